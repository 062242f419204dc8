"""A small sweep that launches EVERY kernel instance once (compute-sanitizer racecheck / synccheck / memcheck
target): block kernel CAP 1024 / 4096 / 32768-arena, with and without knobs; lean kernel CAP 1024 / 4096 / arena;
a schedule trace.  Results are checked against the oracle so a sanitizer run is also a parity run.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from paper_2411_07447_b200 import presets, simsweep, workloads  # noqa: E402
from parity import compare, run_case_list  # noqa: E402

A100 = ["llama3-8b_a100_linear"]


def small(seed, n, online=False):
    return workloads.random_small(seed, n, max_len=6, online=online, S=64)


cases = []
for n in (40, 1500, 4200):  # CAP 1024 / 4096 / arena
    for nm, kw in (("vllm-srf", {}), ("sarathi", {}), ("vllm", {"knobs": simsweep.KNOB_HOL, "max_seqs": 8}),
                   ("rank-i", {}), ("sarathi-srf-hist", {}), ("vllm-pf", {})):
        cases.append((simsweep.preset_config(nm, 60, S=64, **kw), small(n, n, online=n > 1000), A100))
# the Eq. (3) roofline models (the lean kernel's per-lane term table, cdiv) and K = 4 mixed models
THEO = ["llama3-70b_a100x4_theoretical"]
K4 = ["llama3-8b_a100_linear", "llama3-8b_h100_theoretical", "llama3-70b_a100x4_linear", "llama3-70b_h100x4_theoretical"]
for n in (40, 1500, 4200):
    cases.append((simsweep.preset_config("vllm-srf", 60, S=64), small(n + 1, n, online=n > 1000), THEO))
    cases.append((simsweep.preset_config("sarathi", 60, S=64), small(n + 2, n, online=n > 1000), THEO))
cases.append((simsweep.preset_config("sarathi-srf", 60, S=64), small(7, 40), K4))
g, ors = run_case_list(cases)
bad = []
for i in range(len(cases)):
    bad += compare(g, ors, i, label=f"case{i}")
print("variants covered:", len(cases), "mismatches:", len(bad))
for b in bad[:10]:
    print(b)
c = simsweep.preset_config("vllm", 12)
_, log = simsweep.sim_run_traced(c, [workloads.fixed(2, 4, 3)], [simsweep.load_cost_models()[A100[0]]])
print("trace steps:", len(log.steps))
sys.exit(1 if bad else 0)
