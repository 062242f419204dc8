"""Per-simulation timing + phase profile of the step kernel (profiling build).

    python tools/probe.py            (on a GPU box; builds libsimsweep_prof.so first if needed)

Times single simulations (one launch each) with CUDA events and prints
us/step plus the share of thread-0 cycles per phase (arrivals, build P,
admission rounds, features+cost, process, run list), rounds and breaks per step.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_07447_b200 import build  # noqa: E402

PRODUCT = "--product" in sys.argv  # use the product library (no phase counters), e.g. under ncu
if not PRODUCT:
    prof_lib = os.environ.get("PROBE_LIB") or build.LIB.replace(".so", "_prof.so")
    if not os.path.exists(prof_lib) or "--rebuild" in sys.argv:  # noqa
        build.build(profile=True)
    os.environ["SIMSWEEP_LIB"] = prof_lib

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_07447_b200 import simsweep, sweep, workloads  # noqa: E402

L = simsweep.lib()
if not PRODUCT:
    L.sim_debug_read.restype = ctypes.c_int
    L.sim_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_int32]
pcms = simsweep.load_cost_models()
cm = [pcms["llama3-8b_a100_linear"]]
PH = ["arrive", "buildP", "rounds", "feat+cost", "process", "runlist"]

if "--one" in sys.argv:  # a single simulation (for ncu: -k regex:sim_kernel -s 1 -c 1)
    j = sys.argv.index("--one")
    cases = [(sys.argv[j + 1], int(sys.argv[j + 2]), int(sys.argv[j + 3]))]
else:
  cases = [("vllm", 128, 1024), ("vllm", 256, 1024), ("vllm", 1024, 1024), ("vllm-srf", 1024, 1024), ("sarathi", 1024, 1024), ("sarathi-srf", 1024, 1024),
         ("vllm", 1, 1024), ("sarathi", 1, 1024), ("sarathi-nohy", 1024, 1024), ("vllm-hy-srf", 64, 1024),
         ("sarathi-cs", 256, 256), ("vllm", 16, 16), ("sarathi-nocp-srf", 4, 512)]
print(f"{'case':28s} {'steps':>7s} {'ms':>8s} {'us/step':>8s} {'rnd/st':>6s} {'brk/st':>6s} {'sorts':>6s} " +
      " ".join(f"{p:>9s}" for p in PH))
for (nm, I, O) in cases:
    wl = workloads.fixed(I, O, 1024)
    cfgs = [simsweep.preset_config(nm, 100_000)]
    ds = simsweep.DeviceSweep(cfgs, [wl], cm)
    ds.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ds.launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    r = ds.fetch().results[0]
    prof = np.zeros(24, np.int64)
    if not PRODUCT:
        L.sim_debug_read(prof.ctypes.data, 1)
    steps = int(r["steps"])
    tot = prof[[0, 1, 2, 3, 4, 5]].sum() + prof[10]
    tot = prof[[0, 1, 2, 3, 4, 5, 10]].sum()
    share = " ".join(f"{100.0 * prof[i] / max(tot, 1):8.1f}%" for i in range(6))
    share += " | warp-mode/st %.2f closedR/st %.2f chunks/st %.1f wbrk/st %.2f" % tuple(prof[i] / steps for i in (11, 12, 13, 14))
    full = max(int(prof[16]), 1)
    share += f" | full steps {full} ({1000 * ms / full:.2f} us/full step), run steps {int(prof[17])}"
    print(f"{nm + f' {I}/{O}':28s} {steps:7d} {ms:8.2f} {1000 * ms / steps:8.2f} {prof[6] / steps:6.2f} "
          f"{prof[7] / steps:6.2f} {prof[8]:6d} {share}  cyc/step={tot / steps:.0f}")
