"""Per-region instructions and stall samples per unit of the lean kernel (region = a block of sim_lean.cuh found by
marker comments).   LEAN_SRC=... python tools/lean_regions2.py REP LIB KERNEL_SUBSTR units"""
import collections
import os
import re
import subprocess
import sys

sys.argv += []
here = os.path.dirname(os.path.abspath(__file__))
src_path = os.environ.get("LEAN_SRC") or os.path.join(here, "..", "paper_2411_07447_b200", "csrc", "sim_lean.cuh")
src = open(src_path).read().split("\n")
marks = [("---- (1) a2", "arrivals"), ("if (n_done == n)", "loop-checks"),
         ("auto hist_sum", "hist_sum"), ("auto rnew", "misc-lambdas"), ("auto admit_chunk", "admit_chunk"),
         ("auto run_prefills", "run_prefills"), ("auto kv_pass", "wait_scan"), ("auto nth_head", "nth_head"),
         ("auto decode_group", "decode_group"), ("// apply: evict", "evict_apply"), ("if (pfirst) {  // vLLM", "dispatch"),
         ("if (tok == 0) {", "idle"), ("---- (3) a9", "compensate"), ("// the prefill entries:", "process"),
         ("if (n_pb + n_new > 0)", "feature_reduce"), ("// decode completions:", "completion_scan"),
         ("// the new decodes join", "new_decodes"), ("// a9: lane k", "cost"), ("steps++;", "counters"),
         ("// event times", "events"), ("// this step's victims", "victims"), ("---- (4) steady", "steady"),
         ("if (hist && ndone > 0)", "runlist"), ("if (nmov > 0) {  // SRF", "srf_merge"),
         ("nrun = cnt;", "runlist-end"), ("---- a11", "epilogue")]
starts = []
for i, l in enumerate(src, 1):
    for k, nm in marks:
        if k in l and (not starts or starts[-1][1] != nm):
            starts.append((i, nm))
starts.sort()


def region(ln):
    nm = "prologue"
    for a, n in starts:
        if ln >= a:
            nm = n
    return nm


rep, lib, kname, unit = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
env = dict(os.environ)
out = subprocess.run([sys.executable, os.path.join(here, "lean_lines.py"), rep, lib, kname, "1", "100000"],
                     capture_output=True, text=True, env=env).stdout
E, S = collections.Counter(), collections.Counter()
for l in out.split("\n")[2:]:
    f = l.split()
    if len(f) < 4:
        continue
    try:
        samp, ins, ln = float(f[0]), float(f[1]), f[3]
    except ValueError:
        continue
    r = region(int(ln)) if ln.isdigit() else "?"
    E[r] += ins
    S[r] += samp
te = sum(E.values())
print(f"{'region':18s} {'instr/unit':>10s} {'samples%':>9s}")
for r, v in sorted(E.items(), key=lambda x: -x[1]):
    print(f"{r:18s} {v / unit:10.1f} {S[r]:9.1f}")
print(f"{'total':18s} {te / unit:10.1f}")
