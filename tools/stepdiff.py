"""Diff the per-step summary of the GPU (profiling build, config 0) against the oracle trace.
    python tools/stepdiff.py PRESET I O [W] [M]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_07447_b200 import build
os.environ["SIMSWEEP_LIB"] = build.LIB.replace(".so", "_prof.so")
import numpy as np, torch
import oracle as o
from paper_2411_07447_b200 import simsweep, workloads, presets
name, I, O = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
W = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
M = int(sys.argv[5]) if len(sys.argv) > 5 else 100_000
wl = workloads.fixed(I, O, W)
L = simsweep.lib()
L.sim_debug_steps.argtypes = [ctypes.c_void_p, ctypes.c_int32]
cfg = simsweep.preset_config(name, M)
ds = simsweep.DeviceSweep([cfg], [wl], [simsweep.load_cost_models()["llama3-8b_a100_linear"]])
ds.launch(); torch.cuda.synchronize()
g = ds.fetch()
steps = int(g.results["steps"][0])
dbg = np.zeros((65536, 6), np.int32)
L.sim_debug_steps(dbg.ctypes.data, 65536)
p = presets.preset(name)
r = o.run(o.make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=p["C"], M=M, reserve=p["reserve"]), wl.I, wl.O, wl.T,
          o.load_cost_models()["llama3-8b_a100_linear"], trace=True, trace_cap=1 << 28)
print("gpu steps", steps, "oracle steps", r.steps)
pre = 0
j = 0
for st in r.steps_list:
    pre += len(st["events"])
    exp = (st["step"], st["tok"], st["U"], len(st["entries"]), pre)
    d = tuple(int(x) for x in dbg[j][:5])
    if d != exp:
        print("first divergence at step", st["step"], "gpu", d, "oracle", exp)
        for back in range(max(0, j - 3), j + 2):
            s2 = r.steps_list[back]
            print("  oracle step", s2["step"], "tok", s2["tok"], "U", s2["U"], "n", len(s2["entries"]),
                  "events", s2["events"][:6], "entries(head)", s2["entries"][:4], "...", s2["entries"][-3:])
            print("  gpu   ", dbg[back])
        break
    j += 1
    if j >= steps:
        break
else:
    print("no divergence in", j, "steps")
