"""Per-step GPU summary (profiling build, config 0) vs the oracle trace for one random knob case of the tests.
    python tools/stepdiff_case.py SEED [COST_NAME]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2411_07447_b200 import build
os.environ["SIMSWEEP_LIB"] = build.LIB.replace(".so", "_prof.so")
import numpy as np, torch
import oracle as o
from paper_2411_07447_b200 import simsweep
from tests_util_knobs import random_knob_case
seed = int(sys.argv[1])
cname = sys.argv[2] if len(sys.argv) > 2 else ("llama3-8b_a100_linear" if seed % 2 else "llama3-70b_h100x4_theoretical")
wl, oc, _, knobs = random_knob_case(seed)
cfg = simsweep.make_config(oc.order, oc.hybrid, oc.chunked, oc.replacement, C=oc.C, M=oc.M, S=oc.S, **knobs)
L = simsweep.lib()
L.sim_debug_steps.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ds = simsweep.DeviceSweep([cfg], [wl], [simsweep.load_cost_models()[cname]])
ds.launch(); torch.cuda.synchronize()
g = ds.fetch()
steps = int(g.results["steps"][0])
dbg = np.zeros((65536, 6), np.int32)
L.sim_debug_steps(dbg.ctypes.data, 65536)
r = o.run(oc, wl.I, wl.O, wl.T, o.load_cost_models()[cname], trace=True, trace_cap=1 << 24)
print("case", seed, knobs, "order", oc.order, "hybrid", oc.hybrid, "chunked", oc.chunked, "repl", oc.replacement,
      "C", oc.C, "M", oc.M, "| gpu steps", steps, g.status(0), "oracle steps", r.steps, r.status)
pre, j = 0, 0
for st in r.steps_list:
    pre += len(st["events"])
    exp = (st["step"], st["tok"], st["U"], len(st["entries"]), pre)
    d = tuple(int(x) for x in dbg[j][:5])
    if d != exp:
        print("first divergence at step", st["step"], "gpu (step,tok,U,nB,pre)", d, "oracle", exp)
        for back in range(max(0, j - 3), j + 2):
            s2 = r.steps_list[back]
            print("  oracle step", s2["step"], "tok", s2["tok"], "U", s2["U"], "n", len(s2["entries"]),
                  "events", s2["events"][:6], "entries", s2["entries"][:8])
            print("  gpu   ", dbg[back])
        break
    j += 1
    if j >= steps:
        break
else:
    print("no divergence in", j, "steps")
