"""Co-residency experiment: N copies of one simulation in one launch (1 or 2 CTAs per SM)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2411_07447_b200 import simsweep, workloads
name, I, O = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cm = [simsweep.load_cost_models()["llama3-8b_a100_linear"]]
wl = workloads.fixed(I, O, 1024)
for N in (1, 148, 296, 444):
    cfgs = [simsweep.preset_config(name, 100_000) for _ in range(N)]
    ds = simsweep.DeviceSweep(cfgs, [wl], cm)
    ds.launch(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.launch(); e1.record(); torch.cuda.synchronize()
    print(f"{name} {I}/{O} N={N:4d}: {e0.elapsed_time(e1):8.2f} ms")
