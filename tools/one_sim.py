"""Launch one grid simulation (or a few) for profiling: python tools/one_sim.py PRESET I O [W] [reps]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_07447_b200 import simsweep, workloads

name, I, O = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
W = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
cm = simsweep.load_cost_models()["llama3-8b_a100_linear"]
ds = simsweep.DeviceSweep([simsweep.preset_config(name, 100_000)], [workloads.fixed(I, O, W)], [cm])
for _ in range(reps):
    ds.launch()
torch.cuda.synchronize()
r = ds.fetch()
print(name, I, O, r.status(0), int(r.results["steps"][0]))
