"""Launch one simulation alone (one CTA) for profiling.

    python tools/one_sim.py PRESET I O [W] [reps]        a grid cell
    python tools/one_sim.py --full "SUBSTRING" [reps]    the first full-sweep simulation whose label contains SUBSTRING
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_07447_b200 import simsweep, sweep, workloads  # noqa: E402

if sys.argv[1] == "--full":
    cfgs, wls, cms, labels = sweep.full_sweep()
    i = next(k for k, lb in enumerate(labels) if sys.argv[2] in " ".join(map(str, lb)))
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    ds = simsweep.DeviceSweep([simsweep.SimConfig.from_buffer_copy(cfgs[i])], wls, cms)
    what = " ".join(map(str, labels[i]))
else:
    name, I, O = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    W = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    cm = simsweep.load_cost_models()["llama3-8b_a100_linear"]
    ds = simsweep.DeviceSweep([simsweep.preset_config(name, 100_000)], [workloads.fixed(I, O, W)], [cm])
    what = f"{name} {I} {O} W={W}"
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds.launch()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
r = ds.fetch()
print(what, r.status(0), "steps", int(r.results["steps"][0]), "formed", int(r.results["formed_steps"][0]),
      f"{1e3 * dt:.2f} ms (last launch, wall)")
