"""Alone-times of the critical simulations (grid top cells, the full sweep's AzureConv 70B runs), one CTA each, CUDA
events, best of 3.  Compare builds with SIMSWEEP_LIB=path python tools/crit_times.py.  Prints one line per
simulation and the max."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_07447_b200 import simsweep, sweep, workloads  # noqa: E402

GRID = [("vllm-srf", 256, 1024), ("vllm", 256, 1024), ("sarathi-srf", 1024, 1024), ("sarathi-srf", 256, 1024),
        ("vllm-srf", 128, 1024), ("vllm-srf", 64, 1024), ("sarathi-srf", 512, 1024), ("sarathi-srf", 2, 1024),
        ("sarathi", 1024, 1024), ("vllm-srf", 1024, 1024)]
FULL = ["online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9",
        "online-70B vllm llama3-70b_a100x4_theoretical M=100000 azureconv s4"]
cm = simsweep.load_cost_models()["llama3-8b_a100_linear"]
s = torch.cuda.Stream()


def t(ds):
    best = 1e30
    ds.launch(s)
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ds.launch(s)
        e1.record(s)
        s.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


worst = 0.0
for name, I, O in GRID:
    ms = t(simsweep.DeviceSweep([simsweep.preset_config(name, 100_000)], [workloads.fixed(I, O, 1024)], [cm]))
    worst = max(worst, ms)
    print(f"{name:14s} {I:5d} {O:5d} {ms:8.2f} ms", flush=True)
if "--grid" not in sys.argv:
    cfgs, wls, cms, labels = sweep.full_sweep()
    for f in FULL:
        i = next(k for k, lb in enumerate(labels) if f in " ".join(map(str, lb)))
        ms = t(simsweep.DeviceSweep([simsweep.SimConfig.from_buffer_copy(cfgs[i])], wls, cms))
        print(f"{f:70s} {ms:8.2f} ms", flush=True)
print(f"grid max {worst:.2f} ms  [{os.environ.get('SIMSWEEP_LIB', 'default lib')}]")
