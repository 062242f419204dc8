"""Mixed co-residency: 148 copies of A and 148 of B in one launch, interleaved so that each SM holds one of
each, vs. A alone and B alone (I-cache contention test)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2411_07447_b200 import simsweep, workloads
cm = [simsweep.load_cost_models()["llama3-8b_a100_linear"]]
A = ("sarathi-srf", 1024, 1024)
B = ("vllm", 1, 1024)
wls = [workloads.fixed(A[1], A[2], 1024), workloads.fixed(B[1], B[2], 1024)]
def run(cfgs, order=None):
    ds = simsweep.DeviceSweep(cfgs, wls, cm, order=order)
    ds.launch(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.launch(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
ca = [simsweep.preset_config(A[0], 100_000, workload=0) for _ in range(148)]
cb = [simsweep.preset_config(B[0], 100_000, workload=1) for _ in range(148)]
print("A x148 alone", run(ca))
print("B x148 alone", run(cb))
print("A+B blocks [A*148, B*148]", run(ca + cb))
inter = [c for pair in zip(ca, cb) for c in pair]
print("A,B interleaved", run(inter))
print("A x296", run(ca + ca))
