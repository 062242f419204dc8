"""Throughput of the cost-model analytics kernels vs the oracle on a sample.
    python tools/analytics_bench.py      (GPU box)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as o  # noqa: E402
from oracle import analytics as an  # noqa: E402
from paper_2411_07447_b200 import simsweep  # noqa: E402

P = simsweep.load_cost_models()
OC = o.load_cost_models()
names = sorted(P)
rng = np.random.default_rng(1)
n = 1 << 20
shapes = np.stack([rng.integers(1, 129, n), rng.integers(1, 8193, n), rng.integers(0, 131_073, n),
                   rng.integers(0, 257, n), rng.integers(0, 131_073, n)], axis=1).astype(np.int64)
simsweep.sim_batch_times([P[k] for k in names], shapes[:1024])  # warm
t0 = time.perf_counter()
g = simsweep.sim_batch_times([P[k] for k in names], shapes)
t1 = time.perf_counter()
gpu_rate = len(names) * n / (t1 - t0)
t2 = time.perf_counter()
ref = [an.shape_time(OC[names[0]], *(int(x) for x in s)) for s in shapes[:2000]]
t3 = time.perf_counter()
assert np.array_equal(g[0][:2000], np.array(ref))
q = [(np_, c, nd, 1 << 20, tau) for np_ in (8, 32, 128) for nd in (8, 32, 128) for c in range(1, 4097, 16)
     for tau in (0.25, 1.0)]
t4 = time.perf_counter()
f = simsweep.sim_slo_frontier([P[k] for k in names], q)
t5 = time.perf_counter()
print(f"batch_times: {len(names)} models x {n} shapes in {1e3 * (t1 - t0):.1f} ms end to end "
      f"({gpu_rate / 1e6:.1f} M evaluations/s); oracle {2000 / (t3 - t2) / 1e3:.1f} k/s on one core")
print(f"slo_frontier: {len(names)} x {len(q)} queries (21-step bisections) in {1e3 * (t5 - t4):.1f} ms")
