"""GPU parity of the cost-model analytics: the C-ABI kernels vs oracle/analytics.py,
element by element, on the same shapes and the same frozen cost models.  Batch times, swap times and intervals
are compared at 0 ULP (same expression order, Q36); frontiers are integers (exact)."""
import numpy as np
import pytest

import oracle as o
from oracle import analytics as an
from paper_2411_07447_b200 import simsweep

pytestmark = pytest.mark.gpu
OCMS = o.load_cost_models()
PCMS = simsweep.load_cost_models()
NAMES = sorted(OCMS)


def shapes_grid(seed=0, n=400):
    rng = np.random.default_rng(seed)
    out = [(1, 1, 0, 0, 0), (0, 1, 0, 1, 0), (0, 1, 0, 256, 100_000), (128, 4096, 0, 0, 0), (8, 512, 1000, 8, 4000),
           (1, 1, 130_000, 0, 0), (3, 127, 5, 0, 0), (3, 128, 5, 0, 0), (3, 129, 5, 0, 0)]  # ceil(c/H) edges
    while len(out) < n:
        n_p = int(rng.integers(0, 129))
        n_d = int(rng.integers(0 if n_p else 1, 257))
        out.append((n_p, int(rng.integers(1, 8193)), int(rng.integers(0, 131_073)), n_d, int(rng.integers(0, 131_073))))
    return out


def test_batch_times_bit_exact():
    shapes = shapes_grid()
    g = simsweep.sim_batch_times([PCMS[k] for k in NAMES], shapes)
    for a, name in enumerate(NAMES):
        ref = np.array([an.shape_time(OCMS[name], *s) for s in shapes])
        assert np.array_equal(g[a], ref), (name, np.flatnonzero(g[a] != ref)[:5])


def test_batch_times_match_the_simulators_batches():
    # a simulated batch and its shape get the same d_j: SPEC single request I=2, O=3 under the A100 model --
    # prefill (c=2, m=0) then two decodes (m=2, m=3): t_done = d1 + d2 + d3
    from paper_2411_07447_b200 import workloads
    cm = PCMS["llama3-8b_a100_theoretical"]
    wl = workloads.Workload(np.array([2], np.int32), np.array([3], np.int32), np.zeros(1))
    r = simsweep.sim_sweep([simsweep.preset_config("vllm", 100_000)], [wl], [cm])
    d = simsweep.sim_batch_times([cm], [(1, 2, 0, 0, 0), (0, 1, 0, 1, 2), (0, 1, 0, 1, 3)])[0]
    assert r.request_times(0)[1][0, 0] == (d[0] + d[1]) + d[2]


def slo_queries():
    q = []
    for n_p in (0, 8, 32, 128):  # Fig. SLO: 8 / 32 / 128 prefills and decodes
        for n_d in (0, 8, 32, 128):
            if n_p + n_d == 0:
                continue
            for c in (1, 16, 128, 512, 2048):
                for tau in (0.05, 0.25, 1.0):
                    q.append((n_p, c, n_d, 200_000, tau))
    return q


def test_slo_frontier_exact():
    q = slo_queries()
    g = simsweep.sim_slo_frontier([PCMS[k] for k in NAMES], q)
    for a, name in enumerate(NAMES):
        ref = [an.slo_frontier(OCMS[name], *x) for x in q]
        assert g[a].tolist() == ref, name
    assert (g == -1).any() and (g == 200_000).any() and ((g > 0) & (g < 200_000)).any()  # all three regimes


def test_kv_break_even_bit_exact():
    N = np.array([1, 2, 3, 16, 99, 100, 128, 129, 1000, 4096, 65_536], np.int64)
    rec, swap, itv = simsweep.sim_kv_break_even([PCMS[k] for k in NAMES], N, 64e9, 100_000)
    for a, name in enumerate(NAMES):
        ref = np.array([an.kv_break_even(OCMS[name], int(x), 64e9, 100_000) for x in N])
        assert np.array_equal(rec[a], ref[:, 0]) and np.array_equal(swap[a], ref[:, 1]) and \
            np.array_equal(itv[a], ref[:, 2]), name


def test_invalid_shapes_rejected():
    cm = [PCMS["llama3-8b_a100_linear"]]
    for bad in [(0, 1, 0, 0, 0), (1, 0, 0, 0, 0), (-1, 1, 0, 1, 0), (1, 1, -1, 0, 0), (1 << 40, 1 << 20, 0, 0, 0)]:
        with pytest.raises(simsweep.SimError, match="invalid argument"):
            simsweep.sim_batch_times(cm, [bad])
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_slo_frontier(cm, [(1, 1, 1, 10, 0.0)])
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_kv_break_even(cm, [0], 64e9, 100_000)


def test_operator_costs_exact():
    """sim_operator_costs vs oracle/analytics.operator_costs: FLOPs, RW and boundness exact,
    times and intensities 0 ULP, on the shape grid x all 12 models."""
    shapes = shapes_grid(seed=3, n=300)
    g = simsweep.sim_operator_costs([PCMS[k] for k in NAMES], shapes)
    assert g.shape == (len(NAMES), len(shapes), len(simsweep.OP_NAMES))
    for a, name in enumerate(NAMES):
        for i, s in enumerate(shapes):
            ref = an.operator_costs(OCMS[name], *s)
            for o_, r in enumerate(ref):
                x = g[a, i, o_]
                assert (int(x["flops"]), int(x["rw"]), int(x["bound"])) == (r["flops"], r["rw"], r["bound"]), (name, s, o_)
                assert float(x["time"]) == r["time"] and float(x["intensity"]) == r["intensity"], (name, s, o_)
    # the paper's limits straight from the GPU: 128 / ~1.98 on Llama-2-7B
    cm = PCMS["llama2-7b_a100_theoretical"]
    lim = simsweep.sim_operator_costs([cm], [(256, 4096, 10_000_000, 0, 0), (0, 1, 0, 256, 10_000_000)])[0]
    assert abs(lim[0, 4]["intensity"] - 128.0) < 0.02 and abs(lim[1, 5]["intensity"] - 2 / (1 / 128 + 1)) < 1e-3
