"""GPU parity of the exact CSP optimum: sim_optimum (parallel relaxation over the dense
state space) vs oracle_optimum (Dijkstra over explicit states), on the same tiny workloads and cost models.
The optimum is compared at 0 ULP, the reachable-state count exactly; on instances too large for the oracle the
GPU optimum must still bound every simulated preset from below."""
import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import presets, simsweep, workloads

pytestmark = pytest.mark.gpu
OCMS = o.load_cost_models()
PCMS = simsweep.load_cost_models()
NAMES = ["llama3-8b_a100_linear", "llama3-8b_h100_theoretical", "llama3-70b_a100x4_theoretical"]


def random_problems(seed, k=40):
    rng = np.random.default_rng(seed)
    out = [([2, 2], [4, 4], 4096, 6), ([3], [4], 2, 6), ([1, 1, 1], [3, 2, 1], 1, 3)]
    while len(out) < k:
        W = int(rng.integers(1, 4))
        I = [int(x) for x in rng.integers(1, 5, W)]
        O = [int(x) for x in rng.integers(1, 4, W)]
        peak = max(i + j - 1 for i, j in zip(I, O))
        out.append((I, O, int(rng.integers(1, sum(I) + 2)), int(rng.integers(peak, 2 * peak + 2))))
    return out


@pytest.mark.parametrize("name", NAMES + ["unit"])
def test_optimum_bit_exact_vs_oracle(name):
    probs = random_problems(7 * len(name))
    pc = simsweep.unit_cost(1.0) if name == "unit" else PCMS[name]
    oc = o.unit_cost(1.0) if name == "unit" else OCMS[name]
    got = simsweep.sim_optimum(probs, pc)
    for (I, O, C, M), (st, rounds, states, opt) in zip(probs, got):
        ost, ostates, oopt = o.optimum(I, O, C, M, oc)
        assert (st, states, opt) == (ost, ostates, oopt), (I, O, C, M)
        assert rounds >= 1


def test_example_A_and_status_codes():
    got = simsweep.sim_optimum([([2, 2], [4, 4], 4096, 6), ([4, 1], [3, 1], 4096, 5), ([64] * 4, [64] * 4, 4096, 10_000)],
                               simsweep.unit_cost(1.0))
    assert got[0][0] == "ok" and got[0][3] == 6.0  # preemption is optimal: 6 batches, 8 preemption-free
    assert got[1][0] == "unreachable" and got[2][0] == "too_large"


def test_paper_csp_shape_lower_bounds_every_preset():
    # O = W = 4, M = max(2I, I + O - 1), here for small I (exact search); every simulated preset
    # (NRF, SRF, PF) must be >= the optimum, and some preset reaches it or comes within its schedule's choices
    cm = PCMS["llama3-8b_a100_theoretical"]
    probs, cases = [], []
    for I in (1, 2, 4):
        M = max(2 * I, I + 3)
        probs.append(([I] * 4, [4] * 4, 4096, M))
    opts = simsweep.sim_optimum(probs, cm)
    names = [n + p for n in presets.GRID_PRESETS for p in ("", "-srf", "-pf")]
    for (I, O, C, M), (st, _, states, opt) in zip(probs, opts):
        assert st == "ok" and states > 1000
        wl = workloads.fixed(I[0], O[0], 4)
        cfgs = [simsweep.preset_config(nm, M) for nm in names]
        g = simsweep.sim_sweep(cfgs, [wl], [cm])
        ms = [float(g.results["makespan"][i][0]) for i in range(len(cfgs)) if g.status(i) == "ok"]
        assert ms and min(ms) >= opt


@pytest.mark.parametrize("name", ["llama3-8b_a100_theoretical", "unit"])
def test_preemption_free_optimum_bit_exact(name):
    probs = random_problems(101 + len(name), k=30)
    pc = simsweep.unit_cost(1.0) if name == "unit" else PCMS[name]
    oc = o.unit_cost(1.0) if name == "unit" else OCMS[name]
    got = simsweep.sim_optimum(probs, pc, no_preempt=True)
    for (I, O, C, M), (st, _, states, opt) in zip(probs, got):
        assert (st, states, opt) == o.optimum(I, O, C, M, oc, no_preempt=True), (I, O, C, M)


def test_identical_requests_merged_on_the_gpu():
    # four identical requests: one multiset per state (oracle pins: tests/test_oracle_optimum.py)
    U = simsweep.unit_cost(1.0)
    got = simsweep.sim_optimum([([1, 1], [1, 1], 4096, 10), ([2, 2], [1, 1], 4096, 10), ([3] * 4, [4] * 4, 4096, 8)], U)
    assert [(g[0], g[2], g[3]) for g in got[:2]] == [("ok", 3, 1.0), ("ok", 6, 1.0)]
    assert got[2][:1] == ("ok",) and (got[2][2], got[2][3]) == o.optimum([3] * 4, [4] * 4, 4096, 8, o.unit_cost(1.0))[1:]


def test_paper_csp_shape_preemption_free():
    """PAPER.md:454-467 (O = W = 4, M = max(2I, I + O - 1), A100 8B theoretical): the exact optimum and the optimum
    over preemption-free schedules (identical requests merged: I = 16 has at most 1.4e6 canonical states against 3.0e7
    ordered ones).  The optimum never exceeds the preemption-free one nor any simulated preset."""
    cm = PCMS["llama3-8b_a100_theoretical"]
    for I in (4, 8, 16):
        M = max(2 * I, I + 3)
        (st, _, states, opt), = simsweep.sim_optimum([([I] * 4, [4] * 4, 4096, M)], cm)
        (st2, _, _, free), = simsweep.sim_optimum([([I] * 4, [4] * 4, 4096, M)], cm, no_preempt=True)
        assert st == st2 == "ok" and opt <= free
        g = simsweep.sim_sweep([simsweep.preset_config(n + p, M) for n in presets.GRID_PRESETS for p in ("", "-srf", "-pf")],
                               [workloads.fixed(I, 4, 4)], [cm])
        assert min(float(g.results["makespan"][i][0]) for i in range(len(g.results)) if g.status(i) == "ok") >= opt
