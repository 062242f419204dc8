"""Oracle pins: the exact CSP optimum (oracle_optimum).

Pinned by closed forms worked out here, Example A by hand (preemption helps), invariants of
the definition (more C or M never hurts; request order does not matter) and the bound it must be: every
schedule the simulator produces satisfies Eq. (4)-(7), so no preset may beat the optimum."""
import math

import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import presets, workloads

UNIT = o.unit_cost(1.0)  # every batch costs 1: the optimum counts batches
CMS = o.load_cost_models()


@pytest.mark.parametrize("I,O,C", [(1, 1, 1), (3, 4, 4096), (5, 2, 2), (7, 3, 3), (4, 1, 1)])
def test_single_request_closed_form(I, O, C):
    # one request: the prefill needs ceil(I/C) batches (a chunk of at most C each, Eq. (5)), every other token one
    # batch (Eq. (6)); no preemption-only batch exists (Q43), so the reachable states are the I partial-prefill
    # states of g = 0, the O-1 filled states and done
    st, n, opt = o.optimum([I], [O], C, I + O - 1, UNIT)
    assert st == "ok" and opt == math.ceil(I / C) + O - 1 and n == I + O


@pytest.mark.parametrize("I,O", [([2, 3], [4, 1]), ([1, 1, 1], [3, 2, 1]), ([3, 2, 1], [1, 2, 3])])
def test_no_contention_closed_form(I, O):
    # C >= sum I and M >= sum (I+O-1): every request prefills in batch 1 and decodes together -> max O batches
    st, _, opt = o.optimum(I, O, sum(I), sum(i + j - 1 for i, j in zip(I, O)), UNIT)
    assert st == "ok" and opt == max(O)


def test_example_A_preemption_is_optimal():
    # SURVEY 8c.9 Example A: r1 = r2 = (I=2, O=4), M = 6.  By hand: both prefill (U=4), both decode (U=6), then one
    # must give up its 3 KVs: r1 decodes twice more (done), r2 refills 4 tokens and decodes once -> 6 batches.  A
    # partial refill alongside r1 does not save a batch (6 + 1 > 6 until r1 is done).  The preemption-free
    # schedule needs 8 (vLLM^pf: "preemption can be optimal").
    st, _, opt = o.optimum([2, 2], [4, 4], 4096, 6, UNIT)
    assert st == "ok" and opt == 6.0
    cfg = o.make_config("prefill_first", 0, 0, "pf", C=4096, M=6, reserve="peak")
    r = o.run(cfg, np.array([2, 2], np.int32), np.array([4, 4], np.int32), np.zeros(2), UNIT)
    assert r.steps == 8


def test_unreachable_when_a_request_never_fits():
    st, _, _ = o.optimum([4, 1], [3, 1], 4096, 5, UNIT)  # 4 + 3 - 1 = 6 > M
    assert st == "unreachable"


def test_order_and_resources():
    cm = CMS["llama3-8b_a100_theoretical"]
    a = o.optimum([3, 1, 2], [2, 3, 1], 4, 6, cm)
    b = o.optimum([2, 3, 1], [1, 2, 3], 4, 6, cm)
    assert a[0] == b[0] == "ok" and a[1] == b[1] and a[2] == b[2]  # the request order does not matter
    for C, M in [(4, 6), (5, 6), (4, 7), (8, 12)]:
        more = o.optimum([3, 1, 2], [2, 3, 1], C + 1, M + 1, cm)
        assert more[2] <= o.optimum([3, 1, 2], [2, 3, 1], C, M, cm)[2]  # more C or M never hurts


ORDERS = ["prefill_first", "decode_first", "rank_org", "rank_i", "rank_o"]


@pytest.mark.parametrize("seed", range(40))
def test_no_preset_beats_the_optimum(seed):
    rng = np.random.default_rng(1000 + seed)
    W = int(rng.integers(1, 4))
    I = rng.integers(1, 4, size=W).astype(np.int32)
    O = rng.integers(1, 4, size=W).astype(np.int32)
    peak = int((I + O - 1).max())
    M = int(rng.integers(peak, 2 * peak + 2))
    C = int(rng.integers(1, int(I.sum()) + 2))
    cm = [UNIT, CMS["llama3-8b_a100_linear"], CMS["llama3-8b_h100_theoretical"]][seed % 3]
    st, _, opt = o.optimum(I, O, C, M, cm)
    assert st == "ok"
    for order in ORDERS:
        for chunked in (0, 1):
            if not chunked and peak > C:
                continue  # a non-chunked preset rejects such a workload (Q35)
            for hybrid in ((0, 1) if order in ("prefill_first", "decode_first") else (1,)):
                for repl, res in (("nrf", "seq"), ("srf", "seq"), ("pf", "peak")):
                    cfg = o.make_config(order, hybrid, chunked, repl, C=C, M=M, reserve=res)
                    r = o.run(cfg, I, O, np.zeros(W), cm)
                    if r.status == "ok":
                        assert opt <= float(r.makespan[0]), (order, chunked, hybrid, repl)


def test_identical_requests_are_merged():
    # identical requests are interchangeable (a permutation of them maps every schedule to one of the same cost),
    # so the search stores a state once per multiset of their local states.  By hand, unit cost, ample C and M:
    #  two (I=1, O=1): {both waiting, one done, both done} = 3 states; one batch serves both.
    #  three (I=1, O=1): 4 states (0..3 done).
    #  two (I=2, O=1): local states {done, m=0, m=1} -> every multiset of size 2 of them is reachable from (0, 0)
    #  by some batch: binom(3 + 1, 2) = 6 states; one batch (c = 2 each) serves both.
    assert o.optimum([1, 1], [1, 1], 4096, 10, UNIT) == ("ok", 3, 1.0)
    assert o.optimum([1, 1, 1], [1, 1, 1], 4096, 10, UNIT) == ("ok", 4, 1.0)
    assert o.optimum([2, 2], [1, 1], 4096, 10, UNIT) == ("ok", 6, 1.0)
    # a mixed instance: the identical pair is merged, the third request is not
    st, n3, _ = o.optimum([2, 2, 1], [1, 1, 1], 4096, 10, UNIT)
    assert st == "ok" and n3 == 6 * 2  # (pair multisets) x (third request: waiting / done)


def test_preemption_free_optimum():
    # Example A without preemption (e = 0 always): r1, r2 = (2, 4), M = 6 -- both cannot run to their peak 5 + 5
    # together, so one finishes first: 4 batches for r1 (prefill + 3 decodes) and 4 for r2 after it, or
    # interleavings that never beat that: 8 ("preemption can be optimal": 6 < 8)
    assert o.optimum([2, 2], [4, 4], 4096, 6, UNIT, no_preempt=True)[2] == 8.0


@pytest.mark.parametrize("seed", range(20))
def test_preemption_free_optimum_bounds(seed):
    # the preemption-free optimum is >= the optimum (fewer schedules) and <= every PF preset (each PF schedule
    # is a preemption-free schedule satisfying Eq. (4)-(7))
    rng = np.random.default_rng(3000 + seed)
    W = int(rng.integers(1, 4))
    I = rng.integers(1, 4, size=W).astype(np.int32)
    O = rng.integers(1, 4, size=W).astype(np.int32)
    peak = int((I + O - 1).max())
    M = int(rng.integers(peak, 2 * peak + 2))
    C = int(rng.integers(1, int(I.sum()) + 2))
    cm = [UNIT, CMS["llama3-8b_a100_linear"]][seed % 2]
    _, _, opt = o.optimum(I, O, C, M, cm)
    st, _, free = o.optimum(I, O, C, M, cm, no_preempt=True)
    assert st == "ok" and opt <= free
    for order in ("prefill_first", "decode_first"):
        for chunked in (0, 1):
            if not chunked and peak > C:
                continue
            cfg = o.make_config(order, 1, chunked, "pf", C=C, M=M, reserve="peak")
            r = o.run(cfg, I, O, np.zeros(W), cm)
            if r.status == "ok":
                assert free <= float(r.makespan[0])
