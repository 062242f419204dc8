"""Oracle pins: cost-model analytics (oracle/analytics.py).

Expected values are the paper's own arithmetic (Eq. (9)), closed forms of the linear model
solved here by hand (not by the oracle's code path), the plain scan definition of the SLO frontier, and the
directions the paper states.
"""
import math

import pytest

import oracle as o
from oracle import analytics as an

CMS = o.load_cost_models()
PCIE5_X16 = 64e9  # bytes/s: the host link of the swap alternative (Q42)


def test_eq9_paper_arithmetic():
    # t^N_recom / N in [3.3e-6, 1.3e-3] s with M = 100K -> break-even interval in [0.33, 130] s.
    # A unit cost model charges d per batch whatever it holds, so recompute(N) = d and t/N = d/N.
    _, _, lo = an.kv_break_even(o.unit_cost(3.3e-3), 1000, 1.0, 100_000)  # 3.3e-3 / 1000 = 3.3e-6 s per KV
    _, _, hi = an.kv_break_even(o.unit_cost(1.3e-3), 1, 1.0, 100_000)  # 1.3e-3 s per KV
    assert math.isclose(lo, 0.33, rel_tol=1e-12) and math.isclose(hi, 130.0, rel_tol=1e-12)


def test_kv_bytes_and_swap_time():
    # Llama-2-7B: 2 (K, V) x 32 layers x 32 KV heads x 128 x 2 B = 524 288 B per token (PAPER.md:302 dims)
    cm = CMS["llama2-7b_h100_theoretical"]
    assert an.kv_bytes_per_token(cm) == 524_288
    _, swap, _ = an.kv_break_even(cm, 100, PCIE5_X16, 100_000)
    assert swap == 100 * 524_288 / 64e9


def _linear_frontier(cm, n_p, c, n_d, m_max, tau):
    """t(m) = L (A + B m) for the linear model, solved for the largest m with t <= tau (hand algebra)."""
    a0, a1, b0, b1, b2, b3, b4, d0, d1, d2 = list(cm.lin)
    A = a0 + a1 * (n_p * c + n_d)
    B = 0.0
    if n_p:
        A += b0 + b1 * n_p * c * c + b3 * n_p * c
        B += b2 * n_p * c + b4 * n_p
    if n_d:
        A += d0 + d2 * n_d
        B += d1 * n_d
    L = cm.layers
    if L * A > tau:
        return -1
    if B == 0:
        return m_max
    return min(m_max, int(math.floor((tau / L - A) / B)))


@pytest.mark.parametrize("name", ["llama3-8b_a100_linear", "llama3-8b_h100_linear", "llama3-70b_h100x4_linear",
                                  "llama2-7b_a100_linear"])
@pytest.mark.parametrize("shape", [(8, 128, 8), (32, 512, 32), (128, 64, 128), (0, 1, 64), (16, 2048, 0)])
def test_slo_frontier_linear_closed_form(name, shape):
    cm = CMS[name]
    n_p, c, n_d = shape
    m_max = 1 << 20
    m = an.slo_frontier(cm, n_p, c, n_d, m_max, 1.0)  # the paper's 1 s TPOT threshold
    ref = _linear_frontier(cm, n_p, c, n_d, m_max, 1.0)
    assert abs(m - ref) <= 1  # a boundary within one rounding of the closed form
    if m >= 0:  # ... and exactly the definition at the boundary
        assert an.shape_time(cm, n_p, c, m, n_d, m) <= 1.0
        assert m == m_max or an.shape_time(cm, n_p, c, m + 1, n_d, m + 1) > 1.0


@pytest.mark.parametrize("name", ["llama3-8b_a100_theoretical", "llama3-70b_a100x4_theoretical", "llama3-8b_h100_linear"])
def test_slo_bisection_equals_scan(name):
    cm = CMS[name]
    base = an.shape_time(cm, 4, 256, 0, 4, 0)
    for tau in (0.5 * base, base, 1.02 * base, 1.1 * base, 3 * base):
        for m_max in (0, 1, 37, 300):
            assert an.slo_frontier(cm, 4, 256, 4, m_max, tau) == an.slo_frontier_scan(cm, 4, 256, 4, m_max, tau)


def test_batch_time_monotone_in_every_shape_variable():
    # the bisection needs d non-decreasing in m; the cost models are monotone in every feature
    for name, cm in CMS.items():
        for (n_p, c, n_d) in [(1, 1, 0), (8, 128, 8), (0, 1, 32), (64, 512, 0)]:
            ts = [an.shape_time(cm, n_p, c, m, n_d, m) for m in (0, 1, 10, 100, 1000, 10_000, 100_000)]
            assert all(a <= b for a, b in zip(ts, ts[1:])), name
        assert an.shape_time(cm, 1, 100, 0, 0, 0) <= an.shape_time(cm, 1, 101, 0, 0, 0) <= \
            an.shape_time(cm, 2, 101, 0, 0, 0) <= an.shape_time(cm, 2, 101, 0, 1, 0), name


@pytest.mark.parametrize("name", sorted(CMS))
def test_swap_wins_for_few_kvs(name):
    # for few KVs swapping beats recomputing, "since (1) suffers from a fixed cost of loading model
    # weights": the refill of 1 KV costs at least one weight load
    cm = CMS[name]
    rec1, swap1, _ = an.kv_break_even(cm, 1, PCIE5_X16, 100_000)
    assert swap1 < rec1 / 100


def test_recompute_wins_for_many_kvs_on_a_slow_link():
    # recomputing beats swapping for many KVs.  Under the paper's own Eq. (2) (quadratic
    # attention traffic) this needs a slow host link: with PCIe 3.0 x16 (16 GB/s) and Llama-2-7B (MHA, 512 KB
    # of K and V per token) recomputing 4096 KVs is cheaper, with PCIe 5.0 it is not (Q42)
    cm = CMS["llama2-7b_h100_theoretical"]
    rec, swap16, _ = an.kv_break_even(cm, 4096, 16e9, 100_000)
    _, swap64, _ = an.kv_break_even(cm, 4096, PCIE5_X16, 100_000)
    assert rec < swap16 and swap64 < rec


def test_break_even_interval_decreases_with_N():
    # "the KVs of longer requests have smaller break-even intervals" (weight-load-bound range)
    cm = CMS["llama3-8b_h100_theoretical"]
    iv = [an.kv_break_even(cm, N, PCIE5_X16, 100_000)[2] for N in (1, 2, 4, 8, 16, 32, 64, 128, 256)]
    assert all(a > b for a, b in zip(iv, iv[1:]))


# ---------------------------------------------------------------- per-operator roofline classification
# "What Makes a Batch Compute-Bound?", Eq. (3) per operator.

def _tiny_cost(flops=1.0, bw=1.0):
    c = o.OracleCost()
    c.mode, c.layers, c.h, c.f, c.H, c.NQ, c.NKV, c.e, c.tp = 1, 1, 2, 3, 1, 2, 1, 2, 1
    c.flops, c.bw, c.link_bw = flops, bw, 1.0
    return c


def test_operator_costs_tiny_hand_sums():
    # tiny dims h=2, f=3, H=1, N_Q=2, N_KV=1, e=2 B, FLOPS = BW = 1; one prefill (c=2, m=0), N = 2 (the hand sums
    # of test_oracle_cost.py::test_theoretical_hand_sum_prefill):
    #  QKV  F 32, RW 20 el = 40 B -> time 40, intensity 1.6, memory-bound (32 < 40)
    #  O    F 16, RW 12 el -> 24, 4/3        G+U F 48, RW 28 el -> 56, 12/7     Down F 24, RW 16 el -> 32, 1.5
    #  prefill attn F 32, RW 32 el -> 64, 1.0; no decode entry -> absent
    ops = an.operator_costs(_tiny_cost(), 1, 2, 0, 0, 0)
    assert [(x["op"], x["flops"], x["rw"], x["time"], x["bound"]) for x in ops] == [
        ("qkv", 32, 20, 40.0, 0), ("o", 16, 12, 24.0, 0), ("gate_up", 48, 28, 56.0, 0), ("down", 24, 16, 32.0, 0),
        ("attn_prefill", 32, 32, 64.0, 0), ("attn_decode", 0, 0, 0.0, -1)]
    assert [x["intensity"] for x in ops[:5]] == [32 / 20, 16 / 12, 48 / 28, 24 / 16, 1.0]
    # the same batch on a GPU with 100x the bandwidth: every operator now takes FLOPs / FLOPS -> compute-bound
    fast = an.operator_costs(_tiny_cost(bw=100.0), 1, 2, 0, 0, 0)
    assert [(x["time"], x["bound"]) for x in fast[:5]] == [(32.0, 1), (16.0, 1), (48.0, 1), (24.0, 1), (32.0, 1)]
    # one decode (c = 1, m = 3), N = 1: attention F = 4*1*4*1*2 = 32, RW = 2*1*1*2 + 2*1*4*2 + 2*1*4*1*1 = 28
    dec = an.operator_costs(_tiny_cost(), 0, 1, 0, 1, 3)
    assert dec[4]["bound"] == -1 and (dec[5]["flops"], dec[5]["rw"], dec[5]["time"]) == (32, 28, 56.0)


def test_attention_intensity_limits_paper():
    # as c, m and B grow the attention intensity converges to 2 / (1/H + ceil(c/H) N_KV / (c N_Q));
    # Llama-2-7B (H = 128, N_Q = N_KV = 32): 128 for large-c prefills, 2 / (1/128 + 1) ~ 1.98 for decodes.
    cm = CMS["llama2-7b_a100_theoretical"]
    assert (cm.H, cm.NQ, cm.NKV) == (128, 32, 32)
    pre = an.operator_costs(cm, 256, 4096, 10_000_000, 0, 0)[4]["intensity"]
    dec = an.operator_costs(cm, 0, 1, 0, 256, 10_000_000)[5]["intensity"]
    assert abs(pre - 128.0) / 128.0 < 1e-4
    assert abs(dec - 2.0 / (1.0 / 128.0 + 1.0)) < 1e-4 and abs(dec - 2.0) < 0.02


def test_remark_attention_memory_bound_matmuls_can_be_compute_bound():
    # Remark: "Attentions are memory-bound. Only matmuls can be compute-bound, when c is large
    # enough to surpass the cost of loading fixed-size model weights."  On every A100 / H100 model of the paper.
    names = [k for k in CMS if k.endswith("theoretical")]
    shapes = [(1, 1, 0, 0, 0), (8, 4096, 0, 0, 0), (64, 4096, 100_000, 0, 0), (0, 1, 0, 256, 4096),
              (1, 512, 1000, 1024, 100_000), (128, 2048, 2048, 128, 2048)]
    for nm in names:
        for s in shapes:
            ops = an.operator_costs(CMS[nm], *s)
            assert all(x["bound"] in (0, -1) for x in ops[4:]), (nm, s)  # attention: memory-bound (or absent)
        small = an.operator_costs(CMS[nm], 1, 1, 0, 0, 0)
        big = an.operator_costs(CMS[nm], 8, 4096, 0, 0, 0)  # N = 32768 tokens
        assert all(x["bound"] == 0 for x in small[:4]), nm   # c = 1: weight loading dominates
        assert all(x["bound"] == 1 for x in big[:4]), nm     # large c: FLOPs dominate


def test_operator_times_sum_to_the_batch_time():
    # Eq. (3) summed over the operators in batch_time's order, times the layers, IS the theoretical batch time
    # (tp = 1: no All_Reduce term) -- bit for bit, the same additions in the same order (Q36)
    for nm in [k for k in CMS if k.endswith("theoretical") and CMS[k].tp == 1]:
        for s in [(1, 1, 0, 0, 0), (3, 129, 5, 7, 4000), (0, 1, 0, 64, 100_000), (128, 4096, 0, 0, 0)]:
            t = 0.0
            for x in an.operator_costs(CMS[nm], *s):
                if x["bound"] >= 0:
                    t = t + x["time"]
            assert float(CMS[nm].layers) * t == an.shape_time(CMS[nm], *s), (nm, s)
