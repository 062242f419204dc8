"""Oracle pins: the batch-latency model (Eq. (1)-(3)).

Expected values are the paper's printed examples, closed-form limits, or hand
sums over tiny made-up model dimensions (worked out in the comments).
"""
import numpy as np
import pytest

import oracle as o

CMS = o.load_cost_models()


def test_eq1_spec_example():
    # (c=1, m=0, B=1, H=128, N_Q=32) -> 4*1*1*1*128*32 = 16 384 FLOPs
    F, _ = o.attention_cost(1, 0, 1, 128, 32, 32)
    assert F == 16384


def test_matmul_example():
    # c=2, in=3, out=5 -> 60 FLOPs; RW 15 + 6 + 10 = 31 elements = 62 bytes at 2 B/element
    F, RW = o.matmul_cost(2, 3, 5)
    assert (F, 2 * RW) == (60, 62)
    F, RW = o.matmul_cost(0, 4096, 4096)  # c = 0: weights still loaded
    assert (F, RW) == (0, 4096 * 4096)


def test_attention_intensity_limits():
    # intensity -> 2 / (1/H + ceil(c/H) N_KV / (c N_Q)); Llama-2-7B (H=128, N_Q=N_KV=32):
    # 128 for large-c prefills, 2/(1/128 + 1) ~ 1.98 for decodes.
    F, RW = o.attention_cost(4096, 0, 100_000, 128, 32, 32)
    assert abs(F / RW - 128) / 128 < 0.02
    F, RW = o.attention_cost(1, 100_000, 100_000, 128, 32, 32)
    assert abs(F / RW - 2 / (1 / 128 + 1)) < 1e-3 and abs(F / RW - 2) / 2 < 0.05


def test_eq2_additive_over_identical_requests():
    # Eq. (1) is linear in B exactly; Eq. (2)'s (c+m)B terms are additive, the 2cHN_Q term is per call
    F1, R1 = o.attention_cost(7, 30, 1, 128, 32, 8)
    F5, R5 = o.attention_cost(7, 30, 5, 128, 32, 8)
    assert F5 == 5 * F1
    assert R5 - 2 * 7 * 128 * 32 == 5 * (R1 - 2 * 7 * 128 * 32)


def _tiny(mode, tp=1):
    c = o.OracleCost()
    c.mode, c.layers, c.h, c.f, c.H, c.NQ, c.NKV, c.e, c.tp = mode, 1, 2, 3, 1, 2, 1, 2, tp
    c.flops = c.bw = c.link_bw = 1.0
    return c


def test_theoretical_hand_sum_prefill():
    # tiny dims h=2, f=3, H=1, N_Q=2, N_KV=1, e=2 B, FLOPS = BW = 1; one prefill (c=2, m=0), N = 2:
    #  QKV  in 2 out 4: F 32, RW 8+4+8 = 20 el = 40 B -> 40
    #  O    in 2 out 2: F 16, RW 4+4+4 = 12 el = 24 B -> 24
    #  G+U  in 2 out 6: F 48, RW 12+4+12 = 28 el = 56 B -> 56
    #  Down in 3 out 2: F 24, RW 6+6+4 = 16 el = 32 B -> 32
    #  prefill attn: F 4*2*2*1*2 = 32; RW 2*2*1*2 + 2*2*2*2 + 2*2*2*1*1 = 32 el = 64 B -> 64
    assert o.batch_time(_tiny(1), [(2, 0, True)]) == 40 + 24 + 56 + 32 + 64


def test_theoretical_hand_sum_hybrid_tp():
    # add a decode (c=1, m=5), N = 3:
    #  QKV F 48, RW 8+6+12=26 -> 52 | O F 24, RW 4+6+6=16 -> 32 | G+U F 72, RW 12+6+18=36 -> 72
    #  Down F 36, RW 6+9+6=21 -> 42 | prefill attn 64 | decode attn F 4*1*6*1*2 = 48,
    #  RW 2*1*1*2 + 2*1*6*2 + 2*1*6*1*1 = 40 el = 80 B -> 80            total 342
    ents = [(2, 0, True), (1, 5, False)]
    assert o.batch_time(_tiny(1), ents) == 342
    # tp = 2: two All_Reduce of (2 e N h (tp-1) / tp) / link_bw = (2*2*3*2*1/2)/1 = 12 each -> 366
    assert o.batch_time(_tiny(1, tp=2), ents) == 366


def test_linear_hand_sum():
    # lin = 1..10, 2 layers; prefill (c=3, m=2) + decode (m=4): N = 4
    # t = 1 + 2*4 = 9; prefill 3 + 4*9 + 5*6 + 6*3 + 7*2 = 101; decode 8 + 9*4 + 10*1 = 54 -> 164 * 2
    c = _tiny(0)
    c.layers = 2
    for j in range(10):
        c.lin[j] = float(j + 1)
    assert o.batch_time(c, [(3, 2, True), (1, 4, False)]) == 328
    assert o.batch_time(c, [(1, 4, False)]) == 2 * (1 + 2 * 1 + 8 + 9 * 4 + 10)


def test_linear_spec_stub():
    # t = 0.01 + 0.001 * sum c, sum c = 990 -> 1.0 s
    c = _tiny(0)
    c.lin[0], c.lin[1] = 0.01, 0.001
    assert abs(o.batch_time(c, [(990, 0, True)]) - 1.0) < 1e-12


@pytest.mark.parametrize("name", sorted(CMS))
def test_monotone_in_every_feature(name):
    # "Since the cost models are monotonic": adding tokens or KVs never lowers batch time
    cm = CMS[name]
    rng = np.random.default_rng(0)
    for _ in range(200):
        k = int(rng.integers(1, 6))
        ents = [(int(rng.integers(1, 512)), int(rng.integers(0, 4096)), True) for _ in range(k)]
        ents += [(1, int(rng.integers(0, 4096)), False) for _ in range(int(rng.integers(0, 6)))]
        t0 = o.batch_time(cm, ents)
        assert t0 > 0
        j = int(rng.integers(0, len(ents)))
        c, m, p = ents[j]
        bumped = list(ents)
        bumped[j] = (c + (1 if p else 0), m + 1, p)
        assert o.batch_time(cm, bumped) >= t0
        assert o.batch_time(cm, ents + [(1, 10, False)]) >= t0


def test_hist_predict_pins():
    H = np.zeros((18, 18), np.int32)
    assert o.hist_predict(H, 100) == 256  # empty -> prior
    # SURVEY 8(c.6) pin: bucket bI = 6 (I in [64,128)) holds O = {10 x 9, 500}: n = 10, rank ceil(9) = 9,
    # 9th smallest in bO = 3 ([8,16)) -> upper edge 15
    H[6, 3], H[6, 8] = 9, 1
    assert o.hist_predict(H, 100) == 15
    # row with n = 3 < 8 falls back to the global column sums: col3 = 9, col5 = 3, n = 12,
    # rank ceil(10.8) = 11 -> reached at bO = 5 -> 63
    H[2, 5] = 3
    assert o.hist_predict(H, 5) == 63
    # n = 8 exactly, all in bO = 0 -> 1
    H2 = np.zeros((18, 18), np.int32)
    H2[0, 0] = 8
    assert o.hist_predict(H2, 1) == 1
