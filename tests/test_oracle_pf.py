"""Oracle pins for the preemption-free schedulers: ``*^pf``
(reserve I + O - 1 at admission, Table 2) and Orca (reserve
S, decode-first, hybrid, no chunking; Table 2).

Pinned against hand traces, the log verifier (tests/verifier.py, which
re-derives holdings from the reserve rule alone), a reduction to the base
scheduler when the reserve never binds, and the paper's Sec. 4.2 / 4.3
findings as directional bounds.
"""
import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import presets, workloads
from verifier import verify

A100 = "llama3-8b_a100_linear"


def pcfg(name, M, S=4096, **kw):
    p = presets.preset(name, S=S)
    return o.make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=kw.pop("C", p["C"]), M=M, S=S,
                         reserve=p["reserve"], **kw)


def run_fixed(name, I, O, W, M, cm=None):
    wl = workloads.fixed(I, O, W)
    return o.run(pcfg(name, M), wl.I, wl.O, wl.T, cm or o.load_cost_models()[A100])


def test_preset_table():
    assert presets.preset("vllm-pf")["reserve"] == presets.RESERVE_PEAK
    assert presets.preset("vllm-pf")["replacement"] == presets.REPL_PF
    p = presets.preset("orca")
    assert (p["order"], p["hybrid"], p["chunked"], p["reserve"], p["replacement"], p["C"]) == (
        presets.ORDER_DECODE_FIRST, 1, 0, presets.RESERVE_CONTEXT, presets.REPL_PF, 4096)
    with pytest.raises(KeyError):
        presets.preset("orca-srf")


def test_config_validation():
    wl = workloads.fixed(2, 2, 2)
    for repl, res in [("pf", "seq"), ("nrf", "peak"), ("srf", "context")]:
        with pytest.raises(ValueError):
            o.run(o.make_config("prefill_first", 0, 0, repl, C=64, M=64, reserve=res), wl.I, wl.O, wl.T, o.unit_cost())


def test_context_reserve_never_fits():
    """Q35 extended: an Orca reserve S > M can never be admitted -> never_fits, not a deadlock."""
    r = o.run(pcfg("orca", 100, S=128), [2], [2], [0.0], o.unit_cost())
    assert r.status == "never_fits"
    assert o.run(pcfg("orca", 128, S=128), [2], [2], [0.0], o.unit_cost()).status == "ok"


def test_example_a_pf_hand_trace():
    """Example A (two requests I=2, O=4, M=6) under vLLM^pf: each reserves I+O-1 = 5, so only one runs at a
    time: r0 prefill + 3 decodes, then r1 -- 8 steps, no preemption (the non-PF schedule preempts)."""
    cfg = pcfg("vllm-pf", 6)
    r = o.run(cfg, [2, 2], [4, 4], [0.0, 0.0], o.unit_cost(1.0), trace=True)
    assert r.status == "ok" and r.steps == 8 and r.preemptions == 0
    assert list(r.t_first[0]) == [1.0, 5.0] and list(r.t_done[0]) == [4.0, 8.0]
    assert [s["U"] for s in r.steps_list] == [5] * 8
    base = o.run(pcfg("vllm", 6), [2, 2], [4, 4], [0.0, 0.0], o.unit_cost(1.0))
    assert base.preemptions > 0


def test_orca_hand_trace():
    """Orca, S = 10, M = 20, three requests I=2, O=3: each reserves S = 10, so two run concurrently and the
    third waits for a release: steps {p0,p1}, {d0,d1}, {d0,d1} -> done; {p2}, {d2}, {d2}."""
    cfg = pcfg("orca", 20, S=10)
    r = o.run(cfg, [2, 2, 2], [3, 3, 3], [0.0] * 3, o.unit_cost(1.0), trace=True)
    assert r.status == "ok" and r.steps == 6 and r.preemptions == 0
    assert list(r.t_done[0]) == [3.0, 3.0, 6.0] and list(r.t_first[0]) == [1.0, 1.0, 4.0]
    assert [len(s["entries"]) for s in r.steps_list] == [2, 2, 2, 1, 1, 1]
    assert [s["U"] for s in r.steps_list] == [20, 20, 20, 10, 10, 10]


@pytest.mark.parametrize("seed", range(120))
def test_random_pf_configs_verify(seed):
    """Random workloads under *^pf / Orca reserves: every step satisfies Eq. (4)-(7) with holdings
    max(reserve, m + c) (re-derived by the verifier), no preemption ever, conservation without refills."""
    rng = np.random.default_rng(70_000 + seed)
    W = int(rng.integers(1, 25))
    S = 64
    wl = workloads.random_small(70_000 + seed, W, max_len=int(rng.integers(2, 17)), online=bool(rng.integers(0, 2)),
                                S=S)
    order = ["prefill_first", "decode_first", "rank_org", "rank_i", "rank_o"][int(rng.integers(0, 5))]
    reserve = ["peak", "context"][int(rng.integers(0, 2))]
    chunked = int(rng.integers(0, 2))
    hybrid = int(rng.integers(0, 2)) if order in ("prefill_first", "decode_first") else 1
    peak = int((wl.I.astype(int) + wl.O - 1).max())
    C = int(rng.integers(1, 3 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
    lo = peak if reserve == "peak" else S
    M = -1 if rng.random() < 0.1 else int(rng.integers(lo, 4 * lo + 1))
    cfg = o.make_config(order, hybrid, chunked, "pf", C=C, M=M, S=S, reserve=reserve)
    r = o.run(cfg, wl.I, wl.O, wl.T, o.load_cost_models()["llama3-8b_a100_theoretical"], trace=True)
    assert r.status == "ok"
    outs = dict(t_first=list(r.t_first[0]), t_done=list(r.t_done[0]), n_preempt=list(r.n_preempt),
                refill=list(r.refill))
    viol = verify(r.steps_list, list(wl.I), list(wl.O), list(wl.T), C, M, outs, hybrid=bool(hybrid), reserve=reserve,
                  S=S)
    assert viol == []
    assert r.preemptions == 0 and int(r.refill.sum()) == 0
    assert r.processed_tokens == int((wl.I.astype(int) + wl.O - 1).sum())


def test_verifier_catches_wrong_reserve():
    """The verifier really checks the reserve: the vLLM^pf trace of Example A read with reserve s fails."""
    r = o.run(pcfg("vllm-pf", 6), [2, 2], [4, 4], [0.0, 0.0], o.unit_cost(1.0), trace=True)
    assert verify(r.steps_list, [2, 2], [4, 4], [0.0, 0.0], 4096, 6, reserve="peak") == []
    assert any("reported U" in v for v in verify(r.steps_list, [2, 2], [4, 4], [0.0, 0.0], 4096, 6, reserve="seq"))


@pytest.mark.parametrize("base", ["vllm", "sarathi", "sarathi-cs", "sarathi-nocp", "vllm-hy", "sarathi-nohy"])
def test_pf_reduces_to_base_without_contention(base):
    """When M >= sum_i (I_i + O_i - 1) no reserve ever binds: *^pf visits in the same (admission) order as
    NRF and admits the same candidates, so its schedule equals the base scheduler's (which never preempts)."""
    wl = workloads.mix(("LILO", "SISO"), 48, 5)
    M = int((wl.I.astype(int) + wl.O - 1).sum())
    cm = o.load_cost_models()[A100]
    a = o.run(pcfg(base, M), wl.I, wl.O, wl.T, cm)
    b = o.run(pcfg(base + "-pf", M), wl.I, wl.O, wl.T, cm)
    assert a.preemptions == 0 and b.preemptions == 0
    assert a.steps == b.steps and a.batch_entries == b.batch_entries
    assert np.array_equal(a.t_done, b.t_done) and np.array_equal(a.t_first, b.t_first)


def test_orca_concurrency_bounded_by_M_over_S():
    """Orca reserves S per request: at most floor(M / S) requests run at once, whatever I, O."""
    wl = workloads.fixed(8, 16, 64)
    r = o.run(pcfg("orca", 1000, S=128), wl.I, wl.O, wl.T, o.unit_cost(1.0), trace=True)
    for st in r.steps_list:
        assert st["U"] % 128 == 0 and st["U"] <= 1000
        assert len(st["entries"]) <= 1000 // 128
    assert r.batch_entries / r.steps == pytest.approx(1000 // 128, rel=0.15)


@pytest.mark.parametrize("I", [1, 1024])
def test_pf_effective_batch_size(I):
    """PF schedulers' average batch size is close to M/(I+O): ~98 for I=1 and ~49 for
    I=1024 at O = W = 1024, M = 100K.  Bound: within 10%."""
    for name in ("vllm-pf", "sarathi-pf", "sarathi-cs-pf"):
        r = run_fixed(name, I, 1024, 1024, 100_000)
        assert r.preemptions == 0
        assert r.batch_entries / r.steps == pytest.approx(100_000 / (I + 1024), rel=0.10)


def test_pf_tradeoff_at_high_contention():
    """PAPER.md:164-167 (O = W = 1024, M = 100K): PF versions have lower latency and TPOT than their
    non-PF versions; TTFT rises -- by orders of magnitude for vLLM and Sarathi_{C=S} ("up to 1000x"), but
    only modestly for Sarathi ("1.7x")."""
    ttft_ratio = {}
    for base in ("vllm", "sarathi", "sarathi-cs"):
        ttft_ratio[base] = 0.0
        for I in (1, 1024):
            a = run_fixed(base, I, 1024, 1024, 100_000)
            b = run_fixed(base + "-pf", I, 1024, 1024, 100_000)
            assert a.preemptions > 0 and b.preemptions == 0
            assert b.mean_latency[0] < a.mean_latency[0]
            assert b.mean_tpot[0] < a.mean_tpot[0]
            ttft_ratio[base] = max(ttft_ratio[base], b.mean_ttft[0] / a.mean_ttft[0])
    assert ttft_ratio["vllm"] > 100 and ttft_ratio["sarathi-cs"] > 100
    assert 1.0 < ttft_ratio["sarathi"] < 10


def test_small_M_reversal():
    """PAPER.md:194-200 (O = 32, W = 1024): under M = 100 preemption *reduces* latency (PF is up to ~2x
    slower: 1.9x vLLM, 2x Sarathi), while at M = 10K avoiding preemption pays."""
    for base in ("vllm", "sarathi"):
        worst = 0.0
        for I in (8, 32):
            a = run_fixed(base, I, 32, 1024, 100)
            b = run_fixed(base + "-pf", I, 32, 1024, 100)
            worst = max(worst, b.mean_latency[0] / a.mean_latency[0])
        assert 1.2 < worst < 3.0
        a = run_fixed(base, 8, 32, 1024, 10_000)
        b = run_fixed(base + "-pf", 8, 32, 1024, 10_000)
        assert b.mean_latency[0] < a.mean_latency[0]
