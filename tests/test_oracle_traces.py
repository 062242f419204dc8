"""Oracle pins: hand-traced schedules on tiny workloads.

Every expected value below was derived BY HAND from Algorithm 1
(PAPER.md:1512-1563), the GetNextBatch text, Eq. (4)-(6)
 and the DESIGN.md readings -- not by running the oracle.
Batch entries are (request id, phase 1=prefill/0=decode, c, m_before); U is
the KV holding right after admission; events are (victim, m discarded).
A unit-cost stub (every batch costs 1 s) makes times = step counts.
"""
import pytest

import oracle as o

UNIT = o.unit_cost()


def _run(order, hybrid, chunked, repl, C, M, I, O, T=None):
    T = T if T is not None else [0.0] * len(I)
    cfg = o.make_config(order, hybrid, chunked, repl, C=C, M=M)
    return o.run(cfg, I, O, T, UNIT, trace=True)


def _sched(r):
    return [(s["U"], s["entries"], s["events"]) for s in r.steps_list]


def test_spec_single_request():
    # I=2, O=3, unit cost -> prefill, decode, decode; TTFT 1, TPOT (3-1)/2 = 1, makespan 3
    r = _run("prefill_first", 0, 0, "nrf", 4096, 100, [2], [3])
    assert r.status == "ok" and r.steps == 3
    assert r.t_first[0][0] == 1.0 and r.t_done[0][0] == 3.0
    assert r.mean_ttft[0] == 1.0 and r.mean_tpot[0] == 1.0 and r.makespan[0] == 3.0
    assert [e for (_, e, _) in _sched(r)] == [[(0, 1, 2, 0)], [(0, 0, 1, 2)], [(0, 0, 1, 3)]]


@pytest.mark.parametrize("repl", ["nrf", "srf"])
def test_example_A_preemption(repl):
    # vLLM, C=4096, M=6, r1=r2=(I=2,O=4).  Step 3: r1 needs 4 > held 3 -> U would be 7 > 6 ->
    # victim r2 (newest / equal m, later admission) frees 3; step 4: refill of r2 (4 KVs) does not fit
    # (waiting never preempts, Q5); step 5: r2 refills I+g = 4 tokens and regenerates its 3rd token.
    r = _run("prefill_first", 0, 0, repl, 4096, 6, [2, 2], [4, 4])
    assert _sched(r) == [
        (4, [(0, 1, 2, 0), (1, 1, 2, 0)], []),
        (6, [(0, 0, 1, 2), (1, 0, 1, 2)], []),
        (4, [(0, 0, 1, 3)], [(1, 3)]),
        (5, [(0, 0, 1, 4)], []),
        (4, [(1, 1, 4, 0)], []),
        (5, [(1, 0, 1, 4)], []),
    ]
    assert r.steps == 6 and r.preemptions == 1
    assert list(r.refill) == [0, 3] and list(r.n_preempt) == [0, 1]
    assert r.processed_tokens == 13  # (2+4-1)*2 + 3 refilled: conservation
    assert list(r.t_first[0]) == [1.0, 1.0] and list(r.t_done[0]) == [4.0, 6.0]


def test_example_B_nrf():
    # vLLM, C=4096, M=12, r1=(1,6), r2=(1,6), r3=(5,4).  Step 3: r1 -> 11, r2 -> 12, r3 needs 13 and
    # has no lower-retention victim (it is the newest) -> self-preempts, freeing 6.
    r = _run("prefill_first", 0, 0, "nrf", 4096, 12, [1, 1, 5], [6, 6, 4])
    assert _sched(r) == [
        (7, [(0, 1, 1, 0), (1, 1, 1, 0), (2, 1, 5, 0)], []),
        (10, [(0, 0, 1, 1), (1, 0, 1, 1), (2, 0, 1, 5)], []),
        (6, [(0, 0, 1, 2), (1, 0, 1, 2)], [(2, 6)]),
        (8, [(0, 0, 1, 3), (1, 0, 1, 3)], []),
        (10, [(0, 0, 1, 4), (1, 0, 1, 4)], []),
        (12, [(0, 0, 1, 5), (1, 0, 1, 5)], []),
        (7, [(2, 1, 7, 0)], []),
        (8, [(2, 0, 1, 7)], []),
    ]
    assert list(r.refill) == [0, 0, 6] and r.processed_tokens == 26
    assert list(r.t_done[0]) == [6.0, 6.0, 8.0]


def test_example_B_srf():
    # Same workload under SRF: running visited by decreasing m (Q3): r3, r1, r2.  Step 3: r3 -> 11,
    # r1 -> 12; r2 needs 13 and no running request has lower retention than r2 -> self-preempt (frees 2).
    r = _run("prefill_first", 0, 0, "srf", 4096, 12, [1, 1, 5], [6, 6, 4])
    assert _sched(r) == [
        (7, [(0, 1, 1, 0), (1, 1, 1, 0), (2, 1, 5, 0)], []),
        (10, [(2, 0, 1, 5), (0, 0, 1, 1), (1, 0, 1, 1)], []),
        (10, [(2, 0, 1, 6), (0, 0, 1, 2)], [(1, 2)]),
        (12, [(2, 0, 1, 7), (0, 0, 1, 3)], []),
        (7, [(1, 1, 3, 0)], []),
        (9, [(0, 0, 1, 4), (1, 0, 1, 3)], []),
        (11, [(0, 0, 1, 5), (1, 0, 1, 4)], []),
        (6, [(1, 0, 1, 5)], []),
    ]
    assert list(r.refill) == [0, 2, 0] and r.processed_tokens == 22
    assert list(r.t_done[0]) == [7.0, 8.0, 4.0]


def test_example_C_chunked_hybrid():
    # Sarathi-style (decode-first, hybrid, chunked), C=4, M=inf, r1=(6,2), r2=(3,2).
    r = _run("decode_first", 1, 1, "nrf", 4, -1, [6, 3], [2, 2])
    assert [e for (_, e, _) in _sched(r)] == [
        [(0, 1, 4, 0)],
        [(0, 1, 2, 4), (1, 1, 2, 0)],
        [(0, 0, 1, 6), (1, 1, 1, 2)],  # last 1-token chunk is still a prefill (Q17)
        [(1, 0, 1, 3)],
    ]
    assert list(r.t_first[0]) == [2.0, 3.0] and list(r.t_done[0]) == [3.0, 4.0]
    assert r.processed_tokens == 11
    # vLLM with C=4 cannot run r1 (I=6 > C, non-chunked): never fits (Q35)
    assert _run("prefill_first", 0, 0, "nrf", 4, -1, [6, 3], [2, 2]).status == "never_fits"


def test_example_D_online():
    # D1: r2 arrives at 1.5, after step 1 ends at 1 -> admitted at step 3
    r = _run("prefill_first", 0, 0, "nrf", 4096, -1, [2, 1], [2, 1], [0.0, 1.5])
    assert r.steps == 3 and list(r.t_first[0]) == [1.0, 3.0] and list(r.t_done[0]) == [2.0, 3.0]
    assert r.mean_ttft[0] == (1.0 + 1.5) / 2 and r.mean_tpot[0] == 1.0  # O=1 excluded from TPOT
    # D2: idle jump to T=5 is not a step
    r = _run("prefill_first", 0, 0, "nrf", 4096, -1, [1, 1], [1, 1], [0.0, 5.0])
    assert r.steps == 2 and r.idle_jumps == 1 and r.makespan[0] == 6.0
    assert list(r.t_first[0] - [0.0, 5.0]) == [1.0, 1.0]
    # D3: T <= clock is inclusive: r2 (T=2.0) joins at step 3 which starts at 2.0
    r = _run("prefill_first", 0, 0, "nrf", 4096, -1, [2, 1], [2, 1], [0.0, 2.0])
    assert [s["start"] for s in r.steps_list] == [0.0, 1.0, 2.0]
    assert r.steps_list[2]["entries"] == [(1, 1, 1, 0)]


@pytest.mark.parametrize("name,order,hy,ch,steps,ttft2,batches", [
    ("vllm", "prefill_first", 0, 0, 4, 2.0, [[(0, 1, 2)], [(1, 1, 3)], [(0, 0, 1)], [(0, 0, 1)]]),
    ("vllm-hy", "prefill_first", 1, 0, 3, 2.0, [[(0, 1, 2)], [(1, 1, 3), (0, 0, 1)], [(0, 0, 1)]]),
    ("sarathi-nocp", "decode_first", 1, 0, 3, 2.0, [[(0, 1, 2)], [(0, 0, 1), (1, 1, 3)], [(0, 0, 1)]]),
    ("sarathi-nohy", "decode_first", 0, 0, 4, 4.0, [[(0, 1, 2)], [(0, 0, 1)], [(0, 0, 1)], [(1, 1, 3)]]),
    ("sarathi", "decode_first", 1, 1, 3, 2.0, [[(0, 1, 2), (1, 1, 2)], [(0, 0, 1), (1, 1, 1)], [(0, 0, 1)]]),
])
def test_example_E_presets_differ(name, order, hy, ch, steps, ttft2, batches):
    # r1=(2,3), r2=(3,1), C=4 for every preset, M=inf (SURVEY 8(c.9) Example E)
    r = _run(order, hy, ch, "nrf", 4, -1, [2, 3], [3, 1])
    assert r.steps == steps and r.t_first[0][1] == ttft2
    assert [[(i, p, c) for (i, p, c, _) in e] for (_, e, _) in _sched(r)] == batches
    assert r.processed_tokens == 7  # (2+3-1) + (3+1-1), no preemption


def test_fig3_memory_rule():
    # Fig. 3 caption: with M = 8, holdings 4 + 2 + 3 > 8 after the batch -> r3 not admitted.
    # r1 (I=4) and r2 (I=2) fit (4 + 2 = 6); r3 (I=3) would need 6 + 3 = 9 > 8.
    r = _run("prefill_first", 0, 0, "nrf", 4096, 8, [4, 2, 3], [1, 1, 1])
    assert r.steps_list[0]["entries"] == [(0, 1, 4, 0), (1, 1, 2, 0)]
    assert r.steps_list[1]["entries"] == [(2, 1, 3, 0)]


def test_status_codes():
    assert _run("prefill_first", 0, 0, "nrf", 4096, -1, [4096], [2]).status == "too_long"  # I+O-1 > S
    assert _run("prefill_first", 0, 0, "nrf", 4096, 10, [8], [4]).status == "never_fits"  # 11 > M
    assert _run("decode_first", 1, 1, "nrf", 4, -1, [4096], [1]).status == "ok"  # chunked: fits
    cfg = o.make_config("prefill_first", 0, 0, "nrf", C=4096, M=-1, max_steps=2)
    assert o.run(cfg, [1], [5], [0.0], UNIT).status == "max_steps"
