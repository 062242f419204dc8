"""Oracle pins: the alternative-reading knobs (Q10/Q16 alternatives).

Hand traces under the unit cost (every batch costs 1, so times count batches), worked out in the comments, plus
the log verifier and the knob invariants (|B| <= max_seqs; a waiting admission leaves the watermark free) on
random configurations."""
import numpy as np
import pytest

import oracle as o
from tests_util_knobs import random_knob_case
from verifier import verify

UNIT = o.unit_cost(1.0)


def run(I, O, order="prefill_first", hybrid=0, chunked=0, repl="nrf", C=4096, M=-1, **kw):
    cfg = o.make_config(order, hybrid, chunked, repl, C=C, M=M, **kw)
    return o.run(cfg, np.array(I, np.int32), np.array(O, np.int32), np.zeros(len(I)), UNIT, trace=True)


def test_hol_blocks_the_rest_of_the_waiting_group():
    # vLLM, M = 6: r0 = (2, 3), r1 = (5, 1), r2 = (1, 1).  Step 1 visits R_w in order: r0 fits (U = 2), r1 needs
    # 2 + 5 > 6 and is skipped.  Frozen reading (Q10, continue): r2 fits (U = 3) and finishes at step 1; r0
    # decodes at steps 2 and 3 (U = 3, 4) while r1 still does not fit; r1 runs alone at step 4.
    # Head-of-line blocking: r1's failure ends R_w's visit, so r2 waits until step 4, where r1 (U = 5) and r2
    # (U = 6) are admitted together.  Both take 4 batches; r2 finishes at 1 vs 4.
    base = run([2, 5, 1], [3, 1, 1], M=6)
    hol = run([2, 5, 1], [3, 1, 1], M=6, knobs=o.KNOB_HOL)
    assert base.steps == hol.steps == 4
    assert list(base.t_done[0]) == [3.0, 4.0, 1.0]
    assert list(hol.t_done[0]) == [3.0, 4.0, 4.0]


def test_max_seqs_caps_the_batch():
    # vLLM, three (I=2, O=2) requests, max_seqs = 2: step 1 prefills r1, r2 (r3 hits the cap); step 2 prefills r3
    # alone (the decodes fail the phase check, no hybrid); step 3 decodes r1, r2 (r3's decode hits the cap);
    # step 4 decodes r3.  Without the cap: one prefill batch and one decode batch.
    assert run([2, 2, 2], [2, 2, 2], max_seqs=2).steps == 4
    assert run([2, 2, 2], [2, 2, 2]).steps == 2
    r = run([2, 2, 2], [2, 2, 2], max_seqs=2)
    assert max(len(s["entries"]) for s in r.steps_list) == 2


def test_watermark_keeps_kvs_free_for_running_requests():
    # vLLM, M = 10, watermark 3, two (I=4, O=2): r1 is admitted (0 + 4 + 3 <= 10), r2 is not (4 + 4 + 3 > 10)
    # although it would fit (8 <= 10); r1 decodes and finishes at step 2, r2 prefills at step 3 and decodes at 4.
    assert run([4, 4], [2, 2], M=10, kv_watermark=3).steps == 4
    assert run([4, 4], [2, 2], M=10).steps == 2
    # a request whose peak plus the watermark exceeds M can never be admitted into an empty cache (Q35)
    assert run([4, 4], [2, 2], M=10, kv_watermark=6).status == "never_fits"


@pytest.mark.parametrize("seed", range(120))
def test_random_knob_configs_verify(seed):
    wl, cfg, (C, M, hybrid), knobs = random_knob_case(seed)
    r = o.run(cfg, wl.I, wl.O, wl.T, o.load_cost_models()["llama3-8b_a100_theoretical"], trace=True)
    assert r.status == "ok"
    outs = dict(t_first=list(r.t_first[0]), t_done=list(r.t_done[0]), n_preempt=list(r.n_preempt),
                refill=list(r.refill))
    assert verify(r.steps_list, list(wl.I), list(wl.O), list(wl.T), C, cfg.M, outs, hybrid=bool(hybrid),
                  kv_block=knobs.get("kv_block", 1)) == []
    if knobs["max_seqs"]:
        assert max(len(s["entries"]) for s in r.steps_list) <= knobs["max_seqs"]


def test_nrf_by_arrival_keeps_a_refilled_request_in_place():
    # vLLM, M = 5: r0 = (3, 1), r1 = (3, 2), r2 = (1, 2).  Step 1: r0 (U = 3) and r2 (U = 4) prefill, r1 does not fit
    # (6 > 5); r0 finishes.  Step 2: r1 prefills (U = 4; r2's decode fails the phase check).  Step 3 decodes:
    # * frozen NRF (admission order, Q6): r2 (seq 2) first -> U = 5; r1 (seq 3) needs 6 > 5 with no newer admission
    #   to evict -> self-preempts; r2 finishes at 3; r1 refills (4 tokens) and finishes at 4;
    # * by arrival (T, id): r1 (id 1) first -> U = 5; r2 (id 2) self-preempts; r1 finishes at 3, r2 at 4.
    assert list(run([3, 3, 1], [1, 2, 2], M=5).t_done[0]) == [1.0, 4.0, 3.0]
    assert list(run([3, 3, 1], [1, 2, 2], M=5, knobs=o.KNOB_NRF_ARRIVAL).t_done[0]) == [1.0, 3.0, 4.0]


def test_srf_visiting_in_admission_order():
    # vLLM-SRF, M = 4: r0 = (1, 3), r1 = (2, 3).  Step 1 prefills both (U = 3).  Step 2 decodes:
    # * frozen SRF (visit by m descending, Q3): r1 (m 2) decodes (U = 4); r0 (m 1) has no lower-retention
    #   victim and self-preempts; r1 finishes at 3 while r0's refill (2 tokens) waits, refills at 4, ends at 5;
    # * admission order, SRF only for victims: r0 (seq 1) decodes first (U = 4); r1's only lower-m request r0 is
    #   already in B, so r1 self-preempts; r0 finishes at 3, r1 refills (3 tokens) at 4 and ends at 5.
    base = run([1, 2], [3, 3], repl="srf", M=4)
    alt = run([1, 2], [3, 3], repl="srf", M=4, knobs=o.KNOB_SRF_VISIT_ADMISSION)
    assert list(base.t_done[0]) == [5.0, 3.0] and list(alt.t_done[0]) == [3.0, 5.0]


def test_paged_kv_blocks():
    # vLLM, KV in blocks of 4 tokens, M = 12 tokens = 3 blocks: r0 = r1 = (I=4, O=2), r2 = (1, 1).  Step 1 admits
    # all three (one block each: U = 3); r2 finishes (U = 2).  Step 2: r0's decode opens its second block (U = 3);
    # r1's needs a fourth block, and with no newer admission to evict r1 self-preempts; r0 finishes.  Step 3: r1
    # refills its 5 tokens (2 blocks) and finishes.  Per token (Q15 frozen) nothing is short: 2 steps.
    per_token = run([4, 4, 1], [2, 2, 1], M=12)
    paged = run([4, 4, 1], [2, 2, 1], M=12, kv_block=4)
    assert (per_token.steps, per_token.preemptions) == (2, 0) and list(per_token.t_done[0]) == [2.0, 2.0, 1.0]
    assert (paged.steps, paged.preemptions) == (3, 1) and list(paged.t_done[0]) == [2.0, 3.0, 1.0]
    # the capacity is floor(M / b) blocks: a peak of 5 tokens needs 2 blocks, M = 7 tokens holds only one
    assert run([3, 1], [3, 2], M=7).status == "ok" and run([3, 1], [3, 2], M=7, kv_block=4).status == "never_fits"
