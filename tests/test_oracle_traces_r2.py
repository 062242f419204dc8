"""Oracle pins, round 2: hand traces for the three sub-paths the round-1 pins left open.

* SRF+Hist with a LEARNED histogram (>= 8 completions): a row-p90 prediction and a global-column
  fallback prediction each decide an admission/deferral (reading Q31).
* Rank_I / Rank_O over several steps, running requests interleaved with waiting ones by key
  (readings Q20, Q37), including an NRF self-preemption inside the rank order.
* Q2: a preempted request re-enters R_w at its (T, id) place, i.e. AHEAD of a later, never-admitted
  arrival ("appended to R_w" + R_w "ordered by the arrival times" P:1626).

Every expected value is derived BY HAND in the comments from Algorithm 1, the
GetNextBatch text, Eq. (6) and the readings, not by running
the oracle.  Entries are (id, phase 1=prefill/0=decode, c, m_before); events are (victim, m discarded).
A unit-cost stub (every batch costs 1 s) makes the clock equal the step count.
"""
import oracle as o

UNIT = o.unit_cost()


def _run(order, hybrid, chunked, repl, C, M, I, O, T=None):
    T = T if T is not None else [0.0] * len(I)
    cfg = o.make_config(order, hybrid, chunked, repl, C=C, M=M)
    return o.run(cfg, I, O, T, UNIT, trace=True)


def _entries(r):
    return [s["entries"] for s in r.steps_list]


# ---------------------------------------------------------------- SRF+Hist, learned histogram
# vLLM order ({R_w, R_r}, no hybrid, no chunking), C = 4096, M = 27.
#   r0..r7 = (I=8, O=2) at T=0  -> row bI = 3 (8 <= I < 16), column bO = 1 (2 <= O < 4)
#   r8     = (I=2, O=4) at T=0  -> row bI = 1, column bO = 2
#   r9     = (I=8, O=1), r10 = (I=8, O=1), r11 = (I=2, O=1) arrive at T=20
# Q31: O_hat(I) = 2^(b+1) - 1 for the nearest-rank p90 bucket b of the I-row if it holds >= 8
# completions, else of the global column sums if they hold >= 8, else the prior 256.  Defer a
# waiting candidate iff something is running and U + sum_running max(O_hat - g, 0) + s + rem > M.
#
# Steps 1-16 (prior 256, fewer than 8 completions): at step 2k+1 nothing is running, so the first
# waiting request r_k (k <= 7) is admitted without the deferral test (U = 8); every later waiting
# candidate is deferred, e.g. r1: 8 + 256 + 8 + 256 > 27.  Step 2k+2 decodes r_k (held max(8, 9) = 9
# <= 27), which generates its 2nd token and completes.  After step 16: H[3][1] = 8.
# Step 17 (clock 16; r9-r11 not arrived): r8 alone, nothing running -> admitted, prefill c = 2.
#   (Its row bI = 1 is empty, the column holds 8 -> O_hat = 3: the learned value is now in force.)
# Steps 18-20: r8 decodes (m 2 -> 3 -> 4 -> 5), g = 4 = O at step 20 -> H[1][2] = 1.
# Step 21 (clock 20, arrivals T = 20 <= 20 inclusive, Q21):
#   row 3 holds 8 (all bO = 1): target ceil(0.9*8) = 8 reached at b = 1 -> O_hat(I=8) = 3   (ROW)
#   row 1 holds 1 < 8 -> column {b1: 8, b2: 1}, n = 9, target ceil(8.1) = 9: cum(b1) = 8 < 9,
#   cum(b2) = 9 -> O_hat(I=2) = 7                                                        (COLUMN)
#   r9:  nothing running -> admitted; U = 8, running rem = 3 - 0 = 3.
#   r10: 8 + 3 + 8 + 3 = 22 <= 27 -> admitted (KV 16 <= 27); U = 16, running rem 6.
#        (had the column been used for row 3: 8 + 7 + 8 + 7 = 30 > 27 -> deferred)
#   r11: 16 + 6 + 2 + 7 = 31 > 27 -> DEFERRED although its KVs fit (16 + 2 = 18 <= 27).
#        (with O_hat = 3 it would be 27 <= 27 -> admitted: the column's outlier decides)
#   B = {r9 p8, r10 p8}; both complete (O = 1).
# Step 22: r11 alone -> admitted, completes.  22 steps, no preemption.
def test_srf_hist_learned_histogram_row_and_column():
    I = [8] * 8 + [2, 8, 8, 2]
    O = [2] * 8 + [4, 1, 1, 1]
    T = [0.0] * 9 + [20.0] * 3
    r = _run("prefill_first", 0, 0, "srf_hist", 4096, 27, I, O, T)
    expect = []
    for k in range(8):
        expect += [[(k, 1, 8, 0)], [(k, 0, 1, 8)]]
    expect += [[(8, 1, 2, 0)], [(8, 0, 1, 2)], [(8, 0, 1, 3)], [(8, 0, 1, 4)]]
    expect += [[(9, 1, 8, 0), (10, 1, 8, 0)], [(11, 1, 2, 0)]]
    assert r.status == "ok" and r.preemptions == 0
    assert _entries(r) == expect
    assert list(r.t_done[0]) == [2.0 * (k + 1) for k in range(8)] + [20.0, 21.0, 21.0, 22.0]
    # the same workload under plain SRF (no deferral) packs step 1: r0, r1, r2 (24), r8 (26 <= 27)
    p = _run("prefill_first", 0, 0, "srf", 4096, 27, I, O, T)
    assert [e[0] for e in p.steps_list[0]["entries"]] == [0, 1, 2, 8]


def test_hist_predict_learned_values():
    # the two predictions of step 21 above, straight from the prediction rule (Q31)
    H = [[0] * 18 for _ in range(18)]
    H[3][1] = 8
    H[1][2] = 1
    assert o.hist_predict(H, 8) == 3 and o.hist_predict(H, 15) == 3   # row 3 (n = 8)
    assert o.hist_predict(H, 2) == 7 and o.hist_predict(H, 3) == 7    # row 1 (n = 1) -> column (n = 9)
    assert o.hist_predict(H, 1) == 7 and o.hist_predict(H, 100) == 7  # empty rows -> column
    H[3][1] = 7                                                        # 8 completions in all: column
    assert o.hist_predict(H, 8) == 7                                  # {b1: 7, b2: 1}: cum(b1) 7 < 8
    H[1][2] = 0
    assert o.hist_predict(H, 8) == 256                                 # 7 < 8 anywhere: the prior


# ---------------------------------------------------------------- Rank_I / Rank_O over several steps
# One group [W u R] sorted by (key, T, id), hybrid on, no chunking (Q20, Q37).  C = 7, M = inf.
#   r0 = (I=1, O=3), r1 = (I=5, O=3) at T=0; r2 = (I=3, O=2), r3 = (I=4, O=1) arrive at T=1.
#   Every peak I+O-1 (3, 7, 4, 4) fits C = 7, as a non-chunked preset requires (Q35).
def test_rank_i_interleaves_running_and_waiting():
    # Rank_I (key I):
    # step 1 (clock 0): r0 p1 (tok 1), r1 p5 (tok 6).
    # step 2 (clock 1, r2/r3 arrive): order r0 (1, running), r2 (3, waiting), r3 (4, waiting),
    #         r1 (5, running): r0 d (tok 1), r2 p3 (tok 4), r3 p4 -> 8 > 7 rejected (the visit goes on,
    #         Q10), r1 d (tok 5).
    # step 3: order r0 (d), r2 (d), r3 (p), r1 (d): tok 1, 2, 6, 7 <= 7 -> everything completes
    #         (r0 g 3, r2 g 2, r3 g 1, r1 g 3).
    r = _run("rank_i", 1, 0, "nrf", 7, -1, [1, 5, 3, 4], [3, 3, 2, 1], [0.0, 0.0, 1.0, 1.0])
    assert _entries(r) == [
        [(0, 1, 1, 0), (1, 1, 5, 0)],
        [(0, 0, 1, 1), (2, 1, 3, 0), (1, 0, 1, 5)],
        [(0, 0, 1, 2), (2, 0, 1, 3), (3, 1, 4, 0), (1, 0, 1, 6)],
    ]
    assert list(r.t_done[0]) == [3.0, 3.0, 3.0, 3.0]


def test_rank_o_interleaves_running_and_waiting():
    # Rank_O (key O, ties by (T, id)):
    # step 1: r0 (O 3, id 0), r1 (O 3, id 1): r0 p1, r1 p5 (tok 6).
    # step 2: order r3 (1, waiting), r2 (2, waiting), r0 (3, running), r1 (3, running):
    #         r3 p4 (tok 4), r2 p3 (tok 7), r0 d -> 8 > 7 and r1 d -> 8 > 7 rejected.  r3 completes.
    # step 3: order r2 (2), r0 (3), r1 (3): three decodes; r2 g 2 completes.
    # step 4: r0 d, r1 d -> g 3: both complete.
    r = _run("rank_o", 1, 0, "nrf", 7, -1, [1, 5, 3, 4], [3, 3, 2, 1], [0.0, 0.0, 1.0, 1.0])
    assert _entries(r) == [
        [(0, 1, 1, 0), (1, 1, 5, 0)],
        [(3, 1, 4, 0), (2, 1, 3, 0)],
        [(2, 0, 1, 3), (0, 0, 1, 1), (1, 0, 1, 5)],
        [(0, 0, 1, 2), (1, 0, 1, 6)],
    ]
    assert list(r.t_done[0]) == [4.0, 4.0, 3.0, 2.0]


def test_rank_i_self_preemption_and_refill():
    # Rank_I, C = 4096, M = 6, NRF victims (Q20).  r0 = (I=1, O=4), r1 = (I=2, O=3), r2 = (I=3, O=1).
    # step 1: r0 p1 (U 1), r1 p2 (U 3), r2 p3 (U 6 <= 6).  r2 completes, frees 3 -> U 3.
    # step 2: r0 d (held 1 -> 2: U 4), r1 d (2 -> 3: U 5).
    # step 3: r0 d (2 -> 3: U 6); r1 d needs 3 -> 4: 7 > 6; pool = running, not in B, lower retention
    #         than r1 (NRF: larger admission seq) = {} (r0 is in B and older) -> r1 self-preempts (Q8),
    #         frees 3 -> U 3; event (1, m 3).
    # step 4: group by I: running r0 (1), waiting r1 (2, s = I + g = 4): r0 d (3 -> 4: U 4) -> g 4,
    #         completes; r1 refill 4 + 4 = 8 > 6 -> skipped (a waiting candidate never preempts, Q5).
    # step 5: r1 refill p4 (m 0) -> token 3 = O: completes.
    r = _run("rank_i", 1, 0, "nrf", 4096, 6, [1, 2, 3], [4, 3, 1])
    assert [(s["U"], s["entries"], s["events"]) for s in r.steps_list] == [
        (6, [(0, 1, 1, 0), (1, 1, 2, 0), (2, 1, 3, 0)], []),
        (5, [(0, 0, 1, 1), (1, 0, 1, 2)], []),
        (3, [(0, 0, 1, 2)], [(1, 3)]),
        (4, [(0, 0, 1, 3)], []),
        (4, [(1, 1, 4, 0)], []),
    ]
    assert r.preemptions == 1 and list(r.refill) == [0, 3, 0]
    assert r.processed_tokens == 14  # (1+4-1) + (2+3-1) + (3+1-1) = 11, + 3 refilled: conservation


# ---------------------------------------------------------------- Q2: re-entry at the (T, id) place
# vLLM (prefill-first, no hybrid), NRF, C = 4096, M = 6, offline.
#   r0 = (I=2, O=4), r1 = (I=2, O=4), r2 = (I=4, O=1)
# step 1: r0 p2 (U 2), r1 p2 (U 4); r2 needs 4: 8 > 6 -> skipped (never admitted so far).
# step 2: r2 skipped (8 > 6); R_r: r0 d (U 5), r1 d (U 6).
# step 3: r2 skipped (10 > 6); r0 d needs 3 -> 4: 7 > 6 -> victim = newest admitted not in B = r1
#         (frees 3, U 3), then r0 admitted (U 4).  r1 re-enters R_w with g = 2 (s = 4).
# step 4: R_w in (T, id) order = [r1, r2] (Q2: r1 is AHEAD of the never-admitted r2): both need 4:
#         8 > 6 -> skipped; r0 d (U 5) -> g 4, completes (frees 5).
# step 5: R_w = [r1, r2]: r1 refill p4 (U 4); r2: 8 > 6 -> skipped.   (A tail append -- the
#         alternative reading -- would visit r2 first and admit it instead.)
# step 6: r2 skipped (4 + 4 > 6); r1 d (U 5) -> g 4, completes.
# step 7: r2 p4 -> completes.
def test_q2_preempted_request_reenters_ahead_of_later_arrival():
    r = _run("prefill_first", 0, 0, "nrf", 4096, 6, [2, 2, 4], [4, 4, 1])
    assert [(s["U"], s["entries"], s["events"]) for s in r.steps_list] == [
        (4, [(0, 1, 2, 0), (1, 1, 2, 0)], []),
        (6, [(0, 0, 1, 2), (1, 0, 1, 2)], []),
        (4, [(0, 0, 1, 3)], [(1, 3)]),
        (5, [(0, 0, 1, 4)], []),
        (4, [(1, 1, 4, 0)], []),
        (5, [(1, 0, 1, 4)], []),
        (4, [(2, 1, 4, 0)], []),
    ]
    assert list(r.t_done[0]) == [4.0, 6.0, 7.0] and list(r.t_first[0]) == [1.0, 1.0, 7.0]
    assert r.preemptions == 1 and list(r.refill) == [0, 3, 0]


def test_q2_online_reentry_by_arrival_time():
    # The same order holds for online arrivals: R_w is ordered by (T, id), so a preempted request that
    # ARRIVED earlier is ahead of one that arrived later, whatever their admission history.
    # r0 = (I=2, O=4, T=0), r1 = (I=2, O=4, T=0), r2 = (I=4, O=1, T=2.5); vLLM NRF, M = 6.
    # steps 1-3 as above (r2 arrives at 2.5 > 2 = clock before step 3: not yet waiting at step 3).
    # step 4 (clock 3 >= 2.5): R_w = [r1 (T 0), r2 (T 2.5)] -> both skipped; r0 d completes.
    # step 5: r1 refill first (U 4); r2 skipped.  step 6: r1 d completes.  step 7: r2.
    r = _run("prefill_first", 0, 0, "nrf", 4096, 6, [2, 2, 4], [4, 4, 1], [0.0, 0.0, 2.5])
    assert [s["entries"] for s in r.steps_list][4:] == [[(1, 1, 4, 0)], [(1, 0, 1, 4)], [(2, 1, 4, 0)]]
    assert list(r.t_done[0]) == [4.0, 6.0, 7.0]
