"""Oracle pins: closed-form schedules and paper invariants.

Each expected count is derived from the algorithm by arithmetic (stated in the
comment), independent of the oracle's code.
"""
import math

import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import presets, workloads

CMS = o.load_cost_models()
A100_8B = CMS["llama3-8b_a100_linear"]

PAPER_TABLE = {  # PAPER.md:48-54, Table "Schedulers used": priority, hybrid, chunked, C (S = 4096)
    "vllm": ("prefill", 0, 0, 4096),
    "sarathi": ("decode", 1, 1, 512),
    "sarathi-cs": ("decode", 1, 1, 4096),
    "sarathi-nocp": ("decode", 1, 0, 4096),
    "vllm-hy": ("prefill", 1, 0, 4096),
    "sarathi-nohy": ("decode", 0, 0, 4096),
}


def _cfg(name, M, S=4096, **kw):
    p = presets.preset(name, S=S)
    return o.make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=p["C"], M=M, S=S, **kw)


def test_preset_table_matches_paper():
    for name, (prio, hy, ch, C) in PAPER_TABLE.items():
        p = presets.preset(name)
        assert p["order"] == (0 if prio == "prefill" else 1), name
        assert (p["hybrid"], p["chunked"], p["C"]) == (hy, ch, C), name
    assert presets.preset("vllm-srf")["replacement"] == 1
    assert presets.preset("sarathi-srf-hist")["replacement"] == 2


@pytest.mark.parametrize("name", presets.GRID_PRESETS)
def test_config1_closed_form(name):
    # Config [1]: W=32, I=O=16.  Every preset admits all 32 prompts in step 1 (32*16 = 512 <= C for all,
    # Sarathi exactly fills C=512), then 15 decode steps of 32; KV peak 32*(16+16-1) = 992 < M.
    wl = workloads.fixed(16, 16, 32)
    r = o.run(_cfg(name, 100_000), wl.I, wl.O, wl.T, A100_8B, trace=True)
    assert r.status == "ok" and r.steps == 16 and r.preemptions == 0
    st = r.steps_list
    assert [(len(s["entries"]), s["tok"]) for s in st] == [(32, 512)] + [(32, 32)] * 15
    assert st[-1]["U"] == 32 * 31 and r.processed_tokens == 32 * 31
    d = [s["d"] for s in st]
    clock = 0.0
    for x in d:
        clock = clock + x
    assert (r.t_first[0] == d[0]).all() and (r.t_done[0] == clock).all()


def test_config1_all_presets_identical_schedule():
    wl = workloads.fixed(16, 16, 32)
    base = None
    for name in presets.GRID_PRESETS:
        r = o.run(_cfg(name, 100_000), wl.I, wl.O, wl.T, A100_8B, trace=True)
        sched = [sorted(s["entries"]) for s in r.steps_list]
        if base is None:
            base = (sched, list(r.t_done[0]))
        assert (sched, list(r.t_done[0])) == base, name


@pytest.mark.parametrize("O", [1, 2, 5])
def test_chunked_prefill_closed_form(O):
    # W=1, I=1024, C=512 chunked: two prefill chunks (token only after the 2nd, Eq. 6) + O-1 decodes
    r = o.run(_cfg("sarathi", 100_000), [1024], [O], [0.0], A100_8B, trace=True)
    assert r.steps == 2 + O - 1
    assert [e[0][2] for e in (s["entries"] for s in r.steps_list[:2])] == [512, 512]
    d = [s["d"] for s in r.steps_list]
    assert r.t_first[0][0] == d[0] + d[1]


@pytest.mark.parametrize("W,I,O", [(64, 128, 8), (100, 100, 5), (7, 1024, 3), (33, 1, 4)])
def test_sarathi_nohy_closed_form(W, I, O):
    # no hybrid + decode-first: each prefill batch admits k = floor(C/I) requests, then decode-only batches
    # persist until they all complete: ceil(W/k) * O steps.
    k = 4096 // I
    r = o.run(_cfg("sarathi-nohy", -1), [I] * W, [O] * W, [0.0] * W, A100_8B)
    assert r.steps == math.ceil(W / k) * O and r.preemptions == 0


@pytest.mark.parametrize("W,I,O", [(100, 100, 5), (64, 128, 8), (1000, 3, 2), (5, 4096, 1)])
def test_vllm_infinite_M_closed_form(W, I, O):
    # prefill-first, no hybrid, M = inf, W <= C: ceil(W/floor(C/I)) prefill batches, then O-1 decode batches
    k = 4096 // I
    r = o.run(_cfg("vllm", -1), [I] * W, [O] * W, [0.0] * W, A100_8B)
    assert r.steps == math.ceil(W / k) + O - 1 and r.preemptions == 0


def test_w32_grid_no_preemption():
    # "Under low contention (W = 32), no evictions occur across all schedulers":
    # 32 * (I+O-1) <= 32 * 2047 < 100 000 = M.
    for name in presets.GRID_PRESETS:
        for I in (1, 32, 1024):
            for O in (1, 32, 1024):
                wl = workloads.fixed(I, O, 32)
                r = o.run(_cfg(name, 100_000), wl.I, wl.O, wl.T, A100_8B)
                assert r.status == "ok" and r.preemptions == 0, (name, I, O)


def test_offline_schedule_independent_of_cost_model():
    # Offline (all T = 0) GetNextBatch never reads the clock (a2 admits everything at step 0), so every
    # integer output is identical under any cost model, and a K=4 shared run
    # reproduces each single-model run's times bit for bit.
    names = ["llama3-8b_a100_linear", "llama3-8b_h100_theoretical", "llama3-70b_a100x4_linear",
             "llama3-70b_h100x4_theoretical"]
    wl = workloads.fixed(64, 256, 1024)
    runs = [o.run(_cfg("vllm", 100_000), wl.I, wl.O, wl.T, CMS[nm]) for nm in names]
    for r in runs[1:]:
        assert (r.steps, r.preemptions, r.processed_tokens, r.sum_U) == \
               (runs[0].steps, runs[0].preemptions, runs[0].processed_tokens, runs[0].sum_U)
        assert (r.refill == runs[0].refill).all()
    shared = o.run(_cfg("vllm", 100_000), wl.I, wl.O, wl.T, [CMS[nm] for nm in names])
    for k, r in enumerate(runs):
        assert (shared.t_done[k] == r.t_done[0]).all() and (shared.t_first[k] == r.t_first[0]).all()
        assert shared.makespan[k] == r.makespan[0]


def test_srf_hist_deferral_hand_trace():
    # SRF+Hist (reading Q31), empty histogram -> prior O_hat = 256, M = 1000, 5 x (I=10, O=3),
    # vLLM order.  Step 1: r0 admitted (nothing running); r1: 10 + 256 + 10 + 256 = 532 <= M; r2: 20 + 512
    # + 266 = 798; r3: 30 + 768 + 266 = 1064 > M -> deferred, r4 too.  Steps 2-3 decode r0-r2 (r3: 30+3 +
    # 3*(256-1) + 266 = 1064 and 33 + 3*(256-2) + 266 = 1061 > M).  Only 3 completions (< 8 observations):
    # still the prior.  Step 4 admits r3 (nothing running) and r4 (532), steps 5-6 decode.  -> 6 steps.
    r = o.run(_cfg("vllm-srf-hist", 1000), [10] * 5, [3] * 5, [0.0] * 5, o.unit_cost(), trace=True)
    assert r.steps == 6
    assert [[e[0] for e in s["entries"]] for s in r.steps_list] == [[0, 1, 2]] * 3 + [[3, 4]] * 3
    assert o.run(_cfg("vllm-srf", 1000), [10] * 5, [3] * 5, [0.0] * 5, o.unit_cost()).steps == 3


def test_rank_orders():
    # App. D: Rank_I visits small I first, Rank_O small O first; one group, hybrid on.
    I, O = [512, 8, 16], [16, 512, 8]
    cfg = o.make_config("rank_i", 1, 0, "nrf", C=4096, M=-1)
    r = o.run(cfg, I, O, [0.0] * 3, o.unit_cost(), trace=True)
    assert [e[0] for e in r.steps_list[0]["entries"]] == [1, 2, 0]
    cfg = o.make_config("rank_i", 1, 0, "nrf", C=600, M=-1)  # 8 + 16 + 100 = 124; + 512 = 636 > 600
    r = o.run(cfg, [512, 8, 16, 100], [1, 1, 1, 1], [0.0] * 4, o.unit_cost(), trace=True)
    assert [e[0] for e in r.steps_list[0]["entries"]] == [1, 2, 3]  # 8+16+100; 512 does not fit any more
    cfg = o.make_config("rank_o", 1, 0, "nrf", C=4096, M=-1)
    r = o.run(cfg, I, O, [0.0] * 3, o.unit_cost(), trace=True)
    assert [e[0] for e in r.steps_list[0]["entries"]] == [2, 0, 1]
