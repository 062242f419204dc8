"""GPU parity of the per-step schedule trace (sim_run_traced, the schedule log of PAPER.md:714-719)
against the oracle's own trace of the same run: every step's (step, U, tok), its batch entries (id, phase, c,
m_before) in admission order and its preemptions (id, m) in the order they happened -- integers bit-exact --
and the step's start clock and batch time d_j at 0 ULP."""
import io

import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import presets, simsweep, workloads
from parity import cost_models, oracle_config
from tests_util_knobs import random_knob_case

pytestmark = pytest.mark.gpu
A100 = ["llama3-8b_a100_linear"]
UNIT = [("unit", 1.0)]


def W(I, O, T=None, name="hand"):
    T = [0.0] * len(I) if T is None else T
    return workloads.Workload(np.array(I, np.int32), np.array(O, np.int32), np.array(T, np.float64), name)


def traced(cfg, wl, names, caps=(1 << 16, 1 << 20, 1 << 16)):
    ocms, pcms = cost_models()
    c = simsweep.SimConfig.from_buffer_copy(cfg)
    c.workload, c.n_cost = 0, len(names)
    for k in range(len(names)):
        c.cost[k] = k
    cms = [simsweep.unit_cost(nm[1]) if isinstance(nm, tuple) else pcms[nm] for nm in names]
    ocost = [o.unit_cost(nm[1]) if isinstance(nm, tuple) else ocms[nm] for nm in names]
    g, log = simsweep.sim_run_traced(c, [wl], cms, caps=caps)
    r = o.run(oracle_config(c), wl.I, wl.O, wl.T, ocost, trace=True, trace_cap=1 << 25)
    return g, log, r


def assert_same_trace(cfg, wl, names, label, caps=(1 << 16, 1 << 20, 1 << 16)):
    g, log, r = traced(cfg, wl, names, caps)
    assert g.status(0) == r.status, (label, g.status(0), r.status)
    a, b = log.steps_list(), r.steps_list
    assert len(a) == len(b) == int(g.results["steps"][0]), (label, len(a), len(b))
    for x, y in zip(a, b):
        assert x == y, f"{label}: first divergence at step {y['step']}:\n gpu    {str(x)[:600]}\n oracle {str(y)[:600]}"
    # the totals the C-ABI reports are the result's counters
    assert len(log.entries) == int(g.results["batch_entries"][0]) and len(log.events) == int(g.results["preemptions"][0])
    return g, log


def test_hand_traces():
    cfg = simsweep.make_config
    cases = [
        (cfg(0, 0, 0, 0, C=4096, M=6), W([2, 2], [4, 4])),
        (cfg(0, 0, 0, 1, C=4096, M=6), W([2, 2], [4, 4])),
        (cfg(0, 0, 0, 0, C=4096, M=12), W([1, 1, 5], [6, 6, 4])),
        (cfg(0, 0, 0, 1, C=4096, M=12), W([1, 1, 5], [6, 6, 4])),
        (cfg(1, 1, 1, 0, C=4, M=-1), W([6, 3], [2, 2])),
        (cfg(0, 0, 0, 0, C=4096, M=-1), W([2, 1], [2, 1], [0.0, 1.5])),
        (cfg(0, 0, 0, 0, C=4096, M=-1), W([1, 1], [1, 1], [0.0, 5.0])),
        (cfg(0, 0, 0, 2, C=1000, M=1000), W([10] * 5, [3] * 5)),
        (cfg(0, 0, 0, 0, C=4096, M=8), W([4, 2, 3], [1, 1, 1])),
    ]
    for i, (c, wl) in enumerate(cases):
        assert_same_trace(c, wl, UNIT, f"hand{i}")


def test_config1_presets_and_four_cost_models():
    wl = workloads.fixed(16, 16, 32)
    for nm in presets.GRID_PRESETS:
        for sfx in ("", "-srf"):
            assert_same_trace(simsweep.preset_config(nm + sfx, 100_000), wl, A100, nm + sfx)
    names = ["llama3-8b_a100_linear", "llama3-8b_a100_theoretical", "llama3-70b_h100x4_linear", ("unit", 0.5)]
    assert_same_trace(simsweep.preset_config("sarathi-srf", 2_000), workloads.fixed(40, 24, 64), names, "K=4")


@pytest.mark.parametrize("block", range(4))
def test_random_knob_cases(block):
    for seed in range(40 * block, 40 * block + 40):
        wl, oc, _, knobs = random_knob_case(seed)
        c = simsweep.make_config(oc.order, oc.hybrid, oc.chunked, oc.replacement, C=oc.C, M=oc.M, S=oc.S, **knobs)
        assert_same_trace(c, wl, A100 if seed % 2 else ["llama3-70b_h100x4_theoretical"], f"knob case {seed}")


@pytest.mark.parametrize("block", range(2))
def test_random_default_instance_cases(block):
    # configs without knobs: the schedule is traced in the knob instance, so the same configs through sim_sweep
    # (the default instance, steady runs compressed) must give the traced run's results
    rng = np.random.default_rng(900 + block)
    for t in range(30):
        nm = presets.names()[int(rng.integers(0, len(presets.names())))]
        wl = workloads.random_small(4000 + 100 * block + t, int(rng.integers(1, 60)), max_len=int(rng.integers(2, 40)),
                                    online=bool(rng.integers(0, 2)), S=96)
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        c = simsweep.preset_config(nm, int(rng.integers(peak, 4 * peak + 1)), S=96)
        g, log = assert_same_trace(c, wl, A100, f"{nm} case {t}")
        c2 = simsweep.SimConfig.from_buffer_copy(c)
        c2.workload, c2.n_cost, c2.cost[0] = 0, 1, 0
        g2 = simsweep.sim_sweep([c2], [wl], [cost_models()[1]["llama3-8b_a100_linear"]])
        for f in ("status", "steps", "preemptions", "batch_entries", "sum_U", "visits", "makespan"):
            assert np.array_equal(g.results[f], g2.results[f]), (nm, t, f)
        assert np.array_equal(g.t_done, g2.t_done) and np.array_equal(g.refill, g2.refill)


def test_preemption_thrash_and_run_compression_off():
    # vLLM under KV pressure: evictions, refills and self-preemptions in most steps; the traced run
    # forms every step, including those the product kernel compresses into steady decode runs
    for nm in ("vllm", "vllm-srf", "sarathi", "sarathi-srf", "vllm-hy-srf", "sarathi-nohy"):
        g, log = assert_same_trace(simsweep.preset_config(nm, 6_000), workloads.fixed(96, 160, 192), A100, nm)
        if nm.startswith("vllm"):
            assert len(log.events) > 0
    # small capacities: the log is fetched again with the exact sizes
    assert_same_trace(simsweep.preset_config("vllm", 6_000), workloads.fixed(96, 160, 192), A100, "caps", caps=(3, 5, 1))


def test_pf_orca_rank_and_online():
    wl = workloads.fixed(64, 96, 128)
    for nm in ("vllm-pf", "sarathi-pf", "orca", "rank-i", "rank-o-srf"):
        assert_same_trace(simsweep.preset_config(nm, 8_000), wl, A100, nm)
    wl = workloads.random_small(7, 200, max_len=64, online=True, S=4096)
    for nm in ("vllm-srf-hist", "sarathi-srf", "vllm"):
        assert_same_trace(simsweep.preset_config(nm, 3_000), wl, A100, "online " + nm)


def test_grid_thrash_cell_full_size():
    # the bench's critical-path simulation at its BASELINE configs[1] size (W = 1024, M = 100 000)
    g, log = assert_same_trace(simsweep.preset_config("vllm-srf", 100_000), workloads.fixed(128, 1024, 1024), A100,
                               "vllm-srf 128/1024", caps=(1 << 14, 1 << 22, 1 << 16))
    assert len(log.steps) == 11151


def test_large_window_variant_trace():
    wl = workloads.fixed(3, 4, 4500)  # n > 4096: the global-arena kernel instance
    assert_same_trace(simsweep.preset_config("sarathi", 3_000), wl, A100, "n=4500")


def test_schedule_log_csv():
    g, log = assert_same_trace(simsweep.preset_config("vllm", 12), W([2, 2], [4, 4]), UNIT, "csv")
    buf = io.StringIO()
    log.to_csv(buf)
    rows = buf.getvalue().strip().split("\n")
    assert rows[0] == "batch,start_s,duration_s,request,phase,c,m_before,event"
    assert len(rows) == 1 + len(log.entries) + len(log.events)
    assert rows[1].split(",")[3:7] == ["0", "prefill", "2", "0"]
