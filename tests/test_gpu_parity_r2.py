"""GPU parity, round 2: the CUDA path (through the C-ABI) vs the CPU oracle on the configurations round 1 left
untested -- the new hand traces (tests/test_oracle_traces_r2.py), the whole W = 32 half of the north-star grid,
K = 4 shared cost models across a grid slice, and the int32-holdings capacity boundary.  Integers bit-exact,
per-request fp64 times 0 ULP, means within 1e-9 relative (tests/parity.py)."""
import numpy as np
import pytest

from paper_2411_07447_b200 import presets, simsweep, workloads
from parity import compare, run_case_list

pytestmark = pytest.mark.gpu
P = presets
A100 = ["llama3-8b_a100_linear"]
UNIT = [("unit", 1.0)]
K4 = ["llama3-8b_a100_linear", "llama3-8b_h100_linear", "llama3-70b_a100x4_linear", "llama3-70b_h100x4_linear"]


def cfg(order, hybrid, chunked, repl, C, M, S=4096, **kw):
    return simsweep.make_config(order, hybrid, chunked, repl, C=C, M=M, S=S, **kw)


def W(I, O, T=None, name="hand"):
    T = [0.0] * len(I) if T is None else T
    return workloads.Workload(np.array(I, np.int32), np.array(O, np.int32), np.array(T, np.float64), name)


def assert_parity(cases, processes=0):
    g, ors = run_case_list(cases, processes=processes)
    bad = []
    for i in range(len(cases)):
        bad += compare(g, ors, i, label=f"case{i}:{cases[i][1].name}")
    assert bad == [], "\n".join(bad[:40])
    return g, ors


def test_round2_hand_traces():
    hist_I = [8] * 8 + [2, 8, 8, 2]
    hist_O = [2] * 8 + [4, 1, 1, 1]
    hist_T = [0.0] * 9 + [20.0] * 3
    cases = [
        (cfg(0, 0, 0, P.REPL_SRF_HIST, 4096, 27), W(hist_I, hist_O, hist_T), UNIT),          # learned histogram
        (cfg(0, 0, 0, P.REPL_SRF, 4096, 27), W(hist_I, hist_O, hist_T), UNIT),               # its SRF control
        (cfg(P.ORDER_RANK_I, 1, 0, 0, 7, -1), W([1, 5, 3, 4], [3, 3, 2, 1], [0, 0, 1, 1]), UNIT),
        (cfg(P.ORDER_RANK_O, 1, 0, 0, 7, -1), W([1, 5, 3, 4], [3, 3, 2, 1], [0, 0, 1, 1]), UNIT),
        (cfg(P.ORDER_RANK_I, 1, 0, 0, 4096, 6), W([1, 2, 3], [4, 3, 1]), UNIT),              # rank self-preemption
        (cfg(0, 0, 0, 0, 4096, 6), W([2, 2, 4], [4, 4, 1]), UNIT),                           # Q2 re-entry
        (cfg(0, 0, 0, 0, 4096, 6), W([2, 2, 4], [4, 4, 1], [0.0, 0.0, 2.5]), UNIT),          # Q2 online
    ]
    g, _ = assert_parity(cases)
    assert [int(g.results["steps"][i]) for i in (0, 2, 3, 4, 5, 6)] == [22, 3, 4, 5, 7, 7]
    assert g.request_times(0)[1][0].tolist() == [2.0 * (k + 1) for k in range(8)] + [20.0, 21.0, 21.0, 22.0]
    assert g.request_times(5)[1][0].tolist() == [4.0, 6.0, 7.0]


def test_grid_w32_all_cells():
    """The W = 32 half of the north-star sweep: 6 presets x {NRF, SRF} x all 121 (I, O) cells (
    P:986: W = 32 never preempts at M = 100K), every output compared with the oracle."""
    vals = workloads.grid_values()
    cases = [(simsweep.preset_config(nm + sfx, 100_000), workloads.fixed(I, O, 32), A100)
             for nm in P.GRID_PRESETS for sfx in ("", "-srf") for I in vals for O in vals]
    g, _ = assert_parity(cases, processes=16)
    assert int(g.results["preemptions"].sum()) == 0


@pytest.mark.parametrize("name", P.GRID_PRESETS)
def test_grid_slice_four_cost_models(name):
    """K = 4 cost models ({8B, 70B} x {A100, H100}) charged on one schedule across a slice of the W = 1024 grid:
    per-request times of every model 0 ULP against the oracle's K = 4 run (fact 2: offline schedules are
    cost-model independent)."""
    cells = [(1, 1), (1, 1024), (16, 256), (128, 1024), (1024, 1), (1024, 1024), (64, 64), (512, 512), (4, 32)]
    cases = [(simsweep.preset_config(name + sfx, 100_000), workloads.fixed(I, O, 1024), K4)
             for sfx in ("", "-srf") for (I, O) in cells]
    assert_parity(cases, processes=9)


def test_holdings_capacity_boundary():
    """M infinite: the int32 KV holdings.  n = 32768 requests of (I, O = 2), S = 131072, C = 2^30 (16384
    prefills per step).  I = 65534: the bound sum(I + O - 1) = 2 147 450 880 < 2^31 -> simulated, equal to the
    oracle (which holds U in int64; its largest U is 2 * 16384 * 65534).  I = 65535 / 65536: the bound reaches
    2^31 -> SIM_S_CAPACITY (include/simsweep.h), no silent wrap."""
    big = 1 << 30
    ok = (cfg(0, 0, 0, 0, big, -1, S=131072), workloads.fixed(65534, 2, 32768), A100)
    g, ors = assert_parity([ok])
    assert int(g.results["sum_U"][0]) == ors[0].sum_U > 2 ** 31
    over = [(cfg(0, 0, 0, 0, big, -1, S=131072), workloads.fixed(I, 2, 32768), A100) for I in (65535, 65536)]
    cfgs = []
    for i, (c, wl, _) in enumerate(over):
        c = simsweep.SimConfig.from_buffer_copy(c)
        c.workload = i
        cfgs.append(c)
    r = simsweep.sim_sweep(cfgs, [w for _, w, _ in over], [simsweep.load_cost_models()[A100[0]]])
    assert [r.status(0), r.status(1)] == ["capacity", "capacity"]
    # the same workloads with a finite M are simulated (U <= M < 2^30)
    fin = (cfg(0, 0, 0, 0, big, 100_000_000, S=131072), workloads.fixed(65536, 2, 32768), A100)
    assert_parity([fin])


def _with_lean(flag, fn):
    import os
    old = os.environ.get("SIMSWEEP_LEAN")
    os.environ["SIMSWEEP_LEAN"] = flag
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["SIMSWEEP_LEAN"]
        else:
            os.environ["SIMSWEEP_LEAN"] = old


@pytest.mark.parametrize("block", range(2))
def test_block_kernel_still_matches(block):
    """The block kernel (sim_step.cuh) keeps every configuration it owns (rank orders, knobs, SRF+Hist, traces);
    with SIMSWEEP_LEAN=0 it also runs the ones the lean kernel owns, so both stay parity-checked on the same
    cases: random contention configs and full-size grid cells against the oracle."""
    cases = []
    for seed in range(12000 + block * 50, 12000 + block * 50 + 50):
        rng = np.random.default_rng(seed)
        Wn = int(rng.integers(8, 600))
        wl = workloads.random_small(seed, Wn, max_len=int(rng.integers(4, 200)), online=bool(rng.integers(0, 2)), S=512)
        o_ = int(rng.integers(0, 2))
        r = int(rng.integers(0, 2))
        chunked = int(rng.integers(0, 2)) if o_ == 1 else 0
        hybrid = int(rng.integers(0, 2))
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        C = int(rng.integers(max(1, peak // 4), 2 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
        M = int(rng.integers(peak, 6 * peak + 1))
        cases.append((cfg(o_, hybrid, chunked, r, C, M, S=512), wl, A100))
    for nm in ("vllm-srf", "sarathi"):
        cases.append((simsweep.preset_config(nm, 100_000), workloads.fixed(128, 1024, 1024), A100))
    g_block, _ = _with_lean("0", lambda: assert_parity(cases))
    g_lean, _ = assert_parity(cases)
    for f in ("steps", "preemptions", "batch_entries", "processed_tokens", "sum_U", "visits"):
        assert np.array_equal(g_block.results[f], g_lean.results[f]), f
    assert g_block.t_done.tobytes() == g_lean.t_done.tobytes()


def test_lean_large_window_azureconv():
    """The lean kernel's arena variant (n > 4096: workload state in the caller's workspace, the waiting bitmap in
    shared memory) on the AzureConv-like trace at full size (N = 19 700) under vLLM / Sarathi x NRF / SRF / PF."""
    wl = workloads.azureconv(2)
    cases = [(simsweep.preset_config(nm, 100_000, S=131072), wl, A100)
             for nm in ("vllm", "vllm-srf", "sarathi", "sarathi-srf", "vllm-pf")]
    assert_parity(cases, processes=len(cases))


_FULL = {}
CRITICAL = ["online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9",
            "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s3",
            "online-70B vllm llama3-70b_a100x4_theoretical M=100000 azureconv s4"]


def _full_oracle_job(i):
    """Simulation i of sweep.full_sweep() on the CPU oracle (the parent builds the sweep before forking)."""
    import oracle as o
    cfgs, wls, ocost = _FULL["sweep"]
    c, w = cfgs[i], wls[cfgs[i].workload]
    oc = o.make_config(c.order, c.hybrid, c.chunked, c.replacement, C=c.C, M=c.M, S=c.S, max_steps=c.max_steps,
                       n_cost=c.n_cost, reserve=c.reserve)
    return i, o.run(oc, w.I, w.O, w.T, [ocost[c.cost[k]] for k in range(c.n_cost)])


def test_full_sweep_bench_launch_sampled():
    """The north-star sweep (BASELINE configs [1]-[5], sweep.full_sweep: 3554 simulations, K = 4 grids, online
    LongForm / AzureConv runs, heterogeneous mixes) in bench.py's launch configuration: one sim_sweep_device call
    over device-resident inputs in LPT order, every kernel variant running concurrently.  Compared with the oracle on
    a sample: every 31st simulation with n <= 4096, and of the AzureConv-size (arena variant) runs the three
    longest-estimated, the measured critical path (bench.py config.critical_path: the 70B A100x4 theoretical runs
    below) and every 40th of the rest; integers bit-exact, per-request times 0 ULP for every cost model, means 1e-9
    relative."""
    import multiprocessing as mp
    import os

    import oracle as o
    import torch

    from paper_2411_07447_b200 import sweep
    from parity import compare

    cfgs, wls, cms, labels = sweep.full_sweep()
    order = sweep.partition_lpt(sweep.estimate(cfgs, wls), 1)[0]
    ds = simsweep.DeviceSweep(cfgs, wls, cms, device="cuda", order=np.asarray(order, np.int32))
    ds.launch()
    torch.cuda.synchronize()
    g = ds.fetch()
    small = [i for i in order if wls[cfgs[i].workload].n <= 4096]
    big = [i for i in order if wls[cfgs[i].workload].n > 4096]
    crit = [i for i in big if " ".join(map(str, labels[i])) in CRITICAL]
    sample = small[::31] + big[:3] + crit + [i for i in big[3::40] if i not in crit]
    ocms = o.load_cost_models()
    names = {bytes(v): k for k, v in simsweep.load_cost_models().items()}
    _FULL["sweep"] = (cfgs, wls, [ocms[names[bytes(c)]] for c in cms])
    jobs = sorted(sample, key=lambda i: -(wls[cfgs[i].workload].n > 4096))  # the long oracle runs first
    with mp.get_context("fork").Pool(min(len(os.sched_getaffinity(0)), len(jobs))) as pool:
        ors = dict(pool.map(_full_oracle_job, jobs, chunksize=1))
    bad = []
    for i in sample:
        bad += compare(g, ors, i, label=" ".join(map(str, labels[i])))
    assert len(crit) == len(CRITICAL) and all(g.status(i) == "ok" for i in crit)
    assert bad == [], "\n".join(bad[:40])


def test_lean_occupancy_knob_keeps_results():
    """sim_set_lean_ctas_per_sm changes only how many simulations share an SM: a grid slice run at 1, 2, 5 per SM
    and the auto rule gives byte-identical results and per-request outputs (and the first one equals the oracle)."""
    cases = [(simsweep.preset_config(nm, 100_000), workloads.fixed(I, O, 1024), A100)
             for nm in ("vllm-srf", "sarathi") for I, O in ((16, 64), (128, 256))]
    outs = []
    try:
        for k in (1, 2, 5, 0):
            simsweep.set_lean_ctas_per_sm(k)
            g, _ = run_case_list(cases) if outs else assert_parity(cases)
            outs.append((g.results.tobytes(), g.t_first.tobytes(), g.t_done.tobytes(), g.n_preempt.tobytes()))
    finally:
        simsweep.set_lean_ctas_per_sm(0)
    assert all(o == outs[0] for o in outs[1:])
