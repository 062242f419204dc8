"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element, on the same seeded inputs.  Integers bit-exact, per-request fp64
times 0 ULP, means within 1e-9 relative."""
import numpy as np
import pytest

from paper_2411_07447_b200 import presets, simsweep, workloads
from parity import compare, run_case_list

pytestmark = pytest.mark.gpu
P = presets
A100 = ["llama3-8b_a100_linear"]
UNIT = [("unit", 1.0)]


def cfg(order, hybrid, chunked, repl, C, M, S=4096, **kw):
    return simsweep.make_config(order, hybrid, chunked, repl, C=C, M=M, S=S, **kw)


def assert_parity(cases, processes=0):
    g, ors = run_case_list(cases, processes=processes)
    bad = []
    for i in range(len(cases)):
        bad += compare(g, ors, i, label=f"case{i}:{cases[i][1].name}")
    assert bad == [], "\n".join(bad[:40])
    return g, ors


def W(I, O, T=None, name="hand"):
    T = [0.0] * len(I) if T is None else T
    return workloads.Workload(np.array(I, np.int32), np.array(O, np.int32), np.array(T, np.float64), name)


def test_hand_traces():
    cases = [
        (cfg(0, 0, 0, 0, 4096, 6), W([2, 2], [4, 4]), UNIT),  # A nrf
        (cfg(0, 0, 0, 1, 4096, 6), W([2, 2], [4, 4]), UNIT),  # A srf
        (cfg(0, 0, 0, 0, 4096, 12), W([1, 1, 5], [6, 6, 4]), UNIT),  # B nrf
        (cfg(0, 0, 0, 1, 4096, 12), W([1, 1, 5], [6, 6, 4]), UNIT),  # B srf
        (cfg(1, 1, 1, 0, 4, -1), W([6, 3], [2, 2]), UNIT),  # C
        (cfg(0, 0, 0, 0, 4, -1), W([6, 3], [2, 2]), UNIT),  # C never fits
        (cfg(0, 0, 0, 0, 4096, -1), W([2, 1], [2, 1], [0.0, 1.5]), UNIT),  # D1
        (cfg(0, 0, 0, 0, 4096, -1), W([1, 1], [1, 1], [0.0, 5.0]), UNIT),  # D2
        (cfg(0, 0, 0, 0, 4096, -1), W([2, 1], [2, 1], [0.0, 2.0]), UNIT),  # D3
        (cfg(0, 0, 0, 2, 1000, 1000), W([10] * 5, [3] * 5), UNIT),  # SRF+Hist trace
        (cfg(0, 0, 0, 0, 4096, 8), W([4, 2, 3], [1, 1, 1]), UNIT),  # Fig. 3
    ]
    for (o_, hy, ch) in [(0, 0, 0), (0, 1, 0), (1, 1, 0), (1, 0, 0), (1, 1, 1)]:  # E
        cases.append((cfg(o_, hy, ch, 0, 4, -1), W([2, 3], [3, 1]), UNIT))
    g, _ = assert_parity(cases)
    assert g.status(5) == "never_fits"


def test_config1_and_presets():
    wl = workloads.fixed(16, 16, 32)
    cases = [(simsweep.preset_config(nm + sfx, 100_000), wl, A100) for nm in P.GRID_PRESETS for sfx in ("", "-srf")]
    g, _ = assert_parity(cases)
    assert all(int(g.results["steps"][i]) == 16 for i in range(len(cases)))


def test_status_codes_and_edges():
    cases = [
        (cfg(0, 0, 0, 0, 4096, -1), W([4096], [2]), UNIT),  # too long
        (cfg(0, 0, 0, 0, 4096, 10), W([8], [4]), UNIT),  # never fits M
        (cfg(1, 1, 1, 0, 4, -1), W([4096], [1]), UNIT),  # chunked long prompt, C = 4
        (cfg(0, 0, 0, 0, 4096, -1, max_steps=2), W([1], [5]), UNIT),  # max steps
        (cfg(1, 1, 1, 1, 1, 50), W([3, 5, 7], [4, 4, 4]), UNIT),  # C = 1
        (cfg(0, 0, 0, 0, 4096, 100_000), W([1], [1]), A100),  # W = 1, O = 1
        (cfg(0, 1, 0, 1, 4096, 100_000), workloads.fixed(1, 1, 1024), A100),  # all O = 1
        (cfg(1, 1, 1, 0, 512, -1), workloads.fixed(1024, 1024, 1024), A100),  # infinite M, max grid cell
        (cfg(0, 0, 0, 1, 4096, 2047), workloads.fixed(1024, 1024, 3), A100),  # M = exactly one peak
    ]
    g, _ = assert_parity(cases)
    assert [g.status(i) for i in range(4)] == ["too_long", "never_fits", "ok", "max_steps"]


@pytest.mark.parametrize("block", range(4))
def test_random_small(block):
    orders_repl = [(o_, r) for o_ in range(5) for r in range(3)]
    cases = []
    for seed in range(block * 100, block * 100 + 100):
        rng = np.random.default_rng(seed)
        Wn = int(rng.integers(1, 40))
        online = bool(rng.integers(0, 2))
        wl = workloads.random_small(seed, Wn, max_len=int(rng.integers(2, 33)), online=online, S=128)
        o_, r = orders_repl[seed % len(orders_repl)]
        chunked = int(rng.integers(0, 2))
        hybrid = int(rng.integers(0, 2)) if o_ < 2 else 1
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        C = int(rng.integers(1, 3 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
        M = -1 if rng.random() < 0.1 else int(rng.integers(peak, 5 * peak + 1))
        names = A100 if rng.random() < 0.5 else ["llama3-70b_h100x4_theoretical"]
        cases.append((cfg(o_, hybrid, chunked, r, C, M, S=128), wl, names))
    assert_parity(cases)


GRID_SAMPLE = [(1, 1), (1, 1024), (1024, 1), (16, 16), (64, 256), (256, 64), (512, 1024), (1024, 1024),
               (4, 512), (128, 1024)]


@pytest.mark.parametrize("name", P.GRID_PRESETS)
def test_grid_w1024_sample(name):
    # BASELINE configs[1] at full size (W = 1024), in the launch configuration bench.py times
    cases = []
    for sfx in ("", "-srf"):
        for (I, O) in GRID_SAMPLE:
            cases.append((simsweep.preset_config(name + sfx, 100_000), workloads.fixed(I, O, 1024), A100))
    assert_parity(cases)


def test_offline_four_cost_models():
    names = ["llama3-8b_a100_linear", "llama3-8b_h100_theoretical", "llama3-70b_a100x4_linear",
             "llama3-70b_h100x4_theoretical"]
    cases = [(simsweep.preset_config(nm, 100_000), workloads.fixed(64, 256, 1024), names)
             for nm in ("vllm", "sarathi-srf")]
    assert_parity(cases)


def test_online_longform_and_hist():
    cases = []
    for seed in (0, 1):
        wl = workloads.longform(seed)
        for nm in ("vllm", "sarathi"):
            for sfx in ("", "-srf", "-srf-hist"):
                cases.append((simsweep.preset_config(nm + sfx, 100_000, S=131072), wl, A100))
    assert_parity(cases)


def test_online_azureconv():
    """BASELINE configs[3] at full size: the AzureConv-like trace (19.7K requests) through
    the 4096-slot ring-buffer variant; every per-request output compared with the oracle."""
    wl = workloads.azureconv(0)
    cases = [(simsweep.preset_config(nm, 100_000, S=131072), wl, A100)
             for nm in ("vllm", "vllm-srf", "sarathi", "sarathi-srf-hist")]
    assert_parity(cases, processes=len(cases))


def test_online_70b_what_ifs():
    wl = workloads.longform(3)
    cases = []
    for cm in ("llama3-70b_a100x4_linear", "llama3-70b_h100x4_theoretical"):
        for sfx in ("", "-srf"):
            for M in (100_000, -1):
                cases.append((simsweep.preset_config("vllm" + sfx, M, S=131072), wl, [cm]))
    assert_parity(cases)


def test_hetero_rank():
    cases = []
    for gen in (lambda s: workloads.sharegpt(s), lambda s: workloads.table_qa(s, long_context=True),
                lambda s: workloads.text_to_sql(s), lambda s: workloads.mix(("LILO", "SILO"), 1024, s)):
        wl = gen(0)
        for nm in ("rank-org", "rank-i", "rank-o"):
            cases.append((simsweep.preset_config(nm, 100_000), wl, A100))
    assert_parity(cases)


def _oracle_grid_job(args):
    name, I, O, M = args
    import oracle as o2
    from paper_2411_07447_b200 import presets as pr
    from paper_2411_07447_b200 import workloads as wk
    p = pr.preset(name)
    wl = wk.fixed(I, O, 1024)
    r = o2.run(o2.make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=p["C"], M=M,
                              reserve=p["reserve"]), wl.I, wl.O, wl.T, o2.load_cost_models()["llama3-8b_a100_linear"])
    return (r.status, [getattr(r, f) for f in ("steps", "preemptions", "batch_entries", "processed_tokens", "sum_U",
                                               "prefill_entries", "idle_jumps", "visits")],
            r.t_first[0].copy(), r.t_done[0].copy(), r.n_preempt.copy(), r.refill.copy(), r.makespan[0])


@pytest.mark.parametrize("M", [100_000])
def test_full_grid_bench_launch(M):
    """BASELINE configs[1] at full size: all 1452 simulations, one sim_sweep_device launch in bench.py's
    configuration (device-resident inputs, LPT order), every output compared with the oracle."""
    import multiprocessing as mp
    import os

    import torch

    from paper_2411_07447_b200 import sweep
    cfgs, wls, cms, labels = sweep.grid_sweep(M=M)
    order = sweep.partition_lpt(sweep.estimate(cfgs, wls), 1)[0]
    ds = simsweep.DeviceSweep(cfgs, wls, cms, device="cuda", order=np.asarray(order, np.int32))
    ds.launch()
    torch.cuda.synchronize()
    g = ds.fetch()
    jobs = [(nm, I, O, M) for (nm, I, O) in labels]
    with mp.get_context("fork").Pool(min(len(os.sched_getaffinity(0)), 64)) as pool:
        ref = pool.map(_oracle_grid_job, jobs, chunksize=4)
    bad = []
    names = ["steps", "preemptions", "batch_entries", "processed_tokens", "sum_U", "prefill_entries", "idle_jumps",
             "visits"]
    for i, (st, ints, tf, td, npre, rf, mk) in enumerate(ref):
        lab = labels[i]
        if g.status(i) != st:
            bad.append(f"{lab} status {g.status(i)} vs {st}")
            continue
        for f, v in zip(names, ints):
            if int(g.results[f][i]) != v:
                bad.append(f"{lab} {f} {int(g.results[f][i])} vs {v}")
        gtf, gtd = g.request_times(i)
        gnp, grf = g.request_counts(i)
        if not (np.array_equal(gtf[0], tf) and np.array_equal(gtd[0], td)):
            bad.append(f"{lab} per-request times differ")
        if not (np.array_equal(gnp, npre) and np.array_equal(grf, rf)):
            bad.append(f"{lab} per-request preemption counts differ")
        if not np.isclose(g.results["makespan"][i][0], mk, rtol=1e-9, atol=0):
            bad.append(f"{lab} makespan")
    assert bad == [], "\n".join(bad[:30])


@pytest.mark.parametrize("block", range(3))
def test_random_medium_contention(block):
    """Larger W and tight M: many preemptions, SRF/NRF, decode-first chunked (R_r^p interleaved with
    R_r^d in the retention order) -- stresses the closed-form decode group."""
    cases = []
    for seed in range(5000 + block * 60, 5000 + block * 60 + 60):
        rng = np.random.default_rng(seed)
        Wn = int(rng.integers(32, 400))
        wl = workloads.random_small(seed, Wn, max_len=int(rng.integers(4, 200)), online=bool(rng.integers(0, 2)),
                                    S=512)
        o_ = int(rng.integers(0, 2))
        r = int(rng.integers(0, 3))
        chunked = int(rng.integers(0, 2))
        hybrid = int(rng.integers(0, 2))
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        C = int(rng.integers(max(1, peak // 4), 2 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
        M = int(rng.integers(peak, 6 * peak + 1))
        cases.append((cfg(o_, hybrid, chunked, r, C, M, S=512), wl, A100))
    assert_parity(cases)


def test_pf_orca_hand_traces():
    """Example A under vLLM^pf (8 sequential steps) and the Orca S-reserve trace (tests/test_oracle_pf.py)."""
    cases = [
        (cfg(0, 0, 0, P.REPL_PF, 4096, 6, reserve=P.RESERVE_PEAK), W([2, 2], [4, 4]), UNIT),
        (cfg(1, 1, 0, P.REPL_PF, 10, 20, S=10, reserve=P.RESERVE_CONTEXT), W([2, 2, 2], [3, 3, 3]), UNIT),
        (simsweep.preset_config("orca", 1000, S=128), workloads.fixed(8, 16, 64), UNIT),
        (simsweep.preset_config("orca", 100, S=128), workloads.fixed(2, 2, 4), UNIT),  # S > M: never fits
    ]
    g, _ = assert_parity(cases)
    assert g.status(3) == "never_fits"
    assert int(g.results["steps"][0]) == 8 and int(g.results["steps"][1]) == 6
    assert int(g.results["preemptions"][:3].sum()) == 0


@pytest.mark.parametrize("name", ["vllm-pf", "sarathi-pf", "sarathi-cs-pf", "sarathi-nocp-pf", "vllm-hy-pf",
                                  "sarathi-nohy-pf", "orca"])
def test_pf_grid_sample(name):
    """E4 (Fig. exp_bin_packing): preemption-free presets on O = W = 1024 plus a spread of
    (I, O), M = 100K -- the PEAK / CONTEXT reserve through the closed-form decode group and the lean loops."""
    cases = [(simsweep.preset_config(name, 100_000), workloads.fixed(I, O, 1024), A100)
             for (I, O) in [(1, 1024), (1024, 1024), (64, 1024), (16, 16), (512, 2), (2, 512), (1, 1), (256, 64)]]
    assert_parity(cases)


def test_varying_M_sweep():
    """E5 (Fig. varying_M): O = 32, W = 1024, M from 100 to 1M, vLLM / Sarathi and their PF
    versions -- the small-M regime where preemption helps and the large-M regime where nothing binds."""
    cases = []
    for nm in ("vllm", "vllm-pf", "sarathi", "sarathi-pf"):
        for M in (100, 1000, 10_000, 1_000_000):
            for I in (8, 64):
                cases.append((simsweep.preset_config(nm, M), workloads.fixed(I, 32, 1024), A100))
    assert_parity(cases)


@pytest.mark.parametrize("block", range(2))
def test_random_pf_contention(block):
    """Random workloads under the PEAK / CONTEXT reserves across all orders, chunking and hybrid settings,
    online and offline, with M tight enough that reserves bind."""
    cases = []
    for seed in range(9000 + block * 60, 9000 + block * 60 + 60):
        rng = np.random.default_rng(seed)
        Wn = int(rng.integers(1, 400))
        S = 512
        wl = workloads.random_small(seed, Wn, max_len=int(rng.integers(4, 200)), online=bool(rng.integers(0, 2)), S=S)
        o_ = int(rng.integers(0, 5))
        res = int(rng.integers(1, 3))
        chunked = int(rng.integers(0, 2))
        hybrid = int(rng.integers(0, 2)) if o_ < 2 else 1
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        C = int(rng.integers(max(1, peak // 4), 2 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
        lo = peak if res == 1 else S
        M = -1 if rng.random() < 0.1 else int(rng.integers(lo, 6 * lo + 1))
        cases.append((cfg(o_, hybrid, chunked, P.REPL_PF, C, M, S=S, reserve=res), wl, A100))
    assert_parity(cases)


def test_large_window_variant():
    """Workloads of n > 4096 requests run the 32768-slot global-arena variant: every order / policy / reserve,
    online and offline, with windows far beyond the 4096-slot shared-memory ring (offline: the whole
    workload is waiting at step 1)."""
    cases = []
    for k, seed in enumerate(range(31_000, 31_012)):
        rng = np.random.default_rng(seed)
        Wn = int(rng.integers(4097, 9000))
        wl = workloads.random_small(seed, Wn, max_len=int(rng.integers(4, 64)), online=bool(k % 2), S=256)
        o_ = k % 5
        r = [0, 1, 1, P.REPL_PF][k % 4] if k != 6 else 2  # SRF+Hist: the oracle's deferral check is O(n) per
        res = (1 + k % 2) if r == P.REPL_PF else 0             # candidate -- one case keeps it affordable
        chunked = int(rng.integers(0, 2))
        hybrid = int(rng.integers(0, 2)) if o_ < 2 else 1
        peak = int((wl.I.astype(int) + wl.O - 1).max())
        C = int(rng.integers(max(1, peak // 2), 4 * peak + 1)) if chunked else int(rng.integers(peak, 4 * peak + 1))
        lo = 256 if res == 2 else peak
        M = int(rng.integers(lo, 20 * lo + 1))
        cases.append((cfg(o_, hybrid, chunked, r, C, M, S=256, reserve=res), wl, A100))
    assert_parity(cases, processes=len(cases))


@pytest.mark.parametrize("block", range(3))
def test_random_knobs(block):
    # alternative readings: head-of-line blocking, max_seqs, KV watermark, on random configs
    from tests_util_knobs import random_knob_case
    cases = []
    for seed in range(block * 80, block * 80 + 80):
        wl, oc, _, knobs = random_knob_case(seed)
        c = cfg(oc.order, oc.hybrid, oc.chunked, oc.replacement, oc.C, oc.M, S=oc.S, **knobs)
        names = A100 if seed % 2 else ["llama3-70b_h100x4_theoretical"]
        cases.append((c, wl, names))
    assert_parity(cases)


def test_knob_hand_traces_and_grid_sample():
    # the oracle's hand traces (tests/test_oracle_knobs.py) and vLLM-like caps on full-size grid cells
    cases = [(cfg(0, 0, 0, 0, 4096, 6, knobs=simsweep.KNOB_HOL), W([2, 5, 1], [3, 1, 1]), UNIT),
             (cfg(0, 0, 0, 0, 4096, -1, max_seqs=2), W([2, 2, 2], [2, 2, 2]), UNIT),
             (cfg(0, 0, 0, 0, 4096, 10, kv_watermark=3), W([4, 4], [2, 2]), UNIT),
             (cfg(0, 0, 0, 0, 4096, 5, knobs=simsweep.KNOB_NRF_ARRIVAL), W([3, 3, 1], [1, 2, 2]), UNIT),
             (cfg(0, 0, 0, 1, 4096, 4, knobs=simsweep.KNOB_SRF_VISIT_ADMISSION), W([1, 2], [3, 3]), UNIT),
             (cfg(0, 0, 0, 0, 4096, 12, kv_block=4), W([4, 4, 1], [2, 2, 1]), UNIT)]
    for name in ("vllm", "sarathi", "vllm-srf", "sarathi-srf"):
        for (I, O) in ((16, 256), (128, 512), (1, 1024)):
            arr = simsweep.KNOB_NRF_ARRIVAL if name == "vllm" else (simsweep.KNOB_SRF_VISIT_ADMISSION if "srf" in name else 0)
            cases.append((simsweep.preset_config(name, 100_000, knobs=simsweep.KNOB_HOL | arr, max_seqs=256,
                                                 kv_watermark=1000), workloads.fixed(I, O, 1024), A100))
            cases.append((simsweep.preset_config(name, 100_000, kv_block=16), workloads.fixed(I, O, 1024), A100))
    g, ors = assert_parity(cases)
    assert [int(g.results["steps"][i]) for i in range(3)] == [4, 4, 4]
    assert g.request_times(3)[1][0].tolist() == [1.0, 3.0, 4.0]
    assert g.request_times(4)[1][0].tolist() == [3.0, 5.0]
    assert g.request_times(5)[1][0].tolist() == [2.0, 3.0, 1.0] and int(g.results["preemptions"][5]) == 1


def test_knobs_on_the_online_traces():
    # the knob kernel instances of the n <= 4096 (LongForm, n = 2000) and global-arena (AzureConv, n = 19 700)
    # variants, with vLLM's system defaults: head-of-line blocking, FCFS running order, max_num_seqs 256, a
    # watermark and blocks of 16 tokens
    lf, az = workloads.longform(5), workloads.azureconv(1)
    vllm_sys = dict(knobs=simsweep.KNOB_HOL | simsweep.KNOB_NRF_ARRIVAL, max_seqs=256, kv_watermark=1000, kv_block=16)
    cases = [(simsweep.preset_config("vllm", 100_000, S=131072, **vllm_sys), lf, A100),
             (simsweep.preset_config("sarathi-srf", 100_000, S=131072, knobs=simsweep.KNOB_SRF_VISIT_ADMISSION,
                                     max_seqs=128, kv_block=16), lf, A100),
             (simsweep.preset_config("vllm", 100_000, S=131072, **vllm_sys), az, A100),
             (simsweep.preset_config("sarathi", 100_000, S=131072, knobs=simsweep.KNOB_HOL, kv_watermark=500), az, A100)]
    g, _ = assert_parity(cases, processes=len(cases))
    assert all(g.status(i) == "ok" for i in range(len(cases)))
