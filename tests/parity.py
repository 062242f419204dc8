"""GPU <-> oracle parity helpers (test infrastructure).

Both sides get the SAME seeded workload arrays and the same frozen cost-model
data; configs are mapped field by field.  The bar (north star): integers
bit-exact; fp64 per-request times within 1e-9 relative -- we assert 0 ULP for
per-request times (same expression, same order: DESIGN.md Q36) and 1e-9
relative for the per-simulation means.
"""
from __future__ import annotations

import numpy as np

import oracle as o
from paper_2411_07447_b200 import simsweep

INT_FIELDS = ["steps", "preemptions", "batch_entries", "processed_tokens", "sum_U", "prefill_entries", "idle_jumps", "visits"]
REL_TOL = 1e-9

_OCMS = None
_PCMS = None


def cost_models():
    global _OCMS, _PCMS
    if _OCMS is None:
        _OCMS = o.load_cost_models()
        _PCMS = simsweep.load_cost_models()
    return _OCMS, _PCMS


def oracle_config(c: simsweep.SimConfig) -> o.OracleConfig:
    return o.make_config(c.order, c.hybrid, c.chunked, c.replacement, C=c.C, M=c.M, S=c.S, max_steps=c.max_steps,
                         n_cost=c.n_cost, reserve=c.reserve, knobs=c.knobs, max_seqs=c.max_seqs,
                         kv_watermark=c.kv_watermark, kv_block=c.kv_block)


def _oracle_job(args):
    c, wl, ocost = args
    return o.run(c, wl.I, wl.O, wl.T, ocost)


def run_case_list(cases, device=-1, processes=0):
    """cases: list of (SimConfig, Workload, [cost names or ('unit', d)]).  Runs all cases in ONE sim_sweep
    call (one kernel launch per variant) and the oracle per case (in `processes` forked workers if > 0).
    Returns (gpu SweepResult, [oracle results])."""
    ocms, pcms = cost_models()
    wls, cms_p, cfgs, ors = [], [], [], []
    cm_index = {}

    def cm_idx(name):
        if name not in cm_index:
            cm_index[name] = len(cms_p)
            if isinstance(name, tuple):
                cms_p.append(simsweep.unit_cost(name[1]))
            else:
                cms_p.append(pcms[name])
        return cm_index[name]

    for (cfg, wl, names) in cases:
        c = simsweep.SimConfig.from_buffer_copy(cfg)
        c.workload = len(wls)
        wls.append(wl)
        idx = [cm_idx(nm) for nm in names]
        c.n_cost = len(idx)
        for k, v in enumerate(idx):
            c.cost[k] = v
        cfgs.append(c)
        ocost = [o.unit_cost(nm[1]) if isinstance(nm, tuple) else ocms[nm] for nm in names]
        ors.append((oracle_config(c), wl, ocost))
    if processes > 0:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(processes) as pool:
            ors = pool.map(_oracle_job, ors, chunksize=1)
    else:
        ors = [_oracle_job(a) for a in ors]
    g = simsweep.sim_sweep(cfgs, wls, cms_p, device=device)
    return g, ors


def compare(g, ors, i, label=""):
    """Assert parity of config i; returns a list of mismatch strings (empty = parity)."""
    r = ors[i]
    bad = []
    gs = g.status(i)
    if gs != r.status:
        return [f"{label} status gpu={gs} oracle={r.status}"]
    if gs != "ok":
        return []
    res = g.results[i]
    for f in INT_FIELDS:
        if int(res[f]) != getattr(r, f):
            bad.append(f"{label} {f}: gpu={int(res[f])} oracle={getattr(r, f)}")
    npre, rf = g.request_counts(i)
    if not np.array_equal(npre, r.n_preempt):
        bad.append(f"{label} n_preempt differs at {np.flatnonzero(npre != r.n_preempt)[:5]}")
    if not np.array_equal(rf, r.refill):
        bad.append(f"{label} refill differs at {np.flatnonzero(rf != r.refill)[:5]}")
    tf, td = g.request_times(i)
    if not np.array_equal(tf, r.t_first):
        bad.append(f"{label} t_first differs (max abs {np.abs(tf - r.t_first).max():.3e})")
    if not np.array_equal(td, r.t_done):
        bad.append(f"{label} t_done differs (max abs {np.abs(td - r.t_done).max():.3e})")
    K = r.t_first.shape[0]
    for f in ("makespan", "mean_latency", "mean_ttft", "mean_tpot"):
        a = np.asarray(res[f][:K], np.float64)
        b = np.asarray(getattr(r, f)[:K], np.float64)
        if not np.allclose(a, b, rtol=REL_TOL, atol=0.0):
            bad.append(f"{label} {f}: gpu={a} oracle={b}")
    return bad
