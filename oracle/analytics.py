"""ORACLE -- test infrastructure only: cost-model analytics, written from the definitions.

Every batch time comes from ``oracle.batch_time`` over an EXPLICIT list of entries (the C++ oracle's
Eq. (1)-(3) / linear model, pinned in tests/test_oracle_cost.py); nothing here shares code with the CUDA path.

  shape_time       d of n_p prefill entries (c, m_p) and n_d decode entries (m_d)
  slo_frontier     max{m in [0, m_max] : d(n_p prefills (c, m), n_d decodes (m)) <= tau}  (Fig. SLO,
                   PAPER.md:567-600; tau = the paper's 1 s TPOT threshold, :574).  Reading (Q41):
                   prefills and decodes share one m.  The definition is a scan over m (slo_frontier_scan);
                   slo_frontier bisects, valid because d is non-decreasing in m (pinned by a property test)
  operator_costs   per operator of Eq. (3) for one layer of a shape: FLOPs, RW elements, time, intensity FLOPs/RW,
                   compute- or memory-bound ("What Makes a Batch Compute-Bound?"), from the
                   oracle's own matmul_cost / attention_cost (Eq. (1)-(2)) summed per request
                   with B = 1 (reading Q24)
  kv_break_even    recompute = d(one prefill entry c = N, m = 0); swap = N * 2 * layers * NKV * H * e / xfer_bw
                   (K and V over the host link); interval = recompute / N * M, the break-even
                   interval t^N_recom M / N of Eq. (9)

Pins (tests/test_oracle_analytics.py): the paper's own arithmetic for Eq. (9) ([3.3e-6, 1.3e-3] s/KV at
M = 100K -> [0.33, 130] s); closed-form frontiers of the linear model; scan == bisection;
monotonicity; swap cheaper than recompute for few KVs, recompute cheaper for many;
intervals decreasing in N ("KVs of longer requests have smaller break-even intervals", :274).
"""
from __future__ import annotations

import oracle as _o


def shape_entries(n_p: int, c: int, m_p: int, n_d: int, m_d: int):
    return [(c, m_p, True)] * int(n_p) + [(1, m_d, False)] * int(n_d)


def shape_time(cost, n_p: int, c: int, m_p: int, n_d: int, m_d: int) -> float:
    return _o.batch_time(cost, shape_entries(n_p, c, m_p, n_d, m_d))


def slo_frontier_scan(cost, n_p: int, c: int, n_d: int, m_max: int, tau: float) -> int:
    """The definition: the largest m in [0, m_max] with d <= tau, or -1 (a plain scan; small m_max only)."""
    best = -1
    for m in range(m_max + 1):
        if shape_time(cost, n_p, c, m, n_d, m) <= tau:
            best = m
    return best


def slo_frontier(cost, n_p: int, c: int, n_d: int, m_max: int, tau: float) -> int:
    """Same value as slo_frontier_scan, by bisection over the non-decreasing d(m)."""
    ok = lambda m: shape_time(cost, n_p, c, m, n_d, m) <= tau  # noqa: E731
    if not ok(0):
        return -1
    lo, hi = 0, m_max + 1
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if ok(mid):
            lo = mid
        else:
            hi = mid
    return lo


def kv_bytes_per_token(cost) -> int:
    """K and V of one token over all layers: 2 * layers * N_KV * H elements of e bytes (Q26)."""
    return 2 * cost.layers * cost.NKV * cost.H * cost.e


def kv_break_even(cost, N: int, xfer_bw: float, M: int):
    """-> (recompute, swap, interval) in seconds for N KVs of one request."""
    t = shape_time(cost, 1, N, 0, 0, 0)
    swap = float(N * kv_bytes_per_token(cost)) / float(xfer_bw)
    return t, swap, (t / float(N)) * float(M)


OPS = ["qkv", "o", "gate_up", "down", "attn_prefill", "attn_decode"]


def _roof(F: int, R: int, cost):
    """Eq. (3): max(FLOPs / GPU_FLOPS, RW / GPU_bandwidth), RW bytes = e * elements (Q26).
    -> (time, compute_bound)."""
    tc = float(F) / cost.flops
    tm = float(R * cost.e) / cost.bw
    return max(tc, tm), tc > tm


def operator_costs(cost, n_p: int, c: int, m_p: int, n_d: int, m_d: int) -> list:
    """-> [dict(op, flops, rw, time, intensity, bound)] for one layer, ops in OPS order.  bound: 1 compute-bound,
    0 memory-bound, -1 absent (no entry of that phase)."""
    N = n_p * c + n_d  # tokens of the batch (the matmuls' c)
    h, f, H, NQ, NKV = cost.h, cost.f, cost.H, cost.NQ, cost.NKV
    mats = [(h, (NQ + 2 * NKV) * H), (NQ * H, h), (h, 2 * f), (f, h)]  # QKV, O, gate+up (SwiGLU, Q27), down
    out = []
    for name, (din, dout) in zip(OPS[:4], mats):
        F, R = _o.matmul_cost(N, din, dout)
        out.append((name, F, R))
    for name, (nb, cc, mm) in ((OPS[4], (n_p, c, m_p)), (OPS[5], (n_d, 1, m_d))):
        if nb == 0:
            out.append((name, None, None))
            continue
        F1, R1 = _o.attention_cost(cc, mm, 1, H, NQ, NKV)  # one request, B = 1 (Q24); identical entries add up
        out.append((name, nb * F1, nb * R1))
    res = []
    for name, F, R in out:
        if F is None:
            res.append(dict(op=name, flops=0, rw=0, time=0.0, intensity=0.0, bound=-1))
            continue
        t, cb = _roof(F, R, cost)
        res.append(dict(op=name, flops=F, rw=R, time=t, intensity=(float(F) / float(R)) if R > 0 else 0.0,
                        bound=1 if cb else 0))
    return res
