"""ORACLE -- test infrastructure only.

ctypes wrapper around ``oracle/liboracle.so`` (plain C++ of Algorithm 1,
see ``oracle/oracle.cpp``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  It does not import the product package, and the product package
never imports it.

Parity status per function:
  oracle_run            pinned: hand traces A-E, closed forms, SPEC S:349,
                        independent log verifier + conservation law, paper
                        invariants (W=32 no preemption, Infinite-M, B <= W)
  oracle_batch_time     pinned: Eq. (1) SPEC example, matmul example,
                        intensity limits 128 / ~2, hand sums
  oracle_hist_predict   pinned: hand-computed histogram examples (Q31)
  oracle_optimum        pinned: single-request and no-contention closed forms, the full reachable-state
                        count, Example A by hand (6 batches vs 8 preemption-free), and the lower bound
                        it must be for every simulated preset (tests/test_oracle_optimum.py)
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

ORDERS = {"prefill_first": 0, "decode_first": 1, "rank_org": 2, "rank_i": 3, "rank_o": 4}
REPLACEMENTS = {"nrf": 0, "srf": 1, "srf_hist": 2, "pf": 3}
RESERVES = {"seq": 0, "peak": 1, "context": 2}
STATUS = {0: "ok", 1: "too_long", 2: "never_fits", 3: "max_steps", 4: "deadlock"}


class OracleConfig(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("hybrid", ctypes.c_int32), ("chunked", ctypes.c_int32),
                ("replacement", ctypes.c_int32), ("S", ctypes.c_int32), ("n_cost", ctypes.c_int32),
                ("C", ctypes.c_int64), ("M", ctypes.c_int64), ("max_steps", ctypes.c_int64),
                ("reserve", ctypes.c_int32), ("knobs", ctypes.c_int32), ("max_seqs", ctypes.c_int32),
                ("kv_block", ctypes.c_int32), ("kv_watermark", ctypes.c_int64)]


KNOB_HOL = 1  # Q10 alternative: head-of-line blocking of the waiting group
KNOB_NRF_ARRIVAL = 2  # Q6 alternative: NRF retention / running order by arrival (T, id)
KNOB_SRF_VISIT_ADMISSION = 4  # Q3 alternative: SRF visits running requests in admission order


class OracleCost(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("layers", ctypes.c_int32), ("h", ctypes.c_int32), ("f", ctypes.c_int32),
                ("H", ctypes.c_int32), ("NQ", ctypes.c_int32), ("NKV", ctypes.c_int32), ("e", ctypes.c_int32),
                ("tp", ctypes.c_int32), ("pad", ctypes.c_int32), ("lin", ctypes.c_double * 10),
                ("flops", ctypes.c_double), ("bw", ctypes.c_double), ("link_bw", ctypes.c_double)]


class OracleSummary(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("pad", ctypes.c_int32), ("steps", ctypes.c_int64),
                ("preemptions", ctypes.c_int64), ("batch_entries", ctypes.c_int64),
                ("processed_tokens", ctypes.c_int64), ("sum_U", ctypes.c_int64), ("prefill_entries", ctypes.c_int64),
                ("idle_jumps", ctypes.c_int64), ("visits", ctypes.c_int64), ("makespan", ctypes.c_double * 4),
                ("mean_latency", ctypes.c_double * 4), ("mean_ttft", ctypes.c_double * 4),
                ("mean_tpot", ctypes.c_double * 4)]


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_run.argtypes = [P(OracleConfig), ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32),
                                    P(ctypes.c_double), P(OracleCost), P(OracleSummary), P(ctypes.c_double),
                                    P(ctypes.c_double), P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_int64),
                                    ctypes.c_int64, P(ctypes.c_double), ctypes.c_int64, P(ctypes.c_int64)]
        _lib.oracle_batch_time.restype = ctypes.c_double
        _lib.oracle_batch_time.argtypes = [P(OracleCost), ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int64),
                                           P(ctypes.c_int32)]
        _lib.oracle_attention_cost.restype = None
        _lib.oracle_attention_cost.argtypes = [ctypes.c_int64] * 6 + [P(ctypes.c_int64), P(ctypes.c_int64)]
        _lib.oracle_matmul_cost.restype = None
        _lib.oracle_matmul_cost.argtypes = [ctypes.c_int64] * 3 + [P(ctypes.c_int64), P(ctypes.c_int64)]
        _lib.oracle_hist_predict.restype = ctypes.c_int64
        _lib.oracle_hist_predict.argtypes = [P(ctypes.c_int32), ctypes.c_int64]
    return _lib


# ---------------------------------------------------------------- cost models
def load_cost_models(path: str | None = None) -> dict:
    """Name -> OracleCost, read from the frozen data file (input data)."""
    path = path or os.path.join(os.path.dirname(_HERE), "data", "cost_models.json")
    with open(path) as fh:
        doc = json.load(fh)
    out = {}
    for c in doc["cost_models"]:
        oc = OracleCost()
        oc.mode = c["mode"]
        for k in ("layers", "h", "f", "H", "NQ", "NKV", "e", "tp"):
            setattr(oc, k, int(c[k]))
        for j, v in enumerate(c["lin"]):
            oc.lin[j] = float(v)
        oc.flops, oc.bw, oc.link_bw = float(c["flops"]), float(c["bw"]), float(c["link_bw"])
        out[c["name"]] = oc
    return out


def unit_cost(d: float = 1.0) -> OracleCost:
    """A linear model with a0 = d and everything else 0, one layer: every batch costs d
    (the SPEC S:349 "unit-cost stub")."""
    oc = OracleCost()
    oc.mode = 0
    oc.layers = 1
    oc.h = oc.f = oc.H = oc.NQ = oc.NKV = 1
    oc.e = 2
    oc.tp = 1
    oc.lin[0] = d
    oc.flops = oc.bw = oc.link_bw = 1.0
    return oc


# ---------------------------------------------------------------- running
@dataclass
class OracleResult:
    status: str
    summary: OracleSummary
    t_first: np.ndarray  # [K, n]
    t_done: np.ndarray
    n_preempt: np.ndarray
    refill: np.ndarray
    trace_i: np.ndarray | None = None
    trace_d: np.ndarray | None = None
    steps_list: list = field(default_factory=list)

    def __getattr__(self, k):
        if k in ("steps", "preemptions", "batch_entries", "processed_tokens", "sum_U", "prefill_entries",
                 "idle_jumps", "visits"):
            return int(getattr(self.summary, k))
        if k in ("makespan", "mean_latency", "mean_ttft", "mean_tpot"):
            return list(getattr(self.summary, k))
        raise AttributeError(k)


def make_config(order, hybrid, chunked, replacement, C, M, S=4096, max_steps=10_000_000, n_cost=1,
                reserve=0, knobs=0, max_seqs=0, kv_watermark=0, kv_block=0) -> OracleConfig:
    c = OracleConfig()
    c.knobs, c.max_seqs, c.kv_watermark, c.kv_block = int(knobs), int(max_seqs), int(kv_watermark), int(kv_block)
    c.order = ORDERS[order] if isinstance(order, str) else int(order)
    c.hybrid, c.chunked = int(bool(hybrid)), int(bool(chunked))
    c.replacement = REPLACEMENTS[replacement] if isinstance(replacement, str) else int(replacement)
    c.S, c.C, c.M, c.max_steps, c.n_cost = int(S), int(C), int(M), int(max_steps), int(n_cost)
    c.reserve = RESERVES[reserve] if isinstance(reserve, str) else int(reserve)
    return c


def run(cfg: OracleConfig, I, O, T, costs, trace: bool = False, trace_cap: int = 1 << 22) -> OracleResult:
    I = np.ascontiguousarray(I, dtype=np.int32)
    O = np.ascontiguousarray(O, dtype=np.int32)
    T = np.ascontiguousarray(T, dtype=np.float64)
    n = int(I.shape[0])
    if not isinstance(costs, (list, tuple)):
        costs = [costs]
    K = len(costs)
    cfg.n_cost = K
    cm_arr = (OracleCost * K)(*costs)
    summ = OracleSummary()
    tf = np.zeros((K, n), np.float64)
    td = np.zeros((K, n), np.float64)
    npre = np.zeros(n, np.int64)
    rf = np.zeros(n, np.int64)
    P = ctypes.POINTER
    if trace:
        ti = np.zeros(trace_cap, np.int64)
        tdd = np.zeros(trace_cap // 4, np.float64)
        lens = np.zeros(2, np.int64)
        ti_p, td_p, lens_p = (ti.ctypes.data_as(P(ctypes.c_int64)), tdd.ctypes.data_as(P(ctypes.c_double)),
                              lens.ctypes.data_as(P(ctypes.c_int64)))
    else:
        ti = tdd = lens = None
        ti_p = td_p = lens_p = None
    rc = lib().oracle_run(ctypes.byref(cfg), n, I.ctypes.data_as(P(ctypes.c_int32)),
                          O.ctypes.data_as(P(ctypes.c_int32)), T.ctypes.data_as(P(ctypes.c_double)), cm_arr,
                          ctypes.byref(summ), tf.ctypes.data_as(P(ctypes.c_double)),
                          td.ctypes.data_as(P(ctypes.c_double)), npre.ctypes.data_as(P(ctypes.c_int64)),
                          rf.ctypes.data_as(P(ctypes.c_int64)), ti_p, trace_cap if trace else 0, td_p,
                          trace_cap // 4 if trace else 0, lens_p)
    if rc != 0:
        raise ValueError(f"oracle_run call error {rc}")
    res = OracleResult(STATUS[summ.status], summ, tf, td, npre, rf)
    if trace:
        if lens[0] < 0:
            raise RuntimeError("oracle trace overflow")
        res.trace_i = ti[: lens[0]].copy()
        res.trace_d = tdd[: lens[1]].copy()
        res.steps_list = parse_trace(res.trace_i, res.trace_d)
    return res


def parse_trace(ti: np.ndarray, td: np.ndarray) -> list:
    """-> list of dict(step, U, tok, start, d, entries=[(id, phase, c, m)], events=[(id, m)])."""
    steps, p, q = [], 0, 0
    while p < len(ti):
        j, ne, nv, U, tok = (int(x) for x in ti[p:p + 5])
        p += 5
        ent = [tuple(int(x) for x in ti[p + 4 * k: p + 4 * k + 4]) for k in range(ne)]
        p += 4 * ne
        ev = [tuple(int(x) for x in ti[p + 2 * k: p + 2 * k + 2]) for k in range(nv)]
        p += 2 * nv
        steps.append(dict(step=j, U=U, tok=tok, start=float(td[q]), d=float(td[q + 1]), entries=ent, events=ev))
        q += 2
    return steps


def batch_time(cost: OracleCost, entries) -> float:
    """entries: iterable of (c, m_before, is_prefill)."""
    entries = list(entries)
    n = len(entries)
    c = np.array([e[0] for e in entries], np.int64)
    m = np.array([e[1] for e in entries], np.int64)
    p = np.array([1 if e[2] else 0 for e in entries], np.int32)
    P = ctypes.POINTER
    return lib().oracle_batch_time(ctypes.byref(cost), n, c.ctypes.data_as(P(ctypes.c_int64)),
                                   m.ctypes.data_as(P(ctypes.c_int64)), p.ctypes.data_as(P(ctypes.c_int32)))


def attention_cost(c, m, B, H, NQ, NKV):
    f, r = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_attention_cost(c, m, B, H, NQ, NKV, ctypes.byref(f), ctypes.byref(r))
    return f.value, r.value


def matmul_cost(c, n_in, n_out):
    f, r = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_matmul_cost(c, n_in, n_out, ctypes.byref(f), ctypes.byref(r))
    return f.value, r.value


class OracleOpt(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("pad", ctypes.c_int32), ("states", ctypes.c_int64),
                ("optimum", ctypes.c_double)]


def optimum(I, O, C: int, M: int, cost: OracleCost, no_preempt: bool = False):
    """Exact CSP optimum (Dijkstra; identical requests merged): -> (status 'ok' | 'unreachable', reachable states,
    min sum_j d_j).  no_preempt: the optimum over preemption-free schedules (e = 0 always)."""
    Ia = np.ascontiguousarray(I, np.int32)
    Oa = np.ascontiguousarray(O, np.int32)
    out = OracleOpt()
    L = lib()
    L.oracle_optimum.restype = ctypes.c_int
    L.oracle_optimum.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                 ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(OracleCost),
                                 ctypes.POINTER(OracleOpt)]
    rc = L.oracle_optimum(len(Ia), Ia.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                          Oa.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(C), int(M), int(bool(no_preempt)),
                          ctypes.byref(cost), ctypes.byref(out))
    if rc < 0:
        raise ValueError(f"oracle_optimum call error {rc}")
    return ("ok" if out.status == 0 else "unreachable"), int(out.states), float(out.optimum)


def hist_predict(hist: np.ndarray, I: int) -> int:
    h = np.ascontiguousarray(hist, dtype=np.int32).reshape(18 * 18)
    return int(lib().oracle_hist_predict(h.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), I))
