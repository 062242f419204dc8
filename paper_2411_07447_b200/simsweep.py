"""Python binding of libsimsweep.so (include/simsweep.h).  Argument marshalling only.

Every step of the simulation runs in the CUDA kernel; there is no CPU
fallback: if the shared library is missing or no sm_100 device is present the
calls raise.  PyTorch is used only for device memory and streams (the
``DeviceSweep`` path).
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

import numpy as np

from . import presets as _presets
from .workloads import Workload

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("SIMSWEEP_LIB") or os.path.join(PKG, "libsimsweep.so")

SIM_MAX_COST = 4
STATUS = {0: "ok", 1: "too_long", 2: "never_fits", 3: "max_steps", 4: "deadlock", 5: "capacity"}


class SimConfig(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("hybrid", ctypes.c_int32), ("chunked", ctypes.c_int32),
                ("replacement", ctypes.c_int32), ("S", ctypes.c_int32), ("workload", ctypes.c_int32),
                ("C", ctypes.c_int64), ("M", ctypes.c_int64), ("max_steps", ctypes.c_int64),
                ("n_cost", ctypes.c_int32), ("cost", ctypes.c_int32 * SIM_MAX_COST), ("reserve", ctypes.c_int32),
                ("knobs", ctypes.c_int32), ("max_seqs", ctypes.c_int32), ("kv_watermark", ctypes.c_int64),
                ("kv_block", ctypes.c_int32), ("pad", ctypes.c_int32)]


KNOB_HOL = 1  # Q10 alternative: head-of-line blocking of the waiting group
KNOB_NRF_ARRIVAL = 2  # Q6 alternative: NRF retention / running order by arrival (T, id)
KNOB_SRF_VISIT_ADMISSION = 4  # Q3 alternative: SRF visits running requests in admission order


class SimWorkload(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("pad", ctypes.c_int32), ("I", ctypes.c_void_p), ("O", ctypes.c_void_p),
                ("T", ctypes.c_void_p)]


class SimCostModel(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("layers", ctypes.c_int32), ("h", ctypes.c_int32), ("f", ctypes.c_int32),
                ("H", ctypes.c_int32), ("NQ", ctypes.c_int32), ("NKV", ctypes.c_int32), ("e", ctypes.c_int32),
                ("tp", ctypes.c_int32), ("pad", ctypes.c_int32), ("lin", ctypes.c_double * 10),
                ("flops", ctypes.c_double), ("bw", ctypes.c_double), ("link_bw", ctypes.c_double)]


class SimResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("pad", ctypes.c_int32), ("steps", ctypes.c_int64),
                ("preemptions", ctypes.c_int64), ("batch_entries", ctypes.c_int64),
                ("processed_tokens", ctypes.c_int64), ("sum_U", ctypes.c_int64), ("prefill_entries", ctypes.c_int64),
                ("idle_jumps", ctypes.c_int64), ("visits", ctypes.c_int64),
                ("makespan", ctypes.c_double * SIM_MAX_COST),
                ("mean_latency", ctypes.c_double * SIM_MAX_COST), ("mean_ttft", ctypes.c_double * SIM_MAX_COST),
                ("mean_tpot", ctypes.c_double * SIM_MAX_COST), ("formed_steps", ctypes.c_int64)]


class SimBatchShape(ctypes.Structure):
    _fields_ = [("n_p", ctypes.c_int64), ("c", ctypes.c_int64), ("m_p", ctypes.c_int64), ("n_d", ctypes.c_int64),
                ("m_d", ctypes.c_int64)]


class SimSloQuery(ctypes.Structure):
    _fields_ = [("n_p", ctypes.c_int64), ("c", ctypes.c_int64), ("n_d", ctypes.c_int64), ("m_max", ctypes.c_int64),
                ("tau", ctypes.c_double)]


SIM_OPT_MAX_N = 4


class SimOptProblem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("I", ctypes.c_int32 * SIM_OPT_MAX_N), ("O", ctypes.c_int32 * SIM_OPT_MAX_N),
                ("flags", ctypes.c_int32), ("C", ctypes.c_int64), ("M", ctypes.c_int64)]


OPT_NO_PREEMPT = 1  # SIM_OPT_NO_PREEMPT: the optimum over preemption-free schedules


class SimOptResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("rounds", ctypes.c_int32), ("states", ctypes.c_int64),
                ("optimum", ctypes.c_double)]


class SimRequestOut(ctypes.Structure):
    _fields_ = [("t_first", ctypes.c_void_p), ("t_done", ctypes.c_void_p), ("n_preempt", ctypes.c_void_p),
                ("refill_tokens", ctypes.c_void_p)]


class SimTrace(ctypes.Structure):  # == sim_trace_t
    _fields_ = [("steps", ctypes.c_void_p), ("cap_steps", ctypes.c_int64), ("entries", ctypes.c_void_p),
                ("cap_entries", ctypes.c_int64), ("events", ctypes.c_void_p), ("cap_events", ctypes.c_int64),
                ("n_steps", ctypes.c_int64), ("n_entries", ctypes.c_int64), ("n_events", ctypes.c_int64)]


# == sim_trace_step_t / sim_trace_entry_t / sim_trace_event_t
TRACE_STEP_DTYPE = np.dtype([("step", "<i8"), ("n_entries", "<i4"), ("n_events", "<i4"), ("U", "<i8"), ("tok", "<i8"),
                             ("start", "<f8"), ("d", "<f8")])
TRACE_ENTRY_DTYPE = np.dtype([("id", "<i4"), ("phase", "<i4"), ("c", "<i4"), ("m_before", "<i4")])
TRACE_EVENT_DTYPE = np.dtype([("id", "<i4"), ("m", "<i4")])

RESULT_DTYPE = np.dtype([("status", "<i4"), ("pad", "<i4"), ("steps", "<i8"), ("preemptions", "<i8"),
                         ("batch_entries", "<i8"), ("processed_tokens", "<i8"), ("sum_U", "<i8"),
                         ("prefill_entries", "<i8"), ("idle_jumps", "<i8"), ("visits", "<i8"), ("makespan", "<f8", (4,)),
                         ("mean_latency", "<f8", (4,)), ("mean_ttft", "<f8", (4,)), ("mean_tpot", "<f8", (4,)),
                         ("formed_steps", "<i8")])
assert RESULT_DTYPE.itemsize == ctypes.sizeof(SimResult)

_lib = None


def lib() -> ctypes.CDLL:
    """Load libsimsweep.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not found: run `python -m paper_2411_07447_b200.build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        L.sim_sweep.restype = ctypes.c_int
        L.sim_sweep.argtypes = [P(SimConfig), ctypes.c_int32, P(SimWorkload), ctypes.c_int32, P(SimCostModel),
                                ctypes.c_int32, P(SimResult), SimRequestOut, ctypes.c_int32]
        L.sim_sweep_device.restype = ctypes.c_int
        L.sim_sweep_device.argtypes = [P(SimConfig), ctypes.c_int32, P(ctypes.c_int32), ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, SimRequestOut,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.sim_validate.restype = ctypes.c_int
        L.sim_validate.argtypes = [P(SimConfig), ctypes.c_int32, P(SimWorkload), ctypes.c_int32, P(SimCostModel),
                                   ctypes.c_int32]
        L.sim_operator_costs.restype = ctypes.c_int
        L.sim_operator_costs.argtypes = [P(SimCostModel), ctypes.c_int32, P(SimBatchShape), ctypes.c_int32,
                                         ctypes.c_void_p, ctypes.c_int32]
        L.sim_run_traced.restype = ctypes.c_int
        L.sim_run_traced.argtypes = [P(SimConfig), P(SimWorkload), ctypes.c_int32, P(SimCostModel), ctypes.c_int32,
                                     P(SimResult), SimRequestOut, P(SimTrace), ctypes.c_int32]
        L.sim_set_lean_ctas_per_sm.argtypes = [ctypes.c_int32]
        L.sim_workspace_bytes.restype = ctypes.c_int64
        L.sim_workspace_bytes.argtypes = [P(SimConfig), ctypes.c_int32, P(ctypes.c_int32)]
        L.sim_request_rows.restype = ctypes.c_int
        L.sim_request_rows.argtypes = [P(SimConfig), ctypes.c_int32, P(SimWorkload), ctypes.c_int32,
                                       P(ctypes.c_int64), P(ctypes.c_int64)]
        L.sim_batch_times.restype = ctypes.c_int
        L.sim_batch_times.argtypes = [P(SimCostModel), ctypes.c_int32, P(SimBatchShape), ctypes.c_int32,
                                      P(ctypes.c_double), ctypes.c_int32]
        L.sim_slo_frontier.restype = ctypes.c_int
        L.sim_slo_frontier.argtypes = [P(SimCostModel), ctypes.c_int32, P(SimSloQuery), ctypes.c_int32,
                                       P(ctypes.c_int64), ctypes.c_int32]
        L.sim_kv_break_even.restype = ctypes.c_int
        L.sim_kv_break_even.argtypes = [P(SimCostModel), ctypes.c_int32, P(ctypes.c_int64), ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int32]
        L.sim_optimum.restype = ctypes.c_int
        L.sim_optimum.argtypes = [P(SimOptProblem), ctypes.c_int32, P(SimCostModel), P(SimOptResult), ctypes.c_int32]
        L.sim_strerror.restype = ctypes.c_char_p
        L.sim_strerror.argtypes = [ctypes.c_int]
        L.sim_version.restype = ctypes.c_char_p
        L.sim_version.argtypes = []
        _lib = L
    return _lib


EXPORTED_SYMBOLS = ["sim_sweep", "sim_sweep_device", "sim_validate", "sim_run_traced", "sim_workspace_bytes",
                    "sim_request_rows", "sim_strerror", "sim_version", "sim_batch_times", "sim_slo_frontier",
                    "sim_kv_break_even", "sim_operator_costs", "sim_optimum", "sim_set_lean_ctas_per_sm"]


def set_lean_ctas_per_sm(k: int) -> None:
    """sim_set_lean_ctas_per_sm: simulations of the lean n <= 1024 kernel per SM (1..5), 0 = auto (include/simsweep.h)."""
    _check(lib().sim_set_lean_ctas_per_sm(int(k)))


def strerror(code: int) -> str:
    return lib().sim_strerror(code).decode()


class SimError(RuntimeError):
    pass


def _check(rc: int):
    if rc < 0:
        raise SimError(f"simsweep error {rc}: {strerror(rc)}")
    return rc


# ------------------------------------------------------------ cost models
def load_cost_models(path: str | None = None) -> dict:
    """Name -> SimCostModel from the frozen data file (input data, Q23)."""
    path = path or os.path.join(ROOT, "data", "cost_models.json")
    with open(path) as fh:
        doc = json.load(fh)
    out = {}
    for c in doc["cost_models"]:
        m = SimCostModel()
        m.mode = int(c["mode"])
        m.layers, m.h, m.f, m.H = int(c["layers"]), int(c["h"]), int(c["f"]), int(c["H"])
        m.NQ, m.NKV, m.e, m.tp = int(c["NQ"]), int(c["NKV"]), int(c["e"]), int(c["tp"])
        for j, v in enumerate(c["lin"]):
            m.lin[j] = float(v)
        m.flops, m.bw, m.link_bw = float(c["flops"]), float(c["bw"]), float(c["link_bw"])
        out[c["name"]] = m
    return out


def unit_cost(d: float = 1.0) -> SimCostModel:
    """Every batch costs d seconds (linear model, a0 = d, one layer)."""
    m = SimCostModel()
    m.mode, m.layers, m.h, m.f, m.H, m.NQ, m.NKV, m.e, m.tp = 0, 1, 1, 1, 1, 1, 1, 2, 1
    m.lin[0] = d
    m.flops = m.bw = m.link_bw = 1.0
    return m


# ------------------------------------------------------------ configs
def make_config(order, hybrid, chunked, replacement, C, M, S=4096, workload=0, cost=(0,),
                max_steps=10_000_000, reserve=0, knobs=0, max_seqs=0, kv_watermark=0, kv_block=0) -> SimConfig:
    c = SimConfig()
    c.knobs, c.max_seqs, c.kv_watermark, c.kv_block = int(knobs), int(max_seqs), int(kv_watermark), int(kv_block)
    c.order, c.hybrid, c.chunked, c.replacement = int(order), int(bool(hybrid)), int(bool(chunked)), int(replacement)
    c.reserve = int(reserve)
    c.S, c.workload, c.C, c.M, c.max_steps = int(S), int(workload), int(C), int(M), int(max_steps)
    cost = list(cost)
    assert 1 <= len(cost) <= SIM_MAX_COST
    c.n_cost = len(cost)
    for k, v in enumerate(cost):
        c.cost[k] = int(v)
    return c


def preset_config(name: str, M: int, S: int = 4096, workload: int = 0, cost=(0,), **kw) -> SimConfig:
    p = _presets.preset(name, S=S)
    return make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=kw.pop("C", p["C"]), M=M, S=S,
                       workload=workload, cost=cost, reserve=p["reserve"], **kw)


@dataclass
class SweepResult:
    results: np.ndarray  # RESULT_DTYPE [n_cfgs]
    t_first: np.ndarray  # float64 [tim_rows]
    t_done: np.ndarray
    n_preempt: np.ndarray  # int64 [rows]
    refill: np.ndarray
    row_off: np.ndarray
    tim_off: np.ndarray
    n_of: np.ndarray  # n of each config's workload
    k_of: np.ndarray  # n_cost of each config

    def status(self, i: int) -> str:
        return STATUS.get(int(self.results["status"][i]), "?")

    def request_times(self, i: int):
        """-> (t_first [K, n], t_done [K, n]) of config i."""
        n, K, o = int(self.n_of[i]), int(self.k_of[i]), int(self.tim_off[i])
        return self.t_first[o:o + K * n].reshape(K, n), self.t_done[o:o + K * n].reshape(K, n)

    def request_counts(self, i: int):
        n, o = int(self.n_of[i]), int(self.row_off[i])
        return self.n_preempt[o:o + n], self.refill[o:o + n]


def _offsets(cfgs, wls):
    n_of = np.array([wls[c.workload].n for c in cfgs], np.int64)
    k_of = np.array([c.n_cost for c in cfgs], np.int64)
    row_off = np.concatenate([[0], np.cumsum(n_of)[:-1]]).astype(np.int64)
    tim_off = np.concatenate([[0], np.cumsum(n_of * k_of)[:-1]]).astype(np.int64)
    return n_of, k_of, row_off, tim_off, int(n_of.sum()), int((n_of * k_of).sum())


def _cfg_array(cfgs):
    return (SimConfig * len(cfgs))(*cfgs)


def _cm_array(cms):
    return (SimCostModel * len(cms))(*cms)


def alloc_outputs(cfgs, wls, alloc=np.zeros):
    """Output arrays for sim_sweep (alloc may return pinned host memory)."""
    n_of, k_of, row_off, tim_off, rows, trows = _offsets(list(cfgs), wls)
    res = np.frombuffer(alloc(len(cfgs) * RESULT_DTYPE.itemsize, np.uint8).data, RESULT_DTYPE)
    return (res, alloc(trows, np.float64), alloc(trows, np.float64), alloc(rows, np.int64), alloc(rows, np.int64))


def io_bytes(cfgs, wls, n_cms):
    """(H2D, D2H) bytes one sim_sweep call moves (for the e2e accounting)."""
    n_of, k_of, row_off, tim_off, rows, trows = _offsets(list(cfgs), wls)
    n = len(cfgs)
    h2d = (ctypes.sizeof(SimConfig) * n + ctypes.sizeof(SimWorkload) * len(wls) + ctypes.sizeof(SimCostModel) * n_cms
           + 4 * n + 16 * n + sum(16 * w.n for w in wls))
    d2h = RESULT_DTYPE.itemsize * n + 16 * trows + 16 * rows
    return int(h2d), int(d2h)


def _wl_array(wls):
    """sim_workload_t[] over host arrays (returned with the arrays it points into, to keep them alive)."""
    keep = []
    warr = (SimWorkload * len(wls))()
    for j, w in enumerate(wls):
        I = np.ascontiguousarray(w.I, np.int32)
        O = np.ascontiguousarray(w.O, np.int32)
        T = np.ascontiguousarray(w.T, np.float64)
        keep += [I, O, T]
        warr[j].n = int(I.shape[0])
        warr[j].I, warr[j].O, warr[j].T = I.ctypes.data, O.ctypes.data, T.ctypes.data
    return warr, keep


def sim_validate(cfgs, wls: list[Workload], cms) -> None:
    """Host-only validation (the checks sim_sweep makes before touching the device); raises SimError."""
    cfgs = list(cfgs)
    warr, _keep = _wl_array(wls)
    _check(lib().sim_validate(_cfg_array(cfgs), len(cfgs), warr, len(wls), _cm_array(cms), len(cms)))


def sim_sweep(cfgs, wls: list[Workload], cms, device: int = -1, out=None) -> SweepResult:
    """Host-buffer entry point: validates, copies in, simulates, copies out (blocking).
    `out` = alloc_outputs(...) to reuse (e.g. pinned) output buffers."""
    cfgs = list(cfgs)
    n_of, k_of, row_off, tim_off, rows, trows = _offsets(cfgs, wls)
    warr, _keep = _wl_array(wls)
    res, tf, td, npre, rf = out if out is not None else alloc_outputs(cfgs, wls)
    req = SimRequestOut(tf.ctypes.data, td.ctypes.data, npre.ctypes.data, rf.ctypes.data)
    rc = lib().sim_sweep(_cfg_array(cfgs), len(cfgs), warr, len(wls), _cm_array(cms), len(cms),
                         res.ctypes.data_as(ctypes.POINTER(SimResult)), req, int(device))
    _check(rc)
    return SweepResult(res, tf, td, npre, rf, row_off, tim_off, n_of, k_of)


class DeviceSweep:
    """All inputs and outputs resident in device memory (torch tensors); launch()
    enqueues sim_sweep_device on a stream without synchronizing."""

    def __init__(self, cfgs, wls: list[Workload], cms, device="cuda", order=None):
        import torch

        self.torch = torch
        self.cfgs = list(cfgs)
        self.wls = wls
        self.dev = torch.device(device)
        sim_validate(self.cfgs, wls, cms)  # the workload contents too: sim_sweep_device only checks config fields
        n_of, k_of, row_off, tim_off, rows, trows = _offsets(self.cfgs, wls)
        self.n_of, self.k_of, self.row_off_np, self.tim_off_np = n_of, k_of, row_off, tim_off
        self.h_cfgs = _cfg_array(self.cfgs)
        self.h_wls_n = (ctypes.c_int32 * len(wls))(*[w.n for w in wls])
        u8 = lambda a: torch.from_numpy(np.frombuffer(bytes(a), np.uint8).copy()).to(self.dev)
        self.d_cfgs = u8(self.h_cfgs)
        self.d_cms = u8(_cm_array(cms))
        self.n_cms = len(cms)
        self.I = torch.from_numpy(np.concatenate([np.asarray(w.I, np.int32) for w in wls])).to(self.dev)
        self.O = torch.from_numpy(np.concatenate([np.asarray(w.O, np.int32) for w in wls])).to(self.dev)
        self.T = torch.from_numpy(np.concatenate([np.asarray(w.T, np.float64) for w in wls])).to(self.dev)
        warr = (SimWorkload * len(wls))()
        off = 0
        for j, w in enumerate(wls):
            warr[j].n = w.n
            warr[j].I = self.I.data_ptr() + 4 * off
            warr[j].O = self.O.data_ptr() + 4 * off
            warr[j].T = self.T.data_ptr() + 8 * off
            off += w.n
        self.d_wls = u8(warr)
        if order is None:
            order = np.arange(len(self.cfgs))
        self.d_order = torch.from_numpy(np.ascontiguousarray(order, np.int32)).to(self.dev)
        self.d_row_off = torch.from_numpy(row_off).to(self.dev)
        self.d_tim_off = torch.from_numpy(tim_off).to(self.dev)
        self.d_results = torch.zeros(len(self.cfgs) * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=self.dev)
        self.t_first = torch.zeros(trows, dtype=torch.float64, device=self.dev)
        self.t_done = torch.zeros(trows, dtype=torch.float64, device=self.dev)
        self.n_preempt = torch.zeros(rows, dtype=torch.int64, device=self.dev)
        self.refill = torch.zeros(rows, dtype=torch.int64, device=self.dev)
        # state of simulations with n > 4096 requests (a per-CTA arena each); none for the grid sweep
        self.ws_bytes = int(_check(lib().sim_workspace_bytes(self.h_cfgs, len(self.cfgs), self.h_wls_n)))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=self.dev)

    def launch(self, stream=None) -> int:
        """Enqueue the sweep on `stream` (torch.cuda.Stream or None = current); returns #kernel launches."""
        s = stream if stream is not None else self.torch.cuda.current_stream(self.dev)
        req = SimRequestOut(self.t_first.data_ptr(), self.t_done.data_ptr(), self.n_preempt.data_ptr(),
                            self.refill.data_ptr())
        rc = lib().sim_sweep_device(self.h_cfgs, len(self.cfgs), self.h_wls_n, len(self.wls), self.d_cfgs.data_ptr(),
                                    self.d_wls.data_ptr(), self.d_cms.data_ptr(), self.n_cms,
                                    self.d_order.data_ptr(), self.d_row_off.data_ptr(), self.d_tim_off.data_ptr(),
                                    self.d_results.data_ptr(), req, ctypes.c_void_p(self.ws.data_ptr()),
                                    self.ws_bytes, ctypes.c_void_p(s.cuda_stream))
        return _check(rc)

    def fetch(self) -> SweepResult:
        res = np.frombuffer(self.d_results.cpu().numpy().tobytes(), RESULT_DTYPE).copy()
        return SweepResult(res, self.t_first.cpu().numpy(), self.t_done.cpu().numpy(), self.n_preempt.cpu().numpy(),
                           self.refill.cpu().numpy(), self.row_off_np, self.tim_off_np, self.n_of, self.k_of)


@dataclass
class ScheduleLog:
    """The per-step schedule of one simulation (sim_run_traced): record arrays in step order."""
    steps: np.ndarray    # TRACE_STEP_DTYPE [n_steps]
    entries: np.ndarray  # TRACE_ENTRY_DTYPE [sum n_entries], each step's batch in admission order
    events: np.ndarray   # TRACE_EVENT_DTYPE [sum n_events], each step's preemptions in order

    def steps_list(self) -> list:
        """-> [dict(step, U, tok, start, d, entries=[(id, phase, c, m_before)], events=[(id, m)])]."""
        out, p, q = [], 0, 0
        ent = self.entries.tolist()
        ev = self.events.tolist()
        for st in self.steps.tolist():
            j, ne, nv, U, tok, start, d = st
            out.append(dict(step=j, U=U, tok=tok, start=start, d=d, entries=[tuple(x) for x in ent[p:p + ne]],
                            events=[tuple(x) for x in ev[q:q + nv]]))
            p += ne
            q += nv
        return out

    def to_csv(self, fh) -> None:
        """SPEC's ScheduleLog columns: batch,start_s,duration_s,request,phase,c,m_before,event -- one row per batch
        entry, then one row per preemption of that step (phase empty, c = 0, m_before = the discarded m)."""
        fh.write("batch,start_s,duration_s,request,phase,c,m_before,event\n")
        for st in self.steps_list():
            head = f"{st['step']},{st['start']!r},{st['d']!r}"
            for (rid, ph, c, m) in st["entries"]:
                fh.write(f"{head},{rid},{'prefill' if ph else 'decode'},{c},{m},\n")
            for (rid, m) in st["events"]:
                fh.write(f"{head},{rid},,0,{m},preempt\n")


def sim_run_traced(cfg, wls: list[Workload], cms, device: int = -1, caps=(1 << 16, 1 << 20, 1 << 16)):
    """One simulation with its schedule: -> (SweepResult of that one config, ScheduleLog).  Buffers start at
    `caps` (steps, entries, events); a longer log is fetched again with exact sizes."""
    cfgs = [cfg]
    warr, _keep = _wl_array(wls)
    cs, ce, cv = (int(x) for x in caps)
    while True:
        res, tf, td, npre, rf = alloc_outputs(cfgs, wls)
        req = SimRequestOut(tf.ctypes.data, td.ctypes.data, npre.ctypes.data, rf.ctypes.data)
        st = np.zeros(max(cs, 1), TRACE_STEP_DTYPE)
        en = np.zeros(max(ce, 1), TRACE_ENTRY_DTYPE)
        ev = np.zeros(max(cv, 1), TRACE_EVENT_DTYPE)
        tr = SimTrace(st.ctypes.data, cs, en.ctypes.data, ce, ev.ctypes.data, cv, 0, 0, 0)
        _check(lib().sim_run_traced(_cfg_array(cfgs), warr, len(wls), _cm_array(cms), len(cms),
                                    res.ctypes.data_as(ctypes.POINTER(SimResult)), req, ctypes.byref(tr), int(device)))
        if tr.n_steps <= cs and tr.n_entries <= ce and tr.n_events <= cv:
            break
        cs, ce, cv = max(cs, tr.n_steps), max(ce, tr.n_entries), max(cv, tr.n_events)
    n_of, k_of, row_off, tim_off, _, _ = _offsets(cfgs, wls)
    log = ScheduleLog(st[:tr.n_steps].copy(), en[:tr.n_entries].copy(), ev[:tr.n_events].copy())
    return SweepResult(res, tf, td, npre, rf, row_off, tim_off, n_of, k_of), log


def lpt_order(cfgs, wls) -> np.ndarray:
    """Longest-processing-time-first launch order from a step-count estimate."""
    est = []
    for c in cfgs:
        w = wls[c.workload]
        I = np.asarray(w.I, np.float64)
        O = np.asarray(w.O, np.float64)
        Meff = float(max(c.M, 1)) if c.M >= 0 else 1e18
        est.append(O.max() + float(((I + 0.5 * O) * O).sum()) / Meff + float(I.sum()) / float(c.C))
    return np.argsort(-np.asarray(est), kind="stable").astype(np.int32)


# ------------------------------------------------------------ cost-model analytics
def sim_batch_times(cms, shapes, device: int = -1) -> np.ndarray:
    """Batch time of every shape (n_p, c, m_p, n_d, m_d) under every model: float64 [len(cms), len(shapes)].
    `shapes` is any [n, 5] integer array-like (an int64 [n, 5] array is passed without copying)."""
    cms = list(cms)
    arr = np.ascontiguousarray(np.asarray(shapes, np.int64).reshape(-1, 5))  # == sim_batch_shape_t[n]
    n = arr.shape[0]
    out = np.zeros(len(cms) * n, np.float64)
    _check(lib().sim_batch_times(_cm_array(cms), len(cms), arr.ctypes.data_as(ctypes.POINTER(SimBatchShape)), n,
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(device)))
    return out.reshape(len(cms), n)


def sim_slo_frontier(cms, queries, device: int = -1) -> np.ndarray:
    """Largest m with batch time <= tau for every query (n_p, c, n_d, m_max, tau) and model (-1: none):
    int64 [len(cms), len(queries)]."""
    cms = list(cms)
    arr = (SimSloQuery * len(queries))()
    for i, (n_p, c, n_d, m_max, tau) in enumerate(queries):
        arr[i].n_p, arr[i].c, arr[i].n_d, arr[i].m_max, arr[i].tau = int(n_p), int(c), int(n_d), int(m_max), float(tau)
    out = np.zeros(len(cms) * len(queries), np.int64)
    _check(lib().sim_slo_frontier(_cm_array(cms), len(cms), arr, len(queries),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(device)))
    return out.reshape(len(cms), len(queries))


def sim_kv_break_even(cms, N, xfer_bw: float, M: int, device: int = -1):
    """-> (recompute, swap, interval), each float64 [len(cms), len(N)] (seconds)."""
    cms = list(cms)
    Nn = np.ascontiguousarray(N, np.int64)
    outs = [np.zeros(len(cms) * len(Nn), np.float64) for _ in range(3)]
    _check(lib().sim_kv_break_even(_cm_array(cms), len(cms), Nn.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                   len(Nn), float(xfer_bw), int(M), outs[0].ctypes.data, outs[1].ctypes.data,
                                   outs[2].ctypes.data, int(device)))
    return tuple(o.reshape(len(cms), len(Nn)) for o in outs)


OP_NAMES = ["qkv", "o", "gate_up", "down", "attn_prefill", "attn_decode"]  # SIM_OP_* order
OP_COST_DTYPE = np.dtype([("flops", "<i8"), ("rw", "<i8"), ("time", "<f8"), ("intensity", "<f8"), ("bound", "<i4"),
                          ("pad", "<i4")])  # == sim_op_cost_t


def sim_operator_costs(cms, shapes, device: int = -1) -> np.ndarray:
    """Per-operator roofline classification of one layer of every shape (n_p, c, m_p, n_d, m_d)
    under every model: OP_COST_DTYPE [len(cms), len(shapes), 6] (operators in OP_NAMES order; bound 1 = compute,
    0 = memory, -1 = absent)."""
    cms = list(cms)
    arr = np.ascontiguousarray(np.asarray(shapes, np.int64).reshape(-1, 5))
    n = arr.shape[0]
    out = np.zeros(len(cms) * n * len(OP_NAMES), OP_COST_DTYPE)
    _check(lib().sim_operator_costs(_cm_array(cms), len(cms), arr.ctypes.data_as(ctypes.POINTER(SimBatchShape)), n,
                                    out.ctypes.data, int(device)))
    return out.reshape(len(cms), n, len(OP_NAMES))


# ------------------------------------------------------------ exact CSP optimum
OPT_STATUS = {0: "ok", 1: "unreachable", 2: "too_large"}


def sim_optimum(problems, cm: SimCostModel, device: int = -1, no_preempt: bool = False):
    """problems: [(I list, O list, C, M)] -> [(status, rounds, reachable states, optimum seconds)].
    no_preempt: the optimum over preemption-free schedules."""
    arr = (SimOptProblem * len(problems))()
    for q, (I, O, C, M) in enumerate(problems):
        arr[q].flags = OPT_NO_PREEMPT if no_preempt else 0
        assert 1 <= len(I) == len(O) <= SIM_OPT_MAX_N
        arr[q].n = len(I)
        for i, (a, b) in enumerate(zip(I, O)):
            arr[q].I[i], arr[q].O[i] = int(a), int(b)
        arr[q].C, arr[q].M = int(C), int(M)
    out = (SimOptResult * len(problems))()
    _check(lib().sim_optimum(arr, len(problems), ctypes.byref(cm), out, int(device)))
    return [(OPT_STATUS[r.status], int(r.rounds), int(r.states), float(r.optimum)) for r in out]
