"""The C-ABI library builds, loads and exports every symbol include/simsweep.h
declares; struct layouts agree between the header (compiled with gcc) and the
ctypes binding.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2411_07447_b200 import build, simsweep

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "simsweep.h")


@pytest.fixture(scope="module")
def L():
    build.build()
    return simsweep.lib()


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(sim_\w+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol(L):
    decl = declared_functions()
    assert set(decl) == set(simsweep.EXPORTED_SYMBOLS)
    for name in decl:
        assert hasattr(L, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", simsweep.LIB_PATH], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", nm), name


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "simsweep.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sim_config_t), '
                   'sizeof(sim_workload_t), sizeof(sim_cost_model_t), sizeof(sim_result_t), '
                   'sizeof(sim_request_out_t), offsetof(sim_config_t, n_cost), offsetof(sim_result_t, makespan));'
                   'printf("%zu\\n", offsetof(sim_config_t, reserve));'
                   'printf("%zu %zu %zu\\n", sizeof(sim_batch_shape_t), sizeof(sim_slo_query_t), offsetof(sim_slo_query_t, tau));'
                   'printf("%zu %zu %zu\\n", sizeof(sim_opt_problem_t), offsetof(sim_opt_problem_t, C), sizeof(sim_opt_result_t));'
                   'printf("%zu %zu %zu %zu %zu\\n", sizeof(sim_trace_step_t), offsetof(sim_trace_step_t, start), '
                   'sizeof(sim_trace_entry_t), sizeof(sim_trace_event_t), sizeof(sim_trace_t));'
                   'printf("%zu %zu\\n", sizeof(sim_op_cost_t), offsetof(sim_op_cost_t, bound));'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(simsweep.SimConfig), ctypes.sizeof(simsweep.SimWorkload),
            ctypes.sizeof(simsweep.SimCostModel), ctypes.sizeof(simsweep.SimResult),
            ctypes.sizeof(simsweep.SimRequestOut), simsweep.SimConfig.n_cost.offset,
            simsweep.SimResult.makespan.offset, simsweep.SimConfig.reserve.offset,
            ctypes.sizeof(simsweep.SimBatchShape), ctypes.sizeof(simsweep.SimSloQuery), simsweep.SimSloQuery.tau.offset,
            ctypes.sizeof(simsweep.SimOptProblem), simsweep.SimOptProblem.C.offset, ctypes.sizeof(simsweep.SimOptResult),
            simsweep.TRACE_STEP_DTYPE.itemsize, simsweep.TRACE_STEP_DTYPE.fields["start"][1],
            simsweep.TRACE_ENTRY_DTYPE.itemsize, simsweep.TRACE_EVENT_DTYPE.itemsize, ctypes.sizeof(simsweep.SimTrace),
            simsweep.OP_COST_DTYPE.itemsize, simsweep.OP_COST_DTYPE.fields["bound"][1]]
    assert got == want
    assert got[0] == 96 and got[-7:] == [48, 32, 16, 8, 72, 40, 32]


def test_version_and_strerror(L):
    assert b"sm_100a" in L.sim_version()
    assert simsweep.strerror(-1).startswith("invalid")
    assert simsweep.strerror(-5).startswith("no sm_100")


def test_request_rows_host_helper(L):
    from paper_2411_07447_b200 import workloads
    wls = [workloads.fixed(4, 4, 10), workloads.fixed(2, 2, 3)]
    cfgs = [simsweep.preset_config("vllm", 100, workload=0, cost=(0, 1)),
            simsweep.preset_config("sarathi", 100, workload=1)]
    warr = (simsweep.SimWorkload * 2)()
    for j, w in enumerate(wls):
        warr[j].n = w.n
    r, t = ctypes.c_int64(), ctypes.c_int64()
    rc = L.sim_request_rows((simsweep.SimConfig * 2)(*cfgs), 2, warr, 2, ctypes.byref(r), ctypes.byref(t))
    assert rc == 0 and (r.value, t.value) == (13, 23)
    cfgs[0].workload = 7
    assert L.sim_request_rows((simsweep.SimConfig * 2)(*cfgs), 2, warr, 2, ctypes.byref(r), ctypes.byref(t)) == -1


def test_no_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2411_07447_b200 import workloads
    wl = workloads.fixed(2, 2, 4)
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_sweep([simsweep.preset_config("vllm", 100)], [wl], [simsweep.unit_cost()])
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_batch_times([simsweep.unit_cost()], [(1, 1, 0, 0, 0)])
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_slo_frontier([simsweep.unit_cost()], [(1, 1, 1, 10, 1.0)])
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_kv_break_even([simsweep.unit_cost()], [4], 64e9, 100)
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_optimum([([2, 2], [4, 4], 4096, 6)], simsweep.unit_cost())
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_operator_costs([simsweep.unit_cost()], [(1, 1, 0, 0, 0)])
    with pytest.raises(simsweep.SimError, match="no sm_100"):
        simsweep.sim_run_traced(simsweep.preset_config("vllm", 100), [wl], [simsweep.unit_cost()])


def test_invalid_calls_rejected_before_device(L):
    from paper_2411_07447_b200 import workloads
    wl = workloads.fixed(2, 2, 4)
    bad = simsweep.preset_config("vllm", 100)
    bad.order = 9
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_sweep([bad], [wl], [simsweep.unit_cost()])
    wl2 = workloads.Workload(np.array([1, 1], np.int32), np.array([1, 1], np.int32), np.array([1.0, 0.0]))
    with pytest.raises(simsweep.SimError, match="invalid workload"):
        simsweep.sim_sweep([simsweep.preset_config("vllm", 100)], [wl2], [simsweep.unit_cost()])
    with pytest.raises(simsweep.SimError, match="cost"):
        simsweep.sim_sweep([simsweep.preset_config("vllm", 100, cost=(3,))], [wl], [simsweep.unit_cost()])
    with pytest.raises(simsweep.SimError, match="invalid argument"):  # analytics: shapes checked on the host
        simsweep.sim_batch_times([simsweep.unit_cost()], [(0, 1, 0, 0, 0)])
    bad_cm = simsweep.unit_cost()
    bad_cm.mode = 7
    with pytest.raises(simsweep.SimError, match="cost"):
        simsweep.sim_slo_frontier([bad_cm], [(1, 1, 1, 10, 1.0)])
    # the schedule trace: a NULL trace, negative or unbacked capacities, a bad config -- before any device work
    cfgs = simsweep._cfg_array([simsweep.preset_config("vllm", 100)])
    warr, _keep = simsweep._wl_array([wl])
    cm = simsweep._cm_array([simsweep.unit_cost()])
    res = np.zeros(1, simsweep.RESULT_DTYPE)
    req = simsweep.SimRequestOut(None, None, None, None)
    rp = res.ctypes.data_as(ctypes.POINTER(simsweep.SimResult))
    assert L.sim_run_traced(cfgs, warr, 1, cm, 1, rp, req, None, -1) == -1
    for tr in (simsweep.SimTrace(None, -1, None, 0, None, 0, 0, 0, 0), simsweep.SimTrace(None, 4, None, 0, None, 0, 0, 0, 0)):
        assert L.sim_run_traced(cfgs, warr, 1, cm, 1, rp, req, ctypes.byref(tr), -1) == -1
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_run_traced(bad, [wl], [simsweep.unit_cost()])
    with pytest.raises(simsweep.SimError, match="invalid argument"):  # the optimum: C >= 1
        simsweep.sim_optimum([([2], [2], 0, 6)], simsweep.unit_cost())


def test_workspace_bytes_host_query(L):
    """sim_workspace_bytes is host-only: 0 for workloads of <= 4096 requests, a header plus one arena per
    simulation of a larger workload; sim_sweep_device rejects a missing workspace before touching the GPU."""
    from paper_2411_07447_b200 import workloads
    small = [simsweep.preset_config("vllm", 100_000, workload=0)]
    n = (ctypes.c_int32 * 2)(1024, 19_700)
    assert L.sim_workspace_bytes(simsweep._cfg_array(small), 1, n) == 0
    big = [simsweep.preset_config(nm, 100_000, workload=1) for nm in ("vllm", "sarathi", "vllm-pf")]
    b1 = L.sim_workspace_bytes(simsweep._cfg_array(big[:1]), 1, n)
    b3 = L.sim_workspace_bytes(simsweep._cfg_array(big), 3, n)
    assert b1 > 32768 * 51 and b3 - 256 == 3 * (b1 - 256)
    assert L.sim_workspace_bytes(None, 1, n) == -1
    req = simsweep.SimRequestOut(1, 1, 1, 1)
    rc = L.sim_sweep_device(simsweep._cfg_array(big), 3, n, 2, 1, 1, 1, 1, None, 1, 1, 1, req, None, 0, None)
    assert rc == -1


def test_device_entry_validates_configs(L):
    """sim_sweep_device checks every config field it can without the workload contents (enums, knob
    bits, C, M, S, n_cost, workload and cost indices) and returns SIM_EINVAL / SIM_ECOST before any device work;
    a valid call with dummy (non-NULL) device pointers would launch, so only rejected calls are made here."""
    n = (ctypes.c_int32 * 2)(16, 16)
    req = simsweep.SimRequestOut(1, 1, 1, 1)

    def call(c, n_wls=2, n_cms=1):
        return L.sim_sweep_device(simsweep._cfg_array([c]), 1, n, n_wls, 1, 1, 1, n_cms, None, 1, 1, 1, req, None, 0,
                                  None)

    def mk(**kw):
        c = simsweep.preset_config("vllm", 1000)
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    for bad in (mk(workload=-1), mk(workload=2), mk(order=5), mk(replacement=4), mk(knobs=8), mk(C=0),
                mk(C=(1 << 30) + 1), mk(M=(1 << 30) + 1), mk(S=0), mk(n_cost=0), mk(n_cost=5), mk(hybrid=2),
                mk(replacement=3), mk(kv_block=-1), mk(max_seqs=-1)):
        assert call(bad) == -1
    c = mk()
    c.cost[0] = 1
    assert call(c) == -3  # cost index out of range (n_cms = 1)
    assert call(mk(), n_wls=0) == -1


def test_sim_validate_host_checks(L):
    from paper_2411_07447_b200 import workloads
    wl = workloads.fixed(2, 2, 4)
    simsweep.sim_validate([simsweep.preset_config("vllm", 100)], [wl], [simsweep.unit_cost()])  # ok: no raise
    online = workloads.Workload(np.array([1, 1], np.int32), np.array([1, 1], np.int32), np.array([0.0, 1.0]))
    with pytest.raises(simsweep.SimError, match="invalid workload"):  # n_cost > 1 needs an offline workload
        simsweep.sim_validate([simsweep.preset_config("vllm", 100, cost=(0, 0))], [online], [simsweep.unit_cost()])
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_validate([simsweep.preset_config("vllm", 100, workload=-1)], [wl], [simsweep.unit_cost()])


def test_operator_costs_rejects_bad_input(L):
    cm = simsweep.load_cost_models()["llama3-8b_a100_theoretical"]
    with pytest.raises(simsweep.SimError, match="invalid argument"):
        simsweep.sim_operator_costs([cm], [(0, 1, 0, 0, 0)])
    bad = simsweep.unit_cost()
    bad.bw = 0.0
    with pytest.raises(simsweep.SimError, match="cost"):
        simsweep.sim_operator_costs([bad], [(1, 1, 0, 0, 0)])


def test_lean_ctas_per_sm_setter(L):
    """sim_set_lean_ctas_per_sm is host-only: 0 (auto) .. 5 accepted, anything else SIM_EINVAL."""
    for k in range(6):
        assert L.sim_set_lean_ctas_per_sm(k) == 0
    assert L.sim_set_lean_ctas_per_sm(-1) == -1  # SIM_EINVAL
    assert L.sim_set_lean_ctas_per_sm(6) == -1
    assert L.sim_set_lean_ctas_per_sm(0) == 0
    with pytest.raises(simsweep.SimError):
        simsweep.set_lean_ctas_per_sm(9)
