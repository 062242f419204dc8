"""The paper's CSP experiment shape: O = W = 4, M = max(2I, I + O - 1), exact optimum on the GPU
(sim_optimum) next to the best simulated preset, its preemption-free version and the oracle's Dijkstra time on the
small instances.   python tools/optimum_bench.py [I ...]     (GPU box)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as o  # noqa: E402
from paper_2411_07447_b200 import presets, simsweep, workloads  # noqa: E402

cm_name = "llama3-8b_a100_theoretical"
pc = simsweep.load_cost_models()[cm_name]
oc = o.load_cost_models()[cm_name]
Is = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16, 32, 64]
simsweep.sim_optimum([([1], [1], 1, 1)], pc)  # warm
print(f"{'I':>3} {'M':>4} {'states':>10} {'rounds':>6} {'gpu_ms':>8} {'oracle_ms':>9} {'optimum':>10} {'opt_free':>10} "
      f"{'best':>10} {'best_pf':>10}  opt/best  opt/pf  opt/free")
for I in Is:
    M = max(2 * I, I + 3)
    t0 = time.perf_counter()
    st, rounds, states, opt = simsweep.sim_optimum([([I] * 4, [4] * 4, 4096, M)], pc)[0]
    t1 = time.perf_counter()
    _, _, _, free = simsweep.sim_optimum([([I] * 4, [4] * 4, 4096, M)], pc, no_preempt=True)[0]
    ot = float("nan")
    if states < 300_000:
        t2 = time.perf_counter()
        ost, ostates, oopt = o.optimum([I] * 4, [4] * 4, 4096, M, oc)
        ot = 1e3 * (time.perf_counter() - t2)
        assert (ost, ostates, oopt) == (st, states, opt)
    names = [n + p for n in presets.GRID_PRESETS for p in ("", "-srf")]
    pf = [n + "-pf" for n in presets.GRID_PRESETS]
    g = simsweep.sim_sweep([simsweep.preset_config(n, M) for n in names + pf], [workloads.fixed(I, 4, 4)], [pc])
    ms = [float(g.results["makespan"][i][0]) if g.status(i) == "ok" else float("inf") for i in range(len(names + pf))]
    best, best_pf = min(ms[:len(names)]), min(ms[len(names):])
    print(f"{I:3d} {M:4d} {states:10d} {rounds:6d} {1e3 * (t1 - t0):8.1f} {ot:9.1f} {opt:10.6f} {free:10.6f} {best:10.6f} "
          f"{best_pf:10.6f}  {opt / best:8.4f} {opt / best_pf:7.4f} {opt / free:8.4f}", flush=True)
