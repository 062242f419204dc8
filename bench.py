#!/usr/bin/env python
"""bench.py -- simulated scheduler steps/s of the B200 step-level simulator.

One bench STEP = one pass of the whole hot path (rows a1-a12) over one sweep:

* --workload grid (default): BASELINE configs[1], the high-contention grid -- 6 schedulers x I, O in
  {1, 2, ..., 1024} x W = 1024 x {NRF, SRF}, A100 Llama-3-8B linear cost model, KV recomputation, M = 100 000
  (1 452 simulations);
* --workload full: the north-star sweep, configs [1]-[5] (sweep.full_sweep: both grids with K = 4 cost models,
  the online LongForm / AzureConv traces x 10 seeds with the 8B and 70B variants, the heterogeneous mixes with
  the rank orders; 3 554 simulations, 12 266 configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload grid|full] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): STRONG scaling -- the one sweep is LPT-sharded over the ranks
(sweep.ShardedSweep), each rank simulates its shard and all outputs (result rows + per-request slabs) are gathered
to rank 0 by one all_gather over NVLink inside the timed step; value = steps of the sweep / max-over-ranks time.
The floor is the longest single simulation (a dependent chain of steps), reported as config.critical_path.
--impl reference times the CPU oracle (oracle/, the only other thing this file may run) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated scheduler steps/sec (sweep configs/sec in config) vs host oracle"
UNIT = "steps/s"
DTYPE = "i32+f64"  # integer state machine; fp64 only for time
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2: flushed between timed iterations
SM_COUNT = 148
INT_LANES_PER_SM_CLK = 128  # 4 SMSPs x (16 alu + 16 fma-pipe int lanes) per clock (B300_MICROARCH "Pipe rates")
OPS_PER_VISIT = 10  # algorithmic int ops per candidate visit
OPS_PER_ENTRY = 12  # algorithmic int ops per batch entry (Eq. 6 update + features)


def _env_dist():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def build_sweep(workload: str):
    """-> (cfgs, wls, cms, labels, config description)."""
    from paper_2411_07447_b200 import sweep

    if workload == "grid":
        cfgs, wls, cms, labels = sweep.grid_sweep(M=100_000)
        desc = {"workload": "BASELINE configs[1] grid: 6 presets (vllm, sarathi, sarathi-cs, sarathi-nocp, vllm-hy, "
                            "sarathi-nohy) x I,O in {1..1024 pow2} x W=1024 x {NRF,SRF} = 1452 simulations, "
                            "llama3-8b A100 linear cost model, M=100000, offline; LPT-sharded over the GPUs",
                "simulations": len(cfgs), "configs": len(cfgs), "W": 1024, "S": 4096, "M": 100_000}
    else:
        cfgs, wls, cms, labels = sweep.full_sweep()
        desc = {"workload": "north-star sweep, BASELINE configs[1]-[5]: grids W in {32,1024} x 6 presets x "
                            "{NRF,SRF} x 121 (I,O) cells, each schedule under K=4 cost models (8B/70B x A100/H100 "
                            "linear); online LongForm-like and AzureConv-like traces x 10 seeds x {vllm C=S, sarathi "
                            "C=512} x {NRF,SRF,SRF+Hist} (8B/A100) and x 70B {A100x4,H100x4} x {linear,theoretical} "
                            "x {NRF,SRF} x {M=100000, infinite}; heterogeneous mixes (ShareGPT, table-QA, "
                            "text-to-SQL, long-context variants, App. D pairs) x 10 seeds x Rank_org/I/O",
                "simulations": len(cfgs), "configs": int(sum(c.n_cost for c in cfgs)), "M": 100_000}
    desc["l2"] = "flushed between timed iterations (256 MiB)"
    return cfgs, wls, cms, labels, desc


# ---------------------------------------------------------------- oracle (CPU) legs
_SWEEP_CACHE = {}


def _oracle_job(args):
    """Simulation i of the sweep on the CPU oracle (the worker rebuilds the same seeded sweep once)."""
    workload, i = args
    import oracle as o
    from paper_2411_07447_b200 import simsweep

    if workload not in _SWEEP_CACHE:
        cfgs, wls, cms, labels, _ = build_sweep(workload)
        ocms = o.load_cost_models()
        names = {bytes(v): k for k, v in simsweep.load_cost_models().items()}
        _SWEEP_CACHE[workload] = (cfgs, wls, [ocms[names[bytes(c)]] for c in cms])
    cfgs, wls, ocost = _SWEEP_CACHE[workload]
    c = cfgs[i]
    w = wls[c.workload]
    oc = o.make_config(c.order, c.hybrid, c.chunked, c.replacement, C=c.C, M=c.M, S=c.S, max_steps=c.max_steps,
                       reserve=c.reserve)
    r = o.run(oc, w.I, w.O, w.T, [ocost[c.cost[k]] for k in range(c.n_cost)])
    return r.steps, r.batch_entries


def run_oracle(workload, idx, cores: int):
    import multiprocessing as mp

    import oracle

    oracle.build()
    jobs = [(workload, int(i)) for i in idx]
    t0 = time.perf_counter()
    if cores > 1:
        with mp.get_context("fork").Pool(cores) as pool:
            out = pool.map(_oracle_job, jobs, chunksize=1)
    else:
        out = [_oracle_job(j) for j in jobs]
    dt = time.perf_counter() - t0
    return sum(s for s, _ in out), dt


def oracle_list(workload: str, cfgs, wls):
    """The simulations the oracle legs run: the whole list for the grid; for the north-star sweep (whose online
    AzureConv runs take the oracle minutes each) a bounded stratified sample, longest-estimated first."""
    from paper_2411_07447_b200 import sweep

    order = list(sweep.partition_lpt(sweep.estimate(cfgs, wls), 1)[0])
    if workload == "grid":
        return order, f"the full list ({len(order)} simulations)"
    n_big = sum(1 for c in cfgs if wls[c.workload].n > 4096)
    pick = [i for i in order if wls[cfgs[i].workload].n <= 4096][::8]
    return pick, (f"every 8th simulation (LPT order) of the {len(order) - n_big} with n <= 4096 requests "
                  f"({len(pick)} simulations); the {n_big} AzureConv-size runs are left out (minutes each)")


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def bench_reference(args, rank, world):
    if rank != 0:
        return 0
    cfgs, wls, cms, labels, desc = build_sweep(args.workload)
    idx, sample = oracle_list(args.workload, cfgs, wls)
    cores = min(host_cores(), len(idx))
    for _ in range(args.warmup):
        run_oracle(args.workload, idx[: max(1, len(idx) // 16)], cores)
    times, steps = [], 0
    for _ in range(args.steps):
        s, dt = run_oracle(args.workload, idx, cores)
        times.append(dt)
        steps = s
    ms = 1000.0 * statistics.mean(times)
    value = steps / (ms / 1000.0)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": desc | {"reference": "CPU oracle (oracle/oracle.cpp, g++ -O2), multiprocessing over simulations"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{sample}, all {cores} host cores"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for ln in open(self.path):
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [x for x in sm if x > 500] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


# ---------------------------------------------------------------- our arm
def bench_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_07447_b200 import simsweep, sweep

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfgs, wls, cms, labels, desc = build_sweep(args.workload)
    # ONE sweep, LPT-sharded over the ranks (strong scaling); each shard longest-first on its GPU
    sh = sweep.ShardedSweep(cfgs, wls, cms, device=dev)
    order = sh.mine
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def one_step():
        n = sh.launch(stream)
        if world > 1:  # a12: the only collective -- all outputs (rows + per-request slabs) to rank 0 over NVLink
            with torch.cuda.stream(stream):
                sh.gather()
        return n

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_step()
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    ev = []
    launches = 0
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            launches += sh.launch(stream)
            e1.record(stream)
            if world > 1:
                sh.gather()
            e2.record(stream)
            ev.append((e0, e1, e2))
    stream.synchronize()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    kern_ms = [a.elapsed_time(b) for a, b, c in ev]
    res = sh.local().results
    bad = int((res["status"] != 0).sum())
    sums = [int(res[f].sum()) for f in ("steps", "formed_steps", "visits", "batch_entries")]
    ms = statistics.mean(step_ms)
    kms = statistics.mean(kern_ms)
    if world > 1:
        t = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
        c = torch.tensor(sums + [bad, launches], dtype=torch.int64, device=dev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        tot = [int(x) for x in c.tolist()]
        sums, bad, launches_all = tot[:4], tot[4], tot[5]
    else:
        launches_all = launches
    steps_all, formed_all, visits_all, entries_all = sums
    value = steps_all / (ms / 1000.0)
    n_cfgs = int(sum(c.n_cost for c in cfgs))

    # critical path (outside the timed region): the longest-estimated simulations of this rank and those with the
    # most formed steps, each launched alone.  The sweep can never be shorter than its longest simulation (each
    # simulation is one dependent chain of steps); at N > 1 this bounds the strong-scaling curve.
    critical = None
    if rank == 0 and not args.no_critical:
        top = list(dict.fromkeys([int(order[j]) for j in range(min(40, len(order)))] +
                                 [int(order[j]) for j in np.argsort(-res["formed_steps"])[:24]]))
        alone = []
        for i in top:
            one = simsweep.DeviceSweep([simsweep.SimConfig.from_buffer_copy(cfgs[int(i)])], wls, cms, device=dev)
            one.launch(stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one.launch(stream)
            e1.record(stream)
            stream.synchronize()
            alone.append((e0.elapsed_time(e1), int(i)))
        lm, li = max(alone)
        j = order.index(li)
        critical = {"longest_simulation_alone_ms": lm, "longest_simulation": " ".join(map(str, labels[li])),
                    "its_steps": int(res["steps"][j]), "its_formed_steps": int(res["formed_steps"][j]),
                    "sweep_kernel_over_longest": kms / lm,
                    "probed": f"{len(top)} simulations (largest LPT estimates and formed-step counts), each alone"}

    # e2e: the public host API (sim_sweep: pinned H2D + kernel + D2H, blocking), every step
    e2e = None
    if not args.no_e2e:
        pin = lambda n, dt: torch.empty(int(n), dtype={np.uint8: torch.uint8, np.float64: torch.float64,  # noqa: E731
                                                       np.int64: torch.int64}[dt], pin_memory=True).numpy()
        pwls = []
        for w in wls:
            Ip = torch.from_numpy(w.I.copy()).pin_memory().numpy()
            Op = torch.from_numpy(w.O.copy()).pin_memory().numpy()
            Tp = torch.from_numpy(w.T.copy()).pin_memory().numpy()
            pwls.append(type(w)(Ip, Op, Tp, w.name))
        sub = sh.plan.shard_configs(rank)  # this rank's shard, in LPT order
        out = simsweep.alloc_outputs(sub, wls, alloc=pin) if sub else None

        def e2e_step():
            r = simsweep.sim_sweep(sub, pwls, cms, device=local_rank, out=out) if sub else sweep._empty_result()
            if world > 1:  # host results -> rank 0 (rows + per-request slabs), one all_gather
                sweep.gather_results(r, sh.plan, rank, device=dev)
                torch.cuda.synchronize(dev)

        e2e_step()  # warm
        if world > 1:
            dist.barrier()
        walls = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            e2e_step()
            walls.append(time.perf_counter() - t0)
        ems = 1000.0 * statistics.mean(walls)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t[0])
        io = [simsweep.io_bytes(sh.plan.shard_configs(r), wls, len(cms)) for r in range(world) if sh.plan.shards[r]]
        e2e = {"value": steps_all / (ems / 1000.0), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": sum(a for a, _ in io), "d2h_bytes_per_step": sum(b for _, b in io),
               "api": "simsweep.sim_sweep (C-ABI sim_sweep, pinned host buffers, blocking)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = _measured_peaks()
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_ops = SM_COUNT * INT_LANES_PER_SM_CLK * clk_mhz * 1e6
    ops = OPS_PER_VISIT * visits_all + OPS_PER_ENTRY * entries_all
    achieved = ops / (kms / 1000.0)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "latest_ncu_summary.json")
    if os.path.exists(prof) and args.workload == "grid":
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic",
        "config": desc | {"configs_per_s": n_cfgs / (ms / 1000.0), "kernel_ms": kms,
                          "steps_per_sweep": steps_all, "formed_steps_per_sweep": formed_all,
                          "formed_steps_per_s": formed_all / (ms / 1000.0),
                          "batch_entries_per_sweep": entries_all, "batch_entries_per_s": entries_all / (ms / 1000.0),
                          "candidate_visits_per_sweep": visits_all, "failed_simulations": bad,
                          "critical_path": critical},
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tintop/s",
                     "frac": achieved / peak_ops, "traffic": traffic,
                     "kernel": "simsweep::sim_lean_kernel<1024> (+ sim_kernel for rank / knob / SRF+Hist / n > 4096)",
                     "work": f"{OPS_PER_VISIT} int ops/candidate visit + {OPS_PER_ENTRY}/batch entry: the method's "
                             f"algorithmic work (SURVEY 8(d)); the kernel executes less (decode epochs, steady runs)"},
        "clocks": clk, "gpu_launches": launches_all,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        idx, sample = oracle_list(args.workload, cfgs, wls)
        cores = min(host_cores(), len(idx))
        s, dt = run_oracle(args.workload, idx, cores)
        cpu = {"value": s / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{sample}: {s} steps in {dt:.2f} s wall on {cores} host cores"}
        if args.workload == "grid":  # "single-thread" next to "all host cores", same full list
            s1, dt1 = run_oracle(args.workload, idx, 1)
            cpu["value_1core"] = s1 / dt1
            cpu["sample_1core"] = f"{sample}: {s1} steps in {dt1:.2f} s on 1 core"
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", choices=["grid", "full"], default="grid")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-critical", action="store_true")
    args = ap.parse_args()
    rank, world, local_rank = _env_dist()
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    return bench_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
