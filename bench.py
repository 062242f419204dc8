#!/usr/bin/env python
"""bench.py -- simulated scheduler steps/s of the B200 step-level simulator.

One bench STEP = one pass of the whole hot path (rows a1-a12) over BASELINE
configs[1]: the high-contention grid, 6 schedulers x I, O in {1, 2, ..., 1024}
x W = 1024 x {NRF, SRF}, A100 Llama-3-8B linear cost model, KV recomputation,
M = 100 000 (1 452 simulations, one sim_sweep_device launch [+ the gather at N > 1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): STRONG scaling -- the one sweep is
LPT-sharded over the ranks (sweep.ShardedSweep), each rank simulates its shard
and all outputs (result rows + per-request slabs) are gathered to rank 0 by one
all_gather over NVLink inside the timed step; value = steps of the sweep /
max-over-ranks time.  The floor is the longest single simulation (a dependent
chain of steps), reported as config.critical_path.
--impl reference times the CPU oracle (oracle/, the only other thing this file
may run) on the host cores over a bounded sample of the same grid.
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


def workload_desc(world: int):
    return {"workload": "BASELINE configs[1] grid: 6 presets (vllm, sarathi, sarathi-cs, sarathi-nocp, vllm-hy, "
                        "sarathi-nohy) x I,O in {1..1024 pow2} x W=1024 x {NRF,SRF} = 1452 simulations, "
                        "llama3-8b A100 linear cost model, M=100000, offline; LPT-sharded over the GPUs",
            "simulations": 1452, "W": 1024, "S": 4096, "M": 100_000,
            "l2": "flushed between timed iterations (256 MiB)"}


# ---------------------------------------------------------------- oracle (CPU) legs
def _oracle_job(args):
    name, I, O, W, M = args
    import oracle as o
    from paper_2411_07447_b200 import presets

    p = presets.preset(name)
    cfg = o.make_config(p["order"], p["hybrid"], p["chunked"], p["replacement"], C=p["C"], M=M, reserve=p["reserve"])
    cm = o.load_cost_models()["llama3-8b_a100_linear"]
    from paper_2411_07447_b200 import workloads

    wl = workloads.fixed(I, O, W)
    r = o.run(cfg, wl.I, wl.O, wl.T, cm)
    return r.steps, r.batch_entries


def oracle_sample(stride: int, M: int = 100_000):
    """Every stride-th simulation of the grid, in the grid's natural (preset, policy, I, O) order."""
    from paper_2411_07447_b200 import presets, workloads

    vals = workloads.grid_values()
    labels = [(nm + pol, I, O) for nm in presets.GRID_PRESETS for pol in ("", "-srf") for I in vals for O in vals]
    return [(nm, I, O, 1024, M) for (nm, I, O) in labels[::stride]]


def run_oracle(jobs, cores: int):
    import multiprocessing as mp

    import oracle

    oracle.build()
    t0 = time.perf_counter()
    if cores > 1:
        with mp.get_context("fork").Pool(cores) as pool:
            out = pool.map(_oracle_job, jobs, chunksize=1)
    else:
        out = [_oracle_job(j) for j in jobs]
    dt = time.perf_counter() - t0
    return sum(s for s, _ in out), dt


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def bench_reference(args, rank, world):
    if rank != 0:
        return 0
    stride = 8
    jobs = oracle_sample(stride)
    cores = min(host_cores(), len(jobs))
    for _ in range(args.warmup):
        run_oracle(jobs[: max(1, len(jobs) // 8)], cores)
    times, steps = [], 0
    for _ in range(args.steps):
        s, dt = run_oracle(jobs, cores)
        times.append(dt)
        steps = s
    ms = 1000.0 * statistics.mean(times)
    value = steps / (ms / 1000.0)
    sample = f"every {stride}th simulation of the rank-0 grid ({len(jobs)} of 1452), all cores, multiprocessing"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": workload_desc(1) | {"reference": "CPU oracle (oracle/oracle.cpp), g++ -O2"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
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
    cfgs, wls, cms, labels = sweep.grid_sweep(M=100_000)
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
    steps_rank = int(res["steps"].sum())
    visits_rank = int(res["visits"].sum())
    entries_rank = int(res["batch_entries"].sum())
    ms = statistics.mean(step_ms)
    kms = statistics.mean(kern_ms)
    if world > 1:
        t = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
        c = torch.tensor([steps_rank, visits_rank, entries_rank, bad, launches], dtype=torch.int64, device=dev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        steps_all, visits_all, entries_all, bad, launches_all = (int(x) for x in c.tolist())
    else:
        steps_all, visits_all, entries_all, launches_all = steps_rank, visits_rank, entries_rank, launches
    value = steps_all / (ms / 1000.0)
    n_sims = len(cfgs)

    # critical path (outside the timed region): the longest-estimated simulations, each launched alone.  The
    # sweep can never be shorter than its longest simulation (each simulation is one dependent chain of steps).
    critical = None
    if rank == 0 and not args.no_critical:
        # the 48 largest step-count estimates plus the 16 largest visit counts of this sweep (the estimate misses
        # vLLM's preemption thrash at small I, whose steps are all full steps)
        top = list(dict.fromkeys([int(order[j]) for j in range(min(48, len(order)))] +
                                 [int(order[j]) for j in np.argsort(-res["visits"])[:16]]))
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
        critical = {"longest_simulation_alone_ms": lm, "longest_simulation": "%s I=%d O=%d" % labels[li],
                    "its_steps": int(res["steps"][order.index(li)]), "sweep_kernel_over_longest": kms / lm,
                    "probed": f"{len(top)} simulations (largest LPT estimates and visit counts), each launched alone"}

    # e2e: the public host API (sim_sweep: pinned H2D + kernel + D2H, blocking), every step
    e2e = None
    if not args.no_e2e:
        pin = lambda n, dt: torch.empty(int(n), dtype={np.uint8: torch.uint8, np.float64: torch.float64,
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
        io = [simsweep.io_bytes(sh.plan.shard_configs(r), wls, len(cms)) for r in range(world)
              if sh.plan.shards[r]]
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
    ops_rank = OPS_PER_VISIT * visits_rank + OPS_PER_ENTRY * entries_rank
    achieved = ops_rank / (kms / 1000.0)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "latest_ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic",
        "config": workload_desc(world) | {"configs_per_s": n_sims / (ms / 1000.0), "kernel_ms": kms,
                                          "steps_per_sweep": steps_all, "batch_entries_per_sweep": entries_all,
                                          "candidate_visits_per_sweep": visits_all, "failed_simulations": bad,
                                          "critical_path": critical},
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tintop/s",
                     "frac": achieved / peak_ops, "traffic": traffic,
                     "kernel": "simsweep::sim_kernel<256,1024>",
                     "work": f"{OPS_PER_VISIT} int ops/candidate visit + {OPS_PER_ENTRY}/batch entry (DESIGN.md 5)"},
        "clocks": clk, "gpu_launches": launches_all,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        stride = 4
        jobs = oracle_sample(stride)
        cores = min(host_cores(), len(jobs))
        s, dt = run_oracle(jobs, cores)
        jobs1 = oracle_sample(48)  # one core: "single-thread" next to "all host cores"
        s1, dt1 = run_oracle(jobs1, 1)
        line["cpu_baseline"] = {"value": s / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"every {stride}th simulation of the grid ({len(jobs)} of 1452), "
                                          f"{s} steps in {dt:.2f} s wall on {cores} host cores",
                                "value_1core": s1 / dt1,
                                "sample_1core": f"every 48th simulation ({len(jobs1)}), {s1} steps in {dt1:.2f} s on 1 core"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
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
