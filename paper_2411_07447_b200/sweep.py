"""Sweep construction, LPT sharding across ranks and the final result gather (row a12).

Simulations are independent (single-instance serving), so a
sweep shards with no data-path communication: each rank simulates its shard
with one ``sim_sweep_device`` launch and the only collective is the final
gather of fixed-size per-simulation result rows (sim_result_t, 200 B) to rank
0 (NCCL over NVLink on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from . import presets, simsweep, workloads

GRID_COST = "llama3-8b_a100_linear"


def grid_sweep(M: int = 100_000, W: int = 1024, policies=("", "-srf"), preset_names=None, S: int = 4096,
               cost_names=(GRID_COST,), values=None):
    """BASELINE configs[1]: 6 schedulers x I, O in {1,2,...,1024} x W, A100 8B cost model, recompute
    (PAPER.md:25-57), for each replacement policy.  Returns (cfgs, wls, cost_model_list, labels)."""
    preset_names = preset_names or presets.GRID_PRESETS
    values = values or workloads.grid_values()
    pcms = simsweep.load_cost_models()
    cms = [pcms[c] for c in cost_names]
    wls, cfgs, labels = [], [], []
    for I in values:
        for O in values:
            wls.append(workloads.fixed(I, O, W))
    for name in preset_names:
        for pol in policies:
            for wi, (I, O) in enumerate([(I, O) for I in values for O in values]):
                cfgs.append(simsweep.preset_config(name + pol, M, S=S, workload=wi, cost=tuple(range(len(cms)))))
                labels.append((name + pol, I, O))
    return cfgs, wls, cms, labels


def varying_m_sweep(Ms=(100, 1_000, 10_000, 100_000, 1_000_000), O: int = 32, W: int = 1024,
                    preset_names=("vllm", "sarathi", "sarathi-cs"), policies=("", "-pf"), S: int = 4096,
                    cost_names=(GRID_COST,), values=None):
    """E5 (Fig. varying_M): O = 32, W = 1024, I over the grid values, M from 100 to 1M, each
    scheduler and its preemption-free version.  Configs whose requests exceed M report never_fits.
    Returns (cfgs, wls, cost_model_list, labels (name, I, M))."""
    values = values or workloads.grid_values()
    pcms = simsweep.load_cost_models()
    cms = [pcms[c] for c in cost_names]
    wls = [workloads.fixed(I, O, W) for I in values]
    cfgs, labels = [], []
    for name in preset_names:
        for pol in policies:
            for M in Ms:
                for wi, I in enumerate(values):
                    cfgs.append(simsweep.preset_config(name + pol, M, S=S, workload=wi, cost=tuple(range(len(cms)))))
                    labels.append((name + pol, I, M))
    return cfgs, wls, cms, labels


def estimate(cfgs, wls) -> np.ndarray:
    """Step-count estimate per simulation (LPT key): max O + KV-time area / M + sum I / C (area = sum (I + O/2) O,
    or the reserve times O under the preemption-free reserves)."""
    est = np.empty(len(cfgs))
    for i, c in enumerate(cfgs):
        w = wls[c.workload]
        I = np.asarray(w.I, np.float64)
        O = np.asarray(w.O, np.float64)
        Meff = float(max(c.M, 1)) if c.M >= 0 else 1e18
        if c.reserve == 1:  # PEAK: the whole reserve I + O - 1 is held while running
            area = float(((I + O - 1) * O).sum())
        elif c.reserve == 2:  # CONTEXT: S per running request
            area = float(c.S) * float(O.sum())
        else:
            area = float(((I + 0.5 * O) * O).sum())
        est[i] = O.max() + area / Meff + float(I.sum()) / float(c.C)
    return est


def partition_lpt(est, n_ranks: int) -> list:
    """Longest-processing-time-first greedy: each simulation (longest first) goes to the
    least-loaded rank.  Returns per-rank lists of config indices (each in LPT order)."""
    order = np.argsort(-np.asarray(est), kind="stable")
    load = np.zeros(n_ranks)
    shards = [[] for _ in range(n_ranks)]
    for i in order:
        r = int(np.argmin(load))
        shards[r].append(int(i))
        load[r] += est[i]
    return shards


def gather_results(local: np.ndarray, local_idx, n_total: int, group=None, device=None):
    """Gather per-simulation result rows (RESULT_DTYPE) of every rank to rank 0, reassembled in
    global config order.  One all_gather of a fixed-size padded slab (the only collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        out = np.zeros(n_total, simsweep.RESULT_DTYPE)
        out[np.asarray(local_idx, np.int64)] = local
        return out
    item = simsweep.RESULT_DTYPE.itemsize
    counts = torch.tensor([len(local_idx)], dtype=torch.int64, device=device if device is not None else "cpu")
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    cap = int(max(int(c.item()) for c in allc))
    slab = np.zeros(cap * item + 8 * cap, np.uint8)
    slab[: len(local_idx) * item] = np.frombuffer(local.tobytes(), np.uint8)
    slab[cap * item: cap * item + 8 * len(local_idx)] = np.frombuffer(
        np.asarray(local_idx, np.int64).tobytes(), np.uint8)
    dev = device if device is not None else torch.device("cpu")
    t = torch.from_numpy(slab).to(dev)
    big = torch.empty(world * t.numel(), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(big, t, group=group)
    if dist.get_rank(group) != 0:
        return None
    buf = big.cpu().numpy().reshape(world, -1)
    out = np.zeros(n_total, simsweep.RESULT_DTYPE)
    for r in range(world):
        c = int(allc[r].item())
        rows = np.frombuffer(buf[r, : c * item].tobytes(), simsweep.RESULT_DTYPE)
        idx = np.frombuffer(buf[r, cap * item: cap * item + 8 * c].tobytes(), np.int64)
        out[idx] = rows
    return out


def run_sharded(cfgs, wls, cms, group=None, device="cuda"):
    """Simulate a sweep over all ranks of `group` (LPT shards), gather results on rank 0.
    Returns (results on rank 0 / None elsewhere, this rank's shard indices, this rank's SweepResult)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shards = partition_lpt(estimate(cfgs, wls), world)
    mine = shards[rank]
    sub = [simsweep.SimConfig.from_buffer_copy(cfgs[i]) for i in mine]
    ds = simsweep.DeviceSweep(sub, wls, cms, device=device, order=np.arange(len(sub)))
    ds.launch()
    local = ds.fetch()
    full = gather_results(local.results, mine, len(cfgs), group=group, device=ds.dev)
    return full, mine, local
