"""Sweep construction, LPT sharding across ranks and the final result gather (row a12).

Simulations are independent (single-instance serving), so a
sweep shards with no data-path communication: each rank simulates its shard
with one ``sim_sweep_device`` launch and the only collective is the final
gather of the outputs to rank 0 (NCCL over NVLink on GPUs; gloo in the CPU
tests).  The gather moves the per-simulation rows AND the per-request slabs
(t_first, t_done, n_preempt, refill), so rank 0 ends with exactly what one
sim_sweep over the whole sweep returns.
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


K4_LINEAR = ("llama3-8b_a100_linear", "llama3-8b_h100_linear", "llama3-70b_a100x4_linear", "llama3-70b_h100x4_linear")


def full_sweep(seeds=range(10), grid_W=(32, 1024), M: int = 100_000, online: bool = True, hetero: bool = True):
    """The north-star sweep (BASELINE.json north_star): BASELINE configs [1]-[5] in one list.

    * [1] + [2]: the 6 grid presets x {NRF, SRF} x I, O in {1, 2, ..., 1024} x W in {32, 1024}, each schedule
      charged under K = 4 cost models at once ({8B, 70B} x {A100, H100}, linear; offline schedules are
      cost-model independent) -- 2 x 1 452 simulations, 4 x that many configs;
    * [3]: online LongForm-like and AzureConv-like traces x seeds x {vLLM (C = S), Sarathi
      (C = 512)} x {NRF, SRF, SRF+Hist}, Llama-3-8B / A100, M = 100 000, S = 128K;
    * [4]: the same traces x Llama-3-70B on 4 x A100 and 4 x H100 x {NRF, SRF} x {M, infinite M} x {linear,
      theoretical} (vLLM order);
    * [5]: W = 1024 heterogeneous mixes (ShareGPT-like, table-QA, text-to-SQL, their long-context variants, App. D
      SILO+LISO and SISO+LILO pairs) x seeds x Rank_org / Rank_I / Rank_O.
    Returns (cfgs, wls, cost_model_list, labels); labels are (config-class, name, workload) strings."""
    pcms = simsweep.load_cost_models()
    cost_names = list(K4_LINEAR) + ["llama3-70b_a100x4_theoretical", "llama3-70b_h100x4_theoretical"]
    cms = [pcms[c] for c in cost_names]
    cix = {c: i for i, c in enumerate(cost_names)}
    wls, cfgs, labels = [], [], []

    def add_wl(w):
        wls.append(w)
        return len(wls) - 1

    vals = workloads.grid_values()
    for W in grid_W:
        base = len(wls)
        for I in vals:
            for O in vals:
                add_wl(workloads.fixed(I, O, W))
        for name in presets.GRID_PRESETS:
            for pol in ("", "-srf"):
                for j, (I, O) in enumerate([(I, O) for I in vals for O in vals]):
                    cfgs.append(simsweep.preset_config(name + pol, M, workload=base + j,
                                                       cost=tuple(cix[c] for c in K4_LINEAR)))
                    labels.append(("grid", f"{name}{pol} W={W}", f"I={I} O={O}"))
    if online:
        S = 131072
        for seed in seeds:
            for kind, gen in (("longform", workloads.longform), ("azureconv", workloads.azureconv)):
                wi = add_wl(gen(seed))
                for name in ("vllm", "sarathi"):
                    for pol in ("", "-srf", "-srf-hist"):
                        cfgs.append(simsweep.preset_config(name + pol, M, S=S, workload=wi,
                                                           cost=(cix["llama3-8b_a100_linear"],)))
                        labels.append(("online-8B", f"{name}{pol}", f"{kind} s{seed}"))
                for cm in ("llama3-70b_a100x4", "llama3-70b_h100x4"):
                    for mode in ("linear", "theoretical"):
                        for pol in ("", "-srf"):
                            for MM in (M, -1):
                                cfgs.append(simsweep.preset_config("vllm" + pol, MM, S=S, workload=wi,
                                                                   cost=(cix[f"{cm}_{mode}"],)))
                                labels.append(("online-70B", f"vllm{pol} {cm}_{mode} M={'inf' if MM < 0 else MM}",
                                               f"{kind} s{seed}"))
    if hetero:
        for seed in seeds:
            mixes = [workloads.sharegpt(seed), workloads.table_qa(seed), workloads.table_qa(seed, long_context=True),
                     workloads.text_to_sql(seed), workloads.text_to_sql(seed, long_context=True),
                     workloads.mix(("SILO", "LISO"), 1024, seed), workloads.mix(("SISO", "LILO"), 1024, seed)]
            for w in mixes:
                wi = add_wl(w)
                for name in ("rank-org", "rank-i", "rank-o"):
                    cfgs.append(simsweep.preset_config(name, M, workload=wi, cost=(cix["llama3-8b_a100_linear"],)))
                    labels.append(("hetero", name, w.name))
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


class ShardPlan:
    """The LPT partition of one sweep over `world` ranks and the layout of every rank's output slab.

    Every rank computes the same plan from the same configs (a pure function of the sweep), so the gather needs
    no count exchange.  A rank's slab is [result rows | t_first | t_done | n_preempt | refill] of its shard in
    shard order (the layout sim_sweep gives a sweep of those configs), padded to the largest slab.
    """

    def __init__(self, cfgs, wls, world: int):
        self.cfgs, self.wls, self.world = list(cfgs), wls, int(world)
        self.n_total = len(self.cfgs)
        self.shards = partition_lpt(estimate(self.cfgs, wls), self.world)
        self.n_of = np.array([wls[c.workload].n for c in self.cfgs], np.int64)
        self.k_of = np.array([c.n_cost for c in self.cfgs], np.int64)
        self.row_off = np.concatenate([[0], np.cumsum(self.n_of)[:-1]]).astype(np.int64)
        self.tim_off = np.concatenate([[0], np.cumsum(self.n_of * self.k_of)[:-1]]).astype(np.int64)
        self.rows, self.trows = int(self.n_of.sum()), int((self.n_of * self.k_of).sum())
        item = simsweep.RESULT_DTYPE.itemsize
        self.sizes = []  # per rank: (n_cfgs, rows, tim_rows)
        for sh in self.shards:
            sh = np.asarray(sh, np.int64)
            self.sizes.append((len(sh), int(self.n_of[sh].sum()), int((self.n_of[sh] * self.k_of[sh]).sum())))
        self.slab_bytes = [item * c + 16 * t + 16 * r for (c, r, t) in self.sizes]
        self.cap = max(max(self.slab_bytes), 8)

    def shard_configs(self, rank: int):
        return [simsweep.SimConfig.from_buffer_copy(self.cfgs[i]) for i in self.shards[rank]]

    def scatter_index(self, rank: int):
        """Global row indices of rank's per-request rows (rows, tim_rows) in its shard order."""
        rix, tix = [], []
        for i in self.shards[rank]:
            n, k = int(self.n_of[i]), int(self.k_of[i])
            rix.append(self.row_off[i] + np.arange(n, dtype=np.int64))
            tix.append(self.tim_off[i] + np.arange(n * k, dtype=np.int64))
        cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)  # noqa: E731
        return cat(rix), cat(tix)


def pack_slab(plan: ShardPlan, rank: int, results_u8, t_first, t_done, n_preempt, refill, out=None):
    """This rank's outputs (torch tensors on any device) -> one uint8 slab of plan.cap bytes."""
    import torch

    dev = results_u8.device
    slab = out if out is not None else torch.zeros(plan.cap, dtype=torch.uint8, device=dev)
    off = 0
    for t in (results_u8, t_first, t_done, n_preempt, refill):
        if t.numel() == 0:  # (an empty shard)
            continue
        b = t.contiguous().view(torch.uint8).reshape(-1)
        slab[off: off + b.numel()].copy_(b)
        off += b.numel()
    return slab


class Assembler:
    """Rank 0: the gathered slabs [world x cap] -> the full sweep's outputs in global config order (device ops)."""

    def __init__(self, plan: ShardPlan, device):
        import torch

        self.plan, self.dev = plan, device
        self.idx = []
        for r in range(plan.world):
            rix, tix = plan.scatter_index(r)
            self.idx.append((torch.as_tensor(np.asarray(plan.shards[r], np.int64), device=device),
                             torch.as_tensor(rix, device=device), torch.as_tensor(tix, device=device)))
        item = simsweep.RESULT_DTYPE.itemsize
        self.res = torch.zeros((plan.n_total, item), dtype=torch.uint8, device=device)
        self.tf = torch.zeros(plan.trows, dtype=torch.float64, device=device)
        self.td = torch.zeros(plan.trows, dtype=torch.float64, device=device)
        self.npre = torch.zeros(plan.rows, dtype=torch.int64, device=device)
        self.rf = torch.zeros(plan.rows, dtype=torch.int64, device=device)

    def assemble(self, big):
        import torch

        item = simsweep.RESULT_DTYPE.itemsize
        buf = big.reshape(self.plan.world, self.plan.cap)
        for r, (nc, nr, nt) in enumerate(self.plan.sizes):
            if nc == 0:
                continue
            ci, rix, tix = self.idx[r]
            b = buf[r]
            o = 0
            self.res.index_copy_(0, ci, b[o: o + nc * item].reshape(nc, item))
            o += nc * item
            for dst, ix, cnt in ((self.tf, tix, nt), (self.td, tix, nt), (self.npre, rix, nr), (self.rf, rix, nr)):
                dst.index_copy_(0, ix, b[o: o + 8 * cnt].view(dst.dtype))
                o += 8 * cnt
        return self

    def result(self) -> simsweep.SweepResult:
        p = self.plan
        res = np.frombuffer(self.res.cpu().numpy().tobytes(), simsweep.RESULT_DTYPE).copy()
        return simsweep.SweepResult(res, self.tf.cpu().numpy(), self.td.cpu().numpy(), self.npre.cpu().numpy(),
                                    self.rf.cpu().numpy(), p.row_off, p.tim_off, p.n_of, p.k_of)


def gather_slabs(plan: ShardPlan, slab, group=None):
    """The sweep's only collective: all_gather_into_tensor of every rank's padded output slab (NCCL over NVLink on
    GPUs, gloo on CPU).  Returns the [world * cap] uint8 tensor (every rank receives it; rank 0 assembles)."""
    import torch
    import torch.distributed as dist

    big = torch.empty(plan.world * plan.cap, dtype=torch.uint8, device=slab.device)
    dist.all_gather_into_tensor(big, slab, group=group)
    return big


def gather_results(local: simsweep.SweepResult, plan: ShardPlan, rank: int, group=None, device=None):
    """Host-side gather of one rank's SweepResult (numpy) to a full SweepResult on rank 0 (None elsewhere):
    per-simulation rows AND the per-request slabs (t_first, t_done, n_preempt, refill)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = device if device is not None else torch.device("cpu")
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
    slab = pack_slab(plan, rank, t(local.results, np.uint8), t(local.t_first, np.float64), t(local.t_done, np.float64),
                     t(local.n_preempt, np.int64), t(local.refill, np.int64))
    big = gather_slabs(plan, slab, group) if world > 1 else slab
    if rank != 0:
        return None
    return Assembler(plan, dev).assemble(big).result()


def _empty_result():
    z = np.zeros(0, np.int64)
    return simsweep.SweepResult(np.zeros(0, simsweep.RESULT_DTYPE), np.zeros(0), np.zeros(0), z, z.copy(), z, z, z, z)


class ShardedSweep:
    """One sweep partitioned over the ranks of `group` (LPT), each shard simulated by one sim_sweep_device call on
    this rank's GPU, the outputs gathered to rank 0 by one all_gather of padded slabs (device tensors, NCCL)."""

    def __init__(self, cfgs, wls, cms, group=None, device="cuda"):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.dev = torch.device(device)
        self.plan = ShardPlan(cfgs, wls, self.world)
        self.mine = self.plan.shards[self.rank]
        sub = self.plan.shard_configs(self.rank)
        # a rank whose shard is empty (fewer simulations than ranks) still joins the collective with a zero slab
        self.ds = simsweep.DeviceSweep(sub, wls, cms, device=self.dev, order=np.arange(len(sub))) if sub else None
        self.slab = torch.zeros(self.plan.cap, dtype=torch.uint8, device=self.dev)
        self.asm = Assembler(self.plan, self.dev) if self.rank == 0 else None

    def launch(self, stream=None) -> int:
        return self.ds.launch(stream) if self.ds is not None else 0

    def gather(self):
        """Pack this rank's device outputs, all_gather the slabs, assemble on rank 0 (enqueued on the current
        stream).  Returns the number of collectives issued."""
        if self.ds is not None:
            d = self.ds
            pack_slab(self.plan, self.rank, d.d_results, d.t_first, d.t_done, d.n_preempt, d.refill, out=self.slab)
        big = gather_slabs(self.plan, self.slab, self.group) if self.world > 1 else self.slab
        if self.rank == 0:
            self.asm.assemble(big)
        return 1 if self.world > 1 else 0

    def local(self) -> simsweep.SweepResult:
        return self.ds.fetch() if self.ds is not None else _empty_result()

    def result(self):
        """The full sweep's SweepResult on rank 0 (after gather()), None elsewhere."""
        return self.asm.result() if self.rank == 0 else None


def run_sharded(cfgs, wls, cms, group=None, device="cuda"):
    """Simulate a sweep over all ranks of `group` (LPT shards), gather every output to rank 0.
    Returns (full SweepResult on rank 0 / None elsewhere, this rank's shard indices, this rank's SweepResult)."""
    sh = ShardedSweep(cfgs, wls, cms, group=group, device=device)
    sh.launch()
    sh.gather()
    return sh.result(), sh.mine, sh.local()
