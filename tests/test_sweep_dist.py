"""Multi-GPU sweep plumbing (row a12) on CPU: LPT sharding and the result gather over a
gloo process group of world size 2 (127.0.0.1).  The GPU test checks that sharded
simulation reproduces the unsharded results byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_07447_b200 import simsweep, sweep, workloads


def test_partition_lpt_covers_and_balances():
    est = np.random.default_rng(0).lognormal(3, 1.5, size=1000)
    for n in (1, 2, 3, 8):
        shards = sweep.partition_lpt(est, n)
        flat = sorted(i for sh in shards for i in sh)
        assert flat == list(range(1000))
        loads = [est[sh].sum() for sh in shards]
        assert max(loads) - min(loads) <= est.max() + 1e-9  # LPT bound: imbalance <= the largest job
        for sh in shards:  # longest first within a shard
            assert all(est[sh[i]] >= est[sh[i + 1]] for i in range(len(sh) - 1))


def test_grid_sweep_shape():
    cfgs, wls, cms, labels = sweep.grid_sweep()
    assert len(cfgs) == 6 * 2 * 121 and len(wls) == 121 and len(labels) == len(cfgs)
    assert all(w.n == 1024 for w in wls)
    assert {lab[0] for lab in labels} == {p + s for p in ("vllm", "sarathi", "sarathi-cs", "sarathi-nocp", "vllm-hy",
                                                          "sarathi-nohy") for s in ("", "-srf")}


def test_varying_m_sweep_shape():
    cfgs, wls, cms, labels = sweep.varying_m_sweep()
    assert len(cfgs) == 3 * 2 * 5 * 11 and len(wls) == 11 and all(w.n == 1024 and int(w.O[0]) == 32 for w in wls)
    pf = [c for c, lab in zip(cfgs, labels) if lab[0].endswith("-pf")]
    assert len(pf) == len(cfgs) // 2 and all(c.replacement == 3 and c.reserve == 1 for c in pf)
    assert sorted({lab[2] for lab in labels}) == [100, 1_000, 10_000, 100_000, 1_000_000]


def test_pf_grid_sweep_and_estimate():
    """E4 grid: the PF versions are just another policy suffix; the LPT estimate charges their full reserve."""
    cfgs, wls, cms, labels = sweep.grid_sweep(policies=("", "-pf"), preset_names=["vllm"])
    est = sweep.estimate(cfgs, wls)
    i = labels.index(("vllm", 1, 1024))
    j = labels.index(("vllm-pf", 1, 1024))
    assert est[j] > est[i]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _toy_sweep(n_cfgs):
    """n_cfgs configs over 5 workloads of different sizes, K = 1 or 2 cost models (ragged slabs)."""
    wls = [workloads.fixed(1, 1, n) for n in (3, 1, 7, 2, 5)]
    cfgs = [simsweep.preset_config("vllm", 100, workload=i % 5, cost=(0,) * (1 + i % 2)) for i in range(n_cfgs)]
    return cfgs, wls


def _fingerprint(plan, rank):
    """The outputs rank `rank` would produce for its shard, each value a function of its GLOBAL position."""
    sh = plan.shards[rank]
    nc, nr, nt = plan.sizes[rank]
    res = np.zeros(nc, simsweep.RESULT_DTYPE)
    res["steps"] = np.asarray(sh, np.int64) * 7 + 3
    res["makespan"][:, 0] = np.asarray(sh) * 0.5
    rix, tix = plan.scatter_index(rank)
    local = simsweep.SweepResult(res, tix * 1.25, tix * 2.5 + 1, rix * 3, rix * 5 + 2, None, None, None, None)
    assert local.t_first.shape == (nt,) and local.n_preempt.shape == (nr,)
    return local


def _gather_worker(rank, world, port, n_total, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfgs, wls = _toy_sweep(n_total)
    plan = sweep.ShardPlan(cfgs, wls, world)
    full = sweep.gather_results(_fingerprint(plan, rank), plan, rank)
    if rank == 0:
        np.savez(out_path, res=full.results, tf=full.t_first, td=full.t_done, np_=full.n_preempt, rf=full.refill,
                 ro=full.row_off, to=full.tim_off)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total,world", [(137, 2), (1, 2), (3, 4)])
def test_gather_gloo(tmp_path, n_total, world):
    """Ragged shards, and more ranks than simulations (empty shards still join the collective)."""
    out = str(tmp_path / "full.npz")
    mp.spawn(_gather_worker, args=(world, _free_port(), n_total, out), nprocs=world, join=True)
    z = np.load(out, allow_pickle=False)
    full = z["res"]
    assert full.dtype == simsweep.RESULT_DTYPE and full.shape == (n_total,)
    assert (full["steps"] == np.arange(n_total) * 7 + 3).all()
    assert np.array_equal(full["makespan"][:, 0], np.arange(n_total) * 0.5)
    cfgs, wls = _toy_sweep(n_total)
    n_of = np.array([wls[c.workload].n for c in cfgs])
    k_of = np.array([c.n_cost for c in cfgs])
    rows, trows = int(n_of.sum()), int((n_of * k_of).sum())
    # every per-request row landed at its global row (the layout of one unsharded sim_sweep)
    assert np.array_equal(z["tf"], np.arange(trows) * 1.25) and np.array_equal(z["td"], np.arange(trows) * 2.5 + 1)
    assert np.array_equal(z["np_"], np.arange(rows) * 3) and np.array_equal(z["rf"], np.arange(rows) * 5 + 2)
    assert np.array_equal(z["ro"], np.concatenate([[0], np.cumsum(n_of)[:-1]]))


def test_shard_plan_layout():
    cfgs, wls = _toy_sweep(40)
    for world in (1, 3, 64):
        plan = sweep.ShardPlan(cfgs, wls, world)
        assert sorted(i for sh in plan.shards for i in sh) == list(range(40))
        rows = np.concatenate([plan.scatter_index(r)[0] for r in range(world)])
        trows = np.concatenate([plan.scatter_index(r)[1] for r in range(world)])
        assert sorted(rows.tolist()) == list(range(plan.rows)) and sorted(trows.tolist()) == list(range(plan.trows))
        assert plan.cap % 8 == 0 and plan.cap >= max(plan.slab_bytes)


@pytest.mark.gpu
def test_sharded_equals_unsharded():
    """Independent simulations: splitting a sweep into LPT shards (one launch each, as N ranks would), packing each
    shard's device outputs into its slab and assembling the slabs gives exactly the unsharded outputs -- result rows
    and every per-request slab byte for byte (SURVEY 8(e) byte-identity check)."""
    import torch

    cfgs, wls, cms, labels = sweep.grid_sweep(values=[1, 16, 256, 1024])
    whole = simsweep.DeviceSweep(cfgs, wls, cms)
    whole.launch()
    ref = whole.fetch()
    for world in (2, 3, 8, 200):  # 200 > 48 simulations: empty shards
        plan = sweep.ShardPlan(cfgs, wls, world)
        slabs = []
        for r in range(world):
            sub = plan.shard_configs(r)
            slab = torch.zeros(plan.cap, dtype=torch.uint8, device="cuda")
            if sub:
                ds = simsweep.DeviceSweep(sub, wls, cms, order=np.arange(len(sub)))
                ds.launch()
                sweep.pack_slab(plan, r, ds.d_results, ds.t_first, ds.t_done, ds.n_preempt, ds.refill, out=slab)
            slabs.append(slab)
        full = sweep.Assembler(plan, torch.device("cuda")).assemble(torch.cat(slabs)).result()
        assert full.results.tobytes() == ref.results.tobytes(), world
        for a, b in ((full.t_first, ref.t_first), (full.t_done, ref.t_done), (full.n_preempt, ref.n_preempt),
                     (full.refill, ref.refill)):
            assert a.tobytes() == b.tobytes(), world


@pytest.mark.gpu
def test_run_sharded_single_rank():
    """run_sharded without a process group (world 1) returns the unsharded outputs."""
    cfgs, wls, cms, labels = sweep.grid_sweep(values=[2, 64], preset_names=["vllm", "sarathi"])
    full, mine, local = sweep.run_sharded(cfgs, wls, cms)
    ref = simsweep.sim_sweep(cfgs, wls, cms)
    assert sorted(mine) == list(range(len(cfgs)))
    assert full.results.tobytes() == ref.results.tobytes() and full.t_done.tobytes() == ref.t_done.tobytes()
