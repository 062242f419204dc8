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


def _gather_worker(rank, world, port, n_total, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    est = np.arange(n_total, 0, -1, dtype=np.float64) ** 1.5
    shards = sweep.partition_lpt(est, world)
    mine = shards[rank]
    local = np.zeros(len(mine), simsweep.RESULT_DTYPE)
    local["steps"] = np.asarray(mine) * 7 + 3  # a per-config fingerprint
    local["status"] = 0
    local["makespan"][:, 0] = np.asarray(mine) * 0.5
    full = sweep.gather_results(local, mine, n_total)
    if rank == 0:
        np.save(out_path, full)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


def test_gather_gloo_world2(tmp_path):
    n_total = 137  # ragged: shards of unequal size
    out = str(tmp_path / "full.npy")
    mp.spawn(_gather_worker, args=(2, _free_port(), n_total, out), nprocs=2, join=True)
    full = np.load(out, allow_pickle=False)
    assert full.dtype == simsweep.RESULT_DTYPE and full.shape == (n_total,)
    assert (full["steps"] == np.arange(n_total) * 7 + 3).all()
    assert np.array_equal(full["makespan"][:, 0], np.arange(n_total) * 0.5)


@pytest.mark.gpu
def test_sharded_equals_unsharded():
    """Independent simulations: splitting a sweep into LPT shards (one launch each, as N ranks would)
    and reassembling gives exactly the unsharded results (SURVEY 8(e) byte-identity check)."""
    cfgs, wls, cms, labels = sweep.grid_sweep(values=[1, 16, 256, 1024])
    whole = simsweep.DeviceSweep(cfgs, wls, cms)
    whole.launch()
    ref = whole.fetch()
    for world in (2, 3, 8):
        shards = sweep.partition_lpt(sweep.estimate(cfgs, wls), world)
        full = np.zeros(len(cfgs), simsweep.RESULT_DTYPE)
        for sh in shards:
            if not sh:
                continue
            sub = [simsweep.SimConfig.from_buffer_copy(cfgs[i]) for i in sh]
            ds = simsweep.DeviceSweep(sub, wls, cms)
            ds.launch()
            r = ds.fetch()
            full[np.asarray(sh)] = r.results
            for j, i in enumerate(sh):
                a = r.request_times(j)
                b = ref.request_times(i)
                assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
        assert full.tobytes() == ref.results.tobytes(), world
