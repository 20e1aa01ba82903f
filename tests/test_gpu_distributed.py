"""The sharded driver on a real GPU: GpuShardBackend (sm_100a kernels) with an NCCL
process group at world size 1 (the pool gives one GPU per call), and with 2 and 3
ranks sharing cuda:0 over gloo collectives on the device tensors: histogram
all_reduce, objective partial combine, padded repair-candidate all_gather.  Must
equal the single-GPU fit and the oracle byte for byte.  (The same host logic with a
CPU stand-in backend runs in test_distributed_gloo.py.)"""

import os
import socket

import numpy as np
import pytest

from helpers import mixture_codes, random_tables

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_fit_sharded_nccl_world1_equals_fit(oracle):
    import torch
    import torch.distributed as dist

    import paper_1709_03708_b200 as pqk
    from paper_1709_03708_b200.distributed import fit_sharded

    tables = random_tables(4, 256, seed=11, sub_dim=8)
    codes = mixture_codes(30_011, 4, 256, 80, seed=5)
    k, iters, seed = 300, 6, 9
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        res = fit_sharded(codes, len(codes), tables, k, iters, seed)
    finally:
        dist.destroy_process_group()
    single = pqk.fit(codes, tables, k, iters, seed, initial_centers=None)
    ref = oracle.fit(codes, tables, k, iters, seed, scan=oracle.assign_c)
    np.testing.assert_array_equal(res.labels, ref["labels"])
    np.testing.assert_array_equal(res.centers, ref["centers"])
    assert [s.objective for s in res.trace] == [t["objective"] for t in ref["trace"]]
    assert [s.repaired_clusters for s in res.trace] == [t["repaired"] for t in ref["trace"]]
    np.testing.assert_array_equal(res.labels, single.labels)
    assert sum(t["repaired"] for t in ref["trace"]) > 0


def _worker_gloo(rank, world, port, codes, tables, k, iters, seed, out):
    import torch
    import torch.distributed as dist

    from paper_1709_03708_b200.distributed import fit_sharded, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, ln = shard_bounds(len(codes), world, rank)
    res = fit_sharded(codes[off:off + ln], len(codes), tables, k, iters, seed)
    np.savez(f"{out}_{rank}.npz", labels=res.labels, centers=res.centers,
             obj=np.array([s.objective for s in res.trace]), rep=np.array([s.repaired_clusters for s in res.trace]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fit_sharded_gpu_backend_multi_rank(tmp_path, oracle, world):
    """world ranks (processes) sharing cuda:0, each running GpuShardBackend on its own
    tree-aligned shard; collectives over gloo on the device tensors (one GPU per call in
    this pool: no NCCL peers).  Exercises the real multi-rank data path of the GPU
    backend: histogram allreduce, objective partials, padded repair candidates."""
    import torch.multiprocessing as mp

    tables = random_tables(4, 256, seed=13, sub_dim=8)
    codes = mixture_codes(24_007, 4, 256, 60, seed=6)
    k, iters, seed = 400, 6, 4
    out = str(tmp_path / "r")
    mp.start_processes(_worker_gloo, args=(world, _port(), codes, tables, k, iters, seed, out), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(f"{out}_{r}.npz") for r in range(world)]
    ref = oracle.fit(codes, tables, k, iters, seed, scan=oracle.assign_c)
    np.testing.assert_array_equal(np.concatenate([p["labels"] for p in parts]), ref["labels"])
    for p in parts:
        np.testing.assert_array_equal(p["centers"], ref["centers"])
        assert list(p["obj"]) == [t["objective"] for t in ref["trace"]]
        assert list(p["rep"]) == [t["repaired"] for t in ref["trace"]]
    assert sum(t["repaired"] for t in ref["trace"]) > 0
