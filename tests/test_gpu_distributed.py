"""The sharded driver on a real GPU: NCCL process group (world size 1 — the pool
gives one GPU per call), GpuShardBackend (sm_100a kernels), NCCL all_reduce of the
device histograms, objective partial combine, repair-candidate merge.  Must equal
the single-GPU fit and the oracle byte for byte.  (World sizes 2 and 3 of the same
host logic run on CPU/gloo in test_distributed_gloo.py.)"""

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
