"""Multi-process (world_size 2 and 3, gloo, CPU) test of the sharded Lloyd driver.

The host logic of paper_1709_03708_b200.distributed (tree-aligned shards,
objective partial combine, histogram allreduce, repair-candidate merge, global
init_centers) runs unchanged; the per-shard compute is a CPU backend built from
the oracle (test-only stand-in for the GPU ShardEngine).  The result must be the
single-process reference result byte for byte.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import mixture_codes, random_tables


class CpuShardBackend:
    def __init__(self, codes_local, offset, tables, k):
        from oracle import pqk_oracle as O

        self.O = O
        self.codes = np.ascontiguousarray(codes_local, dtype=np.uint8)
        self.n = len(codes_local)
        self.offset = offset
        self.t = tables
        self.k = k
        self.m = tables.shape[0]
        self.l = tables.shape[1]

    def upload_centers(self, c):
        return np.array(c, dtype=np.uint8)

    def assign(self, centers):
        if self.n:
            self.labels, self.sd = self.O.assign_c(self.codes, centers, self.t, threads=1, want_sd=True)
        else:
            self.labels, self.sd = np.zeros(0, np.uint32), np.zeros(0)

    def sync(self):
        pass

    def objective_tensor(self):
        if self.n == 0:
            return torch.zeros(2, dtype=torch.float64)
        return torch.tensor([np.add.reduce(np.sqrt(self.sd)), np.add.reduce(self.sd)], dtype=torch.float64)

    def histogram(self):
        h = self.O.histogram(self.codes, self.labels, self.k, self.l).astype(np.int32)
        self.hist = torch.from_numpy(np.ascontiguousarray(h))
        self.counts = torch.from_numpy(np.bincount(self.labels.astype(np.intp), minlength=self.k).astype(np.int32))
        return self.hist, self.counts

    def vote(self):
        hist = self.hist.numpy()
        counts = self.counts.numpy()
        self.new = np.zeros((self.k, self.m), np.uint8)
        nnz = 0
        for ki in np.flatnonzero(counts > 0):
            for m in range(self.m):
                nnz += int(np.count_nonzero(hist[ki, m]))
                self.new[ki, m] = self.O.vote_argmin(hist[ki, m], self.t[m])
        st = np.zeros(16, np.int64)
        st[2] = nnz
        st[3] = int((counts == 0).sum())
        st[4] = int((counts > 0).sum())
        return st

    def local_candidates(self, e):
        keys = self.sd.view(np.uint64)
        idx = np.arange(self.n) + self.offset
        order = np.lexsort((idx, ~keys))[:e]
        pk = np.zeros(e, np.uint64)
        pi = np.full(e, np.iinfo(np.int64).max, np.int64)
        pr = np.zeros((e, self.m), np.uint8)
        pk[: len(order)] = keys[order]
        pi[: len(order)] = idx[order]
        pr[: len(order)] = self.codes[order]
        return torch.from_numpy(pk.view(np.int64)), torch.from_numpy(pi), torch.from_numpy(pr)

    def counts_tensor(self):
        return self.counts

    def apply_repair_rows(self, empty_idx, rows):
        self.new[empty_idx.numpy()] = rows.numpy()

    def take_new_centers(self):
        return self.new.copy()

    def centers_host(self, c):
        return c

    def labels_host(self):
        return self.labels


def _worker(rank, world, port, codes, tables, k, iters, seed, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1709_03708_b200.distributed import fit_sharded, shard_bounds

    off, ln = shard_bounds(len(codes), world, rank)
    local = codes[off : off + ln]
    backend = CpuShardBackend(local, off, tables, k)
    res = fit_sharded(local, len(codes), tables, k, iters, seed, backend=backend)
    np.savez(f"{out_path}_{rank}.npz", labels=res.labels, centers=res.centers,
             obj=np.array([s.objective for s in res.trace]), obj_sq=np.array([s.objective_sq for s in res.trace]),
             rep=np.array([s.repaired_clusters for s in res.trace]),
             nnz=np.array([np.nan if s.mean_histogram_nnz is None else s.mean_histogram_nnz for s in res.trace]),
             conv=np.array(res.converged))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fit_equals_single_process(tmp_path, world):
    from oracle import pqk_oracle as O

    tables = random_tables(4, 256, seed=11, sub_dim=8)
    codes = mixture_codes(6007, 4, 256, 40, seed=5)
    k, iters, seed = 150, 6, 9
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(world, _free_port(), codes, tables, k, iters, seed, out), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(f"{out}_{r}.npz") for r in range(world)]
    labels = np.concatenate([p["labels"] for p in parts])
    ref = O.fit(codes, tables, k, iters, seed, scan=O.assign_c)
    np.testing.assert_array_equal(labels, ref["labels"])
    for p in parts:
        np.testing.assert_array_equal(p["centers"], ref["centers"])
        assert list(p["obj"]) == [t["objective"] for t in ref["trace"]]
        assert list(p["obj_sq"]) == [t["objective_sq"] for t in ref["trace"]]
        assert list(p["rep"]) == [t["repaired"] for t in ref["trace"]]
        assert bool(p["conv"]) == ref["converged"]
    assert sum(t["repaired"] for t in ref["trace"]) > 0  # the repair merge was exercised
