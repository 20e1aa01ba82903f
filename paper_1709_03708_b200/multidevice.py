"""Single-process multi-GPU Lloyd iteration: ``fit(..., devices=[0, 1, ...])``.

The reference's ``fit`` is one call (clustering.py:377-388); this module keeps it one
call on several GPUs of one node, without a process group.  Codes are row-sharded
along the top splits of numpy's summation tree (:func:`pairwise.tree_split`, as in
:mod:`.distributed`), so per-device objective subtrees combine bit-exactly.  Per
iteration:

1. every device runs assign -> objective sums -> histogram on its shard (the same
   kernels as one GPU; nothing crosses devices);
2. the histogram/count exchange runs over peer memory: device d sums its slice of
   clusters [k0_d, k1_d) from every device's K x M x L histogram with
   ``pqk_peer_sum_device`` (direct NVLink loads; a reduce-scatter in one kernel) and
   the K counts in full;
3. device d votes on its slice only (clustering.py:349-356) and the new center rows
   are gathered into every device with peer copies (K x MP bytes in total);
4. one host read per device (objective sums + stats) applies the stop rule; empty
   clusters take the global top-E farthest codes (sd desc, index asc) from the
   devices' local candidates (clustering.py:460-466).

A device may be listed more than once (shards sharing one GPU): the exchange then
reads the same device's memory, which is how the tests exercise this path on a
one-GPU box.  Results equal single-GPU ``fit`` and the reference bit for bit.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib, engine
from ._lib import STATS_LEN, call
from .pairwise import tree_combine, tree_split

try:
    import torch
except ImportError as exc:  # pragma: no cover
    raise ImportError("paper_1709_03708_b200.multidevice needs PyTorch") from exc


def _addr(t: "torch.Tensor", byte_offset: int = 0) -> int:
    return t.data_ptr() + int(byte_offset)


class _Shard:
    """One device's slice of the codes plus its exchange buffers."""

    def __init__(self, codes_local: np.ndarray, offset: int, tables: np.ndarray, k: int, device: int,
                 k0: int, k1: int):
        self.dev = torch.device("cuda", int(device))
        self.dt = engine.device_tables(tables, self.dev)
        self.n = len(codes_local)
        self.offset = int(offset)
        self.k0, self.k1 = int(k0), int(k1)
        m, l_count = self.dt.m, self.dt.l
        with torch.cuda.device(self.dev):
            codes_dev = engine.upload_codes(codes_local, m, self.dev)
            self.eng = engine.ShardEngine(codes_dev, self.dt, k, self.dev, base_index=offset)
            nh = k * m * l_count
            # histogram | counts in one buffer (peers read it); reduced counts separately
            self.xbuf = torch.zeros(nh + k, dtype=torch.int32, device=self.dev)
            self.eng.hist = self.xbuf[:nh]
            self.eng.counts = self.xbuf[nh:]
            self.counts_red = torch.zeros(k, dtype=torch.int32, device=self.dev)
            self.ev_local = torch.cuda.Event()
            self.ev_voted = torch.cuda.Event()
            self.pin_obj = torch.empty(2, dtype=torch.float64).pin_memory()
            self.pin_stats = torch.empty(STATS_LEN, dtype=torch.int64).pin_memory()

    def stream(self) -> "torch.cuda.Stream":
        return torch.cuda.current_stream(self.dev)


class MultiDeviceLloyd:
    """The iteration of fit over G devices of one process (see the module docstring)."""

    def __init__(self, codes: np.ndarray, tables: np.ndarray, k: int, devices):
        devices = [int(d) for d in devices]
        if not devices or len(devices) > 16:
            raise ValueError("devices must list 1 to 16 CUDA device indices")
        for d in devices:
            engine.device_of(d)  # raises without CUDA (no CPU fallback)
        lib = _lib.load()
        distinct = sorted(set(devices))
        if len(distinct) > 1:
            arr = (C.c_int32 * len(distinct))(*distinct)
            _lib.check(lib.pqk_enable_peer_access(arr, len(distinct)), "pqk_enable_peer_access")
        self.lib = lib
        self.n = len(codes)
        if self.n >= 2**32:
            raise ValueError("N must be < 2^32 (uint32 counts, 32-bit repair key index)")
        self.k = int(k)
        self.m = tables.shape[0]
        self.l = tables.shape[1]
        g = len(devices)
        bounds = tree_split(self.n, g)
        ks = [self.k * i // g for i in range(g + 1)]  # vote slices
        self.shards = [_Shard(codes[off:off + ln], off, tables, self.k, dev, ks[i], ks[i + 1])
                       for i, ((off, ln), dev) in enumerate(zip(bounds, devices))]
        self.mp = self.shards[0].dt.mp

    # -- one iteration ------------------------------------------------------------------
    def upload_centers(self, centers: np.ndarray) -> list:
        out = []
        for sh in self.shards:
            with torch.cuda.device(sh.dev):
                out.append(engine.upload_codes(centers, self.m, sh.dev))
        return out

    def iteration(self, cur: list) -> tuple[float, float, np.ndarray, float, float]:
        """Assign + exchange + sliced vote + gather; returns (objective, objective_sq,
        summed stats, assign seconds, update seconds) and leaves the voted centers in
        every shard's ``eng.new_centers`` (repair not yet applied)."""
        m, l_count, k = self.m, self.l, self.k
        t0 = time.perf_counter()
        for sh, c in zip(self.shards, cur):
            with torch.cuda.device(sh.dev):
                sh.eng.stats.zero_()
                if sh.n:
                    sh.eng.assign(c)
                    sh.eng.objective()
                sh.eng.histogram()
                sh.ev_local.record(sh.stream())
        hist_bytes = k * m * l_count * 4
        g = len(self.shards)
        for sh in self.shards:
            with torch.cuda.device(sh.dev):
                s = sh.stream()
                for other in self.shards:
                    s.wait_event(other.ev_local)
                stream = C.c_void_p(s.cuda_stream)
                row = m * l_count * 4
                if sh.k1 > sh.k0:
                    ptrs = (C.c_void_p * g)(*[_addr(o.xbuf, sh.k0 * row) for o in self.shards])
                    call("pqk_peer_sum_device", ptrs, g, (sh.k1 - sh.k0) * m * l_count,
                         C.c_void_p(_addr(sh.xbuf, sh.k0 * row)), stream)
                ptrs = (C.c_void_p * g)(*[_addr(o.xbuf, hist_bytes) for o in self.shards])
                call("pqk_peer_sum_device", ptrs, g, k, C.c_void_p(_addr(sh.counts_red)), stream)
                if sh.k1 > sh.k0:
                    t = sh.dt
                    call("pqk_vote16_device", C.c_void_p(_addr(sh.xbuf, sh.k0 * row)),
                         C.c_void_p(_addr(sh.counts_red, sh.k0 * 4)), sh.k1 - sh.k0, m, l_count, engine._ptr(t.t64),
                         engine._ptr(None if t.fp64_only else t.t32), engine._ptr(None if t.fp64_only else t.t16),
                         C.c_void_p(_addr(sh.eng.new_centers, sh.k0 * self.mp)), engine._ptr(sh.eng.stats), stream)
                sh.ev_voted.record(s)
        # gather: every device copies the other slices' new rows (peer loads)
        for sh in self.shards:
            with torch.cuda.device(sh.dev):
                s = sh.stream()
                stream = C.c_void_p(s.cuda_stream)
                for other in self.shards:
                    if other is sh or other.k1 == other.k0:
                        continue
                    s.wait_event(other.ev_voted)
                    words = (other.k1 - other.k0) * self.mp // 4
                    ptrs = (C.c_void_p * 1)(_addr(other.eng.new_centers, other.k0 * self.mp))
                    call("pqk_peer_sum_device", ptrs, 1, words,
                         C.c_void_p(_addr(sh.eng.new_centers, other.k0 * self.mp)), stream)
                sh.pin_obj.copy_(sh.eng.obj, non_blocking=True)
                sh.pin_stats.copy_(sh.eng.stats, non_blocking=True)
        for sh in self.shards:
            sh.stream().synchronize()
        t1 = time.perf_counter()
        stats = np.zeros(STATS_LEN, np.int64)
        for sh in self.shards:
            stats += sh.pin_stats.numpy()
        s1 = tree_combine(self.n, [float(sh.pin_obj[0]) if sh.n else 0.0 for sh in self.shards])
        s2 = tree_combine(self.n, [float(sh.pin_obj[1]) if sh.n else 0.0 for sh in self.shards])
        return (engine.mean_from_sum(s1, self.n), engine.mean_from_sum(s2, self.n), stats, t1 - t0, 0.0)

    def repair(self, e: int) -> None:
        """Empty clusters (ascending) take the global top-e codes by (sd desc, index asc)."""
        counts = self.shards[0].counts_red.cpu().numpy().view(np.uint32)
        empty = np.flatnonzero(counts == 0)
        keys, index, rows = [], [], []
        for sh in self.shards:
            if sh.n == 0:
                continue
            kk, ii = sh.eng.repair_candidates(e)
            ii_h = ii.cpu().numpy()
            keys.append(kk.cpu().numpy().view(np.uint64))
            index.append(ii_h)
            rows.append(engine.download_codes(sh.eng.codes[torch.from_numpy(ii_h - sh.offset).to(sh.dev)], self.m))
        keys, index, rows = np.concatenate(keys), np.concatenate(index), np.concatenate(rows)
        order = np.lexsort((index, ~keys))[: len(empty)]  # sd desc (as ~bits asc), then index asc
        for sh in self.shards:
            with torch.cuda.device(sh.dev):
                idx = torch.from_numpy(empty.astype(np.int64)).to(sh.dev)
                sh.eng.new_centers[idx] = engine.upload_codes(rows[order], self.m, sh.dev)

    def labels_host(self) -> np.ndarray:
        return np.concatenate([sh.eng.labels_host() for sh in self.shards if sh.n])


def fit_multi_device(codes: np.ndarray, t, k: int, centers: np.ndarray, max_iterations: int, update: str, devices):
    """The Lloyd loop of fit (clustering.py:437-482) over several devices of this process."""
    from .clustering import ClusteringResult, IterationStats

    drv = MultiDeviceLloyd(codes, t.tables, k, devices)
    cur = drv.upload_centers(centers)
    trace = []
    previous = None
    converged = False
    m_count = t.num_subspaces
    for iteration in range(1, max_iterations + 1):
        objective, objective_sq, stats, a_s, _ = drv.iteration(cur)
        if previous is not None and objective == previous:
            trace.append(IterationStats(iteration, objective, objective_sq, a_s, 0.0))
            converged = True
            break
        start = time.perf_counter()
        empty = int(stats[_lib.STAT_EMPTY])
        if empty:
            drv.repair(empty)
        for sh, c in zip(drv.shards, cur):
            with torch.cuda.device(sh.dev):
                c.copy_(sh.eng.new_centers)
        filled = int(stats[_lib.STAT_FILLED])
        nnz_total = int(stats[_lib.STAT_NNZ_TOTAL])
        mean_nnz = nnz_total / (filled * m_count) if filled else 0.0
        trace.append(IterationStats(iteration, objective, objective_sq, a_s, time.perf_counter() - start,
                                    repaired_clusters=empty,
                                    mean_histogram_nnz=None if update == "naive" else mean_nnz))
        previous = objective
    labels = drv.labels_host().copy()
    final = engine.download_codes(cur[0], m_count).astype(np.uint8)
    for sh in drv.shards:
        torch.cuda.synchronize(sh.dev)
    return ClusteringResult(final, labels, trace, len(trace), converged)
