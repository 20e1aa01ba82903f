"""Multi-GPU compressed-domain Lloyd iteration (one process per GPU).

Codes are row-sharded along the top splits of numpy's pairwise-summation tree
(:func:`pairwise.tree_split`), so each rank sums its objective subtree locally
and the host combines G partials in tree order — bit-identical to the
single-GPU / reference ``np.mean``.  Tables and centers are replicated; the
vote is deterministic on identical reduced histograms, so centers need no
broadcast.  Per iteration:

1. assign on the local shard (no communication);
2. allgather of 2 float64 objective partials;
3. allreduce(sum) of the K x M x L int32 histograms and K counts — the one bulk
   collective (NCCL over NVLink on GPUs, gloo in the CPU tests);
4. replicated vote;
5. if E clusters are empty: every rank proposes its local top-E (sd desc, global
   index asc) codes, an allgather collects them and every rank merges them with two
   stable device sorts and applies the same E rows (no host round trip).

The loop is written against a small backend protocol so that the same host
logic runs with the GPU :class:`GpuShardBackend` (product) and, in tests, with a
CPU backend over gloo.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .pairwise import tree_combine, tree_split

try:
    import torch
    import torch.distributed as dist
except ImportError as exc:  # pragma: no cover
    raise ImportError("paper_1709_03708_b200.distributed needs torch.distributed") from exc


@dataclass
class StepStats:
    objective: float
    objective_sq: float
    empty: int
    filled: int
    nnz_total: int
    assign_seconds: float
    update_seconds: float


class GpuShardBackend:
    """Backend over :class:`engine.ShardEngine` (sm_100a kernels)."""

    def __init__(self, codes_local: np.ndarray, offset: int, tables: np.ndarray, k: int, device=None, *,
                 graphs: bool = True):
        from . import engine

        self.graphs = graphs
        self.engine_mod = engine
        self.dev = engine.device_of(device)
        self.m = tables.shape[0]
        self.dt = engine.device_tables(tables, self.dev)
        with torch.cuda.device(self.dev):
            codes_dev = engine.upload_codes(codes_local, self.m, self.dev)
        self.eng = engine.ShardEngine(codes_dev, self.dt, k, self.dev, base_index=offset)
        self.n = len(codes_local)
        self.offset = offset

    def enable_fused_exchange(self, world: int, rank: int) -> None:
        """Put the histogram, the counts and one (sum sqrt sd, sum sd) slot per rank in one
        int32 buffer, so a single SUM allreduce per iteration exchanges all three: each rank
        writes its float64 partials into its own slot and zeros elsewhere, and integer sums
        with zeros reproduce the bit patterns exactly (replaces an all_gather + 2 allreduces)."""
        nh, nc = self.eng.hist.numel(), self.eng.counts.numel()
        pad = (nh + nc) & 1  # 8-byte alignment of the float64 slots
        buf = torch.zeros(nh + nc + pad + 4 * world, dtype=torch.int32, device=self.dev)
        self.eng.hist = buf[:nh]
        self.eng.counts = buf[nh:nh + nc]
        self._xbuf = buf
        self._xtail = buf[nh + nc + pad:].view(torch.float64).view(world, 2)
        self._xrank = rank

    def _fill_exchange_slot(self) -> None:
        if getattr(self, "_xbuf", None) is not None:
            self._xtail.zero_()
            if self.n:
                self._xtail[self._xrank].copy_(self.eng.obj)

    def upload_centers(self, centers: np.ndarray):
        return self.engine_mod.upload_codes(centers, self.m, self.dev)

    def assign(self, centers_dev) -> None:
        if not hasattr(self, "_ev"):
            self._ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True, external=True),
                        torch.cuda.Event(enable_timing=True)]
        self._ev[0].record()
        self.eng.assign(centers_dev)
        self._ev[1].record()

    def sync(self) -> None:
        torch.cuda.current_stream(self.dev).synchronize()

    def histogram(self):
        self.eng.histogram()
        return self.eng.hist, self.eng.counts

    def vote(self) -> np.ndarray:
        self.eng.vote()
        self._ev[2].record()
        return self.eng.stats_host()

    # -- CUDA-graph phases (the driver uses them when present) ------------------
    # local_phase = assign -> objective partials -> histogram (no communication);
    # update_phase = vote.  The first call of each runs eagerly (lazy set-up), the next
    # one captures a graph that later calls replay; the collectives stay outside.
    def local_phase(self, centers_dev):
        if not hasattr(self, "_ev"):
            # _ev[1] is recorded inside the captured graph: an external event node fires on replay
            self._ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True, external=True),
                        torch.cuda.Event(enable_timing=True)]
        if self.n == 0:
            self.assign(centers_dev)
            obj = self.objective_tensor()
            self._fill_exchange_slot()
            return obj, *self.histogram()
        g = getattr(self, "_graph_local", None)
        if g is None:
            self._ev[0].record()
            self.eng.assign(centers_dev)
            self._ev[1].record()
            self.eng.objective()
            self._fill_exchange_slot()
            self.eng.histogram()
            if self.graphs and getattr(self, "_local_eager_done", False):
                self._cur = centers_dev.clone()
                self._graph_local = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(device=self.dev)
                with torch.cuda.graph(self._graph_local, capture_error_mode="thread_local"):
                    self.eng.assign(self._cur)
                    self._ev[1].record()
                    # objective partials on a parallel branch beside the histogram
                    fork = torch.cuda.Event()
                    fork.record()
                    side.wait_event(fork)
                    with torch.cuda.stream(side):
                        self.eng.objective()
                        self._fill_exchange_slot()
                    join = torch.cuda.Event()
                    join.record(side)
                    self.eng.histogram()
                    torch.cuda.current_stream(self.dev).wait_event(join)
                # the capture did not run the work: this iteration's results come from the
                # eager launches above
            self._local_eager_done = True
        else:
            self._cur.copy_(centers_dev)
            self._ev[0].record()
            g.replay()
        return self.eng.obj, self.eng.hist, self.eng.counts

    def update_phase(self) -> np.ndarray:
        g = getattr(self, "_graph_update", None)
        if g is None:
            self.eng.vote()
            if self.graphs and getattr(self, "_update_eager_done", False):
                self._graph_update = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._graph_update, capture_error_mode="thread_local"):
                    self.eng.vote()
            self._update_eager_done = True
        else:
            g.replay()
        self._ev[2].record()
        return self.eng.stats  # on the device: the driver reads it with the objective partials

    def read_host(self, parts_t, st_dev):
        """Objective partials and vote stats: two async copies into pinned host buffers and
        one stream sync (a pageable .cpu() of a concatenation cost ~0.1 ms per iteration)."""
        key = (tuple(parts_t.shape), st_dev.numel())
        if getattr(self, "_pin_key", None) != key:
            self._pin_parts = torch.empty(parts_t.shape, dtype=torch.float64).pin_memory()
            self._pin_st = torch.empty(st_dev.numel(), dtype=torch.int64).pin_memory()
            self._pin_key = key
        self._pin_parts.copy_(parts_t, non_blocking=True)
        self._pin_st.copy_(st_dev.reshape(-1), non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        self.last_stats = self._pin_st.numpy().copy()
        return self._pin_parts.numpy().copy(), self.last_stats

    def step_seconds(self) -> tuple[float, float]:
        """Device time of the last assign and of everything after it up to the vote
        (CUDA events; valid once vote()'s host read has synchronised)."""
        return self._ev[0].elapsed_time(self._ev[1]) / 1e3, self._ev[1].elapsed_time(self._ev[2]) / 1e3

    def objective_tensor(self):
        """(sum sqrt(sd), sum sd) of the local subtree, float64 on the device (no host sync)."""
        if self.n == 0:
            return torch.zeros(2, dtype=torch.float64, device=self.dev)
        self.eng.objective()
        return self.eng.obj

    def local_candidates(self, e: int):
        """Local top-e (sd desc, global index asc) padded to exactly e entries, on the device:
        keys (int64 bit patterns of sd), global index (int64; padding = int64 max), code rows."""
        keys, index = self.eng.repair_candidates(e)
        got = len(index)
        pk = torch.zeros(e, dtype=torch.int64, device=self.dev)
        pi = torch.full((e,), np.iinfo(np.int64).max, dtype=torch.int64, device=self.dev)
        pr = torch.zeros((e, self.m), dtype=torch.uint8, device=self.dev)
        if got:
            pk[:got] = keys
            pi[:got] = index
            pr[:got] = self.eng.codes[(index - self.offset).clamp_(min=0)][:, : self.m]
        return pk, pi, pr

    @property
    def tensor_device(self):
        return self.dev

    def counts_tensor(self):
        return self.eng.counts  # the allreduced counts (int32 view of uint32)

    def apply_repair_rows(self, empty_idx, rows) -> None:
        self.eng.new_centers[empty_idx, : self.m] = rows

    def take_new_centers(self):
        return self.eng.new_centers.clone()

    def centers_host(self, centers_dev) -> np.ndarray:
        return self.engine_mod.download_codes(centers_dev, self.m)

    def labels_host(self) -> np.ndarray:
        return self.eng.labels_host()


def _allgather_obj(values, group) -> list:
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, values, group=group)
    return out


def merge_candidates(parts, e: int):
    """Global top-e by (sd desc, index asc) from per-rank candidate lists."""
    keys = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.uint64)
    index = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.int64)
    rows = np.concatenate([p[2] for p in parts]) if parts else np.zeros((0, 1), np.uint8)
    order = np.lexsort((index, ~keys))[:e]  # primary: key desc (as ~key asc), then index asc
    return keys[order], index[order], rows[order]


def merge_candidates_device(gk: "torch.Tensor", gi: "torch.Tensor", gr: "torch.Tensor", e: int) -> "torch.Tensor":
    """Rows of the global top-e candidates by (sd desc, index asc), on the tensors' device.

    gk: (world, e) int64 bit patterns of non-negative float64 sd (they order like the
    values); gi: (world, e) int64 global indices (padding = int64 max, key 0); gr:
    (world, e, M) uint8 rows.  Two stable sorts (index, then key descending) replace the
    host lexsort of :func:`merge_candidates` (clustering.py:460-466 order)."""
    keys = gk.reshape(-1)
    idx = gi.reshape(-1)
    rows = gr.reshape(-1, gr.shape[-1])
    o1 = torch.argsort(idx, stable=True)
    o2 = torch.argsort(keys[o1], stable=True, descending=True)
    return rows[o1[o2[:e]]]


def empty_clusters_device(counts: "torch.Tensor", e: int) -> "torch.Tensor":
    """The e empty clusters in ascending order (counts == 0) without a host round trip."""
    return torch.argsort((counts != 0).to(torch.int8), stable=True)[:e]


class DistributedLloyd:
    """Sharded PQk-means fit; every rank calls the same methods in lockstep."""

    def __init__(self, backend, n_total: int, k: int, m: int, group=None):
        self.b = backend
        self.n_total = int(n_total)
        if self.n_total >= 2**32:
            raise ValueError("n_total must be < 2^32 (uint32 counts, 32-bit repair key index)")
        self.k = int(k)
        self.m = int(m)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.fused = hasattr(backend, "enable_fused_exchange")
        if self.fused:
            backend.enable_fused_exchange(self.world, self.rank)

    def init_centers(self, seed: int, codes_local: np.ndarray) -> np.ndarray:
        """clustering.py:149-157 over the global index space, rows gathered from owners."""
        rng = np.random.default_rng(seed)
        idx = rng.choice(self.n_total, size=self.k, replace=False)
        lo, hi = self.b.offset, self.b.offset + self.b.n
        mine = {int(i): codes_local[int(i) - lo] for i in idx if lo <= i < hi}
        parts = _allgather_obj(mine, self.group)
        rows = {}
        for p in parts:
            rows.update(p)
        return np.stack([rows[int(i)] for i in idx]).astype(np.uint8)

    def _gather(self, t: "torch.Tensor") -> "torch.Tensor":
        """all_gather of a fixed-shape tensor (NCCL on GPUs, gloo on CPU) -> (world, *shape)."""
        if self.world == 1:
            return t.unsqueeze(0)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t.contiguous(), group=self.group)
        return torch.stack(out)

    def iteration(self, centers_dev, previous: float | None) -> tuple[StepStats, object, bool]:
        """One Lloyd iteration; returns (stats, next centers, stopped)."""
        # Everything up to the vote is queued without a host sync (the GPU never idles
        # between the scan and the update); the one host read is the vote's stats.  The
        # update is computed even on the stopping iteration and then discarded (the
        # reference stops before updating, clustering.py:450-452: same results).
        t0 = time.perf_counter()
        if hasattr(self.b, "local_phase"):  # GPU backend: CUDA-graph phases
            obj_t, hist, counts = self.b.local_phase(centers_dev)
        else:
            self.b.assign(centers_dev)
            obj_t = self.b.objective_tensor()
            hist, counts = self.b.histogram()
        if self.fused:  # one allreduce: histogram, counts and the per-rank objective slots
            if self.world > 1:
                dist.all_reduce(self.b._xbuf, op=dist.ReduceOp.SUM, group=self.group)
            parts_t = self.b._xtail
        else:
            parts_t = self._gather(obj_t)  # stream-ordered collectives
            if self.world > 1:
                dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=self.group)
                dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=self.group)
        if hasattr(self.b, "update_phase"):
            # one device->host read for the objective partials and the vote stats
            st_dev = self.b.update_phase()
            if hasattr(self.b, "read_host"):
                parts, stats = self.b.read_host(parts_t, st_dev)
            else:
                both = torch.cat([parts_t.reshape(-1).view(torch.int64), st_dev.reshape(-1)]).cpu().numpy()
                parts = both[: parts_t.numel()].view(np.float64).reshape(parts_t.shape)
                stats = both[parts_t.numel():]
        else:
            stats = self.b.vote()
            parts = parts_t.cpu().numpy()
        t1 = time.perf_counter()
        if hasattr(self.b, "step_seconds"):
            assign_seconds, vote_seconds = self.b.step_seconds()
        else:
            assign_seconds, vote_seconds = t1 - t0, 0.0
        s1 = tree_combine(self.n_total, list(parts[:, 0]))
        s2 = tree_combine(self.n_total, list(parts[:, 1]))
        objective = float(np.float64(s1) / self.n_total)
        objective_sq = float(np.float64(s2) / self.n_total)
        if previous is not None and objective == previous:
            return StepStats(objective, objective_sq, 0, 0, 0, assign_seconds, 0.0), centers_dev, True
        empty_n = int(stats[3])
        if empty_n:
            # stream-ordered on the device: no host read of the counts, no host merge
            pk, pi, pr = self.b.local_candidates(empty_n)
            rows = merge_candidates_device(self._gather(pk), self._gather(pi), self._gather(pr), empty_n)
            self.b.apply_repair_rows(empty_clusters_device(self.b.counts_tensor(), empty_n), rows)
        nxt = self.b.take_new_centers()
        update_seconds = vote_seconds + (time.perf_counter() - t1)
        st = StepStats(objective, objective_sq, empty_n, int(stats[4]), int(stats[2]), assign_seconds, update_seconds)
        return st, nxt, False


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(offset, length) of this rank's tree-aligned shard."""
    return tree_split(n_total, world)[rank]


def fit_sharded(codes_local: np.ndarray, n_total: int, tables, k: int, max_iterations: int = 20, seed: int = 0, *,
                update: str = "sparse", initial_centers=None, backend=None, group=None):
    """``fit`` over row-sharded codes (clustering.py:377-482 semantics).

    ``codes_local`` must be this rank's :func:`shard_bounds` slice.  Returns a
    ``ClusteringResult`` whose labels are the local shard's labels.
    """
    from .clustering import ClusteringResult, IterationStats
    from .pq import _validate_codes, as_tables

    t = as_tables(tables)
    m_count = t.num_subspaces
    codes_local = _validate_codes(codes_local, m_count, t.num_codewords)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    offset, length = shard_bounds(n_total, world, rank)
    if length != len(codes_local):
        raise ValueError(f"rank {rank} holds {len(codes_local)} codes, expected the tree-aligned shard of {length}")
    if not 1 <= k <= n_total:
        raise ValueError(f"k must be in [1, {n_total}], got {k}")
    if backend is None:
        backend = GpuShardBackend(codes_local, offset, t.tables, k)
    drv = DistributedLloyd(backend, n_total, k, m_count, group)
    if initial_centers is None:
        centers = drv.init_centers(seed, codes_local)
    else:
        centers = _validate_codes(initial_centers, m_count, t.num_codewords).astype(np.uint8)
    cur = backend.upload_centers(centers)
    trace = []
    previous = None
    converged = False
    for iteration in range(1, max_iterations + 1):
        st, nxt, stop = drv.iteration(cur, previous)
        if stop:
            trace.append(IterationStats(iteration, st.objective, st.objective_sq, st.assign_seconds, 0.0))
            converged = True
            break
        mean_nnz = st.nnz_total / (st.filled * m_count) if st.filled else 0.0
        trace.append(
            IterationStats(
                iteration,
                st.objective,
                st.objective_sq,
                st.assign_seconds,
                st.update_seconds,
                repaired_clusters=st.empty,
                mean_histogram_nnz=None if update == "naive" else mean_nnz,
            )
        )
        cur = nxt
        previous = st.objective
    return ClusteringResult(backend.centers_host(cur).astype(np.uint8), backend.labels_host().copy(), trace,
                            len(trace), converged)
