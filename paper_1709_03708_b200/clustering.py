"""K-means on PQ codes, B200-native drop-in for ``pqclust.clustering``'s hot path.

Public names, signatures, return types and ``ValueError`` messages follow the
reference (/root/reference/pkg/src/pqclust/clustering.py); the iteration runs
resident on one GPU (or sharded over several, :mod:`.distributed`) through the
sm_100a kernels of ``libpqk_b200.so``:

- ``fit``        clustering.py:377-482  (assign -> sd -> objective -> stop? ->
                 counts -> sparse vote -> repair, per iteration)
- ``assign``     clustering.py:255-282  (strategy dispatch; "linear_scan" is the GPU scan)
- registry       clustering.py:200-226  (same protection / messages)
- ``select_assignment_strategy`` clustering.py:229-252
- ``init_centers`` clustering.py:149-157 (numpy Generator.choice on the host, O(K))
- ``pq_cost`` / ``pq_cost_sq`` clustering.py:285-324 (device sums, numpy's tree)
- ``IterationStats`` / ``ClusteringResult`` clustering.py:27-65

``b200_assign_strategy`` is the function to register in the *reference*
registry: ``pqclust.register_assignment_strategy("b200", b200_assign_strategy)``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import engine
from .pq import _validate_codes, as_tables


@dataclass
class IterationStats:
    """Per-iteration record (clustering.py:27-42)."""

    iteration: int
    objective: float
    objective_sq: float
    assign_seconds: float
    update_seconds: float
    repaired_clusters: int = 0
    mean_histogram_nnz: float | None = None


@dataclass
class ClusteringResult:
    """Output of a clustering run (clustering.py:45-65)."""

    centers: np.ndarray
    labels: np.ndarray
    trace: list[IterationStats] = field(default_factory=list)
    iterations_run: int = 0
    converged: bool = False


@dataclass(frozen=True)
class FrequencyHistogram:
    """Counts of codeword indices inside one (cluster, subspace) pair (clustering.py:68-83)."""

    counts: np.ndarray
    support: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.support)


def build_histogram(subindices: np.ndarray, num_codewords: int) -> FrequencyHistogram:
    """Tally subindices into L bins (clustering.py:86-105; host-side input helper)."""
    values = np.asarray(subindices)
    if values.ndim != 1:
        raise ValueError(f"subindices must be 1-d, got shape {values.shape}")
    if values.size and (values.min() < 0 or values.max() >= num_codewords):
        raise ValueError(
            f"subindices must lie in [0, {num_codewords}), got range [{values.min()}, {values.max()}]"
        )
    counts = np.bincount(values.astype(np.intp), minlength=num_codewords)
    return FrequencyHistogram(counts, np.flatnonzero(counts))


def update_center_sparse(histograms, tables) -> np.ndarray:
    """One center from per-subspace member histograms by sparse voting on the GPU (clustering.py:125-146)."""
    t = as_tables(tables)
    if len(histograms) != t.num_subspaces:
        raise ValueError(f"expected {t.num_subspaces} histograms, got {len(histograms)}")
    hist = np.zeros((1, t.num_subspaces, t.num_codewords), dtype=np.int64)
    for m, h in enumerate(histograms):
        if h.nnz == 0:
            raise ValueError(f"histogram for subspace {m} is empty")
        hist[0, m, : len(h.counts)] = h.counts
    return engine.vote_host(hist, t.tables)[0]


def update_center_naive(member_codes: np.ndarray, tables) -> np.ndarray:
    """One center by candidate scan (clustering.py:108-122); same argmin as the vote, computed on the GPU."""
    t = as_tables(tables)
    codes = _validate_codes(member_codes, t.num_subspaces, t.num_codewords)
    if len(codes) == 0:
        raise ValueError("cannot update a center from an empty cluster")
    hist = np.stack([np.bincount(codes[:, m].astype(np.intp), minlength=t.num_codewords)
                     for m in range(t.num_subspaces)])[None]
    return engine.vote_host(hist, t.tables)[0]


def init_centers(codes: np.ndarray, k: int, seed: int = 0) -> np.ndarray:
    """Pick K initial centers by sampling input codes without replacement."""
    codes = np.asarray(codes)
    if codes.ndim != 2:
        raise ValueError(f"codes must be 2-d, got shape {codes.shape}")
    if not 1 <= k <= len(codes):
        raise ValueError(f"k must be in [1, {len(codes)}], got {k}")
    rng = np.random.default_rng(seed)
    return codes[rng.choice(len(codes), size=k, replace=False)].copy()


# ---------------------------------------------------------------------------
# assignment strategies
AssignStrategy = Callable[[np.ndarray, np.ndarray, object, int], np.ndarray]


def _gpu_linear_scan(codes: np.ndarray, centers: np.ndarray, tables, threads: int = 1) -> np.ndarray:
    """Exhaustive nearest-center scan on the GPU; exactly the reference labels."""
    t = as_tables(tables)
    return engine.assign_host(codes, centers, t.tables)


def b200_assign_strategy(codes: np.ndarray, centers: np.ndarray, tables, threads: int = 1) -> np.ndarray:
    """AssignStrategy for the reference registry (clustering.py:200, :207-216).

    ``threads`` is advisory and ignored; codes/centers may be any integer dtype.
    """
    t = as_tables(tables)
    codes = _validate_codes(codes, t.num_subspaces, t.num_codewords)
    centers = _validate_codes(centers, t.num_subspaces, t.num_codewords)
    if len(centers) == 0:
        raise ValueError("centers must be non-empty")
    return _gpu_linear_scan(codes, centers, t, threads)


_ASSIGNMENT_STRATEGIES: dict[str, AssignStrategy] = {
    "linear_scan": _gpu_linear_scan,
}


def register_assignment_strategy(name: str, strategy: AssignStrategy) -> None:
    if not name:
        raise ValueError("strategy name must be non-empty")
    _ASSIGNMENT_STRATEGIES[name] = strategy


def unregister_assignment_strategy(name: str) -> None:
    if name == "linear_scan":
        raise ValueError("the linear_scan strategy cannot be removed")
    _ASSIGNMENT_STRATEGIES.pop(name, None)


def registered_assignment_strategies() -> tuple[str, ...]:
    return tuple(_ASSIGNMENT_STRATEGIES)


def select_assignment_strategy(codes: np.ndarray, tables, k: int, seed: int = 0) -> str:
    """Fastest registered strategy on 10 sampled queries (singleton: no timing)."""
    if len(_ASSIGNMENT_STRATEGIES) == 1:
        return next(iter(_ASSIGNMENT_STRATEGIES))
    t = as_tables(tables)
    codes = _validate_codes(codes, t.num_subspaces, t.num_codewords)
    rng = np.random.default_rng(seed)
    centers = init_centers(codes, min(k, len(codes)), seed)
    queries = codes[rng.integers(0, len(codes), size=min(10, len(codes)))]
    best_name = ""
    best_time = math.inf
    for name, strategy in _ASSIGNMENT_STRATEGIES.items():
        start = time.perf_counter()
        strategy(queries, centers, t, 1)
        elapsed = time.perf_counter() - start
        if elapsed < best_time:
            best_name, best_time = name, elapsed
    return best_name


def assign(codes: np.ndarray, centers: np.ndarray, tables, threads: int = 1, strategy: str = "linear_scan") -> np.ndarray:
    """uint32 labels of the nearest center per code, lowest index on ties."""
    t = as_tables(tables)
    codes = _validate_codes(codes, t.num_subspaces, t.num_codewords)
    centers = _validate_codes(centers, t.num_subspaces, t.num_codewords)
    if len(centers) == 0:
        raise ValueError("centers must be non-empty")
    if strategy not in _ASSIGNMENT_STRATEGIES:
        raise ValueError(f"unknown assignment strategy {strategy!r}")
    return _ASSIGNMENT_STRATEGIES[strategy](codes, centers, t, threads)


# ---------------------------------------------------------------------------
# costs
def _assigned_sd(codes, centers, assignment, tables) -> tuple[np.ndarray, object]:
    t = as_tables(tables)
    codes = _validate_codes(codes, t.num_subspaces, t.num_codewords)
    assignment = np.asarray(assignment)
    if assignment.shape != (len(codes),):
        raise ValueError(f"assignment must have shape ({len(codes)},), got {assignment.shape}")
    if len(assignment) and assignment.max() >= len(centers):
        raise ValueError(
            f"assignment references center {assignment.max()} but only {len(centers)} centers exist"
        )
    return codes, t


def _cost_pair(codes, centers, assignment, tables) -> tuple[float, float]:
    codes, t = _assigned_sd(codes, centers, assignment, tables)
    n = len(codes)
    if n == 0:
        return 0.0, 0.0
    centers = np.asarray(centers)
    dev = engine.device_of()
    import torch

    dt = engine.device_tables(t.tables, dev)
    with torch.cuda.device(dev):
        a = engine.upload_codes(codes, dt.m, dev)
        b = engine.upload_codes(_validate_codes(centers, t.num_subspaces, t.num_codewords), dt.m, dev)
        idx = torch.from_numpy(np.ascontiguousarray(assignment, dtype=np.int64).astype(np.uint32).view(np.int32)).to(dev)
        sd = torch.empty(n, dtype=torch.float64, device=dev)
        engine.call(
            "pqk_paired_distance_device",
            engine._ptr(a),
            engine._ptr(b),
            engine._ptr(idx),
            n,
            dt.m,
            dt.l,
            engine._ptr(dt.t64),
            engine._ptr(sd),
            engine._stream(dev),
        )
        return engine.mean_objectives(sd, n, dev)


def pq_cost(codes, centers, assignment, tables) -> float:
    """Mean symmetric distance (non-squared) of points to assigned centers."""
    return _cost_pair(codes, centers, assignment, tables)[0]


def pq_cost_sq(codes, centers, assignment, tables) -> float:
    """Mean squared symmetric distance of points to assigned centers."""
    return _cost_pair(codes, centers, assignment, tables)[1]


# ---------------------------------------------------------------------------
def fit(
    codes: np.ndarray,
    tables,
    k: int,
    max_iterations: int = 20,
    seed: int = 0,
    *,
    threads: int = 1,
    update: str = "sparse",
    strategy: str | None = None,
    initial_centers: np.ndarray | None = None,
    device: int | None = None,
    devices: list[int] | None = None,
) -> ClusteringResult:
    """Cluster PQ codes with k-means in the compressed domain on the GPU.

    Same semantics as the reference ``fit``: sampled (or given) initial centers,
    alternate assignment and sparse-voting update, stop when the objective
    repeats exactly or after ``max_iterations``, empty clusters re-seeded on the
    farthest codes.  ``threads`` is accepted and ignored (results never depend
    on it).  The returned labels are those of the last assignment.

    ``devices=[0, 1, ...]`` shards the codes over several GPUs of this process
    (:mod:`.multidevice`: peer-memory histogram exchange, sliced vote); the result is
    identical to one GPU.  It needs the built-in scan (``strategy`` None or
    "linear_scan").
    """
    import torch

    t = as_tables(tables)
    m_count, l_count = t.num_subspaces, t.num_codewords
    codes = _validate_codes(codes, m_count, l_count)
    if not 1 <= k <= len(codes):
        raise ValueError(f"k must be in [1, {len(codes)}], got {k}")
    if max_iterations < 1:
        raise ValueError(f"max_iterations must be positive, got {max_iterations}")
    if update not in ("sparse", "naive"):
        raise ValueError(f"update must be 'sparse' or 'naive', got {update!r}")
    if initial_centers is None:
        centers = init_centers(codes, k, seed)
    else:
        centers = _validate_codes(initial_centers, m_count, l_count).astype(np.uint8)
        if len(centers) != k:
            raise ValueError(f"initial_centers has {len(centers)} rows, expected k={k}")
    if strategy is None:
        strategy = select_assignment_strategy(codes, t, k, seed)
    if strategy not in _ASSIGNMENT_STRATEGIES:
        raise ValueError(f"unknown assignment strategy {strategy!r}")
    external = None if _ASSIGNMENT_STRATEGIES[strategy] is _gpu_linear_scan else _ASSIGNMENT_STRATEGIES[strategy]
    if devices is not None:
        if external is not None:
            raise ValueError("devices=... runs the built-in GPU scan; use strategy='linear_scan'")
        from .multidevice import fit_multi_device

        return fit_multi_device(codes, t, k, centers, max_iterations, update, devices)

    dev = engine.device_of(device)
    with torch.cuda.device(dev):
        codes_dev = engine.upload_codes(codes, m_count, dev)
        return _fit_on_device(codes_dev, len(codes), t, k, centers, max_iterations, update, external, codes, threads,
                              dev)


def fit_device(
    codes_dev,
    n: int,
    tables,
    k: int,
    max_iterations: int = 20,
    seed: int = 0,
    *,
    update: str = "sparse",
    initial_centers: np.ndarray | None = None,
    device: int | None = None,
) -> ClusteringResult:
    """``fit`` on codes already resident on the GPU (extension for data streamed from
    files, io.load_codes): ``codes_dev`` is the (N, MP) uint8 device layout with
    validated subindices.  Initial centers are the rows the reference's
    ``init_centers`` would pick (clustering.py:149-157), gathered on the device."""
    import torch

    t = as_tables(tables)
    m_count, l_count = t.num_subspaces, t.num_codewords
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    if max_iterations < 1:
        raise ValueError(f"max_iterations must be positive, got {max_iterations}")
    if update not in ("sparse", "naive"):
        raise ValueError(f"update must be 'sparse' or 'naive', got {update!r}")
    dev = engine.device_of(device)
    with torch.cuda.device(dev):
        if initial_centers is None:
            idx = np.random.default_rng(seed).choice(n, size=k, replace=False)
            rows = codes_dev.index_select(0, torch.from_numpy(idx.astype(np.int64)).to(dev))
            centers = engine.download_codes(rows, m_count)
        else:
            centers = _validate_codes(initial_centers, m_count, l_count).astype(np.uint8)
            if len(centers) != k:
                raise ValueError(f"initial_centers has {len(centers)} rows, expected k={k}")
        return _fit_on_device(codes_dev, n, t, k, centers, max_iterations, update, None, None, 1, dev)


# Replay the device part of each Lloyd iteration from CUDA graphs (engine.IterationGraphs)
# after the first, eager iteration: ~45 kernel launches become two graph launches.
USE_CUDA_GRAPHS = True


def _fit_on_device(codes_dev, n, t, k, centers, max_iterations, update, external, codes, threads, dev):
    """The Lloyd loop of fit (clustering.py:437-482) on a device code buffer."""
    import torch

    m_count = t.num_subspaces
    device_scan = external is None
    with torch.cuda.device(dev):
        dt = engine.device_tables(t.tables, dev)
        cur = engine.upload_codes(centers, m_count, dev)
        eng = engine.ShardEngine(codes_dev, dt, k, dev)
        trace: list[IterationStats] = []
        previous = None
        converged = False
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        graphs = None  # CUDA graphs of the iteration body, captured after iteration 1
        use_graphs = USE_CUDA_GRAPHS
        for iteration in range(1, max_iterations + 1):
            # One stream-ordered iteration: assign, objective sums, histogram and the
            # (speculative) vote into the next-centers buffer, then a single host read of
            # objective + stats.  If the stop rule fires the vote result is discarded, so
            # the observable semantics are the reference's (clustering.py:442-481).
            ev[0].record()
            if graphs is not None:
                graphs.main.replay()
                ev_assigned = graphs.ev_assigned
            else:
                if device_scan:
                    eng.assign(cur)
                else:
                    host_centers = engine.download_codes(cur, m_count)
                    lab = np.asarray(external(codes, host_centers, t, threads), dtype=np.uint32)
                    eng.labels[:n].copy_(torch.from_numpy(lab.view(np.int32)).to(dev))
                    eng.distances_for_labels(cur)
                ev[1].record()
                ev_assigned = ev[1]
                eng.objective()
                eng.histogram()
                eng.vote()
            ev[2].record()
            sums, stats = eng.read_obj_stats()
            assign_seconds = ev[0].elapsed_time(ev_assigned) / 1e3
            objective = engine.mean_from_sum(sums[0], n)
            objective_sq = engine.mean_from_sum(sums[1], n)
            if previous is not None and objective == previous:
                trace.append(IterationStats(iteration, objective, objective_sq, assign_seconds, 0.0))
                converged = True
                break

            start = time.perf_counter()
            empty = int(stats[engine._lib.STAT_EMPTY])
            if empty:
                if graphs is not None:
                    graphs.repair.replay()
                else:
                    eng.repair()
            cur.copy_(eng.new_centers)
            torch.cuda.current_stream(dev).synchronize()
            update_seconds = ev_assigned.elapsed_time(ev[2]) / 1e3 + (time.perf_counter() - start)
            filled = int(stats[engine._lib.STAT_FILLED])
            nnz_total = int(stats[engine._lib.STAT_NNZ_TOTAL])
            mean_nnz = nnz_total / (filled * m_count) if filled else 0.0
            trace.append(
                IterationStats(
                    iteration,
                    objective,
                    objective_sq,
                    assign_seconds,
                    update_seconds,
                    repaired_clusters=empty,
                    mean_histogram_nnz=None if update == "naive" else mean_nnz,
                )
            )
            previous = objective
            if graphs is None and device_scan and use_graphs and iteration < max_iterations:
                graphs = engine.IterationGraphs(eng, cur)
        labels = eng.labels_host().copy()
        final_centers = engine.download_codes(cur, m_count).astype(np.uint8)
    return ClusteringResult(final_centers, labels, trace, len(trace), converged)
