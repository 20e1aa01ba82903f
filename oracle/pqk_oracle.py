"""CPU oracle for the PQk-means hot path — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference algorithm (arXiv 1709.03708,
/root/reference/pkg/src/pqclust) used as the checker of the B200 kernels.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may
import it; the product package never does.

Pinning: every function is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports /root/reference and
writes ``tests/golden/*.npz``) in ``tests/test_oracle_golden.py``.

Semantics restated (file:line of the reference):
- assign_linear_scan    clustering.py:167-197  fp64 gather-add in ascending m starting
                        from 0.0, np.argmin (lowest index on ties)
- paired_distance_sq    pq.py:271-290           fp64 ascending m
- objective             clustering.py:448-449   np.mean (numpy pairwise summation)
- pairwise_sum          numpy/_core/src/umath/loops_utils.h.src (restated in Python)
- histogram             clustering.py:344-347   bincount(labels*L + codes[:,m])
- vote_argmin           clustering.py:349-354   argmin_j sum_s h_s T[s][j], lowest j;
                        the reference evaluates the votes with an OpenBLAS dgemv
                        (order unpinned); the oracle decides the exact-arithmetic
                        argmin: fp64 votes with a rounding certificate, exact
                        rational arithmetic (fractions.Fraction) on near ties.
- sparse_update_all     clustering.py:327-356
- repair                clustering.py:460-466
- fit                   clustering.py:377-482
- encode                pq.py:205-231, _nearest pq.py:114-116 (scipy cdist
                        sqeuclidean = sequential fp64 sum of (x-c)^2, no FMA)
- build_distance_tables pq.py:254-268
- train_codebook        pq.py:127-202 (_lloyd_subspace, empty-codeword reseed)
- cluster_means         baselines.py:26-37      per-dimension np.bincount with weights:
                        float64 sums in increasing point index, / counts
- original_space_error  baselines.py:385-413    np.sum((p - m)**2, axis=1) (pairwise
                        over the row), np.mean(np.sqrt(.)) (pairwise over N)
- binarize              baselines.py:212-234    sign of the float64 projection (exact
                        rational sign here; the reference's dgemm order is unpinned)
- hamming / majority    baselines.py:242-288    popcount(xor), 2 * ones > count
- bkmeans_fit           baselines.py:291-382
"""

from __future__ import annotations

import ctypes as C
import math
import os
from fractions import Fraction
from pathlib import Path

import numpy as np

_CHUNK_BUDGET = 1 << 22  # clustering.py:24


def chunk_bounds(n: int, k: int) -> list[tuple[int, int]]:
    """clustering.py:160-164 (depends on N and K only)."""
    chunk = max(1, min(8192, _CHUNK_BUDGET // max(k, 1)))
    return [(s, min(s + chunk, n)) for s in range(0, n, chunk)]


def assign_linear_scan(codes: np.ndarray, centers: np.ndarray, tables: np.ndarray) -> np.ndarray:
    """clustering.py:167-197: labels = argmin_k sum_m T[m][x^m][c_k^m] (fp64, ascending m)."""
    codes = np.asarray(codes)
    centers = np.asarray(centers)
    n, m_count = codes.shape
    k = len(centers)
    restricted = [np.ascontiguousarray(tables[m][:, centers[:, m]]) for m in range(m_count)]
    labels = np.empty(n, dtype=np.uint32)
    for start, stop in chunk_bounds(n, k):
        acc = np.zeros((stop - start, k), dtype=np.float64)
        for m in range(m_count):
            acc += restricted[m][codes[start:stop, m]]
        labels[start:stop] = np.argmin(acc, axis=1)
    return labels


def paired_distance_sq(tables: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """pq.py:271-290."""
    acc = np.zeros(len(a), dtype=np.float64)
    for m in range(tables.shape[0]):
        acc += tables[m][a[:, m], b[:, m]]
    return acc


def pairwise_sum(a) -> float:
    """numpy's pairwise summation (loops_utils.h.src, PW_BLOCKSIZE=128), pure Python."""
    a = [float(x) for x in a]

    def rec(lo: int, n: int) -> float:
        if n < 8:
            res = 0.0
            for i in range(n):
                res += a[lo + i]
            return res
        if n <= 128:
            r = a[lo : lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, len(a))


def objective(sd_sq: np.ndarray) -> tuple[float, float]:
    """clustering.py:448-449."""
    return float(np.mean(np.sqrt(sd_sq))), float(np.mean(sd_sq))


def histogram(codes: np.ndarray, labels: np.ndarray, k: int, l_count: int) -> np.ndarray:
    """clustering.py:344-347 for every m: (K, M, L) int64."""
    m_count = codes.shape[1]
    joint = labels.astype(np.int64) * l_count
    out = np.empty((k, m_count, l_count), dtype=np.int64)
    for m in range(m_count):
        out[:, m, :] = np.bincount(joint + codes[:, m], minlength=k * l_count).reshape(k, l_count)
    return out


def vote_argmin(counts_row: np.ndarray, table: np.ndarray) -> int:
    """Exact-arithmetic argmin_j sum_s h_s T[s][j], lowest j on exact ties (clustering.py:349-354)."""
    support = np.flatnonzero(counts_row)
    w = counts_row[support].astype(np.float64)
    rows = table[support]
    votes = w @ rows
    order = np.argsort(votes, kind="stable")
    best, second = int(order[0]), (int(order[1]) if len(order) > 1 else None)
    if second is None:
        return best
    v1, v2 = votes[best], votes[second]
    margin = 4.0 * (len(support) + 2) * 2.0**-53
    if v2 - v1 > margin * v2:
        return best
    # near tie: exact rationals for every candidate inside the band
    band = v1 + 2 * margin * max(v2, 1e-300) + 1e-300
    cands = [j for j in range(table.shape[1]) if votes[j] <= band]
    exact = {
        j: sum(Fraction(int(counts_row[s])) * Fraction(float(table[s, j])) for s in support) for j in cands
    }
    lo = min(exact.values())
    return min(j for j, v in exact.items() if v == lo)


def sparse_update_all(codes, labels, counts, tables) -> tuple[np.ndarray, float]:
    """clustering.py:327-356 (exact-arithmetic vote argmin)."""
    k = len(counts)
    m_count, l_count = tables.shape[0], tables.shape[1]
    centers = np.zeros((k, m_count), dtype=np.uint8)
    filled = np.flatnonzero(counts > 0)
    hist = histogram(codes, labels, k, l_count)
    nnz_total = 0
    for m in range(m_count):
        for ki in filled:
            row = hist[ki, m]
            nnz_total += int(np.count_nonzero(row))
            centers[ki, m] = vote_argmin(row, tables[m])
    mean_nnz = nnz_total / (len(filled) * m_count) if len(filled) else 0.0
    return centers, mean_nnz


def repair(new_centers: np.ndarray, counts: np.ndarray, sd_sq: np.ndarray, codes: np.ndarray) -> int:
    """clustering.py:460-466; returns the number of repaired clusters."""
    empty = np.flatnonzero(counts == 0)
    if len(empty):
        own = sd_sq.copy()
        for ki in empty:
            far = int(np.argmax(own))
            new_centers[ki] = codes[far]
            own[far] = -np.inf
    return len(empty)


def init_centers(codes: np.ndarray, k: int, seed: int = 0) -> np.ndarray:
    """clustering.py:149-157."""
    rng = np.random.default_rng(seed)
    return codes[rng.choice(len(codes), size=k, replace=False)].copy()


def fit(codes, tables, k, max_iterations=20, seed=0, *, update="sparse", initial_centers=None, scan=None):
    """clustering.py:377-482 restated; returns dict(centers, labels, trace, iterations_run, converged).

    ``scan`` optionally replaces assign_linear_scan (e.g. the C restatement).
    """
    scan = scan or assign_linear_scan
    codes = np.asarray(codes)
    m_count = tables.shape[0]
    centers = init_centers(codes, k, seed) if initial_centers is None else np.asarray(initial_centers).astype(np.uint8)
    trace = []
    labels = np.zeros(len(codes), dtype=np.uint32)
    previous = None
    converged = False
    for iteration in range(1, max_iterations + 1):
        labels = scan(codes, centers, tables)
        sd_sq = paired_distance_sq(tables, codes, centers[labels])
        obj, obj_sq = objective(sd_sq)
        if previous is not None and obj == previous:
            trace.append(dict(iteration=iteration, objective=obj, objective_sq=obj_sq, repaired=0, nnz=None))
            converged = True
            break
        counts = np.bincount(labels.astype(np.intp), minlength=k)
        new_centers, mean_nnz = sparse_update_all(codes, labels, counts, tables)
        rep = repair(new_centers, counts, sd_sq, codes)
        trace.append(
            dict(
                iteration=iteration,
                objective=obj,
                objective_sq=obj_sq,
                repaired=rep,
                nnz=None if update == "naive" else mean_nnz,
            )
        )
        centers = new_centers
        previous = obj
    return dict(centers=centers, labels=labels, trace=trace, iterations_run=len(trace), converged=converged)


def encode(codewords: np.ndarray, vectors: np.ndarray) -> np.ndarray:
    """pq.py:205-231: nearest codeword per subspace, fp64 sequential squared distance."""
    arr = np.atleast_2d(np.asarray(vectors, dtype=np.float32)).astype(np.float64)
    m_count, l_count, sub = codewords.shape
    out = np.empty((len(arr), m_count), dtype=np.uint8)
    for m in range(m_count):
        pts = arr[:, m * sub : (m + 1) * sub]
        cw = codewords[m].astype(np.float64)
        acc = np.zeros((len(arr), l_count), dtype=np.float64)
        for d in range(sub):
            diff = pts[:, None, d] - cw[None, :, d]
            acc += diff * diff
        out[:, m] = np.argmin(acc, axis=1)
    return out


def _nearest_f64(points: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """pq.py:114-116 with scipy cdist("sqeuclidean") restated: sequential (x-c)*(x-c) sums."""
    acc = np.zeros((len(points), len(centers)), dtype=np.float64)
    for d in range(points.shape[1]):
        diff = points[:, None, d] - centers[None, :, d]
        acc += diff * diff
    return np.argmin(acc, axis=1)


def _lloyd_subspace(sub: np.ndarray, num_codewords: int, iterations: int, rng) -> np.ndarray:
    """pq.py:127-152: float64 Lloyd with farthest-point reseed of empty codewords."""
    points = sub.astype(np.float64)
    n = len(points)
    centers = points[rng.choice(n, size=num_codewords, replace=False)].copy()
    for _ in range(iterations):
        labels = _nearest_f64(points, centers)
        counts = np.bincount(labels, minlength=num_codewords)
        sums = np.stack([np.bincount(labels, weights=points[:, d], minlength=num_codewords)
                         for d in range(points.shape[1])], axis=1)  # pq.py:119-124
        filled = counts > 0
        centers[filled] = sums[filled] / counts[filled, None]
        if not filled.all():
            own = np.sum((points - centers[labels]) ** 2, axis=1)
            for slot in np.flatnonzero(~filled):
                far = int(np.argmax(own))
                centers[slot] = points[far]
                labels[far] = slot
                own[far] = -np.inf
    return centers


def train_codebook(train_vectors: np.ndarray, num_subspaces: int, num_codewords: int, iterations: int = 20,
                   seed: int = 0) -> np.ndarray:
    """pq.py:155-202 (one Generator shared across subspaces); returns (M, L, D/M) float32."""
    vectors = np.asarray(train_vectors, dtype=np.float32)
    n, dim = vectors.shape
    sub_dim = dim // num_subspaces
    rng = np.random.default_rng(seed)
    books = np.empty((num_subspaces, num_codewords, sub_dim), dtype=np.float32)
    for m in range(num_subspaces):
        sub = vectors[:, m * sub_dim : (m + 1) * sub_dim]
        books[m] = _lloyd_subspace(sub, num_codewords, iterations, rng).astype(np.float32)
    return books


def build_distance_tables(codewords: np.ndarray) -> np.ndarray:
    """pq.py:254-268: sequential fp64 squared distances between codewords."""
    m_count, l_count, sub = codewords.shape
    t = np.empty((m_count, l_count, l_count), dtype=np.float64)
    for m in range(m_count):
        cw = codewords[m].astype(np.float64)
        acc = np.zeros((l_count, l_count), dtype=np.float64)
        for d in range(sub):
            diff = cw[:, None, d] - cw[None, :, d]
            acc += diff * diff
        t[m] = acc
    return t


def cluster_means(points: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    """baselines.py:26-37: float64 sums in point-index order (a sequential loop, which is
    what np.bincount(weights=...) does), divided by the counts; empty rows stay 0."""
    pts = np.asarray(points, dtype=np.float64)
    lab = np.asarray(labels).astype(np.intp)
    sums = np.zeros((k, pts.shape[1]))
    counts = np.zeros(k)
    for i in range(len(pts)):  # sequential, index order
        sums[lab[i]] += pts[i]
        counts[lab[i]] += 1.0
    out = np.zeros_like(sums)
    filled = counts > 0
    out[filled] = sums[filled] / counts[filled][:, None]
    return out


def row_pairwise_sq(points: np.ndarray, centers: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """np.sum((points - centers[labels])**2, axis=1): numpy's pairwise sum per row."""
    diff2 = (np.asarray(points, dtype=np.float64) - centers[np.asarray(labels).astype(np.intp)]) ** 2
    return np.array([pairwise_sum(r) for r in diff2])


def original_space_error(vectors: np.ndarray, labels: np.ndarray) -> float:
    """baselines.py:385-413."""
    points = np.asarray(vectors, dtype=np.float32).astype(np.float64)
    lab = np.asarray(labels)
    k = int(lab.max()) + 1
    means = cluster_means(points, lab, k)
    sq = row_pairwise_sq(points, means, lab)
    return float(np.float64(pairwise_sum(np.sqrt(sq))) / len(sq))


_POPCOUNT = np.array([bin(v).count("1") for v in range(256)], dtype=np.uint8)


def binarize(rotation: np.ndarray, vectors: np.ndarray) -> np.ndarray:
    """baselines.py:212-234 with the exact sign of x . R_b (Fraction arithmetic on the
    float64 values), packed MSB-first (np.packbits)."""
    x = np.atleast_2d(np.asarray(vectors, dtype=np.float32)).astype(np.float64)
    proj = x @ rotation
    bits = (proj >= 0).astype(np.uint8)
    # exact sign where the float64 product could be off (|proj| below its error bound)
    bound = (x.shape[1] + 2) * 2.0**-52 * (np.abs(x) @ np.abs(rotation))
    for i, b in zip(*np.nonzero(np.abs(proj) <= bound)):
        v = sum(Fraction(float(x[i, k])) * Fraction(float(rotation[k, b])) for k in range(x.shape[1]))
        bits[i, b] = 1 if v >= 0 else 0
    return np.packbits(bits, axis=1)


def hamming_to_centers(codes: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """baselines.py:285-288."""
    xor = codes[:, None, :] ^ centers[None, :, :]
    return _POPCOUNT[xor].sum(axis=2, dtype=np.int64)


def majority_center(member_bits: np.ndarray) -> np.ndarray:
    """baselines.py:253-282: bit = 2 * ones > count (ties give 0)."""
    ones = np.asarray(member_bits).sum(axis=0, dtype=np.int64)
    return (2 * ones > len(member_bits)).astype(np.uint8)


def bkmeans_fit(codes, k, max_iterations=20, seed=0, *, initial_centers=None):
    """baselines.py:291-382 (single-threaded restatement)."""
    packed = np.asarray(codes, dtype=np.uint8)
    n, width = packed.shape
    bits = 8 * width
    if initial_centers is None:
        centers = packed[np.random.default_rng(seed).choice(n, size=k, replace=False)].copy()
    else:
        centers = np.asarray(initial_centers, dtype=np.uint8).copy()
    trace = []
    previous = None
    converged = False
    labels = np.zeros(n, dtype=np.uint32)
    for _ in range(max_iterations):
        labels = np.argmin(hamming_to_centers(packed, centers), axis=1).astype(np.uint32)
        dist = _POPCOUNT[packed ^ centers[labels]].sum(axis=1, dtype=np.int64)
        objective = float(np.mean(dist))
        objective_sq = float(np.mean(dist.astype(np.float64) ** 2))
        if previous is not None and objective == previous:
            trace.append({"objective": objective, "objective_sq": objective_sq, "repaired": 0})
            converged = True
            break
        counts = np.bincount(labels.astype(np.intp), minlength=k)
        new_centers = np.zeros((k, width), dtype=np.uint8)
        for ki in np.flatnonzero(counts > 0):
            members = np.unpackbits(packed[labels == ki], axis=1, count=bits)
            new_centers[ki] = np.packbits(majority_center(members))
        empty = np.flatnonzero(counts == 0)
        own = dist.astype(np.float64)
        for ki in empty:
            far = int(np.argmax(own))
            new_centers[ki] = packed[far]
            own[far] = -np.inf
        trace.append({"objective": objective, "objective_sq": objective_sq, "repaired": len(empty)})
        centers = new_centers
        previous = objective
    return {"centers": centers, "labels": labels, "trace": trace, "converged": converged}


# ---------------------------------------------------------------------------
# C restatement of the scan (oracle/pqk_scan.c), multithreaded, for large cases and
# the CPU baseline.  Built by oracle/Makefile into oracle/libpqk_oracle.so.
_C_LIB = None


def c_lib():
    global _C_LIB
    if _C_LIB is None:
        path = Path(__file__).resolve().parent / "libpqk_oracle.so"
        if not path.exists():
            raise ImportError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(str(path))
        lib.oracle_assign.restype = C.c_int
        lib.oracle_assign.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_void_p, C.c_int32]
        _C_LIB = lib
    return _C_LIB


def assign_c(codes: np.ndarray, centers: np.ndarray, tables: np.ndarray, threads: int | None = None,
             want_sd: bool = False):
    """Same result as assign_linear_scan, computed by the C restatement."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    centers = np.ascontiguousarray(centers, dtype=np.uint8)
    tables = np.ascontiguousarray(tables, dtype=np.float64)
    n, m = codes.shape
    labels = np.empty(n, dtype=np.uint32)
    sd = np.empty(n, dtype=np.float64)
    threads = threads or os.cpu_count() or 1
    rc = c_lib().oracle_assign(codes.ctypes.data, n, m, centers.ctypes.data, len(centers), tables.ctypes.data,
                               tables.shape[1], labels.ctypes.data, sd.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_assign failed ({rc})")
    return (labels, sd) if want_sd else labels
