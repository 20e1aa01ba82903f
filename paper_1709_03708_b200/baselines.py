"""Original-space evaluation of a clustering on the GPU.

Drop-in replacements for the reference's ``cluster_means`` (baselines.py:26-37) and
``original_space_error`` (baselines.py:385-413), bit-identical to numpy: per-cluster
float64 sums in increasing point index (``np.bincount`` with weights), float64 division,
``np.sum((p - m)**2, axis=1)`` in numpy's pairwise order and ``np.mean`` over numpy's
summation tree (csrc/pqk_eval.cu, csrc/pqk_update.cu).  Device tensors are accepted
for data that should stay resident (``*_device`` functions in ``engine``).
"""

from __future__ import annotations

import numpy as np

from . import engine

try:
    import torch
except ImportError as exc:  # pragma: no cover
    raise ImportError("paper_1709_03708_b200.baselines needs torch") from exc


def _labels_int32(labels: np.ndarray, n: int) -> np.ndarray:
    lab = np.asarray(labels)
    if lab.shape != (n,):
        raise ValueError(f"labels must have shape ({n},), got {lab.shape}")
    if lab.size and not np.issubdtype(lab.dtype, np.integer):
        lab_i = lab.astype(np.int64)
        if not np.array_equal(lab_i, lab):
            raise ValueError("labels must be integers")
        lab = lab_i
    if lab.size and lab.min() < 0:
        raise ValueError("labels must be non-negative")  # np.bincount's own condition
    if lab.size and lab.max() >= 2**31 - 1:
        raise ValueError("labels too large")
    return np.ascontiguousarray(lab, dtype=np.int32)


def cluster_means(points: np.ndarray, labels: np.ndarray, k: int, *, device=None) -> np.ndarray:
    """Per-cluster float64 means; rows of empty clusters are zero (baselines.py:26-37)."""
    pts = np.asarray(points)
    if pts.ndim != 2:
        raise ValueError(f"points must be 2-d, got shape {pts.shape}")
    n, d = pts.shape
    lab = _labels_int32(labels, n)
    if lab.size and int(lab.max()) >= k:
        raise ValueError(f"labels must be < k={k}")  # np.bincount(minlength=k) would grow
    if n == 0 or d == 0:
        return np.zeros((k, d), dtype=np.float64)
    dev = engine.device_of(device)
    if pts.dtype == np.float32:
        x = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    else:
        x = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).to(dev)
    means = engine.cluster_means_device(x, torch.from_numpy(lab).to(dev), int(k), dev)
    return means.cpu().numpy()


def original_space_error(vectors: np.ndarray, labels: np.ndarray, *, device=None) -> float:
    """Mean distance of each vector to the mean of its assigned cluster (baselines.py:385-413)."""
    data = np.asarray(vectors, dtype=np.float32)
    labels = np.asarray(labels)
    if data.ndim != 2:
        raise ValueError(f"vectors must be 2-d, got shape {data.shape}")
    if labels.shape != (len(data),):
        raise ValueError(f"labels must have shape ({len(data)},), got {labels.shape}")
    if len(data) == 0:
        raise ValueError("cannot evaluate an empty dataset")
    lab = _labels_int32(labels, len(data))
    k = int(lab.max()) + 1
    dev = engine.device_of(device)
    x = torch.from_numpy(np.ascontiguousarray(data)).to(dev)
    if data.shape[1] == 0:
        return 0.0
    return engine.original_space_error_device(x, torch.from_numpy(lab).to(dev), k, dev)


# ---------------------------------------------------------------------------
# Bk-means baseline: k-means on packed binary codes with Hamming
# assignment and per-bit majority votes (baselines.py:157-382), on the GPU
# (csrc/pqk_binary.cu, plus the PQ path's repair and objective kernels).
from dataclasses import dataclass  # noqa: E402
import time  # noqa: E402

from . import _lib  # noqa: E402
from .clustering import ClusteringResult, IterationStats  # noqa: E402


@dataclass(frozen=True)
class Binarizer:
    """Maps real vectors to B-bit codes by signs of a rotation (baselines.py:157-187).

    Attributes:
        rotation: float64 matrix of shape (D, B) with orthonormal columns. Bit b of a
            vector x is 1 iff (x @ rotation)[b] >= 0.
    """

    rotation: np.ndarray

    def __post_init__(self) -> None:
        rot = np.ascontiguousarray(self.rotation, dtype=np.float64)
        if rot.ndim != 2:
            raise ValueError(f"rotation must be 2-d, got shape {rot.shape}")
        gram = rot.T @ rot
        if not np.allclose(gram, np.eye(rot.shape[1]), atol=1e-6):
            raise ValueError("rotation columns must be orthonormal within 1e-6")
        rot.flags.writeable = False
        object.__setattr__(self, "rotation", rot)

    @property
    def dim(self) -> int:
        return self.rotation.shape[0]

    @property
    def bits(self) -> int:
        return self.rotation.shape[1]


def train_binarizer(dim: int, bits: int, seed: int = 0) -> Binarizer:
    """Random orthonormal rotation (baselines.py:190-209): the reference's seeded Gaussian
    draw and QR with sign-normalised columns.  A one-off (D x B) setup, computed on the
    host with the same numpy/LAPACK calls as the reference so the rotation is identical."""
    if bits % 8 != 0 or bits < 8:
        raise ValueError(f"bits must be a positive multiple of 8, got {bits}")
    if bits > dim:
        raise ValueError(f"bits={bits} exceeds vector dimension {dim}")
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((dim, bits)))
    q = q * np.where(np.diag(r) >= 0, 1.0, -1.0)
    return Binarizer(q)


def binarize(binarizer: Binarizer, vectors: np.ndarray, *, device=None) -> np.ndarray:
    """Packed codes (B/8,) or (N, B/8) (baselines.py:212-234): bit b = (x . R_b >= 0) with
    the exact sign of the float64 projection, MSB first within each byte."""
    arr = np.asarray(vectors, dtype=np.float32)
    single = arr.ndim == 1
    arr = np.atleast_2d(arr)
    if arr.shape[1] != binarizer.dim:
        raise ValueError(f"vectors have dimension {arr.shape[1]}, binarizer expects {binarizer.dim}")
    dev = engine.device_of(device)
    width = binarizer.bits // 8
    n = len(arr)
    out = torch.zeros((max(n, 1), width), dtype=torch.uint8, device=dev)
    stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
    if n:
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        rot = torch.from_numpy(np.array(binarizer.rotation)).to(dev)
        engine.call("pqk_binarize_device", engine._ptr(x), n, binarizer.dim, engine._ptr(rot), binarizer.bits,
                    engine._ptr(out), width, engine._ptr(stats), engine._stream(dev))
    packed = out[:n].cpu().numpy()
    return packed[0] if single else packed


def unpack_bits(codes: np.ndarray, bits: int) -> np.ndarray:
    """Expand packed codes (N, B/8) into a 0/1 matrix (N, B) (baselines.py:237-239)."""
    return np.unpackbits(np.atleast_2d(codes), axis=1, count=bits)


def _wp(width: int) -> int:
    for wp in (4, 8, 16, 32):
        if width <= wp:
            return wp
    raise ValueError(f"binary codes of {8 * width} bits exceed the 256-bit device layout")


def _upload_packed(packed: np.ndarray, dev) -> "torch.Tensor":
    n, width = packed.shape
    wp = _wp(width)
    buf = np.zeros((max(n, 1), wp), dtype=np.uint8)
    buf[:n, :width] = packed
    return torch.from_numpy(buf).to(dev)


def hamming_to_centers(codes: np.ndarray, centers: np.ndarray, *, device=None) -> np.ndarray:
    """Hamming distances between packed codes (N, W) and centers (K, W) (baselines.py:285-288)."""
    a = np.atleast_2d(np.asarray(codes, dtype=np.uint8))
    b = np.atleast_2d(np.asarray(centers, dtype=np.uint8))
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"code widths differ: {a.shape[1]} vs {b.shape[1]}")
    dev = engine.device_of(device)
    n, k = len(a), len(b)
    out = torch.zeros((max(n * k, 1),), dtype=torch.int32, device=dev)
    if n and k:
        a_dev, b_dev = _upload_packed(a, dev), _upload_packed(b, dev)  # kept alive across the call
        engine.call("pqk_hamming_matrix_device", engine._ptr(a_dev), n, _wp(a.shape[1]), engine._ptr(b_dev), k,
                    engine._ptr(out), engine._stream(dev))
    return out[: n * k].cpu().numpy().astype(np.int64).reshape(n, k)


def majority_center(member_bits: np.ndarray, *, device=None) -> np.ndarray:
    """Per-bit majority vote over one cluster's members (baselines.py:253-282): bit b is
    1 iff strictly more than half of the members have it (ties give 0)."""
    bits_arr = np.asarray(member_bits)
    if bits_arr.ndim != 2 or len(bits_arr) == 0:
        raise ValueError(f"member_bits must be a non-empty 2-d 0/1 array, got shape {bits_arr.shape}")
    if bits_arr.size and not np.isin(bits_arr, (0, 1)).all():
        raise ValueError("member_bits entries must be 0 or 1")
    n, nbits = bits_arr.shape
    if nbits == 0:
        return np.zeros(0, dtype=np.uint8)
    padded_bits = -(-nbits // 8) * 8
    packed = np.packbits(bits_arr.astype(np.uint8), axis=1)
    dev = engine.device_of(device)
    wp = _wp(packed.shape[1])
    codes = _upload_packed(packed, dev)
    labels = torch.zeros(n, dtype=torch.int32, device=dev)
    counts = torch.zeros(1, dtype=torch.int32, device=dev)
    ones = torch.zeros(padded_bits, dtype=torch.int32, device=dev)
    newc = torch.zeros((1, wp), dtype=torch.uint8, device=dev)
    stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
    engine.call("pqk_majority_update_device", engine._ptr(codes), n, wp, padded_bits, engine._ptr(labels), 1,
                engine._ptr(counts), engine._ptr(ones), engine._ptr(newc), engine._ptr(stats), engine._stream(dev))
    return np.unpackbits(newc.cpu().numpy()[0])[:nbits].astype(np.uint8)


class _BinaryShard:
    """Device state of a Bk-means fit (codes, centers, labels, sd, counts, ones)."""

    def __init__(self, packed: np.ndarray, k: int, dev):
        self.dev = dev
        self.n, self.width = packed.shape
        self.bits = 8 * self.width
        self.wp = _wp(self.width)
        self.k = k
        self.codes = _upload_packed(packed, dev)
        self.labels = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.sd = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.counts = torch.empty(k, dtype=torch.int32, device=dev)
        self.ones = torch.empty((k, self.bits), dtype=torch.int32, device=dev)
        self.new_centers = torch.zeros((k, self.wp), dtype=torch.uint8, device=dev)
        self.stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
        self.plan = engine.pairwise_plan(self.n, dev)
        self.obj = torch.zeros(2, dtype=torch.float64, device=dev)
        self.repair_ws = engine._empty(_lib.load().pqk_repair_workspace_bytes(self.n, k), dev)

    def upload_centers(self, centers: np.ndarray) -> "torch.Tensor":
        return _upload_packed(centers, self.dev)[: self.k]

    def assign(self, centers_dev) -> None:
        engine.call("pqk_hamming_assign_device", engine._ptr(self.codes), self.n, self.wp, engine._ptr(centers_dev),
                    self.k, engine._ptr(self.labels), engine._ptr(self.sd), None, engine._stream(self.dev))
        engine.objective_sums(self.sd, self.plan, self.obj, self.dev)

    def update(self) -> int:
        engine.call("pqk_majority_update_device", engine._ptr(self.codes), self.n, self.wp, self.bits,
                    engine._ptr(self.labels), self.k, engine._ptr(self.counts), engine._ptr(self.ones),
                    engine._ptr(self.new_centers), engine._ptr(self.stats), engine._stream(self.dev))
        empty = int(self.stats[_lib.STAT_EMPTY].item())
        if empty:
            engine.call("pqk_repair_device", engine._ptr(self.sd), engine._ptr(self.codes), self.n, self.wp,
                        engine._ptr(self.counts), self.k, engine._ptr(self.new_centers), engine._ptr(self.repair_ws),
                        self.repair_ws.numel(), engine._ptr(self.stats), engine._stream(self.dev))
        return empty


def bkmeans_fit(codes: np.ndarray, k: int, max_iterations: int = 20, seed: int = 0, *, threads: int = 1,
                initial_centers: np.ndarray | None = None, device=None) -> ClusteringResult:
    """K-means on packed binary codes (baselines.py:291-382) on the GPU: Hamming assignment
    (lowest index on ties), per-bit majority update, the PQk-means stop rule and
    empty-cluster repair; the trace objective is the mean Hamming distance.  ``threads``
    is accepted for signature compatibility (the GPU ignores it)."""
    packed = np.asarray(codes, dtype=np.uint8)
    if packed.ndim != 2 or packed.shape[1] == 0:
        raise ValueError(f"codes must have shape (N, B/8), got {packed.shape}")
    n, width = packed.shape
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    if max_iterations < 1:
        raise ValueError(f"max_iterations must be positive, got {max_iterations}")
    if initial_centers is None:
        rng = np.random.default_rng(seed)
        centers = packed[rng.choice(n, size=k, replace=False)].copy()
    else:
        centers = np.asarray(initial_centers, dtype=np.uint8).copy()
        if centers.shape != (k, width):
            raise ValueError(f"initial_centers must have shape ({k}, {width}), got {centers.shape}")
    dev = engine.device_of(device)
    with torch.cuda.device(dev):
        sh = _BinaryShard(packed, k, dev)
        cur = sh.upload_centers(centers)
        trace: list[IterationStats] = []
        previous = None
        converged = False
        for iteration in range(1, max_iterations + 1):
            t0 = time.perf_counter()
            sh.assign(cur)
            s = sh.obj.cpu().numpy()
            assign_seconds = time.perf_counter() - t0
            objective = engine.mean_from_sum(s[0], n)
            objective_sq = engine.mean_from_sum(s[1], n)
            if previous is not None and objective == previous:
                trace.append(IterationStats(iteration, objective, objective_sq, assign_seconds, 0.0))
                converged = True
                break
            t1 = time.perf_counter()
            empty = sh.update()
            nxt = sh.new_centers.clone()
            torch.cuda.current_stream(dev).synchronize()
            update_seconds = time.perf_counter() - t1
            trace.append(IterationStats(iteration, objective, objective_sq, assign_seconds, update_seconds,
                                        repaired_clusters=empty))
            cur = nxt
            previous = objective
        centers_out = cur.cpu().numpy()[:, :width].copy()
        labels = sh.labels.cpu().numpy().astype(np.uint32)
    return ClusteringResult(centers_out, labels, trace, len(trace), converged)
