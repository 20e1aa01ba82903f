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
