"""Seeded synthetic stand-ins for the BASELINE.json workloads.

The paper's datasets (SIFT1M/1B, Deep1B, ILSVRC) are not available; these
generators produce inputs with the shapes and value distributions the configs
describe.  Host numpy, used by bench.py and the tests; not part
of the measured path.

- ``mixture``     config 1 / 5: isotropic Gaussian mixture, means U[0,100]^D, sigma 5
- ``sift_like``   config 2 / 4: clip(round(Gamma(0.6, 30))) dims, 8 blocks of 16
                  L2-normalised to 512 (order: gamma -> block scale -> round -> clip)
- ``deep_like``   config 3: ReLU of a Gaussian mixture (means N(0,1), sigma 0.5),
                  L2-normalised
- ``train_codebook_fast`` a short Lloyd on a sample (BLAS distances) for bench set-up;
                  only its tables feed the Lloyd-iteration benchmark.
"""

from __future__ import annotations

import numpy as np


def stage_seed(seed: int, stage: int) -> int:
    """Per-stage seed like the reference CLI's derive_seed (cli.py:47-49)."""
    return int(np.random.SeedSequence([seed, stage]).generate_state(1)[0])


def mixture(n: int, dim: int, components: int, seed: int, *, low=0.0, high=100.0, sigma=5.0, chunk=1 << 18):
    rng = np.random.default_rng(seed)
    means = rng.uniform(low, high, size=(components, dim)).astype(np.float64)
    out = np.empty((n, dim), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        lab = rng.integers(0, components, size=e - s)
        out[s:e] = (means[lab] + rng.normal(0.0, sigma, size=(e - s, dim))).astype(np.float32)
    return out


def sift_like(n: int, seed: int, *, dim=128, blocks=8, chunk=1 << 17):
    rng = np.random.default_rng(seed)
    out = np.empty((n, dim), dtype=np.float32)
    bd = dim // blocks
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        g = rng.gamma(0.6, 30.0, size=(e - s, blocks, bd))
        norm = np.sqrt((g * g).sum(axis=2, keepdims=True))
        g = g * (512.0 / np.maximum(norm, 1e-12))
        out[s:e] = np.clip(np.rint(g), 0, 255).reshape(e - s, dim).astype(np.float32)
    return out


def deep_like(n: int, seed: int, *, dim=4096, components=10_000, sigma=0.5, chunk=1 << 12):
    rng = np.random.default_rng(seed)
    means = rng.normal(0.0, 1.0, size=(components, dim)).astype(np.float32)
    out = np.empty((n, dim), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        lab = rng.integers(0, components, size=e - s)
        x = means[lab] + rng.normal(0.0, sigma, size=(e - s, dim)).astype(np.float32)
        x = np.maximum(x, 0.0)
        x /= np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-12)
        out[s:e] = x
    return out


def train_codebook_fast(sample: np.ndarray, m: int, l_count: int = 256, iterations: int = 8, seed: int = 0):
    """Per-subspace Lloyd with BLAS distances (bench set-up only)."""
    rng = np.random.default_rng(seed)
    n, dim = sample.shape
    sub = dim // m
    books = np.empty((m, l_count, sub), dtype=np.float32)
    for mm in range(m):
        pts = sample[:, mm * sub : (mm + 1) * sub].astype(np.float64)
        cen = pts[rng.choice(n, size=l_count, replace=False)].copy()
        p2 = (pts * pts).sum(1)
        for _ in range(iterations):
            d = p2[:, None] - 2.0 * pts @ cen.T + (cen * cen).sum(1)[None, :]
            lab = np.argmin(d, axis=1)
            cnt = np.bincount(lab, minlength=l_count)
            sums = np.zeros_like(cen)
            np.add.at(sums, lab, pts)
            filled = cnt > 0
            cen[filled] = sums[filled] / cnt[filled, None]
            if not filled.all():
                far = np.argsort(-d[np.arange(n), lab])[: int((~filled).sum())]
                cen[~filled] = pts[far]
        books[mm] = cen.astype(np.float32)
    return books
