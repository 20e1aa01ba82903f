"""GPU parity of pqk_histogram_device (clustering.py:344-347 bincount per subspace and the
counts of clustering.py:458) against the oracle: the cluster-tiled counting-sort path
(bucket count -> scan -> scatter -> shared-memory tile counts) for K up to ~1e6 at M=4,
and the global-atomic path beyond its bucket limit.  Integer counts: exact equality."""

import numpy as np
import pytest

from oracle import pqk_oracle as O

pytestmark = pytest.mark.gpu


def _run(codes, labels, k, l_count, to_host=True):
    import torch

    from paper_1709_03708_b200 import _lib
    from paper_1709_03708_b200.engine import _ptr, _stream

    dev = torch.device("cuda:0")
    n, m = codes.shape
    mp = _lib.padded_m(m)
    d_codes = torch.zeros((max(n, 1), mp), dtype=torch.uint8, device=dev)
    if n:
        d_codes[:n, :m] = torch.from_numpy(codes).to(dev)
    d_labels = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint32).view(np.int32)).to(dev)
    # garbage-filled outputs: the kernel must write every entry (zeros included)
    hist = torch.full((k, m, l_count), -1, dtype=torch.int32, device=dev)
    counts = torch.full((k,), -1, dtype=torch.int32, device=dev)
    _lib.call("pqk_histogram_device", _ptr(d_codes), n, m, l_count, _ptr(d_labels), k, _ptr(hist), _ptr(counts),
              _stream(dev))
    torch.cuda.synchronize(dev)
    if not to_host:
        return hist, counts
    return hist.cpu().numpy().astype(np.int64), counts.cpu().numpy().astype(np.int64)


def _check(codes, labels, k, l_count):
    hist, counts = _run(codes, labels, k, l_count)
    exp = O.histogram(codes, labels, k, l_count)
    np.testing.assert_array_equal(hist, exp)
    np.testing.assert_array_equal(counts, np.bincount(labels.astype(np.int64), minlength=k))


@pytest.mark.parametrize(
    "n,k,m,l_count",
    [
        (200_000, 100_000, 4, 256),  # config 4's K: 4167 tiles of 24 clusters, most clusters empty
        (300_000, 10_000, 4, 256),  # config 2's K
        (100_000, 20_003, 16, 256),  # config 5's M, K not a multiple of the tile
        (50_000, 999, 3, 12),  # padded codes (M=3 -> 4 bytes), short codebooks
        (40_000, 7, 8, 64),
        (10_000, 1, 2, 256),
        (1, 5, 4, 256),
    ],
)
def test_histogram_random(n, k, m, l_count):
    rng = np.random.default_rng(n + k + m)
    codes = rng.integers(0, l_count, size=(n, m), dtype=np.uint8)
    labels = rng.integers(0, k, size=n).astype(np.uint32)
    _check(codes, labels, k, l_count)


def test_histogram_empty_input():
    hist, counts = _run(np.zeros((0, 4), np.uint8), np.zeros(0, np.uint32), 300, 256)
    assert not hist.any() and not counts.any()


def test_histogram_skewed():
    """One giant cluster of identical codes plus a clustered tail (same-address shared atomics)."""
    rng = np.random.default_rng(3)
    n, k = 300_000, 50_000
    codes = np.repeat(rng.integers(0, 256, size=(1, 4), dtype=np.uint8), n, axis=0)
    labels = np.full(n, 31_337, dtype=np.uint32)
    tail = rng.random(n) < 0.2
    labels[tail] = rng.integers(0, 64, size=int(tail.sum()))
    codes[tail, 1] = rng.integers(0, 3, size=int(tail.sum()))
    _check(codes, labels, k, 256)


def test_histogram_clustered_mixture():
    from helpers import mixture_codes

    codes = mixture_codes(120_000, 4, 256, 500, seed=9)
    rng = np.random.default_rng(10)
    labels = rng.integers(0, 30_000, size=len(codes)).astype(np.uint32)
    _check(codes, labels, 30_000, 256)


def test_histogram_atomic_path_beyond_bucket_limit():
    """M=24: 4 clusters per 96 KB tile, so K=170,000 exceeds the 40,960-bucket limit and the
    global-atomic kernel runs (a 4.2 GB table)."""
    rng = np.random.default_rng(5)
    n, k, m = 30_000, 170_000, 24
    codes = rng.integers(0, 256, size=(n, m), dtype=np.uint8)
    labels = rng.integers(0, k, size=n).astype(np.uint32)
    import torch

    hist, counts = _run(codes, labels, k, 256, to_host=False)
    # compare the touched clusters densely; the whole table must sum to n*m (no stray -1)
    exp_counts = np.bincount(labels.astype(np.int64), minlength=k)
    np.testing.assert_array_equal(counts.cpu().numpy(), exp_counts)
    touched = np.unique(labels)
    rel = np.searchsorted(touched, labels)
    exp = O.histogram(codes, rel.astype(np.uint32), len(touched), 256)
    got = hist[torch.from_numpy(touched.astype(np.int64)).to(hist.device)].cpu().numpy()
    np.testing.assert_array_equal(got, exp)
    assert int(hist.min()) == 0 and int(hist.sum(dtype=torch.int64)) == n * m


@pytest.mark.skipif(bool(__import__("os").environ.get("PQK_HIST_MODE")), reason="already inside a forced-mode child")
@pytest.mark.parametrize("mode", ["tiled", "atomic"])
def test_histogram_forced_path(mode):
    """The cases above again with one path forced for every shape (PQK_HIST_MODE is read
    once per process, so each mode runs in a child pytest)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, PQK_HIST_MODE=mode)
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(here, "test_gpu_histogram.py"), "-k", "random or empty or skewed or mixture"],
        env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
