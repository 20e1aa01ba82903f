"""GPU original-space evaluation: cluster_means and
original_space_error (baselines.py:26-37, 385-413) bit-identical to the reference's
golden outputs and to the oracle, incl. empty clusters, float64 inputs, d > 128
(recursive pairwise rows) and a larger skewed case through the radix sort."""

import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_eval_golden(pqk):
    g = load("baselines")
    for i in range(int(g["ncases"])):
        x, lab, k = g[f"b{i}_x"], g[f"b{i}_labels"], int(g[f"b{i}_k"])
        assert pqk.cluster_means(x.astype(np.float64), lab, k).tobytes() == g[f"b{i}_means"].tobytes(), i
        assert pqk.cluster_means(x, lab, k).tobytes() == g[f"b{i}_means32"].tobytes(), i
        assert pqk.original_space_error(x, lab) == float(g[f"b{i}_err"]), i


def test_eval_large_skewed_matches_oracle(pqk, oracle):
    """200k points, K=3000 with a Zipf-like label skew (one cluster holds ~10%): three
    radix passes over 12-bit labels, long member lists, multi-level scans."""
    rng = np.random.default_rng(5)
    n, d, k = 200_000, 24, 3000
    x = (rng.normal(size=(n, d)) * 3 + 1).astype(np.float32)
    lab = np.minimum(rng.zipf(1.3, size=n) - 1, k - 1).astype(np.int64)
    lab[:: 97] = k - 1
    got = pqk.cluster_means(x, lab, k)
    ref = np.zeros((k, d))
    cnt = np.bincount(lab, minlength=k)
    sums = np.stack([np.bincount(lab, weights=x[:, j].astype(np.float64), minlength=k) for j in range(d)], axis=1)
    np.divide(sums, cnt[:, None], out=ref, where=cnt[:, None] > 0)
    assert got.tobytes() == ref.tobytes()
    err = pqk.original_space_error(x, lab)
    sq = np.sum((x.astype(np.float64) - ref[lab]) ** 2, axis=1)
    assert err == float(np.mean(np.sqrt(sq)))


def test_eval_validation(pqk):
    x = np.zeros((10, 3), np.float32)
    with pytest.raises(ValueError, match="2-d"):
        pqk.original_space_error(np.zeros(5, np.float32), np.zeros(5, int))
    with pytest.raises(ValueError, match="shape"):
        pqk.original_space_error(x, np.zeros(9, int))
    with pytest.raises(ValueError, match="empty"):
        pqk.original_space_error(np.zeros((0, 3), np.float32), np.zeros(0, int))
    with pytest.raises(ValueError, match="non-negative"):
        pqk.cluster_means(x, -np.ones(10, int), 3)
