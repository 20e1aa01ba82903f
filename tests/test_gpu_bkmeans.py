"""GPU Bk-means baseline against the reference's golden outputs
(baselines.py:157-382): binarize, hamming_to_centers, majority_center, bkmeans_fit
(labels, centers, trace objectives, repairs, convergence), plus the reference tests'
known answers (test_baselines.py) and a larger case against the oracle."""

import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_binarize_golden(pqk):
    g = load("bkmeans")
    for i in range(int(g["nbin"])):
        dim, bits, seed = (int(v) for v in g[f"z{i}_args"])
        bz = pqk.train_binarizer(dim, bits, seed=seed)
        assert bz.rotation.tobytes() == g[f"z{i}_rot"].tobytes(), i
        assert np.array_equal(pqk.binarize(bz, g[f"z{i}_x"]), g[f"z{i}_codes"]), i
        assert np.array_equal(pqk.binarize(bz, g[f"z{i}_x"][3]), g[f"z{i}_codes"][3]), i


def test_hamming_and_majority(pqk, oracle):
    g = load("bkmeans")
    assert np.array_equal(pqk.hamming_to_centers(g["h_a"], g["h_b"]), g["h_d"])
    members = np.array([[1, 0], [1, 0], [1, 1]], dtype=np.uint8)
    assert np.array_equal(pqk.majority_center(members), [1, 0])
    assert np.array_equal(pqk.majority_center(np.array([[1, 0], [0, 0]], dtype=np.uint8)), [0, 0])
    assert np.array_equal(pqk.majority_center(np.array([[0, 1, 1]], dtype=np.uint8)), [0, 1, 1])
    rng = np.random.default_rng(3)
    m = rng.integers(0, 2, size=(41, 37)).astype(np.uint8)
    assert np.array_equal(pqk.majority_center(m), oracle.majority_center(m))
    with pytest.raises(ValueError, match="non-empty"):
        pqk.majority_center(np.empty((0, 4), dtype=np.uint8))
    with pytest.raises(ValueError, match="0 or 1"):
        pqk.majority_center(np.array([[0, 2]], dtype=np.uint8))


def test_bkmeans_golden(pqk):
    g = load("bkmeans")
    for i in range(int(g["nfit"])):
        k, it, seed = (int(v) for v in g[f"f{i}_args"])
        init = g[f"f{i}_init"] if len(g[f"f{i}_init"]) else None
        res = pqk.bkmeans_fit(g[f"f{i}_codes"], k, max_iterations=it, seed=seed, initial_centers=init)
        assert np.array_equal(res.centers, g[f"f{i}_centers"]), i
        assert np.array_equal(res.labels, g[f"f{i}_labels"]), i
        assert [s.objective for s in res.trace] == list(g[f"f{i}_obj"]), i
        assert [s.objective_sq for s in res.trace] == list(g[f"f{i}_obj_sq"]), i
        assert [s.repaired_clusters for s in res.trace] == list(g[f"f{i}_rep"]), i
        assert res.converged == bool(g[f"f{i}_conv"]), i


def test_bkmeans_reference_known_answers(pqk):
    packed = np.array([[0x00, 0x00]] * 4 + [[0xFF, 0xFF]] * 4, dtype=np.uint8)
    initial = np.array([[0x00, 0x00], [0xFF, 0xFF]], dtype=np.uint8)
    res = pqk.bkmeans_fit(packed, 2, initial_centers=initial)
    assert res.converged
    assert np.array_equal(res.labels, [0] * 4 + [1] * 4)
    assert np.array_equal(res.centers, initial)
    assert res.trace[-1].objective == 0.0
    with pytest.raises(ValueError, match="k must be"):
        pqk.bkmeans_fit(packed, 0)
    with pytest.raises(ValueError, match="codes must have shape"):
        pqk.bkmeans_fit(packed.ravel(), 2)
    with pytest.raises(ValueError, match="initial_centers"):
        pqk.bkmeans_fit(packed, 2, initial_centers=np.zeros((2, 3), np.uint8))
    with pytest.raises(ValueError, match="max_iterations"):
        pqk.bkmeans_fit(packed, 2, max_iterations=0)


def test_bkmeans_larger_matches_oracle(pqk, oracle):
    """20k 64-bit codes from binarized SIFT-like vectors, K=500 (several center tiles of
    the assignment kernel are not needed at this K; ties and repairs occur)."""
    from paper_1709_03708_b200 import synth

    x = synth.sift_like(20_000, 7)
    bz = pqk.train_binarizer(128, 64, seed=3)
    codes = pqk.binarize(bz, x)
    assert np.array_equal(codes, oracle.binarize(bz.rotation, x))
    res = pqk.bkmeans_fit(codes, 500, max_iterations=6, seed=2)
    ref = oracle.bkmeans_fit(codes, 500, 6, 2)
    assert np.array_equal(res.labels, ref["labels"])
    assert np.array_equal(res.centers, ref["centers"])
    assert [s.objective for s in res.trace] == [t["objective"] for t in ref["trace"]]


def test_hamming_assign_many_center_tiles(pqk, oracle):
    """K = 30,000 centers of 128 bits: ten shared-memory tiles of the assignment kernel."""
    rng = np.random.default_rng(8)
    codes = rng.integers(0, 256, size=(3000, 16), dtype=np.uint8)
    centers = rng.integers(0, 256, size=(30_000, 16), dtype=np.uint8)
    centers[12_345] = codes[7]  # an exact hit in a late tile
    import torch

    from paper_1709_03708_b200 import baselines, engine

    dev = engine.device_of()
    lab = torch.empty(3000, dtype=torch.int32, device=dev)
    dist = torch.empty(3000, dtype=torch.int32, device=dev)
    codes_dev, centers_dev = baselines._upload_packed(codes, dev), baselines._upload_packed(centers, dev)
    engine.call("pqk_hamming_assign_device", engine._ptr(codes_dev), 3000, 16, engine._ptr(centers_dev), 30_000,
                engine._ptr(lab), None, engine._ptr(dist), engine._stream(dev))
    d = oracle.hamming_to_centers(codes, centers)
    assert np.array_equal(lab.cpu().numpy(), np.argmin(d, axis=1))
    assert np.array_equal(dist.cpu().numpy(), d.min(axis=1))
    assert lab.cpu().numpy()[7] == 12_345
