"""GPU codebook training (pq.train_codebook, pq.py:155-202) vs the reference's own
codewords: small cases incl. empty-codeword reseeds, and the full BASELINE config-1
codebook (20,000 x 128 sample, M=4, L=256, 20 iterations)."""

import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_train_golden(pqk):
    g = load("train")
    for i in range(int(g["ncases"])):
        m, l_count, it, seed = (int(v) for v in g[f"t{i}_args"])
        book = pqk.train_codebook(g[f"t{i}_x"], m, l_count, iterations=it, seed=seed)
        assert book.codewords.tobytes() == g[f"t{i}_book"].tobytes(), i


def test_train_config1_codebook(pqk):
    """Regenerate config 1's training sample (make_golden.make_config1) and reproduce
    the reference codebook bit for bit."""
    rng = np.random.default_rng(1234)
    means = rng.uniform(0.0, 100.0, size=(1000, 128))
    lab = rng.integers(0, 1000, size=100_000)
    vectors = (means[lab] + rng.normal(0.0, 5.0, size=(100_000, 128))).astype(np.float32)
    sample = vectors[np.random.default_rng(1235).choice(100_000, 20_000, replace=False)]
    book = pqk.train_codebook(sample, 4, 256, iterations=20, seed=1)
    assert book.codewords.tobytes() == load("config1")["codebook"].tobytes()


def test_train_validation(pqk):
    data = np.zeros((100, 10), dtype=np.float32)
    with pytest.raises(ValueError, match="divisible"):
        pqk.train_codebook(data, 3, 8)
    with pytest.raises(ValueError, match="num_codewords"):
        pqk.train_codebook(data, 2, 300)
    with pytest.raises(ValueError, match="training vectors"):
        pqk.train_codebook(data[:5], 2, 8)
    with pytest.raises(ValueError, match="iterations"):
        pqk.train_codebook(data, 2, 8, iterations=0)
