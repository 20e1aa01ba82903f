"""Edge cases of the public API on the GPU, against the reference's behaviour (via the
oracle / reference semantics): empty inputs, single rows, maximum codeword counts,
K = N, all-identical codes, single-vector encode, and the reference's error messages."""

import numpy as np
import pytest

from helpers import random_codebook, random_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_empty_inputs(pqk, oracle):
    book = random_codebook(4, 256, 8, seed=1)
    tables = oracle.build_distance_tables(book)
    empty = np.zeros((0, 32), np.float32)
    codes = pqk.encode(pqk.PQCodebook(book), empty)
    assert codes.shape == (0, 4) and codes.dtype == np.uint8
    labels = pqk.assign(np.zeros((0, 4), np.uint8), np.zeros((3, 4), np.uint8), tables)
    assert labels.shape == (0,) and labels.dtype == np.uint32
    sd = pqk.paired_distance_sq(tables, np.zeros((0, 4), np.uint8), np.zeros((0, 4), np.uint8))
    assert sd.shape == (0,)
    with pytest.raises(ValueError, match="k must be"):
        pqk.fit(np.zeros((0, 4), np.uint8), tables, 1)


def test_single_vector_and_single_row(pqk, oracle):
    book = random_codebook(2, 256, 16, seed=2)
    x = np.random.default_rng(3).normal(size=32).astype(np.float32)
    code = pqk.encode(pqk.PQCodebook(book), x)
    assert code.shape == (2,) and np.array_equal(code, oracle.encode(book, x[None])[0])
    tables = oracle.build_distance_tables(book)
    res = pqk.fit(code[None], tables, 1, max_iterations=3)
    assert np.array_equal(res.labels, [0]) and res.trace[-1].objective == 0.0


def test_k_equals_n_and_identical_codes(pqk, oracle):
    tables = random_tables(4, 256, seed=4, sub_dim=4)
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 256, size=(500, 4)).astype(np.uint8)
    res = pqk.fit(codes, tables, 500, max_iterations=4, seed=1)
    ref = oracle.fit(codes, tables, 500, max_iterations=4, seed=1, scan=oracle.assign_c)
    assert np.array_equal(res.labels, ref["labels"]) and res.trace[0].objective == 0.0
    same = np.repeat(codes[:1], 300, axis=0)
    res = pqk.fit(same, tables, 7, max_iterations=5, seed=2)
    ref = oracle.fit(same, tables, 7, max_iterations=5, seed=2, scan=oracle.assign_c)
    assert np.array_equal(res.labels, ref["labels"]) and np.array_equal(res.centers, ref["centers"])
    assert [s.repaired_clusters for s in res.trace] == [t["repaired"] for t in ref["trace"]]


@pytest.mark.parametrize("l_count", [2, 3, 255, 256])
def test_codeword_counts(pqk, oracle, l_count):
    """L from the minimum to the maximum (MAX_CODEWORDS = 256): encode and a short fit."""
    book = random_codebook(3, l_count, 8, seed=l_count)
    x = np.random.default_rng(l_count).normal(size=(3000, 24)).astype(np.float32)
    codes = pqk.encode(pqk.PQCodebook(book), x)
    assert np.array_equal(codes, oracle.encode(book, x))
    tables = oracle.build_distance_tables(book)
    res = pqk.fit(codes, tables, min(20, len(np.unique(codes, axis=0))), max_iterations=4, seed=3)
    ref = oracle.fit(codes, tables, min(20, len(np.unique(codes, axis=0))), max_iterations=4, seed=3,
                     scan=oracle.assign_c)
    assert np.array_equal(res.labels, ref["labels"]) and np.array_equal(res.centers, ref["centers"])


def test_reference_error_messages(pqk, oracle):
    tables = random_tables(2, 8, seed=6)
    codes = np.zeros((10, 2), np.uint8)
    with pytest.raises(ValueError, match="max_iterations must be positive"):
        pqk.fit(codes, tables, 2, max_iterations=0)
    with pytest.raises(ValueError, match="update must be"):
        pqk.fit(codes, tables, 2, update="dense")
    with pytest.raises(ValueError, match="initial_centers has 3 rows"):
        pqk.fit(codes, tables, 2, initial_centers=np.zeros((3, 2), np.uint8))
    with pytest.raises(ValueError, match="unknown assignment strategy"):
        pqk.assign(codes, codes[:2], tables, strategy="nope")
    with pytest.raises(ValueError):
        pqk.assign(np.full((3, 2), 9, np.uint8), codes[:2], tables)  # subindex >= L


@pytest.mark.parametrize("k,distinct", [(30_000, 100), (5000, 4000), (2100, 50)])
def test_repair_many_empty_clusters(pqk, oracle, k, distinct):
    """E close to K (the sorted-candidate network covers up to min(N, K) = 2^15 keys and
    more): one fit iteration's repair must place exactly the reference's farthest codes
    (clustering.py:460-466: sd descending, lowest index first)."""
    rng = np.random.default_rng(k + distinct)
    tables = random_tables(4, 256, seed=distinct)
    protos = rng.integers(0, 256, size=(distinct, 4))
    codes = protos[rng.integers(0, distinct, size=40_000)].astype(np.uint8)
    res = pqk.fit(codes, tables, k, max_iterations=2, seed=5)
    ref = oracle.fit(codes, tables, k, max_iterations=2, seed=5, scan=lambda c, ce, t: oracle.assign_c(c, ce, t))
    assert res.trace[0].repaired_clusters == ref["trace"][0]["repaired"] > k // 3
    np.testing.assert_array_equal(res.centers, ref["centers"])
    np.testing.assert_array_equal(res.labels, ref["labels"])
