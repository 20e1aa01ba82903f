"""GPU parity of the assignment scan (labels + exact fp64 sd) against the oracle.

Mirrors the reference's own assignment tests: brute force
(test_clustering.py:119-133), ties toward the low index incl. duplicate centers
(:135-143), acceptance C4 lattice ties + duplicated center rows
(test_acceptance.py:175-236); plus every padded-M kernel variant and sizes that
exercise multi-pass persistent scheduling.
"""

import numpy as np
import pytest

from helpers import lattice_tables, mixture_codes, random_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def _check(pqk, oracle, codes, centers, tables):
    from paper_1709_03708_b200 import engine

    labels, sd = engine.assign_host(codes, centers, tables, want_sd=True)
    expect = oracle.assign_c(codes, centers, tables)
    assert labels.dtype == np.uint32
    np.testing.assert_array_equal(labels, expect)
    exp_sd = oracle.paired_distance_sq(tables, codes.astype(np.int64), centers[expect].astype(np.int64))
    assert sd.tobytes() == exp_sd.tobytes()


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 12, 16, 24, 32, 40])
@pytest.mark.parametrize("l_count", [4, 16, 256])
def test_random_tables_all_widths(pqk, oracle, m, l_count):
    rng = np.random.default_rng(1000 * m + l_count)
    tables = random_tables(m, l_count, seed=m + l_count)
    codes = rng.integers(0, l_count, size=(1500, m)).astype(np.uint8)
    centers = rng.integers(0, l_count, size=(77, m)).astype(np.uint8)
    _check(pqk, oracle, codes, centers, tables)


def test_ties_toward_low_index(pqk):
    tables = lattice_tables(1, 8)
    codes = np.array([[3]], dtype=np.uint8)
    assert pqk.assign(codes, np.array([[2], [4]], dtype=np.uint8), tables)[0] == 0
    assert pqk.assign(codes, np.array([[4], [2]], dtype=np.uint8), tables)[0] == 0
    assert pqk.assign(codes, np.array([[5], [5], [2]], dtype=np.uint8), tables)[0] == 2
    assert pqk.assign(codes, np.array([[5], [5]], dtype=np.uint8), tables)[0] == 0


@pytest.mark.parametrize("trial", range(10))
def test_lattice_ties_and_duplicate_centers(pqk, oracle, trial):
    rng = np.random.default_rng(404 + trial)
    m = int(rng.choice([1, 2, 4]))
    tables = lattice_tables(m, 16)
    codes = rng.integers(0, 16, size=(2000, m)).astype(np.uint8)
    centers = rng.integers(0, 16, size=(40, m)).astype(np.uint8)
    centers[5] = centers[2]
    centers[30] = centers[2]
    _check(pqk, oracle, codes, centers, tables)


@pytest.mark.parametrize("n,k,m", [(100_000, 1000, 4), (60_000, 4096, 4), (50_000, 700, 8), (30_000, 333, 16)])
def test_large_multipass(pqk, oracle, n, k, m):
    rng = np.random.default_rng(n + k + m)
    tables = random_tables(m, 256, seed=7, sub_dim=8)
    codes = mixture_codes(n, m, 256, 500, seed=k)
    centers = codes[rng.choice(n, size=k, replace=False)]
    _check(pqk, oracle, codes, centers, tables)


def test_single_center_and_all_identical(pqk, oracle):
    tables = random_tables(4, 64, seed=3)
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 64, size=(999, 4)).astype(np.uint8)
    _check(pqk, oracle, codes, codes[:1], tables)
    _check(pqk, oracle, codes, np.repeat(codes[:1], 50, axis=0), tables)


def test_strategy_plugin_any_dtype(pqk, oracle):
    tables = random_tables(3, 16, seed=8)
    rng = np.random.default_rng(7)
    codes = rng.integers(0, 16, size=(120, 3)).astype(np.int64)
    centers = rng.integers(0, 16, size=(9, 3)).astype(np.int16)[:, ::1]
    got = pqk.b200_assign_strategy(codes, centers, type("T", (), {"tables": tables})(), 8)
    np.testing.assert_array_equal(got, oracle.assign_linear_scan(codes, centers, tables))


def test_validation(pqk):
    tables = random_tables(2, 8)
    codes = np.zeros((4, 2), dtype=np.uint8)
    with pytest.raises(ValueError, match="non-empty"):
        pqk.assign(codes, np.empty((0, 2), dtype=np.uint8), tables)
    with pytest.raises(ValueError, match="unknown assignment strategy"):
        pqk.assign(codes, codes[:1], tables, strategy="nope")
    with pytest.raises(ValueError, match="shape"):
        pqk.assign(np.zeros((4, 3), dtype=np.uint8), codes[:1], tables)
