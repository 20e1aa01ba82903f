"""GPU `fit` parity with the oracle: labels, centers, objective traces (exact
floats), repaired clusters, histogram occupancy, iterations and convergence.

Known answers from the reference tests (test_clustering.py:233-305): K=N reaches
objective 0; separated groups recovered; empty cluster reseeded on the farthest
code; sparse/naive agree; monotone squared objective (C3).
"""

import numpy as np
import pytest

from helpers import lattice_tables, mixture_codes, random_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def _compare(res, ref):
    np.testing.assert_array_equal(res.labels, ref["labels"])
    np.testing.assert_array_equal(res.centers, ref["centers"])
    assert res.iterations_run == ref["iterations_run"]
    assert res.converged == ref["converged"]
    for s, r in zip(res.trace, ref["trace"]):
        assert s.objective == r["objective"]
        assert s.objective_sq == r["objective_sq"]
        assert s.repaired_clusters == r["repaired"]
        assert s.mean_histogram_nnz == r["nnz"]


@pytest.mark.parametrize("trial", range(12))
def test_fit_matches_oracle_random(pqk, oracle, trial):
    rng = np.random.default_rng(30 + trial)
    m = int(rng.choice([1, 2, 3, 4, 8]))
    l_count = int(rng.choice([8, 32, 256]))
    tables = random_tables(m, l_count, seed=100 + trial)
    n = int(rng.integers(200, 6000))
    codes = rng.integers(0, l_count, size=(n, m)).astype(np.uint8)
    k = int(rng.integers(2, 60))
    res = pqk.fit(codes, tables, k, max_iterations=15, seed=trial)
    ref = oracle.fit(codes, tables, k, max_iterations=15, seed=trial, scan=oracle.assign_c)
    _compare(res, ref)
    sq = [s.objective_sq for s in res.trace]
    assert all(b <= a for a, b in zip(sq, sq[1:]))


@pytest.mark.parametrize("trial", range(4))
def test_fit_clustered_with_repairs(pqk, oracle, trial):
    m = 4
    tables = random_tables(m, 256, seed=7 + trial, sub_dim=8)
    codes = mixture_codes(20000, m, 256, 300, seed=trial)
    res = pqk.fit(codes, tables, 400, max_iterations=6, seed=trial)
    ref = oracle.fit(codes, tables, 400, max_iterations=6, seed=trial, scan=oracle.assign_c)
    _compare(res, ref)


def test_k_equals_n_reaches_zero_objective(pqk):
    tables = lattice_tables(2, 32)
    rng = np.random.default_rng(20)
    codes = np.unique(rng.integers(0, 32, size=(64, 2), dtype=np.uint8), axis=0)
    result = pqk.fit(codes, tables, len(codes), seed=0)
    assert result.converged
    assert result.trace[-1].objective == 0.0
    assert result.trace[-1].objective_sq == 0.0
    assert len(set(result.labels.tolist())) == len(codes)


def test_separated_groups_recovered(pqk):
    tables = lattice_tables(1, 200)
    codes = np.array([0, 1, 2, 99, 100, 101, 197, 198, 199], dtype=np.uint8).reshape(-1, 1)
    initial = np.array([[1], [100], [198]], dtype=np.uint8)
    result = pqk.fit(codes, tables, 3, seed=0, initial_centers=initial)
    assert result.converged
    assert np.array_equal(result.labels, np.repeat([0, 1, 2], 3))
    assert np.array_equal(result.centers, initial)


def test_empty_cluster_reseeded_on_farthest_code(pqk):
    tables = lattice_tables(1, 6)
    codes = np.array([[0], [0], [5], [5]], dtype=np.uint8)
    initial = np.array([[0], [0]], dtype=np.uint8)
    result = pqk.fit(codes, tables, 2, seed=0, initial_centers=initial)
    assert result.trace[0].repaired_clusters == 1
    assert result.converged
    assert np.array_equal(result.labels, [0, 0, 1, 1])


def test_sparse_and_naive_agree(pqk):
    rng = np.random.default_rng(31)
    tables = random_tables(4, 64, seed=32)
    codes = rng.integers(0, 64, size=(3000, 4), dtype=np.uint8)
    sparse = pqk.fit(codes, tables, 12, seed=5, update="sparse")
    naive = pqk.fit(codes, tables, 12, seed=5, update="naive")
    assert np.array_equal(sparse.labels, naive.labels)
    assert np.array_equal(sparse.centers, naive.centers)
    assert [s.objective for s in sparse.trace] == [s.objective for s in naive.trace]
    assert all(s.mean_histogram_nnz is None for s in naive.trace)
    assert any(s.mean_histogram_nnz is not None for s in sparse.trace)


def test_validation(pqk):
    tables = lattice_tables(1, 4)
    codes = np.zeros((5, 1), dtype=np.uint8)
    with pytest.raises(ValueError, match="k must be"):
        pqk.fit(codes, tables, 0)
    with pytest.raises(ValueError, match="k must be"):
        pqk.fit(codes, tables, 6)
    with pytest.raises(ValueError, match="max_iterations"):
        pqk.fit(codes, tables, 2, max_iterations=0)
    with pytest.raises(ValueError, match="update must be"):
        pqk.fit(codes, tables, 2, update="fancy")
    with pytest.raises(ValueError, match="initial_centers has"):
        pqk.fit(codes, tables, 2, initial_centers=np.zeros((3, 1), dtype=np.uint8))


@pytest.mark.parametrize("m,n,k,iters", [(16, 120_000, 3000, 4), (32, 30_000, 700, 3), (12, 20_000, 1500, 3)])
def test_fit_long_codes_matches_oracle(pqk, oracle, m, n, k, iters):
    """Long codes (BASELINE config 5's M=16, and M=32 / a padded M=12) on clustered data:
    the M=16/32 scan variants, their vote and repair paths, several K chunks."""
    tables = random_tables(m, 256, seed=50 + m, sub_dim=4)
    codes = mixture_codes(n, m, 256, 400, seed=m)
    res = pqk.fit(codes, tables, k, max_iterations=iters, seed=m)
    ref = oracle.fit(codes, tables, k, max_iterations=iters, seed=m, scan=oracle.assign_c)
    _compare(res, ref)


def test_graph_replay_equals_eager(pqk, oracle, monkeypatch):
    """Iterations 2.. replay CUDA graphs (engine.IterationGraphs); same result as eager
    launches and as the oracle, with repairs inside the replayed iterations."""
    from paper_1709_03708_b200 import clustering, engine

    tables = random_tables(4, 256, seed=21, sub_dim=8)
    codes = mixture_codes(20_011, 4, 256, 50, seed=22)
    k, iters, seed = 500, 8, 3
    made = []
    real = engine.IterationGraphs

    def spy(*a, **kw):
        g = real(*a, **kw)
        made.append(g)
        return g

    monkeypatch.setattr(engine, "IterationGraphs", spy)
    graphed = pqk.fit(codes, tables, k, iters, seed)
    assert len(made) == 1 and made[0].main_launches > 0 and made[0].repair_launches > 0
    monkeypatch.setattr(clustering, "USE_CUDA_GRAPHS", False)
    eager = pqk.fit(codes, tables, k, iters, seed)
    ref = oracle.fit(codes, tables, k, iters, seed, scan=oracle.assign_c)
    for res in (graphed, eager):
        np.testing.assert_array_equal(res.labels, ref["labels"])
        np.testing.assert_array_equal(res.centers, ref["centers"])
        assert [s.objective for s in res.trace] == [t["objective"] for t in ref["trace"]]
        assert [s.repaired_clusters for s in res.trace] == [t["repaired"] for t in ref["trace"]]
    assert sum(t["repaired"] for t in ref["trace"][1:]) > 0
