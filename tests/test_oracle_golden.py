"""Pin the oracle to the reference: every golden vector in tests/golden was
produced by running the reference package (tests/golden/make_golden.py).  These
tests run on CPU (`-m "not gpu"`)."""

import numpy as np
import pytest

from golden_io import fit_case, fit_expect, load, same_nnz, tables
from oracle import pqk_oracle as O


def test_tables_rebuilt_bit_exact():
    g = load("tables_mean")
    for i in range(4):
        t = O.build_distance_tables(g[f"b{i}_codebook"] if f"b{i}_codebook" in g else g[f"b{i}_codewords"])
        import hashlib

        assert hashlib.sha256(t.tobytes()).hexdigest() == str(g[f"b{i}_tables_sha256"])
        pick = g[f"b{i}_pick"]
        assert t[pick[:, 0], pick[:, 1], pick[:, 2]].tobytes() == g[f"b{i}_values"].tobytes()


def test_assign_golden():
    g = load("assign")
    for i in range(int(g["ncases"])):
        t = tables(g, f"c{i}_")
        codes, centers = g[f"c{i}_codes"], g[f"c{i}_centers"]
        expect = g[f"c{i}_labels"]
        np.testing.assert_array_equal(O.assign_linear_scan(codes, centers, t), expect)
        labels, sd = O.assign_c(codes, centers, t, threads=4, want_sd=True)
        np.testing.assert_array_equal(labels, expect)
        assert sd.tobytes() == g[f"c{i}_sd"].tobytes()
        assert O.paired_distance_sq(t, codes, centers[expect]).tobytes() == g[f"c{i}_sd"].tobytes()


def _check_fit(res, exp):
    np.testing.assert_array_equal(res["labels"], exp["labels"])
    np.testing.assert_array_equal(res["centers"], exp["centers"])
    assert res["iterations_run"] == exp["iterations_run"]
    assert res["converged"] == exp["converged"]
    assert [t["objective"] for t in res["trace"]] == list(exp["objective"])
    assert [t["objective_sq"] for t in res["trace"]] == list(exp["objective_sq"])
    assert [t["repaired"] for t in res["trace"]] == list(exp["repaired"])
    assert all(same_nnz(t["nnz"], e) for t, e in zip(res["trace"], exp["nnz"]))


def test_fit_golden():
    g = load("fit")
    for i in range(int(g["ncases"])):
        c = fit_case(g, i)
        res = O.fit(c["codes"], c["tables"], c["k"], c["it"], c["seed"], update=c["update"],
                    initial_centers=c["init"], scan=O.assign_c)
        _check_fit(res, fit_expect(g, f"f{i}_"))


def test_config1_full_size_golden():
    """BASELINE.json configs[0] (N=1e5, K=1e3, M=4, 10 iterations), reference outputs."""
    g = load("config1")
    t = O.build_distance_tables(g["codebook"])
    import hashlib

    assert hashlib.sha256(t.tobytes()).hexdigest() == str(g["tables_sha256"])
    np.testing.assert_array_equal(O.encode(g["codebook"], g["vectors_head"]), g["codes_head"])
    res = O.fit(g["codes"], t, 1000, 10, 7, scan=O.assign_c)
    _check_fit(res, fit_expect(g, ""))


def test_encode_golden():
    g = load("encode")
    for i in range(int(g["ncases"])):
        np.testing.assert_array_equal(O.encode(g[f"e{i}_codewords"], g[f"e{i}_vectors"]), g[f"e{i}_codes"])
    for t in ("t0", "t1"):
        np.testing.assert_array_equal(O.encode(g[f"{t}_codewords"], g[f"{t}_vectors"]), g[f"{t}_codes"])


def test_vote_golden():
    g = load("vote")
    cache = {}
    for i in range(int(g["ncases"])):
        key = str(g[f"v{i}_key"])
        if key not in cache:
            cache[key] = tables(g, key + "_")
        t = cache[key]
        members = g[f"v{i}_members"]
        got = [O.vote_argmin(np.bincount(members[:, m], minlength=t.shape[1]), t[m]) for m in range(t.shape[0])]
        np.testing.assert_array_equal(got, g[f"v{i}_center"])


def test_objective_tree_golden():
    g = load("tables_mean")
    for n in g["sizes"]:
        x = g[f"m{n}_x"]
        mean = g[f"m{n}_mean"]
        assert O.pairwise_sum(np.sqrt(x)) / n == mean[0]
        assert O.pairwise_sum(x) / n == mean[1]
        assert O.objective(x) == (mean[0], mean[1])


def test_train_codebook_golden():
    """Oracle restatement of pq.train_codebook vs the reference's own codewords."""
    g = load("train")
    for i in range(int(g["ncases"])):
        m, l_count, it, seed = (int(v) for v in g[f"t{i}_args"])
        got = O.train_codebook(g[f"t{i}_x"], m, l_count, iterations=it, seed=seed)
        assert got.tobytes() == g[f"t{i}_book"].tobytes(), i


def test_baselines_golden():
    """Oracle cluster_means / original_space_error vs the reference's own outputs."""
    g = load("baselines")
    for i in range(int(g["ncases"])):
        x, lab, k = g[f"b{i}_x"], g[f"b{i}_labels"], int(g[f"b{i}_k"])
        assert O.cluster_means(x.astype(np.float64), lab, k).tobytes() == g[f"b{i}_means"].tobytes(), i
        assert O.cluster_means(x, lab, k).tobytes() == g[f"b{i}_means32"].tobytes(), i
        assert O.original_space_error(x, lab) == float(g[f"b{i}_err"]), i


def test_bkmeans_golden():
    """Oracle Bk-means pieces vs the reference's own outputs (baselines.py:157-382)."""
    g = load("bkmeans")
    for i in range(int(g["nbin"])):
        assert np.array_equal(O.binarize(g[f"z{i}_rot"], g[f"z{i}_x"]), g[f"z{i}_codes"]), i
    assert np.array_equal(O.hamming_to_centers(g["h_a"], g["h_b"]), g["h_d"])
    reps = 0
    for i in range(int(g["nfit"])):
        k, it, seed = (int(v) for v in g[f"f{i}_args"])
        init = g[f"f{i}_init"] if len(g[f"f{i}_init"]) else None
        ref = O.bkmeans_fit(g[f"f{i}_codes"], k, it, seed, initial_centers=init)
        assert np.array_equal(ref["centers"], g[f"f{i}_centers"]), i
        assert np.array_equal(ref["labels"], g[f"f{i}_labels"]), i
        assert [t["objective"] for t in ref["trace"]] == list(g[f"f{i}_obj"]), i
        assert [t["objective_sq"] for t in ref["trace"]] == list(g[f"f{i}_obj_sq"]), i
        assert [t["repaired"] for t in ref["trace"]] == list(g[f"f{i}_rep"]), i
        assert ref["converged"] == bool(g[f"f{i}_conv"]), i
        reps += int(np.sum(g[f"f{i}_rep"]))
    assert reps > 0  # the repair path is exercised
