"""GPU product vs the reference's own outputs (golden vectors from
tests/golden/make_golden.py): assign + sd, fit traces (incl. BASELINE config 1 at
full size), encode, sparse vote, objective tree."""

import numpy as np
import pytest

from golden_io import fit_case, fit_expect, load, same_nnz, tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_assign_golden(pqk):
    from paper_1709_03708_b200 import engine

    g = load("assign")
    for i in range(int(g["ncases"])):
        t = tables(g, f"c{i}_")
        codes, centers = g[f"c{i}_codes"], g[f"c{i}_centers"]
        np.testing.assert_array_equal(pqk.assign(codes, centers, t), g[f"c{i}_labels"])
        labels, sd = engine.assign_host(codes, centers, t, want_sd=True)
        np.testing.assert_array_equal(labels, g[f"c{i}_labels"])
        assert sd.tobytes() == g[f"c{i}_sd"].tobytes()
        assert pqk.paired_distance_sq(t, codes, centers[labels]).tobytes() == g[f"c{i}_sd"].tobytes()


def _check(res, exp):
    np.testing.assert_array_equal(res.labels, exp["labels"])
    np.testing.assert_array_equal(res.centers, exp["centers"])
    assert res.labels.dtype == np.uint32 and res.centers.dtype == np.uint8
    assert res.iterations_run == exp["iterations_run"]
    assert res.converged == exp["converged"]
    assert [s.objective for s in res.trace] == list(exp["objective"])
    assert [s.objective_sq for s in res.trace] == list(exp["objective_sq"])
    assert [s.repaired_clusters for s in res.trace] == list(exp["repaired"])
    assert all(same_nnz(s.mean_histogram_nnz, e) for s, e in zip(res.trace, exp["nnz"]))


def test_fit_golden(pqk):
    g = load("fit")
    for i in range(int(g["ncases"])):
        c = fit_case(g, i)
        res = pqk.fit(c["codes"], c["tables"], c["k"], c["it"], c["seed"], update=c["update"],
                      initial_centers=c["init"])
        _check(res, fit_expect(g, f"f{i}_"))
        zero = g[f"f{i}_update_zero"]
        assert [s.update_seconds == 0.0 for s in res.trace] == list(zero)


def test_config1_full_size_golden(pqk):
    """BASELINE.json configs[0] end to end: reference encode, tables and 10-iteration fit."""
    g = load("config1")
    book = pqk.PQCodebook(g["codebook"])
    np.testing.assert_array_equal(pqk.encode(book, g["vectors_head"]), g["codes_head"])
    t = pqk.build_distance_tables(book)
    import hashlib

    assert hashlib.sha256(t.tables.tobytes()).hexdigest() == str(g["tables_sha256"])
    res = pqk.fit(g["codes"], t, 1000, max_iterations=10, seed=7)
    _check(res, fit_expect(g, ""))


def test_encode_golden(pqk):
    g = load("encode")
    for i in range(int(g["ncases"])):
        got = pqk.encode(pqk.PQCodebook(g[f"e{i}_codewords"]), g[f"e{i}_vectors"])
        np.testing.assert_array_equal(got, g[f"e{i}_codes"])
    for t in ("t0", "t1"):
        np.testing.assert_array_equal(pqk.encode(pqk.PQCodebook(g[f"{t}_codewords"]), g[f"{t}_vectors"]),
                                      g[f"{t}_codes"])


def test_vote_golden(pqk):
    g = load("vote")
    cache = {}
    for i in range(int(g["ncases"])):
        key = str(g[f"v{i}_key"])
        if key not in cache:
            cache[key] = tables(g, key + "_")
        t = cache[key]
        members = g[f"v{i}_members"]
        hists = [pqk.build_histogram(members[:, m], t.shape[1]) for m in range(t.shape[0])]
        np.testing.assert_array_equal(pqk.update_center_sparse(hists, t), g[f"v{i}_center"])
        np.testing.assert_array_equal(pqk.update_center_naive(members, t), g[f"v{i}_center"])


def test_objective_tree_golden():
    import torch

    from paper_1709_03708_b200 import engine

    g = load("tables_mean")
    dev = engine.device_of()
    for n in g["sizes"]:
        x = g[f"m{n}_x"]
        got = engine.mean_objectives(torch.from_numpy(x).to(dev), int(n), dev)
        assert got == tuple(g[f"m{n}_mean"])


def test_reference_plugin_boundary(pqk):
    """b200_assign_strategy behaves like the reference linear scan for the golden cases."""
    g = load("assign")
    for i in range(int(g["ncases"])):
        t = tables(g, f"c{i}_")
        got = pqk.b200_assign_strategy(g[f"c{i}_codes"].astype(np.int32), g[f"c{i}_centers"], t, 8)
        np.testing.assert_array_equal(got, g[f"c{i}_labels"])


def test_build_distance_tables_golden(pqk):
    """pq.build_distance_tables on the GPU vs the reference's tables (SHA-256 of all bytes)."""
    import hashlib

    g = load("tables_mean")
    for i in range(4):
        cw = g[f"b{i}_codebook"] if f"b{i}_codebook" in g else g[f"b{i}_codewords"]
        t = pqk.build_distance_tables(pqk.PQCodebook(cw)).tables
        assert hashlib.sha256(t.tobytes()).hexdigest() == str(g[f"b{i}_tables_sha256"]), i
