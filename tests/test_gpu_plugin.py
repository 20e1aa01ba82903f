"""The reference's own plugin path, run for real.

The unmodified reference package (`pip install --no-deps --target baseline/_ref` of
/root/reference/pkg; git-ignored, it travels with the snapshot) is imported, the B200
scan is registered into *its* strategy registry (clustering.py:207-216) and
`pqclust.fit(..., strategy="b200")` / `pqclust.assign(..., strategy="b200")`
(clustering.py:255-282, 377-482) must equal the reference's own `linear_scan` run.
Two registrations are covered: INTEGRATION.md's ctypes stub (tests/pqclust_b200.py,
calling `pqk_assign_host` / `pqk_encode_host` of the C-ABI) and the package's
`b200_assign_strategy`.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def pqclust():
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "pqclust").exists():
        pytest.skip("reference not installed in baseline/_ref (pip install --no-deps --target baseline/_ref)")
    sys.path.insert(0, str(ref))
    import pqclust as mod

    assert str(ref) in mod.__file__
    yield mod
    for name in ("b200",):
        mod.unregister_assignment_strategy(name)


@pytest.fixture(scope="module")
def stub(pqclust):
    os.environ.setdefault("PQK_B200_LIB", str(ROOT / "paper_1709_03708_b200" / "libpqk_b200.so"))
    import pqclust_b200

    return pqclust_b200


def _workload(pqclust, n, k_true, seed, m=4, dim=32):
    rng = np.random.default_rng(seed)
    protos = rng.normal(scale=4.0, size=(k_true, dim)).astype(np.float32)
    x = (protos[rng.integers(0, k_true, size=n)] + rng.normal(size=(n, dim))).astype(np.float32)
    book = pqclust.train_codebook(x[: min(n, 5000)], m, 256, iterations=5, seed=seed)
    codes = pqclust.encode(book, x)
    return x, book, codes, pqclust.build_distance_tables(book)


def _same_result(a, b):
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.centers, b.centers)
    assert a.iterations_run == b.iterations_run and a.converged == b.converged
    assert [t.objective for t in a.trace] == [t.objective for t in b.trace]
    assert [t.objective_sq for t in a.trace] == [t.objective_sq for t in b.trace]
    assert [t.repaired_clusters for t in a.trace] == [t.repaired_clusters for t in b.trace]


def test_stub_fit_equals_linear_scan(pqclust, stub):
    """INTEGRATION.md's ctypes stub registered into the unmodified pqclust."""
    _, _, codes, tables = _workload(pqclust, 20_000, 300, seed=1)
    stub.enable()
    assert "b200" in pqclust.registered_assignment_strategies()
    got = pqclust.fit(codes, tables, 200, max_iterations=6, seed=3, strategy="b200")
    ref = pqclust.fit(codes, tables, 200, max_iterations=6, seed=3, strategy="linear_scan")
    _same_result(got, ref)


def test_stub_assign_16bit_tier(pqclust, stub):
    """pqclust.assign through the stub where the 16-bit first tier runs (>= 2^31 lookups:
    2e5 codes x 11,000 centers x M=4), against the reference's own linear scan."""
    rng = np.random.default_rng(5)
    _, _, codes, tables = _workload(pqclust, 200_000, 2000, seed=2)
    centers = codes[rng.choice(len(codes), size=11_000, replace=False)]
    stub.enable()
    got = pqclust.assign(codes, centers, tables, strategy="b200")
    ref = pqclust.assign(codes, centers, tables, threads=os.cpu_count() or 1, strategy="linear_scan")
    np.testing.assert_array_equal(got, ref)


def test_stub_encode_equals_reference(pqclust, stub):
    x, book, codes, _ = _workload(pqclust, 30_000, 50, seed=7)
    np.testing.assert_array_equal(stub.b200_encode(book, x), codes)


def test_stub_errors(pqclust, stub):
    _, _, codes, tables = _workload(pqclust, 1000, 10, seed=9)
    with pytest.raises(ValueError):
        stub.b200_assign(codes, codes[:0], tables, 1)  # empty centers -> PQK_EINVAL


def test_package_strategy_fit_equals_linear_scan(pqclust):
    """paper_1709_03708_b200.b200_assign_strategy registered into pqclust (update 'naive' too)."""
    import paper_1709_03708_b200 as pqk

    _, _, codes, tables = _workload(pqclust, 15_000, 100, seed=11, m=8, dim=64)
    pqclust.register_assignment_strategy("b200", pqk.b200_assign_strategy)
    for update in ("sparse", "naive"):
        got = pqclust.fit(codes, tables, 120, max_iterations=5, seed=4, strategy="b200", update=update)
        ref = pqclust.fit(codes, tables, 120, max_iterations=5, seed=4, strategy="linear_scan", update=update)
        _same_result(got, ref)


def test_dropin_fit_equals_reference_fit(pqclust):
    """The drop-in (`import paper_1709_03708_b200 as pqk` instead of pqclust): the whole
    resident iteration on the GPU equals the reference's fit, trace included."""
    import paper_1709_03708_b200 as pqk

    _, _, codes, tables = _workload(pqclust, 20_000, 400, seed=13)
    for update in ("sparse", "naive"):
        got = pqk.fit(codes, pqk.DistanceTables(tables.tables), 250, max_iterations=8, seed=2, update=update)
        ref = pqclust.fit(codes, tables, 250, max_iterations=8, seed=2, update=update)
        _same_result(got, ref)
        assert [t.mean_histogram_nnz for t in got.trace] == [t.mean_histogram_nnz for t in ref.trace]
