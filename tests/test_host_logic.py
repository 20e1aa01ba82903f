"""CPU tests of the host logic and the C-ABI library (no GPU needed)."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from helpers import lattice_tables, random_tables

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    from paper_1709_03708_b200 import _lib

    lib = _lib.load()
    header = (ROOT / "include" / "pqk_b200.h").read_text()
    names = sorted(set(re.findall(r"\b(pqk_\w+)\s*\(", header)))
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), f"{name} declared in pqk_b200.h but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.pqk_abi_version() == 1


def test_padded_m():
    from paper_1709_03708_b200 import _lib

    assert [_lib.padded_m(m) for m in (1, 2, 3, 4, 5, 8, 9, 16, 17, 32, 33)] == [4, 4, 4, 4, 8, 8, 16, 16, 32, 32, 40]


def test_table_scale():
    from paper_1709_03708_b200 import _lib

    lib = _lib.load()

    def scale(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        e, f = C.c_int32(0), C.c_int32(0)
        _lib.check(lib.pqk_table_scale(a.ctypes.data_as(C.c_void_p), a.size, C.byref(e), C.byref(f)))
        return e.value, f.value

    assert scale([0.0, 1.0, 5e3]) == (0, 0)
    e, f = scale([0.0, 1e200, 1e190])
    assert f == 0 and 2.0**-100 <= 1e190 * 2.0**e and 1e200 * 2.0**e <= 2.0**100
    assert scale([0.0, 1e-300, 1e300])[1] == 1  # no fp32 window: fp64-only mode
    with pytest.raises(ValueError, match="non-negative"):
        scale([0.0, -1.0])


@pytest.mark.parametrize("n", [1, 3, 7, 8, 9, 127, 128, 129, 1000, 4097, 100_003, 1_000_000])
def test_pairwise_plan_matches_numpy(n):
    """Evaluate the C-ABI plan in Python: must equal np.add.reduce bit for bit."""
    from oracle import pqk_oracle as O
    from paper_1709_03708_b200 import engine

    rng = np.random.default_rng(n)
    x = rng.random(n) * 10.0 ** rng.integers(-2, 6, size=n)
    leaf_off, leaf_len, depth_start, na, nb = engine.host_plan(n)
    leafval = []
    for off, ln in zip(leaf_off, leaf_len):
        leafval.append(O.pairwise_sum(x[off : off + ln]) if ln < 8 else float(np.add.reduce(x[off : off + ln])))
    vals = None
    for d in range(len(depth_start) - 2, -1, -1):
        s, e = depth_start[d], depth_start[d + 1]
        cur = []
        for i in range(s, e):
            cur.append(leafval[na[i]] if nb[i] < 0 else vals[na[i]] + vals[nb[i]])
        vals = cur
    assert vals[0] == float(np.add.reduce(x))
    assert sum(leaf_len) == n


@pytest.mark.parametrize("n", [5, 128, 129, 1000, 99_999, 1_000_000])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_tree_split_combine(n, parts):
    from paper_1709_03708_b200.pairwise import tree_combine, tree_split

    rng = np.random.default_rng(n + parts)
    x = rng.random(n)
    shards = tree_split(n, parts)
    assert len(shards) == parts
    assert sum(ln for _, ln in shards) == n
    pos = 0
    for off, ln in shards:
        assert off == pos or ln == 0
        pos += ln
    partials = [float(np.add.reduce(x[o : o + ln])) if ln else 0.0 for o, ln in shards]
    assert tree_combine(n, partials) == float(np.add.reduce(x))
    if parts in (2, 4, 8) and n >= 1000:
        sizes = [ln for _, ln in shards]
        assert max(sizes) - min(sizes) <= 8 * parts


def test_merge_candidates():
    from paper_1709_03708_b200.distributed import merge_candidates

    sd = np.array([5.0, 9.0, 9.0, 1.0, 7.0, 9.0])
    keys = sd.view(np.uint64)
    parts = [(keys[:3], np.arange(3), np.arange(3)[:, None]), (keys[3:], np.arange(3, 6), np.arange(3, 6)[:, None])]
    k, idx, rows = merge_candidates(parts, 4)
    assert list(idx) == [1, 2, 5, 4]
    assert list(rows[:, 0]) == [1, 2, 5, 4]


def test_api_validation_without_device():
    import paper_1709_03708_b200 as pqk

    with pytest.raises(ValueError, match="shape"):
        pqk.DistanceTables(np.zeros((3, 3)))
    bad = np.zeros((1, 3, 3))
    bad[0, 1, 1] = 2.0
    with pytest.raises(ValueError, match="diagonal"):
        pqk.DistanceTables(bad)
    asym = np.zeros((1, 3, 3))
    asym[0, 0, 1] = 1.0
    with pytest.raises(ValueError, match="symmetric"):
        pqk.DistanceTables(asym)
    with pytest.raises(ValueError, match="outside"):
        pqk.PQCodebook(np.zeros((2, 257, 3), dtype=np.float32))
    tables = lattice_tables(1, 4)
    codes = np.zeros((5, 1), dtype=np.uint8)
    with pytest.raises(ValueError, match="k must be"):
        pqk.fit(codes, tables, 0)
    with pytest.raises(ValueError, match="max_iterations"):
        pqk.fit(codes, tables, 2, max_iterations=0)
    with pytest.raises(ValueError, match="update must be"):
        pqk.fit(codes, tables, 2, update="fancy")
    with pytest.raises(ValueError, match="initial_centers has"):
        pqk.fit(codes, tables, 2, initial_centers=np.zeros((3, 1), dtype=np.uint8))
    with pytest.raises(ValueError, match=r"\[0, 4\)"):
        pqk.assign(np.array([[4]]), codes[:1], tables)
    with pytest.raises(ValueError, match="integers"):
        pqk.assign(np.array([[0.5]]), codes[:1], tables)
    with pytest.raises(ValueError, match="non-empty"):
        pqk.assign(codes, np.empty((0, 1), dtype=np.uint8), tables)


def test_registry_semantics():
    import paper_1709_03708_b200 as pqk

    assert pqk.registered_assignment_strategies() == ("linear_scan",)
    with pytest.raises(ValueError, match="cannot be removed"):
        pqk.unregister_assignment_strategy("linear_scan")
    with pytest.raises(ValueError, match="non-empty"):
        pqk.register_assignment_strategy("", lambda *a: None)
    assert pqk.select_assignment_strategy(np.empty((0, 2), dtype=np.uint8), random_tables(2, 4), 3) == "linear_scan"
    # importing the package must not touch the reference's registry either
    import sys

    assert "pqclust" not in sys.modules or "b200" not in sys.modules["pqclust"].registered_assignment_strategies()


def test_product_fails_loudly_without_cuda():
    import torch

    import paper_1709_03708_b200 as pqk

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    tables = random_tables(2, 8)
    codes = np.zeros((4, 2), dtype=np.uint8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pqk.assign(codes, codes[:1], tables)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pqk.fit(codes, tables, 2)


def test_init_centers_matches_reference_rule():
    import paper_1709_03708_b200 as pqk

    rng = np.random.default_rng(1)
    codes = rng.permutation(64).reshape(64, 1).astype(np.uint8)
    centers = pqk.init_centers(codes, 10, seed=3)
    expect = codes[np.random.default_rng(3).choice(64, size=10, replace=False)]
    np.testing.assert_array_equal(centers, expect)


def test_integration_stub_is_the_tested_file():
    """INTEGRATION.md's ctypes stub is tests/pqclust_b200.py verbatim (run by test_gpu_plugin)."""
    root = Path(__file__).resolve().parents[1]
    doc = (root / "INTEGRATION.md").read_text()
    start = doc.index("```python\n", doc.index("## ctypes stub")) + len("```python\n")
    block = doc[start : doc.index("```", start)]
    assert block == (root / "tests" / "pqclust_b200.py").read_text()


def test_bench_codebooks_present_and_recipe():
    """bench_assets hold the reference-trained codebook of every bench config (BASELINE recipe)."""
    import bench

    for name, cfg in bench.CONFIGS.items():
        book = bench.make_codebook(name, cfg["m"], cfg["l"])
        assert book.dtype == np.float32 and book.shape == (cfg["m"], cfg["l"], cfg["dim"] // cfg["m"])
        assert bench.CODEBOOK_RECIPES[name]["iterations"] == 20


@pytest.mark.parametrize("world,e", [(1, 5), (2, 7), (3, 40)])
def test_merge_candidates_device_equals_host(world, e):
    """The device merge (two stable sorts) picks the host lexsort's rows, ties and padding included."""
    import torch

    from paper_1709_03708_b200.distributed import empty_clusters_device, merge_candidates, merge_candidates_device

    rng = np.random.default_rng(world * 100 + e)
    sd = rng.choice([0.0, 1.5, 2.25, 7.0, 9.5], size=(world, e))  # many exact ties
    gk = sd.view(np.int64).copy()
    gi = np.sort(rng.choice(10_000, size=(world, e), replace=False), axis=1).astype(np.int64)
    gi[-1, -2:] = np.iinfo(np.int64).max  # padding rows of a short shard
    gk[-1, -2:] = 0
    gr = rng.integers(0, 256, size=(world, e, 4)).astype(np.uint8)
    _, _, rows_h = merge_candidates([(gk.reshape(-1).view(np.uint64), gi.reshape(-1), gr.reshape(-1, 4))], e)
    rows_d = merge_candidates_device(torch.from_numpy(gk), torch.from_numpy(gi), torch.from_numpy(gr), e)
    np.testing.assert_array_equal(rows_d.numpy(), rows_h)
    counts = torch.from_numpy(rng.integers(0, 3, size=50).astype(np.int32))
    z = np.flatnonzero(counts.numpy() == 0)
    np.testing.assert_array_equal(empty_clusters_device(counts, len(z)).numpy(), z)
