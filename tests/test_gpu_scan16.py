"""GPU parity of the fixed-point first tiers of the assignment: the 8-bit tier with
top-T chunk keys (pqk_hscan8.cuh, padded M = 4) and the 16-bit tier (pqk_hscan.cuh).

The default mode engages a fixed-point tier only above 2^31 lookups, so the small cases
below force it (scan mode 2: 8-bit at M <= 4, 16-bit above; mode 4: 16-bit at every M)
and also force the fp32 list tier for any list length (modes 3 and 5), then compare
labels and sd_sq byte for byte with the oracle's linear scan
(clustering.py:167-197: float64, ascending m, lowest index on ties) and with the fp32
path (mode 1).  Cases: random tables at every supported width, lattice tables with
massive exact ties, duplicated centres, tables spanning huge scales (saturated
entries), clustered codes, partial last chunks, a fit, and a multi-pass size.
"""

import numpy as np
import pytest

from helpers import lattice_tables, mixture_codes, random_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1709_03708_b200 import _lib

    lib = _lib.load()
    yield lib
    _lib.check(lib.pqk_set_scan_mode(0), "scan mode")


def _assign(lib, mode, codes, centers, tables):
    from paper_1709_03708_b200 import _lib, engine

    _lib.check(lib.pqk_set_scan_mode(mode), "scan mode")
    try:
        return engine.assign_host(codes, centers, tables, want_sd=True)
    finally:
        _lib.check(lib.pqk_set_scan_mode(0), "scan mode")


def _check(lib, oracle, codes, centers, tables, modes=(2, 3, 4, 5)):
    expect = oracle.assign_c(codes, centers, tables)
    exp_sd = oracle.paired_distance_sq(tables, codes.astype(np.int64), centers[expect].astype(np.int64))
    if codes.shape[1] > 4:  # modes 4 / 5 only differ from 2 / 3 at padded M = 4
        modes = tuple(md for md in modes if md not in (4, 5))
    for mode in modes:
        labels, sd = _assign(lib, mode, codes, centers, tables)
        np.testing.assert_array_equal(labels, expect, err_msg=f"mode {mode}")
        assert sd.tobytes() == exp_sd.tobytes(), f"mode {mode}"


def test_scan_mode_abi(lib):
    from paper_1709_03708_b200 import _lib

    assert lib.pqk_get_scan_mode() == 0
    assert lib.pqk_set_scan_mode(7) == _lib.PQK_EINVAL
    assert lib.pqk_get_scan_mode() == 0


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 12, 16])
@pytest.mark.parametrize("l_count", [4, 256])
def test_random_tables_widths(lib, oracle, m, l_count):
    rng = np.random.default_rng(77 * m + l_count)
    tables = random_tables(m, l_count, seed=3 * m + l_count)
    codes = rng.integers(0, l_count, size=(3000, m)).astype(np.uint8)
    centers = rng.integers(0, l_count, size=(203, m)).astype(np.uint8)  # partial last chunk
    _check(lib, oracle, codes, centers, tables)


@pytest.mark.parametrize("trial", range(6))
def test_lattice_ties_duplicates(lib, oracle, trial):
    rng = np.random.default_rng(9100 + trial)
    m = int(rng.choice([1, 2, 4, 8]))
    tables = lattice_tables(m, 16)
    codes = rng.integers(0, 16, size=(4000, m)).astype(np.uint8)
    centers = codes[rng.integers(0, 4000, size=150)].copy()
    centers[rng.integers(0, 150, size=50)] = centers[3]
    _check(lib, oracle, codes, centers, tables)


@pytest.mark.parametrize("span", [1e-30, 1e6, 1e30])
def test_wide_dynamic_range(lib, oracle, span):
    """Tables mixing tiny and huge distances: most entries saturate or round to 0."""
    rng = np.random.default_rng(int(np.log10(span)) + 50)
    m, l_count = 4, 64
    book = rng.standard_normal((m, l_count, 2)) * np.where(rng.random((m, l_count, 1)) < 0.1, span, 1.0)
    from oracle import pqk_oracle as O

    tables = O.build_distance_tables(book.astype(np.float32))
    if not np.all(np.isfinite(tables)):
        pytest.skip("float32 overflow in the codebook")
    codes = rng.integers(0, l_count, size=(3000, m)).astype(np.uint8)
    centers = rng.integers(0, l_count, size=(120, m)).astype(np.uint8)
    _check(lib, oracle, codes, centers, tables)


@pytest.mark.parametrize("m", [4, 8, 16])
def test_clustered_codes_multi_pass(lib, oracle, m):
    """Enough codes for several persistent passes per CTA and centres near the codes."""
    rng = np.random.default_rng(m)
    l_count = 256
    tables = random_tables(m, l_count, seed=11 * m, sub_dim=4)
    codes = mixture_codes(60_000 if m < 16 else 30_000, m, l_count, 400, seed=m)
    centers = codes[rng.choice(len(codes), size=1000, replace=False)].copy()
    _check(lib, oracle, codes, centers, tables, modes=(1, 2, 3, 4, 5))


def test_single_center_and_k_equals_n(lib, oracle):
    rng = np.random.default_rng(5)
    tables = random_tables(4, 32, seed=5)
    codes = rng.integers(0, 32, size=(500, 4)).astype(np.uint8)
    _check(lib, oracle, codes, codes[:1].copy(), tables)
    _check(lib, oracle, codes, codes.copy(), tables)


@pytest.mark.parametrize("k", [2, 33, 64, 95, 161, 192, 193])
def test_fewer_chunks_than_keys(lib, oracle, k):
    """The 8-bit tier keeps T = 6 chunk keys per code: K below / at / just above 6 chunks
    of 32 leaves sentinel keys (no bound from unstored chunks) or a partial last chunk."""
    rng = np.random.default_rng(k)
    tables = random_tables(4, 256, seed=k, sub_dim=4)
    codes = mixture_codes(5000, 4, 256, 50, seed=k)
    centers = codes[rng.choice(len(codes), size=k, replace=False)].copy()
    _check(lib, oracle, codes, centers, tables)


@pytest.mark.parametrize("trial", range(3))
def test_cross_chunk_ties(lib, oracle, trial):
    """Exact ties between centres of different chunks: the 8-bit finalisation visits the
    stored chunks by key, not by index, and must still return the lowest index."""
    rng = np.random.default_rng(700 + trial)
    tables = lattice_tables(4, 8)
    codes = rng.integers(0, 8, size=(6000, 4)).astype(np.uint8)
    centers = rng.integers(0, 8, size=(400, 4)).astype(np.uint8)
    _check(lib, oracle, codes, centers, tables)


def test_fit_parity_forced(lib, oracle):
    from paper_1709_03708_b200 import _lib
    import paper_1709_03708_b200 as pqk

    tables = random_tables(4, 256, seed=8, sub_dim=4)
    codes = mixture_codes(20_000, 4, 256, 300, seed=8)
    _lib.check(lib.pqk_set_scan_mode(2), "scan mode")
    try:
        res = pqk.fit(codes, tables, 200, max_iterations=5, seed=3)
    finally:
        _lib.check(lib.pqk_set_scan_mode(0), "scan mode")
    ref = oracle.fit(codes, tables, 200, max_iterations=5, seed=3, scan=oracle.assign_c)
    np.testing.assert_array_equal(res.labels, ref["labels"])
    np.testing.assert_array_equal(res.centers, ref["centers"])
    assert [s.objective for s in res.trace] == [t["objective"] for t in ref["trace"]]
    _lib.check(lib.pqk_set_scan_mode(4), "scan mode")
    try:
        res16 = pqk.fit(codes, tables, 200, max_iterations=5, seed=3)
    finally:
        _lib.check(lib.pqk_set_scan_mode(0), "scan mode")
    np.testing.assert_array_equal(res16.labels, ref["labels"])
    np.testing.assert_array_equal(res16.centers, ref["centers"])


@pytest.mark.parametrize("kind", ["random", "lattice", "scaled", "heavy", "huge", "empty_rows"])
def test_vote_fp16_stage(oracle, kind):
    """The vote's tensor-core first stage (L = 256) decides the exact-arithmetic argmin
    (clustering.py:349-354, lowest j on ties) or hands over to the fp64 stages: counts
    < 2048 (one accumulator), heavy counts (lo/hi split), counts >= 2^22 (tile handed
    over whole), and empty clusters between filled ones; 600 clusters = 5 row tiles."""
    from paper_1709_03708_b200 import engine

    rng = np.random.default_rng({"random": 1, "lattice": 2, "scaled": 3, "heavy": 4, "huge": 5, "empty_rows": 6}[kind])
    m, l_count, k = 2, 256, 600
    if kind == "lattice":
        tables = lattice_tables(m, l_count)  # integer distances: exact ties are common
    else:
        tables = random_tables(m, l_count, seed=17, sub_dim=3)
        if kind == "scaled":
            tables = tables * 1e-30
    hist = np.zeros((k, m, l_count), dtype=np.int64)
    for kk in range(k):
        for mm in range(m):
            nnz = int(rng.integers(1, 40))
            sup = rng.choice(l_count, size=nnz, replace=False)
            hi = {"heavy": 10**6, "huge": 2**26}.get(kind, 50)
            hist[kk, mm, sup] = rng.integers(1, hi, size=nnz)
    if kind == "huge":
        hist[::3] %= 5000  # tiles mixing small, split and too-large counts
    if kind == "empty_rows":
        hist[rng.random(k) < 0.4] = 0
    got = engine.vote_host(hist, tables)
    for kk in range(k):
        if not hist[kk].any():
            continue  # empty cluster: left for the repair
        for mm in range(m):
            assert got[kk, mm] == oracle.vote_argmin(hist[kk, mm], tables[mm]), (kk, mm)


@pytest.mark.parametrize("m,lookup_bytes", [(4, 1), (8, 2)])
def test_default_mode_large_problem_uses_fixed_point_tier(lib, oracle, m, lookup_bytes):
    """Default mode at >= 2^31 lookups: the 8-bit tier runs at M = 4 and the 16-bit tier at
    M = 8 (1- / 2-byte lookups in the stats); labels / sd_sq still equal the oracle's
    linear scan on clustered codes."""
    import torch

    from paper_1709_03708_b200 import _lib, engine

    rng = np.random.default_rng(31)
    l_count = 256
    tables = random_tables(m, l_count, seed=31, sub_dim=8)
    codes = mixture_codes(700_000, m, l_count, 3000, seed=31)
    centers = codes[rng.choice(len(codes), size=800, replace=False)].copy()
    assert len(codes) * len(centers) * m >= 2**31
    dev = engine.device_of()
    dt = engine.device_tables(tables, dev)
    with torch.cuda.device(dev):
        eng = engine.ShardEngine(engine.upload_codes(codes, m, dev), dt, len(centers), dev)
        eng.assign(engine.upload_codes(centers, m, dev))
        labels, sd = eng.labels_host(), eng.sd_host()
        st = eng.stats.cpu().numpy()
    assert int(st[_lib.STAT_LOOKUP_BYTES]) == lookup_bytes
    expect, exp_sd = oracle.assign_c(codes, centers, tables, want_sd=True)
    np.testing.assert_array_equal(labels, expect)
    assert sd.tobytes() == exp_sd.tobytes()


@pytest.mark.skipif(bool(__import__("os").environ.get("PQK_VOTE_SIMT")), reason="already inside the SIMT child")
def test_vote_simt_stage_child():
    """The SIMT shared-table first stage (PQK_VOTE_SIMT=1, read once per process) on the
    same vote cases, in a child pytest."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, PQK_VOTE_SIMT="1")
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(here, "test_gpu_scan16.py"), "-k", "test_vote_fp16_stage"],
        env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
