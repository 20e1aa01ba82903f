"""GPU parity of the remaining kernels: encoder, objective tree, paired distance,
host-buffer C-ABI step."""

import ctypes as C

import numpy as np
import pytest

from helpers import random_codebook, random_tables

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,l_count,sub", [(4, 256, 32), (3, 12, 4), (8, 256, 16), (2, 64, 64), (16, 256, 8), (1, 256, 3)])
def test_encode_matches_oracle(oracle, m, l_count, sub):
    import paper_1709_03708_b200 as pqk

    cw = random_codebook(m, l_count, sub, seed=m * 7 + sub)
    rng = np.random.default_rng(6)
    vectors = rng.normal(size=(3000, m * sub)).astype(np.float32)
    got = pqk.encode(pqk.PQCodebook(cw), vectors)
    np.testing.assert_array_equal(got, oracle.encode(cw, vectors))


def test_encode_ties_toward_low_index():
    import paper_1709_03708_b200 as pqk

    book = pqk.PQCodebook(np.array([[[0.0], [3.0], [3.0], [7.0]]], dtype=np.float32))
    assert pqk.encode(book, np.array([3.0], dtype=np.float32))[0] == 1
    grid = np.arange(4, dtype=np.float32).reshape(1, 4, 1)
    assert pqk.encode(pqk.PQCodebook(grid), np.array([0.5], dtype=np.float32))[0] == 0


# 1_048_876 / 2_102_153: unbalanced trees whose deepest level is small (74 / 1250 nodes) under levels of 8192 / 16384
@pytest.mark.parametrize("n", [1, 5, 8, 9, 100, 128, 129, 255, 1000, 8193, 100_000, 1_048_876, 1_234_567, 2_102_153])
def test_objective_tree_matches_numpy(n):
    import torch

    from paper_1709_03708_b200 import engine

    rng = np.random.default_rng(n)
    sd = rng.random(n) * 10.0 ** rng.integers(-3, 5, size=n)
    dev = engine.device_of()
    got = engine.mean_objectives(torch.from_numpy(sd).to(dev), n, dev)
    assert got == (float(np.mean(np.sqrt(sd))), float(np.mean(sd)))


def test_paired_distance_exact(oracle):
    import paper_1709_03708_b200 as pqk

    tables = random_tables(4, 16, seed=17, sub_dim=3)
    rng = np.random.default_rng(18)
    a = rng.integers(0, 16, size=(500, 4), dtype=np.uint8)
    b = rng.integers(0, 16, size=(500, 4), dtype=np.uint8)
    got = pqk.paired_distance_sq(tables, a, b)
    assert got.tobytes() == oracle.paired_distance_sq(tables, a, b).tobytes()


def test_lloyd_step_host_abi(oracle):
    from paper_1709_03708_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    tables = random_tables(4, 256, seed=9, sub_dim=8)
    codes = rng.integers(0, 256, size=(20000, 4)).astype(np.uint8)
    centers = codes[rng.choice(20000, 300, replace=False)].copy()
    labels = np.empty(20000, np.uint32)
    newc = np.empty((300, 4), np.uint8)
    obj2 = np.empty(2, np.float64)
    stats = np.empty(_lib.STATS_LEN, np.int64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    _lib.check(lib.pqk_lloyd_step_host(p(codes), 20000, 4, p(centers), 300, p(tables), 256, p(labels), p(newc),
                                       p(obj2), p(stats), 0))
    ref = oracle.fit(codes, tables, 300, max_iterations=1, initial_centers=centers, scan=oracle.assign_c)
    np.testing.assert_array_equal(labels, ref["labels"])
    np.testing.assert_array_equal(newc, ref["centers"])
    sd = oracle.paired_distance_sq(tables, codes, centers[labels])
    assert obj2[0] / 20000 == float(np.mean(np.sqrt(sd)))
    assert stats[_lib.STAT_EMPTY] == ref["trace"][0]["repaired"]
