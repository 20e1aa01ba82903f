"""Single-process multi-GPU fit (paper_1709_03708_b200.multidevice): peer-memory
histogram exchange (pqk_peer_sum_device), sliced vote and center gather.

The pool gives one GPU per call, so the shards share cuda:0 (devices=[0, 0, ...]): the
exchange then reads the same device's buffers through the same kernel.  Results must
equal one-GPU fit and the oracle bit for bit (clustering.py:377-482)."""

import ctypes as C

import numpy as np
import pytest

from helpers import mixture_codes, random_tables

pytestmark = pytest.mark.gpu


def _same(a, b):
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.centers, b.centers)
    assert a.iterations_run == b.iterations_run and a.converged == b.converged
    assert [t.objective for t in a.trace] == [t.objective for t in b.trace]
    assert [t.objective_sq for t in a.trace] == [t.objective_sq for t in b.trace]
    assert [t.repaired_clusters for t in a.trace] == [t.repaired_clusters for t in b.trace]
    assert [t.mean_histogram_nnz for t in a.trace] == [t.mean_histogram_nnz for t in b.trace]


@pytest.mark.parametrize("g", [1, 2, 3, 8])
def test_peer_sum(g):
    import torch

    from paper_1709_03708_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(g)
    for count, off in [(1, 0), (7, 1), (4096, 0), (100_003, 3)]:
        bufs = [torch.from_numpy(rng.integers(0, 2**20, size=count + off, dtype=np.int64).astype(np.int32)).cuda()
                for _ in range(g)]
        out = torch.zeros(count + off, dtype=torch.int32, device="cuda")
        ptrs = (C.c_void_p * g)(*[b.data_ptr() + 4 * off for b in bufs])
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.pqk_peer_sum_device(ptrs, g, count, C.c_void_p(out.data_ptr() + 4 * off), s))
        exp = sum(b.cpu().numpy().astype(np.int64) for b in bufs)[off:].astype(np.uint32).view(np.int32)
        np.testing.assert_array_equal(out.cpu().numpy()[off:], exp)
        # in place (out aliases peer 0)
        _lib.check(lib.pqk_peer_sum_device(ptrs, g, count, C.c_void_p(bufs[0].data_ptr() + 4 * off), s))
        np.testing.assert_array_equal(bufs[0].cpu().numpy()[off:], exp)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0], [0] * 8])
def test_fit_devices_equals_single_and_oracle(oracle, devices):
    import paper_1709_03708_b200 as pqk

    tables = random_tables(4, 256, seed=5)
    codes = mixture_codes(20_000, 4, 256, 150, seed=6)
    got = pqk.fit(codes, tables, 200, max_iterations=6, seed=2, devices=devices)
    one = pqk.fit(codes, tables, 200, max_iterations=6, seed=2)
    _same(got, one)
    ref = oracle.fit(codes, tables, 200, max_iterations=6, seed=2)
    np.testing.assert_array_equal(got.labels, ref["labels"])
    np.testing.assert_array_equal(got.centers, ref["centers"])


def test_fit_devices_repairs_long_codes_small_l(oracle):
    """Many empty clusters (repair across shards), M=16 and L=13 (no fp16 vote tables)."""
    import paper_1709_03708_b200 as pqk

    tables = random_tables(16, 13, seed=8)
    rng = np.random.default_rng(9)
    codes = np.repeat(rng.integers(0, 13, size=(300, 16)), 10, axis=0).astype(np.uint8)
    rng.shuffle(codes)
    got = pqk.fit(codes, tables, 900, max_iterations=4, seed=3, devices=[0, 0, 0])
    assert any(t.repaired_clusters for t in got.trace)
    _same(got, pqk.fit(codes, tables, 900, max_iterations=4, seed=3))
    ref = oracle.fit(codes, tables, 900, max_iterations=4, seed=3)
    np.testing.assert_array_equal(got.centers, ref["centers"])


def test_fit_devices_more_devices_than_clusters():
    import paper_1709_03708_b200 as pqk

    tables = random_tables(4, 256, seed=1)
    codes = mixture_codes(3000, 4, 256, 5, seed=1)
    _same(pqk.fit(codes, tables, 2, max_iterations=5, seed=1, devices=[0, 0, 0]),
          pqk.fit(codes, tables, 2, max_iterations=5, seed=1))


def test_fit_devices_config2_workload():
    """Config 2 (1e6 codes, K=1e4, 16-bit first tier) over 4 shards."""
    import torch

    import bench
    import paper_1709_03708_b200 as pqk

    wl = bench.build_workload("c2", torch.device("cuda", 0))
    codes, tables = wl["codes_host"], wl["tables"]
    init = codes[bench.center_indices(len(codes), 10_000)]
    _same(pqk.fit(codes, tables, 10_000, max_iterations=3, initial_centers=init, devices=[0, 0, 0, 0]),
          pqk.fit(codes, tables, 10_000, max_iterations=3, initial_centers=init))


def test_fit_devices_rejects_external_strategy():
    import paper_1709_03708_b200 as pqk

    tables = random_tables(2, 16, seed=1)
    codes = mixture_codes(100, 2, 16, 3, seed=1)
    pqk.register_assignment_strategy("ext", lambda c, ce, t, th: np.zeros(len(c), np.uint32))
    try:
        with pytest.raises(ValueError):
            pqk.fit(codes, tables, 3, strategy="ext", devices=[0, 0])
    finally:
        pqk.unregister_assignment_strategy("ext")
