"""tcgen05 diagnostic: one 128x256xK fp16 tile through UMMA descriptors, TMEM and
tcgen05.ld must equal the fp64 product of the same fp16 operands (products of fp16
pairs are exact in fp32; the fp32 accumulation is checked to 1e-6 relative)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_tcgen05_tile(k):
    import torch

    from paper_1709_03708_b200 import _lib, engine

    dev = engine.device_of()
    rng = np.random.default_rng(k)
    a = rng.integers(-8, 9, size=(128, k)).astype(np.float16) + rng.random((128, k)).astype(np.float16)
    b = rng.integers(-8, 9, size=(256, k)).astype(np.float16) + rng.random((256, k)).astype(np.float16)
    da = torch.from_numpy(a).to(dev)
    db = torch.from_numpy(b).to(dev)
    dc = torch.zeros((128, 256), dtype=torch.float32, device=dev)
    _lib.call("pqk_tc_selftest", C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), C.c_void_p(dc.data_ptr()), k,
              C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    got = dc.cpu().numpy().astype(np.float64)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    scale = np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64)).T
    assert np.all(np.abs(got - ref) <= 1e-6 * scale + 1e-6), np.max(np.abs(got - ref))
