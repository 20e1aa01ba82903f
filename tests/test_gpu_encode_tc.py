"""Tensor-core encoder (tcgen05, fp16 hi/lo split + certificate + fp64 fallback)
against the oracle (pq.py:205-231 semantics: fp64 sequential (x-c)^2, lowest index
on ties).  Shapes with dsub in {8, 16, 32, 64} take the tcgen05 path."""

import numpy as np
import pytest

from helpers import random_codebook

pytestmark = pytest.mark.gpu


def _encode(cw, x):
    import paper_1709_03708_b200 as pqk

    return pqk.encode(pqk.PQCodebook(cw), x)


@pytest.mark.parametrize("m,sub,l_count,n", [(4, 32, 256, 5000), (8, 16, 256, 3001), (2, 64, 256, 1000),
                                              (1, 32, 100, 777), (4, 16, 7, 129), (3, 32, 256, 1),
                                              (16, 8, 256, 2000), (2, 8, 33, 500), (5, 64, 256, 300),
                                              (2, 96, 256, 700), (3, 128, 100, 1300), (1, 256, 256, 400),
                                              (2, 512, 256, 300)])
def test_tc_encode_random(oracle, m, sub, l_count, n):
    cw = random_codebook(m, l_count, sub, seed=m * 100 + sub + l_count)
    x = np.random.default_rng(n).normal(size=(n, m * sub)).astype(np.float32)
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


def test_tc_encode_integer_data_and_ties(oracle):
    """SIFT-like integer vectors (x exactly fp16: the lo-x pass is skipped) and exact
    ties from duplicated codewords and vectors placed on codewords."""
    rng = np.random.default_rng(3)
    x = np.clip(np.rint(rng.gamma(0.6, 30.0, size=(4096, 128))), 0, 255).astype(np.float32)
    cw = x[rng.choice(4096, 256, replace=False)].reshape(256, 4, 32).transpose(1, 0, 2).copy()
    cw[:, 17] = cw[:, 3]  # duplicated codeword: ties must go to index 3
    got = _encode(cw, x)
    np.testing.assert_array_equal(got, oracle.encode(cw, x))


@pytest.mark.parametrize("scale", [1e-30, 1e-6, 1e6, 1e30])
def test_tc_encode_extreme_scales(oracle, scale):
    cw = (random_codebook(4, 256, 32, seed=9) * scale).astype(np.float32)
    x = (np.random.default_rng(1).normal(size=(700, 128)) * scale).astype(np.float32)
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


def test_tc_encode_config1_golden():
    """Reference encode output on BASELINE config 1 vectors (tests/golden/config1.npz)."""
    from golden_io import load

    g = load("config1")
    np.testing.assert_array_equal(_encode(g["codebook"], g["vectors_head"]), g["codes_head"])


def test_tc_encode_rows_outside_codebook_range(oracle):
    """Rows whose |s x|^2 exceeds the fp16 extension range (vectors ~1e4 x the codebook
    scale) and all-zero rows must go through the exact path and still match."""
    cw = random_codebook(4, 256, 32, seed=21)
    x = np.random.default_rng(22).normal(size=(1000, 128)).astype(np.float32)
    x[::7] *= 1e4
    x[3::11] = 0.0
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_encode_non_finite_vectors_follow_np_argmin(oracle, bad):
    """np.argmin over cdist rows: a NaN distance is the minimum (first NaN wins)."""
    cw = random_codebook(4, 256, 32, seed=2)
    x = np.random.default_rng(4).normal(size=(300, 128)).astype(np.float32)
    x[5, 3] = bad
    x[77, 100] = bad
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


_SIMT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1709_03708_b200 as pqk
d = np.load(sys.argv[2])
np.save(sys.argv[3], pqk.encode(pqk.PQCodebook(d["cw"]), d["x"]))
"""


def test_tc_encode_many_tiles_matches_simt_path(tmp_path, oracle):
    """~11 tiles x 4 subspaces per CTA (buffer reuse across items): the tcgen05 path must
    equal the SIMT certified path (run in a subprocess with PQK_ENCODE_SIMT=1) and, on a
    20,000-row sample spanning both halves, the oracle; the fp64 fallback must stay rare."""
    import os
    import subprocess
    import sys

    import torch

    from paper_1709_03708_b200 import _lib, engine

    rng = np.random.default_rng(11)
    n = 200_000
    cw = random_codebook(4, 256, 32, seed=12)
    x = rng.normal(size=(n, 128)).astype(np.float32)
    x[: n // 2] = np.rint(x[: n // 2] * 20)  # half integer-valued (2-pass), half general (3-pass)
    dev = engine.device_of()
    stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
    tc_codes = engine.encode_device(torch.from_numpy(x).to(dev), torch.from_numpy(cw).to(dev), 4, 256, dev,
                                    stride=4, stats=stats).cpu().numpy()
    flagged = int(stats[_lib.STAT_ENCODE_FLAGGED].item())
    np.savez(tmp_path / "in.npz", cw=cw, x=x)
    env = dict(os.environ, PQK_ENCODE_SIMT="1")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    subprocess.run([sys.executable, "-c", _SIMT_SCRIPT, root, str(tmp_path / "in.npz"), str(tmp_path / "out.npy")],
                   check=True, env=env)
    np.testing.assert_array_equal(tc_codes, np.load(tmp_path / "out.npy"))
    rows = np.sort(rng.choice(n, size=20_000, replace=False))
    np.testing.assert_array_equal(tc_codes[rows], oracle.encode(cw, x[rows]))
    # the integer half lies ~20x outside the codebook's range (distances ~ |x|^2, gaps ~ |x||c|):
    # the fp32 certificate leaves ~0.2% of its pairs to the exact path
    assert flagged < n * 4 * 3e-3, flagged  # the stats slot counts every uncertified pair


def test_tc_encode_sift_like_flag_rate(oracle):
    """SIFT-like data with the config-2 / config-4 reference codebooks (bench_assets): the
    certificate must cover almost every pair, and every code must equal the oracle's."""
    import torch

    import bench
    from paper_1709_03708_b200 import _lib, engine, synth

    x = synth.sift_like(40_000, 5)
    dev = engine.device_of()
    for cfg in ("c2", "c4"):
        cw = bench.make_codebook(cfg, 4, 256)
        stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
        codes = engine.encode_device(torch.from_numpy(x).to(dev), torch.from_numpy(np.asarray(cw)).to(dev), 4, 256,
                                     dev, stride=4, stats=stats).cpu().numpy()
        assert int(stats[_lib.STAT_ENCODE_FLAGGED].item()) < 40_000 * 4 * 1e-3
        np.testing.assert_array_equal(codes, oracle.encode(cw, x))


def test_tc_encode_config3_shape(oracle):
    """BASELINE config 3's shape: 4096-D deep-feature-like vectors, M=8 (512-D subspaces,
    the K-streamed tensor-core kernel), codewords drawn from the data."""
    from paper_1709_03708_b200 import synth

    x = synth.deep_like(3000, 11, components=300)
    rng = np.random.default_rng(2)
    cw = x[rng.choice(3000, 256, replace=False)].reshape(256, 8, 512).transpose(1, 0, 2).copy()
    cw += rng.normal(0, 1e-3, size=cw.shape).astype(np.float32)
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


def test_tck_prepared_operands_follow_codebook_changes(oracle):
    """The K-streamed path keeps its prepared codebook operands between calls with the same
    codebook (pointer, shape, contents); an in-place change of the codebook must be seen."""
    import torch

    from paper_1709_03708_b200 import engine

    rng = np.random.default_rng(31)
    cw = rng.normal(size=(2, 256, 128)).astype(np.float32)
    x = rng.normal(size=(900, 256)).astype(np.float32)
    dev = engine.device_of()
    xd = torch.from_numpy(x).to(dev)
    cd = torch.from_numpy(cw).to(dev)
    for step in range(3):
        got = engine.encode_device(xd, cd, 2, 256, dev).cpu().numpy()
        np.testing.assert_array_equal(got, oracle.encode(cw, x), err_msg=f"step {step}")
        if step == 0:
            continue  # step 1 reuses the prepared operands
        cw[1, 7] += 0.5  # in place, same device pointer
        cd.copy_(torch.from_numpy(cw))


@pytest.mark.parametrize("l_count", [256, 100, 33])
def test_tck_candidate_masks_small_codebooks_ties_and_non_finite(oracle, l_count):
    """K-streamed path (dsub = 128): near-duplicate and duplicated codewords (pairs the
    tensor-core certificate must hand on with a candidate mask), fewer than 256 codewords,
    and rows with NaN / inf (every codeword is a candidate: np.argmin's NaN rule)."""
    rng = np.random.default_rng(l_count)
    cw = rng.normal(size=(2, l_count, 128)).astype(np.float32)
    cw[0, 5] = cw[0, 2]  # exact tie: the lower index wins
    cw[1, 7] = cw[1, 3] + np.float32(1e-6)  # near tie
    cw[1, l_count - 1] = cw[1, 0] * np.float32(1 + 2e-7)
    x = rng.normal(size=(4000, 256)).astype(np.float32)
    x[:300, :128] = cw[0, 2] + rng.normal(0, 1e-3, size=(300, 128)).astype(np.float32)
    x[300:600, 128:] = cw[1, 3] + rng.normal(0, 1e-4, size=(300, 128)).astype(np.float32)
    x[600:700, 128:] = cw[1, 0]
    x[700, 3] = np.nan
    x[701, 130] = np.inf
    x[702, 5] = -np.inf
    x[703] = np.nan
    np.testing.assert_array_equal(_encode(cw, x), oracle.encode(cw, x))


def test_tck_single_cta_variant_and_many_items(tmp_path, oracle):
    """K-streamed path with many items per CTA (accumulator, ring and hand-over reuse; odd
    tile count, so the last CTA pair holds one real tile; nk = 5 chunks, so the transform
    groups swap chunk parity every item): the default CTA-pair kernel (cta_group::2) and,
    in a subprocess with PQK_ENCODE_TCK_PAIR=0, the single-CTA kernel must both equal the oracle."""
    import os
    import subprocess
    import sys

    rng = np.random.default_rng(77)
    n, m, dsub = 128 * 332 + 57, 2, 160
    cw = rng.normal(size=(m, 256, dsub)).astype(np.float32)
    x = rng.normal(size=(n, m * dsub)).astype(np.float32)
    x[::7] = np.rint(x[::7] * 4)  # rows whose fp16 split has no lo part
    want = oracle.encode(cw, x)
    np.testing.assert_array_equal(_encode(cw, x), want)
    np.savez(tmp_path / "in.npz", cw=cw, x=x)
    env = dict(os.environ, PQK_ENCODE_TCK_PAIR="0")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    subprocess.run([sys.executable, "-c", _SIMT_SCRIPT, root, str(tmp_path / "in.npz"), str(tmp_path / "out.npy")],
                   check=True, env=env)
    np.testing.assert_array_equal(np.load(tmp_path / "out.npy"), want)
