"""GPU streaming pipeline: fvecs/bvecs -> device unpack -> encoder ->
PQKC file, and PQKC file -> device codes -> fit, against the reference semantics (the
oracle encoder, the reference's PQKC bytes) and its diagnostics."""

import struct

import numpy as np
import pytest

from helpers import random_codebook

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pqk():
    import paper_1709_03708_b200 as pqk

    return pqk


def test_encode_fvecs_matches_oracle(tmp_path, pqk, oracle):
    from paper_1709_03708_b200 import io as pio

    rng = np.random.default_rng(1)
    x = (rng.normal(size=(20_011, 64)) * 4).astype(np.float32)
    cw = random_codebook(4, 256, 16, seed=3) * 4
    pio.write_fvecs(tmp_path / "x.fvecs", x)
    book = pqk.PQCodebook(cw)
    n = pio.encode_fvecs(book, tmp_path / "x.fvecs", tmp_path / "x.pqkc", chunk_records=4096)  # 5 chunks + tail
    assert n == len(x)
    pio.write_codes(tmp_path / "ref.pqkc", oracle.encode(cw, x), 256)
    assert (tmp_path / "x.pqkc").read_bytes() == (tmp_path / "ref.pqkc").read_bytes()


def test_encode_bvecs(tmp_path, pqk, oracle):
    from paper_1709_03708_b200 import io as pio

    rng = np.random.default_rng(2)
    x = rng.integers(0, 256, size=(3000, 32)).astype(np.float32)
    cw = (random_codebook(2, 64, 16, seed=4) * 40 + 128).astype(np.float32)
    pio.write_bvecs(tmp_path / "x.bvecs", x)
    pio.encode_fvecs(pqk.PQCodebook(cw), tmp_path / "x.bvecs", tmp_path / "x.pqkc", bvecs=True, chunk_records=1000)
    codes, m, l_count = pio.read_codes(tmp_path / "x.pqkc")
    assert np.array_equal(codes, oracle.encode(cw, x)) and (m, l_count) == (2, 64)


def test_encode_fvecs_diagnostics(tmp_path, pqk):
    from paper_1709_03708_b200 import io as pio

    book = pqk.PQCodebook(random_codebook(2, 16, 4, seed=5))
    x = np.ones((50, 8), np.float32)
    p = tmp_path / "x.fvecs"
    pio.write_fvecs(p, x)
    raw = bytearray(p.read_bytes())
    raw[36 * 17: 36 * 17 + 4] = struct.pack("<i", 5)  # record 17 declares dimension 5
    p.write_bytes(bytes(raw))
    with pytest.raises(pio.FormatError, match="record 17 declares dimension 5, expected 8"):
        pio.encode_fvecs(book, p, tmp_path / "o.pqkc", chunk_records=8)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(ValueError, match="does not divide into records of dimension 8"):
        pio.encode_fvecs(book, p, tmp_path / "o.pqkc")
    p.write_bytes(b"")
    with pytest.raises(ValueError, match="no vectors to encode"):
        pio.encode_fvecs(book, p, tmp_path / "o.pqkc")
    pio.write_fvecs(p, np.ones((9, 4), np.float32))  # 9 x 20 bytes = 5 x 36 bytes
    with pytest.raises(ValueError, match="vectors have dimension 4, codebook expects 8"):
        pio.encode_fvecs(book, p, tmp_path / "o.pqkc")


def test_load_codes_and_fit_codes_file(tmp_path, pqk, oracle):
    from paper_1709_03708_b200 import engine
    from paper_1709_03708_b200 import io as pio
    from helpers import mixture_codes, random_tables

    codes = mixture_codes(30_001, 4, 256, 60, seed=8)
    tables = random_tables(4, 256, seed=9, sub_dim=8)
    pio.write_codes(tmp_path / "c.pqkc", codes, 256)
    dev_codes, n, m, l_count = pio.load_codes(tmp_path / "c.pqkc", chunk_records=7000)
    assert (n, m, l_count) == (30_001, 4, 256)
    assert np.array_equal(engine.download_codes(dev_codes, 4), codes)
    res = pio.fit_codes_file(tmp_path / "c.pqkc", tables, 200, max_iterations=5, seed=3)
    ref = pqk.fit(codes, tables, 200, max_iterations=5, seed=3)
    assert np.array_equal(res.labels, ref.labels) and np.array_equal(res.centers, ref.centers)
    assert [s.objective for s in res.trace] == [s.objective for s in ref.trace]


def test_load_codes_diagnostics(tmp_path):
    from paper_1709_03708_b200 import io as pio

    codes = (np.arange(40, dtype=np.uint8).reshape(20, 2) % 4)
    pio.write_codes(tmp_path / "c", codes, 4)
    raw = (tmp_path / "c").read_bytes()
    hdr = struct.calcsize("<4sIQII")
    bad = bytearray(raw)
    bad[hdr + 2 * 13 + 1] = 9
    (tmp_path / "b").write_bytes(bytes(bad))
    with pytest.raises(pio.FormatError, match="record 13 holds subindex 9, must be below L=4"):
        pio.load_codes(tmp_path / "b", chunk_records=6)
    bad[hdr + 2 * 3] = 5  # an earlier chunk's error wins over the truncation of a later one
    (tmp_path / "bt").write_bytes(bytes(bad)[: hdr + 2 * 15 + 1])
    with pytest.raises(pio.FormatError, match="record 3 holds subindex 5"):
        pio.load_codes(tmp_path / "bt", chunk_records=6)
    (tmp_path / "t").write_bytes(raw[: hdr + 2 * 15 + 1])
    with pytest.raises(pio.FormatError, match="truncated record 15"):
        pio.load_codes(tmp_path / "t", chunk_records=6)
    (tmp_path / "x").write_bytes(raw + b"\x01")
    with pytest.raises(pio.FormatError, match="trailing bytes after 20 records"):
        pio.load_codes(tmp_path / "x", chunk_records=6)
