"""File formats (reference io.py): writers produce the reference's bytes (golden files
written by the reference itself), readers round-trip them and raise the reference's
diagnostics on damaged files.  Host-only (no GPU)."""

import struct

import numpy as np
import pytest

from golden_io import load

from paper_1709_03708_b200 import io as pio
from paper_1709_03708_b200.pq import PQCodebook


@pytest.fixture(scope="module")
def g():
    return load("io")


def _bytes(path):
    return np.frombuffer(path.read_bytes(), dtype=np.uint8)


def test_writers_match_reference_bytes(tmp_path, g):
    pio.write_fvecs(tmp_path / "a", g["vec"])
    pio.write_bvecs(tmp_path / "b", g["bvec"])
    pio.write_codes(tmp_path / "c", g["codes"], 200)
    pio.write_codebook(tmp_path / "d", PQCodebook(g["book"]))
    pio.write_binary_codes(tmp_path / "e", g["packed"])
    pio.write_labels(tmp_path / "f", g["labels"])
    for name, ref in zip("abcdef", ["fvecs", "bvecs", "pqkc", "pqcb", "pqkb", "labels"]):
        assert np.array_equal(_bytes(tmp_path / name), g[f"file_{ref}"]), ref


def test_readers_round_trip_reference_files(tmp_path, g):
    for name in ("fvecs", "bvecs", "pqkc", "pqcb", "pqkb", "labels"):
        (tmp_path / name).write_bytes(g[f"file_{name}"].tobytes())
    assert np.array_equal(pio.read_fvecs(tmp_path / "fvecs"), g["vec"])
    assert np.array_equal(pio.read_bvecs(tmp_path / "bvecs"), g["bvec"])
    codes, m, l_count = pio.read_codes(tmp_path / "pqkc")
    assert np.array_equal(codes, g["codes"]) and (m, l_count) == (6, 200)
    assert pio.read_codes_header(tmp_path / "pqkc") == (53, 6, 200)
    assert np.array_equal(pio.read_codebook(tmp_path / "pqcb").codewords, g["book"])
    packed, bits = pio.read_binary_codes(tmp_path / "pqkb")
    assert np.array_equal(packed, g["packed"]) and bits == 24
    assert np.array_equal(pio.read_labels(tmp_path / "labels"), g["labels"])
    chunks = list(pio.iter_fvecs(tmp_path / "fvecs", chunk_records=5))
    assert [len(c) for c in chunks] == [5] * 7 + [2]
    assert np.array_equal(np.concatenate(list(pio.iter_codes(tmp_path / "pqkc", chunk_records=10))), g["codes"])


def test_vector_file_diagnostics(tmp_path):
    p = tmp_path / "v.fvecs"
    pio.write_fvecs(p, np.ones((3, 4), np.float32))
    raw = bytearray(p.read_bytes())
    raw[20:24] = struct.pack("<i", 3)  # record 1 (offset 20) declares dimension 3
    p.write_bytes(bytes(raw))
    with pytest.raises(pio.FormatError, match="record 1 declares dimension 3, expected 4"):
        pio.read_fvecs(p)
    pio.write_fvecs(p, np.ones((3, 4), np.float32))
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(pio.FormatError, match="truncated record 2"):
        pio.read_fvecs(p)
    p.write_bytes(b"\x01\x00")
    with pytest.raises(pio.FormatError, match="truncated record 0"):
        pio.read_fvecs(p)
    p.write_bytes(struct.pack("<i", -1) + b"\x00" * 8)
    with pytest.raises(pio.FormatError, match="record 0 declares dimension -1"):
        pio.read_fvecs(p)
    p.write_bytes(b"")
    assert pio.read_fvecs(p).shape == (0, 0)
    with pytest.raises(ValueError, match="shape"):
        pio.write_fvecs(p, np.ones(3, np.float32))
    with pytest.raises(ValueError, match="integers in"):
        pio.write_bvecs(p, np.full((2, 2), 256))


def test_code_file_diagnostics(tmp_path):
    p = tmp_path / "c.pqkc"
    codes = np.arange(20, dtype=np.uint8).reshape(10, 2) % 4
    pio.write_codes(p, codes, 4)
    raw = p.read_bytes()
    hdr = struct.calcsize("<4sIQII")
    (tmp_path / "m").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(pio.FormatError, match="bad magic"):
        pio.read_codes(tmp_path / "m")
    (tmp_path / "v").write_bytes(raw[:4] + struct.pack("<I", 9) + raw[8:])
    with pytest.raises(pio.FormatError, match="version 9"):
        pio.read_codes(tmp_path / "v")
    (tmp_path / "t").write_bytes(raw[: hdr + 7])
    with pytest.raises(pio.FormatError, match="truncated record 3"):
        pio.read_codes(tmp_path / "t")
    bad = bytearray(raw)
    bad[hdr + 3] = 7
    (tmp_path / "b").write_bytes(bytes(bad))
    with pytest.raises(pio.FormatError, match="record 1 holds subindex 7"):
        pio.read_codes(tmp_path / "b")
    (tmp_path / "x").write_bytes(raw + b"\x00")
    with pytest.raises(pio.FormatError, match="trailing bytes"):
        pio.read_codes(tmp_path / "x")
    (tmp_path / "h").write_bytes(struct.pack("<4sIQII", b"PQKC", 1, 1, 0, 4))
    with pytest.raises(pio.FormatError, match="invalid header"):
        pio.read_codes(tmp_path / "h")
    with pytest.raises(ValueError, match="num_codewords"):
        pio.write_codes(p, codes, 1)
    with pytest.raises(ValueError, match="below L=4"):
        pio.write_codes(p, codes + 4, 4)


def test_codes_writer(tmp_path):
    codes = np.arange(24, dtype=np.uint8).reshape(12, 2) % 8
    with pio.CodesWriter(tmp_path / "w", 12, 2, 8) as w:
        w.write(codes[:5])
        w.write(codes[5:])
    pio.write_codes(tmp_path / "r", codes, 8)
    assert (tmp_path / "w").read_bytes() == (tmp_path / "r").read_bytes()
    with pytest.raises(ValueError, match="geometry"):
        pio.CodesWriter(tmp_path / "z", 4, 0, 8)
    w = pio.CodesWriter(tmp_path / "z", 4, 2, 8)
    with pytest.raises(ValueError, match=r"shape \(n, 2\)"):
        w.write(np.zeros((2, 3), np.uint8))
    with pytest.raises(ValueError, match="below L=8"):
        w.write(np.full((1, 2), 8, np.uint8))
    w.write(np.zeros((2, 2), np.uint8))
    with pytest.raises(ValueError, match="header promised 4"):
        w.close()


def test_other_file_diagnostics(tmp_path):
    p = tmp_path / "cb"
    pio.write_codebook(p, PQCodebook(np.ones((2, 4, 3), np.float32)))
    raw = p.read_bytes()
    (tmp_path / "a").write_bytes(raw[:10])
    with pytest.raises(pio.FormatError, match="truncated PQCB header"):
        pio.read_codebook(tmp_path / "a")
    (tmp_path / "b").write_bytes(raw[:-4])
    with pytest.raises(pio.FormatError, match="truncated PQCB payload"):
        pio.read_codebook(tmp_path / "b")
    (tmp_path / "c").write_bytes(raw + b"\x00")
    with pytest.raises(pio.FormatError, match="trailing bytes"):
        pio.read_codebook(tmp_path / "c")
    (tmp_path / "d").write_bytes(struct.pack("<4sIQ", b"PQKB", 12, 1) + b"\x00\x00")
    with pytest.raises(pio.FormatError, match="multiple of 8"):
        pio.read_binary_codes(tmp_path / "d")
    (tmp_path / "e").write_bytes(b"\x00" * 5)
    with pytest.raises(pio.FormatError, match="multiple of 4"):
        pio.read_labels(tmp_path / "e")
    with pytest.raises(ValueError, match="uint32"):
        pio.write_labels(tmp_path / "f", np.array([-1]))
