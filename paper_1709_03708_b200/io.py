"""Dataset / artifact files of the reference and the GPU streaming pipeline.

Formats (little-endian, reference io.py:1-19): fvecs / bvecs records ``[int32 d | d
components]``; PQKC codes (``"PQKC", version u32, N u64, M u32, L u32`` + N*M bytes);
PQCB codebooks (``"PQCB", version u32, D u32, M u32, L u32`` + M*L*(D/M) float32);
PQKB binary codes (``"PQKB", B u32, N u64`` + N*B/8 bytes); bare uint32 label files.
The host readers keep the reference's diagnostics (the offending record is named) and
stream fixed-size chunks; the device pipeline moves raw file bytes through pinned
buffers to the GPU, where ``pqk_unpack_*_device`` validate and unpack them:

* :func:`encode_fvecs` — fvecs/bvecs file -> GPU encoder -> PQKC file (cli.py:107-131),
  disk reads on a worker thread overlapping H2D, unpack, encode and D2H;
* :func:`load_codes` — PQKC file -> validated device code buffer, then
  :func:`fit_codes_file` runs ``fit`` on it without a host copy of the codes.
"""

from __future__ import annotations

import os
import queue
import struct
import threading
from pathlib import Path
from typing import Iterator

import numpy as np

from .pq import MAX_CODEWORDS, PQCodebook

FORMAT_VERSION = 1
_PQKC = struct.Struct("<4sIQII")
_PQCB = struct.Struct("<4sIIII")
_PQKB = struct.Struct("<4sIQ")
_NO_ERROR = np.iinfo(np.uint64).max


class FormatError(ValueError):
    """A file does not conform to its declared format."""


def _take(fh, nbytes: int, path, what: str) -> bytes:
    data = fh.read(nbytes)
    if len(data) != nbytes:
        raise FormatError(f"{path}: truncated {what} ({len(data)} of {nbytes} bytes)")
    return data


# ---------------------------------------------------------------------------
# fvecs / bvecs (io.py:50-144)
class _VecFile:
    """Geometry of an fvecs/bvecs file from its first record; chunked raw access."""

    def __init__(self, path, itemsize: int):
        self.path = path
        self.itemsize = itemsize
        self.size = os.path.getsize(path)
        self.dim = 0
        self.record_bytes = 0
        if self.size == 0:
            return
        if self.size < 4:
            raise FormatError(f"{path}: truncated record 0")
        with open(path, "rb") as fh:
            (self.dim,) = struct.unpack("<i", fh.read(4))
        if self.dim <= 0:
            raise FormatError(f"{path}: record 0 declares dimension {self.dim}")
        self.record_bytes = 4 + itemsize * self.dim

    def blocks(self, chunk_records: int) -> Iterator[tuple[int, np.ndarray]]:
        """(first record index, uint8 block of shape (count, record_bytes)) per chunk."""
        if self.size == 0:
            return
        with open(self.path, "rb") as fh:
            first = 0
            while True:
                data = fh.read(self.record_bytes * chunk_records)
                if not data:
                    return
                count, rest = divmod(len(data), self.record_bytes)
                if rest:  # checked before the dimensions of this chunk, as the reference does
                    raise FormatError(f"{self.path}: truncated record {first + count}")
                block = np.frombuffer(data, dtype=np.uint8).reshape(count, self.record_bytes)
                self.check_dims(block[:, :4].copy().view("<i4").ravel(), first)
                yield first, block
                first += count

    def check_dims(self, dims: np.ndarray, first: int) -> None:
        bad = np.flatnonzero(dims != self.dim)
        if len(bad):
            i = int(bad[0])
            raise FormatError(f"{self.path}: record {first + i} declares dimension {dims[i]}, expected {self.dim}")


def iter_fvecs(path, chunk_records: int = 65536) -> Iterator[np.ndarray]:
    """Stream an fvecs file as float32 chunks of shape (n_i, D)."""
    vf = _VecFile(path, 4)
    for _, block in vf.blocks(chunk_records):
        yield np.ascontiguousarray(block[:, 4:]).view("<f4").reshape(len(block), vf.dim).astype(np.float32)


def read_fvecs(path) -> np.ndarray:
    """Load a whole fvecs file as a float32 array of shape (N, D)."""
    parts = list(iter_fvecs(path))
    return np.concatenate(parts) if parts else np.empty((0, 0), dtype=np.float32)


def _write_records(path, payload: np.ndarray, dim: int) -> None:
    n = len(payload)
    head = np.full((n, 1), dim, dtype="<i4").view(np.uint8)
    with open(path, "wb") as fh:
        fh.write(np.concatenate([head, payload.view(np.uint8).reshape(n, -1)], axis=1).tobytes())


def write_fvecs(path, vectors: np.ndarray) -> None:
    """Write float32 vectors of shape (N, D) as an fvecs file."""
    data = np.ascontiguousarray(vectors, dtype="<f4")
    if data.ndim != 2 or data.shape[1] == 0:
        raise ValueError(f"vectors must have shape (N, D), D >= 1, got {data.shape}")
    _write_records(path, data, data.shape[1])


def iter_bvecs(path, chunk_records: int = 65536) -> Iterator[np.ndarray]:
    """Stream a bvecs file as float32 chunks (byte components widened)."""
    vf = _VecFile(path, 1)
    for _, block in vf.blocks(chunk_records):
        yield block[:, 4:].astype(np.float32)


def read_bvecs(path) -> np.ndarray:
    """Load a whole bvecs file, widened to float32."""
    parts = list(iter_bvecs(path))
    return np.concatenate(parts) if parts else np.empty((0, 0), dtype=np.float32)


def write_bvecs(path, vectors: np.ndarray) -> None:
    """Write integer-valued vectors in [0, 255] as a bvecs file."""
    data = np.asarray(vectors)
    if data.ndim != 2 or data.shape[1] == 0:
        raise ValueError(f"vectors must have shape (N, D), D >= 1, got {data.shape}")
    if not np.array_equal(np.rint(data), data) or data.min(initial=0) < 0 or data.max(initial=0) > 255:
        raise ValueError("bvecs components must be integers in [0, 255]")
    _write_records(path, np.ascontiguousarray(data, dtype=np.uint8), data.shape[1])


# ---------------------------------------------------------------------------
# PQKC code files (io.py:151-276)
def _check_code_values(arr: np.ndarray, num_codewords: int, what: str) -> None:
    if arr.size and int(arr.max()) >= num_codewords:
        raise ValueError(f"{what} {arr.max()}, must be below L={num_codewords}")


def write_codes(path, codes: np.ndarray, num_codewords: int) -> None:
    """Write uint8 PQ codes of shape (N, M) as a PQKC file."""
    arr = np.ascontiguousarray(codes, dtype=np.uint8)
    if arr.ndim != 2 or arr.shape[1] == 0:
        raise ValueError(f"codes must have shape (N, M), M >= 1, got {arr.shape}")
    if not 2 <= num_codewords <= MAX_CODEWORDS:
        raise ValueError(f"num_codewords must be in [2, {MAX_CODEWORDS}], got {num_codewords}")
    _check_code_values(arr, num_codewords, "codes contain index")
    with open(path, "wb") as fh:
        fh.write(_PQKC.pack(b"PQKC", FORMAT_VERSION, arr.shape[0], arr.shape[1], num_codewords))
        fh.write(arr.tobytes())


class CodesWriter:
    """Incremental PQKC writer: the header carries the promised record count and
    ``close`` checks that exactly that many records were written."""

    def __init__(self, path, n: int, m: int, num_codewords: int) -> None:
        if m < 1 or not 2 <= num_codewords <= MAX_CODEWORDS:
            raise ValueError(f"invalid code geometry M={m}, L={num_codewords}")
        self._path, self._n, self._m, self._l = path, n, m, num_codewords
        self._written = 0
        self._fh = open(path, "wb")
        self._fh.write(_PQKC.pack(b"PQKC", FORMAT_VERSION, n, m, num_codewords))

    def write(self, codes: np.ndarray) -> None:
        arr = np.ascontiguousarray(codes, dtype=np.uint8)
        if arr.ndim != 2 or arr.shape[1] != self._m:
            raise ValueError(f"chunk must have shape (n, {self._m}), got {arr.shape}")
        _check_code_values(arr, self._l, "chunk contains index")
        self._fh.write(arr.tobytes())
        self._written += len(arr)

    def close(self) -> None:
        self._fh.close()
        if self._written != self._n:
            raise ValueError(f"{self._path}: wrote {self._written} records, header promised {self._n}")

    def __enter__(self) -> "CodesWriter":
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        if exc_type is None:
            self.close()
        else:
            self._fh.close()


def read_codes_header(path) -> tuple[int, int, int]:
    """Return (N, M, L) from a PQKC header."""
    with open(path, "rb") as fh:
        magic, version, n, m, l_count = _PQKC.unpack(_take(fh, _PQKC.size, path, "PQKC header"))
    if magic != b"PQKC":
        raise FormatError(f"{path}: bad magic {magic!r}, expected b'PQKC'")
    if version != FORMAT_VERSION:
        raise FormatError(f"{path}: unsupported PQKC version {version}")
    if m == 0 or not 2 <= l_count <= MAX_CODEWORDS:
        raise FormatError(f"{path}: invalid header fields M={m}, L={l_count}")
    return n, m, l_count


def _code_chunks(path, chunk_records: int, into=None) -> Iterator[tuple[int, int, object]]:
    """(first record, count, buffer) per chunk of a PQKC payload: a bytes object, or the
    filled prefix of ``into`` (a writable uint8 buffer of chunk_records * M bytes)."""
    n, m, _ = read_codes_header(path)
    with open(path, "rb") as fh:
        fh.seek(_PQKC.size)
        first = 0
        while first < n:
            want = min(chunk_records, n - first)
            if into is None:
                buf = fh.read(want * m)
                got = len(buf)
            else:
                buf = memoryview(into)[: want * m]
                got = fh.readinto(buf)
            count = got // m
            if count < want:
                raise FormatError(f"{path}: truncated record {first + count} (header promises {n} records)")
            yield first, count, buf
            first += count
        if fh.read(1):
            raise FormatError(f"{path}: trailing bytes after {n} records")


def iter_codes(path, chunk_records: int = 262144) -> Iterator[np.ndarray]:
    """Stream a PQKC file as uint8 chunks of shape (n_i, M)."""
    _, m, l_count = read_codes_header(path)
    for first, count, buf in _code_chunks(path, chunk_records):
        chunk = np.frombuffer(buf, dtype=np.uint8).reshape(count, m)
        if chunk.size and int(chunk.max()) >= l_count:
            flat = int(np.argmax(chunk.ravel() >= l_count))
            raise FormatError(f"{path}: record {first + flat // m} holds subindex {chunk.ravel()[flat]}, "
                              f"must be below L={l_count}")
        yield chunk.copy()


def read_codes(path) -> tuple[np.ndarray, int, int]:
    """Load a PQKC file. Returns (codes of shape (N, M), M, L)."""
    _, m, l_count = read_codes_header(path)
    parts = list(iter_codes(path))
    return (np.concatenate(parts) if parts else np.empty((0, m), np.uint8)), m, l_count


# ---------------------------------------------------------------------------
# PQCB codebooks, PQKB binary codes, labels (io.py:279-371)
def write_codebook(path, codebook: PQCodebook) -> None:
    """Write a PQCodebook as a PQCB file."""
    m, l_count, _ = codebook.codewords.shape
    with open(path, "wb") as fh:
        fh.write(_PQCB.pack(b"PQCB", FORMAT_VERSION, codebook.dim, m, l_count))
        fh.write(np.ascontiguousarray(codebook.codewords, dtype="<f4").tobytes())


def read_codebook(path) -> PQCodebook:
    """Load a PQCB file into a PQCodebook."""
    with open(path, "rb") as fh:
        magic, version, dim, m, l_count = _PQCB.unpack(_take(fh, _PQCB.size, path, "PQCB header"))
        if magic != b"PQCB":
            raise FormatError(f"{path}: bad magic {magic!r}, expected b'PQCB'")
        if version != FORMAT_VERSION:
            raise FormatError(f"{path}: unsupported PQCB version {version}")
        if m == 0 or dim % m != 0 or not 2 <= l_count <= MAX_CODEWORDS:
            raise FormatError(f"{path}: invalid header fields D={dim}, M={m}, L={l_count}")
        payload = _take(fh, 4 * m * l_count * (dim // m), path, "PQCB payload")
        if fh.read(1):
            raise FormatError(f"{path}: trailing bytes after codebook payload")
    return PQCodebook(np.frombuffer(payload, dtype="<f4").reshape(m, l_count, dim // m).copy())


def write_binary_codes(path, packed: np.ndarray) -> None:
    """Write packed binary codes of shape (N, B/8) as a PQKB file."""
    arr = np.ascontiguousarray(packed, dtype=np.uint8)
    if arr.ndim != 2 or arr.shape[1] == 0:
        raise ValueError(f"packed codes must have shape (N, B/8), got {arr.shape}")
    with open(path, "wb") as fh:
        fh.write(_PQKB.pack(b"PQKB", 8 * arr.shape[1], len(arr)))
        fh.write(arr.tobytes())


def read_binary_codes(path) -> tuple[np.ndarray, int]:
    """Load a PQKB file. Returns (packed codes of shape (N, B/8), B)."""
    with open(path, "rb") as fh:
        magic, bits, n = _PQKB.unpack(_take(fh, _PQKB.size, path, "PQKB header"))
        if magic != b"PQKB":
            raise FormatError(f"{path}: bad magic {magic!r}, expected b'PQKB'")
        if bits == 0 or bits % 8 != 0:
            raise FormatError(f"{path}: bit count {bits} is not a positive multiple of 8")
        payload = _take(fh, n * (bits // 8), path, "PQKB payload")
        if fh.read(1):
            raise FormatError(f"{path}: trailing bytes after {n} records")
    return np.frombuffer(payload, dtype=np.uint8).reshape(n, bits // 8).copy(), bits


def write_labels(path, labels: np.ndarray) -> None:
    """Write cluster labels as a bare little-endian uint32 array."""
    arr = np.asarray(labels)
    if arr.ndim != 1:
        raise ValueError(f"labels must be 1-d, got shape {arr.shape}")
    if arr.size and (arr.min() < 0 or arr.max() > np.iinfo(np.uint32).max):
        raise ValueError("labels must fit in uint32")
    Path(path).write_bytes(np.ascontiguousarray(arr, dtype="<u4").tobytes())


def read_labels(path) -> np.ndarray:
    """Load a bare uint32 label array."""
    raw = Path(path).read_bytes()
    if len(raw) % 4:
        raise FormatError(f"{path}: size {len(raw)} is not a multiple of 4")
    return np.frombuffer(raw, dtype="<u4").copy()


# ---------------------------------------------------------------------------
# GPU streaming pipeline
def _device_error(err, first_bad_message) -> None:
    vals = err.cpu().numpy().view(np.uint64)
    if int(vals[0]) != int(_NO_ERROR):
        raise FormatError(first_bad_message(int(vals[0]), int(vals[1])))


def encode_fvecs(codebook: PQCodebook, data_path, out_path, *, chunk_records: int = 1 << 20, bvecs: bool = False,
                 device=None) -> int:
    """Encode an fvecs (or bvecs) file into a PQKC file on the GPU (cli.py:107-131).

    Raw records are read on a worker thread into pinned buffers, copied to the device,
    validated and unpacked there (``pqk_unpack_vecs_device``), encoded by the tensor-core
    encoder, and the codes are appended through :class:`CodesWriter`.  Returns N."""
    import torch

    from . import _lib, engine

    itemsize = 1 if bvecs else 4
    size = os.path.getsize(data_path)
    record_bytes = 4 + itemsize * codebook.dim
    if size % record_bytes:
        raise ValueError(f"{data_path}: size {size} does not divide into records of dimension {codebook.dim}")
    n = size // record_bytes
    if n == 0:
        raise ValueError(f"{data_path}: no vectors to encode")
    vf = _VecFile(data_path, itemsize)
    if vf.dim != codebook.dim:
        raise ValueError(f"{data_path}: vectors have dimension {vf.dim}, codebook expects {codebook.dim}")
    dev = engine.device_of(device)
    m, l_count = codebook.num_subspaces, codebook.num_codewords
    chunk = min(chunk_records, n)
    nslots = 3
    with torch.cuda.device(dev):
        pinned = [torch.empty(chunk * record_bytes, dtype=torch.uint8).pin_memory() for _ in range(nslots)]
        h2d_done = [torch.cuda.Event() for _ in range(nslots)]
        raw_dev = torch.empty(chunk * record_bytes + 16, dtype=torch.uint8, device=dev)
        vec_dev = torch.empty((chunk, codebook.dim), dtype=torch.float32, device=dev)
        cw_dev = torch.from_numpy(np.array(codebook.codewords, dtype=np.float32)).to(dev)
        err = torch.full((2,), -1, dtype=torch.int64, device=dev)
        stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
        codes_pin = torch.empty((chunk, m), dtype=torch.uint8).pin_memory()
        stream = torch.cuda.current_stream(dev)
        filled: queue.Queue = queue.Queue()
        free: queue.Queue = queue.Queue()
        for s in range(nslots):
            free.put(s)
        stop = threading.Event()

        def reader():
            try:
                with open(data_path, "rb") as fh:
                    first = 0
                    while first < n and not stop.is_set():
                        s = free.get()
                        if s is None:
                            return
                        h2d_done[s].synchronize()  # the copy that last read this slot has finished
                        count = min(chunk, n - first)
                        view = pinned[s].numpy()[: count * record_bytes]
                        if fh.readinto(memoryview(view)) != count * record_bytes:
                            raise FormatError(f"{data_path}: truncated record {first}")
                        filled.put((first, count, s))
                        first += count
                filled.put(None)
            except BaseException as exc:  # surfaced on the consumer side
                filled.put(exc)

        worker = threading.Thread(target=reader, daemon=True)
        worker.start()
        try:
            with CodesWriter(out_path, n, m, l_count) as writer:
                while True:
                    item = filled.get()
                    if item is None:
                        break
                    if isinstance(item, BaseException):
                        raise item
                    first, count, s = item
                    raw_dev[: count * record_bytes].copy_(pinned[s][: count * record_bytes], non_blocking=True)
                    h2d_done[s].record(stream)
                    free.put(s)
                    engine.call("pqk_unpack_vecs_device", engine._ptr(raw_dev), count, codebook.dim, itemsize, first,
                                engine._ptr(vec_dev), engine._ptr(err), engine._stream(dev))
                    codes = engine.encode_device(vec_dev[:count], cw_dev, m, l_count, dev, stride=m, stats=stats)
                    codes_pin[:count].copy_(codes, non_blocking=True)
                    stream.synchronize()
                    _device_error(err, lambda i, d: f"{data_path}: record {i} declares dimension "
                                                    f"{np.uint32(d).view(np.int32)}, expected {codebook.dim}")
                    writer.write(codes_pin[:count].numpy())
        finally:
            stop.set()
            free.put(None)
            worker.join()
    return n


def load_codes(path, *, chunk_records: int = 1 << 22, device=None):
    """Stream a PQKC file onto the GPU: returns (codes_dev (N, MP) uint8, N, M, L).

    Payload chunks are read into pinned memory and validated on the device (the first
    subindex >= L is reported exactly as :func:`iter_codes` reports it)."""
    import torch

    from . import _lib, engine

    n, m, l_count = read_codes_header(path)
    dev = engine.device_of(device)
    mp = _lib.padded_m(m)
    chunk = max(1, min(chunk_records, n))
    with torch.cuda.device(dev):
        codes_dev = torch.zeros((max(n, 1), mp), dtype=torch.uint8, device=dev)
        pinned = [torch.empty(chunk * m, dtype=torch.uint8).pin_memory() for _ in range(2)]
        raw_dev = torch.empty(chunk * m, dtype=torch.uint8, device=dev)
        err = torch.full((2,), -1, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev)

        def check():  # subindex errors of the chunks submitted so far, in file order
            _device_error(err, lambda pos, v: f"{path}: record {pos // m} holds subindex {v}, "
                                              f"must be below L={l_count}")

        with open(path, "rb") as fh:
            fh.seek(_PQKC.size)

            def read(first, slot):
                want = min(chunk, n - first)
                got = fh.readinto(memoryview(pinned[slot].numpy()[: want * m]))
                if got // m < want:
                    stream.synchronize()
                    check()  # an earlier chunk's bad subindex is reported first, as iter_codes does
                    raise FormatError(f"{path}: truncated record {first + got // m} (header promises {n} records)")
                return want

            first, slot = 0, 0
            count = read(0, 0) if n else 0
            while first < n:
                raw_dev[: count * m].copy_(pinned[slot][: count * m], non_blocking=True)
                engine.call("pqk_unpack_codes_device", engine._ptr(raw_dev), count, m, l_count, first,
                            engine._ptr(codes_dev[first:]), mp, engine._ptr(err), engine._stream(dev))
                nxt_first = first + count
                nxt = read(nxt_first, slot ^ 1) if nxt_first < n else 0  # disk read overlaps the GPU work
                stream.synchronize()  # raw_dev and pinned[slot] are free again
                check()
                first, count, slot = nxt_first, nxt, slot ^ 1
            if fh.read(1):
                raise FormatError(f"{path}: trailing bytes after {n} records")
    return codes_dev, n, m, l_count


def fit_codes_file(path, tables, k: int, max_iterations: int = 20, seed: int = 0, *, update: str = "sparse",
                   initial_centers=None, device=None):
    """``fit`` on a PQKC file: codes streamed to the GPU (:func:`load_codes`), clustered
    there (clustering.fit_device) without a host copy."""
    from .clustering import fit_device
    from .pq import as_tables

    codes_dev, n, m, l_count = load_codes(path, device=device)
    t = as_tables(tables)
    if (t.num_subspaces, t.num_codewords) != (m, l_count):
        raise ValueError(f"{path}: codes have M={m}, L={l_count}; tables have M={t.num_subspaces}, "
                         f"L={t.num_codewords}")
    return fit_device(codes_dev, n, t, k, max_iterations, seed, update=update, initial_centers=initial_centers,
                      device=device)
