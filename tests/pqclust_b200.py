"""Register the B200 linear scan in pqclust's strategy registry (opt-in)."""
import ctypes as C
import os

import numpy as np

from pqclust.clustering import register_assignment_strategy

_lib = C.CDLL(os.environ.get("PQK_B200_LIB", "libpqk_b200.so"))  # paper_1709_03708_b200/libpqk_b200.so
_lib.pqk_assign_host.restype = C.c_int
_lib.pqk_assign_host.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32]
_lib.pqk_encode_host.restype = C.c_int
_lib.pqk_encode_host.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_void_p, C.c_int32]
_lib.pqk_last_error.restype = C.c_char_p


def _check(rc):
    if rc:
        msg = _lib.pqk_last_error().decode()
        raise (ValueError if rc == 1 else MemoryError if rc == 3 else RuntimeError)(msg)


def b200_assign(codes, centers, tables, threads):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)      # validated upstream (clustering.py:276-279)
    centers = np.ascontiguousarray(centers, dtype=np.uint8)
    t = np.ascontiguousarray(tables.tables, dtype=np.float64)
    labels = np.empty(len(codes), dtype=np.uint32)
    _check(_lib.pqk_assign_host(codes.ctypes.data, len(codes), codes.shape[1], centers.ctypes.data,
                                len(centers), t.ctypes.data, t.shape[1], labels.ctypes.data, None, 0))
    return labels


def b200_encode(codebook, vectors):
    """pq.encode(codebook, vectors) on the GPU (pq.py:205-231)."""
    x = np.ascontiguousarray(vectors, dtype=np.float32)
    cw = np.ascontiguousarray(codebook.codewords, dtype=np.float32)
    m, l_count, _ = cw.shape
    codes = np.empty((len(x), m), dtype=np.uint8)
    _check(_lib.pqk_encode_host(x.ctypes.data, len(x), x.shape[1], cw.ctypes.data, m, l_count,
                                codes.ctypes.data, 0))
    return codes


def enable():
    register_assignment_strategy("b200", b200_assign)   # explicit: never on import
