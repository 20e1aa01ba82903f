"""ctypes binding of ``libpqk_b200.so`` (declared in ``include/pqk_b200.h``).

This is the same binding a maintainer of the reference would add to reach the
C-ABI.  Every call returns a ``pqk_status_t``; non-zero
statuses raise ``ValueError`` (PQK_EINVAL), ``MemoryError`` (PQK_ENOMEM) or
``RuntimeError``.  There is no fallback: if the library is missing the import of
any compute entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PQK_B200_LIB", _PKG / "libpqk_b200.so"))

PQK_OK, PQK_EINVAL, PQK_ECUDA, PQK_ENOMEM, PQK_EUNSUPPORTED = range(5)

STAT_UNIQUE_CENTERS = 0
STAT_FLAGGED = 1
STAT_FLAGGED_FP64 = 9
STAT_LOOKUP_BYTES = 10
STAT_NNZ_TOTAL = 2
STAT_EMPTY = 3
STAT_FILLED = 4
STAT_VOTE_EXACT = 5
STAT_ENCODE_FLAGGED = 6
STAT_NCHUNKS = 7
STAT_VOTE_FP64 = 8
STATS_LEN = 24

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t

# name -> (restype, argtypes); the full C-ABI of include/pqk_b200.h
SIGNATURES: dict[str, tuple] = {
    "pqk_abi_version": (C.c_int, []),
    "pqk_last_error": (C.c_char_p, []),
    "pqk_device_info": (C.c_int, [_i32, C.POINTER(_i32), C.POINTER(_i32)]),
    "pqk_padded_m": (_i32, [_i32]),
    "pqk_set_scan_mode": (C.c_int, [_i32]),
    "pqk_get_scan_mode": (_i32, []),
    "pqk_launch_count": (_i64, []),
    "pqk_set_profile_events": (C.c_int, [_p, _p]),
    "pqk_table_scale": (C.c_int, [_p, _i64, C.POINTER(_i32), C.POINTER(_i32)]),
    "pqk_pairwise_plan_size": (C.c_int, [_i64, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64)]),
    "pqk_pairwise_plan_build": (C.c_int, [_i64, _p, _p, _p, _p, _p]),
    "pqk_tables_to_f32": (C.c_int, [_p, _i32, _i32, _i32, _p, _p]),
    "pqk_pad_codes_device": (C.c_int, [_p, _i64, _i32, _p, _p]),
    "pqk_assign_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "pqk_assign_device": (
        C.c_int,
        [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _i32, _p, _sz, _p, _p, _p, _p],
    ),
    "pqk_paired_distance_device": (C.c_int, [_p, _p, _p, _i64, _i32, _i32, _p, _p, _p]),
    "pqk_histogram_device": (C.c_int, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p]),
    "pqk_vote_device": (C.c_int, [_p, _p, _i64, _i32, _i32, _p, _p, _p, _p, _p]),
    "pqk_vote_tables16_device": (C.c_int, [_p, _i32, _i32, _p, _p]),
    "pqk_vote16_device": (C.c_int, [_p, _p, _i64, _i32, _i32, _p, _p, _p, _p, _p, _p]),
    "pqk_repair_workspace_bytes": (_sz, [_i64, _i64]),
    "pqk_repair_device": (C.c_int, [_p, _p, _i64, _i32, _p, _i64, _p, _p, _sz, _p, _p]),
    "pqk_repair_candidates_device": (C.c_int, [_p, _i64, _i64, _i64, _p, _sz, _p, _p, _p]),
    "pqk_objective_workspace_bytes": (_sz, [_i64, _i64]),
    "pqk_objective_device": (C.c_int, [_p, _i64, _i64, _i32, _p, _p, _p, _p, _p, _p, _sz, _p, _p]),
    "pqk_encode_device": (C.c_int, [_p, _i64, _i32, _p, _i32, _i32, _p, _i32, _p, _p]),
    "pqk_assign_host": (C.c_int, [_p, _i64, _i32, _p, _i64, _p, _i32, _p, _p, _i32]),
    "pqk_encode_host": (C.c_int, [_p, _i64, _i32, _p, _i32, _i32, _p, _i32]),
    "pqk_lloyd_step_host": (C.c_int, [_p, _i64, _i32, _p, _i64, _p, _i32, _p, _p, _p, _p, _i32]),
    "pqk_host_release": (C.c_int, [_i32]),
    "pqk_tc_selftest": (C.c_int, [_p, _p, _p, _i32, _p]),
    "pqk_peer_sum_device": (C.c_int, [_p, _i32, _i64, _p, _p]),
    "pqk_enable_peer_access": (C.c_int, [_p, _i32]),
    "pqk_smem_probe": (C.c_int, [_i32, _i32, C.POINTER(C.c_double), C.POINTER(C.c_double), _p]),
    "pqk_tmem_probe": (C.c_int, [_i32, _i32, C.POINTER(C.c_double), C.POINTER(C.c_double), _p]),
    "pqk_train_workspace_bytes": (_sz, [_i64, _i32]),
    "pqk_train_step_device": (C.c_int, [_p, _i64, _i32, _i32, _i32, _p, _i32, _p, _p, _p, _p, _p, _sz, _p, _p]),
    "pqk_build_tables_device": (C.c_int, [_p, _i32, _i32, _i32, _p, _p]),
    "pqk_cluster_means_workspace_bytes": (_sz, [_i64, _i32]),
    "pqk_cluster_means_device": (C.c_int, [_p, _i32, _i64, _i32, _p, _i32, _p, _p, _p, _sz, _p]),
    "pqk_assigned_sq_device": (C.c_int, [_p, _i32, _i64, _i32, _p, _p, _p, _p]),
    "pqk_binarize_device": (C.c_int, [_p, _i64, _i32, _p, _i32, _p, _i32, _p, _p]),
    "pqk_hamming_assign_device": (C.c_int, [_p, _i64, _i32, _p, _i64, _p, _p, _p, _p]),
    "pqk_hamming_matrix_device": (C.c_int, [_p, _i64, _i32, _p, _i64, _p, _p]),
    "pqk_majority_update_device": (C.c_int, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p, _p, _p]),
    "pqk_unpack_vecs_device": (C.c_int, [_p, _i64, _i32, _i32, _i64, _p, _p, _p]),
    "pqk_unpack_codes_device": (C.c_int, [_p, _i64, _i32, _i32, _i64, _p, _i32, _p, _p]),
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the library (once) and attach the C signatures; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1709_03708_b200._build` "
            "(the CUDA extension is required; there is no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pqk_abi_version() != 1:
        raise ImportError("libpqk_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    """Map a pqk_status_t to the reference's exception types."""
    if status == PQK_OK:
        return
    msg = load().pqk_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == PQK_EINVAL:
        raise ValueError(msg)
    if status == PQK_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def padded_m(m: int) -> int:
    return int(load().pqk_padded_m(int(m)))
