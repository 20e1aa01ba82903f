"""Build the sm_100a shared library in-tree (nvcc, no torch types in the ABI).

The library lands next to this file as ``libpqk_b200.so`` so it travels with the
repository snapshot to the GPU box.  ``python -m paper_1709_03708_b200._build``
rebuilds it; ``__graft_entry__.build()`` calls :func:`build`.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libpqk_b200.so"
SOURCES = ["pqk_abi.cu", "pqk_assign.cu", "pqk_update.cu", "pqk_encode.cu", "pqk_encode_tc.cu", "pqk_train.cu",
           "pqk_eval.cu", "pqk_binary.cu", "pqk_ingest.cu", "pqk_probe.cu",
           "pqk_peer.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a into one shared library."""
    if not force and not _stale():
        return LIB
    objdir = PKG / "_obj"
    objdir.mkdir(exist_ok=True)
    flags = [
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC",
        "-Xptxas",
        "-v" if verbose else "-O3",
        "-I",
        str(INCLUDE),
        "-I",
        str(CSRC),
        *ARCH,
    ]
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc(), "-c", str(CSRC / src), "-o", str(obj), *flags]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", *ARCH, "-o", str(tmp), *objs, "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
