"""Loading helpers for the reference-generated golden vectors (tests/golden/*.npz)."""

import hashlib
from functools import lru_cache
from pathlib import Path

import numpy as np

from oracle import pqk_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


def tables(g: dict, prefix: str) -> np.ndarray:
    """Rebuild the reference tables from the stored codebook and check their hash."""
    t = O.build_distance_tables(g[f"{prefix}codebook"])
    sha = hashlib.sha256(t.tobytes()).hexdigest()
    assert sha == str(g[f"{prefix}tables_sha256"]), f"{prefix}: rebuilt tables differ from the reference's"
    return t


def fit_case(g: dict, i: int) -> dict:
    p = f"f{i}_"
    init = g[p + "init"]
    return dict(
        tables=tables(g, p),
        codes=g[p + "codes"],
        k=int(g[p + "k"]),
        seed=int(g[p + "seed"]),
        it=int(g[p + "it"]),
        update=str(g[p + "update"]),
        init=None if init.size == 0 else init,
    )


def fit_expect(g: dict, prefix: str) -> dict:
    return dict(
        labels=g[prefix + "labels"],
        centers=g[prefix + "centers"],
        objective=g[prefix + "objective"],
        objective_sq=g[prefix + "objective_sq"],
        repaired=g[prefix + "repaired"],
        nnz=g[prefix + "nnz"],
        iterations_run=int(g[prefix + "iterations_run"]),
        converged=bool(g[prefix + "converged"]),
    )


def same_nnz(a, b) -> bool:
    a = np.nan if a is None else a
    return (np.isnan(a) and np.isnan(b)) or a == b
