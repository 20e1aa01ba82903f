"""Seeded input generators shared by the tests (mirroring the reference tests'
`random_tables` / `lattice_tables`, test_clustering.py:29-39)."""

import numpy as np

from oracle import pqk_oracle as O


def random_codebook(m, l_count, sub_dim=2, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((m, l_count, sub_dim)).astype(np.float32)


def random_tables(m, l_count, seed=0, sub_dim=2):
    return O.build_distance_tables(random_codebook(m, l_count, sub_dim, seed))


def lattice_tables(m, l_count):
    grid = np.arange(l_count, dtype=np.float32).reshape(l_count, 1)
    return O.build_distance_tables(np.broadcast_to(grid, (m, l_count, 1)).copy())


def mixture_codes(n, m, l_count, k_true, seed):
    """Clustered codes: each point copies a prototype code with a few byte edits."""
    rng = np.random.default_rng(seed)
    protos = rng.integers(0, l_count, size=(k_true, m))
    lab = rng.integers(0, k_true, size=n)
    codes = protos[lab].copy()
    flip = rng.random((n, m)) < 0.2
    codes[flip] = rng.integers(0, l_count, size=int(flip.sum()))
    return codes.astype(np.uint8)
