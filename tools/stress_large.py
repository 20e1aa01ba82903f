"""Randomised parity sweep of the default assignment path at sizes where the fixed-point
first tiers run (>= 2^31 lookups): N up to 3e6 codes, K up to 1e5 centres, M in 1..16,
L in {16, 64, 256}, clustered / lattice (massive ties) / uniform codes, duplicated centres;
labels and paired distances against the oracle's C linear scan (all host threads).

usage: python tools/stress_large.py [seconds]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1709_03708_b200 as pqk  # noqa: E402
from helpers import lattice_tables, mixture_codes, random_tables  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(time.time()))
t0 = time.time()
cases = 0
while time.time() - t0 < budget:
    m = int(rng.choice([1, 2, 3, 4, 4, 4, 8, 16]))
    l_count = int(rng.choice([16, 64, 256, 256]))
    kind = str(rng.choice(["mixture", "lattice", "uniform"]))
    k = int(rng.choice([1000, 5000, 20000, 100000]))
    n = int(min(3_000_000, max(200_000, (2**31 + 2**30) // (k * m) + 1)))
    if kind == "lattice":
        tables = lattice_tables(m, l_count)
    else:
        tables = random_tables(m, l_count, seed=int(rng.integers(1 << 30)), sub_dim=int(rng.integers(1, 9)))
    if kind == "mixture":
        codes = mixture_codes(n, m, l_count, int(rng.integers(10, 5000)), seed=int(rng.integers(1 << 30)))
    else:
        codes = rng.integers(0, l_count, size=(n, m)).astype(np.uint8)
    centers = codes[rng.choice(n, size=k, replace=False)].copy()
    if rng.random() < 0.3:
        centers[rng.integers(0, k, size=k // 10)] = centers[0]
    t1 = time.time()
    labels = pqk.assign(codes, centers, tables)
    sd = pqk.paired_distance_sq(tables, codes, centers[labels])
    t_gpu = time.time() - t1
    ref, ref_sd = O.assign_c(codes, centers, tables, want_sd=True)
    cases += 1
    ok = np.array_equal(labels, ref) and np.array_equal(sd, ref_sd)
    print(f"case {cases}: m={m} l={l_count} {kind} n={n} k={k} gpu {t_gpu:.2f}s {'ok' if ok else 'MISMATCH'}",
          flush=True)
    if not ok:
        np.savez("gpurun_out/stress_large_fail.npz", codes=codes, centers=centers, tables=tables)
        sys.exit(1)
print(f"ok: {cases} large assignment cases in {time.time() - t0:.0f}s")
