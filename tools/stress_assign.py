"""Randomised parity sweep of the GPU assignment (labels and paired distances) and a
short fit against the oracle: lattice (integer) tables with massive ties, duplicated
centers, tiny/huge table scales, all code widths.

usage: python tools/stress_assign.py [seconds] [scan_mode]
  scan_mode: 0 default tiers, 1 fp32 first, 2 16-bit first tier at any size, 3 as 2 with
  the fp32 list tier for any list length (pqk_set_scan_mode)"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1709_03708_b200 as pqk  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
from paper_1709_03708_b200 import _lib  # noqa: E402

_lib.check(_lib.load().pqk_set_scan_mode(mode), "scan mode")
rng = np.random.default_rng(int(time.time()) + 1)
t0 = time.time()
cases = 0
while time.time() - t0 < budget:
    m = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 32]))
    l_count = int(rng.choice([2, 7, 64, 256]))
    kind = rng.choice(["random", "lattice", "scaled"])
    sub = int(rng.integers(1, 5))
    book = rng.normal(size=(m, l_count, sub))
    if kind == "lattice":
        book = np.rint(book * 2)
    if kind == "scaled":
        book *= 10.0 ** rng.uniform(-40, 40)
    tables = O.build_distance_tables(book.astype(np.float32))
    if not np.all(np.isfinite(tables)):
        continue
    n = int(rng.integers(1, 20000))
    k = int(rng.integers(1, min(n, 3000) + 1))
    codes = rng.integers(0, l_count, size=(n, m)).astype(np.uint8)
    centers = codes[rng.integers(0, n, size=k)].copy()
    if rng.random() < 0.3:
        centers[rng.integers(0, k, size=k // 3)] = centers[0]
    labels = pqk.assign(codes, centers, tables)
    ref_labels, ref_sd = O.assign_c(codes, centers, tables, want_sd=True)
    sd = pqk.paired_distance_sq(tables, codes, centers[labels])
    cases += 1
    if not (np.array_equal(labels, ref_labels) and np.array_equal(sd, ref_sd)):
        print("MISMATCH", dict(m=m, l=l_count, kind=kind, n=n, k=k), flush=True)
        np.savez("gpurun_out/stress_assign_fail.npz", codes=codes, centers=centers, tables=tables)
        sys.exit(1)
    if cases % 10 == 0 and n >= k >= 2:
        res = pqk.fit(codes, tables, min(k, 200), max_iterations=3, seed=cases)
        ref = O.fit(codes, tables, min(k, 200), max_iterations=3, seed=cases, scan=O.assign_c)
        if not (np.array_equal(res.labels, ref["labels"]) and np.array_equal(res.centers, ref["centers"])):
            print("FIT MISMATCH", dict(m=m, l=l_count, kind=kind, n=n, k=k), flush=True)
            sys.exit(1)
print(f"ok: {cases} assignment cases in {time.time() - t0:.0f}s (scan mode {mode})")
