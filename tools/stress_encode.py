"""Randomised parity sweep of the GPU encoder (all tensor-core and SIMT paths) against the
oracle: distributions chosen to stress the certificate (near-ties from duplicated and
perturbed codewords, integer data, heavy tails, sparse rows, tiny and huge scales).

usage: python tools/stress_encode.py [seconds]   (PQK_STRESS_TCK=1: only subspace widths
of the K-streamed tensor-core kernel, up to 12,000 rows)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1709_03708_b200 as pqk  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(time.time()))
t0 = time.time()
cases = pairs = 0
while time.time() - t0 < budget:
    tck_only = os.environ.get("PQK_STRESS_TCK") == "1"
    sub = int(rng.choice([96, 128, 160, 224, 256, 512, 1024] if tck_only else [8, 16, 32, 64, 96, 128, 256, 512, 24]))
    m = int(rng.choice([1, 2, 4, 8]))
    l_count = int(rng.choice([2, 17, 100, 256, 256, 256]))
    # (the oracle's float64 pass bounds the case size: ~1e7 vector elements take ~20 s)
    n = int(rng.integers(1, max(300, min(12000, 10_000_000 // (sub * m))) if tck_only
                         else (6000 if sub * m <= 512 else 1500)))
    scale = float(10.0 ** rng.uniform(-6, 6))
    kind = rng.choice(["normal", "int", "heavy", "sparse", "near_tie"])
    d = sub * m
    if kind == "int":
        x = np.rint(rng.normal(size=(n, d)) * 20)
    elif kind == "heavy":
        x = rng.standard_t(2, size=(n, d))
    elif kind == "sparse":
        x = rng.normal(size=(n, d)) * (rng.random((n, d)) < 0.2)
    else:
        x = rng.normal(size=(n, d))
    x = (x * scale).astype(np.float32)
    cw = x[rng.integers(0, n, size=l_count)].reshape(l_count, m, sub).transpose(1, 0, 2).copy()
    if kind == "near_tie":  # codewords nearly equidistant from many vectors
        cw[:, 1::2] = cw[:, 0::2][:, : cw[:, 1::2].shape[1]] * np.float32(1 + 1e-6)
    cw += (rng.normal(size=cw.shape) * scale * 1e-3).astype(np.float32)
    if tck_only:
        print(dict(sub=sub, m=m, l=l_count, n=n, kind=str(kind)), flush=True)
    got = pqk.encode(pqk.PQCodebook(cw), x)
    ref = O.encode(cw, x)
    cases += 1
    pairs += n * m
    if not np.array_equal(got, ref):
        bad = np.argwhere(got != ref)
        print("MISMATCH", dict(sub=sub, m=m, l=l_count, n=n, scale=scale, kind=kind), bad[:5], flush=True)
        np.savez("gpurun_out/stress_fail.npz", x=x, cw=cw, got=got, ref=ref)
        sys.exit(1)
print(f"ok: {cases} cases, {pairs} (vector, subspace) pairs in {time.time() - t0:.0f}s")
