"""Train the bench workloads' PQ codebooks with the reference's own pq.train_codebook.

BASELINE.json recipe per config (20 Lloyd iterations per subspace, seeded sample):
  c1  20,000-vector mixture sample (1,000 components), M=4
  c2  100,000-vector SIFT-like sample, M=4
  c3  100,000-vector deep-feature-like sample (4096-D), M=8
  c4  1,000,000-vector SIFT-like sample, M=4
  c5  1,000,000-vector mixture sample (100,000 components), M=16

Runs in the build container (imports the unmodified reference from baseline/_ref, the
pip install of /root/reference, or /root/reference/pkg/src) and writes
bench_assets/<cfg>_codebook.npy.  bench.py loads these for both arms (the reference arm
never touches the GPU kernels), and its b200 arm re-trains the same sample with the GPU
pq.train_codebook and reports whether the bytes agree.

    python tools/make_bench_codebooks.py c4 c2 ...
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists():
        sys.path.insert(0, str(p))
        break

import bench  # noqa: E402  (CODEBOOK_RECIPES, codebook_sample)


def main(names):
    import pqclust

    out_dir = ROOT / "bench_assets"
    out_dir.mkdir(exist_ok=True)
    for name in names:
        rec = bench.CODEBOOK_RECIPES[name]
        t0 = time.time()
        sample = bench.codebook_sample(name)
        t1 = time.time()
        book = pqclust.train_codebook(sample, rec["m"], 256, iterations=rec["iterations"], seed=rec["seed"])
        cw = np.asarray(book.codewords, dtype=np.float32)
        np.save(out_dir / f"{name}_codebook.npy", cw)
        print(f"{name}: sample {sample.shape} in {t1 - t0:.1f}s, reference train_codebook {time.time() - t1:.1f}s, "
              f"sha256 {hashlib.sha256(cw.tobytes()).hexdigest()[:16]}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c5", "c3"])
