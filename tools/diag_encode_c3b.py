"""Dev diagnostic: config-3 encode as bench.py runs it (trained codebook, device vectors)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1709_03708_b200 import _lib, engine, synth  # noqa: E402

dev = engine.device_of()
t0 = time.perf_counter()
book = bench.make_codebook("c3", 8, 256)
print(f"codebook {time.perf_counter() - t0:.1f}s")
cw = torch.from_numpy(book).to(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
vec = bench.deep_like_gpu(n, 123, dev)
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine.encode_device(vec, cw, 8, 256, dev, stride=8, stats=stats)
    torch.cuda.synchronize()
    print(f"encode {n}: {(time.perf_counter() - t0) * 1e3:.2f} ms flagged {int(stats[_lib.STAT_ENCODE_FLAGGED].item())}")
