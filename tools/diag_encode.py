"""Dev diagnostic: tensor-core encoder time, flag rate and parity on SIFT-like data.

usage: python tools/diag_encode.py [n] [m]   (n vectors of 128-D, m subspaces)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine, synth  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

dev = engine.device_of()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4
x = synth.sift_like(n, 5)
sample = synth.sift_like(20_000, 6)
cw = synth.train_codebook_fast(sample, m, 256, iterations=4, seed=1)
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
xd = torch.from_numpy(x).to(dev)
cd = torch.from_numpy(cw).to(dev)
codes = engine.encode_device(xd, cd, m, 256, dev, stride=m, stats=stats).cpu().numpy()
print("flagged", int(stats[_lib.STAT_ENCODE_FLAGGED].item()), "of", n * m)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    engine.encode_device(xd, cd, m, 256, dev, stride=m)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
gbs = n * (4 * 128 + m) / (ms / 1e3) / 1e9
print(f"encode {n} x 128 (M={m}): {ms:.3f} ms  {n / ms / 1e3:.1f} M vec/s  {gbs:.0f} GB/s ({gbs / 6545.3 * 100:.1f}% HBM)")
k = min(n, 20_000)
ref = O.encode(cw, x[:k])
print(f"mismatch on first {k}:", int((codes[:k] != ref).sum()))
