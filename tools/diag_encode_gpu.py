"""Dev diagnostic: tensor-core encoder on device-generated SIFT-like vectors with a bench
codebook (config 4's by default): time per call, HBM fraction, flagged pairs, and parity of
a row sample against the oracle.

usage: python tools/diag_encode_gpu.py [n (default 7.8e6)] [config (c4)]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402
from paper_1709_03708_b200 import _lib, engine  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 7_812_500
cfgn = sys.argv[2] if len(sys.argv) > 2 else "c4"
cfg = bench.CONFIGS[cfgn]
m = cfg["m"]
dev = engine.device_of()
book = bench.make_codebook(cfgn, m, 256)
x = bench.sift_like_gpu(n, 12345, dev)
cw = torch.from_numpy(np.array(book)).to(dev)
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
codes = engine.encode_device(x, cw, m, 256, dev, stride=m, stats=stats)
torch.cuda.synchronize()
print("flagged pairs", int(stats[_lib.STAT_ENCODE_FLAGGED].item()), "of", n * m)
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    engine.encode_device(x, cw, m, 256, dev, stride=m)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
gbs = n * (4 * x.shape[1] + m) / (ms / 1e3) / 1e9
print(f"encode {n} x {x.shape[1]} (M={m}): median {ms:.3f} ms, min {min(ts):.3f}  {gbs:.0f} GB/s "
      f"({gbs / 6454.6 * 100:.1f}% of measured HBM)")
rows = np.sort(np.random.default_rng(1).choice(n, size=20_000, replace=False))
xr = x[torch.from_numpy(rows).to(dev)].cpu().numpy()
mm = int((codes.cpu().numpy()[rows] != O.encode(book, xr)).sum())
print("mismatch on 20000 sampled rows:", mm)
sys.exit(1 if mm else 0)
