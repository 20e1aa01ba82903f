"""Dev diagnostic: encoder at config 3's shape (D=4096, M=8, dsub=512): time and parity."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine, synth  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

dev = engine.device_of()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000
x = synth.deep_like(n, 5, components=1000)
rng = np.random.default_rng(1)
cw = x[rng.choice(n, 256, replace=False)].reshape(256, 8, 512).transpose(1, 0, 2).copy()
xd, cd = torch.from_numpy(x).to(dev), torch.from_numpy(cw).to(dev)
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
codes = engine.encode_device(xd, cd, 8, 256, dev, stride=8, stats=stats)
torch.cuda.synchronize()
t0 = time.perf_counter()
engine.encode_device(xd, cd, 8, 256, dev, stride=8)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"encode {n} x 4096 (M=8): {dt * 1e3:.2f} ms, {n / dt / 1e6:.3f} M vec/s, "
      f"{n * 4096 * 4 / dt / 1e9:.1f} GB/s; flagged {int(stats[_lib.STAT_ENCODE_FLAGGED].item())}")
k = min(n, 2000)
print("mismatch vs oracle on first", k, ":", int((codes.cpu().numpy()[:k] != O.encode(cw, x[:k])).sum()))
