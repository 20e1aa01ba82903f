import sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from helpers import random_codebook
from oracle import pqk_oracle as O
from paper_1709_03708_b200 import _lib, engine
rng = np.random.default_rng(11)
n = 200_000
cw = random_codebook(4, 256, 32, seed=12)
x = rng.normal(size=(n, 128)).astype(np.float32)
x[: n // 2] = np.rint(x[: n // 2] * 20)
dev = engine.device_of()
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
tc = engine.encode_device(torch.from_numpy(x).to(dev), torch.from_numpy(cw).to(dev), 4, 256, dev, stride=4, stats=stats).cpu().numpy()
print("flagged", int(stats[_lib.STAT_ENCODE_FLAGGED].item()))
ref = O.encode(cw, x)
bad = np.argwhere(tc != ref)
print("mismatches", len(bad))
if len(bad):
    tiles = bad[:, 0] // 128
    w = tiles // 37
    print("by item index w (tile // 37):", dict(zip(*np.unique(w, return_counts=True))))
    print("by subspace:", dict(zip(*np.unique(bad[:, 1], return_counts=True))))
    print("by t0 (tile % 37):", dict(zip(*np.unique(tiles % 37, return_counts=True))))
    print("rows in tile (first 40):", (bad[:40, 0] % 128).tolist())
for r, m in bad[:20]:
    xs = x[r, 32*m:32*m+32].astype(np.float64)
    d = ((cw[m].astype(np.float64) - xs) ** 2).sum(1)
    o = np.argsort(d)
    print(r, m, "got", tc[r, m], "ref", ref[r, m], "d_got", d[tc[r, m]], "best2", o[:3], d[o[:3]])
