"""Dev diagnostic: tensor-core encoder flag rate and parity on SIFT-like data."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine, synth
from oracle import pqk_oracle as O

dev = engine.device_of()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
x = synth.sift_like(n, 5)
sample = synth.sift_like(20_000, 6)
cw = synth.train_codebook_fast(sample, 4, 256, iterations=4, seed=1)
stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
xd = torch.from_numpy(x).to(dev); cd = torch.from_numpy(cw).to(dev)
codes = engine.encode_device(xd, cd, 4, 256, dev, stride=4, stats=stats).cpu().numpy()
print("flagged", int(stats[_lib.STAT_ENCODE_FLAGGED].item()), "of", n * 4)
ref = O.encode(cw, x[:20000])
print("mismatch on first 20000:", int((codes[:20000] != ref).sum()))
