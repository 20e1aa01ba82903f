import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_03708_b200 import _lib, engine, synth
dev = engine.device_of()
n = 1_000_000
x = synth.sift_like(n, 5)
cw = synth.train_codebook_fast(synth.sift_like(20_000, 6), 4, 256, iterations=3, seed=1)
xd = torch.from_numpy(x).to(dev); cd = torch.from_numpy(cw).to(dev)
engine.encode_device(xd, cd, 4, 256, dev, stride=4)
torch.cuda.synchronize()
os.environ["PQK_ENC_DBG"] = "/tmp/tl.bin"
engine.encode_device(xd, cd, 4, 256, dev, stride=4)
torch.cuda.synchronize()
d = np.fromfile("/tmp/tl.bin", np.int64).reshape(64, 16)
t0 = d[0, 0]
names = ["T.beg", "T.xfull", "T.pre_aempty", "T.aempty_ok", "T.end", "M.beg", "M.afull_ok", "M.tempty0_ok", "M.tempty1_ok", "E.beg", "E.tfull0_ok", "E.pre_tfull1", "E.tfull1_ok", "E.end", "M.h0issued", "M.h1issued"]
print("item " + " ".join(f"{n:>12s}" for n in names))
for w in range(0, 24):
    print(f"{w:4d} " + " ".join(f"{(d[w, i] - t0) if d[w, i] else -1:12d}" for i in range(16)))
