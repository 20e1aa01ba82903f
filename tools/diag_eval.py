"""Dev diagnostic: time the original-space evaluation pieces at config 2's size."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import engine, synth  # noqa: E402

dev = engine.device_of()
n, d, k = 1_000_000, 128, 10_000
x = torch.from_numpy(synth.sift_like(n, 3)).to(dev)
lab = torch.from_numpy(np.random.default_rng(1).integers(0, k, size=n).astype(np.int32)).to(dev)
plan = engine.pairwise_plan(n, dev)
out2 = torch.zeros(2, dtype=torch.float64, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for rep in range(3):
    torch.cuda.synchronize()
    ev[0].record()
    means = engine.cluster_means_device(x, lab, k, dev)
    ev[1].record()
    sq = engine.assigned_sq_device(x, means, lab, dev)
    ev[2].record()
    engine.objective_sums(sq, plan, out2, dev)
    ev[3].record()
    torch.cuda.synchronize()
    print(f"means {ev[0].elapsed_time(ev[1]):.3f} ms  sq {ev[1].elapsed_time(ev[2]):.3f} ms  "
          f"objective {ev[2].elapsed_time(ev[3]):.3f} ms")
