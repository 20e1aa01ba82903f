"""Dev check: per-iteration wall time of the Lloyd iteration eager vs CUDA-graph replay
(c1 and c2 shapes), plus equality of the results."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine, synth  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

for n, k in ((100_000, 1000), (1_000_000, 10_000)):
    rng = np.random.default_rng(0)
    tables = O.build_distance_tables(rng.normal(size=(4, 256, 32)).astype(np.float32))
    codes = rng.integers(0, 256, size=(n, 4)).astype(np.uint8)
    c0 = codes[rng.choice(n, k, replace=False)]
    dev = engine.device_of()
    dt = engine.device_tables(tables, dev)
    res = {}
    for mode in ("eager", "graph"):
        eng = engine.ShardEngine(engine.upload_codes(codes, 4, dev), dt, k, dev)
        cur = engine.upload_codes(c0, 4, dev)
        g = None
        times, objs = [], []
        for it in range(12):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if g is None:
                eng.assign(cur)
                eng.objective()
                eng.histogram()
                eng.vote()
            else:
                g.main.replay()
            sums, st = eng.read_obj_stats()
            if st[_lib.STAT_EMPTY]:
                if g is None:
                    eng.repair()
                else:
                    g.repair.replay()
            cur.copy_(eng.new_centers)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            objs.append(sums[1])
            if mode == "graph" and g is None:
                g = engine.IterationGraphs(eng, cur)
        res[mode] = (objs, cur.cpu().numpy(), eng.labels.cpu().numpy())
        print(f"n={n} k={k} {mode}: median iteration {np.median(times[2:]) * 1e3:.3f} ms "
              f"(launches main={getattr(g, 'main_launches', '-')}, repair={getattr(g, 'repair_launches', '-')})",
              flush=True)
    assert res["eager"][0] == res["graph"][0]
    assert np.array_equal(res["eager"][1], res["graph"][1])
    assert np.array_equal(res["eager"][2], res["graph"][2])
print("ok")
