"""Dev diagnostic: where the C-ABI host step's time goes (config 2 shapes): pinned H2D /
D2H bandwidth for the step's buffers, the device-only iteration, and pqk_lloyd_step_host."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine  # noqa: E402
from oracle import pqk_oracle as O  # noqa: E402

n, k, m = 1_000_000, 10_000, 4
rng = np.random.default_rng(0)
tables = O.build_distance_tables(rng.normal(size=(m, 256, 32)).astype(np.float32))
codes = rng.integers(0, 256, size=(n, m)).astype(np.uint8)
cent = codes[rng.choice(n, k, replace=False)].copy()
dev = torch.device("cuda", 0)
lib = _lib.load()


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


pc = torch.from_numpy(codes).pin_memory()
pt = torch.from_numpy(np.array(tables)).pin_memory()
dc = torch.empty_like(pc, device=dev)
dt = torch.empty_like(pt, device=dev)
print(f"H2D codes 4 MB: {timed(lambda: dc.copy_(pc, non_blocking=True)):.3f} ms")
print(f"H2D tables 2 MB: {timed(lambda: dt.copy_(pt, non_blocking=True)):.3f} ms")
lab = torch.empty(n, dtype=torch.int32).pin_memory()
dl = torch.empty(n, dtype=torch.int32, device=dev)
print(f"D2H labels 4 MB: {timed(lambda: lab.copy_(dl, non_blocking=True)):.3f} ms")
big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dbig = torch.empty_like(big, device=dev)
t = timed(lambda: dbig.copy_(big, non_blocking=True), 5)
print(f"H2D 256 MB: {t:.3f} ms = {256 * 1.048576 / t:.1f} GB/s")

pin_c = torch.from_numpy(cent).pin_memory()
pin_new = torch.empty((k, m), dtype=torch.uint8).pin_memory()
obj2 = np.zeros(2)
stats = np.zeros(_lib.STATS_LEN, np.int64)
p = lambda t: C.c_void_p(t.data_ptr())
pa = lambda a: a.ctypes.data_as(C.c_void_p)


def host_step():
    _lib.check(lib.pqk_lloyd_step_host(p(pc), n, m, p(pin_c), k, p(pt), 256, p(lab), p(pin_new), pa(obj2),
                                       pa(stats), 0))


host_step()
print(f"pqk_lloyd_step_host: {timed(host_step):.3f} ms")
# device-only iteration for comparison
eng = engine.ShardEngine(engine.upload_codes(codes, m, dev), engine.device_tables(tables, dev), k, dev)
cur = engine.upload_codes(cent, m, dev)


def dev_step():
    eng.assign(cur)
    eng.objective()
    eng.histogram()
    eng.vote()
    eng.read_obj_stats()


dev_step()
print(f"device iteration: {timed(dev_step):.3f} ms")

flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ts = []
for _ in range(10):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host_step()
    ts.append(time.perf_counter() - t0)
print(f"pqk_lloyd_step_host after L2 flush: {np.median(ts) * 1e3:.3f} ms (min {min(ts) * 1e3:.3f}, max {max(ts) * 1e3:.3f})")
ts = []
for _ in range(10):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_step()
    ts.append(time.perf_counter() - t0)
print(f"device iteration after L2 flush: {np.median(ts) * 1e3:.3f} ms")
