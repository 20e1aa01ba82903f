"""A/B of the assignment scan tiers on a bench workload: the default first tier (mode 0:
8-bit at padded M = 4, 16-bit otherwise), the 16-bit tier (mode 4) and the fp32 scan
(mode 1).  Labels and sd_sq must be bit-identical; prints
the per-assign time of each mode, the first-tier scan kernel time (profile events) and
the flagged counts.  Also runs a few Lloyd iterations per mode and compares centres.

usage: python tools/diag_scan16.py [c1|c2|c3s|c4s|c5s|c4] [reps] [mode_a (default 0)] [mode_b (default 4)]
  c3s/c4s/c5s: the config's codes at a reduced N (same K, M) so the run stays short."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1709_03708_b200 import _lib, engine, synth  # noqa: E402
from paper_1709_03708_b200.pq import PQCodebook, build_distance_tables  # noqa: E402

cfgn = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mode_a = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 2: force the first tier (small configs)
mode_b = int(sys.argv[4]) if len(sys.argv) > 4 else 4  # 4: 16-bit tier at M = 4
base = cfgn.rstrip("s")
cfg = dict(bench.CONFIGS[base])
n = {"c3s": 1_000_000, "c4s": 4_000_000, "c5s": 2_000_000}.get(cfgn, cfg["n"])
k, m, l_count = cfg["k"], cfg["m"], cfg["l"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
lib = _lib.load()
book = bench.make_codebook(base, m, l_count)
tables = build_distance_tables(PQCodebook(book)).tables
mp = _lib.padded_m(m)
cw = torch.from_numpy(np.array(book)).to(dev)
if cfg.get("gpu_data"):
    gen = {"mixture": bench.mixture_gpu, "sift": bench.sift_like_gpu, "deep": bench.deep_like_gpu}[cfg["gpu_data"]]
    codes = torch.empty((n, mp), dtype=torch.uint8, device=dev)
    step = (1 << 31) // (4 * cfg["dim"])
    for s in range(0, n, step):
        e = min(n, s + step)
        vec = gen(e - s, synth.stage_seed(bench.SEED, 1000 + s // step), dev)
        codes[s:e] = engine.encode_device(vec, cw, m, l_count, dev, stride=mp)
        del vec
else:
    vec = torch.from_numpy(bench.make_vectors(base, n, 0)).to(dev)
    codes = engine.encode_device(vec, cw, m, l_count, dev, stride=mp)
    del vec
torch.cuda.synchronize()
dt = engine.device_tables(tables, dev)
eng = engine.ShardEngine(codes, dt, k, dev)
rng = np.random.default_rng(bench.SEED)
codes_host = engine.download_codes(codes, m)
centers0 = codes_host[rng.choice(n, size=k, replace=False)].copy()

ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
ev1.record()
torch.cuda.synchronize()
lib.pqk_set_profile_events(ev0.cuda_event, ev1.cuda_event)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def run(mode, centers_host):
    _lib.check(lib.pqk_set_scan_mode(mode), "scan mode")
    cur = torch.zeros((k, mp), dtype=torch.uint8, device=dev)
    cur[:, :m] = torch.from_numpy(centers_host).to(dev)
    eng.assign(cur)
    torch.cuda.synchronize()
    tot, scan = [], []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.assign(cur)
        b.record()
        torch.cuda.synchronize()
        tot.append(a.elapsed_time(b))
        scan.append(ev0.elapsed_time(ev1))
    st = eng.stats.cpu().numpy()
    return (eng.labels[:n].clone(), eng.sd[:n].clone(), float(np.median(tot)), float(np.median(scan)),
            int(st[_lib.STAT_FLAGGED]), int(st[_lib.STAT_FLAGGED_FP64]), int(st[_lib.STAT_LOOKUP_BYTES]),
            int(st[_lib.STAT_UNIQUE_CENTERS]))


ok = True
cur_centers = centers0
for it in range(3):
    r0 = run(mode_a, cur_centers)
    r2 = run(mode_b, cur_centers)
    r1 = run(1, cur_centers)
    same = bool(torch.equal(r0[0], r1[0]) and torch.equal(r0[1].view(torch.int64), r1[1].view(torch.int64)))
    same &= bool(torch.equal(r2[0], r1[0]) and torch.equal(r2[1].view(torch.int64), r1[1].view(torch.int64)))
    ok &= same
    u = r0[7]
    print(f"[{cfgn} it{it}] n={n} k={k} m={m} U={u}  mode{mode_a} assign {r0[2]:.3f} ms (first tier {r0[3]:.3f} ms, "
          f"{r0[6]} B lookups, {n * u * m * r0[6] / (r0[3] / 1e3) / 1e9:.0f} GB/s, flagged {r0[4]} -> fp64 {r0[5]})  "
          f"mode{mode_b} assign {r2[2]:.3f} ms (first tier {r2[3]:.3f} ms, {r2[6]} B, flagged {r2[4]} -> fp64 {r2[5]})  "
          f"mode1 assign {r1[2]:.3f} ms (scan32 {r1[3]:.3f} ms, flagged {r1[4]})  "
          f"speedup vs b {r2[2] / r0[2]:.2f}x  identical={same}", flush=True)
    # next centres: one Lloyd update from the mode-0 labels
    eng.objective()
    eng.histogram()
    eng.vote()
    eng.read_obj_stats()
    nc = eng.new_centers[:, :m].cpu().numpy()
    cur_centers = nc
lib.pqk_set_profile_events(None, None)
_lib.check(lib.pqk_set_scan_mode(0), "scan mode")
print("PARITY", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
