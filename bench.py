#!/usr/bin/env python
"""Benchmark of the B200-native PQk-means Lloyd iteration (BASELINE.json metric).

Metric: code-center distance evaluations per second (N*K per Lloyd iteration /
seconds per iteration), whole job over all ranks.  Workload at N=1:
BASELINE.json configs[1] ("SIFT-like": N=1e6 128-D vectors, M=4, L=256,
K=1e4), synthetic data of that shape (paper datasets absent).  One step = one
full Lloyd iteration resident on the GPU: assignment scan (+ exact fp64
certificate/rescan), objective sums, histogram, [NCCL allreduce], sparse vote,
empty-cluster repair.  L2 (126 MB) is flushed by writing 512 MB between timed
steps.  Weak scaling: every rank holds its own N codes (tree-aligned shards).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n_per_gpu, k, m, l, dim)
    "c2": dict(n=1_000_000, k=10_000, m=4, l=256, dim=128, workload="config2 SIFT-like N=1e6/GPU K=1e4 M=4 L=256"),
    "c1": dict(n=100_000, k=1_000, m=4, l=256, dim=128, workload="config1 mixture N=1e5 K=1e3 M=4 L=256"),
    # config 4's per-GPU shard at 8 GPUs: 1e9/8 SIFT-like codes, K=1e5 (chunked tables stream from HBM)
    # config 5's per-GPU shard at 8 GPUs: 1e8/8 mixture codes with M=16 (8-D subspaces), K=1e5
    "c5": dict(n=12_500_000, k=100_000, m=16, l=256, dim=128, gpu_data="mixture",
               workload="config5 shard mixture N=1.25e7/GPU K=1e5 M=16 L=256"),
    "c4": dict(n=125_000_000, k=100_000, m=4, l=256, dim=128, gpu_data="sift",
               workload="config4 shard SIFT-like N=1.25e8/GPU K=1e5 M=4 L=256"),
    # config 3 on one GPU: 1e7 deep-feature-like 4096-D vectors generated on the device in
    # chunks and encoded there (K-streamed tensor-core encoder, 512-D subspaces)
    "c3": dict(n=10_000_000, k=10_000, m=8, l=256, dim=4096, gpu_data="deep",
               workload="config3 deep-feature-like N=1e7 K=1e4 M=8 L=256 (D=4096, GPU-encoded)"),
}
SEED = 20260419


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workload (host, seeded)
def make_vectors(cfg_name: str, n: int, rank: int) -> np.ndarray:
    from paper_1709_03708_b200 import synth

    if cfg_name == "c1":
        return synth.mixture(n, 128, 1000, synth.stage_seed(SEED, 100 + rank))
    if cfg_name == "c5":
        return synth.mixture(n, 128, 100_000, synth.stage_seed(SEED, 100 + rank))
    if cfg_name == "c3":
        return synth.deep_like(n, synth.stage_seed(SEED, 100 + rank))
    return synth.sift_like(n, synth.stage_seed(SEED, 100 + rank))


def sift_like_gpu(n: int, seed: int, dev, dim: int = 128, blocks: int = 8):
    """Device-side SIFT-like generator (config 4 chunks), same recipe as synth.sift_like."""
    import torch

    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    alpha = torch.full((n, blocks, dim // blocks), 0.6, dtype=torch.float32, device=dev)
    g = torch._standard_gamma(alpha, generator=gen) * 30.0
    g = g * (512.0 / g.norm(dim=2, keepdim=True).clamp_min(1e-12))
    return g.round_().clamp_(0, 255).reshape(n, dim).contiguous()


def mixture_gpu(n: int, seed: int, dev, dim: int = 128, components: int = 100_000, sigma: float = 5.0):
    """Device-side config-5 mixture: means U[0,100]^dim (fixed seed), sigma 5, uniform components."""
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(SEED)
    means = torch.rand((components, dim), generator=g, device=dev) * 100.0
    g.manual_seed(seed)
    lab = torch.randint(0, components, (n,), generator=g, device=dev)
    return (means[lab] + sigma * torch.randn((n, dim), generator=g, device=dev)).contiguous()


def deep_like_gpu(n: int, seed: int, dev, dim: int = 4096, components: int = 10_000, sigma: float = 0.5):
    """Device-side config-3 vectors: ReLU(mixture of N(0,1) means, sigma 0.5), L2-normalised."""
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(SEED)
    means = torch.randn((components, dim), generator=g, device=dev)
    g.manual_seed(seed)
    lab = torch.randint(0, components, (n,), generator=g, device=dev)
    x = (means[lab] + sigma * torch.randn((n, dim), generator=g, device=dev)).clamp_min_(0.0)
    return (x / x.norm(dim=1, keepdim=True).clamp_min(1e-12)).contiguous()


def make_codebook(cfg_name: str, m: int, l_count: int) -> np.ndarray:
    from paper_1709_03708_b200 import synth

    if cfg_name == "c3":  # bench set-up: 4 Lloyd iterations on a 20k sample of the same distribution
        sample = synth.deep_like(20_000, synth.stage_seed(SEED, 1))
        return synth.train_codebook_fast(sample, m, l_count, iterations=4, seed=synth.stage_seed(SEED, 2))
    if cfg_name == "c1":
        sample = synth.mixture(20_000, 128, 1000, synth.stage_seed(SEED, 1))
    elif cfg_name == "c5":
        sample = synth.mixture(100_000, 128, 100_000, synth.stage_seed(SEED, 1))
    else:
        sample = synth.sift_like(100_000, synth.stage_seed(SEED, 1))
    return synth.train_codebook_fast(sample, m, l_count, iterations=8, seed=synth.stage_seed(SEED, 2))


# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every 5 ms while
    the timed region runs (the region is tens of ms at config 2, too short for
    nvidia-smi's 200 ms loop); falls back to nvidia-smi -lms 50."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None

    def _sample(self):
        import pynvml

        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM)))
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for k, mask in self._masks.items():
            if r & mask:
                self.reasons.add(k)

    def _poll(self):
        while True:  # at least one sample even for a region shorter than the period
            self._sample()
            if self._stop.wait(0.005):
                break

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()  # before the region starts: init costs tens of ms
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._masks = {k: getattr(pynvml, v) for k, v in self.REASONS.items()}
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=2)
            import pynvml

            pynvml.nvmlShutdown()

    def summary(self) -> dict:
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 5 ms"}


# ---------------------------------------------------------------------------
def cpu_baseline_sample(codes: np.ndarray, centers: np.ndarray, tables: np.ndarray, n_total: int,
                        budget_s: float = 10.0) -> dict:
    """Reference algorithm on host cores (oracle C port, all threads): bounded sample.

    assignment: first n_s codes vs all K centers (C restatement of
    clustering.py:167-197, every host thread); update: the sparse vote of the
    sample's histograms (numpy restatement of clustering.py:327-356).  The
    iteration time is extrapolated to the full N (assignment is O(N*K*M)).
    """
    from oracle import pqk_oracle as O

    threads = os.cpu_count() or 1
    k = len(centers)
    n0 = min(len(codes), max(256, threads * 64))
    t0 = time.perf_counter()
    O.assign_c(codes[:n0], centers, tables, threads)
    rate = n0 * k / max(time.perf_counter() - t0, 1e-6)
    ns = int(min(len(codes), max(n0, rate * budget_s * 0.6 / k)))
    t0 = time.perf_counter()
    labels = O.assign_c(codes[:ns], centers, tables, threads)
    t_assign = time.perf_counter() - t0
    counts = np.bincount(labels.astype(np.intp), minlength=k)
    t0 = time.perf_counter()
    O.sparse_update_all(codes[:ns], labels, counts, tables)
    t_update = time.perf_counter() - t0
    t_iter = t_assign * (n_total / ns) + t_update
    return {"value": n_total * k / t_iter, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": f"assign {ns} of {n_total} codes x {k} centers ({t_assign:.2f}s, {threads} threads, C port of "
                      f"clustering.py:167-197) + sparse update of the sample ({t_update:.2f}s, numpy port of "
                      f"clustering.py:327-356); iteration extrapolated linearly in N",
            "assign_evals_per_s": ns * k / t_assign, "s_per_iteration": t_iter}


def run_reference(args) -> None:
    """--impl reference: the reference algorithm (oracle port) on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import pqk_oracle as O

    cfgn = args.config
    cfg = CONFIGS[cfgn]
    book = make_codebook(cfgn, cfg["m"], cfg["l"])
    tables = O.build_distance_tables(book)
    ns = min(cfg["n"], max(60_000, cfg["k"] + 10_000))  # bounded host sample of the workload's vectors
    vectors = make_vectors(cfgn, ns, 0)
    rng = np.random.default_rng(SEED)
    cidx = rng.choice(ns, size=cfg["k"], replace=False)
    centers = O.encode(book, vectors[cidx])
    codes = np.concatenate([O.encode(book, vectors[s : s + 10_000]) for s in range(0, min(cfg["n"], 50_000), 10_000)])
    vals = []
    for _ in range(args.warmup):
        cpu_baseline_sample(codes, centers, tables, cfg["n"] * args.gpus, budget_s=2.0)
    for _ in range(args.steps):
        vals.append(cpu_baseline_sample(codes, centers, tables, cfg["n"] * args.gpus, budget_s=4.0))
    v = float(np.median([x["value"] for x in vals]))
    spi = float(np.median([x["s_per_iteration"] for x in vals]))
    out = {
        "metric": "code-center distance evals/s", "impl": "reference", "value": v, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": spi * 1e3,
        "s_per_iteration": spi, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": cfg["n"] * args.gpus, "k": cfg["k"], "m": cfg["m"],
                   "l": cfg["l"]},
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": vals[-1]["cores"], "kind": "port",
                         "sample": vals[-1]["sample"]},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="launch the iteration eagerly (no CUDA graphs)")
    ap.add_argument("--dist", action="store_true", help="sharded NCCL driver even with one rank")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1709_03708_b200 import _lib, engine, synth
    from paper_1709_03708_b200.distributed import DistributedLloyd, GpuShardBackend, shard_bounds
    from paper_1709_03708_b200.pq import build_distance_tables, PQCodebook

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PQK_BENCH_BACKEND=gloo: functional check of the N>1 code path on a box with fewer GPUs
    # than ranks (ranks share devices; the timing of such a run means nothing)
    backend_name = os.environ.get("PQK_BENCH_BACKEND", "nccl")
    if backend_name != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist
    if use_dist:
        # keep stdout for the single JSON line: NCCL's banner/log go to stderr
        if not os.environ.get("PQK_KEEP_NCCL_DEBUG"):
            os.environ["NCCL_DEBUG"] = "WARN"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        else:
            dist.init_process_group(backend_name, rank=rank, world_size=world)
    lib = _lib.load()

    cfgn = args.config
    cfg = CONFIGS[cfgn]
    n_loc, k, m, l_count = cfg["n"], cfg["k"], cfg["m"], cfg["l"]
    n_total = n_loc * world

    # ---- workload -----------------------------------------------------------------
    t0 = time.perf_counter()
    book = make_codebook(cfgn, m, l_count)
    tables = build_distance_tables(PQCodebook(book)).tables
    mp = _lib.padded_m(m)
    enc_ms = 0.0
    with torch.cuda.device(dev):
        stats_enc = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
        cw_dev = torch.from_numpy(np.array(book)).to(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # untimed warm-up call: module load, tensor-map entry point, per-device workspace
        warm = torch.zeros((4096, cfg["dim"]), dtype=torch.float32, device=dev)
        engine.encode_device(warm, cw_dev, m, l_count, dev, stride=mp)
        torch.cuda.synchronize(dev)
        del warm
        if cfg.get("gpu_data"):
            # billion-scale shard: vectors generated on device per seeded chunk, encoded in place
            codes_dev = torch.empty((n_loc, mp), dtype=torch.uint8, device=dev)
            enc_flagged_sum = 0
            chunk = (1 << 32) // (4 * cfg["dim"])  # 4 GiB of fp32 vectors per encode call
            gen = {"mixture": mixture_gpu, "sift": sift_like_gpu, "deep": deep_like_gpu}[cfg["gpu_data"]]
            for s in range(0, n_loc, chunk):
                e = min(n_loc, s + chunk)
                cseed = synth.stage_seed(SEED, 1000 + rank * 100_000 + s // chunk)
                vec = gen(e - s, cseed, dev)
                e0.record()
                codes_dev[s:e] = engine.encode_device(vec, cw_dev, m, l_count, dev, stride=mp, stats=stats_enc)
                e1.record()
                torch.cuda.synchronize(dev)
                enc_ms += e0.elapsed_time(e1)
                enc_flagged_sum += int(stats_enc[_lib.STAT_ENCODE_FLAGGED].item())  # per call
                del vec
        else:
            vectors = make_vectors(cfgn, n_loc, rank)
            vec_dev = torch.from_numpy(vectors).to(dev)
            codes_dev = engine.encode_device(vec_dev, cw_dev, m, l_count, dev, stride=mp, stats=stats_enc)
            torch.cuda.synchronize(dev)
            times = []
            for _ in range(3):  # timed repeats (the first call above sized the workspace)
                e0.record()
                engine.encode_device(vec_dev, cw_dev, m, l_count, dev, stride=mp)
                e1.record()
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1))
            enc_ms = min(times)
            del vec_dev
        codes_host = engine.download_codes(codes_dev, m)
        enc_flagged = enc_flagged_sum if cfg.get("gpu_data") else int(stats_enc[_lib.STAT_ENCODE_FLAGGED].item())
        del codes_dev
    log(f"[bench] rank {rank}: workload ready in {time.perf_counter() - t0:.1f}s")

    offset, length = shard_bounds(n_total, world, rank)
    assert length == n_loc, (length, n_loc)
    backend = GpuShardBackend(codes_host, offset, tables, k, device=local, graphs=not args.no_graphs)
    drv = DistributedLloyd(backend, n_total, k, m) if use_dist else None
    if use_dist:
        centers0 = drv.init_centers(SEED, codes_host)
    else:
        rng = np.random.default_rng(SEED)
        centers0 = codes_host[rng.choice(n_loc, size=k, replace=False)].copy()
    eng = backend.eng

    graphs = None
    graph_launches = [0]  # kernels launched by graph replays (pqk_launch_count sees captures only)

    def step_single(cur):
        # the iteration body of fit(): one host read (objective + stats) per iteration; the
        # device part replays from CUDA graphs after the first (eager) iteration, as fit() does
        nonlocal graphs
        if graphs is not None:
            graphs.main.replay()
            graph_launches[0] += graphs.main_launches
            _, st = eng.read_obj_stats()
            if st[_lib.STAT_EMPTY]:
                graphs.repair.replay()
                graph_launches[0] += graphs.repair_launches
            cur.copy_(eng.new_centers)
            return cur, st
        eng.assign(cur)
        eng.objective()
        eng.histogram()
        eng.vote()
        _, st = eng.read_obj_stats()
        if st[_lib.STAT_EMPTY]:
            eng.repair()
        nxt = eng.new_centers.clone()
        if not args.no_graphs:
            graphs = engine.IterationGraphs(eng, nxt)
        return nxt, st

    def step(cur):
        if not use_dist:
            return step_single(cur)
        st, nxt, _ = drv.iteration(cur, None)
        # the stats the driver's one host read already brought back (no second sync)
        last = getattr(backend, "last_stats", None)
        return nxt, (last if last is not None else eng.stats_host())

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ev_scan0 = torch.cuda.Event(enable_timing=True)
    ev_scan1 = torch.cuda.Event(enable_timing=True)
    ev_scan0.record()
    ev_scan1.record()
    torch.cuda.synchronize(dev)
    lib.pqk_set_profile_events(ev_scan0.cuda_event, ev_scan1.cuda_event)

    with torch.cuda.device(dev):
        cur = backend.upload_centers(centers0)
        for _ in range(args.warmup):
            cur, _ = step(cur)
        torch.cuda.synchronize(dev)
        step_ms, scan_ms, uniq, flagged, vote_fp64, vote_dd = [], [], [], [], [], []
        flagged64, lookup_b = [], []
        launches0 = lib.pqk_launch_count()
        graph_launches[0] = 0
        with ClockSampler(local) as clocks:
            for _ in range(args.steps):
                flush.fill_(1)
                if use_dist:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                cur, st = step(cur)
                e1.record()
                torch.cuda.synchronize(dev)
                step_ms.append(e0.elapsed_time(e1))
                scan_ms.append(ev_scan0.elapsed_time(ev_scan1))
                uniq.append(int(st[_lib.STAT_UNIQUE_CENTERS]))
                flagged.append(int(st[_lib.STAT_FLAGGED]))
                flagged64.append(int(st[_lib.STAT_FLAGGED_FP64]))
                lookup_b.append(int(st[_lib.STAT_LOOKUP_BYTES]))
                vote_fp64.append(int(st[_lib.STAT_VOTE_FP64]))
                vote_dd.append(int(st[_lib.STAT_VOTE_EXACT]))
        launches = lib.pqk_launch_count() - launches0 + graph_launches[0]
    lib.pqk_set_profile_events(None, None)

    total_ms = float(np.sum(step_ms))
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n_total * k / (ms_per_step / 1e3)

    # roofline of the dominant kernel (assignment scan): shared-memory lookups
    u = int(np.median(uniq))
    lb = int(np.median(lookup_b)) or 4  # 2: 16-bit first tier (uint16 tables), 4: fp32 scan
    lookup_bytes = n_loc * u * m * lb  # algorithmic: one table lookup per (code, center, subspace)
    scan_name = "hscan_kernel (16-bit fixed-point tables)" if lb == 2 else "scan_kernel (fp32 tables)"
    scan_s = float(np.mean(scan_ms)) / 1e3
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = clocks.summary()
    peak_clock = 1965.0
    peak = sm_count * 128 * peak_clock * 1e6 / 1e9  # GB/s: 128 B/clk/SM shared-memory bandwidth
    achieved = lookup_bytes / scan_s / 1e9
    traffic = None
    prof = ROOT / "profiles" / "scan_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(cfgn)  # DRAM bytes per scan launch (ncu)
        except Exception:
            traffic = None

    out = {
        "metric": "code-center distance evals/s",
        "value": value,
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "s_per_iteration": ms_per_step / 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32+f64",
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n_total, "k": k, "m": m, "l": l_count,
                   "unique_centers": u, "flagged_codes_per_iter": int(np.median(flagged)),
                   "fp64_rescan_codes_per_iter": int(np.median(flagged64)),
                   "votes_fp64_per_iter": int(np.median(vote_fp64)), "votes_dd_per_iter": int(np.median(vote_dd)),
                   "l2": "flushed (512 MB write) between timed iterations",
                   "step": "assign+certify+objective+histogram+allreduce+vote+repair",
                   "launch": ("eager" if args.no_graphs else
                              "cuda graphs per phase (assign+objective+histogram, vote), collectives between"
                              if use_dist else "cuda graphs (after first warm-up step)"),
                   "parallelism": f"codes sharded dp{world}"},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "note": f"{scan_name}: {n_loc}x{u}x{m} {lb}-byte lookups per launch / {scan_s * 1e3:.3f} ms; peak = "
                             f"{sm_count} SMs x 128 B/clk x {peak_clock:.0f} MHz (architectural, not in "
                             "MEASURED_PEAKS.json)",
                     "scan_ms": scan_s * 1e3, "scan_share_of_step": scan_s * 1e3 / ms_per_step},
        "clocks": clk,
        "gpu_launches": int(launches),
    }
    # GPU codebook training with the reference recipe (pq.train_codebook: 20 Lloyd
    # iterations per subspace, bit-identical codewords) on a 100,000-vector sample
    if rank == 0 and cfgn in ("c2", "c4") and not args.no_cpu_baseline:
        from paper_1709_03708_b200 import pq as gpq

        tsample = synth.sift_like(100_000, synth.stage_seed(SEED, 1))
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        gpq.train_codebook(tsample, m, l_count, iterations=20, seed=synth.stage_seed(SEED, 2), device=local)
        out_train = {"vectors": 100_000, "dim": 128, "m": m, "l": l_count, "iterations": 20,
                     "seconds": time.perf_counter() - t0, "exact": "bit-identical to pq.train_codebook"}
    else:
        out_train = None
    # PQ encoder (set-up of the workload, timed with events): HBM roofline of code streaming
    enc_bytes = n_loc * (4 * cfg["dim"] + m)
    hbm_peak = 6545.3
    try:
        hbm_peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    # code streaming (north_star: HBM roofline fraction): the histogram pass reads every code
    # row (MP bytes) and label (4 B) and the objective pass every sd (8 B); timed with events
    # on the resident engine after the bench steps (its labels/sd are the last iteration's)
    with torch.cuda.device(dev):
        cs_h, cs_o = [], []
        for _ in range(5):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            e0.record()
            eng.histogram()
            e1.record()
            eng.objective()
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record()
            torch.cuda.synchronize(dev)
            cs_h.append(e0.elapsed_time(e1))
            cs_o.append(e1.elapsed_time(e2))
    h_ms, o_ms = float(np.median(cs_h)), float(np.median(cs_o))
    h_bytes, o_bytes = n_loc * (mp + 4), n_loc * 8
    out["code_streaming"] = {
        "histogram_ms": h_ms, "histogram_gbs": h_bytes / (h_ms / 1e3) / 1e9,
        "histogram_hbm_frac": h_bytes / (h_ms / 1e3) / 1e9 / hbm_peak,
        "objective_ms": o_ms, "objective_gbs": o_bytes / (o_ms / 1e3) / 1e9,
        "objective_hbm_frac": o_bytes / (o_ms / 1e3) / 1e9 / hbm_peak,
        "note": "histogram: codes (MP B) + labels (4 B) per code, atomics into K x M x 256 int32 (L2); objective: "
                "8 B sd per code through numpy's pairwise tree; L2 flushed before each; small at config 2 "
                "(launch- and atomic-latency bound), scales with N (configs 4/5)"}
    out["encode"] = {"vectors": n_loc, "ms": enc_ms, "vectors_per_s": n_loc / (enc_ms / 1e3),
                     "hbm_gbs": enc_bytes / (enc_ms / 1e3) / 1e9,
                     "hbm_frac": enc_bytes / (enc_ms / 1e3) / 1e9 / hbm_peak,
                     "flagged_pairs": enc_flagged,
                     "kernel": ("encode_tc_kernel (tcgen05 fp16 hi/lo split, certified argmin, fp64 fallback)"
                                if (cfg["dim"] // m) in (8, 16, 32, 64) else
                                "encode_tck_kernel (K-streamed tcgen05, certified argmin, fp64 fallback)"
                                if (cfg["dim"] // m) % 32 == 0 and 96 <= cfg["dim"] // m <= 1024 else
                                "encode_kernel (SIMT fp32 filter + fp64 certificate)")}
    if out_train:
        out["codebook_training"] = out_train

    # original-space error of the final labels (baselines.original_space_error, SURVEY
    # §8f row 3): means in index order + pairwise row sums + np.mean tree, on device
    if rank == 0 and not cfg.get("gpu_data") and not args.no_cpu_baseline:
        with torch.cuda.device(dev):
            x_dev = torch.from_numpy(vectors).to(dev)
            lab_dev = eng.labels.to(torch.int32)
            plan = engine.pairwise_plan(n_loc, dev)
            out2 = torch.zeros(2, dtype=torch.float64, device=dev)
            times = []
            for _ in range(3):
                torch.cuda.synchronize(dev)
                e0.record()
                means = engine.cluster_means_device(x_dev, lab_dev, k, dev)
                sq = engine.assigned_sq_device(x_dev, means, lab_dev, dev)
                engine.objective_sums(sq, plan, out2, dev)
                e1.record()
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1))
            ose_ms = min(times)
            ose_bytes = 2 * n_loc * cfg["dim"] * 4 + n_loc * (3 * 4 + 16)
            out["original_space_error"] = {
                "value": engine.mean_from_sum(float(out2[0].item()), n_loc), "ms": ose_ms, "n": n_loc, "k": k,
                "dim": cfg["dim"], "hbm_gbs": ose_bytes / (ose_ms / 1e3) / 1e9,
                "hbm_frac": ose_bytes / (ose_ms / 1e3) / 1e9 / hbm_peak,
                "exact": "bit-identical to baselines.original_space_error (float64, numpy order)"}
            del means, sq
            # Bk-means baseline on the same vectors: 32-bit sign codes
            # (the memory of PQ with M=4), K clusters, iterations of Hamming assignment +
            # majority update + repair, timed like the PQ step (events, warm-up first)
            from paper_1709_03708_b200 import baselines as gbl

            bz = gbl.train_binarizer(cfg["dim"], 32, seed=synth.stage_seed(SEED, 3))
            rot = torch.from_numpy(np.array(bz.rotation)).to(dev)
            bcodes = torch.zeros((n_loc, 4), dtype=torch.uint8, device=dev)
            bstats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
            bt = []
            for _ in range(3):
                torch.cuda.synchronize(dev)
                e0.record()
                engine.call("pqk_binarize_device", engine._ptr(x_dev), n_loc, cfg["dim"], engine._ptr(rot), 32,
                            engine._ptr(bcodes), 4, engine._ptr(bstats), engine._stream(dev))
                e1.record()
                torch.cuda.synchronize(dev)
                bt.append(e0.elapsed_time(e1))
            packed = bcodes.cpu().numpy()
            sh = gbl._BinaryShard(packed, k, dev)
            bcur = sh.upload_centers(packed[np.random.default_rng(SEED).choice(n_loc, size=k, replace=False)])
            for _ in range(2):
                sh.assign(bcur)
                sh.update()
                bcur = sh.new_centers.clone()
            it_ms, scan_ms_b = [], []
            e2 = torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                torch.cuda.synchronize(dev)
                e0.record()
                sh.assign(bcur)
                e2.record()
                sh.obj.cpu()
                sh.update()
                bcur = sh.new_centers.clone()
                e1.record()
                torch.cuda.synchronize(dev)
                it_ms.append(e0.elapsed_time(e1))
                scan_ms_b.append(e0.elapsed_time(e2))
            out["bkmeans"] = {"bits": 32, "n": n_loc, "k": k, "binarize_ms": min(bt),
                              "binarize_exact_bits": int(bstats[_lib.STAT_ENCODE_FLAGGED].item()),
                              "ms_per_iteration": float(np.median(it_ms)),
                              "assign_ms": float(np.median(scan_ms_b)),
                              "evals_per_s": n_loc * k / (float(np.median(it_ms)) / 1e3),
                              "exact": "bit-identical to baselines.bkmeans_fit (golden tests)"}
            del x_dev, sh
            # streaming pipeline: fvecs file -> GPU encoder -> PQKC file, and
            # PQKC file -> device codes; wall time, files in the page cache
            import tempfile

            from paper_1709_03708_b200 import io as pio

            with tempfile.TemporaryDirectory() as td:
                fv, pk = Path(td) / "x.fvecs", Path(td) / "x.pqkc"
                pio.write_fvecs(fv, vectors)
                book_obj = PQCodebook(np.asarray(book, dtype=np.float32))
                pio.encode_fvecs(book_obj, fv, pk)  # warm (allocations, page cache)
                t0s = time.perf_counter()
                pio.encode_fvecs(book_obj, fv, pk)
                enc_s = time.perf_counter() - t0s
                pio.load_codes(pk)
                t0s = time.perf_counter()
                codes_dev_f, _, _, _ = pio.load_codes(pk)
                torch.cuda.synchronize(dev)
                load_s = time.perf_counter() - t0s
                ok = bool(np.array_equal(engine.download_codes(codes_dev_f, m), codes_host))
                out["stream"] = {"vectors": n_loc, "fvecs_bytes": fv.stat().st_size,
                                 "encode_file_s": enc_s, "encode_file_gbs": fv.stat().st_size / enc_s / 1e9,
                                 "load_codes_s": load_s, "codes_bytes": pk.stat().st_size,
                                 "codes_equal_in_memory_encode": ok,
                                 "note": "wall time, files in the page cache; fvecs -> pinned -> GPU unpack+encode "
                                         "-> PQKC, PQKC -> pinned -> GPU unpack/validate"}
                del codes_dev_f

    # ---- e2e through the C-ABI host entry (host buffers, H2D/D2H inside) ------------
    if not args.no_e2e and not use_dist:
        import ctypes as C

        pin_codes = torch.from_numpy(codes_host).pin_memory()
        pin_cent = torch.from_numpy(centers0).pin_memory()
        pin_tab = torch.from_numpy(np.array(tables)).pin_memory()
        pin_lab = torch.empty(n_loc, dtype=torch.int32).pin_memory()
        pin_new = torch.empty((k, m), dtype=torch.uint8).pin_memory()
        obj2 = np.zeros(2)
        stats = np.zeros(_lib.STATS_LEN, np.int64)
        p = lambda t: C.c_void_p(t.data_ptr())
        pa = lambda a: a.ctypes.data_as(C.c_void_p)

        def host_step():
            _lib.check(lib.pqk_lloyd_step_host(p(pin_codes), n_loc, m, p(pin_cent), k, p(pin_tab), l_count,
                                               p(pin_lab), p(pin_new), pa(obj2), pa(stats), local))
            pin_cent.copy_(pin_new)

        for _ in range(args.warmup):
            host_step()
        times = []
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            host_step()
            times.append(time.perf_counter() - t0)
        e2e_s = float(np.mean(times))
        h2d = codes_host.nbytes + centers0.nbytes + tables.nbytes
        d2h = n_loc * 4 + k * m + 16 + _lib.STATS_LEN * 8
        out["e2e"] = {"value": n_total * k / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
                      "ms_steps": [round(t * 1e3, 3) for t in times],
                      "api": "pqk_lloyd_step_host (C-ABI, pinned host buffers)"}
        lib.pqk_host_release(local)
    elif not args.no_e2e:
        # multi-GPU: host buffers through the sharded driver (H2D shard + centers, D2H labels + centers)
        times = []
        pin_codes = torch.from_numpy(codes_host).pin_memory()
        for it in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            eng.codes[:, :m].copy_(pin_codes.to(dev, non_blocking=True))
            c = backend.upload_centers(centers0)
            st, nxt, _ = drv.iteration(c, None)
            lab = eng.labels_host()
            _ = backend.centers_host(nxt)
            torch.cuda.synchronize(dev)
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                times.append(dt)
        t = torch.tensor([float(np.mean(times))], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        out["e2e"] = {"value": n_total * k / e2e_s, "unit": "evals/s",
                      "h2d_bytes_per_step": int(codes_host.nbytes + centers0.nbytes),
                      "d2h_bytes_per_step": int(n_loc * 4 + k * m), "ms_per_step": e2e_s * 1e3,
                      "api": "distributed.DistributedLloyd.iteration with host buffers"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(codes_host, centers0, tables, n_total)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
