#!/usr/bin/env python
"""Benchmark of the B200-native PQk-means Lloyd iteration (BASELINE.json metric).

Metric: code-center distance evaluations per second (N*K per Lloyd iteration /
seconds per iteration), whole job over all ranks, plus seconds per iteration.
Default workload (north_star): BASELINE.json configs[3]'s per-GPU shard, i.e. the
billion-scale SIFT-like set split over 8 GPUs: N=1.25e8 codes per GPU, K=1e5,
M=4, L=256 (``--config c4``).  ``--config c1|c2|c3|c5`` select the other
configurations (c5 is config 5's per-GPU shard).  Synthetic data of the configs'
shapes and distributions (the paper's datasets are absent); codebooks trained by
the reference's own pq.train_codebook with BASELINE's recipe (bench_assets/).

One step = one full Lloyd iteration resident on the GPU: assignment scan
(+ exact fp64 certificate/rescan), objective sums, histogram, [NCCL allreduce],
sparse vote, empty-cluster repair.  L2 (126 MB) is flushed by writing 512 MB
between timed steps.  Weak scaling: every rank holds its own N codes
(tree-aligned shards of the job's index space).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c4]

``--gpus N`` without WORLD_SIZE in the environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL).  Rank 0 prints one JSON
line.  After the timed steps an untimed iteration is checked against the oracle
(``parity`` in the line: sampled labels/sd, the full histogram, sampled votes,
the repair and the objective, bit for bit).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # config 4's per-GPU shard at 8 GPUs: 1e9/8 SIFT-like codes, K=1e5 (north_star)
    "c4": dict(n=125_000_000, k=100_000, m=4, l=256, dim=128, gpu_data="sift",
               workload="config4 shard SIFT-like N=1.25e8/GPU K=1e5 M=4 L=256"),
    "c2": dict(n=1_000_000, k=10_000, m=4, l=256, dim=128, workload="config2 SIFT-like N=1e6/GPU K=1e4 M=4 L=256"),
    "c1": dict(n=100_000, k=1_000, m=4, l=256, dim=128, workload="config1 mixture N=1e5 K=1e3 M=4 L=256"),
    # config 5's per-GPU shard at 8 GPUs: 1e8/8 mixture codes with M=16 (8-D subspaces), K=1e5
    "c5": dict(n=12_500_000, k=100_000, m=16, l=256, dim=128, gpu_data="mixture",
               workload="config5 shard mixture N=1.25e7/GPU K=1e5 M=16 L=256"),
    # config 3 on one GPU: 1e7 deep-feature-like 4096-D vectors generated on the device in
    # chunks and encoded there (K-streamed tensor-core encoder, 512-D subspaces)
    "c3": dict(n=10_000_000, k=10_000, m=8, l=256, dim=4096, gpu_data="deep",
               workload="config3 deep-feature-like N=1e7 K=1e4 M=8 L=256 (D=4096, GPU-encoded)"),
}
DEFAULT_CONFIG = "c4"
SEED = 20260419
DTYPE = ("u8 fixed-point scan (M<=4; u16 for M 8/16) + f32 filters, f64 exact "
         "(results bit-identical to the float64 reference)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workload (seeded)
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


GPU_GENERATORS = {"mixture": mixture_gpu, "sift": sift_like_gpu, "deep": deep_like_gpu}


def gpu_chunks(cfg: dict, n_loc: int, rank: int):
    """(start, stop, seed) of the device-generated chunks of a rank's shard (4 GiB of fp32 each)."""
    from paper_1709_03708_b200 import synth

    chunk = (1 << 32) // (4 * cfg["dim"])
    return [(s, min(n_loc, s + chunk), synth.stage_seed(SEED, 1000 + rank * 100_000 + s // chunk))
            for s in range(0, n_loc, chunk)]


# BASELINE.json codebook recipe per config: pq.train_codebook (20 Lloyd iterations per
# subspace) on a seeded sample of the config's distribution.  The codebooks are trained
# once by the reference itself (tools/make_bench_codebooks.py -> bench_assets/) so both
# arms read the same bytes; the b200 arm re-trains the sample on the GPU and reports
# whether its codebook equals the reference's (pq.py:155-202).
CODEBOOK_RECIPES = {
    "c1": dict(sample=20_000, m=4, iterations=20),
    "c2": dict(sample=100_000, m=4, iterations=20),
    "c3": dict(sample=100_000, m=8, iterations=20),
    "c4": dict(sample=1_000_000, m=4, iterations=20),
    "c5": dict(sample=1_000_000, m=16, iterations=20),
}
for _r in CODEBOOK_RECIPES.values():
    _r["seed"] = int(np.random.SeedSequence([SEED, 2]).generate_state(1)[0])


def codebook_sample(cfg_name: str) -> np.ndarray:
    from paper_1709_03708_b200 import synth

    n = CODEBOOK_RECIPES[cfg_name]["sample"]
    s = synth.stage_seed(SEED, 1)
    if cfg_name == "c3":
        return synth.deep_like(n, s)
    if cfg_name == "c1":
        return synth.mixture(n, 128, 1000, s)
    if cfg_name == "c5":
        return synth.mixture(n, 128, 100_000, s)
    return synth.sift_like(n, s)


def make_codebook(cfg_name: str, m: int, l_count: int) -> np.ndarray:
    """The reference-trained codebook of the config (bench_assets/, see CODEBOOK_RECIPES)."""
    path = ROOT / "bench_assets" / f"{cfg_name}_codebook.npy"
    if not path.exists():
        raise FileNotFoundError(f"{path} missing: run tools/make_bench_codebooks.py {cfg_name} in the build container")
    book = np.load(path)
    assert book.shape[:2] == (m, l_count), book.shape
    return book


def center_indices(n_total: int, k: int) -> np.ndarray:
    """Initial centers: clustering.py:149-157 (Generator.choice over the job's code index)."""
    return np.random.default_rng(SEED).choice(n_total, size=k, replace=False)


def build_workload(cfg_name: str, dev, rank: int = 0, world: int = 1, n_loc: int | None = None) -> dict:
    """Codebook, tables and this rank's (N_loc, M) codes, encoded on the device exactly as
    the bench does (GPU-generated vectors for configs 3/4/5, host vectors otherwise).

    Returns dict(book, tables, codes_host, n_loc, enc_ms, enc_flagged, vectors | None)."""
    import torch

    from paper_1709_03708_b200 import _lib, engine
    from paper_1709_03708_b200.pq import PQCodebook, build_distance_tables

    cfg = CONFIGS[cfg_name]
    n_loc = cfg["n"] if n_loc is None else int(n_loc)
    m, l_count = cfg["m"], cfg["l"]
    book = make_codebook(cfg_name, m, l_count)
    tables = build_distance_tables(PQCodebook(book)).tables
    mp = _lib.padded_m(m)
    enc_ms = 0.0
    vectors = None
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
            enc_flagged = 0
            gen = GPU_GENERATORS[cfg["gpu_data"]]
            for ci, (s, e, cseed) in enumerate(gpu_chunks(cfg, n_loc, rank)):
                vec = gen(e - s, cseed, dev)
                if ci == 0:  # untimed: sizes the encoder workspace for a full chunk (cudaMalloc)
                    engine.encode_device(vec, cw_dev, m, l_count, dev, stride=mp)
                    torch.cuda.synchronize(dev)
                e0.record()
                codes_dev[s:e] = engine.encode_device(vec, cw_dev, m, l_count, dev, stride=mp, stats=stats_enc)
                e1.record()
                torch.cuda.synchronize(dev)
                enc_ms += e0.elapsed_time(e1)
                enc_flagged += int(stats_enc[_lib.STAT_ENCODE_FLAGGED].item())  # per call
                del vec
        else:
            vectors = make_vectors(cfg_name, n_loc, rank)
            vec_dev = torch.from_numpy(vectors).to(dev)
            codes_dev = engine.encode_device(vec_dev, cw_dev, m, l_count, dev, stride=mp, stats=stats_enc)
            torch.cuda.synchronize(dev)
            enc_flagged = int(stats_enc[_lib.STAT_ENCODE_FLAGGED].item())
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
        del codes_dev
    return dict(book=book, tables=tables, codes_host=codes_host, n_loc=n_loc, enc_ms=enc_ms,
                enc_flagged=enc_flagged, vectors=vectors)


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
# CPU leg: the reference algorithm on the host cores (oracle port), bounded sample
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_step(codes_s: np.ndarray, centers: np.ndarray, tables: np.ndarray, n_total: int, threads: int,
             vote_clusters: int = 2000) -> dict:
    """One bounded sample of the reference iteration on the host cores.

    assignment: the S sampled codes against all K centers (C restatement of
    clustering.py:167-197, all host threads); update: the sparse vote
    (clustering.py:327-356, numpy restatement) of the first `vote_clusters` filled
    clusters of the sample's histograms.  The iteration time is extrapolated
    linearly: assignment x N/S (O(N*K*M)), update x K/vote_clusters.
    """
    from oracle import pqk_oracle as O

    k = len(centers)
    s = len(codes_s)
    t0 = time.perf_counter()
    labels = O.assign_c(codes_s, centers, tables, threads)
    t_assign = time.perf_counter() - t0
    t0 = time.perf_counter()
    counts = np.bincount(labels.astype(np.intp), minlength=k)
    filled = np.flatnonzero(counts > 0)[:vote_clusters]
    l_count = tables.shape[1]
    joint = labels.astype(np.int64) * l_count
    for mm in range(tables.shape[0]):
        hist = np.bincount(joint + codes_s[:, mm], minlength=k * l_count).reshape(k, l_count)
        for ki in filled:
            O.vote_argmin(hist[ki], tables[mm])
    t_update = time.perf_counter() - t0
    kv = max(len(filled), 1)
    t_iter = t_assign * (n_total / s) + t_update * (k / kv)
    return {"value": n_total * k / t_iter, "t_assign": t_assign, "t_update": t_update, "rows": s,
            "vote_clusters": kv, "s_per_iteration": t_iter, "step_s": t_assign + t_update,
            "assign_evals_per_s": s * k / t_assign}


def cpu_sample_rows(k: int, threads: int, budget_s: float, rate_guess: float = 2.5e8) -> int:
    """Rows of a CPU step sized to ~budget_s of assignment (rate_guess evals/s per thread)."""
    return int(max(256, budget_s * rate_guess * threads / max(k, 1)))


def reference_inputs(cfg_name: str, world: int, k: int, rows_max: int) -> tuple[np.ndarray, np.ndarray, dict]:
    """The b200 arm's initial centers and a sample of rank 0's codes, rebuilt for the
    reference arm without the b200 kernels: the same seeded vectors (device-generated
    chunks through torch for configs 3/4/5, host numpy otherwise), encoded on the host
    by the reference's own pq.encode (pqclust from baseline/_ref when installed, else
    the oracle's restatement; both equal the GPU encoder bit for bit)."""
    from paper_1709_03708_b200.distributed import shard_bounds

    cfg = CONFIGS[cfg_name]
    m = cfg["m"]
    n_loc = cfg["n"]
    n_total = n_loc * world
    book = make_codebook(cfg_name, m, cfg["l"])
    cidx = center_indices(n_total, k)
    bounds = [shard_bounds(n_total, world, r) for r in range(world)]
    want = {}  # rank -> local row indices needed (centers; rank 0 also the sample)
    for r, (off, ln) in enumerate(bounds):
        sel = cidx[(cidx >= off) & (cidx < off + ln)] - off
        want[r] = sel
    sample_rows = np.arange(min(rows_max, n_loc))
    rows: dict[tuple[int, int], np.ndarray] = {}
    t0 = time.perf_counter()
    how = "host numpy"
    if cfg.get("gpu_data"):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("the reference arm rebuilds config 3/4/5 vectors with torch on cuda:0")
        dev = torch.device("cuda", 0)
        gen = GPU_GENERATORS[cfg["gpu_data"]]
        how = "torch device generator (same seeds as the b200 arm), rows copied to the host"
        for r in range(world):
            need = np.union1d(want[r], sample_rows) if r == 0 else want[r]
            for s, e, cseed in gpu_chunks(cfg, n_loc, r):
                sel = need[(need >= s) & (need < e)]
                if len(sel) == 0:
                    continue
                vec = gen(e - s, cseed, dev)
                got = vec[torch.from_numpy(sel - s).to(dev)].cpu().numpy()
                for i, row in zip(sel, got):
                    rows[(r, int(i))] = row
                del vec
            torch.cuda.synchronize(dev)
    else:
        for r in range(world):
            vec = make_vectors(cfg_name, n_loc, r)
            need = np.union1d(want[r], sample_rows) if r == 0 else want[r]
            for i in need:
                rows[(r, int(i))] = vec[i]
    t_gen = time.perf_counter() - t0
    keys = [(r, int(i - bounds[r][0])) for i in cidx for r in range(world)
            if bounds[r][0] <= i < bounds[r][0] + bounds[r][1]]
    xc = np.stack([rows[key] for key in keys]).astype(np.float32)
    xs = np.stack([rows[(0, int(i))] for i in sample_rows]).astype(np.float32)
    t0 = time.perf_counter()
    enc, enc_name = reference_encoder()
    both = enc(book, np.concatenate([xc, xs]))
    t_enc = time.perf_counter() - t0
    centers = both[: len(xc)].astype(np.uint8)
    codes_s = both[len(xc):].astype(np.uint8)
    info = {"vectors": how, "encoder": enc_name, "generate_s": round(t_gen, 2), "encode_s": round(t_enc, 2)}
    return centers, codes_s, info


def reference_pqclust():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    p = ROOT / "baseline" / "_ref"
    if p.exists() and str(p) not in sys.path:
        sys.path.insert(0, str(p))
    try:
        import pqclust  # noqa: F401

        return pqclust
    except Exception:
        return None


def reference_encoder():
    pqc = reference_pqclust()
    if pqc is not None:
        return (lambda book, x: pqc.encode(pqc.PQCodebook(np.asarray(book, dtype=np.float32)), x)), \
            "pqclust.encode (reference, baseline/_ref)"
    from oracle import pqk_oracle as O

    return O.encode, "oracle.encode (restatement of pq.py:205-231)"


def pqclust_assign_rate(codes_s: np.ndarray, centers: np.ndarray, book: np.ndarray, threads: int,
                        budget_s: float = 4.0) -> dict | None:
    """The unmodified reference's own assignment (pqclust.assign, linear scan, threads=T)
    on a bounded sample; its labels are compared with the C port's on the same rows."""
    pqc = reference_pqclust()
    if pqc is None:
        return None
    from oracle import pqk_oracle as O

    tables = pqc.build_distance_tables(pqc.PQCodebook(np.asarray(book, dtype=np.float32)))
    k = len(centers)
    s = int(min(len(codes_s), max(64, budget_s * 3e7 * threads / k)))
    t0 = time.perf_counter()
    lab = pqc.assign(codes_s[:s], centers, tables, threads=threads)
    dt = time.perf_counter() - t0
    same = bool(np.array_equal(lab, O.assign_c(codes_s[:s], centers, tables.tables, threads)))
    return {"assign_evals_per_s": s * k / dt, "rows": s, "threads": threads, "seconds": dt,
            "labels_equal_port": same, "api": "pqclust.assign(codes, centers, tables, threads=T) (linear_scan)"}


def run_reference(args) -> None:
    """--impl reference: the reference algorithm on the box's host cores, same inputs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import pqk_oracle as O

    cfgn = args.config
    cfg = CONFIGS[cfgn]
    k = cfg["k"]
    world = args.gpus
    n_total = cfg["n"] * world
    threads = cpu_threads()
    rows_max = min(cfg["n"], cpu_sample_rows(k, threads, 4.0))
    t_setup = time.perf_counter()
    centers, codes_s, info = reference_inputs(cfgn, world, k, rows_max)
    tables = O.build_distance_tables(make_codebook(cfgn, cfg["m"], cfg["l"]))
    info["setup_s"] = round(time.perf_counter() - t_setup, 1)
    # calibrate S so a step's assignment takes ~2.5 s of the host's threads
    cal = cpu_step(codes_s[: min(len(codes_s), max(256, threads * 64))], centers, tables, n_total, threads, 16)
    rows = int(min(len(codes_s), max(256, 2.5 * cal["assign_evals_per_s"] / k)))
    for _ in range(args.warmup):
        cpu_step(codes_s[:rows], centers, tables, n_total, threads)
    vals = [cpu_step(codes_s[:rows], centers, tables, n_total, threads) for _ in range(args.steps)]
    v = float(np.median([x["value"] for x in vals]))
    spi = float(np.median([x["s_per_iteration"] for x in vals]))
    step_ms = float(np.mean([x["step_s"] for x in vals])) * 1e3
    sample = (f"per step: assign {rows} of {n_total} codes x {k} centers (C port of clustering.py:167-197, "
              f"{threads} threads) + sparse vote of {vals[-1]['vote_clusters']} clusters x {cfg['m']} subspaces "
              f"(numpy port of clustering.py:327-356); value = N*K / (assign x N/S + vote x K/clusters)")
    out = {
        "metric": "code-center distance evals/s", "impl": "reference", "value": v, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "s_per_iteration": spi, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n_total, "k": k, "m": cfg["m"], "l": cfg["l"],
                   "inputs": "the b200 arm's initial centers and rank 0's first codes (same seeds, same codebook)",
                   "centers_sha16": _sha16(centers), **info},
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": threads, "kind": "port", "sample": sample,
                         "s_per_iteration": spi,
                         "note": "ms_per_step is one sampled step's wall time; s_per_iteration is the "
                                 "extrapolated full iteration the value is quoted on"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    pq = pqclust_assign_rate(codes_s, centers, make_codebook(cfgn, cfg["m"], cfg["l"]), threads)
    if pq is not None:
        pq["s_per_iteration_assign_only"] = n_total * k / pq["assign_evals_per_s"]
        out["reference_python"] = pq
    print(json.dumps(out), flush=True)


def _sha16(a: np.ndarray) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# ---------------------------------------------------------------------------
# parity: one untimed iteration checked against the oracle
def parity_record(eng, cur_in, codes_host: np.ndarray, tables: np.ndarray, k: int, m: int, l_count: int, *,
                  rows: int = 20_000, votes: int = 2_000, check_hist: bool = True, check_repair: bool = True,
                  seed: int = SEED + 7) -> dict:
    """Bit-exact checks of the engine state after one iteration with centers `cur_in`:
    labels and sd of `rows` sampled codes (oracle C scan, clustering.py:167-197 and
    pq.py:271-290), the objective sums (numpy's pairwise tree, clustering.py:448-449),
    the full K x M x L histogram against bincount of the GPU labels (clustering.py:344-347),
    `votes` sampled (k, m) votes (clustering.py:349-354) and every repaired cluster
    (clustering.py:460-466)."""
    from oracle import pqk_oracle as O

    t0 = time.perf_counter()
    threads = cpu_threads()
    n = eng.n
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(rows, n), replace=False))
    cen = cur_in[:, :m].cpu().numpy()
    lab_g = eng.labels[:n].cpu().numpy().view(np.uint32)
    sd_g = eng.sd[:n].cpu().numpy()
    lab_o, sd_o = O.assign_c(codes_host[idx], cen, tables, threads, want_sd=True)
    rec = {"rows": int(len(idx)), "label_mismatch": int((lab_o != lab_g[idx]).sum()),
           "sd_mismatch": int((sd_o.view(np.uint64) != sd_g[idx].view(np.uint64)).sum())}
    obj = eng.obj.cpu().numpy()
    rec["objective_equal"] = bool(obj[0] == np.sum(np.sqrt(sd_g)) and obj[1] == np.sum(sd_g))
    hist_g = eng.hist[: k * m * l_count].cpu().numpy().view(np.uint32).reshape(k, m, l_count)
    counts_g = eng.counts[:k].cpu().numpy().view(np.uint32)
    if check_hist:
        joint = lab_g.astype(np.int64) * l_count
        bad = 0
        for mm in range(m):
            h = np.bincount(joint + codes_host[:, mm], minlength=k * l_count).reshape(k, l_count)
            bad += int((h != hist_g[:, mm, :]).sum())
        rec["hist_bins"] = int(k * m * l_count)
        rec["hist_mismatch"] = bad
        rec["counts_mismatch"] = int((np.bincount(lab_g.astype(np.intp), minlength=k) != counts_g).sum())
    new_c = eng.new_centers[:, :m].cpu().numpy()
    filled = np.flatnonzero(counts_g > 0)
    pairs = rng.choice(len(filled) * m, size=min(votes, len(filled) * m), replace=False)
    vbad = 0
    for p in pairs:
        ki, mm = int(filled[p // m]), int(p % m)
        vbad += int(O.vote_argmin(hist_g[ki, mm].astype(np.int64), tables[mm]) != new_c[ki, mm])
    rec["votes"] = int(len(pairs))
    rec["vote_mismatch"] = vbad
    empty = np.flatnonzero(counts_g == 0)
    e = len(empty)
    rec["repaired"] = int(e)
    if e and check_repair:
        # farthest codes, sd descending then index ascending (np.argmax picks the first)
        cand = np.argpartition(sd_g, n - e)[n - e:] if e < n else np.arange(n)
        thr = sd_g[cand].min()
        cand = np.flatnonzero(sd_g >= thr)
        order = cand[np.lexsort((cand, -sd_g[cand]))][:e]
        rec["repair_mismatch"] = int((codes_host[order] != new_c[empty]).any(axis=1).sum())
    rec["mismatch"] = int(sum(v for key, v in rec.items() if key.endswith("mismatch")) + (not rec["objective_equal"]))
    rec["seconds"] = round(time.perf_counter() - t0, 1)
    rec["oracle"] = "oracle/pqk_oracle.py + pqk_scan.c (pinned to the reference's outputs, tests/golden)"
    return rec


# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(args) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run, N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    log("[bench] launching", " ".join(cmd[2:6]), "...")
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip encoder/training/streaming side measurements")
    ap.add_argument("--no-graphs", action="store_true", help="launch the iteration eagerly (no CUDA graphs)")
    ap.add_argument("--dist", action="store_true", help="sharded NCCL driver even with one rank")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "b200":
        sys.exit(relaunch_distributed(args))
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1709_03708_b200 import _lib, engine
    from paper_1709_03708_b200.distributed import DistributedLloyd, GpuShardBackend, shard_bounds

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
        # stdout carries only the JSON line: NCCL's log (at the level the caller chose with
        # NCCL_DEBUG, WARN by default) goes to stderr
        os.environ.setdefault("NCCL_DEBUG", "WARN")
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
    mp = _lib.padded_m(m)

    # ---- workload -----------------------------------------------------------------
    t0 = time.perf_counter()
    wl = build_workload(cfgn, dev, rank, world)
    book, tables, codes_host = wl["book"], wl["tables"], wl["codes_host"]
    vectors = wl["vectors"]
    log(f"[bench] rank {rank}/{world}: workload ready in {time.perf_counter() - t0:.1f}s")

    offset, length = shard_bounds(n_total, world, rank)
    assert length == n_loc, (length, n_loc)
    backend = GpuShardBackend(codes_host, offset, tables, k, device=local, graphs=not args.no_graphs)
    drv = DistributedLloyd(backend, n_total, k, m) if use_dist else None
    if use_dist:
        centers0 = drv.init_centers(SEED, codes_host)
    else:
        centers0 = codes_host[center_indices(n_loc, k)].copy()
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
        # measured shared-memory ceiling (roofline denominator), right before the region
        import ctypes as C

        smem_bps, smem_ms = C.c_double(0), C.c_double(0)
        _lib.check(lib.pqk_smem_probe(local, 16384, C.byref(smem_bps), C.byref(smem_ms),
                                      C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)), "pqk_smem_probe")
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
    lb = int(np.median(lookup_b)) or 4  # 1: 8-bit first tier, 2: 16-bit first tier, 4: fp32 scan
    lookup_bytes = n_loc * u * m * lb  # algorithmic: one table lookup per (code, center, subspace)
    scan_name = {1: "hscan8_kernel (8-bit fixed-point tables, top-6 chunk keys)",
                 2: "hscan_kernel (16-bit fixed-point tables)"}.get(lb, "scan_kernel (fp32 tables)")
    scan_s = float(np.mean(scan_ms)) / 1e3
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = clocks.summary()
    arch_peak = sm_count * 128 * 1965.0 * 1e6 / 1e9  # GB/s: 128 B/clk/SM at the max SM clock
    peak = smem_bps.value / 1e9
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
        "dtype": DTYPE,
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n_total, "k": k, "m": m, "l": l_count,
                   "codebook": f"reference pq.train_codebook, {CODEBOOK_RECIPES[cfgn]['sample']}-vector sample, "
                               f"{CODEBOOK_RECIPES[cfgn]['iterations']} iterations (bench_assets/{cfgn}_codebook.npy)",
                   "centers_sha16": _sha16(centers0),
                   "unique_centers": u, "flagged_codes_per_iter": int(np.median(flagged)),
                   "fp64_rescan_codes_per_iter": int(np.median(flagged64)),
                   "votes_fp64_per_iter": int(np.median(vote_fp64)), "votes_dd_per_iter": int(np.median(vote_dd)),
                   "l2": "flushed (512 MB write) between timed iterations",
                   "step": "assign+certify+objective+histogram+allreduce+vote+repair",
                   "launch": ("eager" if args.no_graphs else
                              "cuda graphs per phase (assign+objective+histogram, vote), collectives between"
                              if use_dist else "cuda graphs (after first warm-up step)"),
                   "parallelism": f"codes sharded dp{world}", "backend": backend_name if use_dist else None},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "peak_source": f"measured: pqk_smem_probe (conflict-free LDS.128, one 1024-thread CTA per SM, best of 3, "
                                    f"{smem_ms.value:.2f} ms launch) just before the timed steps; architectural "
                                    f"{sm_count} SMs x 128 B/clk x 1965 MHz = {arch_peak:.0f} GB/s",
                     "frac_of_architectural": achieved / arch_peak,
                     "note": f"{scan_name}: {n_loc}x{u}x{m} {lb}-byte lookups per launch / {scan_s * 1e3:.3f} ms "
                             "(CUDA events around the launch on its stream)",
                     "scan_ms": scan_s * 1e3, "scan_share_of_step": scan_s * 1e3 / ms_per_step,
                     "lookups_per_s": n_loc * u * m / scan_s},
        "clocks": clk,
        "gpu_launches": int(launches),
    }

    # ---- parity: one more (untimed) iteration, checked against the oracle -------------
    if not args.no_parity:
        with torch.cuda.device(dev):
            cur_in = cur.clone()
            cur, _ = step(cur)
            torch.cuda.synchronize(dev)
        if rank == 0:
            out["parity"] = parity_record(eng, cur_in, codes_host, tables, k, m, l_count, check_hist=not use_dist,
                                          check_repair=not use_dist)
            if use_dist:
                out["parity"]["note"] = ("rank 0's shard; the histogram is the allreduced one (votes checked on it); "
                                         "the repair merges all ranks' candidates (checked by tests/test_distributed_gloo.py)")

    hbm_peak = 6545.3
    try:
        hbm_peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    if rank == 0 and not args.no_extras:
        # GPU codebook training with the reference recipe on the same sample: bit-identical?
        from paper_1709_03708_b200 import pq as gpq

        rec = CODEBOOK_RECIPES[cfgn]
        tsample = codebook_sample(cfgn)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        gbook = gpq.train_codebook(tsample, m, l_count, iterations=rec["iterations"], seed=rec["seed"], device=local)
        out["codebook_training"] = {
            "vectors": rec["sample"], "dim": cfg["dim"], "m": m, "l": l_count, "iterations": rec["iterations"],
            "seconds": time.perf_counter() - t0,
            "equal_to_reference": bool(np.array_equal(np.asarray(gbook.codewords), book)),
            "reference": "bench_assets codebook = the reference's own pq.train_codebook on the same sample"}
        del tsample
    # PQ encoder (set-up of the workload, timed with events): HBM roofline of code streaming
    enc_bytes = n_loc * (4 * cfg["dim"] + m)
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
        "note": "histogram: codes (MP B) + labels (4 B) per code in, K x M x 256 int32 table out; objective: "
                "8 B sd per code through numpy's pairwise tree; L2 flushed before each"}
    enc_ms = wl["enc_ms"]
    dsub = cfg["dim"] // m
    out["encode"] = {"vectors": n_loc, "ms": enc_ms, "vectors_per_s": n_loc / (enc_ms / 1e3),
                     "hbm_gbs": enc_bytes / (enc_ms / 1e3) / 1e9,
                     "hbm_frac": enc_bytes / (enc_ms / 1e3) / 1e9 / hbm_peak,
                     "flagged_pairs": wl["enc_flagged"],
                     "kernel": ("encode_tc_kernel (tcgen05 fp16 hi/lo split, certified argmin, fp64 fallback)"
                                if dsub in (8, 16, 32, 64) else
                                "encode_tck_kernel (K-streamed tcgen05, certified argmin, fp64 fallback)"
                                if dsub % 32 == 0 and 96 <= dsub <= 1024 else
                                "encode_kernel (SIMT fp32 filter + fp64 certificate)")}

    # original-space error / Bk-means / file streaming on host-made data
    if rank == 0 and vectors is not None and not args.no_extras:
        extras_host_data(out, eng, vectors, codes_host, book, cfg, k, m, n_loc, dev, hbm_peak)

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
                      "api": "pqk_lloyd_step_host (C-ABI, pinned host buffers): one Lloyd iteration"}
        # the reference plugin's call (AssignStrategy, clustering.py:200): labels of host codes
        pin_cent.copy_(torch.from_numpy(centers0))
        ptimes = []
        for it in range(3):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            _lib.check(lib.pqk_assign_host(p(pin_codes), n_loc, m, p(pin_cent), k, p(pin_tab), l_count, p(pin_lab),
                                           None, local))
            if it:
                ptimes.append(time.perf_counter() - t0)
        pa_s = float(np.mean(ptimes))
        out["e2e"]["plugin_assign"] = {
            "value": n_total * k / pa_s, "unit": "evals/s", "ms_per_call": pa_s * 1e3,
            "h2d_bytes_per_call": int(codes_host.nbytes + centers0.nbytes + tables.nbytes),
            "d2h_bytes_per_call": int(n_loc * 4),
            "api": "pqk_assign_host (C-ABI of the AssignStrategy plugin, INTEGRATION.md), pinned host buffers"}
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
        threads = cpu_threads()
        rows = min(n_loc, cpu_sample_rows(k, threads, 0.05))
        cal = cpu_step(codes_host[:rows], centers0, tables, n_total, threads, 16)
        rows = int(min(n_loc, max(256, 8.0 * cal["assign_evals_per_s"] / k)))
        cb = cpu_step(codes_host[:rows], centers0, tables, n_total, threads)
        out["cpu_baseline"] = {
            "value": cb["value"], "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": f"assign {rows} of {n_total} codes x {k} centers ({cb['t_assign']:.2f}s, {threads} threads, C port "
                      f"of clustering.py:167-197) + sparse vote of {cb['vote_clusters']} clusters ({cb['t_update']:.2f}s, "
                      "numpy port of clustering.py:327-356); iteration extrapolated (assign x N/S, vote x K/clusters)",
            "assign_evals_per_s": cb["assign_evals_per_s"], "s_per_iteration": cb["s_per_iteration"]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def extras_host_data(out, eng, vectors, codes_host, book, cfg, k, m, n_loc, dev, hbm_peak) -> None:
    """original_space_error, Bk-means and the file-streaming pipeline on the config's vectors."""
    import torch

    from paper_1709_03708_b200 import _lib, engine
    from paper_1709_03708_b200.pq import PQCodebook

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
        from paper_1709_03708_b200 import synth

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


if __name__ == "__main__":
    main()
