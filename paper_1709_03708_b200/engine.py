"""Device-resident state of the compressed-domain Lloyd iteration.

PyTorch provides device memory, streams and (in :mod:`.distributed`) NCCL;
every computation is a launch of the sm_100a C-ABI in ``libpqk_b200.so``.
There is no CPU path: without CUDA these functions raise ``RuntimeError``.

Data layout in HBM (one device, one shard of N codes):
  codes    (N, MP) uint8   MP = padded M (pad subspaces are zero)
  t64      (M, L, L) f64   reference DistanceTables, used for every exact result
  t32      (MP, L, L) f32  ldexp-scaled copy, the assignment filter's source
  labels   (N,) int32 (bit pattern of the reference's uint32 labels)
  sd       (N,) f64        distance of each code to its center (clustering.py:447)
  hist     (K, M, L) uint32 member histograms (clustering.py:344-347), in int32 tensors
  counts   (K,) uint32, in an int32 tensor
  centers  (K, MP) uint8 ×2 (current / next)
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import STATS_LEN, call

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise ImportError("paper_1709_03708_b200 needs PyTorch for device memory and streams") from exc


def device_of(device: int | None = None) -> "torch.device":
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1709_03708_b200 runs on a CUDA device (sm_100a); no GPU is visible and there is no CPU fallback"
        )
    _lib.load()
    idx = torch.cuda.current_device() if device is None else int(device)
    return torch.device("cuda", idx)


def _ptr(t: "torch.Tensor | None") -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(dev: "torch.device") -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


# PQK_GUARD=1 (diagnostic; the pool has no compute-sanitizer): every buffer the kernels
# write is allocated between two 64 KB guard zones filled with 0xA5, and check_guards()
# reports any zone a kernel overwrote (an out-of-bounds store into a neighbouring buffer).
_GUARD = os.environ.get("PQK_GUARD", "") == "1"
_GUARD_BYTES = 64 << 10
_GUARDS: list = []


def _alloc(shape, dtype, dev, zero: bool = False) -> "torch.Tensor":
    if not _GUARD:
        return (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=dev)
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    numel = 1
    for s in shape:
        numel *= int(s)
    nbytes = numel * torch.tensor([], dtype=dtype).element_size()
    raw = torch.full((_GUARD_BYTES + nbytes + _GUARD_BYTES,), 0xA5, dtype=torch.uint8, device=dev)
    body = raw[_GUARD_BYTES:_GUARD_BYTES + nbytes]
    if zero:
        body.zero_()
    _GUARDS.append((raw, nbytes))
    return body.view(dtype).view(shape)


def check_guards() -> list:
    """Indices of guarded buffers whose guard zones were overwritten (empty: all intact)."""
    bad = []
    for i, (raw, nbytes) in enumerate(_GUARDS):
        lo = raw[:_GUARD_BYTES]
        hi = raw[_GUARD_BYTES + nbytes:]
        if bool((lo != 0xA5).any()) or bool((hi != 0xA5).any()):
            bad.append(i)
    return bad


def _empty(n_bytes: int, dev) -> "torch.Tensor":
    return _alloc(max(int(n_bytes), 1), torch.uint8, dev)


# ---------------------------------------------------------------------------
# tables
@dataclass
class DeviceTables:
    t64: "torch.Tensor"
    t32: "torch.Tensor"
    m: int
    l: int
    mp: int
    fp64_only: int
    exp2: int
    t16: "torch.Tensor | None" = None  # fp16 vote tables (L = 256), built once


_TABLE_CACHE: dict = {}
_TABLE_LOCK = threading.Lock()


def device_tables(tables: np.ndarray, dev) -> DeviceTables:
    """Upload (M, L, L) float64 tables and build the scaled fp32 filter copy (cached)."""
    t = np.ascontiguousarray(tables, dtype=np.float64)
    # keyed by content (never by identity: a read-only view can still change through a
    # writable base, and the reference recomputes from the array every call)
    key = (dev.index, t.shape, hashlib.blake2b(t.tobytes(), digest_size=16).digest())
    hold = None
    with _TABLE_LOCK:
        hit = _TABLE_CACHE.get(key)
        if hit is not None:
            return hit[0]
    m, l, _ = t.shape
    lib = _lib.load()
    e = C.c_int32(0)
    f64 = C.c_int32(0)
    _lib.check(lib.pqk_table_scale(t.ctypes.data_as(C.c_void_p), t.size, C.byref(e), C.byref(f64)), "pqk_table_scale")
    mp = _lib.padded_m(m)
    t64 = torch.from_numpy(np.array(t)).to(dev)  # (read-only DistanceTables arrays)
    t32 = torch.empty(mp * l * l, dtype=torch.float32, device=dev)
    call("pqk_tables_to_f32", _ptr(t64), m, l, e.value, _ptr(t32), _stream(dev))
    t16 = None
    if l == 256 and not f64.value:
        t16 = torch.empty(m * l * l, dtype=torch.int16, device=dev)
        call("pqk_vote_tables16_device", _ptr(t32), m, l, _ptr(t16), _stream(dev))
    dt = DeviceTables(t64, t32, m, l, mp, int(f64.value), int(e.value), t16)
    with _TABLE_LOCK:
        if len(_TABLE_CACHE) >= 8:
            _TABLE_CACHE.pop(next(iter(_TABLE_CACHE)))
        _TABLE_CACHE[key] = (dt, hold)
    return dt


def upload_codes(codes: np.ndarray, m: int, dev) -> "torch.Tensor":
    """(N, M) integer host codes (already validated) -> (N, MP) uint8 device layout."""
    mp = _lib.padded_m(m)
    host = np.ascontiguousarray(codes, dtype=np.uint8)
    n = host.shape[0]
    if mp == m:
        return torch.from_numpy(host).to(dev)
    out = torch.empty((n, mp), dtype=torch.uint8, device=dev)
    if n:
        raw = torch.from_numpy(host).to(dev)
        call("pqk_pad_codes_device", _ptr(raw), n, m, _ptr(out), _stream(dev))
    return out


def download_codes(codes_dev: "torch.Tensor", m: int) -> np.ndarray:
    return np.ascontiguousarray(codes_dev[:, :m].cpu().numpy())


# ---------------------------------------------------------------------------
# numpy pairwise-sum plan (objective)
@dataclass
class PairwisePlan:
    n: int
    nleaves: int
    ndepth: int
    depth_start: np.ndarray  # host int64 (ndepth+1)
    leaf_off: "torch.Tensor"
    leaf_len: "torch.Tensor"
    node_a: "torch.Tensor"
    node_b: "torch.Tensor"
    ws: "torch.Tensor"


def host_plan(n: int) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """numpy's pairwise_sum tree for n elements (built by the C-ABI helper)."""
    lib = _lib.load()
    nl, nd, nn = C.c_int64(0), C.c_int32(0), C.c_int64(0)
    _lib.check(lib.pqk_pairwise_plan_size(n, C.byref(nl), C.byref(nd), C.byref(nn)), "pqk_pairwise_plan_size")
    leaf_off = np.empty(nl.value, np.int64)
    leaf_len = np.empty(nl.value, np.int32)
    depth_start = np.empty(nd.value + 1, np.int64)
    na = np.empty(nn.value, np.int32)
    nb = np.empty(nn.value, np.int32)
    _lib.check(
        lib.pqk_pairwise_plan_build(
            n, *(x.ctypes.data_as(C.c_void_p) for x in (leaf_off, leaf_len, depth_start, na, nb))
        ),
        "pqk_pairwise_plan_build",
    )
    return leaf_off, leaf_len, depth_start, na, nb


def pairwise_plan(n: int, dev) -> PairwisePlan:
    leaf_off, leaf_len, depth_start, na, nb = host_plan(n)
    ws_bytes = _lib.load().pqk_objective_workspace_bytes(len(leaf_off), len(na))
    return PairwisePlan(
        n,
        len(leaf_off),
        len(depth_start) - 1,
        depth_start,
        torch.from_numpy(leaf_off).to(dev),
        torch.from_numpy(leaf_len).to(dev),
        torch.from_numpy(na).to(dev),
        torch.from_numpy(nb).to(dev),
        _empty(ws_bytes, dev),
    )


def objective_sums(sd: "torch.Tensor", plan: PairwisePlan, out2: "torch.Tensor", dev) -> None:
    """out2 <- (pairwise_sum(sqrt(sd)), pairwise_sum(sd)) exactly as numpy."""
    call(
        "pqk_objective_device",
        _ptr(sd),
        plan.n,
        plan.nleaves,
        plan.ndepth,
        _ptr(plan.leaf_off),
        _ptr(plan.leaf_len),
        plan.depth_start.ctypes.data_as(C.c_void_p),
        _ptr(plan.node_a),
        _ptr(plan.node_b),
        _ptr(plan.ws),
        plan.ws.numel(),
        _ptr(out2),
        _stream(dev),
    )


def mean_from_sum(total: float, n: int) -> float:
    """np.mean's final step: float64 sum divided by the count (true_divide)."""
    return float(np.float64(total) / n)


# ---------------------------------------------------------------------------
class ShardEngine:
    """One device's share of the Lloyd iteration (all N codes on a single GPU)."""

    def __init__(self, codes_dev: "torch.Tensor", tables: DeviceTables, k: int, dev, base_index: int = 0):
        self.dev = dev
        self.tables = tables
        self.codes = codes_dev
        self.n = int(codes_dev.shape[0])
        self.k = int(k)
        self.base_index = int(base_index)
        m, l, mp = tables.m, tables.l, tables.mp
        lib = _lib.load()
        self.labels = _alloc(max(self.n, 1), torch.int32, dev)
        self.sd = _alloc(max(self.n, 1), torch.float64, dev)
        self.ws_bytes = int(lib.pqk_assign_workspace_bytes(max(self.n, 1), self.k, m, l))
        self.ws = _empty(self.ws_bytes, dev)
        self.stats = _alloc(STATS_LEN, torch.int64, dev, zero=True)
        self.hist = _alloc(self.k * m * l, torch.int32, dev)
        self.counts = _alloc(self.k, torch.int32, dev)
        self.new_centers = _alloc((self.k, mp), torch.uint8, dev, zero=True)
        self.rws_bytes = int(lib.pqk_repair_workspace_bytes(max(self.n, 1), self.k))
        self.rws = _empty(self.rws_bytes, dev)
        self.obj = _alloc(2, torch.float64, dev, zero=True)
        self.plan = pairwise_plan(self.n, dev) if self.n else None

    # -- stream-ordered launches ------------------------------------------------
    def assign(self, centers_dev: "torch.Tensor") -> None:
        t = self.tables
        if self.n == 0:
            return
        call(
            "pqk_assign_device",
            _ptr(self.codes),
            self.n,
            t.m,
            t.l,
            _ptr(centers_dev),
            int(centers_dev.shape[0]),
            _ptr(t.t64),
            _ptr(t.t32),
            t.fp64_only,
            _ptr(self.ws),
            self.ws_bytes,
            _ptr(self.labels),
            _ptr(self.sd),
            _ptr(self.stats),
            _stream(self.dev),
        )

    def distances_for_labels(self, centers_dev: "torch.Tensor") -> None:
        """sd <- paired distance of every code to centers[labels] (external strategies)."""
        t = self.tables
        call(
            "pqk_paired_distance_device",
            _ptr(self.codes),
            _ptr(centers_dev),
            _ptr(self.labels),
            self.n,
            t.m,
            t.l,
            _ptr(t.t64),
            _ptr(self.sd),
            _stream(self.dev),
        )

    def objective(self) -> None:
        if self.n:
            objective_sums(self.sd[: self.n], self.plan, self.obj, self.dev)

    def histogram(self) -> None:
        t = self.tables
        call(
            "pqk_histogram_device",
            _ptr(self.codes),
            self.n,
            t.m,
            t.l,
            _ptr(self.labels),
            self.k,
            _ptr(self.hist),
            _ptr(self.counts),
            _stream(self.dev),
        )

    def vote(self) -> None:
        t = self.tables
        call(
            "pqk_vote16_device",
            _ptr(self.hist),
            _ptr(self.counts),
            self.k,
            t.m,
            t.l,
            _ptr(t.t64),
            _ptr(None if t.fp64_only else t.t32),
            _ptr(None if t.fp64_only else t.t16),
            _ptr(self.new_centers),
            _ptr(self.stats),
            _stream(self.dev),
        )

    def repair(self) -> None:
        call(
            "pqk_repair_device",
            _ptr(self.sd),
            _ptr(self.codes),
            self.n,
            self.tables.m,
            _ptr(self.counts),
            self.k,
            _ptr(self.new_centers),
            _ptr(self.rws),
            self.rws_bytes,
            _ptr(self.stats),
            _stream(self.dev),
        )

    def repair_candidates(self, e: int) -> tuple["torch.Tensor", "torch.Tensor"]:
        """Local top-e (sd desc, global index asc) candidates: (uint64 keys, int64 global index)."""
        keys = torch.empty(max(e, 1), dtype=torch.int64, device=self.dev)
        index = torch.empty(max(e, 1), dtype=torch.int64, device=self.dev)
        e_eff = min(e, self.n)
        if e_eff > 0:
            need = int(_lib.load().pqk_repair_workspace_bytes(self.n, max(e_eff, 1)))
            ws = self.rws if need <= self.rws_bytes else _empty(need, self.dev)
            call(
                "pqk_repair_candidates_device",
                _ptr(self.sd),
                self.n,
                self.base_index,
                e_eff,
                _ptr(ws),
                ws.numel(),
                _ptr(keys),
                _ptr(index),
                _stream(self.dev),
            )
        return keys[:e_eff], index[:e_eff]

    # -- host reads ---------------------------------------------------------------
    def read_obj_stats(self) -> tuple[np.ndarray, np.ndarray]:
        """Objective sums and stats with two async D2H copies and one stream sync."""
        if not hasattr(self, "_pin_obj"):
            self._pin_obj = torch.empty(2, dtype=torch.float64).pin_memory()
            self._pin_stats = torch.empty(STATS_LEN, dtype=torch.int64).pin_memory()
        self._pin_obj.copy_(self.obj, non_blocking=True)
        self._pin_stats.copy_(self.stats, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return self._pin_obj.numpy().copy(), self._pin_stats.numpy().copy()

    def stats_host(self) -> np.ndarray:
        return self.stats.cpu().numpy()

    def labels_host(self) -> np.ndarray:
        return self.labels[: self.n].cpu().numpy().view(np.uint32)

    def sd_host(self) -> np.ndarray:
        return self.sd[: self.n].cpu().numpy()


class IterationGraphs:
    """The device part of a Lloyd iteration as two CUDA graphs, replayed every iteration:
    ``main`` = assign(cur) -> [objective sums || histogram -> vote] (~15 kernel launches),
    ``repair`` = the empty-cluster repair (~30 launches of the 12-digit radix select).
    ``cur`` is a fixed (K, MP) centers buffer; the caller refreshes it with
    ``cur.copy_(eng.new_centers)`` between replays.  Capture after one eager iteration
    (lazy device info and kernel attributes are set up by then).  ``ev_assigned`` is an
    external event node recorded after the assignment (per-iteration assign timing)."""

    def __init__(self, eng: ShardEngine, cur: "torch.Tensor"):
        import torch

        self.eng, self.cur = eng, cur
        self.ev_assigned = torch.cuda.Event(enable_timing=True, external=True)
        lib = _lib.load()
        self.main = torch.cuda.CUDAGraph()
        l0 = lib.pqk_launch_count()
        side = torch.cuda.Stream(device=eng.dev)
        with torch.cuda.graph(self.main, capture_error_mode="thread_local"):
            eng.assign(cur)
            self.ev_assigned.record()
            # the objective sums (a latency-bound tree) run on a parallel branch of the graph,
            # beside the histogram and the vote; they share no buffers
            fork = torch.cuda.Event()
            fork.record()
            side.wait_event(fork)
            with torch.cuda.stream(side):
                eng.objective()
            join = torch.cuda.Event()
            join.record(side)
            eng.histogram()
            eng.vote()
            torch.cuda.current_stream(eng.dev).wait_event(join)
        self.main_launches = int(lib.pqk_launch_count() - l0)
        self.repair = torch.cuda.CUDAGraph()
        l0 = lib.pqk_launch_count()
        with torch.cuda.graph(self.repair, capture_error_mode="thread_local"):
            eng.repair()
        self.repair_launches = int(lib.pqk_launch_count() - l0)


# ---------------------------------------------------------------------------
# one-shot host helpers used by the public API
def assign_host(codes: np.ndarray, centers: np.ndarray, tables: np.ndarray, *, device=None, want_sd=False):
    """Labels (and optionally sd) of host codes through ``pqk_assign_host``, the C-ABI of the
    AssignStrategy plugin: a cached per-device context (grow-only buffers, tables compared by
    content) runs only the assignment — no histogram, repair workspace or summation plan."""
    dev = device_of(device)
    c = np.ascontiguousarray(codes, dtype=np.uint8)
    ce = np.ascontiguousarray(centers, dtype=np.uint8)
    t = np.ascontiguousarray(tables, dtype=np.float64)
    n, m = c.shape
    labels = np.empty(n, dtype=np.uint32)
    sd = np.empty(n, dtype=np.float64) if want_sd else None
    lib = _lib.load()
    _lib.check(
        lib.pqk_assign_host(c.ctypes.data, n, m, ce.ctypes.data, len(ce), t.ctypes.data, t.shape[1],
                            labels.ctypes.data, None if sd is None else sd.ctypes.data, dev.index),
        "pqk_assign_host",
    )
    return (labels, sd) if want_sd else labels


def paired_distance_host(tables: np.ndarray, a: np.ndarray, b: np.ndarray, *, device=None) -> np.ndarray:
    dev = device_of(device)
    dt = device_tables(tables, dev)
    n = len(a)
    if n == 0:
        return np.zeros(0, dtype=np.float64)
    with torch.cuda.device(dev):
        a_dev = upload_codes(a, dt.m, dev)
        b_dev = upload_codes(b, dt.m, dev)
        out = torch.empty(n, dtype=torch.float64, device=dev)
        call(
            "pqk_paired_distance_device",
            _ptr(a_dev),
            _ptr(b_dev),
            _ptr(None),
            n,
            dt.m,
            dt.l,
            _ptr(dt.t64),
            _ptr(out),
            _stream(dev),
        )
        return out.cpu().numpy()


def vote_host(hist: np.ndarray, tables: np.ndarray, *, device=None) -> np.ndarray:
    """Sparse-vote centers for (K, M, L) host histograms; (K, M) uint8 (empty rows -> 0)."""
    dev = device_of(device)
    dt = device_tables(tables, dev)
    k = hist.shape[0]
    counts_h = hist[:, 0, :].sum(axis=1) if k else np.zeros(0, np.int64)
    if hist.min(initial=0) < 0 or counts_h.max(initial=0) >= 2**32:
        raise ValueError("histogram counts must be non-negative and fit in uint32")
    with torch.cuda.device(dev):
        # uint32 counts carried in int32 tensors (the kernels read them unsigned)
        h = torch.from_numpy(np.ascontiguousarray(hist, dtype=np.uint32).view(np.int32)).to(dev)
        counts = torch.from_numpy(counts_h.astype(np.uint32).view(np.int32)).to(dev)
        out = torch.zeros((k, dt.mp), dtype=torch.uint8, device=dev)
        stats = torch.zeros(STATS_LEN, dtype=torch.int64, device=dev)
        call("pqk_vote_device", _ptr(h), _ptr(counts), k, dt.m, dt.l, _ptr(dt.t64),
             _ptr(None if dt.fp64_only else dt.t32), _ptr(out), _ptr(stats), _stream(dev))
        return download_codes(out, dt.m)


def mean_objectives(sd_dev: "torch.Tensor", n: int, dev) -> tuple[float, float]:
    """(mean(sqrt(sd)), mean(sd)) with numpy's summation tree, on device."""
    plan = pairwise_plan(n, dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    objective_sums(sd_dev, plan, out, dev)
    s = out.cpu().numpy()
    return mean_from_sum(s[0], n), mean_from_sum(s[1], n)


def encode_host(codewords: np.ndarray, vectors: np.ndarray, *, device=None, stride: int | None = None):
    """(N, D) float32 -> (N, M) uint8 codes on device; returns host codes."""
    dev = device_of(device)
    m, l, sub = codewords.shape
    n, d = vectors.shape
    with torch.cuda.device(dev):
        out = encode_device(
            torch.from_numpy(np.ascontiguousarray(vectors, dtype=np.float32)).to(dev),
            torch.from_numpy(np.array(codewords, dtype=np.float32)).to(dev),  # (read-only codebooks)
            m,
            l,
            dev,
            stride=m,
        )
        return out.cpu().numpy()


def train_codebook_host(vectors: np.ndarray, m: int, l: int, iterations: int, seed: int, *, device=None) -> np.ndarray:
    """Per-subspace Lloyd k-means on the GPU, bit-identical to pq.train_codebook (pq.py:127-202).

    Initial codewords come from the same host Generator draws as the reference; each
    Lloyd step runs in pqk_train_step_device; empty codewords are re-seeded on the
    farthest points (lowest index first) chosen by the device top-E select.
    """
    dev = device_of(device)
    lib = _lib.load()
    vectors = np.ascontiguousarray(vectors, dtype=np.float32)
    n, d = vectors.shape
    sub = d // m
    rng = np.random.default_rng(seed)
    books = np.empty((m, l, sub), dtype=np.float32)
    with torch.cuda.device(dev):
        s = _stream(dev)
        x = torch.from_numpy(vectors).to(dev)
        labels = _alloc(n, torch.int32, dev)
        sums = _alloc(l * sub, torch.float64, dev)
        counts = _alloc(l, torch.int32, dev)
        own = _alloc(n, torch.float64, dev)
        ws_bytes = int(lib.pqk_train_workspace_bytes(n, sub))
        ws = _empty(ws_bytes, dev)
        stats = torch.zeros(STATS_LEN, dtype=torch.int64, device=dev)
        rws_bytes = int(lib.pqk_repair_workspace_bytes(n, l))
        rws = _empty(rws_bytes, dev)
        keys = torch.empty(l, dtype=torch.int64, device=dev)
        index = torch.empty(l, dtype=torch.int64, device=dev)
        for mm in range(m):
            idx = rng.choice(n, size=l, replace=False)
            centers = torch.from_numpy(vectors[idx, mm * sub : (mm + 1) * sub].astype(np.float64)).to(dev).contiguous()
            for _ in range(iterations):
                call("pqk_train_step_device", _ptr(x), n, d, mm * sub, sub, _ptr(centers), l, _ptr(labels), _ptr(sums),
                     _ptr(counts), _ptr(own), _ptr(ws), ws_bytes, _ptr(stats), s)
                e = int(stats[_lib.STAT_EMPTY].item())
                if e:
                    # pq.py:145-151: empty slots (ascending) take the farthest points
                    call("pqk_repair_candidates_device", _ptr(own), n, 0, e, _ptr(rws), rws_bytes, _ptr(keys),
                         _ptr(index), s)
                    slots = torch.from_numpy(np.flatnonzero(counts.cpu().numpy() == 0)).to(dev)
                    far = index[:e]
                    centers[slots] = x[far, mm * sub : (mm + 1) * sub].double()
            books[mm] = centers.cpu().numpy().astype(np.float32)
    return books


def encode_device(vec_dev, cw_dev, m: int, l: int, dev, stride: int | None = None, stats=None):
    n, d = int(vec_dev.shape[0]), int(vec_dev.shape[1])
    stride = m if stride is None else stride
    out = _alloc((n, stride), torch.uint8, dev)
    st = stats if stats is not None else _alloc(STATS_LEN, torch.int64, dev, zero=True)
    if n:
        call("pqk_encode_device", _ptr(vec_dev), n, d, _ptr(cw_dev), m, l, _ptr(out), stride, _ptr(st), _stream(dev))
    return out


# ---------------------------------------------------------------------------
# original-space evaluation (baselines.py:26-37, 385-413)
def cluster_means_device(x_dev: "torch.Tensor", labels_dev: "torch.Tensor", k: int, dev,
                         counts_dev: "torch.Tensor | None" = None) -> "torch.Tensor":
    """(K, D) float64 means of float32/float64 rows grouped by int32 labels in [0, k)."""
    n, d = int(x_dev.shape[0]), int(x_dev.shape[1])
    dtype = 0 if x_dev.dtype == torch.float32 else 1
    means = torch.empty((k, d), dtype=torch.float64, device=dev)
    ws = _empty(_lib.load().pqk_cluster_means_workspace_bytes(n, k), dev)
    call("pqk_cluster_means_device", _ptr(x_dev), dtype, n, d, _ptr(labels_dev), k, _ptr(means), _ptr(counts_dev),
         _ptr(ws), ws.numel(), _stream(dev))
    return means


def assigned_sq_device(x_dev: "torch.Tensor", centers_dev: "torch.Tensor", labels_dev: "torch.Tensor", dev):
    """(N,) float64 np.sum((x - centers[labels])**2, axis=1) in numpy's order."""
    n, d = int(x_dev.shape[0]), int(x_dev.shape[1])
    dtype = 0 if x_dev.dtype == torch.float32 else 1
    sq = torch.empty(n, dtype=torch.float64, device=dev)
    call("pqk_assigned_sq_device", _ptr(x_dev), dtype, n, d, _ptr(centers_dev), _ptr(labels_dev), _ptr(sq),
         _stream(dev))
    return sq


def original_space_error_device(x_dev: "torch.Tensor", labels_dev: "torch.Tensor", k: int, dev) -> float:
    means = cluster_means_device(x_dev, labels_dev, k, dev)
    sq = assigned_sq_device(x_dev, means, labels_dev, dev)
    return mean_objectives(sq, int(x_dev.shape[0]), dev)[0]


def build_tables_host(codewords: np.ndarray, *, device=None) -> np.ndarray:
    """(M, L, L) float64 DistanceTables of (M, L, dsub) float32 codewords, computed on the GPU."""
    cw = np.ascontiguousarray(codewords, dtype=np.float32)
    m, l, dsub = cw.shape
    dev = device_of(device)
    with torch.cuda.device(dev):
        cw_dev = torch.from_numpy(np.array(cw)).to(dev)
        t = torch.empty((m, l, l), dtype=torch.float64, device=dev)
        call("pqk_build_tables_device", _ptr(cw_dev), m, l, dsub, _ptr(t), _stream(dev))
        return t.cpu().numpy()
