"""Histogram timing at the bench configurations' shard sizes: the cluster-tiled path against
the global-atomic kernel (PQK_HIST_MODE=tiled|atomic, each in a child process), L2 flushed before each
launch.  Prints one JSON line per (config, path) with ms and the algorithmic HBM rate
((M_padded + 4) B read per code + K*M*L*4 B table written)."""

import json
import os
import subprocess
import sys

CASES = {"c2": (1_000_000, 10_000, 4), "c3": (10_000_000, 10_000, 8), "c5": (12_500_000, 100_000, 16),
         "c4": (125_000_000, 100_000, 4)}


def child(name):
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1709_03708_b200 import _lib
    from paper_1709_03708_b200.engine import _ptr, _stream

    n, k, m = CASES[name]
    dev = torch.device("cuda:0")
    mp = _lib.padded_m(m)
    g = torch.Generator(device=dev).manual_seed(1)
    codes = torch.randint(0, 256, (n, mp), dtype=torch.uint8, device=dev, generator=g)
    labels = torch.randint(0, k, (n,), dtype=torch.int32, device=dev, generator=g)
    hist = torch.empty((k, m, 256), dtype=torch.int32, device=dev)
    counts = torch.empty((k,), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    times = []
    for it in range(6):
        flush.fill_(it)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        _lib.call("pqk_histogram_device", _ptr(codes), n, m, 256, _ptr(labels), k, _ptr(hist), _ptr(counts),
                  _stream(dev))
        b.record(s)
        torch.cuda.synchronize(dev)
        times.append(a.elapsed_time(b))
    ms = sorted(times[2:])[len(times[2:]) // 2]
    byts = n * (mp + 4) + k * m * 256 * 4
    assert int(counts.sum()) == n and int(hist.sum(dtype=torch.int64)) == n * m
    print(json.dumps({"case": name, "path": os.environ.get("PQK_HIST_MODE", "auto"),
                      "n": n, "k": k, "m": m, "ms": round(ms, 4), "alg_gbs": round(byts / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1])
    else:
        for name in CASES:
            for mode in ("tiled", "atomic"):
                env = dict(os.environ, PQK_HIST_MODE=mode)
                subprocess.run([sys.executable, __file__, name], env=env, check=False, timeout=600)
