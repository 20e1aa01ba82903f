"""bench.py as the driver launches it, at N > 1 ranks.

`python bench.py --gpus 2` (no WORLD_SIZE) must relaunch itself under
torch.distributed.run with two ranks and print ONE JSON line with n_gpus = 2, weak
scaling (the job holds 2 x the per-GPU shard) and a zero-mismatch oracle parity record.
The pool has one GPU per call, so the two ranks share cuda:0 over gloo collectives
(PQK_BENCH_BACKEND=gloo): a functional check of the N > 1 path, not a timing.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_relaunch():
    env = dict(os.environ, PQK_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "2", "--warmup", "3",
         "--no-cpu-baseline", "--no-e2e", "--no-extras"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2
    assert out["scaling"] == "weak"
    assert out["config"]["n"] == 2 * 100_000
    assert out["parity"]["mismatch"] == 0
    assert out["value"] > 0
