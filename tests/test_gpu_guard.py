"""Out-of-bounds store check (the pool does not allow compute-sanitizer).

tools/sanitize_fit.py runs every hot kernel of the path on small and mid-size inputs with
PQK_GUARD=1: the engine allocates each buffer a kernel writes between 64 KB guard zones
of 0xA5 and fails if a zone changed; every result is also compared with the oracle.  Run
twice, for the L2-atomic and the cluster-tiled histogram (PQK_HIST_MODE is read once per
process)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("hist_mode", ["atomic", "tiled"])
def test_guard_zones_and_oracle(hist_mode):
    env = dict(os.environ, PQK_GUARD="1", PQK_HIST_MODE=hist_mode)
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_fit.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "SANITIZE_FIT OK" in res.stdout
    assert "guard zones intact" in res.stdout
