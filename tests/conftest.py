"""Shared pytest setup: the `gpu` marker and import paths.

`-m "not gpu"` runs on the CPU container (oracle vs golden vectors, host logic,
C-ABI symbol checks, gloo multi-process tests); `-m gpu` runs the parity tests
through the C-ABI on a B200.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pqk_oracle

    return pqk_oracle


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
