import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def desk_y32():
    """The desk fixture (m=8192, p=64) as float32 signal rows (m, p)."""
    u8 = golden("desk_patches")["u8"]
    return (u8.astype(np.float64) / 255.0).astype(np.float32)


@pytest.fixture(scope="session")
def desk_y64(desk_y32):
    """Reference-layout p x m float64 view of the float32 desk signals."""
    return desk_y32.T.astype(np.float64)
