import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(GOLDEN / f"{name}.npz")


def golden_camera(z, suffix=""):
    f = z[f"cam_f{suffix}"]
    return SimpleNamespace(
        width=int(z[f"cam_w{suffix}"]), height=int(z[f"cam_h{suffix}"]),
        fx=float(f[0]), fy=float(f[1]), cx=float(f[2]), cy=float(f[3]), c2w=z[f"cam_c2w{suffix}"],
    )


def toy_occupancy_bits():
    z = golden("toy_occupancy_256")
    return z["res"], z["bits"]


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
