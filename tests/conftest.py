"""Test configuration: markers, paths and shared helpers.

`-m "not gpu"` runs here (CPU container): oracle-vs-golden pinning, host
logic, C-ABI symbol/load checks.  `-m gpu` runs on a B200 through gpurun:
the parity tests proper, every one calling through libdvla_b200.so.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")
    # a fresh checkout has no libdvla_b200.so yet: build it (nvcc cross-
    # compiles sm_100a without a GPU; incremental when it exists)
    lib = ROOT / "paper_2605_13276_b200" / "libdvla_b200.so"
    if not lib.exists():
        from paper_2605_13276_b200 import build as _build
        _build.build()


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dev():
    if not cuda_ok():
        pytest.fail("gpu-marked test ran without a CUDA device")
    import torch
    return torch.device("cuda", 0)
