"""Test configuration: markers, import paths, shared helpers.

`-m "not gpu"` runs the CPU suite (oracle pins, C-ABI symbol checks, host
logic); `-m gpu` runs the device parity suite through the C-ABI on a B200.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_1603_01876_b200", "python"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libprg.so")
    config.addinivalue_line("markers", "slow: full-size (BASELINE-scale) property checks")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def rel_l1(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def canonical(uv):
    """Reference test canonicalizer sorted_fully (tests/helpers.hpp:29-34)."""
    uv = np.asarray(uv).reshape(-1, 2)
    return uv[np.lexsort((uv[:, 1], uv[:, 0]))]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
