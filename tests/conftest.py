"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on the CPU-only build container (oracle, host logic, ABI load)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


@pytest.fixture(scope="session")
def golden_codec():
    return dict(np.load(os.path.join(GOLDEN, "codec.npz")))


@pytest.fixture(scope="session")
def golden_layers():
    return dict(np.load(os.path.join(GOLDEN, "layers.npz")))


@pytest.fixture(scope="session")
def golden_nets():
    return dict(np.load(os.path.join(GOLDEN, "nets.npz")))


@pytest.fixture(scope="session")
def golden_memory():
    with open(os.path.join(GOLDEN, "memory.json")) as f:
        return json.load(f)


def rel_err(got, want, floor=1e-8):
    """Worst-case elementwise relative error with an absolute floor
    (reference tests/conftest.py:76-81)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)))


def norm_err(got, want):
    """Normwise relative error ||got-want|| / ||want|| (0 if both zero)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    d = np.linalg.norm(want.ravel())
    e = np.linalg.norm((got - want).ravel())
    return float(e / d) if d > 0 else float(e)
