import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def normrel(a, b, floor=1e-12):
    """Norm-relative error of a against reference b, ignoring entries of b below
    floor * max|b| (FFT-noise-level oracle entries are excluded)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        a = np.stack([np.real(a), np.imag(a)], -1).astype(np.float64)
        b = np.stack([np.real(b), np.imag(b)], -1).astype(np.float64)
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    scale = np.max(np.abs(b)) if b.size else 0.0
    if scale == 0.0:
        return float(np.max(np.abs(a))) if a.size else 0.0
    keep = np.abs(b) >= floor * scale
    return float(np.linalg.norm((a - b)[keep]) / max(np.linalg.norm(b[keep]), 1e-300))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
