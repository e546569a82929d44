"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def bits_equal(a, b) -> bool:
    """Bitwise float comparison (-0.0 != +0.0), as pkg/tests/conftest.py:91-97."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def packed(seed, nc=13, cap=7):
    """Packed arrays with per-cell free space (pkg/tests/test_backends.py:21-39)."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, cap + 1, size=nc).astype(np.int64)
    caps = np.full(nc, cap, dtype=np.int64)
    offs = np.concatenate(([0], np.cumsum(caps[:-1]))).astype(np.int64)
    total = int(caps.sum())
    x, vx, vy, yp = np.zeros(total), np.zeros(total), np.zeros(total), np.zeros(total)
    for j in range(nc):
        n = counts[j]
        sl = slice(offs[j], offs[j] + n)
        x[sl] = rng.random(n)
        vx[sl] = rng.standard_normal(n) * 0.3
        vy[sl] = rng.standard_normal(n) * 0.3
        yp[sl] = rng.standard_normal(n)
    return x, vx, vy, yp, offs, counts


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2404_10270_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
