"""Shared test helpers.  `gpu` tests need a B200 and the built native
library; everything else runs on CPU (driver: pytest -m "not gpu")."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the native library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def smooth_random_field(rng, shape, lo, hi):
    """Low-frequency random surface in [lo, hi] (bilinear-upsampled normals)."""
    h, w = shape
    coarse = rng.standard_normal((max(h // 8, 2), max(w // 8, 2)))
    ys = np.linspace(0.0, coarse.shape[0] - 1.0, h)
    xs = np.linspace(0.0, coarse.shape[1] - 1.0, w)
    yi = np.minimum(ys.astype(int), coarse.shape[0] - 2)
    xi = np.minimum(xs.astype(int), coarse.shape[1] - 2)
    fy = (ys - yi)[:, None]
    fx = (xs - xi)[None, :]
    surf = (coarse[yi][:, xi] * (1 - fy) * (1 - fx) + coarse[yi][:, xi + 1] * (1 - fy) * fx
            + coarse[yi + 1][:, xi] * fy * (1 - fx) + coarse[yi + 1][:, xi + 1] * fy * fx)
    return lo + (surf - surf.min()) * (hi - lo) / (surf.max() - surf.min())


def impulse(shape, at=None):
    h, w = shape
    f = np.zeros(shape)
    f[at if at is not None else (h // 2, w // 2)] = 1.0
    return f


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
