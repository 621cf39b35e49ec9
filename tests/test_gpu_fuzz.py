"""Randomised parity of the large-kernel paths (a short, seeded run of
scripts/fuzz_big.py): images of 1024-2048 px a side, LUT parameter fields
mixing small and huge kernels (sigma up to ~300: primary kernel, stage 2,
shared-memory overflow pass, global-scratch blocks, per-pixel fallback,
streamed host path), one or two passes, float32 / float64 images and
parameters; ~300 sampled pixels per case against the exact per-point GPU
oracle (oracle/dense_oracle_cuda.cu).  Bar: 1e-9 of max |output|."""

import importlib.util
import os

import numpy as np
import pytest

import paper_1003_2022_b200 as rb

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location(
    "fuzz_big", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "fuzz_big.py"))


@pytest.mark.parametrize("seed", [11, 12])
def test_random_large_kernel_fields_match_the_exact_oracle(cuda, seed):
    fuzz = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(fuzz)
    rng = np.random.default_rng(seed)
    lut = rb.default_lut()
    for _ in range(8):
        err, desc = fuzz.run_case(rng, lut, sides=(1024, 1536, 2048), widths=(1024, 1300, 2048))
        assert err < 1e-9, f"{desc}: {err:.3e}"
