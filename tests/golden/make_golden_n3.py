"""Golden fixtures for the three-direction (N=3) kernel, generated from the
REAL reference (build container only: it imports /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_n3.py

The reference has no N=3 filter and no exact N=3 evaluator (SURVEY.md §0
fact 6).  What it does have, and what is recorded here:
  rubs.geometry.direction_vectors(3)      (geometry.py:76-81)
  rubs.geometry.covariance_general(a)     (geometry.py:102-106)
  rubs.oracle.synthesize_kernel(a)        (oracle.py:87-167; spectral
      sampler with alias folding -- accurate to ~1e-3 .. 1e-5 of the peak)
  rubs.oracle.uniform_scales(3, sigma)    (oracle.py:74-76)
They pin the exact N=3 kernel of oracle/dense3_oracle.c
(tests/test_oracle_n3.py).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from rubs import geometry, oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    scales = np.array([
        oracle.uniform_scales(3, 2.0),
        [3.0, 4.0, 5.0],
        [6.0, 1.5, 2.5],
        [2.0, 7.0, 1.0],
        oracle.uniform_scales(3, 5.0),
    ])
    vals, steps, covs = [], [], []
    for a in scales:
        # fixed grid size so the fixtures stack: 257 samples per axis
        hx = 0.5 * float(np.sum(a * np.abs(geometry.direction_vectors(3)[:, 0])))
        hy = 0.5 * float(np.sum(a * np.abs(geometry.direction_vectors(3)[:, 1])))
        extent = 1.2 * max(hx, hy)
        step = 2.0 * extent / 256.0
        k = oracle.synthesize_kernel(a, step=step, extent=extent)
        assert k.values.shape == (257, 257), k.values.shape
        vals.append(k.values)
        steps.append(k.step)
        covs.append(geometry.covariance_general(a))
    np.savez_compressed(os.path.join(OUT, "n3_kernels.npz"), scales=scales,
                        values=np.stack(vals).astype(np.float32), step=np.array(steps),
                        cov=np.stack(covs), directions=geometry.direction_vectors(3),
                        uniform_sigma=np.array([2.0, 5.0]),
                        uniform_scales=np.stack([oracle.uniform_scales(3, 2.0),
                                                 oracle.uniform_scales(3, 5.0)]))


if __name__ == "__main__":
    main()
