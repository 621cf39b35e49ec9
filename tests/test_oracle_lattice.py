"""The two routes of the N=3 lattice (O(1), interpolated) mode agree on the
CPU: the numpy restatement of the O(1) algorithm (oracle/lattice3_port.py:
splat, triple running sums, 8-vertex finite difference, linear interpolation
on the lattice triangles) and the brute-force sum over lattice points with
the exact N=3 kernel (oracle/dense3_oracle.c rubs_oracle3_lattice_points;
the kernel is pinned to the reference's spectral sampler by
tests/test_oracle_n3.py).  Plus the resampling's defining properties and the
error of the mode against the exact N=3 filter."""

import math

import numpy as np
import pytest

import oracle
from oracle import lattice3_port as lp

SIN60 = math.sqrt(3.0) / 2.0


def _all_pts(H, W):
    return np.array([(r, c) for r in range(H) for c in range(W)])


@pytest.mark.parametrize("h", [1.0, 0.5, 0.75])
def test_port_matches_brute_force(h):
    rng = np.random.default_rng(int(h * 100))
    H, W = 36, 44
    f = rng.random((H, W)) - 0.3
    fld = rng.uniform(0.3, 10.0, (H, W, 3))
    got = lp.lattice3(f, fld, h)
    ref = oracle.lattice3_points(f, fld, _all_pts(H, W), h).reshape(H, W)
    assert np.abs(got - ref).max() < 1e-11 * np.abs(ref).max()


def test_splat_keeps_mass_and_first_moments():
    rng = np.random.default_rng(3)
    f = rng.random((20, 24))
    for h in (1.0, 0.6):
        ga = np.arange(-4, int(22 / (SIN60 * h)) + 4)[:, None]
        al = np.arange(-6, int(26 / h + ga.max() / 2) + 6)[None, :]
        fh = lp.splat(f, h, al, ga)
        assert np.array_equal(fh, oracle.splat3(f, h, al, ga))
        px, py = h * (al - 0.5 * ga), SIN60 * h * ga
        r, c = np.mgrid[0:20, 0:24]
        assert abs(fh.sum() - f.sum()) < 1e-11 * f.sum()
        assert abs((fh * px).sum() - (f * c).sum()) < 1e-10 * (f * c).sum()
        assert abs((fh * py).sum() - (f * r).sum()) < 1e-10 * (f * r).sum()


def test_two_passes_keep_constants_inside():
    """m = 2 (a / sqrt(2) per pass on canvases extended by the support, the
    field edge-clamped): away from the border a constant image stays
    constant up to the resampling's aliasing, which shrinks with h."""
    f = np.ones((40, 48))
    fld = np.array([9.0, 8.0, 10.0])
    errs = []
    for h in (1.0, 0.5):
        two = lp.lattice3(f, fld, h, iterations=2)
        errs.append(np.abs(two[16:24, 18:30] - 1.0).max())
    assert errs[0] < 1e-2 and errs[1] < errs[0], errs


def test_error_against_exact_falls_with_kernel_size():
    """The mode's only approximation is the resampling: its error against the
    exact N=3 filter falls as the kernel grows (white-noise image, the worst
    case: every frequency present)."""
    rng = np.random.default_rng(5)
    f = rng.random((72, 72))
    pts = np.array([(r, c) for r in range(24, 48, 3) for c in range(24, 48, 3)])
    errs = []
    for a in (2.0, 4.0, 8.0, 16.0):
        fld = np.array([a, a, a])
        ex = oracle.points3(f, fld, pts)
        lat = oracle.lattice3_points(f, fld, pts, 1.0)
        errs.append(np.abs(lat - ex).max() / np.abs(ex).max())
    assert all(e1 > e2 for e1, e2 in zip(errs, errs[1:])), errs
    assert errs[-1] < 5e-3
