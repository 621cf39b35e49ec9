"""Pin the three-direction (N=3) oracle and host mapping.  CPU only.

The reference has no N=3 filter; its N=3 anchors are the spectral sampler
oracle.synthesize_kernel and geometry.covariance_general / direction_vectors
(golden vectors: tests/golden/make_golden_n3.py).  The exact kernel
(oracle/dense3_oracle.c) must match them to the sampler's own accuracy, and
the numpy row-profile restatement (oracle/port3.py, the algorithm the GPU
runs) must match the exact dense filter to rounding."""

import math

import numpy as np
import pytest

import oracle
from oracle import port3
from conftest import golden, smooth_random_field
from paper_1003_2022_b200 import geometry
from paper_1003_2022_b200.solver import Infeasible


def _grid(n, step):
    x = (np.arange(n) - n // 2) * step
    return np.meshgrid(x, x)  # X1 along columns, X2 along rows


def test_directions_and_covariance_match_reference():
    g = golden("n3_kernels.npz")
    assert np.abs(geometry.direction_vectors(3) - g["directions"]).max() < 1e-15
    for a, cov in zip(g["scales"], g["cov"]):
        assert np.abs(geometry.covariance_general(a) - cov).max() < 1e-13 * np.abs(cov).max()


def test_exact_kernel_matches_reference_spectral_sampler():
    """synthesize_kernel (oracle.py:87-167) folds +-3 alias copies at ~257
    samples per axis: point values good to ~1e-3 of the peak.  The exact
    kernel must sit inside that, everywhere on the grid."""
    g = golden("n3_kernels.npz")
    for a, vals, step in zip(g["scales"], g["values"], g["step"]):
        X1, X2 = _grid(vals.shape[0], step)
        got = oracle.kernel3_values(a, X1, X2)
        ref = vals.astype(np.float64)
        assert np.abs(got - ref).max() < 2e-3 * ref.max()
        # and far tighter on average (the sampler's ripple alternates sign)
        assert np.abs(got - ref).mean() < 1e-4 * ref.max()


def test_exact_kernel_mass_and_moments():
    """Unit mass and covariance sum a_k^2/12 u_k u_k^T, by quadrature of the
    exact (piecewise-linear) kernel on a fine grid."""
    for a in ([3.0, 4.0, 5.0], [6.0, 1.5, 2.5], [2.0, 7.0, 1.0]):
        a = np.array(a)
        step = 0.01
        ext = 0.5 * a[0] + 0.25 * (a[1] + a[2]) + 0.5
        x = np.arange(-ext, ext + step / 2, step)
        X1, X2 = np.meshgrid(x, x)
        v = oracle.kernel3_values(a, X1, X2)
        w = step * step
        assert abs(v.sum() * w - 1.0) < 2e-4
        cov = np.array([[(v * X1 * X1).sum(), (v * X1 * X2).sum()],
                        [(v * X1 * X2).sum(), (v * X2 * X2).sum()]]) * w
        ref = geometry.covariance_general(a)
        assert np.abs(cov - ref).max() < 2e-3 * np.abs(ref).max()


def test_kernel_is_centrally_symmetric_and_supported(rng):
    a = np.array([4.3, 2.2, 6.1])
    x1 = rng.uniform(-8, 8, 4000)
    x2 = rng.uniform(-8, 8, 4000)
    assert np.abs(oracle.kernel3_values(a, x1, x2) - oracle.kernel3_values(a, -x1, -x2)).max() < 1e-15
    hx = 0.5 * a[0] + 0.25 * (a[1] + a[2])
    hy = 0.25 * math.sqrt(3.0) * (a[1] + a[2])
    out = (np.abs(x1) > hx) | (np.abs(x2) > hy)
    assert (oracle.kernel3_values(a, x1[out], x2[out]) == 0.0).all()


@pytest.mark.parametrize("iterations", [1, 2])
def test_port_matches_exact_dense(rng, iterations):
    """Row-profile restatement (the GPU's algorithm) == exact dense filter,
    floored widths included."""
    f = rng.random((37, 45))
    field = rng.uniform(0.0, 9.0, (37, 45, 3))
    field[3, 4] = [0.01, 5.0, 5.0]
    ref = oracle.dense3(f, field, iterations)
    got = port3.filter3(f, field, iterations)
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()


def test_port_uniform_and_smooth_field(rng):
    f = rng.random((40, 33))
    got = port3.filter3(f, np.array([3.0, 2.0, 5.0]))
    assert np.abs(got - oracle.dense3(f, np.array([3.0, 2.0, 5.0]))).max() < 1e-12
    s = smooth_random_field(rng, (40, 33), 2.0, 40.0)
    field = port3.scales3_from_params(s, np.full_like(s, 1.5), np.full_like(s, 0.4))
    assert np.abs(port3.filter3(f, field) - oracle.dense3(f, field)).max() < 1e-12


def test_points_equal_dense(rng):
    f = rng.random((30, 26))
    field = rng.uniform(0.5, 7.0, (30, 26, 3))
    pts = np.array([[0, 0], [29, 25], [15, 3], [7, 20]])
    ref = oracle.dense3(f, field)
    assert np.abs(oracle.points3(f, field, pts) - ref[pts[:, 0], pts[:, 1]]).max() < 1e-14


def test_host_mapping_matches_linear_solve(rng):
    """Closed-form N=3 mapping (product host code) == numpy linear solve of
    covariance_general (oracle), and reproduces covariance_from_params."""
    n = 2000
    th = rng.uniform(0.0, math.pi, n)
    bound = geometry.elongation_bound3(th)
    rho = 1.0 + (np.minimum(bound, 50.0) - 1.0) * rng.uniform(0.0, 0.999, n)
    s = rng.uniform(0.1, 5000.0, n)
    a = geometry.scales3_from_params(s, rho, th)
    b = port3.scales3_from_params(s, rho, th)
    assert np.abs(a - b).max() <= 1e-9 * np.abs(b).max()
    cov = geometry.covariance_general(a)
    ref = geometry.covariance_from_params(s, rho, th)
    assert np.abs(cov - ref).max() <= 1e-12 * s.max()


def test_elongation_bound3_known_values():
    th = np.array([0.0, math.pi / 6, math.pi / 4, math.pi / 3, math.pi / 2, 5 * math.pi / 6])
    b = geometry.elongation_bound3(th)
    assert b[0] == np.inf and b[3] > 1e12
    assert abs(b[1] - 3.0) < 1e-12 and abs(b[4] - 3.0) < 1e-12 and abs(b[5] - 3.0) < 1e-12
    assert abs(b[2] - (2.0 + math.sqrt(3.0))) < 1e-12
    # the bound is where the mapping stops being feasible
    for t in (0.2, 0.5, 1.0, 1.4, 2.2, 2.9):
        u = geometry.elongation_bound3(t)
        geometry.scales3_from_params(10.0, u * (1 - 1e-9), t)
        with pytest.raises(Infeasible):
            geometry.scales3_from_params(10.0, u * (1 + 1e-6), t)
