"""Second-order geometry needed on the filtering path (host side, numpy).

Only the pieces the hot path and its LUT mapping use are here:

* ``as_scale_vector``        validation of a (4,) scale-vector
                             (reference: pkg/src/rubs/geometry.py:63-73)
* ``covariance_of``          scale-vector -> covariance (geometry.py:84-99)
* ``covariance_from_params`` (size, elongation, orientation) -> covariance
                             (geometry.py:153-172)
* ``elongation_bound``       reachable elongation U(phi), used to clamp rho
                             (geometry.py:175-202; vectorised here)

Three-direction (N=3) kernels (BASELINE.json config 3; no reference filter):

* ``direction_vectors``      unit directions at (k-1) pi / n (geometry.py:76-81)
* ``covariance_general``     sum a_k^2 / 12 u_k u_k^T (geometry.py:102-106)
* ``scales3_from_params``    the unique N=3 scales of a covariance (closed form)
* ``elongation_bound3``      reachable N=3 elongation (3 at 30/90/150 degrees)

Size is the covariance trace (geometry.py:20-21).  BASELINE.json quotes
kernel sizes as a Gaussian ``sigma``; this package maps sigma to
size = 2 sigma^2, the trace of sigma^2 I.
"""

from __future__ import annotations

import math

import numpy as np

MIN_ELONGATION_BOUND = 3.0 + 2.0 * math.sqrt(2.0)


def as_scale_vector(a) -> np.ndarray:
    v = np.asarray(a, dtype=np.float64)
    if v.shape != (4,):
        raise ValueError(f"scale-vector must have shape (4,), got {v.shape}")
    if not (np.isfinite(v).all() and (v > 0.0).all()):
        raise ValueError("scale-vector entries must be finite and positive")
    return v


def covariance_of(a) -> np.ndarray:
    """C = 1/24 [[2a1^2+a2^2+a4^2, a2^2-a4^2], [a2^2-a4^2, 2a3^2+a2^2+a4^2]]."""
    sq = np.square(as_scale_vector(a))
    diag = sq[1] + sq[3]
    off = (sq[1] - sq[3]) / 24.0
    return np.array([[(2.0 * sq[0] + diag) / 24.0, off], [off, (2.0 * sq[2] + diag) / 24.0]])


def sigma_to_size(sigma):
    """Gaussian sigma (BASELINE.json) -> covariance trace (reference size)."""
    return 2.0 * np.square(np.asarray(sigma, dtype=np.float64))


def covariance_from_params(size, elongation, orientation):
    """Covariance with trace ``size``, eigenvalue ratio ``elongation`` and
    major axis at ``orientation``; vectorised, returns (..., 2, 2)."""
    s = np.asarray(size, dtype=np.float64)
    r = np.asarray(elongation, dtype=np.float64)
    th = np.asarray(orientation, dtype=np.float64)
    if not (np.isfinite(s).all() and (s > 0.0).all()):
        raise ValueError("size must be positive and finite")
    if not (np.isfinite(r).all() and (r >= 1.0).all()):
        raise ValueError("elongation must be >= 1")
    if ((th < 0.0) | (th >= math.pi)).any():
        raise ValueError("orientation must lie in [0, pi)")
    big = s * r / (1.0 + r)
    small = s / (1.0 + r)
    co, si = np.cos(th), np.sin(th)
    c11 = big * co * co + small * si * si
    c22 = big * si * si + small * co * co
    c12 = (big - small) * co * si
    out = np.empty(np.broadcast(s, r, th).shape + (2, 2))
    out[..., 0, 0] = c11
    out[..., 1, 1] = c22
    out[..., 0, 1] = c12
    out[..., 1, 0] = c12
    return out


def elongation_bound(phi):
    """U(phi) = (1 + nu + sqrt(1 + nu^2)) / (1 - 1/(nu + sqrt(1 + nu^2))),
    nu = |cot 2 phi|; +inf on the four box directions, 3 + 2 sqrt 2 midway."""
    p = np.asarray(phi, dtype=np.float64)
    if ((p < 0.0) | (p >= math.pi)).any():
        raise ValueError("orientation must lie in [0, pi)")
    s2 = np.sin(2.0 * p)
    with np.errstate(divide="ignore", invalid="ignore"):
        nu = np.abs(np.cos(2.0 * p) / s2)
        root = np.hypot(1.0, nu)
        val = (1.0 + nu + root) / (1.0 - 1.0 / (nu + root))
    val = np.where(np.abs(nu - 1.0) < 4e-16, MIN_ELONGATION_BOUND, val)
    principal = (p == 0.0) | (p == 0.25 * math.pi) | (p == 0.5 * math.pi) | (p == 0.75 * math.pi)
    val = np.where(principal | (s2 == 0.0) | ~np.isfinite(nu), np.inf, val)
    return float(val) if np.ndim(val) == 0 else val


def direction_vectors(n: int) -> np.ndarray:
    """Unit direction vectors (cos, sin) at angles (k-1) pi / n, k = 1..n."""
    if n < 2:
        raise ValueError("need at least two directions")
    ang = np.arange(n) * (math.pi / n)
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1)


def covariance_general(scales) -> np.ndarray:
    """Covariance of an n-direction kernel: sum_k a_k^2 / 12 u_k u_k^T."""
    a = np.asarray(scales, dtype=np.float64)
    u = direction_vectors(a.shape[-1])
    return np.einsum("...k,ki,kj->...ij", a * a / 12.0, u, u)


_INV_SQRT3 = 1.0 / math.sqrt(3.0)


def _n3_coeffs(th):
    """p_k = lam_max alpha_k + lam_min beta_k for the three N=3 squared
    scales / 12 (p1 = C11 - C22/3, p2,3 = 2/3 C22 +- 2/sqrt3 C12)."""
    co, si = np.cos(th), np.sin(th)
    cc, ss, cs = co * co, si * si, co * si
    alpha = np.stack([cc - ss / 3.0, 2.0 / 3.0 * ss + 2.0 * _INV_SQRT3 * cs,
                      2.0 / 3.0 * ss - 2.0 * _INV_SQRT3 * cs], axis=-1)
    beta = np.stack([ss - cc / 3.0, 2.0 / 3.0 * cc - 2.0 * _INV_SQRT3 * cs,
                     2.0 / 3.0 * cc + 2.0 * _INV_SQRT3 * cs], axis=-1)
    return alpha, beta


def scales3_from_params(size, elongation, orientation):
    """The three-direction scales whose covariance (covariance_general) is
    covariance_from_params(size, elongation, orientation); three unknowns for
    three covariance entries, so the solution is unique.  Raises Infeasible
    beyond the N=3 elongation bound (some a_k^2 < 0).  Returns (..., 3).
    Mirrors the device mapping of rubs_b200_filter3_params."""
    from .solver import Infeasible
    cov = covariance_from_params(size, elongation, orientation)
    s = np.asarray(size, dtype=np.float64)
    c11, c22, c12 = cov[..., 0, 0], cov[..., 1, 1], cov[..., 0, 1]
    p = np.stack([c11 - c22 / 3.0, c22 * (2.0 / 3.0) + c12 * (2.0 * _INV_SQRT3),
                  c22 * (2.0 / 3.0) - c12 * (2.0 * _INV_SQRT3)], axis=-1)
    if (p < -1e-12 * np.broadcast_to(s, p.shape[:-1])[..., None]).any():
        raise Infeasible("elongation beyond the three-direction bound at this orientation")
    return np.sqrt(12.0 * np.maximum(p, 0.0))


def elongation_bound3(phi):
    """Largest elongation an N=3 kernel reaches at orientation phi: +inf on
    the box directions (0, 60, 120 degrees), 3 midway (30, 90, 150)."""
    p = np.asarray(phi, dtype=np.float64)
    if ((p < 0.0) | (p >= math.pi)).any():
        raise ValueError("orientation must lie in [0, pi)")
    alpha, beta = _n3_coeffs(p)
    with np.errstate(divide="ignore", invalid="ignore"):
        lim = np.where(alpha < -1e-15, -beta / alpha, np.inf)
    val = lim.min(axis=-1)
    return float(val) if np.ndim(val) == 0 else val
