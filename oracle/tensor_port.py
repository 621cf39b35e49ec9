"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's
structure-tensor / adaptive smoothing pipeline (pkg/src/rubs/tensor.py).

Used by tests/ (checker for csrc/rubs_tensor.cu) and bench.py's CPU legs;
nothing in ``paper_1003_2022_b200`` may import it.  Pinned against golden
vectors from the real reference (tests/golden/make_golden.py tensor).

The filter steps are pluggable: ``filt(f, field, iterations)`` defaults to
the exact dense oracle (oracle.dense), which makes this the exact pipeline;
``port.filter_space_variant`` gives the reference's own fast path.

Restated (citations are /root/reference/pkg/src/rubs/tensor.py):
  structure_tensor         52-75   (reflect pad, central differences,
                                    isotropic window c = max(ws sqrt 6, 0.05))
  _bound_vectorised        77-86
  anisotropy_from_tensor   90-171  (eigen split, theta, rho cases, clamp,
                                    percentile size map, isotropic fallback)
  adaptive_smooth          174-224 (rho cap, lookup, two filters, gain)
"""

from __future__ import annotations

import math

import numpy as np

EIG_REL, EIG_ABS = 1e-8, 1e-12
SCALE_FLOOR = 0.05


def _dense(f, field, iterations=1):
    import oracle
    return oracle.dense(f, field, iterations)


def structure_tensor(f, window_sigma=1.5, filt=_dense):
    f = np.asarray(f, dtype=np.float64)
    pad = np.pad(f, 1, mode="reflect")
    gx = 0.5 * (pad[1:-1, 2:] - pad[1:-1, :-2])
    gy = 0.5 * (pad[2:, 1:-1] - pad[:-2, 1:-1])
    j = np.stack([gx * gx, gx * gy, gy * gy], axis=-1)
    if window_sigma > 0.0:
        c = max(window_sigma * math.sqrt(6.0), SCALE_FLOOR)
        for k in range(3):
            j[..., k] = filt(j[..., k], np.full(4, c))
    return j


def bound_vectorised(phi):
    s2 = np.sin(2.0 * phi)
    c2 = np.cos(2.0 * phi)
    with np.errstate(divide="ignore"):
        nu = np.abs(c2 / s2)
    root = np.hypot(1.0, nu)
    with np.errstate(invalid="ignore"):
        out = (1.0 + nu + root) / (1.0 - 1.0 / (nu + root))
    return np.where(np.isfinite(nu), out, np.inf)


def anisotropy_from_tensor(j, noise_sigma, size_range=None, bound_fraction=0.95, iso_gain=1.0):
    j = np.asarray(j, dtype=np.float64)
    j11, j12, j22 = j[..., 0], j[..., 1], j[..., 2]
    tr = j11 + j22
    disc = np.hypot(j11 - j22, 2.0 * j12)
    lmax = 0.5 * (tr + disc)
    lmin = 0.5 * (tr - disc)
    thr = EIG_REL * tr + EIG_ABS
    has_major = lmax > thr
    has_minor = lmin > thr
    theta = np.mod(0.5 * np.arctan2(2.0 * j12, j11 - j22) + 0.5 * math.pi, math.pi)
    theta[~has_major] = 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = lmax / lmin
    rho = np.where(has_major & has_minor, ratio, np.where(has_major, np.maximum(1.0, lmax), 1.0))
    rho = np.minimum(rho, bound_fraction * bound_vectorised(theta))
    rho = np.maximum(rho, 1.0)
    if size_range is None:
        size_range = (0.5, 3.0 * noise_sigma * noise_sigma + 0.5)
    s_min, s_max = size_range
    q05, q95 = np.percentile(tr, [5.0, 95.0])
    if q95 - q05 > 1e-300:
        size = s_max + (tr - q05) * (s_min - s_max) / (q95 - q05)
    else:
        size = np.full_like(tr, 0.5 * (s_min + s_max))
    size = np.clip(size, s_min, s_max)
    iso = ~has_major
    sigma_iso = max(iso_gain * noise_sigma * noise_sigma, 1.0)
    size[iso] = sigma_iso * sigma_iso / 3.0
    rho[iso] = 1.0
    return size, rho, theta, iso


def adaptive_smooth(f, noise_sigma, lut, window_sigma=1.5, iterations=1, bound_fraction=0.95,
                    size_range=None, iso_gain=1.0, filt=_dense, j=None):
    """``lut`` = (rho_grid, phi_grid, entries); ``j`` = a structure tensor
    to start from instead of computing one (isolates the later stages)."""
    from oracle import port
    f = np.asarray(f, dtype=np.float64)
    if j is None:
        j = structure_tensor(f, window_sigma, filt)
    size, rho, theta, _ = anisotropy_from_tensor(j, noise_sigma, size_range, bound_fraction, iso_gain)
    rho_grid, phi_grid, entries = lut
    rho = np.minimum(rho, rho_grid[-1] * (1.0 - 1e-9))
    field = port.lookup_many(rho_grid, phi_grid, entries, size, rho, theta)
    out = filt(f, field, iterations)
    gain = filt(np.ones_like(f), field, iterations)
    return np.where(np.abs(gain) > 1e-6, out / np.where(gain == 0.0, 1.0, gain), out)


def stripe_image(shape=(160, 160), period=8.0, angle=0.3, contrast=1.0):
    """oracle.py:351-363 (synthetic oriented stripes in [0, contrast])."""
    h, w = shape
    x1 = np.arange(w, dtype=np.float64)[None, :]
    x2 = np.arange(h, dtype=np.float64)[:, None]
    phase = -math.sin(angle) * x1 + math.cos(angle) * x2
    return (0.5 * contrast) * (np.sin(2.0 * math.pi * phase / period) + 1.0)


def add_gaussian_noise(image, target_psnr_db, peak=1.0, seed=0):
    """oracle.py:366-372 (white noise sized for a target PSNR)."""
    sigma = peak / 10.0 ** (target_psnr_db / 20.0)
    return image + np.random.default_rng(seed).normal(0.0, sigma, size=np.shape(image))


def psnr(reference, estimate, peak=1.0):
    """oracle.py:375-383."""
    mse = float(np.mean((np.asarray(reference, float) - np.asarray(estimate, float)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)
