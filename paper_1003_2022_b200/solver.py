"""Covariance -> scale-vector mapping, host side (numpy, vectorised).

The hot path consumes per-pixel scale-vectors either directly (the
reference's (H, W, 4) field) or through the reference's lookup table,
which the device evaluates fused into the filter kernel
(``rubs_b200_filter_params``).  The table itself is built here once per
process, the same way the reference builds it:

* ``optimize_scale_vector``  kurtosis moment matching, closed-form cubic +
                             one Newton polish per root, candidates
                             {t_lo, t_hi, roots}, ties to the smallest t
                             (reference: pkg/src/rubs/solver.py:93-200)
* ``build_lut``              n_rho x n_phi unit-size table, rho geometric on
                             [1, rho_max], phi cell-centred on [0, pi/4)
                             (solver.py:250-281)
* ``ScaleLut``               the table (solver.py:232-247)

Unlike the reference this solver is vectorised over any number of
covariances, so a per-pixel exact field (BASELINE config 1) costs
milliseconds instead of seconds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .geometry import covariance_from_params

_DIR = np.array([1.0, -1.0, 1.0, -1.0])


class Infeasible(ValueError):
    """No positive scale-vector reproduces the covariance (solver.py:64-78)."""


class OutOfGrid(ValueError):
    """Lookup parameters outside the table grid (solver.py:81-82)."""


@dataclass(frozen=True)
class ScaleLut:
    rho_grid: np.ndarray
    phi_grid: np.ndarray
    entries: np.ndarray

    @property
    def rho_max(self) -> float:
        return float(self.rho_grid[-1])


def _cov_parts(c):
    c = np.asarray(c, dtype=np.float64)
    if c.shape[-2:] != (2, 2):
        raise ValueError(f"covariance must be 2x2, got shape {c.shape}")
    if not np.isfinite(c).all():
        raise ValueError("covariance entries must be finite")
    c11, c12, c21, c22 = c[..., 0, 0], c[..., 0, 1], c[..., 1, 0], c[..., 1, 1]
    if (np.abs(c12 - c21) > 1e-12 * (np.abs(c12) + np.abs(c21) + 1.0)).any():
        raise ValueError("covariance must be symmetric")
    tr = c11 + c22
    det = c11 * c22 - c12 * c21
    if ((tr <= 0.0) | (c11 <= 0.0) | (c22 <= 0.0) | (det <= 1e-12 * tr * tr)).any():
        raise ValueError("covariance must be positive definite")
    return c11, c12, c22


def _line(c11, c12, c22, eps):
    """Squared scales p(t) = base + t (1,-1,1,-1) meeting the covariance."""
    k1, k2, k3 = 24.0 * c11, 24.0 * c12, 24.0 * c22
    base = np.stack([0.5 * (k1 - k2 - 2.0), k2 + 1.0, 0.5 * (k3 - k2 - 2.0),
                     np.ones_like(k1)], axis=-1)
    lo = np.maximum(-base[..., 0], -base[..., 2]) + eps
    hi = np.minimum(base[..., 1], base[..., 3]) - eps
    return base, lo, hi


def _objective(base, t):
    p = base + t[..., None] * _DIR
    q = p * p
    return (q * q).sum(axis=-1) + (q[..., 0] + q[..., 2]) * (q[..., 1] + q[..., 3])


def _stationary_points(base):
    """Real roots of d/dt objective (a cubic), each Newton-polished once."""
    b1, b2, b3, b4 = (base[..., k] for k in range(4))
    al, be = b1 + b3, b2 + b4
    z3 = 32.0
    z2 = 24.0 * (b1 - b2 + b3 - b4)
    z1 = 16.0 * (b1 * b1 + b2 * b2 + b3 * b3 + b4 * b4) - 8.0 * al * be
    z0 = (4.0 * (b1 ** 3 - b2 ** 3 + b3 ** 3 - b4 ** 3)
          + 2.0 * al * (b2 * b2 + b4 * b4) - 2.0 * be * (b1 * b1 + b3 * b3))
    B, C, D = z2 / z3, z1 / z3, z0 / z3
    p = C - B * B / 3.0
    q = 2.0 * B ** 3 / 27.0 - B * C / 3.0 + D
    shift = -B / 3.0
    disc = (q / 2.0) ** 2 + (p / 3.0) ** 3
    roots = np.full(base.shape[:-1] + (3,), np.nan)
    one = disc > 0.0
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.sqrt(np.where(one, disc, 0.0))
        s1, s2 = -q / 2.0 + r, -q / 2.0 - r
        cr = lambda x: np.copysign(np.abs(x) ** (1.0 / 3.0), x)  # noqa: E731
        roots[..., 0] = np.where(one, cr(s1) + cr(s2) + shift, np.nan)
        zero_p = (~one) & (p == 0.0)
        roots[..., 0] = np.where(zero_p, shift, roots[..., 0])
        three = (~one) & (p != 0.0)
        m = 2.0 * np.sqrt(np.where(three, -p / 3.0, 1.0))
        arg = np.clip(3.0 * q / (p * m), -1.0, 1.0)
        ph = np.arccos(np.where(three, arg, 0.0)) / 3.0
        for k in range(3):
            val = m * np.cos(ph - 2.0 * math.pi * k / 3.0) + shift
            roots[..., k] = np.where(three, val, roots[..., k])
        # one Newton polish (solver.py:185-188)
        t = roots
        d1 = ((z3 * t + z2[..., None]) * t + z1[..., None]) * t + z0[..., None]
        d2 = (3.0 * z3 * t + 2.0 * z2[..., None]) * t + z1[..., None]
        roots = np.where(d2 != 0.0, t - d1 / np.where(d2 != 0.0, d2, 1.0), t)
    return roots


def optimize_line_position(c, eps: float = 1e-6):
    """(base, t_lo, t_hi, t0) for one or many covariances."""
    c11, c12, c22 = _cov_parts(c)
    base, lo, hi = _line(c11, c12, c22, eps)
    if (lo > hi).any():
        raise Infeasible("elongation exceeds the reachable bound at this orientation")
    roots = _stationary_points(base)
    ok = (roots >= lo[..., None] - 1e-10) & (roots <= hi[..., None] + 1e-10)
    roots = np.clip(roots, lo[..., None], hi[..., None])
    cand = np.concatenate([lo[..., None], hi[..., None], roots], axis=-1)
    valid = np.concatenate([np.ones(lo.shape + (2,), bool), ok & np.isfinite(roots)], axis=-1)
    cand = np.where(valid, cand, np.inf)
    order = np.argsort(cand, axis=-1, kind="stable")
    cand = np.take_along_axis(cand, order, axis=-1)
    vals = np.where(np.isfinite(cand), _objective(base[..., None, :], np.where(np.isfinite(cand), cand, 0.0)), np.inf)
    t0 = np.take_along_axis(cand, np.argmin(vals, axis=-1)[..., None], axis=-1)[..., 0]
    return base, lo, hi, t0


def optimize_scale_vector(c, eps: float = 1e-6) -> np.ndarray:
    """Scale-vector(s) realising covariance(s) c with minimal kurtosis norm."""
    base, _, _, t0 = optimize_line_position(c, eps)
    return np.sqrt(base + t0[..., None] * _DIR)


def build_lut(n_rho: int = 64, n_phi: int = 64, rho_max: float = 5.8, eps: float = 1e-6,
              check_tol: float = 1e-9) -> ScaleLut:
    if n_rho < 2 or n_phi < 2:
        raise ValueError("grid needs at least 2 points per axis")
    if not 1.0 < rho_max < 3.0 + 2.0 * math.sqrt(2.0):
        raise ValueError("rho_max must lie in (1, 3 + 2*sqrt(2))")
    rho_grid = np.exp(np.linspace(0.0, math.log(rho_max), n_rho))
    rho_grid[0] = 1.0
    phi_grid = (np.arange(n_phi) + 0.5) * (0.25 * math.pi / n_phi)
    R, PH = np.meshgrid(rho_grid, phi_grid, indexing="ij")
    target = covariance_from_params(np.ones_like(R), R, PH)
    entries = optimize_scale_vector(target, eps)
    sq = entries * entries
    got = np.empty_like(target)
    got[..., 0, 0] = (2.0 * sq[..., 0] + sq[..., 1] + sq[..., 3]) / 24.0
    got[..., 1, 1] = (2.0 * sq[..., 2] + sq[..., 1] + sq[..., 3]) / 24.0
    got[..., 0, 1] = got[..., 1, 0] = (sq[..., 1] - sq[..., 3]) / 24.0
    err = np.linalg.norm(got - target, axis=(-2, -1)) / np.linalg.norm(target, axis=(-2, -1))
    if (err > check_tol).any():
        raise RuntimeError(f"LUT covariance error {err.max():.3e} exceeds {check_tol:.1e}")
    return ScaleLut(rho_grid, phi_grid, np.ascontiguousarray(entries))


_DEFAULT = {}


def default_lut() -> ScaleLut:
    """The reference's default 64 x 64, rho_max 5.8 table, built once."""
    if "lut" not in _DEFAULT:
        _DEFAULT["lut"] = build_lut()
    return _DEFAULT["lut"]


# ---------------------------------------------------------------------------
# Table files (the reference's save_lut / load_lut, solver.py:351-395):
# magic "RUBS", then little-endian u32 version 1, n_rho, n_phi, the two grids
# and the entries (n_rho, n_phi, 4) as little-endian f64, orientation
# fastest, components innermost.  Written atomically.

LUT_MAGIC = b"RUBS"
LUT_VERSION = 1


def save_lut(lut: ScaleLut, path) -> None:
    import struct
    from .pgmio import atomic_write_bytes
    rg = np.asarray(lut.rho_grid, dtype="<f8")
    pg = np.asarray(lut.phi_grid, dtype="<f8")
    en = np.ascontiguousarray(lut.entries, dtype="<f8")
    if en.shape != (rg.shape[0], pg.shape[0], 4):
        raise ValueError("table entries must be (n_rho, n_phi, 4)")
    atomic_write_bytes(path, LUT_MAGIC + struct.pack("<III", LUT_VERSION, rg.shape[0], pg.shape[0])
                       + rg.tobytes() + pg.tobytes() + en.tobytes())


def load_lut(path) -> ScaleLut:
    import struct
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < 16 or data[:4] != LUT_MAGIC:
        raise ValueError("not a scale lookup table (bad magic)")
    version, n_rho, n_phi = struct.unpack_from("<III", data, 4)
    if version != LUT_VERSION:
        raise ValueError(f"unsupported table version {version}")
    need = 16 + 8 * (n_rho + n_phi + 4 * n_rho * n_phi)
    if len(data) != need:
        raise ValueError(f"truncated table: {len(data)} bytes, expected {need}")
    vals = np.frombuffer(data, "<f8", (need - 16) // 8, 16).astype(np.float64)
    rho_grid, phi_grid = vals[:n_rho].copy(), vals[n_rho:n_rho + n_phi].copy()
    entries = vals[n_rho + n_phi:].reshape(n_rho, n_phi, 4).copy()
    if (np.diff(rho_grid) <= 0.0).any() or (np.diff(phi_grid) <= 0.0).any():
        raise ValueError("table grids must be strictly increasing")
    if not (np.isfinite(entries).all() and (entries > 0.0).all()):
        raise ValueError("table entries must be positive and finite")
    return ScaleLut(rho_grid, phi_grid, entries)
