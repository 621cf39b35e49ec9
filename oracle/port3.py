"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the three-direction
(N=3) filter path, the checker for the GPU's N=3 kernel and the CPU baseline
of bench.py's N=3 config.  The product package never imports it.

The reference has no N=3 filter (PAPER.md:285, 662:
60/120-degree running sums are off the pixel lattice).  What is restated
here is this repo's exact N=3 algorithm, whose reference
anchors are the kernel (geometry.direction_vectors / covariance_general,
geometry.py:76-81, 102-106; oracle.synthesize_kernel, oracle.py:87-167) and
the filter semantics of engine.filter_space_variant (engine.py:265-324:
zero padding, floor 0.05 before the 1/sqrt(m) scaling, edge-clamped field on
iterated canvases).

Row-profile form: the N=3 box spline sliced at height y is, along x, the
box of width a1 convolved with the indicator of the chord [L(y), U(y)] of
the parallelogram spanned by the 60/120-degree boxes, times
K = 2 / (sqrt3 a1 a2 a3).  With S_j(t) = sum_m f[j, m] max(t - m, 0) (the
row's double running sum, piecewise linear between integers),

  out(n) = K sum_d [S(n1 + h - L) - S(n1 + h - U) - S(n1 - h - L) + S(n1 - h - U)],

j = n2 - d, h = a1 / 2, L(d) = max(-a2/2 - d/sqrt3, d/sqrt3 - a3/2),
U(d) = min(a2/2 - d/sqrt3, d/sqrt3 + a3/2), |d| <= (a2 + a3) sqrt3 / 4.
"""

from __future__ import annotations

import math

import numpy as np

SCALE_FLOOR = 0.05
SQRT3 = math.sqrt(3.0)


def scales3_from_params(size, elongation, orientation):
    """(size, elongation, orientation) -> N=3 scales by solving
    C = sum_k a_k^2 / 12 u_k u_k^T (covariance_general, geometry.py:102-106)
    with numpy's linear solver -- independent of the product's closed form.
    Returns (..., 3); NaN where the covariance is out of reach (some
    a_k^2 < 0)."""
    s = np.asarray(size, np.float64)
    r = np.asarray(elongation, np.float64)
    t = np.asarray(orientation, np.float64)
    s, r, t = np.broadcast_arrays(s, r, t)
    big, small = s * r / (1.0 + r), s / (1.0 + r)
    c, sn = np.cos(t), np.sin(t)
    c11 = big * c * c + small * sn * sn
    c22 = big * sn * sn + small * c * c
    c12 = (big - small) * c * sn
    ang = np.arange(3) * (math.pi / 3.0)
    u = np.stack([np.cos(ang), np.sin(ang)], axis=-1)
    A = np.stack([u[:, 0] ** 2, u[:, 1] ** 2, u[:, 0] * u[:, 1]], axis=0) / 12.0  # rows: c11, c22, c12
    rhs = np.stack([c11, c22, c12], axis=-1)
    sq = np.linalg.solve(A, rhs[..., None])[..., 0]
    tol = 1e-12 * s[..., None]
    sq = np.where(sq < -tol, np.nan, np.maximum(sq, 0.0))
    return np.sqrt(sq)


def _prep(field, shape, div):
    fld = np.asarray(field, np.float64)
    if fld.shape == (3,):
        fld = np.broadcast_to(fld, (*shape, 3))
    return np.maximum(fld, SCALE_FLOOR) / div


def _row_S(img, c_lo):
    """S[j, e] = S_j(c_lo - 1 + e), e = 0 .. w + 1 (region-local, restarted
    at column c_lo; zero below it)."""
    h, w = img.shape
    C = np.cumsum(img, axis=1)
    S = np.zeros((h, w + 2))
    S[:, 2:] = np.cumsum(C, axis=1)  # S(c_lo + k + 1) = sum_{m <= k} C[m]
    return S


def _eval(S, rows, t):
    """Piecewise-linear S_j at real local coordinates t (entry units)."""
    k = np.floor(t)
    ki = k.astype(np.int64)
    n = S.shape[1]
    lo = np.clip(ki, 0, n - 1)
    hi = np.clip(ki + 1, 0, n - 1)
    v0 = S[rows, lo]
    v1 = S[rows, hi]
    out = v0 + (t - k) * (v1 - v0)
    out = np.where(ki < 0, 0.0, out)
    # beyond the last entry S is linear with slope C[-1] (no further mass)
    past = ki >= n - 1
    if past.any():
        slope = S[rows, n - 1] - S[rows, n - 2]
        out = np.where(past, S[rows, n - 1] + (t - (n - 1)) * slope, out)
    return out


def pass3(cur, cur_c0, cur_r0, a, pc_lo, pr_lo, pw, ph):
    """One pass: output pixels (pc_lo + x, pr_lo + y), x < pw, y < ph, of
    the image `cur` whose element [r, c] sits at lattice (cur_c0 + c,
    cur_r0 + r); `a` = (ph, pw, 3) floored scaled scales."""
    ch, cw = cur.shape
    S = _row_S(cur, 0)
    a1, a2, a3 = a[..., 0], a[..., 1], a[..., 2]
    K = 2.0 / (SQRT3 * a1 * a2 * a3)
    hy = 0.25 * SQRT3 * (a2 + a3)
    D = int(math.ceil(hy.max())) if hy.size else 0
    ny = (pr_lo + np.arange(ph))[:, None] * np.ones((1, pw), np.int64)
    nx = (pc_lo + np.arange(pw))[None, :] * np.ones((ph, 1), np.int64)
    # local entry coordinate of lattice x: e = x - cur_c0 + 1
    x = (nx - cur_c0 + 1).astype(np.float64)
    h = 0.5 * a1
    acc = np.zeros((ph, pw))
    for d in range(-D, D + 1):
        live = np.abs(d) <= hy
        j = ny - d - cur_r0
        inside = live & (j >= 0) & (j < ch)
        if not inside.any():
            continue
        yd = d / SQRT3
        L = np.maximum(-0.5 * a2 - yd, yd - 0.5 * a3)
        U = np.maximum(np.minimum(0.5 * a2 - yd, yd + 0.5 * a3), L)
        rows = np.clip(j, 0, ch - 1)
        e1 = _eval(S, rows, x + h - L)
        e2 = _eval(S, rows, x + h - U)
        e3 = _eval(S, rows, x - h - L)
        e4 = _eval(S, rows, x - h - U)
        acc += np.where(inside, (e1 - e2) - (e3 - e4), 0.0)
    return K * acc


def support3(a):
    """Global integer support radii (rx, ry) of floored, scaled scales."""
    rx = int(np.ceil(0.5 * a[..., 0] + 0.25 * (a[..., 1] + a[..., 2])).max()) + 1
    ry = int(np.ceil(0.25 * SQRT3 * (a[..., 1] + a[..., 2])).max()) + 1
    return rx, ry


def filter3(f, field, iterations: int = 1):
    """N=3 space-variant filter (iterations passes), numpy."""
    f = np.asarray(f, np.float64)
    H, W = f.shape
    div = math.sqrt(iterations)
    fld = np.asarray(field, np.float64)
    full = _prep(fld, (H, W), div)
    rx, ry = support3(full)
    cur, c0, r0 = f, 0, 0
    for p in range(iterations):
        remain = iterations - 1 - p
        pc_lo, pr_lo = -remain * rx, -remain * ry
        pw, ph = W + 2 * remain * rx, H + 2 * remain * ry
        rr = np.clip(pr_lo + np.arange(ph), 0, H - 1)
        cc = np.clip(pc_lo + np.arange(pw), 0, W - 1)
        a = full[rr][:, cc]
        cur = pass3(cur, c0, r0, a, pc_lo, pr_lo, pw, ph)
        c0, r0 = pc_lo, pr_lo
    return cur


def filter3_band(f, field, lo, hi):
    """One pass, output rows [lo, hi) of the whole-image result, from the
    image rows the band reads (exact by zero padding); bench.py's CPU
    baseline unit of work."""
    f = np.asarray(f, np.float64)
    H, W = f.shape
    a = _prep(np.asarray(field, np.float64)[lo:hi], (hi - lo, W), 1.0)
    _, ry = support3(a)
    r0, r1 = max(0, lo - ry), min(H, hi + ry)
    return pass3(f[r0:r1], 0, r0, a, 0, lo, W, hi - lo)
