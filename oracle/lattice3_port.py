"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the O(1) "lattice" mode
of the three-direction (N=3) filter: the checker for csrc/rubs_n3_lattice.cu
and the CPU baseline of bench.py's lattice config.  The product package never
imports it.

The paper's O(1) algorithm (eq. keyeqn) needs running sums
along every box direction; 60 and 120 degrees are off the pixel lattice, so
the image must be interpolated.  This mode does it the
way the paper's own relation (link2) suggests: on a lattice that CONTAINS the
three directions -- the triangular lattice p(al, ga) = h (al u1 + ga u3) --
everything after the resampling is exact:

1. f_hex[p] = sum_m f[m] hat((m - p) / h)   (adjoint of linear interpolation
   on the lattice triangles: keeps mass and first moments);
2. G = triple running sum of f_hex along (1, 0), (0, 1), (1, 1) in (al, ga)
   -- the lattice vectors h u1, h u3 and h u2 = h (u1 + u3);
3. F(y) = (h / sin60) Lin[G](y - h u2) is the continuous triple integral of
   the f_hex delta train (the three-direction box spline with unit scales on
   this lattice is the linear "hat" element, centred at h u2);
4. out(n) = 1 / (a1 a2 a3) sum_{s in {+-1}^3} (s1 s2 s3) F(n + sum_k s_k a_k u_k / 2)
   -- the 8-vertex finite difference (FD_mesh with N = 3).

So out(n) = sum_p f_hex[p] beta_a(n)(n - p) exactly: the EXACT N=3 kernel
applied to the resampled image (brute force: oracle.lattice3_points).  The
only approximation against the exact N=3 filter is step 1.

Region: the whole image plus the largest support, one restart; float64 sums
(fine at the small sizes the tests use; the device sums are exact integers).
"""

from __future__ import annotations

import math

import numpy as np

SCALE_FLOOR = 0.05
SIN60 = math.sqrt(3.0) / 2.0
U = np.array([[1.0, 0.0], [0.5, SIN60], [-0.5, SIN60]])  # u1, u2, u3 as (x = column, y = row)


def hat(da, dg):
    m = np.maximum(np.maximum(np.abs(da), np.abs(dg)), np.abs(da - dg))
    return np.maximum(0.0, 1.0 - m)


def splat(f, h, al, ga, r0: int = 0, c0: int = 0):
    """f_hex at lattice indices (al, ga) (broadcast integer arrays); f[0, 0]
    is pixel (r0, c0) of the global lattice, zero outside f."""
    f = np.asarray(f, np.float64)
    H, W = f.shape
    px = h * (al - 0.5 * ga)
    py = SIN60 * h * ga
    cb, rb = np.floor(px).astype(np.int64), np.floor(py).astype(np.int64)
    acc = np.zeros(np.broadcast(al, ga).shape)
    for dr in (0, 1):
        for dc in (0, 1):
            r, c = rb + dr, cb + dc
            ok = (r >= r0) & (r < r0 + H) & (c >= c0) & (c < c0 + W)
            dg = (r - py) / (SIN60 * h)
            da = (c - px) / h + 0.5 * dg
            acc += np.where(ok, f[np.clip(r - r0, 0, H - 1), np.clip(c - c0, 0, W - 1)], 0.0) * hat(da, dg)
    return acc


def support3(a):
    """(rx, ry) per pixel, as dense3_oracle.c support3."""
    rx = np.ceil(0.5 * a[..., 0] + 0.25 * (a[..., 1] + a[..., 2])).astype(np.int64) + 1
    ry = np.ceil(0.5 * SIN60 * (a[..., 1] + a[..., 2])).astype(np.int64) + 1
    return rx, ry


def lattice_pass(cur, r0, c0, a, out_r0, out_c0, h):
    """One lattice-mode pass: output pixels (out_r0 + i, out_c0 + j) for the
    prepared scales a (oh, ow, 3), input canvas cur with cur[0, 0] at global
    pixel (r0, c0)."""
    oh, ow = a.shape[:2]
    if oh == 0 or ow == 0:
        return np.zeros((oh, ow))
    rx, ry = support3(a)
    RX, RY = int(rx.max()) + 2, int(ry.max()) + 2
    gh = SIN60 * h
    g_lo = math.floor((out_r0 - RY) / gh) - 2
    g_hi = math.ceil((out_r0 + oh - 1 + RY) / gh) + 2
    a_lo = math.floor((out_c0 - RX) / h + 0.5 * g_lo) - 2
    a_hi = math.ceil((out_c0 + ow - 1 + RX) / h + 0.5 * g_hi) + 2
    ga = np.arange(g_lo, g_hi + 1)[:, None]
    al = np.arange(a_lo, a_hi + 1)[None, :]
    G = splat(cur, h, al, ga, r0, c0)
    G = np.cumsum(np.cumsum(G, axis=1), axis=0)
    for r in range(1, G.shape[0]):  # diagonal (1, 1): G[ga, al] += G[ga - 1, al - 1]
        G[r, 1:] += G[r - 1, :-1]
    Y, X = np.meshgrid(np.arange(out_r0, out_r0 + oh, dtype=np.float64),
                       np.arange(out_c0, out_c0 + ow, dtype=np.float64), indexing="ij")
    # base position of the pixel in lattice coordinates, shifted by -h u2;
    # integer part + fraction, so that each vertex adds a SMALL offset
    gb = Y / gh - 1.0
    ab = X / h + 0.5 * (Y / gh) - 1.0
    gi, ai = np.floor(gb), np.floor(ab)
    gf, af = gb - gi, ab - ai
    acc = np.zeros((oh, ow))
    for s in np.array(np.meshgrid([1, -1], [1, -1], [1, -1], indexing="ij")).reshape(3, -1).T:
        ox = 0.5 * (s[0] * a[..., 0] * U[0, 0] + s[1] * a[..., 1] * U[1, 0] + s[2] * a[..., 2] * U[2, 0])
        oy = 0.5 * (s[0] * a[..., 0] * U[0, 1] + s[1] * a[..., 1] * U[1, 1] + s[2] * a[..., 2] * U[2, 1])
        og = oy / gh
        oa = ox / h + 0.5 * og
        tg, ta = gf + og, af + oa
        fg, fa = np.floor(tg), np.floor(ta)
        wg, wa = tg - fg, ta - fa
        g0 = (gi + fg).astype(np.int64) - g_lo
        a0 = (ai + fa).astype(np.int64) - a_lo
        G00 = G[g0, a0]
        G11 = G[g0 + 1, a0 + 1]
        low = wa >= wg
        G10 = G[g0, a0 + 1]
        G01 = G[g0 + 1, a0]
        lin = np.where(low, G00 + wa * (G10 - G00) + wg * (G11 - G10),
                       G00 + wg * (G01 - G00) + wa * (G11 - G01))
        acc += np.prod(s) * lin
    return acc * (h / (SIN60 * a[..., 0] * a[..., 1] * a[..., 2]))


def _raw_field(field, shape):
    fld = np.asarray(field, np.float64)
    if fld.shape == (3,):
        fld = np.broadcast_to(fld, (*shape, 3))
    return fld


def lattice3(f, field, h: float = 1.0, iterations: int = 1):
    """The lattice-mode N=3 filter with the semantics of
    filter_space_variant (engine.py:285-324): floor 0.05, then a / sqrt(m)
    for m > 1 passes, intermediate passes on canvases extended by the global
    support with the field edge-clamped."""
    f = np.asarray(f, np.float64)
    H, W = f.shape
    if H == 0 or W == 0:
        return np.zeros((H, W))
    raw = np.maximum(_raw_field(field, (H, W)), SCALE_FLOOR)
    if iterations > 1:
        raw = raw / math.sqrt(iterations)
    rx, ry = support3(raw)
    grx, gry = int(rx.max()), int(ry.max())
    cur, r0, c0 = f, 0, 0
    for p in range(iterations):
        remain = iterations - 1 - p
        orow, ocol = -remain * gry, -remain * grx
        oh, ow = H + 2 * remain * gry, W + 2 * remain * grx
        rr = np.clip(np.arange(orow, orow + oh), 0, H - 1)
        cc = np.clip(np.arange(ocol, ocol + ow), 0, W - 1)
        a = raw[rr[:, None], cc[None, :]]
        cur = lattice_pass(cur, r0, c0, a, orow, ocol, h)
        r0, c0 = orow, ocol
    return cur
