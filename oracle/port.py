"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference fast path.

This module is the CPU "port" of the reference algorithm.  It exists for
two jobs and no others:

* the ``cpu_baseline`` leg of ``bench.py`` and ``bench.py --impl
  reference`` (the reference package itself cannot travel to the GPU box),
* a second checker for the GPU path (oracle "B": the same algorithm run on
  crops / small images), next to the exact dense oracle in
  ``dense_oracle.c``.

Nothing in ``paper_1003_2022_b200`` may import it.  It is pinned against
golden vectors produced by the real reference (tests/golden/make_golden.py).

Algorithm restated (citations are /root/reference/pkg/src/rubs/...):

* ``preintegrate``      engine.py:145-201  (canvas geometry 169-180,
                        four sweeps 186-193, 2^53 guard 195-200)
* ``interpolate``       zp.py:186-228      (7-tap quadratic, clamped reads)
* ZP table              zp.py:89-137 fits it numerically; the exact dyadic
                        values (multiples of 1/8) are hard-coded here
* ``apply_mesh``        engine.py:219-244  (16 vertices, signs, weight)
* ``read_margins``      engine.py:247-262
* ``filter_space_variant`` engine.py:265-324 (floor, 1/sqrt(m), passes)
* ``lookup_many``       solver.py:289-335
"""

from __future__ import annotations

import math

import numpy as np

SQRT2 = math.sqrt(2.0)
SCALE_FLOOR = 0.05
GUARD = float(2 ** 53)

# --- ZP table --------------------------------------------------------------
# Per partition q: seven (dx, dy) offsets, (0, 0) first then lexicographic,
# and the coefficients of (1, d1, d2, d1^2, d1*d2, d2^2) in units of 1/8.
_ZP_ROWS = {
    0: [((0, 0), (4, 0, 0, -4, 0, -4)), ((-1, 0), (1, 4, 0, 4, 0, 0)),
        ((0, -1), (1, 0, 4, -2, 4, 2)), ((0, 1), (1, 0, -4, -2, -4, 2)),
        ((1, -1), (0, 0, 0, 2, -4, 2)), ((1, 0), (1, -4, 0, 0, 0, -4)),
        ((1, 1), (0, 0, 0, 2, 4, 2))],
    1: [((0, 0), (4, 0, 0, -4, 0, -4)), ((-1, 0), (1, 4, 0, 2, 4, -2)),
        ((-1, 1), (0, 0, 0, 2, -4, 2)), ((0, -1), (1, 0, 4, 0, 0, 4)),
        ((0, 1), (1, 0, -4, -4, 0, 0)), ((1, 0), (1, -4, 0, 2, -4, -2)),
        ((1, 1), (0, 0, 0, 2, 4, 2))],
    2: [((0, 0), (4, 0, 0, -4, 0, -4)), ((-1, -1), (0, 0, 0, 2, 4, 2)),
        ((-1, 0), (1, 4, 0, 2, -4, -2)), ((0, -1), (1, 0, 4, -4, 0, 0)),
        ((0, 1), (1, 0, -4, 0, 0, 4)), ((1, -1), (0, 0, 0, 2, -4, 2)),
        ((1, 0), (1, -4, 0, 2, 4, -2))],
    3: [((0, 0), (4, 0, 0, -4, 0, -4)), ((-1, -1), (0, 0, 0, 2, 4, 2)),
        ((-1, 0), (1, 4, 0, 0, 0, -4)), ((-1, 1), (0, 0, 0, 2, -4, 2)),
        ((0, -1), (1, 0, 4, -2, -4, 2)), ((0, 1), (1, 0, -4, -2, 4, 2)),
        ((1, 0), (1, -4, 0, 4, 0, 0))],
}
ZP_OFFSETS = np.array([[o for o, _ in _ZP_ROWS[q]] for q in range(4)], dtype=np.int64)
ZP_COEFFS = np.array([[c for _, c in _ZP_ROWS[q]] for q in range(4)], dtype=np.float64) / 8.0

# Vertex bit patterns: bit k of i says whether width k enters vertex i.
VERTEX_BITS = ((np.arange(16)[:, None] >> np.arange(4)[None, :]) & 1).astype(np.float64)
VERTEX_SIGNS = np.where(VERTEX_BITS.sum(axis=1) % 2 == 0, 1.0, -1.0)


def load_table_dump(text):
    """Coefficients (4, 7, 6) from zp.dump_polynomial_table() text, in this
    module's offset order."""
    out = ZP_COEFFS.copy()
    for ln in text.splitlines()[1:]:
        v = ln.split()
        q, dx, dy = int(v[0]), int(v[1]), int(v[2])
        j = [tuple(o) for o in ZP_OFFSETS[q]].index((dx, dy))
        out[q, j] = [float(t) for t in v[3:]]
    return out


def _quad(c, d1, d2):
    return c[0] + d1 * (c[1] + c[3] * d1 + c[4] * d2) + d2 * (c[2] + c[5] * d2)


def partition(d1, d2):
    return 2 * (np.asarray(d1 + d2) >= 0.0).astype(np.int64) + (np.asarray(d1 - d2) >= 0.0)


def interpolate(plane, col0, row0, x1, x2, coeffs=None):
    """F(x) = sum_n plane[n] Z(x - n), reads clamped to the plane edge.
    ``coeffs`` overrides the exact dyadic table (e.g. with the reference's
    least-squares fit, to reproduce its rounding)."""
    table = ZP_COEFFS if coeffs is None else coeffs
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    shape = np.broadcast_shapes(x1.shape, x2.shape)
    xa = np.broadcast_to(x1, shape).reshape(-1)
    ya = np.broadcast_to(x2, shape).reshape(-1)
    rows, cols = plane.shape
    flat = plane.reshape(-1)
    n1 = np.floor(xa + 0.5).astype(np.int64)
    n2 = np.floor(ya + 0.5).astype(np.int64)
    d1 = n1 - xa
    d2 = n2 - ya
    q = partition(d1, d2)
    res = np.empty(xa.shape)
    for p in range(4):
        idx = np.flatnonzero(q == p)
        if idx.size == 0:
            continue
        e1, e2 = d1[idx], d2[idx]
        cb, rb = n1[idx] - col0, n2[idx] - row0
        acc = np.zeros(idx.size)
        for j in range(7):
            dx, dy = ZP_OFFSETS[p, j]
            cc = np.clip(cb + dx, 0, cols - 1)
            rr = np.clip(rb + dy, 0, rows - 1)
            acc += _quad(table[p, j], e1, e2) * flat[rr * cols + cc]
        res[idx] = acc
    return res.reshape(shape)


def preintegrate(f, col0=0, row0=0, need_cols=None, need_rows=None, guard=True):
    """Four running-sum sweeps on the reference canvas.  Returns
    (plane, c_lo, r_lo) with plane[r, c] at lattice (c_lo + c, r_lo + r)."""
    f = np.asarray(f, dtype=np.float64)
    if f.ndim != 2:
        raise ValueError("image must be 2-D")
    h, w = f.shape
    if need_cols is None:
        need_cols = (col0 - 2, col0 + w + 1)
    if need_rows is None:
        need_rows = (row0 - 2, row0 + h + 1)
    c_lo = min(int(need_cols[0]), col0)
    r_lo = min(int(need_rows[0]), row0 - 1)
    r_hi = max(int(need_rows[1]), row0 + h - 1)
    c_hi = max(int(need_cols[1]), col0 + w - 1) + (r_hi - row0) + 1
    plane = np.zeros((r_hi - r_lo + 1, c_hi - c_lo + 1))
    plane[row0 - r_lo:row0 - r_lo + h, col0 - c_lo:col0 - c_lo + w] = f
    g = plane[row0 - r_lo:]
    np.cumsum(g, axis=1, out=g)
    g *= SQRT2
    for r in range(1, g.shape[0]):
        g[r, 1:] += g[r - 1, :-1]
    np.cumsum(g, axis=0, out=g)
    g *= SQRT2
    for r in range(1, g.shape[0]):
        g[r, :-1] += g[r - 1, 1:]
    if guard:
        peak = float(np.abs(g).max()) if g.size else 0.0
        if peak >= GUARD:
            raise OverflowError(f"running sums reached {peak:.3e}, beyond 2^53")
    return plane, c_lo, r_lo


def mesh_pieces(field):
    a1, a2, a3, a4 = (field[..., k] for k in range(4))
    p2 = a2 / SQRT2
    p4 = a4 / SQRT2
    t1 = 0.5 * a1 + 0.5 * (p2 - p4) - 0.5
    t2 = 0.5 * a3 + 0.5 * (p2 + p4) - 1.5
    w = 1.0 / (a1 * a2 * a3 * a4)
    return a1, a3, p2, p4, t1, t2, w


def apply_mesh(plane, c_lo, r_lo, field, cols, rows, coeffs=None):
    a1, a3, p2, p4, t1, t2, w = mesh_pieces(field)
    xb = cols[None, :] + t1
    yb = rows[:, None] + t2
    acc = np.zeros(field.shape[:2])
    for i in range(16):
        b1, b2, b3, b4 = VERTEX_BITS[i]
        acc += VERTEX_SIGNS[i] * interpolate(
            plane, c_lo, r_lo, xb - (b1 * a1 + b2 * p2 - b4 * p4), yb - (b2 * p2 + b3 * a3 + b4 * p4),
            coeffs)
    return acc * w


def read_margins(field):
    a1, a3, p2, p4, t1, t2, _ = mesh_pieces(field)
    left = max(0, math.ceil(-float((t1 - a1 - p2).min())) + 2)
    right = max(0, math.ceil(float((t1 + p4).max())) + 2)
    below = max(0, math.ceil(-float((t2 - a3 - p2 - p4).min())) + 2)
    above = max(0, math.ceil(float(t2.max())) + 2)
    return left, right, below, above


def prepare_field(field, shape, iterations):
    field = np.asarray(field, dtype=np.float64)
    if field.shape == (4,):
        field = np.broadcast_to(field, (*shape, 4))
    if field.shape != (*shape, 4):
        raise ValueError("scale field shape mismatch")
    if not np.all(np.isfinite(field)):
        raise ValueError("scale field entries must be finite")
    return np.maximum(field, SCALE_FLOOR) / math.sqrt(iterations)


def filter_space_variant(f, field, iterations=1, guard=True, coeffs=None):
    """The reference engine's output (engine.py:265-324), same canvases."""
    f = np.asarray(f, dtype=np.float64)
    if f.ndim != 2:
        raise ValueError("image must be 2-D")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    h, w = f.shape
    fld = prepare_field(field, (h, w), iterations)
    left, right, below, above = read_margins(fld)
    cur, col0, row0 = f, 0, 0
    for p in range(iterations):
        k = iterations - 1 - p
        pc, pr = -k * left, -k * below
        pw, ph = w + k * (left + right), h + k * (below + above)
        fp = np.pad(fld, ((k * below, k * above), (k * left, k * right), (0, 0)), mode="edge")
        plane, c_lo, r_lo = preintegrate(
            cur, col0, row0, (pc - left, pc + pw - 1 + right), (pr - below, pr + ph - 1 + above), guard)
        cur = apply_mesh(plane, c_lo, r_lo, fp,
                         np.arange(pc, pc + pw, dtype=np.float64), np.arange(pr, pr + ph, dtype=np.float64),
                         coeffs)
        col0, row0 = pc, pr
    return cur


def filter_window(f_crop, crop_r0, crop_c0, field_win, r0, c0):
    """One pass, output pixels [r0, r0 + h) x [c0, c0 + w) (h, w = the
    window's field shape) of an image of which ``f_crop`` holds rows
    [crop_r0, ...) x cols [crop_c0, ...) -- the crop must contain every
    pixel the window's kernels read (its own read margins around it; the
    rest of the image is zero as far as the window is concerned).  Exact by
    linearity and zero padding (test_engine.py:115-124).  Only the window's
    pixels are meshed: a halo costs pre-integration only (0.6 % of the
    reference's time per element), so the bands / tiles of the CPU baseline
    do not pay the mesh for their halos."""
    fld = prepare_field(field_win, np.asarray(field_win).shape[:2], 1)
    h, w = fld.shape[:2]
    left, right, below, above = read_margins(fld)
    plane, c_lo, r_lo = preintegrate(f_crop, crop_c0, crop_r0, (c0 - left, c0 + w - 1 + right),
                                     (r0 - below, r0 + h - 1 + above), guard=False)
    return apply_mesh(plane, c_lo, r_lo, fld, np.arange(c0, c0 + w, dtype=np.float64),
                      np.arange(r0, r0 + h, dtype=np.float64))


def filter_band(f, field, row_lo, row_hi, iterations=1):
    """Rows [row_lo, row_hi) of the filtered image (the reference's output
    with the band's own canvases; exact by linearity and zero padding,
    reference tests test_engine.py:175-184); used to run the CPU baseline on
    independent row bands.  One pass: ``filter_window`` on the band.  Two
    passes: pass 1 on the rows of the extended domain the band's pass 2
    reads (edge-clamped field, engine.py:295-323), then pass 2 on the band;
    only pass 1's halo rows are extra mesh work."""
    f = np.asarray(f, dtype=np.float64)
    h, w = f.shape
    field = np.asarray(field, dtype=np.float64)
    if field.shape == (4,):
        field = np.broadcast_to(field, (h, w, 4))
    if iterations == 1:
        fld = prepare_field(field[row_lo:row_hi], (row_hi - row_lo, w), 1)
        _, _, below, above = read_margins(fld)
        lo, hi = max(0, row_lo - below), min(h, row_hi + above)
        return filter_window(f[lo:hi], lo, 0, field[row_lo:row_hi], row_lo, 0)
    if iterations != 2:
        return filter_space_variant(f, field, iterations, guard=False)[row_lo:row_hi]
    fld = prepare_field(field, (h, w), 2)
    left, right, below, above = read_margins(fld)  # whole-field margins, as the reference
    p_lo, p_hi = row_lo - below, row_hi + above  # pass-1 rows the band reads
    pc, pw = -left, w + left + right
    rows1 = np.arange(p_lo, p_hi)
    cols1 = np.arange(pc, pc + pw)
    fp = fld[np.clip(rows1, 0, h - 1)][:, np.clip(cols1, 0, w - 1)]
    lo, hi = max(0, p_lo - below), min(h, p_hi + above)
    plane, c_lo, r_lo = preintegrate(f[lo:hi], 0, lo, (pc - left, pc + pw - 1 + right),
                                     (p_lo - below, p_hi - 1 + above), guard=False)
    cur = apply_mesh(plane, c_lo, r_lo, fp, cols1.astype(np.float64), rows1.astype(np.float64))
    plane, c_lo, r_lo = preintegrate(cur, pc, p_lo, (-left, w - 1 + right),
                                     (row_lo - below, row_hi - 1 + above), guard=False)
    return apply_mesh(plane, c_lo, r_lo, fld[row_lo:row_hi], np.arange(w, dtype=np.float64),
                      np.arange(row_lo, row_hi, dtype=np.float64))


def lookup_many(rho_grid, phi_grid, entries, size, elongation, orientation):
    """Bilinear LUT lookup with quarter-turn fold (solver.py:289-335)."""
    size = np.asarray(size, dtype=np.float64)
    rho = np.asarray(elongation, dtype=np.float64)
    theta = np.asarray(orientation, dtype=np.float64)
    shape = np.broadcast_shapes(size.shape, rho.shape, theta.shape)
    size, rho, theta = (np.broadcast_to(v, shape) for v in (size, rho, theta))
    rho_max = float(rho_grid[-1])
    if np.any(size <= 0.0) or not np.all(np.isfinite(size)):
        raise ValueError("size must be positive and finite")
    if np.any(rho < 1.0) or not np.all(np.isfinite(rho)):
        raise ValueError("elongation must be >= 1 and finite")
    if np.any((theta < 0.0) | (theta >= math.pi)):
        raise ValueError("orientation must lie in [0, pi)")
    if np.any(rho > rho_max * (1.0 + 1e-12)):
        raise ValueError("elongation beyond table maximum")
    rho = np.minimum(rho, rho_max)
    quarter = 0.25 * math.pi
    q = np.minimum((theta // quarter).astype(np.int64), 3)
    phi = theta - q * quarter
    nr, nph = rho_grid.shape[0], phi_grid.shape[0]
    u = np.clip(np.log(rho) / math.log(rho_max) * (nr - 1), 0.0, nr - 1.0)
    v = np.clip(phi / quarter * nph - 0.5, 0.0, nph - 1.0)
    i0 = np.minimum(u.astype(np.int64), nr - 2)
    j0 = np.minimum(v.astype(np.int64), nph - 2)
    fu = (u - i0)[..., None]
    fv = (v - j0)[..., None]
    e = entries
    mix = (e[i0, j0] * (1.0 - fu) * (1.0 - fv) + e[i0 + 1, j0] * fu * (1.0 - fv)
           + e[i0, j0 + 1] * (1.0 - fu) * fv + e[i0 + 1, j0 + 1] * fu * fv)
    roll = np.array([[(k - s) % 4 for k in range(4)] for s in range(4)])
    out = np.take_along_axis(mix, np.broadcast_to(roll[q], mix.shape), axis=-1)
    return out * np.sqrt(size)[..., None]
