"""Generate the golden fixtures from the REAL reference (run in the build
container only: it imports /root/reference, which does not exist on the GPU
box).  The fixtures pin the oracle restatement (oracle/) and the host-side
solver; the GPU tests then compare the CUDA path against the pinned oracle.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array here comes out of the reference's public functions:
  rubs._exact.kernel_values   (pkg/src/rubs/_exact.py:29)
  rubs.zp.dump_polynomial_table / interpolate (zp.py:186, 232)
  rubs.engine.filter_space_variant / filter_space_invariant / preintegrate
  rubs.oracle.dense_convolve  (oracle.py:177)
  rubs.solver.build_lut / lookup_many / optimize_scale_vector
  rubs.tensor.structure_tensor / anisotropy_from_tensor / adaptive_smooth
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import rubs  # noqa: E402
from rubs import _exact, engine, oracle, solver, zp  # noqa: E402
from rubs.geometry import covariance_from_params, elongation_bound  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def smooth_random_field(rng, shape, lo, hi):
    # same recipe as the reference tests' conftest helper
    h, w = shape
    coarse = rng.standard_normal((max(h // 8, 2), max(w // 8, 2)))
    ys = np.linspace(0.0, coarse.shape[0] - 1.0, h)
    xs = np.linspace(0.0, coarse.shape[1] - 1.0, w)
    yi = np.minimum(ys.astype(int), coarse.shape[0] - 2)
    xi = np.minimum(xs.astype(int), coarse.shape[1] - 2)
    fy = (ys - yi)[:, None]
    fx = (xs - xi)[None, :]
    surf = (coarse[yi][:, xi] * (1 - fy) * (1 - fx) + coarse[yi][:, xi + 1] * (1 - fy) * fx
            + coarse[yi + 1][:, xi] * fy * (1 - fx) + coarse[yi + 1][:, xi + 1] * fy * fx)
    return lo + (surf - surf.min()) * (hi - lo) / (surf.max() - surf.min())


def kernels(rng):
    A = rng.uniform(0.3, 6.0, size=(24, 4))
    A[0] = [1.0, math.sqrt(2.0), 1.0, math.sqrt(2.0)]  # the unit ZP element
    A[1] = [0.05, 0.05, 0.05, 0.05]
    X1 = rng.uniform(-5.0, 5.0, size=(24, 600))
    X2 = rng.uniform(-5.0, 5.0, size=(24, 600))
    X1[:, :25] = np.repeat(np.arange(-2.0, 3.0), 5)[None, :]  # integer offsets
    X2[:, :25] = np.tile(np.arange(-2.0, 3.0), 5)[None, :]
    V = np.stack([_exact.kernel_values(A[i], X1[i], X2[i]) for i in range(A.shape[0])])
    np.savez_compressed(os.path.join(OUT, "kernel_values.npz"), a=A, x1=X1, x2=X2, values=V)


def zp_golden(rng):
    with open(os.path.join(OUT, "zp_table.txt"), "w") as fh:
        fh.write(zp.dump_polynomial_table())
    plane = rng.standard_normal((40, 40))
    q1 = rng.uniform(-3.0, 43.0, 6000)
    q2 = rng.uniform(-3.0, 43.0, 6000)
    q1[:8] = [5.0, 5.5, 5.25, 4.75, 5.25, 4.75, 10.5, 10.0]   # partition ties
    q2[:8] = [5.0, 5.5, 5.25, 5.25, 4.75, 4.75, 10.5, 10.5]
    vals = zp.interpolate(zp.IntegratedImage(plane, col0=-2, row0=3), q1, q2)
    np.savez_compressed(os.path.join(OUT, "interpolate.npz"), plane=plane, col0=-2, row0=3,
                        x1=q1, x2=q2, values=vals)


def engine_golden(rng):
    cases = {}
    # impulse responses (test_engine.py:31-48 style)
    A = rng.uniform(0.7, 2.8, size=(10, 4))
    imp = np.zeros((33, 33))
    imp[16, 16] = 1.0
    cases["impulse_a"] = A
    cases["impulse_out"] = np.stack([engine.filter_space_invariant(imp, a) for a in A])
    off = np.zeros((25, 31))
    off[7, 22] = 1.0
    cases["impulse_off_out"] = engine.filter_space_invariant(off, [1.1, 2.3, 0.8, 1.6])
    # dense-oracle comparisons (test_engine.py:51-78)
    f1 = rng.random((20, 24))
    a1 = np.array([1.4, 1.9, 2.2, 0.9])
    cases["uni_f"], cases["uni_a"] = f1, a1
    cases["uni_ref"] = engine.filter_space_invariant(f1, a1)
    cases["uni_dense"] = oracle.dense_convolve(f1, a1)
    f2 = rng.random((18, 16))
    fld2 = np.stack([smooth_random_field(rng, (18, 16), 0.8, 2.5) for _ in range(4)], axis=-1)
    cases["var_f"], cases["var_field"] = f2, fld2
    cases["var_ref"] = engine.filter_space_variant(f2, fld2)
    cases["var_dense"] = oracle.dense_convolve(f2, fld2)
    f3 = rng.random((14, 15))
    fld3 = np.stack([smooth_random_field(rng, (14, 15), 0.9, 2.0) for _ in range(4)], axis=-1)
    cases["it2_f"], cases["it2_field"] = f3, fld3
    cases["it2_ref"] = engine.filter_space_variant(f3, fld3, iterations=2)
    cases["it2_dense"] = oracle.dense_convolve(f3, fld3, iterations=2)
    f4 = rng.random((31, 27))
    fld4 = np.stack([smooth_random_field(rng, (31, 27), 0.6, 3.5) for _ in range(4)], axis=-1)
    fld4[3:6, 4:9, 1] = 0.01  # widths below the floor
    cases["it3_f"], cases["it3_field"] = f4, fld4
    cases["it3_ref"] = engine.filter_space_variant(f4, fld4, iterations=3)
    cases["floor_dense"] = oracle.dense_convolve(f4, fld4)
    cases["floor_ref"] = engine.filter_space_variant(f4, fld4)
    # 64^2 config-1-style field through the exact optimiser
    H = W = 64
    x = np.arange(W, dtype=float)[None, :] * np.ones((H, 1))
    y = np.arange(H, dtype=float)[:, None] * np.ones((1, W))
    sig = 0.5 + 1.5 * x / (W - 1)
    c = (W - 1) / 2.0
    rho = 1.0 + 2.0 * np.hypot(x - c, y - c) / math.hypot(c, c)
    th = np.mod(np.arctan2(y - c, x - c), math.pi)
    field = np.empty((H, W, 4))
    for i in range(H):
        for j in range(W):
            field[i, j] = solver.optimize_scale_vector(
                covariance_from_params(2.0 * sig[i, j] ** 2, rho[i, j], th[i, j]))
    f5 = np.random.default_rng(0).random((H, W))
    cases["c1s_f"], cases["c1s_field"] = f5, field
    cases["c1s_ref"] = engine.filter_space_variant(f5, field)
    cases["c1s_dense"] = oracle.dense_convolve(f5, field)
    np.savez_compressed(os.path.join(OUT, "engine_small.npz"), **cases)


def preint_golden(rng):
    f = rng.random((12, 10))
    g = engine.preintegrate(f, col0=-3, row0=4, need_cols=(-9, 11), need_rows=(-1, 19))
    g0 = engine.preintegrate(f)
    np.savez_compressed(os.path.join(OUT, "preintegrate.npz"), f=f, plane=g.plane, col0=g.col0,
                        row0=g.row0, plane0=g0.plane, col00=g0.col0, row00=g0.row0)


def solver_golden(rng):
    lut = solver.build_lut()
    n = 4000
    size = rng.uniform(0.2, 600.0, n)
    th = rng.uniform(0.0, math.pi, n)
    rho = rng.uniform(1.0, lut.rho_max, n)
    q = 0.25 * math.pi
    th[:8] = [0.0, q, 2 * q, 3 * q, np.nextafter(q, 0), np.nextafter(2 * q, 0), np.nextafter(math.pi, 0), 1e-300]
    rho[:4] = [1.0, lut.rho_max, lut.rho_max * (1 + 1e-13), 1.0 + 1e-15]
    vals = solver.lookup_many(lut, size, rho, th)
    covs, opt = [], []
    for _ in range(600):
        t = rng.uniform(0.0, math.pi)
        cap = min(elongation_bound(t) * 0.9, 5.5)
        c = covariance_from_params(rng.uniform(0.5, 8.0), rng.uniform(1.0, cap), t)
        covs.append(c)
        opt.append(solver.optimize_scale_vector(c))
    np.savez_compressed(os.path.join(OUT, "solver.npz"), rho_grid=lut.rho_grid, phi_grid=lut.phi_grid,
                        entries=lut.entries, size=size, rho=rho, theta=th, lookup=vals,
                        covs=np.array(covs), opt=np.array(opt))


def config2_style(rng):
    """128^2 config-2-style run (LUT field) through the full reference."""
    H = W = 128
    lut = solver.build_lut()
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    sm = lambda k: (np.sin(2 * math.pi * (0.7 + 0.5 * k) * xx / W + 0.3 * k)  # noqa: E731
                    + np.sin(2 * math.pi * (1.1 + 0.3 * k) * yy / H + 1.7 * k))
    norm = lambda v: (v - v.min()) / (v.max() - v.min())  # noqa: E731
    size = 2.0 * (1.0 + 3.0 * norm(sm(1))) ** 2
    rho = 1.0 + 3.0 * norm(sm(2))
    th = np.mod(2 * math.pi * norm(sm(3)), math.pi)
    th = np.where(th >= math.pi, 0.0, th)
    field = solver.lookup_many(lut, size, rho, th)
    f = np.random.default_rng(7).random((H, W))
    out = engine.filter_space_variant(f, field)
    np.savez_compressed(os.path.join(OUT, "config2_style_128.npz"), f=f, size=size, rho=rho,
                        theta=th, field=field, ref=out)


def tensor_golden():
    """structure_tensor / anisotropy_from_tensor / adaptive_smooth
    (tensor.py:52-224) on stripes + noise, a step edge with flat areas, a
    constant image, and the reference tests' hand-made tensors."""
    from rubs import tensor
    rng = np.random.default_rng(77)
    cases = {}
    stripes = oracle.stripe_image((48, 56), period=7.0, angle=0.5)
    noisy = stripes + rng.normal(0.0, 0.08, stripes.shape)
    step = np.zeros((40, 44))
    step[:, 20:] = 1.0
    step[12:30, 5:12] += rng.normal(0.0, 0.05, (18, 7))
    cases["noisy"], cases["step"] = noisy, step
    for name, img in (("noisy", noisy), ("step", step)):
        cases[f"{name}_j0"] = tensor.structure_tensor(img, window_sigma=0.0)
        j = tensor.structure_tensor(img, window_sigma=1.5)
        cases[f"{name}_j"] = j
        m = tensor.anisotropy_from_tensor(j, 0.1)
        for k in ("size", "elongation", "orientation", "isotropic"):
            cases[f"{name}_{k}"] = getattr(m, k)
        cases[f"{name}_smooth"] = tensor.adaptive_smooth(img, 0.1)
    cases["noisy_smooth2"] = tensor.adaptive_smooth(noisy, 0.2, iterations=2, size_range=(0.5, 4.0))
    cases["flat_smooth"] = tensor.adaptive_smooth(np.full((24, 24), 0.75), 0.1)
    # the reference tests' tensor fields (test_tensor.py:54-110)
    g = np.array([math.cos(0.35), math.sin(0.35)])
    jm = 2.5 * np.outer(g, g)
    phi_g = math.pi / 8 + math.pi / 2
    g2 = np.array([math.cos(phi_g), math.sin(phi_g)])
    jm2 = 10.0 * np.outer(g2, g2)
    hand = np.zeros((6, 6, 3))
    hand[0, :] = (4.0, 0.0, 1.0)
    hand[1, :] = (6.0, 0.0, 2.0)
    hand[2, :] = (jm[0, 0], jm[0, 1], jm[1, 1])
    hand[3, :] = 0.0
    hand[4, :] = (jm2[0, 0], jm2[0, 1], jm2[1, 1])
    hand[5, :3] = (1.0, 0.0, 0.0)
    hand[5, 3:] = (9.0, 0.0, 0.0)
    cases["hand_j"] = hand
    m = tensor.anisotropy_from_tensor(hand, 0.1, size_range=(0.5, 4.0))
    for k in ("size", "elongation", "orientation", "isotropic"):
        cases[f"hand_{k}"] = getattr(m, k)
    np.savez_compressed(os.path.join(OUT, "tensor.npz"), **cases)


def main():
    if sys.argv[1:] == ["tensor"]:
        tensor_golden()
        print("tensor fixtures written to", OUT)
        return
    rng = np.random.default_rng(20240817)
    kernels(rng)
    zp_golden(rng)
    engine_golden(rng)
    preint_golden(rng)
    solver_golden(rng)
    config2_style(rng)
    tensor_golden()
    print("golden fixtures written to", OUT, "(rubs", rubs.__version__, ")")


if __name__ == "__main__":
    main()
