"""Parity of the CUDA path (through the C ABI) with the oracle.

Mirrors the reference's own engine tests (pkg/tests/test_engine.py,
test_acceptance.py 01/02/09, test_zp.py) with the checker swapped for the
pinned oracle (oracle/), then adds the BASELINE configs at full size:
sampled exact-dense checks plus size-independent properties (linearity,
impulse response = exact kernel, zero padding).

Tolerances: abs 1e-12 where the reference asserts 1e-12 (impulses), 1e-9
(relative to max |output|) against the exact dense oracle everywhere else
-- the north_star's target, tighter than the reference's own fast path
manages beyond 256^2.
"""

import math

import numpy as np
import pytest

import oracle
from oracle import port
from conftest import golden, impulse, smooth_random_field
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9


def kernel_at_offsets(a, shape, center):
    h, w = shape
    cy, cx = center
    return oracle.kernel_values(a, np.arange(w, dtype=float)[None, :] - cx,
                                np.arange(h, dtype=float)[:, None] - cy)


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))


def sample_points(rng, H, W, n, extra=()):
    pts = np.stack([rng.integers(0, H, n), rng.integers(0, W, n)], axis=1)
    border = [[0, 0], [0, W - 1], [H - 1, 0], [H - 1, W - 1], [0, W // 2], [H - 1, W // 3],
              [H // 2, 0], [H // 3, W - 1], [1, 1], [H - 2, W - 2]]
    return np.concatenate([pts, np.array(border), np.array(list(extra), dtype=np.int64).reshape(-1, 2)])


# --- reference test_engine.py, through the drop-in API ---------------------


def test_impulse_matches_exact_kernel(cuda, rng):
    for _ in range(10):
        a = rng.uniform(0.7, 2.8, size=4)
        out = rb.filter_space_invariant(impulse((33, 33)), a)
        assert np.abs(out - kernel_at_offsets(a, (33, 33), (16, 16))).max() < 1e-12


def test_impulse_golden(cuda):
    g = golden("engine_small.npz")
    for a, ref in zip(g["impulse_a"], g["impulse_out"]):
        out = rb.filter_space_invariant(impulse((33, 33)), a)
        assert np.abs(out - kernel_at_offsets(a, (33, 33), (16, 16))).max() < 1e-12
        assert np.abs(out - ref).max() < 1e-12
    out = rb.filter_space_invariant(impulse((25, 31), at=(7, 22)), [1.1, 2.3, 0.8, 1.6])
    assert np.abs(out - kernel_at_offsets([1.1, 2.3, 0.8, 1.6], (25, 31), (7, 22))).max() < 1e-12


@pytest.mark.parametrize("case,m", [("uni", 1), ("var", 1), ("it2", 2)])
def test_matches_dense_oracle_golden(cuda, case, m):
    g = golden("engine_small.npz")
    f = g[f"{case}_f"]
    fld = g["uni_a"] if case == "uni" else g[f"{case}_field"]
    out = rb.filter_space_variant(f, fld, m)
    assert np.abs(out - g[f"{case}_dense"]).max() < 1e-9
    assert np.abs(out - oracle.dense(f, fld, m)).max() < 1e-9


def test_three_passes_and_floor(cuda):
    g = golden("engine_small.npz")
    f, fld = g["it3_f"], g["it3_field"]
    assert np.abs(rb.filter_space_variant(f, fld) - g["floor_dense"]).max() < 1e-9
    out3 = rb.filter_space_variant(f, fld, 3)
    assert np.abs(out3 - oracle.dense(f, fld, 3)).max() < 1e-9
    assert np.abs(out3 - g["it3_ref"]).max() < 1e-8


def test_config1_style_golden(cuda):
    g = golden("engine_small.npz")
    out = rb.filter_space_variant(g["c1s_f"], g["c1s_field"])
    assert np.abs(out - g["c1s_dense"]).max() < 1e-9


def test_invariant_is_variant_bitwise(cuda, rng):
    f = rng.random((17, 19))
    a = np.array([1.2, 1.7, 2.4, 1.1])
    assert np.array_equal(rb.filter_space_variant(f, rb.ScaleField.uniform(f.shape, a)),
                          rb.filter_space_invariant(f, a))


def test_constant_preserved_for_integer_straight_widths(cuda):
    out = rb.filter_space_invariant(np.ones((28, 28)), [2.0, 1.3, 3.0, 2.6])
    assert np.abs(out[7:-7, 7:-7] - 1.0).max() < 1e-10


def test_fractional_widths_shift_the_constant(cuda):
    out = rb.filter_space_invariant(np.ones((28, 28)), [1.3, 1.1, 0.9, 1.2])
    dev = np.abs(out[8:-8, 8:-8] - 1.0).max()
    assert 1e-3 < dev < 0.1


def test_linearity(cuda, rng):
    a = np.array([1.5, 1.0, 2.0, 1.3])
    f = rng.standard_normal((15, 13))
    g = rng.standard_normal((15, 13))
    lhs = rb.filter_space_invariant(1.5 * f - 0.25 * g, a)
    rhs = 1.5 * rb.filter_space_invariant(f, a) - 0.25 * rb.filter_space_invariant(g, a)
    assert np.abs(lhs - rhs).max() < 1e-10


def test_zero_padding_consistency(cuda, rng):
    f = rng.random((12, 12))
    a = np.array([1.8, 1.2, 1.5, 2.1])
    padded = np.zeros((24, 24))
    padded[6:18, 6:18] = f
    assert np.abs(rb.filter_space_invariant(padded, a)[6:18, 6:18] - rb.filter_space_invariant(f, a)).max() < 1e-11


def test_scale_floor_clamps_bitwise(cuda):
    f = impulse((15, 15))
    assert np.array_equal(rb.filter_space_invariant(f, [0.01] * 4),
                          rb.filter_space_invariant(f, [rb.SCALE_FLOOR] * 4))


def test_overflow_guard_raises(cuda):
    with pytest.raises(OverflowError):
        rb.filter_space_invariant(np.full((64, 256), 1e14), [1.0, 1.0, 1.0, 1.0])


def test_nonfinite_field_raises(cuda):
    fld = np.ones((6, 7, 4))
    fld[3, 2, 1] = np.nan
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((6, 7)), fld)
    fld[3, 2, 1] = np.inf
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((6, 7)), fld)


def test_raw_nonpositive_entries_are_floored(cuda):
    # raw arrays with <= 0 entries are floored, not rejected (engine.py:292)
    f = impulse((11, 11))
    assert np.array_equal(rb.filter_space_variant(f, np.full((11, 11, 4), -3.0)),
                          rb.filter_space_invariant(f, [0.05] * 4))


def test_iterated_impulse_point_symmetry(cuda):
    a = np.array([1.6, 1.8, 2.0, 1.4])
    for m in (1, 2, 3):
        out = rb.filter_space_invariant(impulse((41, 41)), a, iterations=m)
        assert np.abs(out - out[::-1, ::-1]).max() < 1e-11


def test_empty_and_ragged_shapes(cuda, rng):
    assert rb.filter_space_invariant(np.zeros((0, 5)), [1.0] * 4).shape == (0, 5)
    for shape in [(1, 1), (1, 37), (37, 1), (33, 65), (65, 31)]:
        f = rng.random(shape)
        fld = rng.uniform(0.5, 3.0, size=shape + (4,))
        assert np.abs(rb.filter_space_variant(f, fld) - oracle.dense(f, fld)).max() < 1e-9


def test_float32_input_is_upcast(cuda, rng):
    f32 = rng.random((40, 30)).astype(np.float32)
    fld = rng.uniform(0.8, 2.5, size=(40, 30, 4))
    out = rb.filter_space_variant(f32, fld)
    assert out.dtype == np.float64
    assert np.array_equal(out, rb.filter_space_variant(f32.astype(np.float64), fld))


# --- reference test_acceptance.py ------------------------------------------


def test_acceptance_01_space_variant_matches_dense_oracle(cuda, rng):
    shape = (64, 64)
    for _ in range(2):
        f = rng.uniform(0.0, 1.0, size=shape)
        flat = np.broadcast_to(rng.uniform(0.8, 2.4, size=4), shape + (4,)).copy()
        wavy = np.stack([smooth_random_field(rng, shape, 0.7, 2.6) for _ in range(4)], axis=-1)
        for field in (flat, wavy):
            assert np.abs(rb.filter_space_variant(f, field) - oracle.dense(f, field)).max() < 1e-9


def test_acceptance_02_impulse_response_is_sampled_kernel(cuda, rng):
    for a in rng.uniform(0.6, 2.8, size=(25, 4)):
        out = rb.filter_space_invariant(impulse((33, 33)), a)
        assert np.abs(out - kernel_at_offsets(a, (33, 33), (16, 16))).max() < 1e-12


def _flat_cost_ms(torch, f, sizes, reps=5, calls=10):
    """Median over `reps` of the mean device time (CUDA events) of `calls`
    isotropic filters per size s (covariance trace; a = sqrt(3 s), N=4)."""
    out = []
    for s in sizes:
        a = np.full(4, math.sqrt(3.0 * s))
        rb.filter_space_invariant(f, a)
        laps = []
        for _ in range(reps):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(calls):
                rb.filter_space_invariant(f, a)
            t1.record()
            torch.cuda.synchronize()
            laps.append(t0.elapsed_time(t1) / calls)
        out.append(float(np.median(laps)))
    return out


def test_acceptance_03_runtime_flat_across_kernel_sizes(cuda):
    # test_acceptance.py:94-108 (max/min mean time < 1.15 over s = 1..16),
    # timed on the device at 2048^2 (at 512^2 a call is launch-bound: ~20 us)
    torch = cuda
    f = torch.from_numpy(np.random.default_rng(1).uniform(0.0, 1.0, size=(2048, 2048))).cuda()
    means = _flat_cost_ms(torch, f, (1.0, 2.0, 4.0, 8.0, 16.0))
    print("flat cost ms, s = 1..16:", [round(m, 4) for m in means])
    assert max(means) / min(means) < 1.15, means


@pytest.mark.xfail(strict=False, reason="large kernels (s >= 256) take the global-scratch block path: "
                   "measured max/min ~2.4 over s = 1..16384 at 2048^2 (DESIGN.md §4, flat-cost table)")
def test_acceptance_03_flat_up_to_large_kernels(cuda):
    # the same contract extended to s = 16384 (a ~ 222, support ~540 px)
    torch = cuda
    f = torch.from_numpy(np.random.default_rng(1).uniform(0.0, 1.0, size=(2048, 2048))).cuda()
    sizes = (1.0, 16.0, 256.0, 1024.0, 4096.0, 16384.0)
    means = _flat_cost_ms(torch, f, sizes, reps=3, calls=5)
    print("flat cost ms:", dict(zip(sizes, [round(m, 4) for m in means])),
          "max/min", round(max(means) / min(means), 2))
    assert max(means) / min(means) < 1.15, means


def test_acceptance_07_gaussian_correlation_of_the_device_kernel(cuda):
    # test_acceptance.py:160-171 on the device: the impulse response of the
    # filter (the discrete kernel) against the target Gaussian on the same
    # lattice, >= 0.95 for one pass and >= 0.99 for two.  The family is
    # scale-free; size 64 samples the kernel finely enough on integer pixels
    # (the reference engine gives the same correlations to 1e-9).
    n = 161
    f = np.zeros((n, n))
    f[n // 2, n // 2] = 1.0
    y, x = np.mgrid[: n, : n].astype(float) - n // 2
    for rho in (1.0, 2.0, 3.0, 4.0):
        for k in range(5):
            c = rb.covariance_from_params(64.0, rho, k * math.pi / 16.0)
            ci = np.linalg.inv(c)
            g = np.exp(-0.5 * (ci[0, 0] * x * x + 2.0 * ci[0, 1] * x * y + ci[1, 1] * y * y))
            a = rb.optimize_scale_vector(c)
            for m, floor in ((1, 0.95), (2, 0.99)):
                v = rb.filter_space_invariant(f, a, iterations=m)
                corr = float((v * g).sum()) / math.sqrt(float((v * v).sum()) * float((g * g).sum()))
                assert corr >= floor, (rho, k, m, corr)
                # mass and covariance of the discrete kernel: the target up to
                # the fractional-width quirk (reference: <= 0.012 and <= 0.26)
                mass = v.sum()
                cov = np.array([[(v * x * x).sum(), (v * x * y).sum()],
                                [(v * x * y).sum(), (v * y * y).sum()]]) / mass
                assert abs(mass - 1.0) < 0.02 and np.abs(cov - c).max() < 0.01 * np.abs(c).max() + 0.3


def test_acceptance_08_l2_error_decreases_with_passes(cuda):
    # test_acceptance.py:183-189 on the device: more passes of a / sqrt(m)
    # move the discrete kernel strictly closer to its Gaussian limit
    # (the reference engine: 0.0208, 0.0072, 0.0045, 0.0034 for m = 1..4)
    n = 161
    f = np.zeros((n, n))
    f[n // 2, n // 2] = 1.0
    y, x = np.mgrid[: n, : n].astype(float) - n // 2
    a = 4.0 * np.array([1.5, 1.0, 2.0, 1.2])
    c = rb.covariance_of(a)
    ci = np.linalg.inv(c)
    g = np.exp(-0.5 * (ci[0, 0] * x * x + 2.0 * ci[0, 1] * x * y + ci[1, 1] * y * y))
    g /= 2.0 * math.pi * math.sqrt(np.linalg.det(c))
    errs = [math.sqrt(float(((rb.filter_space_invariant(f, a, iterations=m) - g) ** 2).sum()))
            for m in (1, 2, 3, 4)]
    assert all(later < earlier for earlier, later in zip(errs, errs[1:])), errs
    assert errs[0] < 0.025 and errs[-1] < 0.004, errs


# --- ZP interpolation and global pre-integration (API parity) --------------


def test_interpolate_matches_reference_golden(cuda):
    g = golden("interpolate.npz")
    img = rb.IntegratedImage(g["plane"], int(g["col0"]), int(g["row0"]))
    got = rb.interpolate(img, g["x1"], g["x2"])
    assert np.abs(got - g["values"]).max() < 1e-12


def test_interpolate_matches_support_sum(cuda, rng):
    plane = rng.standard_normal((40, 40))
    q1 = rng.uniform(4.0, 35.0, size=10000)
    q2 = rng.uniform(4.0, 35.0, size=10000)
    fast = rb.interpolate(rb.IntegratedImage(plane), q1, q2)
    brute = np.zeros_like(fast)
    n1, n2 = np.round(q1).astype(int), np.round(q2).astype(int)
    unit = np.array([1.0, math.sqrt(2.0), 1.0, math.sqrt(2.0)])
    for d1 in range(-3, 4):
        for d2 in range(-3, 4):
            brute += plane[n2 + d2, n1 + d1] * oracle.kernel_values(unit, q1 - n1 - d1, q2 - n2 - d2)
    assert np.abs(fast - brute).max() < 1e-12


def test_interpolate_polynomial_reproduction(cuda, rng):
    cc, rr = np.meshgrid(np.arange(15.0), np.arange(12.0))
    q1 = rng.uniform(3.0, 11.0, size=200)
    q2 = rng.uniform(3.0, 8.0, size=200)
    got = rb.interpolate(rb.IntegratedImage(2.0 + 0.3 * cc - 0.7 * rr), q1, q2)
    assert np.abs(got - (2.0 + 0.3 * q1 - 0.7 * q2)).max() < 1e-12

    def quad(x1, x2):
        return 2.0 + 0.3 * x1 - 0.7 * x2 + 0.05 * x1 * x1 - 0.11 * x1 * x2 + 0.09 * x2 * x2
    got = rb.interpolate(rb.IntegratedImage(quad(cc, rr)), q1, q2)
    assert np.abs(got - quad(q1, q2) - 0.5 * 0.25 * (2 * 0.05 + 2 * 0.09)).max() < 1e-10


def test_preintegrate_matches_reference_golden(cuda):
    g = golden("preintegrate.npz")
    img = rb.preintegrate(g["f"], col0=-3, row0=4, need_cols=(-9, 11), need_rows=(-1, 19))
    assert (img.col0, img.row0) == (int(g["col0"]), int(g["row0"]))
    assert np.abs(img.plane - g["plane"]).max() <= 1e-13 * np.abs(g["plane"]).max()
    img0 = rb.preintegrate(g["f"])
    assert img0.plane.shape == g["plane0"].shape
    assert np.abs(img0.plane - g["plane0"]).max() <= 1e-13 * np.abs(g["plane0"]).max()


def test_preintegrate_guard(cuda):
    with pytest.raises(OverflowError):
        rb.preintegrate(np.full((64, 256), 1e14))


# --- LUT mapping ------------------------------------------------------------


def test_lookup_many_matches_reference_golden(cuda):
    g = golden("solver.npz")
    lut = rb.ScaleLut(g["rho_grid"], g["phi_grid"], g["entries"])
    got = rb.lookup_many(lut, g["size"], g["rho"], g["theta"])
    assert np.abs(got - g["lookup"]).max() <= 1e-14 * np.abs(g["lookup"]).max()


def test_lookup_out_of_grid_and_invalid(cuda):
    lut = rb.default_lut()
    with pytest.raises(rb.OutOfGrid):
        rb.lookup_many(lut, [1.0], [6.5], [0.3])
    with pytest.raises(ValueError):
        rb.lookup_many(lut, [1.0], [2.0], [math.pi])
    with pytest.raises(ValueError):
        rb.lookup_many(lut, [-1.0], [2.0], [0.3])
    with pytest.raises(ValueError):
        rb.lookup_many(lut, [1.0], [0.5], [0.3])


def test_fused_params_path_equals_field_path(cuda, rng):
    lut = rb.default_lut()
    H, W = 70, 90
    f = rng.random((H, W))
    size = rng.uniform(0.5, 40.0, (H, W))
    rho = rng.uniform(1.0, 5.0, (H, W))
    th = rng.uniform(0.0, math.pi, (H, W))
    fld = rb.lookup_many(lut, size, rho, th)
    fld_port = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, size, rho, th)
    assert np.abs(fld - fld_port).max() < 1e-13 * fld.max()
    fused = rb.filter_space_variant_params(f, size, rho, th, lut)
    via_field = rb.filter_space_variant(f, fld)
    # the same per-pixel arithmetic; both within the exactness target
    exact = oracle.dense(f, fld_port)
    assert rel_err(fused, exact) < REL_TOL
    assert rel_err(via_field, exact) < REL_TOL
    assert rel_err(fused, via_field) < REL_TOL


def test_fused_params_errors(cuda):
    with pytest.raises(rb.OutOfGrid):
        rb.filter_space_variant_params(np.ones((8, 8)), np.ones((8, 8)), np.full((8, 8), 9.0), np.zeros((8, 8)))
    with pytest.raises(ValueError):
        rb.filter_space_variant_params(np.ones((8, 8)), np.zeros((8, 8)), np.ones((8, 8)), np.zeros((8, 8)))


def test_torch_device_path_matches_host_path(cuda, rng):
    torch = cuda
    f = rng.random((50, 70))
    fld = rng.uniform(0.6, 3.0, size=(50, 70, 4))
    host = rb.filter_space_variant(f, fld, 2)
    dev = rb.filter_space_variant(torch.from_numpy(f).cuda(), torch.from_numpy(fld).cuda(), 2)
    assert dev.is_cuda and dev.dtype == torch.float64
    assert np.array_equal(dev.cpu().numpy(), host)


def test_streamed_host_path_equals_device_path(cuda, rng):
    # host buffers take the banded H2D / compute / D2H pipeline; device
    # tensors the single launch -- the same tiles, so the same bits
    torch = cuda
    H, W = 600, 520
    w = workloads.config2(H, W, device="cuda", param_dtype=torch.float32)
    f = w["f"]
    params = (w["size"], w["elong"], w["orient"])
    dev = rb.filter_space_variant_params(torch.from_numpy(f).cuda(), *params).cpu().numpy()
    host = rb.filter_space_variant_params(f, *(p.cpu().numpy() for p in params))
    assert np.array_equal(host, dev)
    # field mode with a block of very wide pixels: their tiles go through
    # the deferred (overflow) launches after the pipeline, rows re-copied
    fld = rng.uniform(0.6, 3.0, size=(H, W, 4))
    fld[300:310, 200:210] = 70.0
    dev = rb.filter_space_variant(torch.from_numpy(f).cuda(), torch.from_numpy(fld).cuda())
    host = rb.filter_space_variant(f, fld)
    assert np.array_equal(host, dev.cpu().numpy())
    pts = sample_points(rng, H, W, 12, extra=[(305, 205), (300, 200), (250, 260)])
    ref = oracle.points(f, fld, pts)
    assert rel_err(host[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def test_streamed_host_path_float32_and_pageable(cuda, rng):
    # float32 image, float64 parameters, no caller-provided result buffer
    torch = cuda
    H, W = 520, 480
    f = rng.random((H, W)).astype(np.float32)
    size = rng.uniform(2.0, 60.0, (H, W))
    rho = rng.uniform(1.0, 3.5, (H, W))
    th = rng.uniform(0.0, math.pi, (H, W))
    host = rb.filter_space_variant_params(f, size, rho, th)
    dev = rb.filter_space_variant_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda()
                                                                        for v in (size, rho, th)))
    assert host.dtype == np.float64 and np.array_equal(host, dev.cpu().numpy())
    lut = rb.default_lut()
    fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, size, rho, th)
    pts = sample_points(rng, H, W, 16)
    assert rel_err(host[pts[:, 0], pts[:, 1]], oracle.points(f.astype(np.float64), fld, pts)) < REL_TOL


# --- BASELINE configs at full size ------------------------------------------


def test_config1_full(cuda, rng):
    w = workloads.config1()
    out = rb.filter_space_variant(w["f"], w["field"])
    floored = np.argwhere((w["field"] < rb.SCALE_FLOOR).any(axis=-1))
    extra = floored[rng.choice(len(floored), min(200, len(floored)), replace=False)] if len(floored) else []
    pts = sample_points(rng, 256, 256, 1500, extra)
    ref = oracle.points(w["f"], w["field"], pts)
    assert rel_err(out[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def _config2_device(cuda):
    torch = cuda
    w = workloads.config2(device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    return w, f


def test_config2_full_sampled_exact(cuda, rng):
    w, f = _config2_device(cuda)
    out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"]).cpu().numpy()
    lut = rb.default_lut()
    s, r, t = (v.double().cpu().numpy() for v in (w["size"], w["elong"], w["orient"]))
    fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, s, r, t)
    floored = np.argwhere((fld < rb.SCALE_FLOOR).any(axis=-1))
    extra = floored[rng.choice(len(floored), min(100, len(floored)), replace=False)] if len(floored) else []
    big = np.argwhere(s > 0.95 * s.max())
    extra = list(extra) + list(big[rng.choice(len(big), min(100, len(big)), replace=False)])
    pts = sample_points(rng, 2048, 2048, 1200, extra)
    ref = oracle.points(w["f"], fld, pts)
    assert rel_err(out[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def test_config2_full_linearity_and_impulses(cuda, rng):
    torch = cuda
    w, f = _config2_device(cuda)
    args = (w["size"], w["elong"], w["orient"])
    g = torch.from_numpy(rng.standard_normal((2048, 2048))).cuda()
    lhs = rb.filter_space_variant_params(1.5 * f - 0.25 * g, *args)
    rhs = 1.5 * rb.filter_space_variant_params(f, *args) - 0.25 * rb.filter_space_variant_params(g, *args)
    assert (lhs - rhs).abs().max().item() < 1e-9 * rhs.abs().max().item()
    # sparse impulses far apart: each response is the exact kernel of the
    # OUTPUT pixel's own scale-vector (space-variant impulse response)
    imp = torch.zeros((2048, 2048), dtype=torch.float64, device="cuda")
    centres = [(300, 300), (1000, 1700), (1800, 400), (5, 2040), (1024, 1024)]
    for (y, x) in centres:
        imp[y, x] = 1.0
    out = rb.filter_space_variant_params(imp, *args).cpu().numpy()
    lut = rb.default_lut()
    for (y, x) in centres:
        ys, xs = np.mgrid[max(0, y - 12):min(2048, y + 13), max(0, x - 12):min(2048, x + 13)]
        fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, *(v.double().cpu().numpy()[ys, xs] for v in args))
        fld = np.maximum(fld, rb.SCALE_FLOOR)
        ref = np.array([oracle.kernel_values(fld[i, j], xs[i, j] - x, ys[i, j] - y)
                        for i in range(ys.shape[0]) for j in range(ys.shape[1])]).reshape(ys.shape)
        assert np.abs(out[ys, xs] - ref).max() < 1e-12


def test_config4_one_image_two_passes(cuda, rng):
    torch = cuda
    w = workloads.config4_image(0, 1024, 1024, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"], iterations=2).cpu().numpy()
    lut = rb.default_lut()
    s, r, t = (v.double().cpu().numpy() for v in (w["size"], w["elong"], w["orient"]))
    fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, s, r, t)
    pts = sample_points(rng, 1024, 1024, 24)
    ref = oracle.points(w["f"].astype(np.float64), fld, pts, iterations=2)
    assert rel_err(out[pts[:, 0], pts[:, 1]], ref) < REL_TOL


# --- large halos (regions beyond shared memory: configs 3 and 5) ----------


def test_large_uniform_kernel_global_regions(cuda, rng):
    # a ~ 150 -> support half-extent ~180 px: 8x8 regions exceed 225 KB,
    # so every tile runs through the global-memory block path
    f = rng.random((700, 600))
    a = np.array([150.0, 131.0, 120.0, 170.0])
    out = rb.filter_space_invariant(f, a)
    pts = sample_points(rng, 700, 600, 24)
    ref = oracle.points(f, a, pts)
    assert rel_err(out[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def _param_impulse_check(out, imp_centres, args, lut, radius):
    for (y, x) in imp_centres:
        ys, xs = np.mgrid[max(0, y - radius):min(out.shape[0], y + radius + 1):7,
                          max(0, x - radius):min(out.shape[1], x + radius + 1):7]
        fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries,
                               *(v[ys, xs] for v in args))
        fld = np.maximum(fld, rb.SCALE_FLOOR)
        ref = np.array([oracle.kernel_values(fld[i, j], xs[i, j] - x, ys[i, j] - y)
                        for i in range(ys.shape[0]) for j in range(ys.shape[1])]).reshape(ys.shape)
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(out[ys, xs] - ref).max() < 1e-9 * scale + 1e-15


def test_config3_shapes_sampled_exact(cuda, rng):
    # config 3 image and fields at 1024^2 (sigma in [1, 32], rho in [1, 6]
    # clamped), N=4 element: mixes the shared-memory and the block path
    torch = cuda
    w = workloads.config3(1024, 1024, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"]).cpu().numpy()
    lut = rb.default_lut()
    s, r, t = (v.double().cpu().numpy() for v in (w["size"], w["elong"], w["orient"]))
    fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, s, r, t)
    big = np.argwhere(s > 0.9 * s.max())
    extra = big[rng.choice(len(big), min(12, len(big)), replace=False)]
    pts = sample_points(rng, 1024, 1024, 24, extra)
    ref = oracle.points(w["f"].astype(np.float64), fld, pts)
    assert rel_err(out[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def test_config5_fields_impulse_response(cuda, rng):
    # config 5's field (sigma up to 256) on 4096^2 with sparse impulses: the
    # response near each impulse is the exact kernel of each output pixel
    torch = cuda
    w = workloads.config5(4096, 4096, device="cuda", param_dtype=torch.float32)
    imp = torch.zeros((4096, 4096), dtype=torch.float64, device="cuda")
    centres = [(700, 800), (2000, 3300), (3500, 1200), (4000, 4000)]
    for (y, x) in centres:
        imp[y, x] = 1.0
    out = rb.filter_space_variant_params(imp, w["size"], w["elong"], w["orient"]).cpu().numpy()
    args = [v.double().cpu().numpy() for v in (w["size"], w["elong"], w["orient"])]
    _param_impulse_check(out, centres, args, rb.default_lut(), 60)


# --- row bands (multi-GPU partition, emulated rank by rank on one GPU) -----


def test_row_bands_reproduce_whole_image_bitwise(cuda):
    torch = cuda
    from paper_1003_2022_b200 import sharding
    H, W = 1024, 768
    w = workloads.config2(H, W, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    params = (w["size"], w["elong"], w["orient"])
    whole = rb.filter_space_variant_params(f, *params)
    lut = rb.default_lut()
    for world in (2, 3, 8):
        parts = []
        for band in sharding.band_bounds(H, world):
            pb = [p[band[0]:band[1]] for p in params]
            m = sharding.read_margins_params(*pb, band[0], H)
            fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries,
                                   *(p.double().cpu().numpy() for p in pb))
            assert tuple(m) == port.read_margins(np.maximum(fld, rb.SCALE_FLOOR))
            n0, n1 = sharding.needed_rows(band, m, H)
            parts.append(sharding.filter_rows_params(f[n0:n1], n0, H, *pb, band[0], band[0],
                                                     band[1] - band[0]))
            # the cheap halo bound the multi-GPU path uses: more rows, same result
            b0, b1 = sharding.needed_rows(band, sharding.halo_bound_params(pb[0], lut), H)
            assert b0 <= n0 and b1 >= n1
            assert torch.equal(sharding.filter_rows_params(f[b0:b1], b0, H, *pb, band[0], band[0],
                                                           band[1] - band[0]), parts[-1])
        assert torch.equal(torch.cat(parts), whole)


# --- batch API (BASELINE config 4: a batch of images, pipelined) -----------


def test_batch_api_equals_per_image_calls(cuda, rng):
    torch = cuda
    imgs, ps = [], []
    for i in range(5):
        w = workloads.config4_image(i, 256, 192, param_dtype=torch.float32)
        imgs.append(w["f"])
        ps.append([v.numpy() for v in (w["size"], w["elong"], w["orient"])])
    for it in (1, 2):
        got = rb.filter_space_variant_params_batch(imgs, *[[p[q] for p in ps] for q in range(3)], iterations=it)
        for f, p, g in zip(imgs, ps, got):
            assert np.array_equal(g, rb.filter_space_variant_params(f, *p, iterations=it))
    # pinned outputs, aliased across the batch (image j lands in outs[j])
    outs = [torch.empty((256, 192), dtype=torch.float64, pin_memory=True).numpy() for _ in range(5)]
    got = rb.filter_space_variant_params_batch(imgs, *[[p[q] for p in ps] for q in range(3)], outs=outs)
    assert all(g is o for g, o in zip(got, outs))
    assert rb.filter_space_variant_params_batch([], [], [], []) == []


def test_batch_api_reports_the_failing_image(cuda, rng):
    torch = cuda
    w = workloads.config4_image(0, 64, 64, param_dtype=torch.float32)
    p = [v.numpy() for v in (w["size"], w["elong"], w["orient"])]
    bad = p[0].copy()
    bad[3, 5] = np.nan
    with pytest.raises(ValueError, match="batch image 2"):
        rb.filter_space_variant_params_batch([w["f"]] * 4, [p[0], p[0], bad, p[0]], [p[1]] * 4, [p[2]] * 4)
    with pytest.raises(ValueError):
        rb.filter_space_variant_params_batch([w["f"], w["f"][:32]], [p[0]] * 2, [p[1]] * 2, [p[2]] * 2)


def test_band_streamed_host_path_large_images(cuda):
    # H >= 8192: host buffers go through the band-complete pipeline
    # (run_streamed_bands): small kernels bitwise equal to the device path
    # (bands on the tile grid), large kernels (block regions cut at band
    # edges) within the precision budget of it
    torch = cuda
    w = workloads.config2(8192, 384, param_dtype=torch.float32)
    p = [v.numpy() for v in (w["size"], w["elong"], w["orient"])]
    host = rb.filter_space_variant_params(w["f"], *p)
    dev = rb.filter_space_variant_params(torch.from_numpy(w["f"]).cuda(), *(torch.from_numpy(v).cuda() for v in p))
    assert np.array_equal(host, dev.cpu().numpy())
    w5 = workloads.config5(8192, 512, param_dtype=torch.float32)
    f = w5["f"].numpy()
    p5 = [v.numpy() for v in (w5["size"], w5["elong"], w5["orient"])]
    host = rb.filter_space_variant_params(f, *p5)
    dev = rb.filter_space_variant_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda() for v in p5)).cpu().numpy()
    assert np.abs(host - dev).max() <= 1e-9 * np.abs(dev).max()


def test_row_bands_with_block_regions_match_whole_image_and_oracle(cuda, rng):
    """Config-5 kernels (sigma up to 256: global-scratch block regions) in
    row bands: the blocks are cut at the band edges, so a band's regions
    differ from the whole-image call's and the results agree within the
    precision budget, not bit for bit; both are within 1e-9 of the exact
    filter."""
    torch = cuda
    from paper_1003_2022_b200 import sharding
    H, W = 4096, 1024
    w = workloads.config5(H, W, device="cuda", param_dtype=torch.float32, image_device="cuda")
    f, params = w["f"], (w["size"], w["elong"], w["orient"])
    lut = rb.default_lut()
    whole = rb.filter_space_variant_params(f, *params)
    scale = float(whole.abs().max())
    parts = []
    for band in sharding.band_bounds(H, 4):
        pb = [p[band[0]:band[1]] for p in params]
        n0, n1 = sharding.needed_rows(band, sharding.halo_bound_params(pb[0], lut), H)
        parts.append(sharding.filter_rows_params(f[n0:n1], n0, H, *pb, band[0], band[0], band[1] - band[0]))
    banded = torch.cat(parts)
    assert float((banded - whole).abs().max()) < 1e-9 * scale
    pts = np.stack([rng.integers(0, H, 400), rng.integers(0, W, 400)], axis=1)
    pts = np.vstack([pts, [[1023, 5], [1024, 5], [2047, 900], [2048, 900], [3071, 77], [3072, 77]]])  # band edges
    idx = torch.as_tensor(pts, device="cuda")
    fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries,
                           *(p[idx[:, 0], idx[:, 1]].double().cpu().numpy() for p in params))
    ref = oracle.points_cuda(f, fld, pts)
    got = banded[idx[:, 0], idx[:, 1]].cpu().numpy()
    assert np.abs(got - ref).max() < 1e-9 * np.abs(ref).max()


def test_needle_kernels_are_reported_not_silent(cuda, rng):
    """A kernel whose own minimal region breaks the float64 precision budget
    (three widths at the floor next to a long one) cannot be held to 1e-9 by
    any region: the call still succeeds, within ~1e-8 of the exact filter,
    and says so (rubs_b200_precision_limited -> PrecisionWarning).  Ordinary
    fields, config-5 kernels included, raise nothing."""
    import warnings
    torch = cuda
    H, W = 96, 88
    f = rng.standard_normal((H, W))
    field = rng.uniform(2.0, 9.0, (H, W, 4))
    field[40, 30] = [0.01, 90.0, 0.01, 0.01]
    field[70, 60] = [0.02, 0.03, 0.01, 75.0]
    with pytest.warns(rb.PrecisionWarning):
        out = rb.filter_space_variant(f, field)
    ref = oracle.dense(f, field)
    assert np.abs(out - ref).max() < 5e-8 * np.abs(ref).max()
    mask = np.ones((H, W), bool)
    mask[40, 30] = mask[70, 60] = False
    assert np.abs(out - ref)[mask].max() < 1e-9 * np.abs(ref).max()
    with warnings.catch_warnings():
        warnings.simplefilter("error", rb.PrecisionWarning)
        rb.filter_space_variant(f, rng.uniform(0.0, 40.0, (H, W, 4)))  # floored entries, no needles
        w = workloads.config5(2048, 512, device="cuda", param_dtype=torch.float32, image_device="cuda")
        rb.filter_space_variant_params(w["f"], w["size"], w["elong"], w["orient"])
        w2 = workloads.config2(512, 512, device="cuda", param_dtype=torch.float32)
        rb.filter_space_variant_params(torch.from_numpy(w2["f"]).cuda(), w2["size"], w2["elong"], w2["orient"])
