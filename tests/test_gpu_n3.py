"""Parity of the three-direction (N=3) CUDA path (csrc/rubs_n3.cu, through
the C ABI) with the exact N=3 oracle (oracle/dense3_oracle.c, pinned to the
reference's spectral sampler and covariance_general by
tests/test_oracle_n3.py).

The N=3 path is exact (no image interpolation), so the bar is the same as
the N=4 path's: 1e-9 relative to max |output| against the exact dense
filter (impulses: the exact kernel to 1e-12)."""

import math

import numpy as np
import pytest

import oracle
from oracle import port3
from conftest import impulse, smooth_random_field
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))


def test_impulse_is_exact_kernel(cuda, rng):
    for _ in range(8):
        a = rng.uniform(0.3, 9.0, size=3)
        out = rb.filter_space_variant3(impulse((41, 45), (20, 22)), a)
        x = np.arange(45, dtype=float)[None, :] - 22
        y = np.arange(41, dtype=float)[:, None] - 20
        assert np.abs(out - oracle.kernel3_values(a, x, y)).max() < 1e-12


def test_random_field_matches_dense(cuda, rng):
    f = rng.random((70, 90))
    field = rng.uniform(0.0, 12.0, (70, 90, 3))
    field[5, 7] = [0.01, 3.0, 9.0]  # floored
    field[60, 80] = [-1.0, 0.0, 4.0]  # raw non-positive entries are floored
    assert rel_err(rb.filter_space_variant3(f, field), oracle.dense3(f, field)) < REL_TOL


def test_smooth_field_float32_image(cuda, rng):
    f = rng.random((96, 80)).astype(np.float32)
    s = smooth_random_field(rng, (96, 80), 2.0, 200.0)
    th = smooth_random_field(rng, (96, 80), 0.0, math.pi - 1e-9)
    rho = np.minimum(smooth_random_field(rng, (96, 80), 1.0, 6.0), 0.95 * rb.elongation_bound3(th))
    field = rb.scales3_from_params(s, rho, th)
    got = rb.filter_space_variant3(f, field)
    assert got.dtype == np.float64
    assert rel_err(got, oracle.dense3(f.astype(np.float64), field)) < REL_TOL


def test_uniform_vector_equals_full_field_bitwise(cuda, rng):
    f = rng.random((50, 61))
    a = np.array([3.3, 5.1, 2.2])
    u = rb.filter_space_variant3(f, a)
    full = rb.filter_space_variant3(f, np.broadcast_to(a, (50, 61, 3)).copy())
    assert np.array_equal(u, full)
    assert rel_err(u, oracle.dense3(f, a)) < REL_TOL


@pytest.mark.parametrize("iterations", [2, 3])
def test_iterations_match_dense(cuda, rng, iterations):
    f = rng.random((30, 34))
    field = rng.uniform(0.5, 6.0, (30, 34, 3))
    assert rel_err(rb.filter_space_variant3(f, field, iterations),
                   oracle.dense3(f, field, iterations)) < REL_TOL


def test_params_path_equals_field_path(cuda, rng):
    H, W = 64, 72
    f = rng.random((H, W))
    s = smooth_random_field(rng, (H, W), 1.0, 300.0)
    th = rng.uniform(0.0, math.pi, (H, W))
    rho = 1.0 + (0.95 * np.minimum(rb.elongation_bound3(th), 40.0) - 1.0) * rng.random((H, W))
    field = port3.scales3_from_params(s, rho, th)
    ref = oracle.dense3(f, field)
    fused = rb.filter_space_variant3_params(f, s, rho, th)
    assert rel_err(fused, ref) < REL_TOL
    # device mapping == oracle's linear solve
    dev = rb.scales3_many(s, rho, th)
    assert np.abs(dev - field).max() <= 1e-9 * field.max()
    # float32 parameters: mapping of the rounded values
    s32, r32, t32 = (v.astype(np.float32) for v in (s, rho, th))
    fused32 = rb.filter_space_variant3_params(f, s32, r32, t32)
    ref32 = oracle.dense3(f, port3.scales3_from_params(s32.astype(float), r32.astype(float),
                                                       t32.astype(float)))
    assert rel_err(fused32, ref32) < REL_TOL


def test_params_errors(cuda):
    f = np.ones((8, 8))
    ok = np.ones((8, 8))
    with pytest.raises(ValueError):
        rb.filter_space_variant3_params(f, -ok, ok, 0.1 * ok)
    with pytest.raises(ValueError):
        rb.filter_space_variant3_params(f, ok, 0.5 * ok, 0.1 * ok)
    with pytest.raises(ValueError):
        rb.filter_space_variant3_params(f, ok, ok, 4.0 * ok)
    with pytest.raises(rb.Infeasible):  # beyond the N=3 bound (3 at 90 degrees)
        rb.filter_space_variant3_params(f, ok, 3.5 * ok, (math.pi / 2) * ok)
    rb.filter_space_variant3_params(f, ok, 2.9 * ok, (math.pi / 2) * ok)


def test_field_errors_and_shapes(cuda, rng):
    f = rng.random((9, 11))
    bad = np.ones((9, 11, 3))
    bad[2, 3, 1] = np.nan
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, bad)
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, np.ones((9, 11, 4)))
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, np.array([1.0, np.inf, 1.0]))
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, np.ones(3), 0)
    with pytest.raises(ValueError):
        rb.filter_space_variant3(np.ones(5), np.ones(3))
    for shape in ((0, 5), (5, 0), (1, 1), (1, 77), (77, 1), (33, 65)):
        g = rng.random(shape)
        out = rb.filter_space_variant3(g, np.array([2.5, 1.5, 3.5]))
        assert out.shape == shape
        if g.size:
            assert rel_err(out, oracle.dense3(g, np.array([2.5, 1.5, 3.5]))) < REL_TOL


def test_linearity(cuda, rng):
    f, g = rng.random((48, 52)), rng.random((48, 52))
    field = rng.uniform(0.5, 8.0, (48, 52, 3))
    lhs = rb.filter_space_variant3(2.5 * f - 1.5 * g, field)
    rhs = 2.5 * rb.filter_space_variant3(f, field) - 1.5 * rb.filter_space_variant3(g, field)
    assert rel_err(lhs, rhs) < 1e-12


def test_torch_device_path_matches_host_path(cuda, rng):
    torch = cuda
    f = rng.random((40, 44))
    field = rng.uniform(0.5, 7.0, (40, 44, 3))
    host = rb.filter_space_variant3(f, field)
    dev = rb.filter_space_variant3(torch.from_numpy(f).cuda(), torch.from_numpy(field).cuda())
    assert np.array_equal(dev.cpu().numpy(), host)
    s = rng.uniform(1.0, 50.0, (40, 44))
    r = np.full((40, 44), 1.7)
    t = rng.uniform(0.0, math.pi, (40, 44))
    hp = rb.filter_space_variant3_params(f, s, r, t)
    dp = rb.filter_space_variant3_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda() for v in (s, r, t)))
    assert np.array_equal(dp.cpu().numpy(), hp)


def test_large_kernels_stream_region_rows(cuda, rng):
    """sigma up to 256 (config 5's range): regions far taller than one
    shared-memory chunk -- rows are streamed; sampled exact check."""
    H, W = 700, 900
    f = rng.random((H, W))
    a = np.array([330.0, 410.0, 260.0])  # hx ~ 350, hy ~ 290
    got = rb.filter_space_variant3(f, a)
    pts = np.array([[0, 0], [H - 1, W - 1], [350, 450], [10, 880], [690, 5], [200, 300]])
    ref = oracle.points3(f, a, pts)
    assert np.abs(got[pts[:, 0], pts[:, 1]] - ref).max() < REL_TOL * np.abs(ref).max()
    # impulse response at this size = exact kernel
    imp = rb.filter_space_variant3(impulse((H, W), (350, 450)), a)
    x = np.arange(W, dtype=float)[None, :] - 450
    y = np.arange(H, dtype=float)[:, None] - 350
    assert np.abs(imp - oracle.kernel3_values(a, x, y)).max() < 1e-15 + 1e-9 * np.abs(imp).max()


def test_config3_n3_sampled_exact(cuda, rng):
    """BASELINE config 3 as named (N=3, sigma 1-32, rho <= 6 clamped to the
    N=3 bound) at full size 8192^2: sampled pixels vs the exact filter."""
    torch = cuda
    w = workloads.config3_n3(param_dtype=torch.float32)
    f = w["f"]
    s, r, t = (v.numpy() for v in (w["size"], w["elong"], w["orient"]))
    out = rb.filter_space_variant3_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda() for v in (s, r, t)))
    H, W = f.shape
    pts = np.stack([rng.integers(0, H, 600), rng.integers(0, W, 600)], axis=1)
    pts = np.concatenate([pts, [[0, 0], [H - 1, W - 1], [0, W - 1], [H - 1, 0], [4000, 0], [0, 5000]]])
    field = port3.scales3_from_params(s[pts[:, 0], pts[:, 1]].astype(float),
                                      r[pts[:, 0], pts[:, 1]].astype(float),
                                      t[pts[:, 0], pts[:, 1]].astype(float))
    f64 = f.astype(np.float64)
    ref = np.empty(len(pts))
    for i, (p, a) in enumerate(zip(pts, field)):
        ref[i] = oracle.points3(f64, a, p[None, :], threads=1)[0]
    got = out[pts[:, 0], pts[:, 1]].cpu().numpy()
    assert np.abs(got - ref).max() < REL_TOL * np.abs(ref).max()


def test_streamed_host_path_equals_device_path(cuda, rng):
    """Host buffers go through the banded H2D / compute / D2H pipeline; the
    tiles are the device path's tiles, so the result is bitwise the same."""
    torch = cuda
    H, W = 700, 333
    f = rng.random((H, W)).astype(np.float32)
    s = smooth_random_field(rng, (H, W), 2.0, 800.0)
    th = smooth_random_field(rng, (H, W), 0.0, math.pi - 1e-9)
    r = np.minimum(smooth_random_field(rng, (H, W), 1.0, 5.0), 0.95 * rb.elongation_bound3(th))
    host = rb.filter_space_variant3_params(f, s, r, th)
    dev = rb.filter_space_variant3_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda() for v in (s, r, th)))
    assert np.array_equal(host, dev.cpu().numpy())
    field = rb.scales3_from_params(s, r, th)
    hf = rb.filter_space_variant3(f, field)
    df = rb.filter_space_variant3(torch.from_numpy(f).cuda(), torch.from_numpy(field).cuda())
    assert np.array_equal(hf, df.cpu().numpy())
    pts = np.array([[0, 0], [699, 332], [128, 10], [127, 300], [400, 200]])
    ref = oracle.points3(f.astype(np.float64), field, pts)
    assert np.abs(hf[pts[:, 0], pts[:, 1]] - ref).max() < REL_TOL * np.abs(ref).max()


def test_row_bands_reproduce_whole_image_bitwise(cuda):
    """Multi-GPU row bands of one N=3 image (each band computed from the
    image rows its reach needs): bitwise equal to the whole-image call."""
    torch = cuda
    from paper_1003_2022_b200 import sharding
    H, W = 1000, 640
    w = workloads.config3_n3(H, W, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    params = (w["size"], w["elong"], w["orient"])
    whole = rb.filter_space_variant3_params(f, *params)
    for world in (2, 3, 8):
        parts = []
        for band in sharding.band_bounds(H, world, sharding.TILE3):
            pb = [p[band[0]:band[1]] for p in params]
            reach = sharding.read_margins3_params(*pb)[1]
            field = np.maximum(port3.scales3_from_params(*(p.double().cpu().numpy() for p in pb)), 0.05)
            hy = 0.25 * math.sqrt(3.0) * (field[..., 1] + field[..., 2])
            assert reach == int(np.ceil(hy).max()) + 1
            n0, n1 = sharding.needed_rows3(band, reach, H)
            parts.append(sharding.filter3_rows_params(f[n0:n1], n0, H, *pb, band[0], band[0],
                                                      band[1] - band[0]))
            b0, b1 = sharding.needed_rows3(band, sharding.reach3_bound_params(pb[0]), H)
            assert b0 <= n0 and b1 >= n1
            assert torch.equal(sharding.filter3_rows_params(f[b0:b1], b0, H, *pb, band[0], band[0],
                                                            band[1] - band[0]), parts[-1])
        assert torch.equal(torch.cat(parts), whole)


def test_kernel_wider_than_the_region_buffer_fails_loudly(cuda):
    """A kernel whose row reach exceeds the shared-memory row buffer (about
    4000 columns) is refused with an error, never computed wrongly."""
    f = np.ones((16, 16))
    with pytest.raises(RuntimeError):
        rb.filter_space_variant3(f, np.array([9000.0, 1.0, 1.0]))
    out = rb.filter_space_variant3(f, np.array([3000.0, 1.0, 1.0]))  # fits
    ref = oracle.dense3(f, np.array([3000.0, 1.0, 1.0]))
    assert np.abs(out - ref).max() < 1e-9 * np.abs(ref).max()


def test_params_path_two_passes(cuda, rng):
    """Fused N=3 mapping with iterated passes (global reach from the mapped
    field, edge-clamped canvases) against the exact two-pass oracle."""
    H, W = 36, 40
    f = rng.random((H, W))
    s = smooth_random_field(rng, (H, W), 2.0, 120.0)
    th = rng.uniform(0.0, math.pi, (H, W))
    rho = 1.0 + (0.9 * np.minimum(rb.elongation_bound3(th), 8.0) - 1.0) * rng.random((H, W))
    ref = oracle.dense3(f, port3.scales3_from_params(s, rho, th), 2)
    got = rb.filter_space_variant3_params(f, s, rho, th, iterations=2)
    assert rel_err(got, ref) < REL_TOL
    dev = rb.filter_space_variant3_params(cuda.from_numpy(f).cuda(), *(cuda.from_numpy(v).cuda() for v in (s, rho, th)),
                                          iterations=2)
    assert np.array_equal(dev.cpu().numpy(), got)
