"""Parity of the N=3 lattice (O(1), interpolated) mode on the GPU
(csrc/rubs_n3_lattice.cu, through the C ABI) with its two CPU routes: the
brute-force sum over lattice points with the exact N=3 kernel
(oracle.lattice3_points) and the numpy restatement (oracle/lattice3_port.py),
which tests/test_oracle_lattice.py pins to each other.

The device sums are exact integers, so the bar is the exact path's: 1e-9
relative to max |output|.  The mode's own error against the exact N=3
filter (the resampling) is reported by bench.py and DESIGN.md §9b, not
tested against a threshold here beyond its fall with kernel size."""

import math

import numpy as np
import pytest

import oracle
from oracle import lattice3_port as lp, port3
from conftest import smooth_random_field
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))


def _pts(H, W):
    return np.array([(r, c) for r in range(H) for c in range(W)])


@pytest.mark.parametrize("h", [1.0, 0.5])
def test_random_field_matches_brute_force(cuda, rng, h):
    H, W = 60, 76
    f = rng.random((H, W))
    field = rng.uniform(0.0, 12.0, (H, W, 3))
    field[5, 7] = [0.01, 3.0, 9.0]  # floored
    got = rb.filter_space_variant3(f, field, mode="lattice", spacing=h)
    ref = oracle.lattice3_points(f, field, _pts(H, W), h).reshape(H, W)
    assert rel_err(got, ref) < REL_TOL


def test_matches_port_and_float32_image(cuda, rng):
    H, W = 96, 80
    f = rng.random((H, W)).astype(np.float32)
    s = smooth_random_field(rng, (H, W), 2.0, 200.0)
    th = smooth_random_field(rng, (H, W), 0.0, math.pi - 1e-9)
    rho = np.minimum(smooth_random_field(rng, (H, W), 1.0, 6.0), 0.95 * rb.elongation_bound3(th))
    field = rb.scales3_from_params(s, rho, th)
    got = rb.filter_space_variant3(f, field, mode="lattice")
    assert got.dtype == np.float64
    assert rel_err(got, lp.lattice3(f.astype(np.float64), field)) < REL_TOL


def test_fused_params_f32_f64(cuda, rng):
    H, W = 70, 66
    f = rng.random((H, W))
    s = smooth_random_field(rng, (H, W), 2.0, 120.0)
    th = smooth_random_field(rng, (H, W), 0.0, math.pi - 1e-9)
    rho = np.minimum(smooth_random_field(rng, (H, W), 1.0, 6.0), 0.95 * rb.elongation_bound3(th))
    ref = oracle.lattice3_points(f, port3.scales3_from_params(s, rho, th), _pts(H, W), 1.0).reshape(H, W)
    got = rb.filter_space_variant3_params(f, s, rho, th, mode="lattice")
    assert rel_err(got, ref) < REL_TOL
    s32, r32, t32 = (v.astype(np.float32) for v in (s, rho, th))
    t32 = np.minimum(t32, np.nextafter(np.float32(math.pi), np.float32(0)))  # [0, pi) after rounding
    ref32 = oracle.lattice3_points(f, port3.scales3_from_params(s32, r32, t32), _pts(H, W), 1.0)
    got32 = rb.filter_space_variant3_params(f, s32, r32, t32, mode="lattice")
    assert rel_err(got32, ref32.reshape(H, W)) < REL_TOL


def test_two_passes_match_port(cuda, rng):
    f = rng.random((50, 58))
    field = rng.uniform(1.0, 9.0, (50, 58, 3))
    got = rb.filter_space_variant3(f, field, 2, mode="lattice")
    assert rel_err(got, lp.lattice3(f, field, 1.0, iterations=2)) < REL_TOL
    got3 = rb.filter_space_variant3(f, field, 3, mode="lattice", spacing=0.5)
    assert rel_err(got3, lp.lattice3(f, field, 0.5, iterations=3)) < REL_TOL


def test_uniform_vector_equals_full_field_bitwise(cuda, rng):
    f = rng.random((50, 61))
    a = np.array([3.3, 5.1, 2.2])
    u = rb.filter_space_variant3(f, a, mode="lattice")
    full = rb.filter_space_variant3(f, np.broadcast_to(a, (50, 61, 3)).copy(), mode="lattice")
    assert np.array_equal(u, full)


def test_torch_equals_host_bitwise(cuda, rng):
    import torch
    f = rng.random((64, 70))
    s = rng.uniform(2.0, 50.0, (64, 70))
    r = rng.uniform(1.0, 2.5, (64, 70))
    t = rng.uniform(0.0, 3.0, (64, 70))
    host = rb.filter_space_variant3_params(f, s, r, t, mode="lattice")
    dev = rb.filter_space_variant3_params(*(torch.from_numpy(v).cuda() for v in (f, s, r, t)), mode="lattice")
    assert np.array_equal(host, dev.cpu().numpy())
    fld = rb.scales3_from_params(s, r, t)
    dev2 = rb.filter_space_variant3(torch.from_numpy(f).cuda(), torch.from_numpy(fld).cuda(), mode="lattice")
    assert np.array_equal(rb.filter_space_variant3(f, fld, mode="lattice"), dev2.cpu().numpy())


def test_linearity(cuda, rng):
    f, g = rng.random((48, 52)), rng.random((48, 52))
    field = rng.uniform(1.0, 8.0, (48, 52, 3))
    lhs = rb.filter_space_variant3(2.0 * f - 3.0 * g, field, mode="lattice")
    rhs = 2.0 * rb.filter_space_variant3(f, field, mode="lattice") - 3.0 * rb.filter_space_variant3(g, field, mode="lattice")
    assert rel_err(lhs, rhs) < 1e-12


def test_scale_invariance_of_quantisation(cuda, rng):
    """The int128 sums are scaled by powers of two per block: scaling the
    image by 2^k scales the output exactly."""
    f = rng.random((40, 45))
    field = rng.uniform(1.0, 6.0, (40, 45, 3))
    base = rb.filter_space_variant3(f, field, mode="lattice")
    for k in (-40, 7, 300):
        assert np.array_equal(rb.filter_space_variant3(np.ldexp(f, k), field, mode="lattice"), np.ldexp(base, k))


def test_zero_and_negative_images(cuda, rng):
    field = rng.uniform(1.0, 6.0, (30, 33, 3))
    assert np.array_equal(rb.filter_space_variant3(np.zeros((30, 33)), field, mode="lattice"), np.zeros((30, 33)))
    f = rng.random((30, 33)) - 0.7
    ref = oracle.lattice3_points(f, field, _pts(30, 33), 1.0).reshape(30, 33)
    assert rel_err(rb.filter_space_variant3(f, field, mode="lattice"), ref) < REL_TOL


def test_errors_and_shapes(cuda, rng):
    f = rng.random((20, 24))
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, [2.0, 2.0, 2.0], mode="lattice", spacing=1.5)
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, [2.0, 2.0, 2.0], mode="hex")
    bad = f.copy()
    bad[3, 4] = np.nan
    with pytest.raises(ValueError):
        rb.filter_space_variant3(bad, [2.0, 2.0, 2.0], mode="lattice")
    with pytest.raises(ValueError):
        rb.filter_space_variant3(f, [2.0, np.inf, 2.0], mode="lattice")
    with pytest.raises(rb.Infeasible):
        rb.filter_space_variant3_params(f, 10.0, 5.9, 0.5 * math.pi, mode="lattice")
    for shape in ((0, 5), (5, 0), (1, 1), (1, 300), (300, 1)):
        g = rng.random(shape)
        got = rb.filter_space_variant3(g, [3.0, 4.0, 2.0], mode="lattice")
        assert got.shape == shape
        if g.size:
            ref = oracle.lattice3_points(g, np.array([3.0, 4.0, 2.0]), _pts(*shape), 1.0).reshape(shape)
            assert rel_err(got, ref) < REL_TOL


def test_large_kernels(cuda, rng):
    """sigma up to ~250 px: supports wider than the image, many blocks."""
    H, W = 400, 360
    f = rng.random((H, W))
    field = np.stack([rng.uniform(300, 700, (H, W)), rng.uniform(200, 600, (H, W)),
                      rng.uniform(250, 650, (H, W))], -1)
    got = rb.filter_space_variant3(f, field, mode="lattice")
    pts = np.stack([rng.integers(0, H, 64), rng.integers(0, W, 64)], 1)
    pts = np.vstack([pts, [[0, 0], [H - 1, W - 1], [0, W - 1], [H - 1, 0]]])
    ref = oracle.lattice3_points(f, field, pts, 1.0)
    assert rel_err(got[pts[:, 0], pts[:, 1]], ref) < REL_TOL


def test_error_against_exact_small_on_smooth_image(cuda, rng):
    """Against the EXACT N=3 filter (the interpolation error of the mode):
    small and falling with the kernel size on a smooth image."""
    H, W = 160, 160
    yy, xx = np.mgrid[0:H, 0:W]
    f = np.sin(xx / 9.0) * np.cos(yy / 13.0) + 0.5
    errs = []
    for a in (4.0, 16.0, 48.0):
        ex = oracle.dense3(f, np.array([a, a, a]))[40:120, 40:120]
        lat = rb.filter_space_variant3(f, np.array([a, a, a]), mode="lattice")[40:120, 40:120]
        errs.append(rel_err(lat, ex))
    assert errs[0] > errs[1] > errs[2] and errs[-1] < 1e-3, errs


def test_config3_full_size_sampled(cuda, rng):
    """BASELINE config 3 at 8192^2 through the fused mapping, checked at
    sampled pixels (borders and corners included) against the brute force."""
    torch = cuda
    w = workloads.config3_n3(param_dtype=torch.float32)
    f = w["f"]
    s, r, t = (v.numpy() for v in (w["size"], w["elong"], w["orient"]))
    out = rb.filter_space_variant3_params(torch.from_numpy(f).cuda(), *(torch.from_numpy(v).cuda() for v in (s, r, t)),
                                          mode="lattice")
    H, W = f.shape
    pts = np.stack([rng.integers(0, H, 400), rng.integers(0, W, 400)], axis=1)
    pts = np.concatenate([pts, [[0, 0], [H - 1, W - 1], [0, W - 1], [H - 1, 0], [4000, 0], [0, 5000]]])
    field = port3.scales3_from_params(s[pts[:, 0], pts[:, 1]].astype(float),
                                      r[pts[:, 0], pts[:, 1]].astype(float),
                                      t[pts[:, 0], pts[:, 1]].astype(float))
    f64 = f.astype(np.float64)
    ref = np.empty(len(pts))
    for i, (p, a) in enumerate(zip(pts, field)):  # one pixel with its own scales
        ref[i] = oracle.lattice3_points(f64, a, p[None, :], 1.0, threads=1)[0]
    got = out[pts[:, 0], pts[:, 1]].cpu().numpy()
    assert np.abs(got - ref).max() < REL_TOL * np.abs(ref).max()


def test_host_pipeline_equals_device_entry(cuda, rng):
    """Host buffers, one pass, >= 2048 rows: the three-stream block pipeline
    (size plane, image chunks, per-block parameters up; rows back per block)
    against the device-pointer entry.  The blocks differ (capped at 1/8 of
    the rows), so the quantisation exponents do: equal far below the bar,
    not bitwise."""
    torch = cuda
    H, W = 2304, 200
    f = rng.random((H, W)).astype(np.float32)
    s = smooth_random_field(rng, (H, W), 2.0, 300.0).astype(np.float32)
    th = np.minimum(smooth_random_field(rng, (H, W), 0.0, math.pi - 1e-6).astype(np.float32),
                    np.nextafter(np.float32(math.pi), np.float32(0)))
    rho = np.minimum(smooth_random_field(rng, (H, W), 1.0, 6.0),
                     0.95 * rb.elongation_bound3(th.astype(np.float64))).astype(np.float32)
    host = rb.filter_space_variant3_params(f, s, rho, th, mode="lattice")
    dev = rb.filter_space_variant3_params(*(torch.from_numpy(v).cuda() for v in (f, s, rho, th)),
                                          mode="lattice").cpu().numpy()
    assert rel_err(host, dev) < 1e-12
    pts = np.stack([rng.integers(0, H, 48), rng.integers(0, W, 48)], axis=1)
    pts = np.vstack([pts, [[0, 0], [H - 1, W - 1], [287, 5], [288, 5], [2303, 0]]])  # block edges too
    field = port3.scales3_from_params(*(v[pts[:, 0], pts[:, 1]].astype(float) for v in (s, rho, th)))
    f64 = f.astype(np.float64)
    ref = np.array([oracle.lattice3_points(f64, a, p[None, :], 1.0, threads=1)[0]
                    for p, a in zip(pts, field)])
    assert np.abs(host[pts[:, 0], pts[:, 1]] - ref).max() < REL_TOL * np.abs(ref).max()
    # errors surface from the pipeline as from the plain path
    bad = s.copy()
    bad[1500, 7] = -1.0
    with pytest.raises(ValueError):
        rb.filter_space_variant3_params(f, bad, rho, th, mode="lattice")
    with pytest.raises(rb.Infeasible):
        rb.filter_space_variant3_params(f, s, np.full_like(rho, 50.0), np.full_like(th, 0.6), mode="lattice")
    fbad = f.copy()
    fbad[2000, 3] = np.inf
    with pytest.raises(ValueError):
        rb.filter_space_variant3_params(fbad, s, rho, th, mode="lattice")


def test_row_bands_reproduce_whole_image(cuda, rng):
    """Lattice-mode row bands (2, 3, 8 bands, each from the image rows its
    halo bound needs): equal to the whole-image call far below the bar (the
    blocks' quantisation exponents differ, so not bitwise)."""
    torch = cuda
    from paper_1003_2022_b200 import sharding
    H, W = 1000, 320
    w = workloads.config3_n3(H, W, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    params = (w["size"], w["elong"], w["orient"])
    whole = rb.filter_space_variant3_params(f, *params, mode="lattice")
    scale = float(whole.abs().max())
    for world in (2, 3, 8):
        parts = []
        for band in sharding.band_bounds(H, world, sharding.TILE3L):
            pb = [p[band[0]:band[1]] for p in params]
            reach = sharding.reach3_lattice_bound(pb[0])
            n0, n1 = sharding.needed_rows3(band, reach, H)
            parts.append(sharding.filter3_lattice_rows_params(f[n0:n1], n0, H, *pb, band[0], band[0],
                                                              band[1] - band[0]))
        assert float((torch.cat(parts) - whole).abs().max()) < 1e-12 * scale


def test_absurd_kernel_sizes_are_refused(cuda, rng):
    """Supports beyond any image (size 1e30) fail with an error, through the
    size bound of the parameter entries and the exact margins of the field
    entries alike."""
    f = rng.random((40, 40))
    ones = np.ones((40, 40))
    with pytest.raises(RuntimeError):
        rb.filter_space_variant3_params(f, ones * 1e30, ones, ones * 0.3, mode="lattice")
    with pytest.raises(RuntimeError):
        rb.filter_space_variant3(f, np.array([1e20, 3.0, 3.0]), mode="lattice")


def test_two_passes_fused_params_match_port(cuda, rng):
    """Iterated passes through the fused-parameter entry: its canvases come
    from the size-plane bound (larger than the exact supports), which changes
    nothing but rounding against the restatement's exact canvases."""
    H, W = 72, 64
    f = rng.random((H, W))
    s = smooth_random_field(rng, (H, W), 4.0, 90.0)
    th = smooth_random_field(rng, (H, W), 0.0, math.pi - 1e-9)
    rho = np.minimum(smooth_random_field(rng, (H, W), 1.0, 5.0), 0.95 * rb.elongation_bound3(th))
    field = port3.scales3_from_params(s, rho, th)
    got = rb.filter_space_variant3_params(f, s, rho, th, 2, mode="lattice")
    assert rel_err(got, lp.lattice3(f, field, 1.0, iterations=2)) < REL_TOL
    got_t = rb.filter_space_variant3_params(*(cuda.from_numpy(v).cuda() for v in (f, s, rho, th)), 2,
                                            mode="lattice").cpu().numpy()
    assert np.array_equal(got, got_t)
