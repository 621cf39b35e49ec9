"""bench.py's parity leg (CPU): per-pixel crops of the exact oracle equal the
whole-image exact filter, for the N=4 LUT, field and N=3 parameter paths."""

import math

import numpy as np

import bench
import oracle
from oracle import port, port3
from paper_1003_2022_b200 import default_lut


def _pts(rng, H, W, n=40):
    p = np.stack([rng.integers(0, H, n), rng.integers(0, W, n)], axis=1)
    return np.concatenate([p, [[0, 0], [H - 1, W - 1], [0, W - 1]]])


def test_parity_check_lut_and_field(rng):
    H, W = 48, 52
    f = rng.random((H, W))
    pts = _pts(rng, H, W)
    size = rng.uniform(1.0, 60.0, len(pts))
    rho = rng.uniform(1.0, 3.0, len(pts))
    th = rng.uniform(0.0, math.pi, len(pts))
    lut = default_lut()
    a = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, size, rho, th)
    # exact whole-image values at each pixel, each with its own kernel
    exact = np.array([oracle.points(f, ai, p[None, :])[0] for p, ai in zip(pts, a)])
    par = np.stack([size, rho, th], axis=1)
    res = bench.parity_check("2", {"pts": pts, "got": exact, "par": par, "n3": False, "f": f})
    assert res["max_rel_err"] < 1e-13
    res = bench.parity_check("1", {"pts": pts, "got": exact, "par": a, "n3": False, "f": f})
    assert res["max_rel_err"] < 1e-13
    bad = exact.copy()
    bad[3] += 1e-6
    assert bench.parity_check("2", {"pts": pts, "got": bad, "par": par, "n3": False, "f": f})[
        "max_rel_err"] > 1e-8


def test_parity_check_three_directions(rng):
    H, W = 40, 44
    f = rng.random((H, W)).astype(np.float32)
    pts = _pts(rng, H, W)
    size = rng.uniform(1.0, 80.0, len(pts))
    th = rng.uniform(0.0, math.pi, len(pts))
    rho = np.minimum(rng.uniform(1.0, 4.0, len(pts)), 2.9)
    a = port3.scales3_from_params(size, rho, th)
    f64 = f.astype(np.float64)
    exact = np.array([oracle.points3(f64, ai, p[None, :])[0] for p, ai in zip(pts, a)])
    par = np.stack([size, rho, th], axis=1)
    res = bench.parity_check("3", {"pts": pts, "got": exact, "par": par, "n3": True, "f": f})
    assert res["max_rel_err"] < 1e-13


def test_parity_check_lattice_mode(rng):
    """Config 3l: the parity figure is against the lattice mode's brute-force
    definition (here fed with the numpy restatement's output), the mode's own
    resampling error against the exact filter is reported beside it."""
    from oracle import lattice3_port as lp
    H, W = 44, 40
    f = rng.random((H, W)).astype(np.float32)
    pts = _pts(rng, H, W, 24)
    size = rng.uniform(4.0, 80.0, (H, W))
    th = rng.uniform(0.0, math.pi, (H, W))
    rho = np.minimum(rng.uniform(1.0, 4.0, (H, W)), 2.9)
    field = port3.scales3_from_params(size, rho, th)
    got = lp.lattice3(f.astype(np.float64), field)[pts[:, 0], pts[:, 1]]
    par = np.stack([v[pts[:, 0], pts[:, 1]] for v in (size, rho, th)], axis=1)
    res = bench.parity_check("3l", {"pts": pts, "got": got, "par": par, "n3": True, "lattice": True, "f": f})
    assert res["max_rel_err"] < 1e-11
    mode = res["mode_error_vs_exact"]
    assert 0.0 < mode["rms_rel"] <= mode["max_rel"] < 0.2


def test_lattice_config_is_listed_with_the_same_config_object_in_both_arms():
    assert "3l" in bench.CONFIGS and bench.SHAPES["3l"] == bench.SHAPES["3"]
    assert bench.bench_config("3l", 1)["path"].startswith("fused closed-form N=3 mapping + O(1) lattice")
    assert bench.row_banded("3l", 8) and not bench.row_banded("3l", 1)  # one image: row bands at N > 1
