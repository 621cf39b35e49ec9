"""Host-side logic of the drop-in API that needs no GPU: validation and
exception mapping (engine.py:285-293, 204-216; geometry.py:63-73), fd_mesh,
geometry helpers, and the synthetic workload generators."""

import math

import numpy as np
import pytest

import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import geometry, workloads


def test_image_must_be_2d():
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((4, 4, 4)), [1.0] * 4)
    with pytest.raises(ValueError):
        rb.filter_space_invariant(np.ones(7), [1.0] * 4)


def test_iterations_validated():
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((4, 4)), np.ones((4, 4, 4)), iterations=0)


def test_field_shape_validated():
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((4, 4)), np.ones((5, 5, 4)))
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((4, 4)), np.ones(3))


def test_thread_cap_env(monkeypatch):
    # test_engine.py:180-187
    monkeypatch.delenv("RUBS_THREADS", raising=False)
    assert rb.thread_cap() == 0
    monkeypatch.setenv("RUBS_THREADS", "4")
    assert rb.thread_cap() == 4
    for bad in ("junk", "-1"):
        monkeypatch.setenv("RUBS_THREADS", bad)
        with pytest.raises(ValueError):
            rb.thread_cap()


def test_uniform_nonfinite_rejected():
    with pytest.raises(ValueError):
        rb.filter_space_variant(np.ones((4, 4)), [1.0, np.nan, 1.0, 1.0])


def test_scale_field_validation():
    with pytest.raises(ValueError):
        rb.ScaleField(np.ones((4, 4, 3)))
    with pytest.raises(ValueError):
        rb.ScaleField(np.zeros((4, 4, 4)))
    sf = rb.ScaleField.uniform((3, 5), [1.0, 2.0, 3.0, 4.0])
    assert sf.shape == (3, 5) and sf.scales.dtype == np.float64


def test_invariant_validates_scale_vector():
    with pytest.raises(ValueError):
        rb.filter_space_invariant(np.ones((4, 4)), [1.0, -1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        rb.filter_space_invariant(np.ones((4, 4)), [1.0, 1.0, 1.0])


def test_fd_mesh_structure(rng):
    a = rng.uniform(0.5, 2.5, size=4)
    mesh = rb.fd_mesh(a)
    assert mesh.offsets.shape == (16, 2)
    assert int(np.sum(mesh.signs == 1)) == 8 and int(np.sum(mesh.signs == -1)) == 8
    assert mesh.weight == pytest.approx(1.0 / float(np.prod(a)), rel=1e-15)


def test_fd_mesh_spec_example():
    # SPEC worked example: a = (2, 2 sqrt2, 2, 2 sqrt2) -> w = 1/32,
    # x_15 = (2, 6), tau = (0.5, 1.5)
    m = rb.fd_mesh([2.0, 2 * math.sqrt(2.0), 2.0, 2 * math.sqrt(2.0)])
    assert m.weight == pytest.approx(1 / 32)
    assert np.allclose(m.offsets[15], [2.0, 6.0])
    assert np.allclose(m.shift, [0.5, 1.5])


def test_elongation_bound_values():
    assert geometry.elongation_bound(math.pi / 8) == pytest.approx(3 + 2 * math.sqrt(2))
    assert math.isinf(geometry.elongation_bound(0.0))
    assert math.isinf(geometry.elongation_bound(math.pi / 4))
    with pytest.raises(ValueError):
        geometry.elongation_bound(math.pi)


def test_covariance_round_trip(rng):
    for _ in range(50):
        th = rng.uniform(0, math.pi)
        cap = min(geometry.elongation_bound(th) * 0.9, 5.5)
        c = geometry.covariance_from_params(rng.uniform(0.5, 8), rng.uniform(1, cap), th)
        a = rb.optimize_scale_vector(c)
        got = geometry.covariance_of(a)
        assert np.linalg.norm(got - c) / np.linalg.norm(c) < 1e-9


def test_infeasible_raises():
    c = geometry.covariance_from_params(2.0, 7.0, math.pi / 8)
    with pytest.raises(rb.Infeasible):
        rb.optimize_scale_vector(c)


def test_workload_config1_shape_and_range():
    w = workloads.config1(32, 32)
    assert w["f"].shape == (32, 32) and w["field"].shape == (32, 32, 4)
    assert np.isfinite(w["field"]).all() and (w["field"] > 0).all()


def test_workload_param_fields_respect_lut_domain():
    w = workloads.config2(64, 64)
    size, rho, th = (v.numpy() for v in (w["size"], w["elong"], w["orient"]))
    assert (size > 0).all() and (rho >= 1.0).all() and (rho <= 5.8).all()
    assert (th >= 0).all() and (th < math.pi).all()
    s = np.sqrt(size / 2.0)
    assert s.min() >= 2.0 - 1e-9 and s.max() <= 16.0 + 1e-9


def test_device_lut_is_cached_per_device(monkeypatch):
    """A LUT handle lives in one device's memory: the cache keys it by
    (table, device), so a call on cuda:1 after cuda:0 gets its own upload
    (mocked upload: no GPU here)."""
    import torch
    from paper_1003_2022_b200 import engine
    made = []

    class FakeDev:
        def __init__(self, d):
            self.d = d

        def __enter__(self):
            return self

        def __exit__(self, *a):
            return False

    monkeypatch.setattr(engine.DeviceLut, "_create", lambda self, lut: made.append(self.device))
    monkeypatch.setattr(torch.cuda, "device", FakeDev)
    monkeypatch.setattr(torch.cuda, "current_device", lambda: 0)
    monkeypatch.setattr(engine, "_LUT_CACHE", {})
    lut = rb.default_lut()
    a0 = engine.device_lut(lut, 0)
    a1 = engine.device_lut(lut, "cuda:1")
    assert a0 is not a1 and (a0.device, a1.device) == (0, 1)
    assert engine.device_lut(lut) is a0  # current device 0
    assert engine.device_lut(lut, torch.device("cuda", 1)) is a1
    assert made == [0, 1]
