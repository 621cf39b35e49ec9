"""Whole-image parity at the BASELINE sizes against the exact dense filter
on the GPU (oracle/dense_oracle_cuda.cu) -- every
output pixel, not a sample.  The GPU oracle is first pinned to the C oracle
(itself pinned to the reference's golden vectors).  Tolerance: 1e-9 of the
output scale (the north_star's target)."""

import numpy as np
import pytest

import oracle
from oracle import port
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9


def rel(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    e = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))
    print(f"max relative error {e:.3e} over {ref.size} pixels")
    return e


def lut_field(size, rho, th):
    lut = rb.default_lut()
    return port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, size, rho, th)


def test_cuda_oracle_matches_c_oracle(cuda, rng):
    f = rng.random((37, 45))
    fld = rng.uniform(0.02, 4.0, (37, 45, 4))
    got = oracle.dense_cuda(f, fld).cpu().numpy()
    assert rel(got, oracle.dense(f, fld)) < 1e-14
    a = np.array([2.3, 1.1, 0.7, 3.4])
    assert rel(oracle.dense_cuda(f, a).cpu().numpy(), oracle.dense(f, a)) < 1e-14
    sub = oracle.dense_cuda(f, fld, rows=(5, 20), cols=(7, 40)).cpu().numpy()
    assert rel(sub, oracle.dense(f, fld)[5:20, 7:40]) < 1e-14


def test_config1_whole_image(cuda):
    w = workloads.config1()
    out = rb.filter_space_variant(w["f"], w["field"])
    assert rel(out, oracle.dense_cuda(w["f"], w["field"]).cpu().numpy()) < REL_TOL


def test_config2_whole_image(cuda):
    torch = cuda
    w = workloads.config2(param_dtype=torch.float32)
    params = [v.numpy() for v in (w["size"], w["elong"], w["orient"])]
    out = rb.filter_space_variant_params(w["f"], *params)
    ref = oracle.dense_cuda(w["f"], lut_field(*params)).cpu().numpy()
    assert rel(out, ref) < REL_TOL


def test_config3_crop_of_the_full_image(cuda):
    # the whole 8192^2 image is filtered; every pixel of a 2048 x 1024 crop
    # is checked (sigma up to 32: ~20k exact kernel taps per pixel)
    torch = cuda
    w = workloads.config3(device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
    out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"])
    r, c = (3000, 5048), (5000, 6024)
    params = [v[r[0]:r[1], c[0]:c[1]].cpu().numpy() for v in (w["size"], w["elong"], w["orient"])]
    # the oracle reads the field only at output pixels: a full-size field
    # array with the crop's values in place
    full = torch.zeros((8192, 8192, 4), dtype=torch.float64, device="cuda")
    full[r[0]:r[1], c[0]:c[1]] = torch.from_numpy(lut_field(*params)).cuda()
    ref = oracle.dense_cuda(f.double(), full, rows=r, cols=c)
    assert rel(out[r[0]:r[1], c[0]:c[1]].cpu().numpy(), ref.cpu().numpy()) < REL_TOL


def test_config5_crop_large_kernels(cuda):
    # config 5's recipe (sigma 2..256) on 4096^2; 128 x 128 pixels around
    # the largest kernels checked exactly (~10^6 taps each)
    torch = cuda
    w = workloads.config5(4096, 4096, device="cuda", param_dtype=torch.float32, image_device="cuda")
    out = rb.filter_space_variant_params(w["f"], w["size"], w["elong"], w["orient"])
    i = int(torch.argmax(w["size"]).item())
    y, x = divmod(i, 4096)
    y = min(max(y, 64), 4096 - 64)
    x = min(max(x, 64), 4096 - 64)
    r, c = (y - 64, y + 64), (x - 64, x + 64)
    params = [v[r[0]:r[1], c[0]:c[1]].cpu().numpy() for v in (w["size"], w["elong"], w["orient"])]
    full = torch.zeros((4096, 4096, 4), dtype=torch.float64, device="cuda")
    full[r[0]:r[1], c[0]:c[1]] = torch.from_numpy(lut_field(*params)).cuda()
    ref = oracle.dense_cuda(w["f"].double(), full, rows=r, cols=c)
    assert rel(out[r[0]:r[1], c[0]:c[1]].cpu().numpy(), ref.cpu().numpy()) < REL_TOL
