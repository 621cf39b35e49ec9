"""TEST INFRASTRUCTURE ONLY -- the parity oracle for the B200 filter path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker.  The product package ``paper_1003_2022_b200`` never
imports it and has no CPU fallback.

Two oracles live here:

* ``dense_oracle.c`` (built into ``oracle/_build/liboracle.so``): the exact
  dense convolution with the exact box-spline kernel -- the reference's
  ``oracle.dense_convolve`` + ``_exact.kernel_values``
  (pkg/src/rubs/oracle.py:177-241, _exact.py:29-106) restated in C, with an
  independent area routine (polygon clipping instead of slice integration).
* ``port.py``: a numpy restatement of the reference fast path (engine.py,
  zp.py, solver.lookup_many), used as the CPU baseline and as oracle "B".
* ``dense_oracle_cuda.cu`` (``dense_cuda``): the same exact dense filter on
  the GPU, for whole-image checks at the BASELINE sizes (tests only; pinned
  to ``dense`` by tests/test_gpu_fullsize.py).

Both are pinned against golden vectors generated from the reference itself
(tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


_CUDA_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_cuda.so")
_cuda_lib = None


def build() -> str:
    """Compile the C oracle (make in oracle/) and, where nvcc exists, its
    GPU copy for whole-image checks (make cuda)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    try:
        subprocess.run(["make", "-s", "-C", _HERE, "cuda"], check=True)
    except (OSError, subprocess.CalledProcessError):
        pass
    return _LIB_PATH


def dense_cuda(f, field, rows=None, cols=None):
    """Exact dense filter (one pass) on the GPU: output rows x cols (ranges,
    default the whole image) of the H x W image ``f``; inputs numpy or torch.
    Same kernel geometry as ``dense`` (dense_oracle_cuda.cu)."""
    import torch
    _cuda()
    ft = torch.as_tensor(f).to("cuda", torch.float64).contiguous()
    fl = torch.as_tensor(field).to("cuda", torch.float64).contiguous()
    H, W = ft.shape
    uniform = int(fl.numel() == 4)
    r0, r1 = rows if rows is not None else (0, H)
    c0, c1 = cols if cols is not None else (0, W)
    out = torch.empty((r1 - r0, c1 - c0), dtype=torch.float64, device="cuda")
    rc = _cuda_lib.rubs_oracle_cuda_dense(ctypes.c_void_p(ft.data_ptr()), H, W,
                                          ctypes.c_void_p(fl.data_ptr()), uniform, r0, c0,
                                          r1 - r0, c1 - c0, ctypes.c_void_p(out.data_ptr()))
    if rc:
        raise RuntimeError(f"oracle cuda error {rc}")
    return out


def _cuda():
    global _cuda_lib
    if _cuda_lib is None:
        if not os.path.exists(_CUDA_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE, "cuda"], check=True)
        L = ctypes.CDLL(_CUDA_LIB_PATH)
        vp, i = ctypes.c_void_p, ctypes.c_int
        L.rubs_oracle_cuda_dense.restype = i
        L.rubs_oracle_cuda_dense.argtypes = [vp, i, i, vp, i, i, i, i, i, vp]
        L.rubs_oracle_cuda_points.restype = i
        L.rubs_oracle_cuda_points.argtypes = [vp, i, i, i, vp, ctypes.c_double, vp, i, vp]
        _cuda_lib = L
    return _cuda_lib


def points_cuda(f, field, pts, div=1.0):
    """Exact one-pass output at lattice points pts = (n, 2) [row, col] on
    the GPU (dense_oracle_cuda.cu points_kernel): ``f`` is the H x W image
    (torch f32 / f64, any device, zero outside), ``field`` the (n, 4) RAW
    scale-vectors of the points (floored at 0.05, then divided by ``div`` =
    sqrt(iterations), as in dense_oracle.c field_at).  Points may lie
    outside the image (intermediate passes).  Returns numpy (n,)."""
    import torch
    ft = torch.as_tensor(f)
    if ft.dtype not in (torch.float32, torch.float64):
        ft = ft.double()
    ft = ft.to("cuda").contiguous()
    H, W = ft.shape
    fl = torch.as_tensor(np.ascontiguousarray(field, np.float64).reshape(-1, 4)).to("cuda")
    pt = torch.as_tensor(np.ascontiguousarray(pts, np.int64).reshape(-1, 2)).to("cuda")
    n = pt.shape[0]
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    rc = _cuda().rubs_oracle_cuda_points(ctypes.c_void_p(ft.data_ptr()), int(ft.dtype == torch.float32),
                                         H, W, ctypes.c_void_p(fl.data_ptr()), float(div),
                                         ctypes.c_void_p(pt.data_ptr()), n, ctypes.c_void_p(out.data_ptr()))
    if rc:
        raise RuntimeError(f"oracle cuda error {rc}")
    return out.cpu().numpy()


def support_radius(a):
    """(rx, ry) of dense_oracle.c support_radius for PREPARED vectors a (n, 4)."""
    a = np.asarray(a, np.float64).reshape(-1, 4)
    diag = (a[:, 1] + a[:, 3]) / np.sqrt(2.0)
    return (np.ceil(0.5 * (a[:, 0] + diag)).astype(np.int64) + 1,
            np.ceil(0.5 * (a[:, 2] + diag)).astype(np.int64) + 1)


def points2_cuda(f, field_of, pts):
    """Exact TWO-pass output (iterations=2: dense_oracle.c passp_at, the
    reference's oracle.py:205-241 semantics) at pixels pts (n, 2).
    ``field_of(rows, cols)`` returns the raw (k, 4) scale-vectors at image
    pixels (already edge-clamped indices are passed).  Pass 1 is evaluated
    on the GPU at every lattice point of the union window of the points'
    pass-2 supports (edge-clamped field, zero-padded image); pass 2 sums
    exact kernel values times those on the host."""
    f_t = f
    H, W = int(f_t.shape[0]), int(f_t.shape[1])
    pts = np.asarray(pts, np.int64).reshape(-1, 2)
    div = np.sqrt(2.0)
    a2 = np.maximum(np.asarray(field_of(pts[:, 0], pts[:, 1]), np.float64), 0.05) / div
    rx, ry = support_radius(a2)
    r0, r1 = int((pts[:, 0] - ry).min()), int((pts[:, 0] + ry).max())
    c0, c1 = int((pts[:, 1] - rx).min()), int((pts[:, 1] + rx).max())
    rr, cc = np.mgrid[r0:r1 + 1, c0:c1 + 1]
    q = np.stack([rr.ravel(), cc.ravel()], axis=1)
    fq = field_of(np.clip(q[:, 0], 0, H - 1), np.clip(q[:, 1], 0, W - 1))
    p1 = points_cuda(f_t, fq, q, div).reshape(rr.shape)
    out = np.empty(len(pts))
    for i, (r, c) in enumerate(pts):
        ys = np.arange(r - ry[i], r + ry[i] + 1)
        xs = np.arange(c - rx[i], c + rx[i] + 1)
        k = kernel_values(a2[i], (c - xs)[None, :].astype(np.float64), (r - ys)[:, None].astype(np.float64))
        out[i] = float((k * p1[ys[0] - r0:ys[-1] - r0 + 1, xs[0] - c0:xs[-1] - c0 + 1]).sum())
    return out


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_int64)
        L.rubs_oracle_kernel.restype = ctypes.c_double
        L.rubs_oracle_kernel.argtypes = [dp, ctypes.c_double, ctypes.c_double]
        L.rubs_oracle_kernel_many.restype = None
        L.rubs_oracle_kernel_many.argtypes = [dp, dp, dp, ctypes.c_int64, dp]
        L.rubs_oracle_points.restype = ctypes.c_int
        L.rubs_oracle_points.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int,
                                         ctypes.c_int, lp, ctypes.c_int64, dp]
        L.rubs_oracle_dense.restype = ctypes.c_int
        L.rubs_oracle_dense.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int,
                                        ctypes.c_int, dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def kernel_values(a, x1, x2):
    """Exact kernel K_a at points (x1, x2) (broadcast)."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(4)
    x1, x2 = np.broadcast_arrays(np.asarray(x1, np.float64), np.asarray(x2, np.float64))
    shape = x1.shape
    x1 = np.ascontiguousarray(x1).reshape(-1)
    x2 = np.ascontiguousarray(x2).reshape(-1)
    out = np.empty(x1.size)
    lib().rubs_oracle_kernel_many(_dp(a), _dp(x1), _dp(x2), x1.size, _dp(out))
    return out.reshape(shape)


def _field_arg(field, shape):
    field = np.asarray(field, dtype=np.float64)
    if field.shape == (4,):
        return np.ascontiguousarray(field), 1
    if field.shape != (*shape, 4):
        raise ValueError("field shape mismatch")
    return np.ascontiguousarray(field), 0


def dense(f, field, iterations=1):
    """Full exact dense filter (reference dense_convolve semantics)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    H, W = f.shape
    fld, uni = _field_arg(field, f.shape)
    out = np.empty((H, W))
    rc = lib().rubs_oracle_dense(_dp(f), H, W, _dp(fld), uni, int(iterations), _dp(out))
    if rc != 0:
        raise RuntimeError(f"oracle dense failed ({rc})")
    return out


def points(f, field, pts, iterations=1, threads=None):
    """Exact filter output at pixels pts = (N, 2) [row, col]; threaded
    (ctypes releases the GIL)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    H, W = f.shape
    fld, uni = _field_arg(field, f.shape)
    pts = np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 2)
    out = np.empty(pts.shape[0])
    n = pts.shape[0]
    if n == 0:
        return out
    threads = threads or min(os.cpu_count() or 1, 64)
    chunks = np.array_split(np.arange(n), min(threads * 4, n))
    L = lib()

    def run(idx):
        if idx.size == 0:
            return
        p = np.ascontiguousarray(pts[idx])
        o = np.empty(idx.size)
        rc = L.rubs_oracle_points(_dp(f), H, W, _dp(fld), uni, int(iterations),
                                  p.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.size, _dp(o))
        if rc != 0:
            raise RuntimeError("oracle points failed")
        out[idx] = o

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, chunks))
    return out


# ---------------------------------------------------------------------------
# Three-direction (N=3) kernel (dense3_oracle.c): exact, test side only.


def _lib3():
    L = lib()
    if not getattr(L, "_n3_ready", False):
        dp = ctypes.POINTER(ctypes.c_double)
        L.rubs_oracle3_kernel_many.restype = None
        L.rubs_oracle3_kernel_many.argtypes = [dp, dp, dp, ctypes.c_int64, dp]
        L.rubs_oracle3_dense.restype = ctypes.c_int
        L.rubs_oracle3_dense.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, ctypes.c_int, dp]
        L.rubs_oracle3_points.restype = ctypes.c_int
        L.rubs_oracle3_points.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, dp]
        L._n3_ready = True
    return L


def kernel3_values(a, x1, x2):
    """Exact N=3 kernel (directions 0/60/120 degrees) at points (x1, x2)."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(3)
    x1, x2 = np.broadcast_arrays(np.asarray(x1, np.float64), np.asarray(x2, np.float64))
    shape = x1.shape
    x1 = np.ascontiguousarray(x1).reshape(-1)
    x2 = np.ascontiguousarray(x2).reshape(-1)
    out = np.empty(x1.size)
    _lib3().rubs_oracle3_kernel_many(_dp(a), _dp(x1), _dp(x2), x1.size, _dp(out))
    return out.reshape(shape)


def _field3_arg(field, shape):
    field = np.asarray(field, dtype=np.float64)
    if field.shape == (3,):
        return np.ascontiguousarray(field), 1
    if field.shape != (*shape, 3):
        raise ValueError("field shape mismatch")
    return np.ascontiguousarray(field), 0


def dense3(f, field, iterations=1):
    """Exact dense N=3 filter (whole image)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    H, W = f.shape
    fld, uni = _field3_arg(field, f.shape)
    out = np.empty((H, W))
    if _lib3().rubs_oracle3_dense(_dp(f), H, W, _dp(fld), uni, int(iterations), _dp(out)) != 0:
        raise RuntimeError("oracle dense3 failed")
    return out


def points3(f, field, pts, threads=None):
    """Exact one-pass N=3 filter at pixels pts = (N, 2) [row, col]; threaded."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    H, W = f.shape
    fld, uni = _field3_arg(field, f.shape)
    pts = np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 2)
    out = np.empty(pts.shape[0])
    n = pts.shape[0]
    if n == 0:
        return out
    threads = threads or min(os.cpu_count() or 1, 64)
    chunks = np.array_split(np.arange(n), min(threads * 4, n))
    L = _lib3()

    def run(idx):
        if idx.size == 0:
            return
        p = np.ascontiguousarray(pts[idx])
        o = np.empty(idx.size)
        if L.rubs_oracle3_points(_dp(f), H, W, _dp(fld), uni,
                                 p.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.size, _dp(o)):
            raise RuntimeError("oracle points3 failed")
        out[idx] = o

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, chunks))
    return out


# ---------------------------------------------------------------------------
# N=3 lattice (O(1), interpolated) mode: brute-force route (dense3_oracle.c).


def _lib3l():
    L = _lib3()
    if not getattr(L, "_n3l_ready", False):
        dp, lp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        L.rubs_oracle3_splat.restype = None
        L.rubs_oracle3_splat.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, lp, lp,
                                         ctypes.c_int64, dp]
        L.rubs_oracle3_lattice_points.restype = ctypes.c_int
        L.rubs_oracle3_lattice_points.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int,
                                                  ctypes.c_double, lp, ctypes.c_int64, dp]
        L._n3l_ready = True
    return L


def splat3(f, h, al, ga):
    """Lattice-mode resampling f_hex at lattice indices (al, ga)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    al, ga = np.broadcast_arrays(np.asarray(al, np.int64), np.asarray(ga, np.int64))
    shape = al.shape
    al, ga = np.ascontiguousarray(al).reshape(-1), np.ascontiguousarray(ga).reshape(-1)
    out = np.empty(al.size)
    lp = ctypes.POINTER(ctypes.c_int64)
    _lib3l().rubs_oracle3_splat(_dp(f), f.shape[0], f.shape[1], float(h), al.ctypes.data_as(lp),
                                ga.ctypes.data_as(lp), al.size, _dp(out))
    return out.reshape(shape)


def lattice3_points(f, field, pts, h=1.0, threads=None):
    """Lattice-mode N=3 filter (one pass) at pixels pts = (N, 2) [row, col],
    by brute force: sum over lattice points p of f_hex[p] beta(n - p)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    H, W = f.shape
    fld, uni = _field3_arg(field, f.shape)
    pts = np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 2)
    out = np.empty(pts.shape[0])
    n = pts.shape[0]
    if n == 0:
        return out
    threads = threads or min(os.cpu_count() or 1, 64)
    chunks = np.array_split(np.arange(n), min(threads * 4, n))
    L = _lib3l()
    lp = ctypes.POINTER(ctypes.c_int64)

    def run(idx):
        if idx.size == 0:
            return
        p = np.ascontiguousarray(pts[idx])
        o = np.empty(idx.size)
        if L.rubs_oracle3_lattice_points(_dp(f), H, W, _dp(fld), uni, float(h), p.ctypes.data_as(lp),
                                         idx.size, _dp(o)):
            raise RuntimeError("oracle lattice3_points failed")
        out[idx] = o

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, chunks))
    return out
