"""Drop-in host API for the reference's filtering engine, backed by sm_100a.

Signatures, argument meaning and exceptions follow
/root/reference/pkg/src/rubs/engine.py and zp.py; the work runs in the CUDA
kernels of csrc/rubs_b200.cu through the C ABI (include/rubs_b200.h).

Accepted inputs
  * numpy / array-likes (the reference's contract): results come back as
    new float64 numpy arrays.  The host buffers go through the library's
    ``*_host`` entry points, which stage the copies themselves.
  * torch CUDA tensors: stay on the device (stream = torch's current
    stream); results are float64 CUDA tensors.

Reference map
  filter_space_variant     engine.py:265-324
  filter_space_invariant   engine.py:327-336
  ScaleField               engine.py:103-125
  fd_mesh / FdMesh         engine.py:64-100
  preintegrate             engine.py:145-201   (global canvas, 2^53 guard)
  interpolate              zp.py:186-228
  lookup_many              solver.py:289-335   (device)
  filter_space_variant_params   lookup_many + filter_space_variant fused
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native
from .geometry import as_scale_vector
from .solver import ScaleLut, default_lut

SCALE_FLOOR = 0.05  # engine.py:58
_SQRT2 = math.sqrt(2.0)
_BITS = ((np.arange(16)[:, None] >> np.arange(4)[None, :]) & 1).astype(np.float64)
_SIGNS = np.where(_BITS.sum(axis=1) % 2 == 0, 1.0, -1.0)


class FdMesh(NamedTuple):
    offsets: np.ndarray
    signs: np.ndarray
    weight: float
    shift: np.ndarray


def fd_mesh(a) -> FdMesh:
    """Finite-difference mesh of one scale-vector (engine.py:85-100)."""
    a1, a2, a3, a4 = as_scale_vector(a)
    p2, p4 = a2 / _SQRT2, a4 / _SQRT2
    ox = _BITS[:, 0] * a1 + _BITS[:, 1] * p2 - _BITS[:, 3] * p4
    oy = _BITS[:, 1] * p2 + _BITS[:, 2] * a3 + _BITS[:, 3] * p4
    return FdMesh(np.stack([ox, oy], axis=-1), _SIGNS.copy(), 1.0 / (a1 * a2 * a3 * a4),
                  np.array([0.5 * a1 + 0.5 * (p2 - p4) - 0.5, 0.5 * a3 + 0.5 * (p2 + p4) - 1.5]))


@dataclass(frozen=True)
class ScaleField:
    """Per-pixel scale-vectors (H, W, 4), all entries finite and positive."""

    scales: np.ndarray

    def __post_init__(self):
        s = np.asarray(self.scales, dtype=np.float64)
        if s.ndim != 3 or s.shape[2] != 4:
            raise ValueError(f"scale field must be (H, W, 4), got {s.shape}")
        if not np.isfinite(s).all() or (s <= 0.0).any():
            raise ValueError("scale field entries must be finite and positive")
        object.__setattr__(self, "scales", s)

    @classmethod
    def uniform(cls, shape, a) -> "ScaleField":
        h, w = shape
        return cls(np.broadcast_to(as_scale_vector(a), (h, w, 4)).copy())

    @property
    def shape(self):
        return self.scales.shape[:2]


@dataclass(frozen=True)
class IntegratedImage:
    """Pre-integrated plane plus the lattice position of plane[0, 0] (zp.py:56-66)."""

    plane: np.ndarray
    col0: int = 0
    row0: int = 0


def thread_cap() -> int:
    """Worker cap from RUBS_THREADS, validated as the reference does
    (engine.py:128-142): unset or 0 means automatic, a negative or
    non-integer value raises ValueError.  The device path is deterministic
    for any value (one launch geometry per shape), so the cap only
    documents the caller's intent; the CPU side here is single-threaded."""
    raw = os.environ.get("RUBS_THREADS", "0")
    try:
        cap = int(raw)
    except ValueError:
        raise ValueError(f"RUBS_THREADS must be an integer, got {raw!r}") from None
    if cap < 0:
        raise ValueError(f"RUBS_THREADS must be >= 0, got {cap}")
    return cap


# ---------------------------------------------------------------------------
def _is_torch(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and t.__name__ == "Tensor"


def _torch():
    import torch
    return torch


def _stream_handle():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _img_dtype_code(dt) -> int:
    return _native.RUBS_F32 if dt == np.float32 else _native.RUBS_F64


def _host_image(f):
    """Reference semantics: np.asarray(f, float64) (engine.py:285); float32
    stays float32 on the wire (the widening to fp64 is exact, done on chip)."""
    arr = np.asarray(f)
    if arr.dtype != np.float32:
        arr = np.asarray(arr, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("image must be 2-D")
    return np.ascontiguousarray(arr)


def _unwrap_field(field):
    """A ScaleField -- this package's or the reference's own ``rubs.ScaleField``
    (callers of the shimmed reference pass theirs) -- is used through its
    ``scales`` array; arrays and tensors pass through."""
    if isinstance(field, ScaleField):
        return field.scales
    if not isinstance(field, np.ndarray) and not _is_torch(field):
        scales = getattr(field, "scales", None)
        if scales is not None:
            return scales
    return field


def _host_field(field, shape):
    field = _unwrap_field(field)
    fld = np.asarray(field, dtype=np.float64)
    if fld.shape == (4,):
        if not np.isfinite(fld).all():
            raise ValueError("scale field entries must be finite")
        return np.ascontiguousarray(fld), True
    if fld.shape != (*shape, 4):
        raise ValueError(f"scale field shape {fld.shape} does not match image {shape}")
    return np.ascontiguousarray(fld), False


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _host_out(out, shape):
    """Optional caller-provided result buffer (e.g. pinned host memory, so
    the device-to-host copy runs at full bandwidth); an extension of the
    reference API, which always allocates."""
    if out is None:
        return np.empty(shape, dtype=np.float64)
    if out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array of the image shape")
    return out


def filter_space_variant(f, field, iterations: int = 1, *, out=None):
    """Filter with a per-pixel kernel in constant time per pixel.

    ``f`` 2-D image (combined with zeros outside); ``field`` ScaleField,
    (H, W, 4) array or (4,) vector; entries below SCALE_FLOOR are clamped.
    Returns float64 of f's shape (numpy, or a CUDA tensor for CUDA input).
    """
    if isinstance(iterations, bool) or int(iterations) != iterations:
        raise ValueError("iterations must be an integer")
    iterations = int(iterations)
    if _is_torch(f):
        return _filter_torch(f, field, iterations)
    img = _host_image(f)
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    fld, uniform = _host_field(field, img.shape)
    H, W = img.shape
    out = _host_out(out, (H, W))
    if H == 0 or W == 0:
        return out
    L = _native.load()
    _native.check(L.rubs_b200_filter_host(_ptr(img), _img_dtype_code(img.dtype), H, W, _ptr(fld),
                                          int(uniform), iterations, _ptr(out)))
    return out


def _filter_torch(f, field, iterations):
    torch = _torch()
    if f.dim() != 2:
        raise ValueError("image must be 2-D")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if not f.is_cuda:
        raise ValueError("torch input must live on a CUDA device")
    if f.dtype not in (torch.float32, torch.float64):
        f = f.to(torch.float64)
    if f.stride(1) != 1:
        f = f.contiguous()
    H, W = f.shape
    out = torch.empty((H, W), dtype=torch.float64, device=f.device)
    field = _unwrap_field(field)
    uniform = False
    if _is_torch(field):
        fld = field.to(device=f.device, dtype=torch.float64)
        if tuple(fld.shape) == (4,):
            host4 = np.ascontiguousarray(fld.cpu().numpy())
            uniform = True
        elif tuple(fld.shape) != (H, W, 4):
            raise ValueError(f"scale field shape {tuple(fld.shape)} does not match image {(H, W)}")
        else:
            if fld.stride(2) != 1 or fld.stride(1) != 4:
                fld = fld.contiguous()
    else:
        arr = np.asarray(field, dtype=np.float64)
        if arr.shape == (4,):
            host4 = np.ascontiguousarray(arr)
            uniform = True
        elif arr.shape != (H, W, 4):
            raise ValueError(f"scale field shape {arr.shape} does not match image {(H, W)}")
        else:
            fld = torch.from_numpy(np.ascontiguousarray(arr)).to(f.device)
    if H == 0 or W == 0:
        return out
    L = _native.load()
    with torch.cuda.device(f.device):
        if uniform:
            if not np.isfinite(host4).all():
                raise ValueError("scale field entries must be finite")
            fptr, ld_field = _ptr(host4), 0
        else:
            fptr, ld_field = ctypes.c_void_p(fld.data_ptr()), fld.stride(0) // 4
        _native.check(L.rubs_b200_filter(
            ctypes.c_void_p(f.data_ptr()), _native.RUBS_F32 if f.dtype == torch.float32 else _native.RUBS_F64,
            H, W, f.stride(0), fptr, int(uniform), ld_field, iterations,
            ctypes.c_void_p(out.data_ptr()), W, _stream_handle()))
    return out


def filter_space_invariant(f, a, iterations: int = 1):
    """Uniform-kernel filtering; bit-identical to the variant path
    (engine.py:327-336)."""
    if _is_torch(f):
        if f.dim() != 2:
            raise ValueError("image must be 2-D")
    else:
        f = _host_image(f)
    a = as_scale_vector(a.detach().cpu().numpy() if _is_torch(a) else a)
    return filter_space_variant(f, a, iterations)


# ---------------------------------------------------------------------------
# LUT mapping on the device


class DeviceLut:
    """A ScaleLut uploaded to one CUDA device (rubs_lut handle; the table
    lives in that device's memory, so a handle serves that device only)."""

    def __init__(self, lut: ScaleLut, device: int | None = None):
        self.lut = lut
        torch = _torch()
        self.device = torch.cuda.current_device() if device is None else int(device)
        with torch.cuda.device(self.device):
            self._create(lut)

    def _create(self, lut):
        L = _native.load()
        h = ctypes.c_void_p()
        rg = np.ascontiguousarray(lut.rho_grid, dtype=np.float64)
        pg = np.ascontiguousarray(lut.phi_grid, dtype=np.float64)
        en = np.ascontiguousarray(lut.entries, dtype=np.float64)
        _native.check(L.rubs_b200_lut_create(_ptr(rg), _ptr(pg), _ptr(en), rg.shape[0], pg.shape[0],
                                             ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                _native.load().rubs_b200_lut_destroy(self.handle)
        except Exception:
            pass


_LUT_CACHE: dict = {}


def _device_index(device) -> int:
    if type(device) is int:
        return device
    torch = _torch()
    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


def device_lut(lut: ScaleLut | None = None, device=None) -> DeviceLut:
    """The device copy of ``lut`` on ``device`` (default: the current CUDA
    device), cached per (table, device)."""
    lut = lut or default_lut()
    dev = _device_index(device)
    key = (id(lut), dev)
    hit = _LUT_CACHE.get(key)
    if hit is None or hit.lut is not lut:
        hit = DeviceLut(lut, dev)
        _LUT_CACHE[key] = hit
    return hit


_DT_CODE = {}  # torch dtype -> RUBS_F32 / RUBS_F64 (filled on first use)


def _raw_stream(device: int) -> int:
    """Handle of torch's current stream on `device` (the raw-pointer query
    torch uses for its own kernel launches: ~0.3 us instead of ~3 us for
    torch.cuda.current_stream().cuda_stream)."""
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(device)
    return torch.cuda.current_stream(device).cuda_stream


def _fast_device_args(f, params):
    """(image dtype code, parameter dtype code) when f and the three
    parameter planes are contiguous float32/float64 CUDA tensors of f's shape
    on f's device, which is the current device, the parameters sharing one
    dtype; else None (the general path converts).  Kept to plain attribute
    reads: it runs on every call (config 2: ~0.4 ms per call)."""
    if not _DT_CODE:
        torch = _torch()
        _DT_CODE.update({torch.float32: _native.RUBS_F32, torch.float64: _native.RUBS_F64})
    fd = _DT_CODE.get(f.dtype)
    if fd is None or not f.is_cuda or not f.is_contiguous():
        return None
    dev = f.get_device()
    if dev != _torch().cuda.current_device():
        return None
    p0 = params[0]
    shape = f.shape
    for p in params:
        if (not _is_torch(p) or p.get_device() != dev or p.dtype != p0.dtype or p.shape != shape
                or not p.is_contiguous()):
            return None
    pd = _DT_CODE.get(p0.dtype)
    return None if pd is None else (fd, pd)


def _params_host(size, elongation, orientation):
    s = np.asarray(size)
    r = np.asarray(elongation)
    t = np.asarray(orientation)
    shape = np.broadcast_shapes(s.shape, r.shape, t.shape)
    dt = np.float32 if all(np.asarray(v).dtype == np.float32 for v in (s, r, t)) else np.float64
    return [np.ascontiguousarray(np.broadcast_to(v, shape), dtype=dt) for v in (s, r, t)], shape, dt


def lookup_many(lut: ScaleLut, size, elongation, orientation):
    """Vectorised bilinear LUT lookup on the device (solver.py:289-335)."""
    (s, r, t), shape, dt = _params_host(size, elongation, orientation)
    torch = _torch()
    n = int(np.prod(shape)) if shape else 1
    out = torch.empty((max(n, 1), 4), dtype=torch.float64, device="cuda")
    if n == 0:
        return np.empty(shape + (4,))
    dl = device_lut(lut)
    ds, dr, dth = (torch.from_numpy(v.reshape(-1)).cuda() for v in (s, r, t))
    L = _native.load()
    _native.check(L.rubs_b200_lookup(dl.handle, ctypes.c_void_p(ds.data_ptr()), ctypes.c_void_p(dr.data_ptr()),
                                     ctypes.c_void_p(dth.data_ptr()),
                                     _native.RUBS_F32 if dt == np.float32 else _native.RUBS_F64, n,
                                     ctypes.c_void_p(out.data_ptr()), _stream_handle()))
    return out.cpu().numpy().reshape(shape + (4,))


def filter_space_variant_params(f, size, elongation, orientation, lut: ScaleLut | None = None,
                                iterations: int = 1, *, out=None):
    """filter_space_variant(f, lookup_many(lut, size, elongation, orientation),
    iterations) with the lookup fused into the filter kernel."""
    iterations = int(iterations)
    dl = device_lut(lut, f.get_device() if _is_torch(f) and f.is_cuda else None)
    L = _native.load()
    if _is_torch(f):
        torch = _torch()
        if f.dim() != 2:
            raise ValueError("image must be 2-D")
        if iterations < 1:
            raise ValueError("iterations must be >= 1")
        H, W = f.shape
        fast = _fast_device_args(f, (size, elongation, orientation))
        if fast is not None:
            # already-placed contiguous CUDA tensors on the current device: no
            # conversions (the wrapper's own cost is part of every call's step)
            fdt, pdt = fast
            out = torch.empty_like(f, dtype=torch.float64)
            rc = L.rubs_b200_filter_params(
                f.data_ptr(), fdt, H, W, W, size.data_ptr(), elongation.data_ptr(),
                orientation.data_ptr(), pdt, W, dl.handle, iterations, out.data_ptr(), W,
                _raw_stream(f.get_device()))
            if rc:
                _native.check(rc)
            return out
        ps = []
        for v in (size, elongation, orientation):
            v = v if _is_torch(v) else torch.as_tensor(np.asarray(v))
            v = v.to(device=f.device)
            if v.dtype not in (torch.float32, torch.float64):
                v = v.to(torch.float64)
            ps.append(v)
        pdt = torch.float32 if all(p.dtype == torch.float32 for p in ps) else torch.float64
        ps = [torch.broadcast_to(p.to(pdt), (H, W)).contiguous() for p in ps]
        if f.dtype not in (torch.float32, torch.float64):
            f = f.to(torch.float64)
        f = f.contiguous()
        out = torch.empty((H, W), dtype=torch.float64, device=f.device)
        with torch.cuda.device(f.device):
            _native.check(L.rubs_b200_filter_params(
                ctypes.c_void_p(f.data_ptr()), _native.RUBS_F32 if f.dtype == torch.float32 else _native.RUBS_F64,
                H, W, W, *(ctypes.c_void_p(p.data_ptr()) for p in ps),
                _native.RUBS_F32 if pdt == torch.float32 else _native.RUBS_F64, W, dl.handle, iterations,
                ctypes.c_void_p(out.data_ptr()), W, _stream_handle()))
        return out
    img = _host_image(f)
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    H, W = img.shape
    (s, r, t), shape, dt = _params_host(size, elongation, orientation)
    if shape != (H, W):
        s, r, t = (np.ascontiguousarray(np.broadcast_to(v, (H, W))) for v in (s, r, t))
    out = _host_out(out, (H, W))
    if H == 0 or W == 0:
        return out
    _native.check(L.rubs_b200_filter_params_host(
        _ptr(img), _img_dtype_code(img.dtype), H, W, _ptr(s), _ptr(r), _ptr(t),
        _native.RUBS_F32 if dt == np.float32 else _native.RUBS_F64, dl.handle, iterations, _ptr(out)))
    return out


def filter_space_variant_params_batch(images, sizes, elongations, orientations,
                                      lut: ScaleLut | None = None, iterations: int = 1, *, outs=None):
    """``[filter_space_variant_params(f, s, r, t, lut, iterations) for ...]``
    over a batch of same-shape host images (BASELINE config 4), pipelined
    on the device: image i+1's inputs upload while image i is filtered and
    image i-1's result comes back (rubs_b200_filter_params_batch_host).
    ``outs``: optional list of C-contiguous float64 host arrays (pinned
    memory lets every copy run asynchronously).  Returns the list of
    results.  An error names the first failing image."""
    iterations = int(iterations)
    n = len(images)
    if not (len(sizes) == len(elongations) == len(orientations) == n):
        raise ValueError("batch lists must have the same length")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if n == 0:
        return []
    imgs = [_host_image(f) for f in images]
    H, W = imgs[0].shape
    if any(im.shape != (H, W) for im in imgs) or len({im.dtype for im in imgs}) != 1:
        raise ValueError("batch images must share one shape and dtype")
    params = []
    pdt = None
    for s, r, t in zip(sizes, elongations, orientations):
        (ps, pr, pt), shape, dt = _params_host(s, r, t)
        if shape != (H, W):
            ps, pr, pt = (np.ascontiguousarray(np.broadcast_to(v, (H, W))) for v in (ps, pr, pt))
        pdt = pdt or dt
        if dt != pdt:
            ps, pr, pt = (np.ascontiguousarray(v, dtype=np.float64) for v in (ps, pr, pt))
            pdt = np.float64
        params.append((ps, pr, pt))
    if pdt == np.float64:
        params = [tuple(np.ascontiguousarray(v, dtype=np.float64) for v in p) for p in params]
    outs = [_host_out(o, (H, W)) for o in (outs or [None] * n)]
    if H == 0 or W == 0:
        return outs
    dl = device_lut(lut)
    L = _native.load()

    def arr(ptrs):
        return (ctypes.c_void_p * n)(*[a.ctypes.data for a in ptrs])
    failed = ctypes.c_int(-1)
    rc = L.rubs_b200_filter_params_batch_host(
        n, arr(imgs), _img_dtype_code(imgs[0].dtype), H, W, arr([p[0] for p in params]),
        arr([p[1] for p in params]), arr([p[2] for p in params]),
        _native.RUBS_F32 if pdt == np.float32 else _native.RUBS_F64, dl.handle, iterations, arr(outs),
        ctypes.byref(failed))
    if rc:
        try:
            _native.check(rc)
        except Exception as e:
            raise type(e)(f"batch image {failed.value}: {e}") from None
    return outs


# ---------------------------------------------------------------------------
# Global-mode pieces kept for API parity (not on the hot path)


def preintegrate(f, *, col0: int = 0, row0: int = 0, need_cols=None, need_rows=None) -> IntegratedImage:
    """Four running-sum sweeps on the reference canvas (engine.py:145-201),
    computed on the device; raises OverflowError past 2^53."""
    torch = _torch()
    img = _host_image(f)
    h, w = img.shape
    if need_cols is None:
        need_cols = (col0 - 2, col0 + w + 1)
    if need_rows is None:
        need_rows = (row0 - 2, row0 + h + 1)
    L = _native.load()
    rows, cols, c_lo, r_lo = (ctypes.c_int64() for _ in range(4))
    L.rubs_b200_preintegrate_shape(h, w, col0, row0, int(need_cols[0]), int(need_cols[1]),
                                   int(need_rows[0]), int(need_rows[1]), ctypes.byref(rows),
                                   ctypes.byref(cols), ctypes.byref(c_lo), ctypes.byref(r_lo))
    dimg = torch.from_numpy(img).cuda()
    plane = torch.empty((rows.value, cols.value), dtype=torch.float64, device="cuda")
    _native.check(L.rubs_b200_preintegrate(
        ctypes.c_void_p(dimg.data_ptr()), _img_dtype_code(img.dtype), h, w, w, col0, row0,
        int(need_cols[0]), int(need_cols[1]), int(need_rows[0]), int(need_rows[1]),
        ctypes.c_void_p(plane.data_ptr()), cols.value, _stream_handle()))
    return IntegratedImage(plane.cpu().numpy(), col0=c_lo.value, row0=r_lo.value)


def interpolate(image: IntegratedImage, x1, x2) -> np.ndarray:
    """F(x) = sum_n g[n] Z(x - n) at arbitrary points, reads clamped to the
    plane edge (zp.py:186-228), on the device."""
    torch = _torch()
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    shape = np.broadcast_shapes(x1.shape, x2.shape)
    xa = np.ascontiguousarray(np.broadcast_to(x1, shape)).reshape(-1)
    ya = np.ascontiguousarray(np.broadcast_to(x2, shape)).reshape(-1)
    plane = np.ascontiguousarray(image.plane, dtype=np.float64)
    dp = torch.from_numpy(plane).cuda()
    dx, dy = torch.from_numpy(xa).cuda(), torch.from_numpy(ya).cuda()
    out = torch.empty(xa.shape[0], dtype=torch.float64, device="cuda")
    L = _native.load()
    _native.check(L.rubs_b200_interpolate(
        ctypes.c_void_p(dp.data_ptr()), plane.shape[0], plane.shape[1], plane.shape[1], int(image.col0),
        int(image.row0), ctypes.c_void_p(dx.data_ptr()), ctypes.c_void_p(dy.data_ptr()), xa.shape[0],
        ctypes.c_void_p(out.data_ptr()), _stream_handle()))
    return out.cpu().numpy().reshape(shape)


# ---------------------------------------------------------------------------
# Three-direction (N=3) box spline (BASELINE.json config 3).  Not in the
# reference: these extend filter_space_variant's
# semantics (engine.py:265-324) to the 0/60/120-degree kernel, computed
# exactly on the device (csrc/rubs_n3.cu).


def _host_field3(field, shape):
    fld = np.asarray(field, dtype=np.float64)
    if fld.shape == (3,):
        if not np.isfinite(fld).all():
            raise ValueError("scale field entries must be finite")
        return np.ascontiguousarray(fld), True
    if fld.shape != (*shape, 3):
        raise ValueError(f"three-direction scale field shape {fld.shape} does not match image {shape}")
    return np.ascontiguousarray(fld), False


def _check_iterations(iterations) -> int:
    if isinstance(iterations, bool) or int(iterations) != iterations:
        raise ValueError("iterations must be an integer")
    if int(iterations) < 1:
        raise ValueError("iterations must be >= 1")
    return int(iterations)


def _torch_image(f):
    torch = _torch()
    if f.dim() != 2:
        raise ValueError("image must be 2-D")
    if not f.is_cuda:
        raise ValueError("torch input must live on a CUDA device")
    if f.dtype not in (torch.float32, torch.float64):
        f = f.to(torch.float64)
    return f.contiguous()


def _n3_mode(mode, spacing) -> bool:
    """True for the O(1) lattice mode; validates its spacing."""
    if mode not in ("exact", "lattice"):
        raise ValueError(f"mode must be 'exact' or 'lattice', got {mode!r}")
    if mode == "lattice" and not (0.125 <= float(spacing) <= 1.0):
        raise ValueError("lattice spacing must be in [0.125, 1]")
    return mode == "lattice"


def filter_space_variant3(f, field, iterations: int = 1, *, out=None, mode: str = "exact",
                          spacing: float = 1.0):
    """Three-direction filter: per-pixel scales (a1, a2, a3) along 0, 60 and
    120 degrees.  ``field`` is (H, W, 3) or (3,); entries below SCALE_FLOOR
    are clamped, passes use a / sqrt(iterations) like filter_space_variant.
    ``mode="exact"`` computes the N=3 filter exactly (O(kernel height) per
    pixel); ``mode="lattice"`` is the paper's O(1) algorithm on the
    triangular lattice of the given ``spacing`` (the image resampled once,
    DESIGN.md §9b).  Returns float64 of f's shape (numpy, or a CUDA tensor for
    CUDA input)."""
    iterations = _check_iterations(iterations)
    lattice = _n3_mode(mode, spacing)
    L = _native.load()
    if _is_torch(f):
        torch = _torch()
        f = _torch_image(f)
        H, W = f.shape
        res = torch.empty((H, W), dtype=torch.float64, device=f.device)
        fld = field.detach().cpu().numpy() if _is_torch(field) and tuple(field.shape) == (3,) else field
        if _is_torch(fld):
            if tuple(fld.shape) != (H, W, 3):
                raise ValueError(f"three-direction scale field shape {tuple(fld.shape)} does not match image {(H, W)}")
            dfl = fld.to(device=f.device, dtype=torch.float64).contiguous()
            uniform, fptr = False, ctypes.c_void_p(dfl.data_ptr())
        else:
            arr, uniform = _host_field3(fld, (H, W))
            if uniform:
                fptr = _ptr(arr)
            else:
                dfl = torch.from_numpy(arr).to(f.device)
                fptr = ctypes.c_void_p(dfl.data_ptr())
        if H == 0 or W == 0:
            return res
        fdt = _native.RUBS_F32 if f.dtype == torch.float32 else _native.RUBS_F64
        with torch.cuda.device(f.device):
            if lattice:
                _native.check(L.rubs_b200_filter3_lattice(
                    ctypes.c_void_p(f.data_ptr()), fdt, H, W, W, fptr, int(uniform), W, iterations,
                    float(spacing), ctypes.c_void_p(res.data_ptr()), W, _stream_handle()))
            else:
                _native.check(L.rubs_b200_filter3(
                    ctypes.c_void_p(f.data_ptr()), fdt, H, W, W, fptr, int(uniform), W, iterations,
                    ctypes.c_void_p(res.data_ptr()), W, _stream_handle()))
        return res
    img = _host_image(f)
    fld, uniform = _host_field3(field, img.shape)
    H, W = img.shape
    out = _host_out(out, (H, W))
    if H == 0 or W == 0:
        return out
    if lattice:
        _native.check(L.rubs_b200_filter3_lattice_host(_ptr(img), _img_dtype_code(img.dtype), H, W,
                                                       _ptr(fld), int(uniform), iterations,
                                                       float(spacing), _ptr(out)))
    else:
        _native.check(L.rubs_b200_filter3_host(_ptr(img), _img_dtype_code(img.dtype), H, W, _ptr(fld),
                                               int(uniform), iterations, _ptr(out)))
    return out


def filter_space_variant3_params(f, size, elongation, orientation, iterations: int = 1, *, out=None,
                                 mode: str = "exact", spacing: float = 1.0):
    """filter_space_variant3(f, scales3_from_params(size, elongation,
    orientation), iterations, mode=mode, spacing=spacing) with the
    (closed-form) mapping fused into the filter kernel.  Raises Infeasible
    beyond the N=3 elongation bound."""
    iterations = _check_iterations(iterations)
    lattice = _n3_mode(mode, spacing)
    L = _native.load()
    if _is_torch(f):
        torch = _torch()
        if f.dim() == 2:
            fast = _fast_device_args(f, (size, elongation, orientation))
            if fast is not None:
                H, W = f.shape
                res = torch.empty((H, W), dtype=torch.float64, device=f.device)
                if H and W:
                    stream = torch.cuda.current_stream(f.device).cuda_stream
                    if lattice:
                        _native.check(L.rubs_b200_filter3_lattice_params(
                            f.data_ptr(), fast[0], H, W, W, size.data_ptr(), elongation.data_ptr(),
                            orientation.data_ptr(), fast[1], W, iterations, float(spacing),
                            res.data_ptr(), W, stream))
                    else:
                        _native.check(L.rubs_b200_filter3_params(
                            f.data_ptr(), fast[0], H, W, W, size.data_ptr(), elongation.data_ptr(),
                            orientation.data_ptr(), fast[1], W, iterations, res.data_ptr(), W, stream))
                return res
        f = _torch_image(f)
        H, W = f.shape
        ps = []
        for v in (size, elongation, orientation):
            v = v if _is_torch(v) else torch.as_tensor(np.asarray(v))
            v = v.to(device=f.device)
            if v.dtype not in (torch.float32, torch.float64):
                v = v.to(torch.float64)
            ps.append(v)
        pdt = torch.float32 if all(p.dtype == torch.float32 for p in ps) else torch.float64
        ps = [torch.broadcast_to(p.to(pdt), (H, W)).contiguous() for p in ps]
        res = torch.empty((H, W), dtype=torch.float64, device=f.device)
        if H == 0 or W == 0:
            return res
        fdt = _native.RUBS_F32 if f.dtype == torch.float32 else _native.RUBS_F64
        pcode = _native.RUBS_F32 if pdt == torch.float32 else _native.RUBS_F64
        pp = [ctypes.c_void_p(p.data_ptr()) for p in ps]
        with torch.cuda.device(f.device):
            if lattice:
                _native.check(L.rubs_b200_filter3_lattice_params(
                    ctypes.c_void_p(f.data_ptr()), fdt, H, W, W, *pp, pcode, W, iterations, float(spacing),
                    ctypes.c_void_p(res.data_ptr()), W, _stream_handle()))
            else:
                _native.check(L.rubs_b200_filter3_params(
                    ctypes.c_void_p(f.data_ptr()), fdt, H, W, W, *pp, pcode, W, iterations,
                    ctypes.c_void_p(res.data_ptr()), W, _stream_handle()))
        return res
    img = _host_image(f)
    H, W = img.shape
    (s, r, t), shape, dt = _params_host(size, elongation, orientation)
    if shape != (H, W):
        s, r, t = (np.ascontiguousarray(np.broadcast_to(v, (H, W))) for v in (s, r, t))
    out = _host_out(out, (H, W))
    if H == 0 or W == 0:
        return out
    pcode = _native.RUBS_F32 if dt == np.float32 else _native.RUBS_F64
    if lattice:
        _native.check(L.rubs_b200_filter3_lattice_params_host(
            _ptr(img), _img_dtype_code(img.dtype), H, W, _ptr(s), _ptr(r), _ptr(t), pcode, iterations,
            float(spacing), _ptr(out)))
    else:
        _native.check(L.rubs_b200_filter3_params_host(
            _ptr(img), _img_dtype_code(img.dtype), H, W, _ptr(s), _ptr(r), _ptr(t), pcode, iterations,
            _ptr(out)))
    return out


def scales3_many(size, elongation, orientation):
    """The N=3 mapping on the device: (..., 3) float64 numpy scales."""
    (s, r, t), shape, dt = _params_host(size, elongation, orientation)
    n = int(np.prod(shape)) if shape else 1
    if n == 0:
        return np.empty(shape + (3,))
    torch = _torch()
    ds, dr, dth = (torch.from_numpy(v.reshape(-1)).cuda() for v in (s, r, t))
    res = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    _native.check(_native.load().rubs_b200_scales3(
        ctypes.c_void_p(ds.data_ptr()), ctypes.c_void_p(dr.data_ptr()), ctypes.c_void_p(dth.data_ptr()),
        _native.RUBS_F32 if dt == np.float32 else _native.RUBS_F64, n, ctypes.c_void_p(res.data_ptr()),
        _stream_handle()))
    return res.cpu().numpy().reshape(shape + (3,))
