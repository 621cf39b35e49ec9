"""Structure-tensor driven adaptive smoothing on the B200 -- the reference's
own caller of the filter path (pkg/src/rubs/tensor.py).

Same functions, arguments and exceptions as the reference module:

  structure_tensor(f, window_sigma=1.5)             tensor.py:52-75
  anisotropy_from_tensor(j, noise_sigma, ...)       tensor.py:90-171
  adaptive_smooth(f, noise_sigma, ...)              tensor.py:174-224

Every step runs on the device (csrc/rubs_tensor.cu through the C ABI):
the gradient / tensor kernel, the three isotropic window passes and the two
space-variant passes are the hot path's own kernels; the 5th / 95th trace
percentiles are exact order statistics from a device radix select.
numpy inputs come back as numpy arrays, torch CUDA tensors stay on the
device.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np

from . import _native
from .engine import _is_torch, _stream_handle, _torch, device_lut
from .solver import ScaleLut, default_lut

__all__ = [
    "structure_tensor",
    "anisotropy_from_tensor",
    "adaptive_smooth",
    "default_lut",
    "AnisotropyMaps",
]


class AnisotropyMaps(NamedTuple):
    """Per-pixel ellipse parameters derived from a structure tensor
    (tensor.py:43-49)."""

    size: object
    elongation: object
    orientation: object
    isotropic: object  # bool: no usable orientation here


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def _device_image(f):
    """(tensor on the device, was_numpy); float32 stays float32 (the
    widening to float64 is exact, on chip), everything else is float64
    like np.asarray(f, dtype=float64) (tensor.py:63)."""
    torch = _torch()
    if _is_torch(f):
        t = f if f.dtype in (torch.float32, torch.float64) else f.to(torch.float64)
        if not t.is_cuda:
            t = t.cuda()
        host = False
    else:
        a = np.asarray(f)
        if a.dtype != np.float32:
            a = np.asarray(a, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        host = True
    if t.dim() != 2:
        raise ValueError("image must be 2-D")
    return t.contiguous(), host


def _dtype_code(t):
    return _native.RUBS_F32 if t.dtype == _torch().float32 else _native.RUBS_F64


def structure_tensor(f, window_sigma: float = 1.5):
    """Gradient structure tensor, shape (H, W, 3): J11, J12, J22
    (tensor.py:52-75)."""
    t, host = _device_image(f)
    window_sigma = float(window_sigma)
    if window_sigma < 0.0:
        raise ValueError("window_sigma must be >= 0")
    torch = _torch()
    H, W = t.shape
    j = torch.zeros((H, W, 3), dtype=torch.float64, device=t.device)
    if H and W:
        with torch.cuda.device(t.device):
            _native.check(_native.load().rubs_b200_structure_tensor(
                _vp(t), _dtype_code(t), H, W, W, window_sigma, _vp(j), _stream_handle()))
    return j.cpu().numpy() if host else j


def anisotropy_from_tensor(j, noise_sigma: float, *, size_range=None, bound_fraction: float = 0.95,
                           iso_gain: float = 1.0) -> AnisotropyMaps:
    """Smoothing-ellipse parameters from a structure tensor
    (tensor.py:90-171)."""
    torch = _torch()
    host = not _is_torch(j)
    jt = torch.as_tensor(np.asarray(j, dtype=np.float64)) if host else j.to(torch.float64)
    if jt.dim() != 3 or jt.shape[2] != 3:
        raise ValueError(f"structure tensor must be (H, W, 3), got {tuple(jt.shape)}")
    if not 0.0 < bound_fraction < 1.0:
        raise ValueError("bound_fraction must lie in (0, 1)")
    if size_range is not None:
        s_min, s_max = (float(v) for v in size_range)
        if not (0.0 < s_min <= s_max):
            raise ValueError("size_range must be positive and ordered")
    jt = jt.cuda().contiguous()
    H, W = jt.shape[:2]
    maps = torch.empty((3, H, W), dtype=torch.float64, device=jt.device)
    iso = torch.empty((H, W), dtype=torch.uint8, device=jt.device)
    if H and W:
        sr = (ctypes.c_double * 2)(*size_range) if size_range is not None else None
        with torch.cuda.device(jt.device):
            _native.check(_native.load().rubs_b200_anisotropy(
                _vp(jt), H, W, float(noise_sigma), sr, float(bound_fraction), float(iso_gain),
                _vp(maps[0]), _vp(maps[1]), _vp(maps[2]), _vp(iso), _stream_handle()))
    out = (maps[0], maps[1], maps[2], iso.bool())
    if host:
        out = tuple(v.cpu().numpy() for v in out)
    return AnisotropyMaps(*out)


def adaptive_smooth(f, noise_sigma: float, *, window_sigma: float = 1.5, iterations: int = 1,
                    lut: ScaleLut | None = None, bound_fraction: float = 0.95, size_range=None,
                    iso_gain: float = 1.0, out=None):
    """Smooth an image with per-pixel oriented elliptical kernels
    (tensor.py:174-224): structure tensor, anisotropy maps, LUT mapping,
    the space-variant filter of f and of a flat image, gain correction.
    ``out`` (extension): a C-contiguous float64 host array (e.g. pinned) to
    receive a numpy caller's result."""
    t, host = _device_image(f)
    if noise_sigma < 0.0:
        raise ValueError("noise_sigma must be >= 0")
    if window_sigma < 0.0:
        raise ValueError("window_sigma must be >= 0")
    if int(iterations) < 1:
        raise ValueError("iterations must be >= 1")
    if not 0.0 < bound_fraction < 1.0:
        raise ValueError("bound_fraction must lie in (0, 1)")
    if size_range is not None:
        s_min, s_max = (float(v) for v in size_range)
        if not (0.0 < s_min <= s_max):
            raise ValueError("size_range must be positive and ordered")
    torch = _torch()
    dl = device_lut(lut if lut is not None else default_lut(), t.device)
    H, W = t.shape
    res = torch.empty((H, W), dtype=torch.float64, device=t.device)
    if H and W:
        sr = (ctypes.c_double * 2)(*size_range) if size_range is not None else None
        with torch.cuda.device(t.device):
            _native.check(_native.load().rubs_b200_adaptive_smooth(
                _vp(t), _dtype_code(t), H, W, W, float(noise_sigma), float(window_sigma),
                int(iterations), dl.handle, float(bound_fraction), sr, float(iso_gain), _vp(res), W,
                _stream_handle()))
    if not host:
        return res
    if out is None:
        return res.cpu().numpy()
    if out.shape != (H, W) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array of the image shape")
    torch.from_numpy(out).copy_(res)
    return out
