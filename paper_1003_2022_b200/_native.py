"""ctypes binding of the C ABI in include/rubs_b200.h.

The shared library is built in-tree (``build_native``) as
``paper_1003_2022_b200/_lib/librubs_b200.so`` for sm_100a.  There is no CPU
fallback: if the library is missing or CUDA is unavailable every entry point
raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_PKG)
LIB_DIR = os.path.join(_PKG, "_lib")
# RUBS_B200_LIB: load an alternative build (A/B experiments; see build_native)
LIB_PATH = os.environ.get("RUBS_B200_LIB") or os.path.join(LIB_DIR, "librubs_b200.so")
CSRC = os.path.join(_PKG, "csrc")
INCLUDE = os.path.join(_REPO, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

(RUBS_OK, RUBS_EVALUE, RUBS_EOVERFLOW, RUBS_EOUTOFGRID, RUBS_ECUDA, RUBS_EUNSUPPORTED,
 RUBS_EINFEASIBLE) = range(7)
RUBS_F32, RUBS_F64 = 0, 1


def build_native(verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile csrc/*.cu into the in-tree shared library (sm_100a).
    ``defines``/``out`` build a variant library for A/B runs."""
    os.makedirs(LIB_DIR, exist_ok=True)
    out = out or LIB_PATH
    srcs = [os.path.join(CSRC, n) for n in ("rubs_b200.cu", "rubs_tensor.cu", "rubs_n3.cu", "rubs_n3_lattice.cu")]
    cmd = ["nvcc", *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", INCLUDE, "-o", out + ".tmp",
           *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)
_dbl = ctypes.c_double

# name -> (restype, argtypes); kept identical to include/rubs_b200.h
SIGNATURES = {
    "rubs_b200_version": (ctypes.c_char_p, []),
    "rubs_b200_last_error": (ctypes.c_char_p, []),
    "rubs_b200_launch_count": (_i64, []),
    "rubs_b200_reset_launch_count": (None, []),
    "rubs_b200_set_profiling": (None, [_int]),
    "rubs_b200_kernel_time": (None, [_int, _dp, _lp]),
    "rubs_b200_reset_kernel_time": (None, []),
    "rubs_b200_dfma_peak": (_int, [_dp, _dp]),
    "rubs_b200_precision_limited": (_int, []),
    "rubs_b200_filter": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _int, _vp, _i64, _vp]),
    "rubs_b200_filter_host": (_int, [_vp, _int, _i64, _i64, _vp, _int, _int, _vp]),
    "rubs_b200_lut_create": (_int, [_vp, _vp, _vp, _int, _int, ctypes.POINTER(_vp)]),
    "rubs_b200_lut_destroy": (None, [_vp]),
    "rubs_b200_lookup": (_int, [_vp, _vp, _vp, _vp, _int, _i64, _vp, _vp]),
    "rubs_b200_filter_params": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _int, _i64, _vp,
                                       _int, _vp, _i64, _vp]),
    "rubs_b200_filter_params_host": (_int, [_vp, _int, _i64, _i64, _vp, _vp, _vp, _int, _vp, _int,
                                            _vp]),
    "rubs_b200_filter_params_batch_host": (_int, [_int, _vp, _int, _i64, _i64, _vp, _vp, _vp, _int, _vp,
                                                  _int, _vp, ctypes.POINTER(_int)]),
    "rubs_b200_filter_rows": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64,
                                     _i64, _vp, _i64, _vp]),
    "rubs_b200_filter_params_rows": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _int,
                                            _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp]),
    "rubs_b200_read_margins": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _int,
                                      ctypes.POINTER(_int), _vp]),
    "rubs_b200_read_margins_params": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _i64, _i64, _i64, _vp,
                                             _int, ctypes.POINTER(_int), _vp]),
    "rubs_b200_preintegrate_shape": (_int, [_i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _lp,
                                            _lp, _lp, _lp]),
    "rubs_b200_preintegrate": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                      _i64, _vp, _i64, _vp]),
    "rubs_b200_interpolate": (_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp]),
    "rubs_b200_structure_tensor": (_int, [_vp, _int, _i64, _i64, _i64, _dbl, _vp, _vp]),
    "rubs_b200_anisotropy": (_int, [_vp, _i64, _i64, _dbl, _vp, _dbl, _dbl, _vp, _vp, _vp, _vp, _vp]),
    "rubs_b200_adaptive_smooth": (_int, [_vp, _int, _i64, _i64, _i64, _dbl, _dbl, _int, _vp, _dbl, _vp,
                                         _dbl, _vp, _i64, _vp]),
    "rubs_b200_filter3": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _int, _vp, _i64, _vp]),
    "rubs_b200_filter3_host": (_int, [_vp, _int, _i64, _i64, _vp, _int, _int, _vp]),
    "rubs_b200_filter3_params": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _int, _i64, _int,
                                        _vp, _i64, _vp]),
    "rubs_b200_filter3_lattice": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _int, _dbl, _vp,
                                         _i64, _vp]),
    "rubs_b200_filter3_lattice_params": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _int, _i64,
                                                _int, _dbl, _vp, _i64, _vp]),
    "rubs_b200_filter3_lattice_params_rows": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _vp,
                                                     _vp, _int, _i64, _i64, _i64, _i64, _dbl, _vp, _i64,
                                                     _vp]),
    "rubs_b200_filter3_lattice_host": (_int, [_vp, _int, _i64, _i64, _vp, _int, _int, _dbl, _vp]),
    "rubs_b200_filter3_lattice_params_host": (_int, [_vp, _int, _i64, _i64, _vp, _vp, _vp, _int, _int,
                                                     _dbl, _vp]),
    "rubs_b200_filter3_params_host": (_int, [_vp, _int, _i64, _i64, _vp, _vp, _vp, _int, _int, _vp]),
    "rubs_b200_scales3": (_int, [_vp, _vp, _vp, _int, _i64, _vp, _vp]),
    "rubs_b200_read_margins3_params": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _i64,
                                              ctypes.POINTER(_int), _vp]),
    "rubs_b200_filter3_params_rows": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                             _int, _i64, _i64, _i64, _i64, _vp, _i64, _vp]),
}


def load(path: str | None = None):
    """Load the shared library (CPU-safe: loading needs no GPU)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"native library {p} is missing; build it with "
            "paper_1003_2022_b200._native.build_native() (no CPU fallback exists)")
    L = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = L
    return L


class PrecisionWarning(RuntimeWarning):
    """A filter call met needle kernels (rubs_b200_precision_limited)."""


def check(rc: int) -> None:
    """Map a C status to the reference's exception classes."""
    if rc == RUBS_OK:
        if _lib is not None and _lib.rubs_b200_precision_limited():
            import warnings
            warnings.warn("some kernels are too anisotropic for the float64 running sums (three widths at "
                          "the 0.05 floor next to a long one): their pixels may be accurate to ~1e-8 "
                          "relative instead of 1e-9", PrecisionWarning, stacklevel=3)
        return
    msg = load().rubs_b200_last_error().decode(errors="replace")
    if rc == RUBS_EVALUE:
        raise ValueError(msg)
    if rc == RUBS_EOVERFLOW:
        raise OverflowError(msg)
    if rc == RUBS_EOUTOFGRID:
        from .solver import OutOfGrid
        raise OutOfGrid(msg)
    if rc == RUBS_EINFEASIBLE:
        from .solver import Infeasible
        raise Infeasible(msg)
    raise RuntimeError(f"rubs_b200 error {rc}: {msg}")
