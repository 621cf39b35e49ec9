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


def build() -> str:
    """Compile the C oracle (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


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
