"""Dev: per-call overhead of the device API on config 2 (2048^2): wall time
per call through the Python API and through a bare ctypes call with
precomputed arguments, against the primary kernel's CUDA-event time."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1003_2022_b200 as rb  # noqa: E402
from paper_1003_2022_b200 import _native, workloads  # noqa: E402
from paper_1003_2022_b200.engine import device_lut  # noqa: E402

w = workloads.config2(device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
p = [w["size"], w["elong"], w["orient"]]
L = _native.load()
n = 200
for _ in range(10):
    rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
L.rubs_b200_reset_kernel_time()
L.rubs_b200_set_profiling(1)
t0 = time.perf_counter()
for _ in range(n):
    rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
api = (time.perf_counter() - t0) / n * 1e3
L.rubs_b200_set_profiling(0)
km, kn = ctypes.c_double(), ctypes.c_int64()
L.rubs_b200_kernel_time(0, ctypes.byref(km), ctypes.byref(kn))
out = torch.empty_like(f)
dl = device_lut(None)
args = (ctypes.c_void_p(f.data_ptr()), _native.RUBS_F64, 2048, 2048, 2048, ctypes.c_void_p(p[0].data_ptr()),
        ctypes.c_void_p(p[1].data_ptr()), ctypes.c_void_p(p[2].data_ptr()), _native.RUBS_F32, 2048, dl.handle, 1,
        ctypes.c_void_p(out.data_ptr()), 2048, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
fn = L.rubs_b200_filter_params
t0 = time.perf_counter()
for _ in range(n):
    fn(*args)
torch.cuda.synchronize()
bare = (time.perf_counter() - t0) / n * 1e3
print(f"API call {api:.4f} ms, bare ctypes call {bare:.4f} ms, pass kernels {km.value / max(kn.value, 1):.4f} ms")
