"""Dev: cost of the pieces of the device fast path in Python (us per call)."""
import ctypes
import os
import sys
import timeit

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1003_2022_b200 as rb  # noqa: E402
from paper_1003_2022_b200 import _native, engine, workloads  # noqa: E402

w = workloads.config2(256, 256, device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
p = (w["size"], w["elong"], w["orient"])
rb.filter_space_variant_params(f, *p)
L = _native.load()
n = 20000


def t(stmt):
    return timeit.timeit(stmt, number=n, globals=globals()) / n * 1e6


print(f"fast_device_args {t('engine._fast_device_args(f, p)'):.2f} us")
print(f"device_lut {t('engine.device_lut(None, f.get_device())'):.2f} us")
print(f"empty_like {t('torch.empty_like(f, dtype=torch.float64)'):.2f} us")
print(f"current_stream {t('torch.cuda.current_stream().cuda_stream'):.2f} us")
print(f"data_ptr x5 {t('f.data_ptr(); p[0].data_ptr(); p[1].data_ptr(); p[2].data_ptr(); f.data_ptr()'):.2f} us")
print(f"get_device {t('f.get_device()'):.2f} us, current_device {t('torch.cuda.current_device()'):.2f} us")
print(f"launch count (ctypes no-arg) {t('L.rubs_b200_launch_count()'):.2f} us")
torch.cuda.synchronize()
print(f"whole call (256^2, kernel ~10 us) {t('rb.filter_space_variant_params(f, *p)'):.2f} us")
