"""Per-call host overhead of the device API (config 2): wall time per call
vs the primary kernel's event time."""
import sys, time, ctypes
sys.path.insert(0, '.')
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads, _native
w = workloads.config2(device="cuda", param_dtype=torch.float32)
f = torch.from_numpy(w["f"]).cuda()
p = [w["size"], w["elong"], w["orient"]]
L = _native.load()
for _ in range(5):
    rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
L.rubs_b200_reset_kernel_time(); L.rubs_b200_set_profiling(1)
n = 200
t0 = time.perf_counter()
for _ in range(n):
    rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / n * 1e3
L.rubs_b200_set_profiling(0)
ms, cnt = ctypes.c_double(), ctypes.c_int64()
L.rubs_b200_kernel_time(0, ctypes.byref(ms), ctypes.byref(cnt))
print(f"wall {el:.4f} ms/call, kernel {ms.value / cnt.value:.4f} ms, overhead {el - ms.value / cnt.value:.4f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(100):
    rb.filter_space_variant_params(f, *p)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
