"""Split one device-API call into Python wrapper time and C-call time."""
import sys, time, ctypes
sys.path.insert(0, '.')
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads, _native
w = workloads.config2(device="cuda", param_dtype=torch.float32)
f = torch.from_numpy(w["f"]).cuda()
p = [w["size"], w["elong"], w["orient"]]
L = _native.load()
real = L.rubs_b200_filter_params
acc = [0.0]
class Wrap:
    def __call__(self, *a):
        t = time.perf_counter(); r = real(*a); acc[0] += time.perf_counter() - t; return r
for _ in range(5):
    rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
L.rubs_b200_filter_params = Wrap()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    rb.filter_space_variant_params(f, *p)
tot = (time.perf_counter() - t0) / n * 1e6
print(f"total {tot:.1f} us/call, inside C {acc[0] / n * 1e6:.1f} us, python {tot - acc[0] / n * 1e6:.1f} us")
