"""Dev probe: raw pinned H2D / D2H bandwidth vs the e2e host-buffer call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

n = 84 * 2**20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print("H2D GB/s", 10 * n / (time.perf_counter() - t) / 1e9)
t = time.perf_counter()
for _ in range(10):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print("D2H GB/s", 10 * n / (time.perf_counter() - t) / 1e9)
s2 = torch.cuda.Stream()
t = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2 = h  # same buffer both ways is fine for bandwidth
        h2.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print("duplex GB/s (each way)", 10 * n / (time.perf_counter() - t) / 1e9)

w = workloads.config2(param_dtype=torch.float32)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
f = pin(w["f"])
ps = [pin(v.numpy()) for v in (w["size"], w["elong"], w["orient"])]
out = pin(np.empty((2048, 2048)))
for _ in range(3):
    rb.filter_space_variant_params(f, *ps, out=out)
t = time.perf_counter()
for _ in range(10):
    rb.filter_space_variant_params(f, *ps, out=out)
dt = (time.perf_counter() - t) / 10
print("e2e ms", dt * 1e3, "Gpx/s", 2048 * 2048 / dt / 1e9, "H2D-bound ms at 55 GB/s", 84e6 / 55e9 * 1e3)
