"""Dev tool: where does the end-to-end (host buffers) time go?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads
w = workloads.config2(param_dtype=torch.float32)
H, W = w["f"].shape
hf = torch.empty((H, W), dtype=torch.float64, pin_memory=True); hf.copy_(torch.from_numpy(w["f"]))
hp = []
for v in (w["size"], w["elong"], w["orient"]):
    t = torch.empty(v.shape, dtype=torch.float32, pin_memory=True); t.copy_(v); hp.append(t.numpy())
lut = rb.default_lut()
for _ in range(3): rb.filter_space_variant_params(hf.numpy(), *hp, lut=lut)
t0 = time.perf_counter(); n = 10
for _ in range(n): rb.filter_space_variant_params(hf.numpy(), *hp, lut=lut)
print("e2e ms/call", (time.perf_counter() - t0) / n * 1e3)
d = torch.empty((H, W), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(n): d.copy_(hf, non_blocking=True)
torch.cuda.synchronize(); print("H2D 32MB pinned ms", (time.perf_counter() - t0) / n * 1e3)
o = torch.empty((H, W), dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(n): o.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("D2H 32MB pinned ms", (time.perf_counter() - t0) / n * 1e3)
out_np = np.empty((H, W))
t0 = time.perf_counter()
for _ in range(n): out_np[...] = 0
print("host memset 32MB ms", (time.perf_counter() - t0) / n * 1e3)
