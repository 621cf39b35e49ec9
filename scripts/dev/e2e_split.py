"""e2e (host-buffer call) time of config 2 vs the bare copies of its bytes."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads
w = workloads.config2(param_dtype=torch.float32)
H, W = w["f"].shape
hf = torch.empty((H, W), dtype=torch.float64, pin_memory=True); hf.copy_(torch.from_numpy(w["f"]))
hp = []
for v in (w["size"], w["elong"], w["orient"]):
    t = torch.empty(v.shape, dtype=v.dtype, pin_memory=True); t.copy_(v); hp.append(t.numpy())
hout = torch.empty((H, W), dtype=torch.float64, pin_memory=True).numpy()
hfn = hf.numpy()
lut = rb.default_lut()
for _ in range(3):
    rb.filter_space_variant_params(hfn, *hp, lut=lut, out=hout)
n = 20
t0 = time.perf_counter()
for _ in range(n):
    rb.filter_space_variant_params(hfn, *hp, lut=lut, out=hout)
e2e = (time.perf_counter() - t0) / n * 1e3
# bare copies of the same bytes, H2D and D2H on two streams
d_in = torch.empty(hf.numel() * 2 + 3 * H * W // 2 * 2, dtype=torch.float64, device="cuda")
hin = torch.empty(d_in.numel(), dtype=torch.float64, pin_memory=True)
d_out = torch.empty((H, W), dtype=torch.float64, device="cuda")
ho = torch.from_numpy(hout)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    with torch.cuda.stream(s1):
        d_in[: (8 + 12) * H * W // 8].copy_(hin[: (8 + 12) * H * W // 8], non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
bare = (time.perf_counter() - t0) / n * 1e3
print(f"e2e {e2e:.3f} ms/call ({H*W/e2e/1e6:.2f} Gpx/s); bare H2D 80 MiB || D2H 32 MiB: {bare:.3f} ms")
