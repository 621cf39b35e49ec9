"""A/B check (dev): bit-level checksum of the config-5 output (or another
config) under the current environment, for comparing kernel variants that
must agree bitwise (e.g. RUBS_B200_BIG_GATHER=l1 vs the windowed gather).

    python scripts/ab_hash.py [config] [H]
"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1003_2022_b200 as rb  # noqa: E402
from paper_1003_2022_b200 import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
if cfg == "5":
    w = workloads.config5(H, H, device="cuda", param_dtype=torch.float32, image_device="cuda")
    f = w["f"]
elif cfg == "3n4":
    w = workloads.config3(H, H, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
else:
    w = workloads.config4_image(0, H, H, device="cuda", param_dtype=torch.float32)
    f = torch.from_numpy(w["f"]).cuda()
p = (w["size"], w["elong"], w["orient"])
it = int(w["iterations"])
out = rb.filter_space_variant_params(f, *p, iterations=it)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = rb.filter_space_variant_params(f, *p, iterations=it)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
bits = out.view(torch.int64).flatten()
idx = torch.arange(bits.numel(), device=bits.device, dtype=torch.int64)
h = int(((bits ^ (idx * 0x9E3779B97F4A7C15)) * 0x100000001B3).sum().item())
print(f"config {cfg} {H}^2: hash {h & 0xFFFFFFFFFFFFFFFF:016x} ms {min(ts):.2f} {ts}")
