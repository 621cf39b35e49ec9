"""A/B timing (dev): config 3 (N=3) through the fused-params entry, device
time per call and a checksum.  RUBS_B200_LIB selects the build.

    python scripts/ab_n3.py [exact|lattice] [H]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

mode = sys.argv[1] if len(sys.argv) > 1 else "lattice"
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
w = workloads.config3_n3(H, H, device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
p = (w["size"], w["elong"], w["orient"])
for _ in range(3):
    out = rb.filter_space_variant3_params(f, *p, mode=mode)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = rb.filter_space_variant3_params(f, *p, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"config 3 {mode} {H}^2: sum {float(out.sum()):.10e} ms {min(ts):.3f} {[round(t, 3) for t in ts]}")
