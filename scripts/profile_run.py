"""Short config-2 run for ncu captures (dev tool): a few filter calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg == "2":
    w = workloads.config2(device="cuda", param_dtype=torch.float32)
else:
    w = workloads.config4_image(0, device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
for _ in range(n):
    out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"], iterations=w["iterations"])
torch.cuda.synchronize()
print("ok", float(out.sum()))
