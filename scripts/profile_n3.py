"""Short config-3 (N=3) run for ncu captures (dev tool): a few filter calls.

    python scripts/profile_n3.py [exact|lattice] [calls]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

mode = sys.argv[1] if len(sys.argv) > 1 else "lattice"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = workloads.config3_n3(device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
for _ in range(n):
    out = rb.filter_space_variant3_params(f, w["size"], w["elong"], w["orient"], mode=mode)
torch.cuda.synchronize()
print("ok", float(out.sum()))
