"""Dev tool: a few config-5-recipe filter calls at a reduced size (ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
w = workloads.config5(n, n, device="cuda", param_dtype=torch.float32, image_device="cuda")
for _ in range(2):
    out = rb.filter_space_variant_params(w["f"], w["size"], w["elong"], w["orient"])
torch.cuda.synchronize()
print("ok", float(out.sum()))
