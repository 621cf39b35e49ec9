"""Per-step device time of one bench config (dev only): is the step time
bimodal across steps / processes?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "3n4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
dev = torch.device("cuda", 0)
w = workloads.config3(device=dev, param_dtype=torch.float32) if cfg == "3n4" else \
    workloads.config5(device=dev, param_dtype=torch.float32, image_device=dev)
f = torch.as_tensor(w["f"]).to(dev)
p = [w["size"], w["elong"], w["orient"]]
ts = []
for i in range(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rb.filter_space_variant_params(f, *p)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(cfg, " ".join(f"{t:.1f}" for t in ts))
print("free GB", torch.cuda.mem_get_info()[0] / 1e9)
