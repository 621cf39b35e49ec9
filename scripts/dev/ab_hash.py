"""A/B of two library builds (dev only): output hash + median step time per
workload.  RUBS_B200_LIB selects the build."""
import hashlib
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

dev = torch.device("cuda", 0)
runs = {}
def add(name, fn):
    runs[name] = fn
w = workloads.config2(device=dev)
f2 = torch.as_tensor(w["f"]).to(dev); p2 = [w["size"], w["elong"], w["orient"]]
add("2", lambda: rb.filter_space_variant_params(f2, *p2))
w = workloads.config3(device=dev, param_dtype=torch.float32)
f3 = torch.as_tensor(w["f"]).to(dev); p3 = [w["size"], w["elong"], w["orient"]]
add("3n4", lambda: rb.filter_space_variant_params(f3, *p3))
w = workloads.config4_image(0, device=dev, param_dtype=torch.float32)
f4 = torch.as_tensor(w["f"]).to(dev); p4 = [w["size"], w["elong"], w["orient"]]
add("4", lambda: rb.filter_space_variant_params(f4, *p4, iterations=2))
w = workloads.config5(8192, 8192, device=dev, param_dtype=torch.float32, image_device=dev)
f5 = torch.as_tensor(w["f"]).to(dev); p5 = [w["size"], w["elong"], w["orient"]]
add("5@8192", lambda: rb.filter_space_variant_params(f5, *p5))
wa = workloads.adaptive_image()
fa = torch.as_tensor(wa["f"]).to(dev)
add("A", lambda: rb.adaptive_smooth(fa, wa["noise_sigma"]))
fc = torch.full((1024, 1024), 0.3, dtype=torch.float64, device=dev)
add("A-flat", lambda: rb.adaptive_smooth(fc, 0.1))
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, fn in runs.items():
    if only and name not in only:
        continue
    out = fn()
    torch.cuda.synchronize()
    h = hashlib.sha1(out.double().cpu().numpy().tobytes()).hexdigest()[:16]
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:8s} {h} {np.median(ts):8.3f} ms")
