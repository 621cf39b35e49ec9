"""Config-5 recipe at a reduced size (dev timing / profiling of the
large-halo path)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads, _native
import ctypes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = workloads.config5(n, n, device="cuda", param_dtype=torch.float32, image_device="cuda")
f, p = w["f"], [w["size"], w["elong"], w["orient"]]
rb.filter_space_variant_params(f, *p)
torch.cuda.synchronize()
L = _native.load()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    rb.filter_space_variant_params(f, *p)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"n={n}: {ms:.2f} ms/call, {n*n/ms/1e6:.2f} Gpx/s")
