"""The lattice mode's own error (dev / DESIGN.md §9b): N=3 lattice mode
against the exact N=3 mode on the config-3 recipe, per lattice spacing.

    python scripts/lattice_error.py [H]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

H = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = workloads.config3_n3(H, H, device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
p = (w["size"], w["elong"], w["orient"])
ex = rb.filter_space_variant3_params(f, *p)
scale = float(ex.abs().max())
print(f"# config-3 recipe at {H}^2 (rectangles + noise 0.05, sigma 1-32); error of mode=lattice against mode=exact,")
print("# relative to max |exact output|; device ms per call (CUDA events)")
print("spacing\tmax_rel\trms_rel\tms")
for h in (1.0, 0.75, 0.5, 0.25):
    for _ in range(2):
        lat = rb.filter_space_variant3_params(f, *p, mode="lattice", spacing=h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lat = rb.filter_space_variant3_params(f, *p, mode="lattice", spacing=h)
    e1.record()
    torch.cuda.synchronize()
    d = (lat - ex)
    print(f"{h:g}\t{float(d.abs().max()) / scale:.3e}\t{float(d.pow(2).mean().sqrt()) / scale:.3e}\t{e0.elapsed_time(e1):.3f}")
# smooth image: the resampling error falls with the kernel size
yy, xx = np.mgrid[0:512, 0:512]
g = torch.from_numpy(np.sin(xx / 9.0) * np.cos(yy / 13.0) + 0.5).cuda()
print("# smooth 512^2 image, uniform isotropic kernels a1 = a2 = a3 = a, spacing 1: max rel error (interior)")
print("a\tmax_rel")
for a in (2.0, 4.0, 8.0, 16.0, 32.0, 64.0):
    v = np.array([a, a, a])
    e = rb.filter_space_variant3(g, v)[128:384, 128:384]
    l = rb.filter_space_variant3(g, v, mode="lattice")[128:384, 128:384]
    print(f"{a:g}\t{float((l - e).abs().max() / e.abs().max()):.3e}")
