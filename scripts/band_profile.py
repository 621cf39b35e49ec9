"""One config-5 row band (dev, for ncu launch lists): world, rank from argv."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads, sharding
H = W = 32768
world, rank = int(sys.argv[1]), int(sys.argv[2])
w = workloads.config5(H, W, device="cuda", param_dtype=torch.float32, image_device="cuda")
f, p = w["f"], [w["size"], w["elong"], w["orient"]]
lut = rb.default_lut()
band = sharding.band_bounds(H, world)[rank]
pb = [v[band[0]:band[1]].contiguous() for v in p]
m = sharding.halo_bound_params(pb[0], lut)
n0, n1 = sharding.needed_rows(band, m, H)
fr = f[n0:n1].contiguous()
del f, w, p
for _ in range(3):
    out = sharding.filter_rows_params(fr, n0, H, *pb, band[0], band[0], band[1] - band[0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = sharding.filter_rows_params(fr, n0, H, *pb, band[0], band[0], band[1] - band[0])
e1.record(); torch.cuda.synchronize()
print("band ms", e0.elapsed_time(e1))
