import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle
from oracle import port
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads
w = workloads.config3(device="cuda", param_dtype=torch.float32)
f = torch.from_numpy(w["f"]).cuda()
out = rb.filter_space_variant_params(f, w["size"], w["elong"], w["orient"])
r, c = (3000, 5048), (5000, 6024)
params = [v[r[0]:r[1], c[0]:c[1]].cpu().numpy() for v in (w["size"], w["elong"], w["orient"])]
lut = rb.default_lut()
fl = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, *params)
full = torch.zeros((8192, 8192, 4), dtype=torch.float64, device="cuda")
full[r[0]:r[1], c[0]:c[1]] = torch.from_numpy(fl).cuda()
ref = oracle.dense_cuda(f.double(), full, rows=r, cols=c).cpu().numpy()
got = out[r[0]:r[1], c[0]:c[1]].cpu().numpy()
err = np.abs(got - ref)
print("max err", err.max(), "ref max", np.abs(ref).max())
idx = np.argsort(err.ravel())[::-1][:6]
flm = np.maximum(fl, 0.05)
for i in idx:
    y, x = divmod(i, got.shape[1])
    a = flm[y, x]
    print(y + r[0], x + c[0], "err %.2e" % err[y, x], "a", np.round(a, 3), "w %.3g" % (1 / a.prod()), "size", params[0][y, x], "rho", params[1][y, x])
big = err > 1e-9
print("pixels > 1e-9:", big.sum(), "rows", np.unique(np.nonzero(big)[0] + r[0])[:20], "cols", np.unique(np.nonzero(big)[1] + c[0])[:20])
