import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
os.chdir('/root/repo')
import numpy as np
from conftest import golden
from oracle import tensor_port, port
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import tensor
g = golden("tensor.npz")
lut = rb.default_lut(); lt = (lut.rho_grid, lut.phi_grid, lut.entries)
f = g["noisy"]
j = tensor.structure_tensor(f, 1.5)
got = tensor.adaptive_smooth(f, 0.1)
size, rho, theta, iso = tensor_port.anisotropy_from_tensor(j, 0.1)
rho = np.minimum(rho, lut.rho_grid[-1] * (1 - 1e-9))
field = np.maximum(port.lookup_many(*lt, size, rho, theta), 0.05)
w = 1 / field.prod(-1)
ex = tensor_port.adaptive_smooth(f, 0.1, lt, j=j)
err = np.abs(got - ex)
idx = np.argsort(err.ravel())[::-1][:8]
for i in idx:
    r, c = divmod(i, f.shape[1])
    print(r, c, "err %.2e" % err[r, c], "w %.3g" % w[r, c], "a", np.round(field[r, c], 3))
print("w max", w.max(), "frac w>1e4", (w > 1e4).mean(), "err median", np.median(err))
# filter stage alone: out = filter(f, field) vs dense
import oracle
out_gpu = rb.filter_space_variant(f, field)
out_ex = oracle.dense(f, field)
e2 = np.abs(out_gpu - out_ex)
print("filter stage max err", e2.max(), "at w", w.ravel()[e2.argmax()])
