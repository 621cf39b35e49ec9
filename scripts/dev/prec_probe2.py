import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from oracle import tensor_port, port
import oracle
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import tensor
rng = np.random.default_rng(9)
img = tensor_port.stripe_image((160, 176), period=13.0, angle=0.9) + rng.normal(0.0, 0.1, (160, 176))
kw = dict(size_range=(0.5, 3000.0))
j = tensor.structure_tensor(img, 1.5)
size, rho, theta, iso = tensor_port.anisotropy_from_tensor(j, 0.1, **kw)
lut = rb.default_lut(); lt = (lut.rho_grid, lut.phi_grid, lut.entries)
rho = np.minimum(rho, lut.rho_grid[-1] * (1 - 1e-9))
field = np.maximum(port.lookup_many(*lt, size, rho, theta), 0.05)
out_g = rb.filter_space_variant(img, field)
out_e = oracle.dense(img, field)
e = np.abs(out_g - out_e)
i = e.argmax(); r, c = divmod(i, img.shape[1])
print("filter stage max abs err", e.max(), "at", r, c, "a", field[r, c], "w", 1/field[r, c].prod())
print("size range", size.min(), size.max(), "frac size>100", (size > 100).mean())
ones_g = rb.filter_space_variant(np.ones_like(img), field)
ones_e = oracle.dense(np.ones_like(img), field)
e2 = np.abs(ones_g - ones_e); i2 = e2.argmax()
print("gain stage max abs err", e2.max(), "gain there", ones_e.ravel()[i2], "min |gain|", np.abs(ones_e).min())
got = tensor.adaptive_smooth(img, 0.1, **kw)
ex = tensor_port.adaptive_smooth(img, 0.1, lt, j=j, **kw)
e3 = np.abs(got - ex); i3 = e3.argmax(); r3, c3 = divmod(i3, img.shape[1])
print("final max err", e3.max(), "at", r3, c3, "gain", ones_e[r3, c3], "out", out_e[r3, c3])
