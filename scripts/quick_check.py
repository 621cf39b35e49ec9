"""Ad-hoc GPU sanity check (dev tool): CUDA path vs exact dense oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

rng = np.random.default_rng(5)
def smooth_field(shape, lo, hi):
    h, w = shape
    c = rng.standard_normal((max(h // 8, 2), max(w // 8, 2)))
    ys = np.linspace(0, c.shape[0] - 1.0, h); xs = np.linspace(0, c.shape[1] - 1.0, w)
    yi = np.minimum(ys.astype(int), c.shape[0] - 2); xi = np.minimum(xs.astype(int), c.shape[1] - 2)
    fy = (ys - yi)[:, None]; fx = (xs - xi)[None, :]
    s = (c[yi][:, xi] * (1 - fy) * (1 - fx) + c[yi][:, xi + 1] * (1 - fy) * fx + c[yi + 1][:, xi] * fy * (1 - fx) + c[yi + 1][:, xi + 1] * fy * fx)
    return lo + (s - s.min()) * (hi - lo) / (s.max() - s.min())

for (H, W, m) in [(18, 16, 1), (20, 24, 1), (14, 15, 2), (64, 64, 1), (40, 50, 2)]:
    f = rng.random((H, W))
    field = np.stack([smooth_field((H, W), 0.8, 2.5) for _ in range(4)], axis=-1)
    t = time.time(); out = rb.filter_space_variant(f, field, m); tg = time.time() - t
    ref = oracle.dense(f, field, m)
    print(f"{H}x{W} m={m}: max abs err {np.abs(out - ref).max():.3e}  gpu {tg*1e3:.1f} ms", flush=True)

# impulse
a = np.array([1.1, 2.3, 0.8, 1.6]); fi = np.zeros((25, 31)); fi[7, 22] = 1
out = rb.filter_space_invariant(fi, a)
x1 = np.arange(31.0)[None, :] - 22; x2 = np.arange(25.0)[:, None] - 7
print("impulse err", np.abs(out - oracle.kernel_values(a, x1, x2)).max())
# config 1
c1 = workloads.config1()
t = time.time(); out = rb.filter_space_variant(c1["f"], c1["field"]); print("config1 gpu s", time.time() - t)
pts = np.stack([rng.integers(0, 256, 400), rng.integers(0, 256, 400)], axis=1)
pts = np.concatenate([pts, [[0, 0], [0, 255], [255, 0], [255, 255]]])
t = time.time(); ref = oracle.points(c1["f"], c1["field"], pts); print("oracle s", time.time() - t)
got = out[pts[:, 0], pts[:, 1]]
print("config1 max rel err", (np.abs(got - ref) / np.abs(ref).max()).max())
# config 2 fused
import torch
c2 = workloads.config2(device="cuda", param_dtype=torch.float32)
f = torch.from_numpy(c2["f"]).cuda()
for it in range(3):
    torch.cuda.synchronize(); t = time.time()
    out = rb.filter_space_variant_params(f, c2["size"], c2["elong"], c2["orient"])
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"config2 fused: {dt*1e3:.2f} ms  {2048*2048/dt/1e9:.2f} Gpx/s")
lut = rb.default_lut()
s, r, th = (v.double().cpu().numpy() for v in (c2["size"], c2["elong"], c2["orient"]))
pts = np.stack([rng.integers(0, 2048, 200), rng.integers(0, 2048, 200)], axis=1)
pts = np.concatenate([pts, [[0, 0], [0, 2047], [2047, 0], [2047, 2047]]])
from oracle import port
field_pts = None
fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, s, r, th)
t = time.time(); ref = oracle.points(c2["f"], fld, pts); print("oracle s", time.time() - t)
o = out.cpu().numpy()
print("config2 max rel err", (np.abs(o[pts[:, 0], pts[:, 1]] - ref) / np.abs(ref).max()).max())
