"""Dev: wall time of one host-buffer call (pinned buffers) vs the device
call, for a config (default 3n4), optionally with RUBS_B200_HOST_TIMING."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1003_2022_b200 as rb  # noqa: E402
from paper_1003_2022_b200 import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3n4"
w = (workloads.config3(param_dtype=torch.float32) if cfg == "3n4" else
     workloads.config5(param_dtype=torch.float32, image_device="cuda"))
f = w["f"] if isinstance(w["f"], np.ndarray) else w["f"].cpu().numpy()
ps = [v.cpu() for v in (w["size"], w["elong"], w["orient"])]


def pin(a):
    t = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
    t.copy_(a)
    return t.numpy()


hf = pin(torch.from_numpy(f))
hp = [pin(v) for v in ps]
ho = torch.empty(f.shape, dtype=torch.float64, pin_memory=True).numpy()
for _ in range(2):
    rb.filter_space_variant_params(hf, *hp, out=ho)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    rb.filter_space_variant_params(hf, *hp, out=ho)
    ts.append(time.perf_counter() - t0)
df = torch.from_numpy(f).cuda()
dp = [v.cuda() for v in ps]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    rb.filter_space_variant_params(df, *dp)
torch.cuda.synchronize()
print(f"{cfg} host call ms {[round(t * 1e3, 2) for t in ts]}, device call ms {(time.perf_counter() - t0) / 3 * 1e3:.2f}")
