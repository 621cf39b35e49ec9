"""Dev: one uniform-kernel filter of a 2048^2 f64 image at size s (a = sqrt(3 s))."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1003_2022_b200 as rb  # noqa: E402

s = float(sys.argv[1])
f = torch.from_numpy(np.random.default_rng(1).random((2048, 2048))).cuda()
a = np.full(4, math.sqrt(3.0 * s))
for _ in range(3):
    rb.filter_space_invariant(f, a)
torch.cuda.synchronize()
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    rb.filter_space_invariant(f, a)
torch.cuda.synchronize()
print(f"s={s}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per call (wall)")
