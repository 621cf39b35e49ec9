"""A/B timing (dev): one isotropic N=4 filter of a 2048^2 float64 image per
size s (the flat-cost table's call), device ms and a checksum.

    python scripts/ab_flat.py 256,512,1024
"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1003_2022_b200 as rb

sizes = [float(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256,512,1024").split(",")]
f = torch.from_numpy(np.random.default_rng(0).random((2048, 2048))).cuda()
for s in sizes:
    a = np.full(4, math.sqrt(3.0 * s))
    for _ in range(3):
        out = rb.filter_space_invariant(f, a)
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = rb.filter_space_invariant(f, a)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"s={s:g}: {min(ts):.4f} ms (median {sorted(ts)[4]:.4f})  sum {float(out.sum()):.12e}")
