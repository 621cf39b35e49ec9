"""Dev probe: one small float64 filter call (TMA region loads) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1003_2022_b200 as rb

rng = np.random.default_rng(1)
for H, W in [(40, 48), (64, 64), (100, 70)]:
    f = rng.random((H, W))
    a = np.array([1.3, 2.1, 1.7, 1.1])
    out = rb.filter_space_invariant(f, a)
    ref = oracle.dense(f, np.broadcast_to(a, (H, W, 4)).copy(), 1)
    print(H, W, "max err", float(np.abs(out - ref).max()), flush=True)
