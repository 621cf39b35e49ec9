import numpy as np, sys
sys.path.insert(0, '.')
import oracle
import paper_1003_2022_b200 as rb
rng = np.random.default_rng(5)
for (H, W, lo, hi) in [(40, 40, 2.0, 2.0), (40, 40, 1.0, 3.0), (40, 40, 0.0, 12.0), (70, 90, 0.0, 12.0)]:
    f = rng.random((H, W))
    field = rng.uniform(lo, hi, (H, W, 3))
    ref = oracle.dense3(f, field)
    got = rb.filter_space_variant3(f, field)
    err = np.abs(got - ref)
    print(H, W, lo, hi, 'max err', err.max(), 'bad px', (err > 1e-9).sum(), np.argwhere(err > 1e-9)[:8].tolist())
    fu = np.ones((H, W))
    print('  ones: ', np.abs(rb.filter_space_variant3(fu, field) - oracle.dense3(fu, field)).max())
