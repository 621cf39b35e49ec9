"""Randomised parity sweep of the large-kernel paths (dev): images of
1024-4096 px a side, LUT parameter fields mixing small and huge kernels
(sigma up to ~300: primary kernel, stage 2, shared-memory overflow pass,
global-scratch blocks, per-pixel fallback, streamed host path), one or two
passes; sampled pixels against the exact per-point GPU oracle
(oracle/dense_oracle_cuda.cu), bar 1e-9 of max |output|.

    python scripts/fuzz_big.py [cases] [seed]
"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from oracle import port
import paper_1003_2022_b200 as rb



def smooth(rng, H, W, lo, hi, waves=3):
    yy, xx = np.mgrid[0:H, 0:W]
    v = sum(np.sin(rng.uniform(0, 6.3) + xx * rng.uniform(-3, 3) / W * 6.3 + yy * rng.uniform(-3, 3) / H * 6.3)
            for _ in range(waves))
    v = (v - v.min()) / max(v.max() - v.min(), 1e-9)
    return lo + (hi - lo) * v


def run_case(rng, lut, sides=(1024, 1536, 2048, 3000, 4096), widths=(1024, 1300, 2048, 4096)):
    """One random case; returns (max relative error at the sampled pixels, description)."""
    H = int(rng.choice(sides))
    W = int(rng.choice(widths))
    f = rng.random((H, W)).astype(np.float32 if rng.random() < 0.5 else np.float64)
    smax = float(10.0 ** rng.uniform(0.3, 2.5))  # sigma up to ~300
    style = int(rng.integers(0, 4))
    sig = smooth(rng, H, W, rng.uniform(0.5, 3.0), smax)
    if style == 1:  # abrupt patches of tiny kernels inside huge ones
        mask = smooth(rng, H, W, 0.0, 1.0, 2) > 0.8
        sig = np.where(mask, rng.uniform(0.4, 1.5), sig)
    elif style == 2:  # per-pixel noise on the size
        sig = sig * rng.uniform(0.5, 1.5, (H, W))
    size = 2.0 * sig * sig
    rho = np.minimum(smooth(rng, H, W, 1.0, rng.uniform(1.0, 5.7)), 5.79)
    th = smooth(rng, H, W, 0.0, math.pi - 1e-6)
    it = 1 if smax > 40 or rng.random() < 0.7 else 2
    pdt = np.float32 if rng.random() < 0.6 else np.float64
    s_, r_, t_ = size.astype(pdt), rho.astype(pdt), th.astype(pdt)
    if pdt == np.float32:
        t_ = np.minimum(t_, np.nextafter(np.float32(math.pi), np.float32(0)))
        r_ = np.minimum(r_, np.float32(5.79))
    host = rng.random() < 0.3
    if host:
        out = torch.from_numpy(rb.filter_space_variant_params(f, s_, r_, t_, lut=lut, iterations=it))
    else:
        out = rb.filter_space_variant_params(*(torch.from_numpy(v).cuda() for v in (f, s_, r_, t_)), lut=lut,
                                             iterations=it).cpu()
    n = 300
    pts = np.stack([rng.integers(0, H, n), rng.integers(0, W, n)], axis=1)
    pts = np.vstack([pts, [[0, 0], [H - 1, W - 1], [0, W - 1], [H - 1, 0]]])
    got = out.numpy()[pts[:, 0], pts[:, 1]]
    if it == 1:
        fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries,
                               *(v[pts[:, 0], pts[:, 1]].astype(np.float64) for v in (s_, r_, t_)))
        ref = oracle.points_cuda(torch.from_numpy(f), fld, pts)
    else:
        def field_of(rows, cols):
            return port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries,
                                    *(v[rows, cols].astype(np.float64) for v in (s_, r_, t_)))
        sub = pts[:24]
        got = got[:24]
        ref = np.concatenate([oracle.points2_cuda(torch.from_numpy(f), field_of, sub[i:i + 8])
                              for i in range(0, len(sub), 8)])
    e = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))
    desc = (f"{H}x{W} {f.dtype} params {np.dtype(pdt).name} sigma<= {smax:.0f} style {style} "
            f"passes {it} {'host' if host else 'device'}")
    return e, desc


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    lut = rb.default_lut()
    t0 = time.time()
    worst = 0.0
    for k in range(cases):
        e, desc = run_case(rng, lut)
        worst = max(worst, e)
        print(f"{'FAIL' if e > 1e-9 else 'ok'} case {k}: {desc}: {e:.2e}", flush=True)
    print(f"{cases} cases, seed {seed}, {time.time() - t0:.0f} s; worst {worst:.2e}")


if __name__ == "__main__":
    main()
