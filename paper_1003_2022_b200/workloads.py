"""Seeded synthetic inputs for BASELINE.json's five configs.

No public dataset is involved: the reference's own tests use synthetic
images only.  Every generator is deterministic in its seed; the same arrays
feed the GPU path and the CPU oracles.

Conventions (recorded in DESIGN.md):
  * x = column, y = row; sigma (BASELINE.json) -> size s = 2 sigma^2.
  * smooth(seed): min-max normalised sum of three sinusoids
    sin(2 pi (fx x / W + fy y / H) + phi), fx, fy ~ U(0.5, 3), phi ~ U(0, 2 pi).
  * rho is clamped to min(rho, 0.95 U(theta), 5.8 (1 - 1e-6)) like
    tensor.py:140 and tensor.py:216 (which use 1 - 1e-9; float32 parameters
    need the wider margin to stay inside the table after rounding).
  * config 3 names N=3 directions (0/60/120 degrees), which the reference
    does not implement: ``config3_n3`` is that workload
    for this repo's exact N=3 path (rho clamped to 0.95 of the N=3 bound,
    min 3 at 30/90/150 degrees); ``config3`` keeps its shapes with the N=4
    ZP element for the reference-anchored path.
"""

from __future__ import annotations

import math

import numpy as np

# a margin that survives float32 rounding (5.8 itself would round up)
RHO_LUT_CAP = 5.8 * (1.0 - 1e-6)


def _torch():
    import torch
    return torch


def smooth(seed: int, H: int, W: int, device="cpu", dtype=None):
    """Three-sinusoid smooth field in [0, 1], evaluated with torch (fp64)."""
    torch = _torch()
    rng = np.random.default_rng(seed)
    fx = rng.uniform(0.5, 3.0, 3)
    fy = rng.uniform(0.5, 3.0, 3)
    ph = rng.uniform(0.0, 2.0 * math.pi, 3)
    x = torch.arange(W, dtype=torch.float64, device=device)[None, :] / W
    y = torch.arange(H, dtype=torch.float64, device=device)[:, None] / H
    acc = torch.zeros((H, W), dtype=torch.float64, device=device)
    for k in range(3):
        acc += torch.sin(2.0 * math.pi * (fx[k] * x + fy[k] * y) + ph[k])
    lo, hi = acc.min(), acc.max()
    acc = (acc - lo) / (hi - lo)
    return acc if dtype is None else acc.to(dtype)


def clamp_rho(rho, theta):
    """rho <- min(rho, 0.95 U(theta), RHO_LUT_CAP) (torch, elementwise)."""
    torch = _torch()
    s2 = torch.sin(2.0 * theta)
    c2 = torch.cos(2.0 * theta)
    nu = torch.abs(c2 / s2)
    root = torch.sqrt(1.0 + nu * nu)
    bound = (1.0 + nu + root) / (1.0 - 1.0 / (nu + root))
    bound = torch.where(torch.isfinite(bound), bound, torch.full_like(bound, float("inf")))
    return torch.clamp(torch.minimum(rho, 0.95 * bound), max=RHO_LUT_CAP)


def _param_fields(H, W, sigma_lo, sigma_hi, rho_hi, seeds, device, dtype):
    torch = _torch()
    sig = sigma_lo + (sigma_hi - sigma_lo) * smooth(seeds[0], H, W, device)
    size = 2.0 * sig * sig
    theta = torch.remainder(2.0 * math.pi * smooth(seeds[2], H, W, device), math.pi)
    theta = torch.where(theta >= math.pi, torch.zeros_like(theta), theta)
    rho = 1.0 + (rho_hi - 1.0) * smooth(seeds[1], H, W, device)
    rho = torch.clamp(clamp_rho(rho, theta), min=1.0)
    out = [size, rho, theta]
    if dtype is not None:
        out = [v.to(dtype) for v in out]
        # float32 rounding must not push theta onto pi
        out[2] = torch.where(out[2] >= math.pi, torch.zeros_like(out[2]), out[2])
        out[1] = torch.clamp(out[1], min=1.0)
    return out


def config1(H: int = 256, W: int = 256):
    """256^2 fp64 uniform[0,1) seed 0; sigma 2->8 along x, rho 1->3 radial,
    theta = atan2(y - c, x - c) mod pi; exact optimiser per pixel -> (H,W,4)."""
    from .geometry import covariance_from_params
    from .solver import optimize_scale_vector
    f = np.random.default_rng(0).random((H, W))
    x = np.arange(W, dtype=np.float64)[None, :] * np.ones((H, 1))
    y = np.arange(H, dtype=np.float64)[:, None] * np.ones((1, W))
    sigma = 2.0 + 6.0 * x / (W - 1)
    c = (W - 1) / 2.0
    cy = (H - 1) / 2.0
    r = np.hypot(x - c, y - cy)
    rho = 1.0 + 2.0 * r / math.hypot(c, cy)
    theta = np.mod(np.arctan2(y - cy, x - c), math.pi)
    theta = np.where(theta >= math.pi, 0.0, theta)
    cov = covariance_from_params(2.0 * sigma * sigma, rho, theta)
    field = optimize_scale_vector(cov)
    return {"name": "config1", "f": f, "field": field, "iterations": 1}


def config2(H: int = 2048, W: int = 2048, device="cpu", param_dtype=None):
    """2048^2 fp64 uniform[0,1) seed 0; sigma in [2,16], rho in [1,4],
    theta in [0,pi) from smooth fields (seeds 1, 2, 3); LUT mapping."""
    f = np.random.default_rng(0).random((H, W))
    size, rho, theta = _param_fields(H, W, 2.0, 16.0, 4.0, (1, 2, 3), device, param_dtype)
    return {"name": "config2", "f": f, "size": size, "elong": rho, "orient": theta, "iterations": 1}


def rectangles_image(H: int, W: int, seed: int = 0, count: int = 512, noise: float = 0.05):
    """Config 3 image: `count` axis-aligned rectangles (sides U(32,1024),
    levels U(0,1)) painted in order on 0.5, plus N(0, noise^2); float32."""
    rng = np.random.default_rng(seed)
    img = np.full((H, W), 0.5, dtype=np.float32)
    for _ in range(count):
        h, w = rng.uniform(32, 1024, 2)
        y0, x0 = rng.uniform(0, H), rng.uniform(0, W)
        lvl = rng.uniform(0.0, 1.0)
        img[int(y0):int(min(H, y0 + h)), int(x0):int(min(W, x0 + w))] = lvl
    img += rng.normal(0.0, noise, (H, W)).astype(np.float32)
    return img


def config3(H: int = 8192, W: int = 8192, device="cpu", param_dtype=None):
    f = rectangles_image(H, W)
    size, rho, theta = _param_fields(H, W, 1.0, 32.0, 6.0, (31, 32, 33), device, param_dtype)
    return {"name": "config3", "f": f, "size": size, "elong": rho, "orient": theta, "iterations": 1}


def clamp_rho3(rho, theta):
    """rho <- min(rho, 0.95 U3(theta)): the three-direction bound
    (geometry.elongation_bound3), torch elementwise."""
    torch = _torch()
    c, s = torch.cos(theta), torch.sin(theta)
    cc, ss, cs = c * c, s * s, c * s
    r3 = 2.0 / math.sqrt(3.0)
    alpha = [cc - ss / 3.0, 2.0 / 3.0 * ss + r3 * cs, 2.0 / 3.0 * ss - r3 * cs]
    beta = [ss - cc / 3.0, 2.0 / 3.0 * cc - r3 * cs, 2.0 / 3.0 * cc + r3 * cs]
    bound = torch.full_like(rho, float("inf"))
    for al, be in zip(alpha, beta):
        lim = torch.where(al < -1e-15, -be / al, torch.full_like(al, float("inf")))
        bound = torch.minimum(bound, lim)
    return torch.clamp(torch.minimum(rho, 0.95 * bound), min=1.0)


def config3_n3(H: int = 8192, W: int = 8192, device="cpu", param_dtype=None):
    """Config 3 as BASELINE.json names it: the 8192^2 float32 rectangles
    image, N=3 directions (0/60/120 degrees), sigma in [1, 32], rho in
    [1, 6] clamped to 0.95 of the N=3 bound, smooth theta; (size, rho,
    theta) map to N=3 scales in closed form (filter_space_variant3_params)."""
    torch = _torch()
    f = rectangles_image(H, W)
    sig = 1.0 + 31.0 * smooth(31, H, W, device)
    size = 2.0 * sig * sig
    theta = torch.remainder(2.0 * math.pi * smooth(33, H, W, device), math.pi)
    theta = torch.where(theta >= math.pi, torch.zeros_like(theta), theta)
    rho = clamp_rho3(1.0 + 5.0 * smooth(32, H, W, device), theta)
    out = [size, rho, theta]
    if param_dtype is not None:
        out = [v.to(param_dtype) for v in out]
        # the 0.95 margin dwarfs float32 rounding of (rho, theta)
        out[2] = torch.where(out[2] >= math.pi, torch.zeros_like(out[2]), out[2])
        out[1] = torch.clamp(out[1], min=1.0)
    return {"name": "config3_n3", "f": f, "size": out[0], "elong": out[1], "orient": out[2],
            "iterations": 1, "directions": 3}


def config4_image(i: int, H: int = 4096, W: int = 4096, device="cpu", param_dtype=None):
    """Image i of config 4's batch: uniform[0,1) fp32 (seed 1000+i), sigma in
    [2,24], rho in [1,4], smooth theta (per-image seeds); two passes."""
    f = np.random.default_rng(1000 + i).random((H, W), dtype=np.float32)
    base = 4000 + 3 * i
    size, rho, theta = _param_fields(H, W, 2.0, 24.0, 4.0, (base, base + 1, base + 2), device, param_dtype)
    return {"name": f"config4[{i}]", "f": f, "size": size, "elong": rho, "orient": theta, "iterations": 2}


def config5(H: int = 32768, W: int = 32768, device="cpu", param_dtype=None, image_device=None):
    """32768^2 fp32 uniform[0,1): generated with torch's Philox on the given
    device (seed 0) -- a 4 GiB numpy draw would dominate the run; sigma in
    [2,256], rho in [1,8] clamped, smooth theta."""
    torch = _torch()
    g = torch.Generator(device=image_device or device)
    g.manual_seed(0)
    f = torch.rand((H, W), generator=g, device=image_device or device, dtype=torch.float32)
    size, rho, theta = _param_fields(H, W, 2.0, 256.0, 8.0, (51, 52, 53), device, param_dtype)
    return {"name": "config5", "f": f, "size": size, "elong": rho, "orient": theta, "iterations": 1}


def adaptive_image(H: int = 2048, W: int = 2048, seed: int = 0, noise: float = 0.1):
    """Workload of the adaptive_smooth pipeline (tensor.py:174-224; SURVEY.md
    §8f): oriented stripes (period 11 px, angle 0.7 rad, oracle.py:351-363
    recipe) plus N(0, noise^2) seeded noise, float64; noise_sigma = noise."""
    x1 = np.arange(W, dtype=np.float64)[None, :]
    x2 = np.arange(H, dtype=np.float64)[:, None]
    phase = -math.sin(0.7) * x1 + math.cos(0.7) * x2
    clean = 0.5 * (np.sin(2.0 * math.pi * phase / 11.0) + 1.0)
    f = clean + np.random.default_rng(seed).normal(0.0, noise, (H, W))
    return {"name": "adaptive", "f": f, "clean": clean, "noise_sigma": noise, "iterations": 1}
