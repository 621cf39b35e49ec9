#!/usr/bin/env python
"""Benchmark of the B200 space-variant filter path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 5|2|1|3|3l|3n4|4|A]

Default workload: BASELINE.json config 5 -- ONE 32768^2 float32 image,
N=4 ZP box spline, sigma up to 256 (the largest configuration that runs on
one GPU), LUT-mapped (size, elongation, orientation) fields in float32, one
pass, fused params path (rubs_b200_filter_params).  One step = one filter
of the whole image.
  N = 1   the whole image on one GPU;
  N > 1   the image is split into N row bands (sharding.RowBandPlan): each
          rank exchanges halo rows with its neighbours over NCCL and filters
          its band (strong scaling: the N ranks share one image per step).
Config 4 is the 64-image batch: each rank filters its 64/N images per step
(two passes each; weak in per-rank work, the batch is fixed).  Other
configs: one image per rank per step (configs 3 with N=3 shard by row bands
like config 5).

``--gpus N`` with no torchrun environment re-launches itself under
``torch.distributed.run`` with N processes (one per GPU); under torchrun,
WORLD_SIZE must equal N.

Printed JSON (rank 0, one line) carries the driver's keys plus
  e2e          the same metric through the public API with HOST buffers
               (pinned H2D of every input and D2H of the result inside the
               timed region; N > 1 row bands: each rank's band and halo rows
               in, its band out)
  roofline     the pass's filter kernels (primary tile kernel + the
               deferred-tile passes, bracketed by CUDA events on the launch
               stream): algorithmic bytes / that time, against
               MEASURED_PEAKS.json; ``traffic`` = ncu DRAM bytes of the same
               kernels (profiles/)
  fp64, smem   the primary kernel against the fp64 pipe and shared-memory
               wavefront rates (configs 2, 3: the bounds that bind there)
  cpu_baseline the reference algorithm (oracle/port.py, numpy) on a bounded
               sample of the same workload, all host cores, rank 0 at N=1
  parity       (same leg, as the checker) max relative error of the GPU
               output at sampled pixels of the workload against the exact
               dense oracle -- BASELINE.json's "max rel err vs oracle"
`--impl reference` prints the same line for the CPU port alone (rank 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Gpixel/s filtered"
UNIT = "Gpixel/s"
CONFIGS = ["5", "2", "1", "3", "3l", "3n4", "4", "A"]
BATCH4 = 64  # config 4: images per step (all ranks together)
# Algorithmic bytes per output pixel: image + per-pixel
# parameters + f64 output, per pass (config 4: both passes, intermediate
# ignored; config 1: the drop-in (H,W,4) f64 field).
BYTES_PER_PX = {"2": 28, "1": 48, "3": 24, "3l": 24, "3n4": 24, "4": 52, "5": 24, "A": 16}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="5", choices=CONFIGS)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--probe-launch", action="store_true",
                   help="start the ranks, all-gather them, print one JSON line, exit (launcher test)")
    return p.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args_n: int) -> int:
    """Re-run this script under torch.distributed.run with N processes."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args_n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
WORKLOADS = {
    "5": "config5: 32768^2 fp32 uniform[0,1) (torch Philox seed 0); N=4 ZP; sigma [2,256] smooth, "
         "rho [1,8] clamped to the LUT, smooth theta (LUT mapping fused, f32 params); one pass",
    "3": "config3: 8192^2 fp32 rectangles + N(0,0.05^2) noise; N=3 directions (0/60/120 deg); "
         "sigma [1,32], rho [1,6] clamped to 0.95 of the N=3 bound, smooth theta; exact N=3 path "
         "(closed-form mapping fused, f32 params)",
    "3l": "config3: 8192^2 fp32 rectangles + N(0,0.05^2) noise; N=3 directions (0/60/120 deg); "
          "sigma [1,32], rho [1,6] clamped to 0.95 of the N=3 bound, smooth theta; O(1) LATTICE mode: "
          "image resampled once onto the triangular lattice (spacing 1), exact integer running sums, "
          "8-vertex finite difference (closed-form mapping fused, f32 params)",
    "3n4": "config3 shapes with the N=4 ZP element: 8192^2 fp32 rectangles + N(0,0.05^2) noise; "
           "sigma [1,32], rho [1,6] clamped, smooth theta (LUT mapping)",
    "2": "config2: 2048^2 fp64 uniform[0,1) seed 0; N=4 ZP box spline; sigma [2,16], rho [1,4], "
         "theta [0,pi) smooth fields (LUT mapping, f32 params)",
    "1": "config1: 256^2 fp64 uniform[0,1) seed 0; sigma 2->8 along x, rho 1->3 radial, "
         "theta=atan2 mod pi; exact optimiser field",
    "4": "config4: batch of 64 4096^2 fp32 uniform[0,1) images (seeds 1000+i); sigma [2,24], rho [1,4], "
         "smooth theta (per-image seeds); N=4 ZP applied twice (iterations=2)",
    "A": "adaptive_smooth pipeline (tensor.py; SURVEY 8f): 2048^2 fp64 stripes + N(0,0.1^2), "
         "noise_sigma 0.1, window 1.5; structure tensor (3 window filters), percentiles, anisotropy, "
         "LUT filter of image and flat image, gain correction",
}
SHAPES = {"5": (32768, 32768), "3": (8192, 8192), "3l": (8192, 8192), "3n4": (8192, 8192), "2": (2048, 2048),
          "1": (256, 256), "4": (4096, 4096), "A": (2048, 2048)}
ITERS = {"4": 2}


def row_banded(cfg: str, world: int) -> bool:
    return cfg in ("5", "3", "3l") and world > 1


def bench_config(cfg: str, world: int) -> dict:
    """The ``config`` object of the JSON line -- identical for both arms."""
    H, W = SHAPES[cfg]
    d = {"workload": WORKLOADS[cfg], "image": [H, W], "iterations": ITERS.get(cfg, 1)}
    if cfg == "4":
        d.update(batch=BATCH4, images_per_rank_per_step=-(-BATCH4 // world),
                 parallelism=f"batch sharded over {world} rank(s), no data-path collective")
    elif row_banded(cfg, world):
        d.update(parallelism=f"one image in {world} row bands, NCCL halo exchange overlapped with "
                             f"the band interior")
    else:
        d.update(parallelism="one image per rank per step" + (" (replicas)" if world > 1 else ""))
    if cfg in ("5", "3", "3l", "3n4", "4"):
        d["l2"] = "inputs + output per step exceed the 126 MB L2 (no flush needed)"
    elif cfg != "1":
        d["l2"] = "4 rotating input/output sets per rank (working set > 126 MB L2)"
    else:
        d["l2"] = "4 rotating input sets (working set < L2: launch-bound config)"
    d["path"] = {"1": "drop-in (H,W,4) f64 field (rubs_b200_filter)",
                 "3": "fused closed-form N=3 mapping + exact N=3 filter (rubs_b200_filter3_params)",
                 "3l": "fused closed-form N=3 mapping + O(1) lattice-mode N=3 filter "
                       "(rubs_b200_filter3_lattice_params)",
                 "A": "rubs_b200_adaptive_smooth"}.get(
        cfg, "fused LUT mapping + filter (rubs_b200_filter_params)")
    return d


def _load_workload(cfg, torch, device, rank=0, image=None):
    from paper_1003_2022_b200 import workloads
    f32 = torch.float32
    if cfg == "2":
        return workloads.config2(device=device, param_dtype=f32)
    if cfg == "1":
        return workloads.config1()
    if cfg in ("3", "3l"):
        return workloads.config3_n3(device=device, param_dtype=f32)
    if cfg == "3n4":
        return workloads.config3(device=device, param_dtype=f32)
    if cfg == "5":
        return workloads.config5(device=device, param_dtype=f32, image_device=device)
    if cfg == "A":
        return workloads.adaptive_image()
    return workloads.config4_image(rank if image is None else image, device=device, param_dtype=f32)


class Work:
    """One rank's workload: device-resident inputs and the step function."""

    def __init__(self, cfg, torch, device, rank, world):
        import paper_1003_2022_b200 as rb
        from paper_1003_2022_b200 import sharding
        self.cfg, self.torch, self.rb = cfg, torch, rb
        self.rank, self.world = rank, world
        self.H, self.W = SHAPES[cfg]
        self.iters = ITERS.get(cfg, 1)
        self.n3 = cfg in ("3", "3l")
        self.n3_mode = "lattice" if cfg == "3l" else "exact"
        self.row_bands = row_banded(cfg, world)
        self.sets = []
        self.lut = rb.default_lut()
        if cfg == "4":
            # the batch: this rank's 64/N images, all resident
            self.images = sharding.batch_indices(BATCH4, world, rank)
            for i in self.images:
                w = _load_workload(cfg, torch, device, image=i)
                self.sets.append({"f": torch.as_tensor(w["f"]).to(device),
                                  "p": [w["size"], w["elong"], w["orient"]]})
            self.px_per_step = float(self.H * self.W) * BATCH4  # all ranks together
            return
        w = _load_workload(cfg, torch, device, rank)
        self.w = w
        if cfg == "A":
            f = torch.as_tensor(w["f"]).to(device)
            self.sets = [{"f": f.clone(), "adaptive": True} for _ in range(4)]
        elif cfg == "1":
            f = torch.as_tensor(w["f"]).to(device)
            fld = torch.as_tensor(w["field"]).to(device)
            self.sets = [{"f": f.clone(), "field": fld.clone()} for _ in range(4)]
        elif cfg == "2":
            f = torch.as_tensor(w["f"]).to(device)
            self.sets = [{"f": f.clone(), "p": [v.clone() for v in (w["size"], w["elong"], w["orient"])]}
                         for _ in range(4)]
        else:
            self.sets = [{"f": torch.as_tensor(w["f"]).to(device), "p": [w["size"], w["elong"], w["orient"]]}]
        if self.row_bands:
            align = (sharding.TILE3L if self.n3_mode == "lattice" else sharding.TILE3) if self.n3 \
                else sharding.TILE
            self.band = sharding.band_bounds(self.H, world, align)[rank]
            s0 = self.sets[0]
            b0, b1 = self.band
            self.own = s0["f"][b0:b1].contiguous()
            self.pb = [p[b0:b1].contiguous() for p in s0["p"]]
            if self.n3_mode == "lattice":
                self.plan = sharding.row_band_plan3_lattice(self.band, self.H, self.pb[0])
            elif self.n3:
                self.plan = sharding.row_band_plan3(self.band, self.H, self.pb[0])
            else:
                self.plan = sharding.row_band_plan(self.band, self.H, self.pb[0], self.lut)
            self.sets = []
            torch.cuda.empty_cache()
            self.px_per_step = float(self.H * self.W)  # the ranks share one image
        else:
            self.px_per_step = float(self.H * self.W) * world

    def step(self, i):
        rb, sharding = self.rb, __import__("paper_1003_2022_b200.sharding", fromlist=["x"])
        if self.row_bands and self.n3_mode == "lattice":
            return sharding.filter3_lattice_row_band(self.own, self.band, self.H, *self.pb, plan=self.plan)
        if self.row_bands and self.n3:
            return sharding.filter3_row_band(self.own, self.band, self.H, *self.pb, plan=self.plan)
        if self.row_bands:
            return sharding.filter_row_band(self.own, self.band, self.H, *self.pb, lut=self.lut,
                                            plan=self.plan)
        if self.cfg == "4":
            out = None
            for s in self.sets:
                out = rb.filter_space_variant_params(s["f"], *s["p"], lut=self.lut, iterations=2)
            return out
        s = self.sets[i % len(self.sets)]
        if "adaptive" in s:
            return rb.adaptive_smooth(s["f"], self.w["noise_sigma"])
        if "p" in s and self.n3:
            return rb.filter_space_variant3_params(s["f"], *s["p"], iterations=self.iters, mode=self.n3_mode)
        if "p" in s:
            return rb.filter_space_variant_params(s["f"], *s["p"], lut=self.lut, iterations=self.iters)
        return rb.filter_space_variant(s["f"], s["field"], self.iters)

    # ---- end to end through the public API with host buffers ------------
    def e2e_setup(self):
        """(call, h2d bytes, d2h bytes, pixels per call) on pinned host
        buffers; every call copies its inputs in and its result out."""
        torch, rb = self.torch, self.rb

        def pinned(t, dtype=None):
            h = torch.empty(t.shape, dtype=dtype or t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        if self.row_bands:
            from paper_1003_2022_b200 import sharding
            # this rank's share as the host scatters it: its band's
            # parameter rows and its band + halo image rows; the band's
            # output rows come back (no exchange: the host holds the rows)
            n0, n1 = self.plan.needs[self.rank]
            b0, b1 = self.band
            # the halo rows live on the neighbours: fetch them once here
            # (setup), as the host scatter would hand them out
            full = sharding.exchange_rows(self.own, self.band, self.plan.bands, self.plan.needs, self.rank)
            hf = pinned(full)
            hp = [pinned(p) for p in self.pb]
            hout = torch.empty((b1 - b0, self.W), dtype=torch.float64, pin_memory=True)
            dev = self.own.device

            def call():
                f_rows = hf.to(dev, non_blocking=True)
                ps = [p.to(dev, non_blocking=True) for p in hp]
                if self.n3_mode == "lattice":
                    out = sharding.filter3_lattice_rows_params(f_rows, n0, self.H, *ps, b0, b0, b1 - b0)
                elif self.n3:
                    out = sharding.filter3_rows_params(f_rows, n0, self.H, *ps, b0, b0, b1 - b0)
                else:
                    out = sharding.filter_rows_params(f_rows, n0, self.H, *ps, b0, b0, b1 - b0, self.lut)
                hout.copy_(out, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return hout
            h2d = hf.numel() * hf.element_size() + sum(p.numel() * p.element_size() for p in hp)
            return call, h2d, hout.numel() * 8, float((b1 - b0) * self.W)
        if self.cfg == "4":
            # the rank's images as pinned host arrays (up to 8 distinct sets,
            # rotating over the rank's 64/N images: every image is copied in
            # and out on every call)
            k = min(len(self.sets), 8)
            hsets = [(pinned(s["f"]).numpy(), [pinned(p).numpy() for p in s["p"]]) for s in self.sets[:k]]
            houts = [torch.empty((self.H, self.W), dtype=torch.float64, pin_memory=True).numpy()
                     for _ in range(2)]

            m = len(self.sets)
            bf = [hsets[j % k][0] for j in range(m)]
            bp = [[hsets[j % k][1][q] for j in range(m)] for q in range(3)]
            bo = [houts[j % 2] for j in range(m)]

            def call():
                # the batch entry point: image j+1 uploads while j is filtered
                # and j-1 returns (rubs_b200_filter_params_batch_host)
                return rb.filter_space_variant_params_batch(bf, *bp, lut=self.lut, iterations=2, outs=bo)
            one = hsets[0][0].nbytes + sum(p.nbytes for p in hsets[0][1])
            return call, one * len(self.sets), self.H * self.W * 8 * len(self.sets), \
                float(self.H * self.W) * len(self.sets)
        s = self.sets[0]
        hout = torch.empty((self.H, self.W), dtype=torch.float64, pin_memory=True).numpy()
        if "adaptive" in s:
            hf = pinned(s["f"]).numpy()
            return (lambda: rb.adaptive_smooth(hf, self.w["noise_sigma"], out=hout)), hf.nbytes, \
                hout.nbytes, float(self.H * self.W)
        if "p" in s:
            hf = pinned(s["f"]).numpy()
            hp = [pinned(p).numpy() for p in s["p"]]
            if self.n3:
                call = lambda: rb.filter_space_variant3_params(hf, *hp, iterations=self.iters, out=hout,  # noqa: E731
                                                               mode=self.n3_mode)
            else:
                call = lambda: rb.filter_space_variant_params(hf, *hp, lut=self.lut,  # noqa: E731
                                                              iterations=self.iters, out=hout)
            return call, hf.nbytes + sum(p.nbytes for p in hp), hout.nbytes, float(self.H * self.W)
        hf = pinned(s["f"]).numpy()
        hfl = pinned(s["field"], torch.float64).numpy()
        return (lambda: rb.filter_space_variant(hf, hfl, self.iters, out=hout)), hf.nbytes + hfl.nbytes, \
            hout.nbytes, float(self.H * self.W)


def pcie_copy_seconds(torch, h2d_bytes, d2h_bytes, device, chunk=256 << 20):
    """Seconds for bare pinned copies of h2d_bytes up and d2h_bytes down,
    concurrently on two streams (the e2e leg's PCIe bound)."""
    try:
        hu = torch.empty(chunk, dtype=torch.uint8, pin_memory=True)
        hd = torch.empty(chunk, dtype=torch.uint8, pin_memory=True)
        du = torch.empty(chunk, dtype=torch.uint8, device=device)
        dd = torch.empty(chunk, dtype=torch.uint8, device=device)
        su, sd = torch.cuda.Stream(device), torch.cuda.Stream(device)

        def run():
            with torch.cuda.stream(su):
                left = h2d_bytes
                while left > 0:
                    n = min(chunk, left)
                    du[:n].copy_(hu[:n], non_blocking=True)
                    left -= n
            with torch.cuda.stream(sd):
                left = d2h_bytes
                while left > 0:
                    n = min(chunk, left)
                    hd[:n].copy_(dd[:n], non_blocking=True)
                    left -= n
            torch.cuda.synchronize(device)
        run()
        t0 = time.perf_counter()
        run()
        return time.perf_counter() - t0
    except RuntimeError:
        return None


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1003_2022_b200 import _native

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    L = _native.load()
    # PrecisionWarning = the filter met needle kernels; the
    # line reports how many calls of this run raised it (0 on every config)
    import warnings
    _rec = warnings.catch_warnings(record=True)
    wlist = _rec.__enter__()
    warnings.simplefilter("always", _native.PrecisionWarning)
    dfma = None
    if rank == 0:
        # measured fp64 FMA peak of this GPU (the fp64 roofline's denominator)
        tf, pms = ctypes.c_double(), ctypes.c_double()
        if L.rubs_b200_dfma_peak(ctypes.byref(tf), ctypes.byref(pms)) == 0:
            dfma = tf.value
    wk = Work(args.config, torch, device, rank, world)
    if rank == 0 and world == 1:
        _WK_FOR_CPU["wk"] = wk

    for i in range(args.warmup):
        wk.step(i)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    L.rubs_b200_reset_launch_count()
    L.rubs_b200_reset_kernel_time()
    L.rubs_b200_set_profiling(1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for i in range(args.steps):
        wk.step(i)
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    L.rubs_b200_set_profiling(0)
    ms_total = ev0.elapsed_time(ev1)
    launches = int(L.rubs_b200_launch_count())
    pass_ms, pass_n = ctypes.c_double(), ctypes.c_int64()
    L.rubs_b200_kernel_time(0, ctypes.byref(pass_ms), ctypes.byref(pass_n))
    all_ms, all_n = ctypes.c_double(), ctypes.c_int64()
    L.rubs_b200_kernel_time(2, ctypes.byref(all_ms), ctypes.byref(all_n))
    clk = clocks.stop() if rank == 0 else None

    t = torch.tensor([ms_total], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = wk.px_per_step * args.steps / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        call, h2d, d2h, px_call = wk.e2e_setup()
        for _ in range(max(2, args.warmup // 2)):
            call()
        if world > 1:
            dist.barrier()
        ksteps = max(3, args.steps // 2) if args.config != "4" else max(2, args.steps // 4)
        t0 = time.perf_counter()
        for _ in range(ksteps):
            call()
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        px_all = wk.px_per_step if (wk.row_bands or args.config == "4") else px_call * world
        # the PCIe bound of the same bytes: bare concurrent pinned copies
        # (H2D on one stream, D2H on another), outside the timed region
        bound_s = pcie_copy_seconds(torch, h2d, d2h, device)
        e2e = {"value": px_all * ksteps / float(te.item()) / 1e9, "unit": UNIT,
               "pcie_bound_value": px_all / bound_s / 1e9 if bound_s else None,
               "pcie_bound_note": "same metric if the call took only the bare concurrent pinned copies of its "
                                  "input and result bytes",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": ksteps, "host_buffers": "pinned (inputs and result)",
               "timing": "wall clock around blocking API calls, max over ranks"
                         + ("; per rank: its band + halo rows in, its band out" if wk.row_bands else "")}

    # one more call outside the timed region: the output at sampled pixels for
    # the parity line (checked against the exact oracle in the CPU leg)
    pin = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out = wk.step(0)
        torch.cuda.synchronize()
        pin = parity_sample(args.config, wk, out)

    result = None
    if rank == 0:
        hbm, sm_max, peak_kind = measured_peaks()
        bpp = BYTES_PER_PX[args.config]
        px_rank_step = wk.px_per_step / (1 if wk.row_bands or args.config == "4" else world)
        if wk.row_bands:
            px_rank_step = float((wk.band[1] - wk.band[0]) * wk.W)
        elif args.config == "4":
            px_rank_step = float(wk.H * wk.W * len(wk.sets))
        kern_s = max(pass_ms.value, 1e-9) / max(1, args.steps) * 1e-3  # filter kernels per step
        achieved = bpp * px_rank_step / kern_s / 1e9
        passes_per_step = pass_n.value / max(1, args.steps)
        fp64 = smem = None
        dp_per_px = DP_INST_PER_PX.get(args.config)
        if dp_per_px:
            # DP lane-instructions / s: the measured DFMA rate (one DFMA per
            # lane-instruction) when the probe ran, else 64 lanes x SMs x clock
            peak_dp = dfma * 1e12 / 2.0 if dfma else 148 * 64 * sm_max * 1e6
            got_dp = dp_per_px * px_rank_step * wk.iters / kern_s
            fp64 = {"achieved_dp_ops_per_s": got_dp, "peak_dp_ops_per_s": peak_dp,
                    "frac": got_dp / peak_dp, "dp_inst_per_px": dp_per_px,
                    "peak_source": "measured DFMA probe (rubs_b200_dfma_peak)" if dfma else
                                   "148 SMs x 64 fp64 lanes x max clock",
                    "measured_dfma_tflops": dfma,
                    "source": "ncu sm__sass_thread_inst_executed_op_fp64 per px"}
        wf_per_px = SMEM_WF_PER_PX.get(args.config)
        if wf_per_px:
            peak_wf = 148 * sm_max * 1e6  # wavefronts / s at max clock
            got_wf = wf_per_px * px_rank_step * wk.iters / kern_s
            smem = {"achieved_wavefronts_per_s": got_wf, "peak_wavefronts_per_s": peak_wf,
                    "frac": got_wf / peak_wf, "wavefronts_per_px": wf_per_px,
                    "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum per px"}
        traffic = TRAFFIC_PER_PASS.get(args.config)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if wk.row_bands else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(args.config, world),
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm,
                         "traffic": traffic[0] if traffic else None,
                         "traffic_note": traffic[1] if traffic else None,
                         "kernel": KERNEL_NOTE.get(args.config, "wide_filter_kernel (the pass's one launch)"),
                         "kernel_ms_per_step": max(pass_ms.value, 0.0) / max(1, args.steps),
                         "passes_per_step": passes_per_step,
                         "algorithmic_bytes_per_px": bpp, "peak_source": peak_kind,
                         "binding_bound": BINDING.get(args.config, "shared-memory wavefronts and issue")},
            "fp64": fp64,
            "smem": smem,
            "dfma_peak_tflops": dfma,
            "gpu_launches": launches,
            "launches_per_step": launches / max(1, args.steps),
            "kernel_share_of_step": all_ms.value / max(ms_total, 1e-9),
            "clocks": clk,
            "precision_warnings": sum(1 for w_ in wlist if issubclass(w_.category, _native.PrecisionWarning)),
        }
        if pin is not None:
            result["_parity_in"] = pin
    _rec.__exit__(None, None, None)
    if world > 1:
        dist.destroy_process_group()
    return result


KERNEL_NOTE = {
    "5": "the pass's filter kernels: wide_filter_kernel (mapping, plan, small kernels) + the "
         "large-halo block passes (big_* kernels); per-kernel split in profiles/",
    "3n4": "the pass's filter kernels: wide_filter_kernel + the large-halo block passes",
    "4": "the filter kernels of both passes of each image",
    "3": "n3_tile_kernel",
    "3l": "the lattice pass: lat_splat / lat_colsum / lat_diagsum / lat_gather kernels",
    "A": "the pipeline's filter launches",
}
BINDING = {
    "5": "on-chip: the 16-vertex gather (L1) and the block regions' scratch traffic (see traffic)",
    "3": "shared-memory wavefronts (see smem)",
    "3l": "HBM traffic of the int128 lattice regions (16 B per lattice point, written by the splat, "
          "swept twice, gathered)",
}
# From the committed ncu captures of the primary kernel (wide_filter_kernel)
# on config 2 (profiles/ncu_r01b_summary.md, final build): fp64 instructions
# executed per output pixel (DADD + DFMA + DMUL, thread level), shared-memory
# wavefronts per output pixel.  Config 3 (N=3, n3_tile_kernel): same file.
DP_INST_PER_PX = {"2": 524, "3": 2147}
SMEM_WF_PER_PX = {"2": 16.39, "3": 53.9}
# DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per pass, summed
# over the pass's kernels, from the ncu launch lists in profiles/.
TRAFFIC_PER_PASS = {
    "2": (105.45e6, "ncu, wide_filter_kernel, profiles/ncu_r01b_summary.md"),
    "3": (1.588e9, "ncu, n3_tile_kernel, profiles/ncu_r01b_summary.md"),
    "3l": (11.57e9, "ncu launch list of one pass, sum over the lat_* kernels "
                    "(profiles/ncu_r02_c3l_launches.csv; algorithmic 1.61 GB: the rest is the int128 lattice "
                    "region, 16 B per lattice point, written by the splat, read and written by the two line "
                    "sums, read by the gather)"),
    "5": (180.2e9, "ncu launch list of one step, sum over the pass's kernels "
                   "(profiles/ncu_r02_c5_launches.csv, split in profiles/ncu_r02_summary.md; algorithmic "
                   "25.8 GB: the rest is the large-halo regions' scratch, 4.5 elements per pixel written "
                   "and re-read by the sweeps, then gathered)"),
}


# ---------------------------------------------------------------------------
# Parity leg (checker only, after the timed region): the GPU output at
# sampled pixels against the exact dense oracle.

PARITY_PX = {"1": 256, "2": 256, "3": 256, "3l": 256, "3n4": 128}


def parity_sample(cfg, wk, out):
    """GPU outputs (and inputs) at the sampled pixels of the workload."""
    torch = wk.torch
    H, W = wk.H, wk.W
    rng = np.random.default_rng(7)
    if cfg == "A":
        return None
    if cfg == "4":
        # 8 x 8 blocks of the last image filtered (two passes), corners incl.
        blocks = [(0, 0), (H - 8, W - 8), (0, W - 8), (H - 8, 0)] + \
                 [(int(rng.integers(0, H - 8)), int(rng.integers(0, W - 8))) for _ in range(4)]
        pts = np.concatenate([np.stack(np.mgrid[y:y + 8, x:x + 8], -1).reshape(-1, 2) for y, x in blocks])
        s = wk.sets[-1]
    else:
        n = PARITY_PX.get(cfg, 2000)
        pts = np.stack([rng.integers(0, H, n), rng.integers(0, W, n)], axis=1)
        pts = np.concatenate([pts, [[0, 0], [H - 1, W - 1], [0, W - 1], [H - 1, 0]]])
        s = wk.sets[0]
    idx = torch.as_tensor(pts, device=out.device)
    got = out[idx[:, 0], idx[:, 1]].double().cpu().numpy()
    if "field" in s:
        par = s["field"][idx[:, 0], idx[:, 1]].double().cpu().numpy()
    else:
        par = np.stack([v[idx[:, 0], idx[:, 1]].double().cpu().numpy() for v in s["p"]], axis=1)
    return {"pts": pts, "got": got, "par": par, "n3": wk.n3, "lattice": wk.n3_mode == "lattice", "f": s["f"],
            "p": s.get("p")}


def parity_check(cfg: str, pin) -> dict:
    """Max relative error of the GPU output at sampled pixels of the bench
    workload against the exact dense oracle (oracle/dense_oracle.c,
    dense3_oracle.c; configs 4 and 5: its GPU copy dense_oracle_cuda.cu,
    pinned to it by tests/test_gpu_baseline_size.py -- the checker, pinned to
    the reference by tests/test_oracle_golden.py, test_oracle_n3.py).  Each
    pixel is evaluated on the crop of the image its kernel reaches (exact:
    zero padding), with its own scale-vector."""
    import math as _m
    import oracle
    from oracle import port, port3
    from paper_1003_2022_b200 import default_lut
    pts, got, par = pin["pts"], pin["got"], pin["par"]
    f = pin["f"]
    lut = default_lut()
    if cfg == "1" or par.shape[1] == 4:
        field = par
    elif pin["n3"]:
        field = port3.scales3_from_params(par[:, 0], par[:, 1], par[:, 2])
    else:
        field = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, par[:, 0], par[:, 1], par[:, 2])
    if cfg in ("4", "5"):
        if cfg == "5":
            ref = oracle.points_cuda(f, field, pts)
            how = "exact dense filter per pixel on the GPU (oracle/dense_oracle_cuda.cu points_kernel)"
        else:
            import torch
            params = pin["p"]

            def field_of(rows, cols):
                r = torch.as_tensor(np.asarray(rows, np.int64), device=params[0].device)
                c = torch.as_tensor(np.asarray(cols, np.int64), device=params[0].device)
                v = [p[r, c].double().cpu().numpy() for p in params]
                return port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, *v)
            ref = np.concatenate([oracle.points2_cuda(f, field_of, pts[i:i + 64])
                                  for i in range(0, len(pts), 64)])
            how = ("exact two-pass dense filter (pass 1 on the GPU over each 8x8 block's window, "
                   "oracle/dense_oracle_cuda.cu; pass 2 exact kernel sums)")
        scale = max(float(np.abs(ref).max()), 1e-300)
        return {"max_rel_err": float(np.abs(got - ref).max() / scale), "pixels": int(len(pts)),
                "oracle": how, "tolerance": 1e-9}
    H, W = f.shape
    if pin.get("lattice"):
        return _parity_lattice(f, field, pts, got)
    ref = np.empty(len(pts))
    for i, ((r, c), a) in enumerate(zip(pts, field)):
        a = np.maximum(a, 0.05)
        if pin["n3"]:
            rx = int(_m.ceil(0.5 * a[0] + 0.25 * (a[1] + a[2]))) + 1
            ry = int(_m.ceil(0.25 * _m.sqrt(3.0) * (a[1] + a[2]))) + 1
        else:
            diag = (a[1] + a[3]) / _m.sqrt(2.0)
            rx = int(_m.ceil(0.5 * (a[0] + diag))) + 1
            ry = int(_m.ceil(0.5 * (a[2] + diag))) + 1
        r0, r1, c0, c1 = max(0, r - ry), min(H, r + ry + 1), max(0, c - rx), min(W, c + rx + 1)
        crop = f[r0:r1, c0:c1]
        crop = (crop.double().cpu().numpy() if hasattr(crop, "cpu") else np.asarray(crop, np.float64))
        q = np.array([[r - r0, c - c0]])
        ref[i] = (oracle.points3(crop, a, q, threads=1) if pin["n3"] else
                  oracle.points(crop, a, q, threads=1))[0]
    scale = max(float(np.abs(ref).max()), 1e-300)
    return {"max_rel_err": float(np.abs(got - ref).max() / scale), "pixels": int(len(pts)),
            "oracle": "exact dense filter per pixel (oracle/dense" + ("3" if pin["n3"] else "") +
                      "_oracle.c) on the crop its kernel reaches",
            "tolerance": 1e-9}


def _parity_lattice(f, field, pts, got) -> dict:
    """Lattice (O(1)) N=3 mode.  ``max_rel_err``: against the mode's own
    definition taken literally -- the brute-force sum of the exact N=3 kernel
    over the resampled image (oracle/dense3_oracle.c
    rubs_oracle3_lattice_points), the 1e-9 bar.  ``mode_error_vs_exact``: the
    mode's resampling error against the exact N=3 filter of the original
    image (dense3_oracle.c), reported, not a pass/fail bar."""
    import math as _m
    import oracle
    H, W = f.shape
    f64 = f.double().cpu().numpy() if hasattr(f, "cpu") else np.asarray(f, np.float64)
    ref = np.empty(len(pts))
    exact = np.empty(len(pts))
    for i, ((r, c), a) in enumerate(zip(pts, field)):
        a = np.maximum(a, 0.05)
        rx = int(_m.ceil(0.5 * a[0] + 0.25 * (a[1] + a[2]))) + 1
        ry = int(_m.ceil(0.25 * _m.sqrt(3.0) * (a[1] + a[2]))) + 1
        # the lattice is anchored at the image origin: the brute force takes
        # the whole image (it only visits the pixel's support)
        ref[i] = oracle.lattice3_points(f64, a, np.array([[r, c]]), 1.0, threads=1)[0]
        r0, r1, c0, c1 = max(0, r - ry), min(H, r + ry + 1), max(0, c - rx), min(W, c + rx + 1)
        exact[i] = oracle.points3(f64[r0:r1, c0:c1], a, np.array([[r - r0, c - c0]]), threads=1)[0]
    scale = max(float(np.abs(ref).max()), 1e-300)
    return {"max_rel_err": float(np.abs(got - ref).max() / scale), "pixels": int(len(pts)),
            "oracle": "lattice mode by brute force: exact N=3 kernel summed over the resampled image "
                      "(oracle/dense3_oracle.c rubs_oracle3_lattice_points)",
            "tolerance": 1e-9,
            "mode_error_vs_exact": {
                "max_rel": float(np.abs(got - exact).max() / max(float(np.abs(exact).max()), 1e-300)),
                "rms_rel": float(np.sqrt(np.mean((got - exact) ** 2)) / max(float(np.abs(exact).max()), 1e-300)),
                "note": "the mode's resampling error against the exact N=3 filter of the original image "
                        "(oracle/dense3_oracle.c), relative to max |output|; reported, not a bar"}}


# ---------------------------------------------------------------------------
# CPU leg: the reference algorithm on the host cores (cpu_baseline and the
# --impl reference arm).  Units are independent windows of the workload,
# exact by linearity + zero padding; a unit's halo costs pre-integration
# only (port.filter_window), not mesh work.

_PORT = {}


def _adaptive_worker(k):
    """One independent adaptive_smooth pipeline (oracle/tensor_port.py with
    the reference fast-path port as its filter) on crop k; returns pixels."""
    import oracle.port as port
    from oracle import tensor_port
    f, lut, noise, c = _PORT["f"], _PORT["lut"], _PORT["noise"], _PORT["crop"]
    r0 = (k * c) % (f.shape[0] - c)
    crop = f[r0:r0 + c, :c]
    tensor_port.adaptive_smooth(crop, noise, lut, filt=lambda a, fld, m=1: port.filter_space_variant(a, fld, m))
    return c * c


def _band3_worker(band):
    """One N=3 row band (oracle/port3.py); returns pixels produced."""
    from oracle import port3
    lo, hi = band
    port3.filter3_band(_PORT["f"], _PORT["field"], lo, hi)
    return (hi - lo) * _PORT["f"].shape[1]


def _band3l_worker(band):
    """One N=3 lattice-mode row band (oracle/lattice3_port.py lattice_pass on
    the band's crop with its support rows); returns pixels produced."""
    from oracle import lattice3_port as lp
    f, field = _PORT["f"], _PORT["field"]
    lo, hi = band
    a = np.maximum(field[lo:hi], lp.SCALE_FLOOR)
    ry = int(lp.support3(a)[1].max()) + 4
    r0, r1 = max(0, lo - ry), min(f.shape[0], hi + ry)
    lp.lattice_pass(f[r0:r1], r0, 0, a, lo, 0, 1.0)
    return (hi - lo) * f.shape[1]


def _band_worker(band):
    """One CPU-port row band (oracle B); returns pixels produced."""
    import oracle.port as port
    f, field, iters = _PORT["f"], _PORT["field"], _PORT["iters"]
    lo, hi = band
    port.filter_band(f, field, lo, hi, iters)
    return (hi - lo) * f.shape[1]


def _window_worker(k):
    """One pre-cut 2-D window of config 5 (crop + window field); returns pixels."""
    import oracle.port as port
    crop, cr0, cc0, fld, r0, c0 = _PORT["windows"][k]
    port.filter_window(crop, cr0, cc0, fld, r0, c0)
    return fld.shape[0] * fld.shape[1]


class CpuPort:
    """The reference algorithm (oracle/port.py, a numpy restatement of the
    reference fast path, pinned to it at 1e-14) on independent units of the
    config's workload, one process per host core."""

    def __init__(self, cfg: str, workers: int | None = None, wk=None):
        import multiprocessing as mp
        from oracle import port
        from paper_1003_2022_b200 import default_lut, workloads
        self.cfg = cfg
        self.cores = workers or os.cpu_count() or 1
        os.environ["OMP_NUM_THREADS"] = "1"
        lut = default_lut()
        self.H, self.W = SHAPES[cfg]
        self.note = ""
        if cfg == "A":
            w = workloads.adaptive_image()
            _PORT.update(f=w["f"], lut=(lut.rho_grid, lut.phi_grid, lut.entries),
                         noise=w["noise_sigma"], crop=256)
            self.jobs = list(range(self.cores))
            self.kind = "adaptive"
        elif cfg == "5":
            # 1024 x 1024 output windows of the real 32768^2 workload (the
            # device-resident image and fields), spread over the image; each
            # window's crop carries its read margins
            self._config5_windows(wk, lut)
            self.kind = "window"
        else:
            if cfg == "1":
                w = workloads.config1()
                field = w["field"]
            elif cfg == "2":
                w = workloads.config2()
            elif cfg in ("3", "3l"):
                from oracle import port3
                w = workloads.config3_n3(2048, 2048)
                self.note = (" (2048^2 instance of the config-3 N=3 recipe; oracle/port3.py)" if cfg == "3" else
                             " (2048^2 instance of the config-3 N=3 recipe; oracle/lattice3_port.py)")
            elif cfg == "3n4":
                w = workloads.config3(2048, 2048)
                self.note = " (2048^2 instance of the config-3 recipe)"
            else:
                w = workloads.config4_image(0)
                self.note = " (image 0 of the batch; two passes: each band's pass 1 covers its halo rows)"
            if cfg in ("3", "3l"):
                field = port3.scales3_from_params(w["size"].numpy(), w["elong"].numpy(), w["orient"].numpy())
            elif cfg != "1":
                field = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, w["size"].numpy(),
                                         w["elong"].numpy(), w["orient"].numpy())
            f = np.asarray(w["f"], dtype=np.float64)
            _PORT.update(f=f, field=field, iters=int(w["iterations"]))
            self.H, self.W = f.shape
            rows = max(64 if cfg != "4" else 128, -(-self.H // self.cores))
            if cfg == "3":
                rows = 32  # bounded sample: the N=3 port costs O(kernel height) per pixel
            self.bands = [(lo, min(self.H, lo + rows)) for lo in range(0, self.H, rows)][: self.cores]
            self.rows = rows
            self.jobs = self.bands
            self.kind = {"3": "band3", "3l": "band3l"}.get(cfg, "band")
        self.cores = len(self.jobs)
        self.pool = mp.get_context("fork").Pool(self.cores)

    def _config5_windows(self, wk, lut):
        import torch
        from oracle import port
        if wk is None:  # the reference arm: the same workload, generated on the device
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
            w = _load_workload("5", torch, dev)
            f, params = w["f"], [w["size"], w["elong"], w["orient"]]
        else:
            f, params = wk.sets[0]["f"] if wk.sets else None, None
            if f is None:
                raise RuntimeError("config-5 CPU windows need the whole-image workload (N=1)")
            params = wk.sets[0]["p"]
        H, W = f.shape
        T = 1024
        n = self.cores
        rng = np.random.default_rng(5)
        wins = []
        for k in range(n):
            r0 = int(rng.integers(0, H // T)) * T
            c0 = int(rng.integers(0, W // T)) * T
            par = [p[r0:r0 + T, c0:c0 + T].double().cpu().numpy() for p in params]
            fld = port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, *par)
            left, right, below, above = port.read_margins(np.maximum(fld, port.SCALE_FLOOR))
            cr0, cr1 = max(0, r0 - below - 1), min(H, r0 + T + above + 1)
            cc0, cc1 = max(0, c0 - left - 1), min(W, c0 + T + right + 1)
            crop = f[cr0:cr1, cc0:cc1].double().cpu().numpy()
            wins.append((crop, cr0, cc0, fld, r0, c0))
        _PORT["windows"] = wins
        self.jobs = list(range(n))
        self.T = T

    def step(self):
        worker = {"adaptive": _adaptive_worker, "window": _window_worker, "band3": _band3_worker,
                  "band3l": _band3l_worker, "band": _band_worker}[self.kind]
        t0 = time.perf_counter()
        px = sum(self.pool.map(worker, self.jobs))
        return px, time.perf_counter() - t0

    def sample(self):
        if self.kind == "adaptive":
            return (f"{self.cores} independent adaptive_smooth pipelines on 256x256 crops of the "
                    f"workload image (numpy restatement of tensor.py with the reference fast-path "
                    f"port as filter, oracle/tensor_port.py), {self.cores} processes x 1 thread")
        if self.kind == "window":
            return (f"{self.cores} output windows of {self.T}x{self.T} px at seeded random places of the "
                    f"config-5 32768^2 image and fields, each from its crop with read margins "
                    f"(halo pre-integrated only); numpy port of the reference fast path "
                    f"(oracle/port.py filter_window), {self.cores} processes x 1 thread")
        return (f"{len(self.bands)} row bands of {self.rows} rows x {self.W} cols "
                f"({sum(h - l for l, h in self.bands)} of {self.H} rows) of {WORKLOADS[self.cfg].split(':')[0]}"
                f"{self.note}, halo rows pre-integrated only; "
                + ("numpy restatement of the exact N=3 row-profile algorithm (oracle/port3.py)"
                   if self.cfg == "3" else
                   "numpy restatement of the N=3 lattice mode (oracle/lattice3_port.py)" if self.cfg == "3l"
                   else "numpy port of the reference fast path (oracle/port.py)")
                + f", {self.cores} processes x 1 thread")

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_port_throughput(cfg: str, steps: int = 1, warmup: int = 1, wk=None):
    cp = CpuPort(cfg, wk=wk)
    try:
        for _ in range(warmup):
            cp.step()
        px = el = 0.0
        for _ in range(steps):
            p, e = cp.step()
            px += p
            el += e
        return px / el / 1e6, cp.cores, cp.sample(), el
    finally:
        cp.close()


def run_reference(args, rank, world):
    if rank != 0:
        return None
    # bounded: a few steps of the CPU sample (each step is a full pass over
    # the sample, ~10-30 s of host work)
    steps = max(1, min(args.steps, 2))
    mpx, cores, sample, el = cpu_port_throughput(args.config, steps=steps, warmup=0)
    v = mpx / 1e3  # Gpixel/s
    return {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": 0,
        "ms_per_step": el / steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if row_banded(args.config, world) else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": bench_config(args.config, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def probe_launch(rank, world, local):
    """Launcher check: every rank joins a process group and reports."""
    import torch
    import torch.distributed as dist
    if world > 1:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        got = [None] * world
        dist.all_gather_object(got, {"rank": rank, "local": local, "pid": os.getpid()})
        dist.destroy_process_group()
    else:
        got = [{"rank": 0, "local": 0, "pid": os.getpid()}]
    if rank == 0:
        print(json.dumps({"probe": True, "n_gpus": world, "ranks": got}), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.probe_launch:
        probe_launch(rank, world, local)
        return
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res = run_ours(args, rank, world, local)
    if rank == 0 and res is not None:
        pin = res.pop("_parity_in", None)
        if world == 1 and not args.no_cpu_baseline:
            wk = None
            if args.config == "5":
                # the CPU windows are cut from the device-resident workload
                wk = _WK_FOR_CPU.get("wk")
            mpx, cores, sample, el = cpu_port_throughput(args.config, steps=1, warmup=0, wk=wk)
            res["cpu_baseline"] = {"value": mpx / 1e3, "unit": UNIT, "cores": cores, "kind": "port",
                                   "sample": sample, "wall_s": el}
            if pin is not None:
                res["parity"] = parity_check(args.config, pin)
        print(json.dumps(res), flush=True)


_WK_FOR_CPU: dict = {}

if __name__ == "__main__":
    main()
