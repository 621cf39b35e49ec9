"""Multi-GPU sharding of the filter path.

Two decompositions, one process per GPU (torch.distributed, NCCL on GPUs,
gloo on CPU for the tests):

* batches (BASELINE config 4): images are independent -- each rank filters
  its own images, there is no data-path collective (``batch_indices``);
* row bands (configs 5 and, with three directions, 3): one large image is split into horizontal bands of
  output rows.  A rank needs the input rows its outputs read -- its band
  grown by the read margins (engine.py:247-262) -- so the one exchange step
  is a halo exchange of image rows with the neighbouring ranks
  (``exchange_rows``), sized by an all-gather of every rank's needs.  Band
  edges sit on the 32-row tile grid, so tiles of the shared-memory path
  reproduce the single-GPU result bit for bit.

The reference has no parallelism at all; its SPEC only asks for
determinism, which this partition keeps.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

TILE = 32


def batch_indices(n_images: int, world: int, rank: int) -> list[int]:
    """Round-robin assignment of a batch's images to ranks."""
    return list(range(rank, n_images, world))


def band_bounds(H: int, world: int, align: int = TILE) -> list[tuple[int, int]]:
    """Contiguous output-row bands, edges multiples of `align` (balanced)."""
    units = -(-H // align)
    base, extra = divmod(units, world)
    out, lo = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        hi = min(H, lo + n * align)
        out.append((min(lo, H), hi))
        lo = hi
    return out


def needed_rows(band: tuple[int, int], margins, H: int, slack: int = 1) -> tuple[int, int]:
    """Input rows a band's outputs read: the band grown by the read margins
    (below, above) plus the one-row slack of the tile regions."""
    r0, r1 = band
    if r1 <= r0:
        return (r0, r0)
    below, above = int(margins[2]), int(margins[3])
    return (max(0, r0 - below - slack), min(H, r1 + above + slack))


def transfers(bands, needs, rank: int):
    """(sends, recvs) of this rank: lists of (peer, lo, hi) global row ranges;
    a rank sends the part of its own band that a peer needs and receives the
    parts of its need owned by peers."""
    sends, recvs = [], []
    own = bands[rank]
    for peer, (n0, n1) in enumerate(needs):
        if peer == rank:
            continue
        lo, hi = max(own[0], n0), min(own[1], n1)
        if lo < hi:
            sends.append((peer, lo, hi))
    n0, n1 = needs[rank]
    for peer, (b0, b1) in enumerate(bands):
        if peer == rank:
            continue
        lo, hi = max(b0, n0), min(b1, n1)
        if lo < hi:
            recvs.append((peer, lo, hi))
    return sends, recvs


def gather_needs(need: tuple[int, int], group=None, device=None):
    """All ranks' (lo, hi) needs (one small all-gather)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([need[0], need[1]], dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [(int(v[0]), int(v[1])) for v in out]


def exchange_rows(own, band, bands, needs, rank: int, group=None):
    """Return the image rows [needs[rank]) given this rank's own rows
    (tensor ``own`` = rows [band)); missing rows come from the peers that
    own them (batched isend/irecv, so NCCL runs them as one group)."""
    import torch
    import torch.distributed as dist
    n0, n1 = needs[rank]
    W = own.shape[1]
    out = torch.empty((n1 - n0, W), dtype=own.dtype, device=own.device)
    lo, hi = max(band[0], n0), min(band[1], n1)
    if lo < hi:
        out[lo - n0:hi - n0] = own[lo - band[0]:hi - band[0]]
    sends, recvs = transfers(bands, needs, rank)
    ops = []
    for peer, s0, s1 in sends:
        ops.append(dist.P2POp(dist.isend, own[s0 - band[0]:s1 - band[0]].contiguous(), peer, group))
    bufs = []
    for peer, r0, r1 in recvs:
        buf = torch.empty((r1 - r0, W), dtype=own.dtype, device=own.device)
        bufs.append((r0, r1, buf))
        ops.append(dist.P2POp(dist.irecv, buf, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r0, r1, buf in bufs:
        out[r0 - n0:r1 - n0] = buf
    return out


class RowBandPlan:
    """One rank's share of a row-band filter, planned once per field.

    The halo reach (below, above) and the all-gather of every rank's needed
    rows happen at construction, not per call.  ``run`` posts the halo
    exchange (batched isend / irecv: NCCL runs it on its own stream), then
    computes the band's INTERIOR output rows -- those whose reads lie inside
    the rank's own rows -- while the transfer is in flight, and only then
    waits for the halo and computes the rows next to the band edges.  The
    output rows are split on the tile grid (``align``), so the shared-memory
    tiles are the ones a single call would use.

    ``filt(f_rows, f_row0, out_row0, out_rows, out)`` computes output rows
    [out_row0, out_row0 + out_rows) into ``out`` from image rows
    [f_row0, f_row0 + len(f_rows)) (the product: ``filter_rows_params``; the
    gloo tests pass the CPU port)."""

    def __init__(self, band, H: int, reach, group=None, align: int = TILE, device=None):
        import torch.distributed as dist
        world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        self.H = H
        self.bands = band_bounds(H, world, align)
        self.band = tuple(band)
        assert self.band == self.bands[self.rank], "band must match band_bounds(H, world)[rank]"
        below, above = int(reach[0]), int(reach[1])
        self.needs = gather_needs(needed_rows(self.band, (0, 0, below, above), H), group, device)
        self.sends, self.recvs = transfers(self.bands, self.needs, self.rank)
        b0, b1 = self.band
        lo = b0 if b0 == 0 else b0 + below + 1  # needed_rows' one-row slack
        hi = b1 if b1 == H else b1 - above - 1
        i0 = b0 + -(-(lo - b0) // align) * align
        i1 = hi if hi == H else b0 + ((hi - b0) // align) * align
        self.interior = (i0, i1) if i1 > i0 else None

    def run(self, own, filt):
        import torch
        import torch.distributed as dist
        b0, b1 = self.band
        n0, n1 = self.needs[self.rank]
        W = own.shape[1]
        ops, bufs = [], []
        for peer, s0, s1 in self.sends:
            ops.append(dist.P2POp(dist.isend, own[s0 - b0:s1 - b0].contiguous(), peer, self.group))
        for peer, r0, r1 in self.recvs:
            buf = torch.empty((r1 - r0, W), dtype=own.dtype, device=own.device)
            bufs.append((r0, r1, buf))
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        out = torch.empty((b1 - b0, W), dtype=torch.float64, device=own.device)
        if self.interior is not None:
            i0, i1 = self.interior
            filt(own, b0, i0, i1 - i0, out[i0 - b0:i1 - b0])
        for req in reqs:
            req.wait()
        if self.interior is not None and not bufs and (n0, n1) == (b0, b1):
            f_need = own
        else:
            f_need = torch.empty((n1 - n0, W), dtype=own.dtype, device=own.device)
            lo, hi = max(b0, n0), min(b1, n1)
            if lo < hi:
                f_need[lo - n0:hi - n0] = own[lo - b0:hi - b0]
            for r0, r1, buf in bufs:
                f_need[r0 - n0:r1 - n0] = buf
        parts = [(b0, b1)] if self.interior is None else [(b0, self.interior[0]), (self.interior[1], b1)]
        for r0, r1 in parts:
            if r1 > r0:
                filt(f_need, n0, r0, r1 - r0, out[r0 - b0:r1 - b0])
        return out


# --- device calls (C ABI) --------------------------------------------------


def read_margins_params(size, elong, orient, row0: int, H: int, lut=None, iterations: int = 1):
    """Exact read margins (left, right, below, above) of parameter rows
    [row0, row0 + rows) (CUDA tensors); engine.py:247-262."""
    import torch
    from . import _native
    from .engine import _stream_handle, device_lut
    dl = device_lut(lut, size.device)
    ps = [v.contiguous() for v in (size, elong, orient)]
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    out4 = (ctypes.c_int * 4)()
    with torch.cuda.device(ps[0].device):
        _native.check(_native.load().rubs_b200_read_margins_params(
            *(ctypes.c_void_p(p.data_ptr()) for p in ps), pdt, ps[0].shape[0], ps[0].shape[1],
            ps[0].stride(0), H, row0, dl.handle, iterations, out4, _stream_handle()))
    return tuple(out4)


def filter_rows_params(f_rows, f_row0: int, H: int, size, elong, orient, p_row0: int,
                       out_row0: int, out_rows: int, lut=None, out=None):
    """Output rows [out_row0, out_row0 + out_rows) of the H-row image whose rows
    [f_row0, f_row0 + len(f_rows)) are given (rubs_b200_filter_params_rows)."""
    import torch
    from . import _native
    from .engine import _stream_handle, device_lut
    dl = device_lut(lut, f_rows.device)
    f_rows = f_rows.contiguous()
    ps = [v.contiguous() for v in (size, elong, orient)]
    W = f_rows.shape[1]
    if out is None:
        out = torch.empty((out_rows, W), dtype=torch.float64, device=f_rows.device)
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    fdt = _native.RUBS_F32 if f_rows.dtype == torch.float32 else _native.RUBS_F64
    with torch.cuda.device(f_rows.device):
        _native.check(_native.load().rubs_b200_filter_params_rows(
            ctypes.c_void_p(f_rows.data_ptr()), fdt, f_row0, f_rows.shape[0], W, f_rows.stride(0), H,
            *(ctypes.c_void_p(p.data_ptr()) for p in ps), pdt, p_row0, ps[0].stride(0), dl.handle,
            out_row0, out_rows, ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_handle()))
    return out


def halo_bound_params(size, lut=None) -> tuple:
    """Read-margin bound (left, right, below, above) of LUT-mapped kernels
    with sizes up to size.max(): every mapped component is a convex blend of
    table entries times sqrt(size) (solver.py:289-335), and the margins of
    engine.py:247-262 grow with each component.  One reduction over the
    band's size plane instead of mapping every pixel (the exact
    read_margins_params costs about half a band's filter time at 8 ranks);
    a wider halo changes nothing but the rows exchanged."""
    from .solver import default_lut
    lut = lut or default_lut()
    smax = float(size.max().item()) if hasattr(size, "max") else float(np.max(size))
    A = max(float(np.max(lut.entries)) * math.sqrt(max(smax, 0.0)), 0.05)
    m = int(math.ceil(0.5 * A + A / math.sqrt(2.0) + 1.5)) + 3
    return (m, m, m, m)


def row_band_plan(band, H: int, size, lut=None, group=None):
    """The RowBandPlan of an N=4 LUT band (halo from ``halo_bound_params``)."""
    m = halo_bound_params(size, lut)
    return RowBandPlan(band, H, (m[2], m[3]), group, TILE, device=size.device)


def filter_row_band(f_own, band, H: int, size, elong, orient, lut=None, group=None, plan=None):
    """One rank's share of a row-band filter: this rank holds image rows
    ``band`` (f_own) and the parameter rows of the same band; returns its
    output rows.  Collective over the group (halo exchange; the needs
    all-gather too unless a ``plan`` from ``row_band_plan`` is given)."""
    plan = plan or row_band_plan(band, H, size, lut, group)

    def filt(f_rows, f_row0, r0, n, out):
        filter_rows_params(f_rows, f_row0, H, size, elong, orient, band[0], r0, n, lut, out=out)

    return plan.run(f_own, filt)


# --- three directions (config 3) -------------------------------------------
# Same decomposition; the N=3 kernel's tiles are 64 rows tall, so band edges
# sit on the 64-row grid (bitwise equal to the whole-image result), and a
# band's reach is the vertical half-extent of its kernels
# (rubs_b200_read_margins3_params).

TILE3 = 64


def read_margins3_params(size, elong, orient):
    """(columns, rows) reach of the N=3 kernels of these parameter rows."""
    import torch
    from . import _native
    from .engine import _stream_handle
    ps = [v.contiguous() for v in (size, elong, orient)]
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    out2 = (ctypes.c_int * 2)()
    with torch.cuda.device(ps[0].device):
        _native.check(_native.load().rubs_b200_read_margins3_params(
            *(ctypes.c_void_p(p.data_ptr()) for p in ps), pdt, ps[0].shape[0], ps[0].shape[1],
            ps[0].stride(0), out2, _stream_handle()))
    return tuple(out2)


def needed_rows3(band, reach_rows: int, H: int):
    """Image rows an N=3 band reads."""
    r0, r1 = band
    if r1 <= r0:
        return (r0, r0)
    return (max(0, r0 - reach_rows), min(H, r1 + reach_rows))


def filter3_rows_params(f_rows, f_row0: int, H: int, size, elong, orient, p_row0: int,
                        out_row0: int, out_rows: int, out=None):
    """N=3 output rows [out_row0, out_row0 + out_rows) of the H-row image whose
    rows [f_row0, f_row0 + len(f_rows)) are given (rubs_b200_filter3_params_rows)."""
    import torch
    from . import _native
    from .engine import _stream_handle
    f_rows = f_rows.contiguous()
    ps = [v.contiguous() for v in (size, elong, orient)]
    W = f_rows.shape[1]
    if out is None:
        out = torch.empty((out_rows, W), dtype=torch.float64, device=f_rows.device)
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    fdt = _native.RUBS_F32 if f_rows.dtype == torch.float32 else _native.RUBS_F64
    with torch.cuda.device(f_rows.device):
        _native.check(_native.load().rubs_b200_filter3_params_rows(
            ctypes.c_void_p(f_rows.data_ptr()), fdt, f_row0, f_rows.shape[0], W, f_rows.stride(0), H,
            *(ctypes.c_void_p(p.data_ptr()) for p in ps), pdt, p_row0, ps[0].stride(0),
            out_row0, out_rows, ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_handle()))
    return out


def reach3_bound_params(size) -> int:
    """Row reach bound of N=3 kernels with sizes up to size.max(): the
    closed-form scales satisfy a_k^2 = 12 p_k <= 15 size (p_k <= (2/3 +
    1/sqrt3) size), and the reach is ceil((a2 + a3) sqrt3 / 4) + 1."""
    smax = float(size.max().item()) if hasattr(size, "max") else float(np.max(size))
    a = max(math.sqrt(15.0 * max(smax, 0.0)), 0.05)
    return int(math.ceil(0.5 * math.sqrt(3.0) * a)) + 2


def row_band_plan3(band, H: int, size, group=None):
    """The RowBandPlan of an N=3 band (64-row grid, reach_bound rows)."""
    reach = reach3_bound_params(size)
    return RowBandPlan(band, H, (reach - 1, reach - 1), group, TILE3, device=size.device)


def filter3_row_band(f_own, band, H: int, size, elong, orient, group=None, plan=None):
    """One rank's share of an N=3 row-band filter (band = band_bounds(H,
    world, TILE3)[rank]); collective over the group, like filter_row_band."""
    plan = plan or row_band_plan3(band, H, size, group)

    def filt(f_rows, f_row0, r0, n, out):
        filter3_rows_params(f_rows, f_row0, H, size, elong, orient, band[0], r0, n, out=out)

    return plan.run(f_own, filt)


# --- three directions, lattice mode (O(1) per pixel) ------------------------
# The lattice pass is exact after the resampling, and a pixel's output only
# depends on the resampled image inside its kernel support, so a band needs
# its kernels' vertical reach plus the resampling footprint (one pixel row)
# of halo; rows beyond that may be missing (they count as zero).  There is no
# tile grid: band edges sit on a 32-row grid for even sizes only.  Bands
# reproduce the whole-image call up to the blocks' quantisation exponents
# (~1e-17 relative), not bit for bit.

TILE3L = 32


def filter3_lattice_rows_params(f_rows, f_row0: int, H: int, size, elong, orient, p_row0: int,
                                out_row0: int, out_rows: int, out=None, spacing: float = 1.0):
    """Lattice-mode N=3 output rows [out_row0, out_row0 + out_rows) of the
    H-row image whose rows [f_row0, f_row0 + len(f_rows)) are given
    (rubs_b200_filter3_lattice_params_rows)."""
    import torch
    from . import _native
    from .engine import _stream_handle
    f_rows = f_rows.contiguous()
    ps = [v.contiguous() for v in (size, elong, orient)]
    W = f_rows.shape[1]
    if out is None:
        out = torch.empty((out_rows, W), dtype=torch.float64, device=f_rows.device)
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    fdt = _native.RUBS_F32 if f_rows.dtype == torch.float32 else _native.RUBS_F64
    with torch.cuda.device(f_rows.device):
        _native.check(_native.load().rubs_b200_filter3_lattice_params_rows(
            ctypes.c_void_p(f_rows.data_ptr()), fdt, f_row0, f_rows.shape[0], W, f_rows.stride(0), H,
            *(ctypes.c_void_p(p.data_ptr()) for p in ps), pdt, p_row0, ps[0].stride(0),
            out_row0, out_rows, float(spacing), ctypes.c_void_p(out.data_ptr()), out.stride(0),
            _stream_handle()))
    return out


def reach3_lattice_bound(size) -> int:
    """Halo rows of a lattice-mode band with sizes up to size.max(): the
    kernels' vertical reach ceil((a2 + a3) sqrt3 / 4) + 1 with a2 + a3 <=
    sqrt(32 size) (a2^2 + a3^2 = 16 C22 <= 16 size), plus the resampling
    footprint (each lattice point draws on pixels within one row)."""
    smax = float(size.max().item()) if hasattr(size, "max") else float(np.max(size))
    a23 = math.sqrt(32.0 * max(smax, 1.0)) * (1.0 + 1e-9) + 0.1
    return int(math.ceil(0.25 * math.sqrt(3.0) * a23)) + 3


def row_band_plan3_lattice(band, H: int, size, group=None):
    """The RowBandPlan of a lattice-mode N=3 band."""
    reach = reach3_lattice_bound(size)
    return RowBandPlan(band, H, (reach - 1, reach - 1), group, TILE3L, device=size.device)


def filter3_lattice_row_band(f_own, band, H: int, size, elong, orient, group=None, plan=None,
                             spacing: float = 1.0):
    """One rank's share of a lattice-mode N=3 row-band filter (band =
    band_bounds(H, world, TILE3L)[rank]); collective over the group."""
    plan = plan or row_band_plan3_lattice(band, H, size, group)

    def filt(f_rows, f_row0, r0, n, out):
        filter3_lattice_rows_params(f_rows, f_row0, H, size, elong, orient, band[0], r0, n, out=out,
                                    spacing=spacing)

    return plan.run(f_own, filt)
