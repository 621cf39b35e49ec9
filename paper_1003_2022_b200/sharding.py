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


# --- device calls (C ABI) --------------------------------------------------


def read_margins_params(size, elong, orient, row0: int, H: int, lut=None, iterations: int = 1):
    """Exact read margins (left, right, below, above) of parameter rows
    [row0, row0 + rows) (CUDA tensors); engine.py:247-262."""
    import torch
    from . import _native
    from .engine import _stream_handle, device_lut
    dl = device_lut(lut)
    ps = [v.contiguous() for v in (size, elong, orient)]
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    out4 = (ctypes.c_int * 4)()
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
    dl = device_lut(lut)
    f_rows = f_rows.contiguous()
    ps = [v.contiguous() for v in (size, elong, orient)]
    W = f_rows.shape[1]
    if out is None:
        out = torch.empty((out_rows, W), dtype=torch.float64, device=f_rows.device)
    pdt = _native.RUBS_F32 if ps[0].dtype == torch.float32 else _native.RUBS_F64
    fdt = _native.RUBS_F32 if f_rows.dtype == torch.float32 else _native.RUBS_F64
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


def filter_row_band(f_own, band, H: int, size, elong, orient, lut=None, group=None):
    """One rank's share of a row-band filter: this rank holds image rows
    ``band`` (f_own) and the parameter rows of the same band; returns its
    output rows.  Collective over the group (needs all-gather + halos)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bands = band_bounds(H, world)
    assert tuple(band) == bands[rank], "band must match band_bounds(H, world)[rank]"
    margins = halo_bound_params(size, lut)
    needs = gather_needs(needed_rows(band, margins, H), group, device=f_own.device)
    f_need = exchange_rows(f_own, band, bands, needs, rank, group)
    return filter_rows_params(f_need, needs[rank][0], H, size, elong, orient, band[0], band[0],
                              band[1] - band[0], lut)


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


def filter3_row_band(f_own, band, H: int, size, elong, orient, group=None):
    """One rank's share of an N=3 row-band filter (band = band_bounds(H,
    world, TILE3)[rank]); collective over the group (needs all-gather +
    halo exchange), like filter_row_band."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bands = band_bounds(H, world, TILE3)
    assert tuple(band) == bands[rank], "band must match band_bounds(H, world, TILE3)[rank]"
    reach = reach3_bound_params(size)
    needs = gather_needs(needed_rows3(band, reach, H), group, device=f_own.device)
    f_need = exchange_rows(f_own, band, bands, needs, rank, group)
    return filter3_rows_params(f_need, needs[rank][0], H, size, elong, orient, band[0], band[0],
                               band[1] - band[0])
