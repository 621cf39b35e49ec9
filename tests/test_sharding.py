"""Multi-GPU partition logic on CPU (gloo, world size 2): batch assignment,
row-band bounds, halo needs and the halo exchange itself.  The filter used
inside the bands here is the CPU port (oracle/port.py) -- the point is the
partition: band results reproduce the whole-image result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1003_2022_b200 import sharding


def test_batch_indices_cover_batch_once():
    for world in (1, 2, 4, 8):
        seen = sorted(i for r in range(world) for i in sharding.batch_indices(64, world, r))
        assert seen == list(range(64))


def test_band_bounds_aligned_and_covering():
    for H in (1, 31, 32, 100, 2048, 32768, 32769):
        for world in (1, 2, 3, 4, 8):
            b = sharding.band_bounds(H, world)
            assert b[0][0] == 0 and b[-1][1] == H
            for (a0, a1), (b0, b1) in zip(b, b[1:]):
                assert a1 == b0
            for r0, r1 in b:
                assert r0 % 32 == 0 or r0 == H
                assert r1 % 32 == 0 or r1 == H


def test_transfers_are_symmetric():
    bands = sharding.band_bounds(1000, 4)
    needs = [sharding.needed_rows(b, (0, 0, 40, 300), 1000) for b in bands]
    sends = {r: sharding.transfers(bands, needs, r)[0] for r in range(4)}
    recvs = {r: sharding.transfers(bands, needs, r)[1] for r in range(4)}
    for r in range(4):
        for peer, lo, hi in recvs[r]:
            assert (r, lo, hi) in sends[peer]
    # a halo wider than one band reaches past the neighbour
    assert any(len(recvs[r]) >= 2 for r in range(4))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, f, field, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as cpu
        H = f.shape[0]
        bands = sharding.band_bounds(H, world)
        band = bands[rank]
        own = torch.from_numpy(f[band[0]:band[1]].copy())
        fld = cpu.prepare_field(field, f.shape, 1)
        margins = cpu.read_margins(fld[band[0]:band[1]])
        needs = sharding.gather_needs(sharding.needed_rows(band, margins, H))
        rows = sharding.exchange_rows(own, band, bands, needs, rank)
        n0, n1 = needs[rank]
        assert np.array_equal(rows.numpy(), f[n0:n1])
        out = cpu.filter_space_variant(rows.numpy(), field[n0:n1])[band[0] - n0:band[1] - n0]
        parts = [None] * world
        dist.all_gather_object(parts, out)
        if rank == 0:
            ret.put(np.concatenate(parts))
    finally:
        dist.destroy_process_group()


def test_row_bands_with_halo_exchange_reproduce_whole_image():
    rng = np.random.default_rng(3)
    H, W = 200, 48
    f = rng.random((H, W))
    field = np.stack([np.full((H, W), 2.0), np.linspace(1.0, 30.0, H)[:, None] * np.ones((1, W)),
                      np.full((H, W), 1.5), np.full((H, W), 3.0)], axis=-1)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    procs = mp.start_processes(_worker, args=(2, _free_port(), f, field, ret), nprocs=2,
                               join=False, start_method="spawn")
    banded = ret.get(timeout=120)  # before join: a queue holding data blocks exit
    procs.join()
    from oracle import port as cpu
    whole = cpu.filter_space_variant(f, field)
    assert banded.shape == whole.shape
    assert np.abs(banded - whole).max() < 1e-9


def _worker3(rank, world, port, f, field, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port3
        H, W = f.shape
        bands = sharding.band_bounds(H, world, sharding.TILE3)
        band = bands[rank]
        own = torch.from_numpy(f[band[0]:band[1]].copy())
        _, ry = port3.support3(np.maximum(field[band[0]:band[1]], 0.05))
        needs = sharding.gather_needs(sharding.needed_rows3(band, ry, H))
        rows = sharding.exchange_rows(own, band, bands, needs, rank)
        n0, n1 = needs[rank]
        assert np.array_equal(rows.numpy(), f[n0:n1])
        a = np.maximum(field[band[0]:band[1]], 0.05)
        out = port3.pass3(rows.numpy(), 0, n0, a, 0, band[0], W, band[1] - band[0])
        parts = [None] * world
        dist.all_gather_object(parts, out)
        if rank == 0:
            ret.put(np.concatenate(parts))
    finally:
        dist.destroy_process_group()


def test_three_direction_row_bands_reproduce_whole_image():
    """N=3 bands (64-row grid, reach = vertical kernel half-extent) with the
    halo exchange at world size 2; the band filter is the numpy restatement."""
    from oracle import port3
    rng = np.random.default_rng(5)
    H, W = 200, 40
    f = rng.random((H, W))
    field = np.stack([np.full((H, W), 3.0), np.linspace(1.0, 60.0, H)[:, None] * np.ones((1, W)),
                      np.full((H, W), 2.5)], axis=-1)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    procs = mp.start_processes(_worker3, args=(2, _free_port(), f, field, ret), nprocs=2,
                               join=False, start_method="spawn")
    banded = ret.get(timeout=120)
    procs.join()
    whole = port3.filter3(f, field)
    assert np.abs(banded - whole).max() < 1e-11


def test_halo_bounds_cover_the_exact_margins(rng):
    """The cheap halo bounds used by the row-band filters are >= the exact
    per-pixel margins (N=4 LUT mapping, N=3 closed form)."""
    import math
    from oracle import port, port3
    from paper_1003_2022_b200 import default_lut
    lut = default_lut()
    n = 4000
    size = rng.uniform(0.1, 2.0e5, n)
    th = rng.uniform(0.0, math.pi, n)
    rho = rng.uniform(1.0, 5.79, n)
    a = np.maximum(port.lookup_many(lut.rho_grid, lut.phi_grid, lut.entries, size, rho, th), 0.05)
    exact = port.read_margins(a)
    bound = sharding.halo_bound_params(size, lut)
    assert all(b >= e for b, e in zip(bound, exact))
    from paper_1003_2022_b200 import elongation_bound3
    rho3 = 1.0 + (np.minimum(elongation_bound3(th), 40.0) - 1.0) * rng.uniform(0.0, 0.95, n)
    a3 = np.maximum(port3.scales3_from_params(size, rho3, th), 0.05)
    assert sharding.reach3_bound_params(size) >= port3.support3(a3)[1]


def _worker_plan(rank, world, port, f, field, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as cpu
        H, W = f.shape
        band = sharding.band_bounds(H, world)[rank]
        fld = cpu.prepare_field(field, f.shape, 1)
        _, _, below, above = cpu.read_margins(fld[band[0]:band[1]])
        plan = sharding.RowBandPlan(band, H, (below, above))
        calls = []

        def filt(f_rows, f_row0, r0, n, out):
            # the CPU port on the given rows only: rows it lacks are zero,
            # so a wrong split or a missing halo row shows up as an error
            calls.append((f_row0, f_rows.shape[0], r0, n))
            out.copy_(torch.from_numpy(cpu.filter_window(f_rows.numpy(), f_row0, 0, field[r0:r0 + n], r0, 0)))

        out = plan.run(torch.from_numpy(f[band[0]:band[1]].copy()), filt)
        res = [None] * world
        dist.all_gather_object(res, (out.numpy(), calls, plan.interior))
        if rank == 0:
            ret.put(res)
    finally:
        dist.destroy_process_group()


def test_row_band_plan_overlaps_interior_and_reproduces_whole_image():
    """RowBandPlan: interior rows from the rank's own rows (before the halo
    arrives), edge rows after the exchange; together == the whole image."""
    rng = np.random.default_rng(11)
    H, W = 320, 40
    f = rng.random((H, W))
    field = np.stack([np.full((H, W), 2.0), np.full((H, W), 6.0), np.full((H, W), 1.5),
                      np.full((H, W), 4.0)], axis=-1)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    procs = mp.start_processes(_worker_plan, args=(2, _free_port(), f, field, ret), nprocs=2,
                               join=False, start_method="spawn")
    res = ret.get(timeout=120)
    procs.join()
    import oracle
    whole = oracle.dense(f, field)  # exact (the whole-image port has ~2e-9 of global-sum error here)
    banded = np.concatenate([r[0] for r in res])
    assert np.abs(banded - whole).max() < 1e-9 * np.abs(whole).max()  # the port's own sum error
    for out, calls, interior in res:
        assert interior is not None  # 160-row bands, ~7-row halos
        # the interior call reads only the rank's own rows
        assert calls[0][2] == interior[0] and calls[0][3] == interior[1] - interior[0]
        assert interior[0] % 32 == 0 and (interior[1] % 32 == 0 or interior[1] == H)
        assert len(calls) == 2  # interior + the one edge facing the other rank


def _worker_lattice(rank, world, port, f, field, size, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import lattice3_port as lp
        H, W = f.shape
        band = sharding.band_bounds(H, world, sharding.TILE3L)[rank]
        plan = sharding.row_band_plan3_lattice(band, H, torch.from_numpy(size[band[0]:band[1]]))
        calls = []

        def filt(f_rows, f_row0, r0, n, out):
            # the numpy restatement of the lattice pass on the given rows only
            # (rows it lacks are zero: a missing halo row shows up as an error)
            calls.append((f_row0, f_rows.shape[0], r0, n))
            a = np.maximum(field[r0:r0 + n], lp.SCALE_FLOOR)
            out.copy_(torch.from_numpy(lp.lattice_pass(f_rows.numpy(), f_row0, 0, a, r0, 0, 1.0)))

        out = plan.run(torch.from_numpy(f[band[0]:band[1]].copy()), filt)
        res = [None] * world
        dist.all_gather_object(res, (out.numpy(), calls, plan.interior))
        if rank == 0:
            ret.put(res)
    finally:
        dist.destroy_process_group()


def test_lattice_mode_row_bands_reproduce_whole_image():
    """N=3 lattice mode in row bands at world size 2: the halo is the
    kernels' reach bound plus the resampling footprint; interior rows are
    filtered from the rank's own rows while the exchange is in flight."""
    from oracle import lattice3_port as lp, port3
    rng = np.random.default_rng(13)
    H, W = 256, 36
    f = rng.random((H, W))
    size = np.linspace(2.0, 40.0, H)[:, None] * np.ones((1, W))
    th = rng.uniform(0.0, np.pi, (H, W))
    rho = np.full((H, W), 1.5)
    field = port3.scales3_from_params(size, rho, th)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    procs = mp.start_processes(_worker_lattice, args=(2, _free_port(), f, field, size, ret), nprocs=2,
                               join=False, start_method="spawn")
    res = ret.get(timeout=120)
    procs.join()
    whole = lp.lattice3(f, field)
    banded = np.concatenate([r[0] for r in res])
    assert np.abs(banded - whole).max() < 1e-10 * np.abs(whole).max()
    for out, calls, interior in res:
        assert interior is not None and len(calls) == 2


def test_lattice_halo_bound_covers_the_support(rng):
    import math
    from oracle import port3
    from paper_1003_2022_b200 import elongation_bound3
    n = 4000
    size = rng.uniform(0.1, 2.0e5, n)
    th = rng.uniform(0.0, math.pi, n)
    rho3 = 1.0 + (np.minimum(elongation_bound3(th), 40.0) - 1.0) * rng.uniform(0.0, 0.999, n)
    a3 = np.maximum(port3.scales3_from_params(size, rho3, th), 0.05)
    ry = int(np.max(port3.support3(a3)[1]))
    assert sharding.reach3_lattice_bound(size) >= ry + 1  # + the resampling footprint
    # the device's own bound (csrc lat_sizebound_kernel) in numpy: a1 <= sqrt(12 s), a2 + a3 <= sqrt(32 s)
    assert np.all(a3[:, 0] <= np.sqrt(12.0 * size) * (1 + 1e-12) + 0.05)
    assert np.all(a3[:, 1] + a3[:, 2] <= np.sqrt(32.0 * size) * (1 + 1e-12) + 0.1)
