"""CPU: the multi-GPU decomposition (paper_2509_08574_b200/shard.py).

* the angle / slab shards partition the work exactly (world_size 2, gloo);
* the decomposition is exact for the reference's Siddon model: concatenated
  angle-shard forward projections and stacked slab adjoints reproduce the
  full operators (checked with the float64 oracle);
* the bench's max-over-ranks device time reduction runs over gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2509_08574_b200 as k
from oracle import Geometry, Grid, Oracle
from paper_2509_08574_b200 import shard
from tests._util import tiny_geometry


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = k.GridSpec((16, 12, 10), (1.0, 1.0, 1.0))
    geom = k.ConeBeamGeometry(1000.0, 1500.0, 8, 8, 1.0, 1.0, k.uniform_angles(7))
    sg = shard.shard_geometry(geom, world, rank)
    sl = shard.slab_grid(grid, world, rank)
    z0, z1 = shard.slab_range(grid.dims[2], world, rank)
    mine = torch.tensor(shard.angle_indices(geom.n_angles(), world, rank).tolist()
                        + [-1] * (4 - sg.n_angles()))
    allang = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allang, mine)
    slabs = [torch.zeros(2, dtype=torch.long) for _ in range(world)]
    dist.all_gather(slabs, torch.tensor([z0, z1]))
    t = torch.tensor([0.5 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((sorted(int(a) for x in allang for a in x if a >= 0),
               [tuple(int(v) for v in s) for s in slabs], float(t.item()),
               sl.origin[2]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    angles, slabs, tmax, oz0 = q.get()
    assert angles == list(range(7))
    assert slabs == [(0, 5), (5, 10)]
    assert tmax == 1.5
    assert oz0 == -5.0


@pytest.mark.parametrize("world", [2, 3, 4])
def test_slab_ranges_cover(world):
    for nz in (1, 7, 64, 256, 513):
        if nz < world:
            continue
        rs = [shard.slab_range(nz, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_decomposition_is_exact_float64():
    """Angle shards of A and slab blocks of A^T reproduce the full operators."""
    ora = Oracle("ora")
    grid = Grid(6, 5, 8, 1.0, 1.1, 0.9)
    geom = tiny_geometry(6, 10, 9)
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, grid.count)
    y = rng.uniform(-1, 1, geom.ray_count)
    full_fwd = ora.forward(grid, geom, x).reshape(geom.n_angles, -1)
    full_adj = ora.adjoint(grid, geom, y).reshape(grid.nz, -1)
    world = 2
    kg = k.GridSpec((grid.nx, grid.ny, grid.nz), (grid.sx, grid.sy, grid.sz),
                    (grid.ox, grid.oy, grid.oz))
    kge = k.ConeBeamGeometry(geom.dso, geom.dsd, geom.nu, geom.nv, geom.pu, geom.pv, geom.angles,
                             geom.offset_u, geom.offset_v)
    for r in range(world):
        sg = shard.shard_geometry(kge, world, r)
        og = Geometry(sg.dso, sg.dsd, sg.nu, sg.nv, sg.pu, sg.pv, sg.angles, sg.offset_u,
                      sg.offset_v)
        part = ora.forward(grid, og, x).reshape(sg.n_angles(), -1)
        np.testing.assert_array_equal(part, full_fwd[shard.angle_indices(geom.n_angles, world, r)])
        sl = shard.slab_grid(kg, world, r)
        osl = Grid(*sl.dims, *sl.spacing, *sl.origin)
        z0, z1 = shard.slab_range(grid.nz, world, r)
        blk = ora.adjoint(osl, geom, y).reshape(z1 - z0, -1)
        np.testing.assert_allclose(blk, full_adj[z0:z1], rtol=1e-12, atol=1e-12)
        sl = shard.slab_grid(kg, world, r, axis="y")
        osl = Grid(*sl.dims, *sl.spacing, *sl.origin)
        y0, y1 = shard.slab_range(grid.ny, world, r)
        blk = ora.adjoint(osl, geom, y).reshape(grid.nz, y1 - y0, grid.nx)
        ref = full_adj.reshape(grid.nz, grid.ny, grid.nx)[:, y0:y1, :]
        np.testing.assert_allclose(blk, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_y_slab_split_and_assemble_round_trip(world):
    """distributed.y_slab / assemble_y_slabs (reference layout, x-fastest)."""
    from paper_2509_08574_b200 import distributed
    grid = k.GridSpec((5, 11, 4), (1.0, 1.0, 1.0))
    vol = np.arange(grid.count(), dtype=np.float32)
    parts = []
    for r in range(world):
        j0, j1 = shard.slab_range(grid.dims[1], world, r)
        sl = distributed.y_slab(vol, grid, j0, j1)
        assert sl.size == 5 * (j1 - j0) * 4
        parts.append(sl)
    np.testing.assert_array_equal(distributed.assemble_y_slabs(parts, grid), vol)
    sg = shard.slab_grid(grid, world, world - 1, axis="y")
    j0, j1 = shard.slab_range(grid.dims[1], world, world - 1)
    assert sg.dims == (5, j1 - j0, 4)
    assert sg.origin[1] == pytest.approx(grid.origin[1] + j0 * grid.spacing[1])


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_balanced_bounds(world):
    """shard.balanced_bounds: contiguous, covering, non-empty slabs on 4-plane
    boundaries, equal totals for uniform weights, thinner slabs where the
    weight is larger."""
    bounds = shard.balanced_bounds(np.ones(64), world)
    assert bounds[0] == 0 and bounds[-1] == 64 and len(bounds) == world + 1
    assert all(b1 > b0 for b0, b1 in zip(bounds, bounds[1:]))
    assert all(b % 4 == 0 for b in bounds)
    sizes = np.diff(bounds)
    assert sizes.max() - sizes.min() <= 4
    w = np.concatenate([np.ones(32), 3 * np.ones(32)])
    b2 = shard.balanced_bounds(w, 2)
    assert b2[1] > 32  # the heavy half gets the thinner slab


def test_slab_bounds_same_for_every_scan_of_a_system():
    """distributed.slab_bounds depends on the system (source, detector), not on
    the scan's angles: prior and follow-up projectors get the same y-slabs;
    the corners of a cube outside the field of view make the outer slabs
    thicker."""
    from paper_2509_08574_b200 import distributed, synth
    cfg = synth.CONFIGS["c3"]
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    g60 = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                             synth.angles(60))
    g360 = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                              synth.angles(360))
    b = distributed.slab_bounds(grid, g60, 8)
    assert b == distributed.slab_bounds(grid, g360, 8)
    sizes = np.diff(b)
    assert sizes[0] > sizes[3] and sizes[-1] > sizes[4]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("dims,nu,pu,off", [((64, 64, 8), 96, 1.0, 0.0), ((48, 80, 4), 40, 1.7, 3.0),
                                            ((256, 256, 4), 384, 0.5, 0.0), ((10, 9, 3), 12, 1.3, -0.4)])
def test_native_slab_bounds_match_python(world, dims, nu, pu, off):
    """kct_slab_bounds (the C++ host's slab split, include/kct.h) is the same
    function as distributed.slab_bounds."""
    import ctypes as C
    from paper_2509_08574_b200 import distributed
    sp = 1.0 if dims[0] != 256 else 0.5
    grid = k.GridSpec(dims, (sp, sp, sp))
    geom = k.ConeBeamGeometry(1000.0, 1500.0, nu, 16, pu, pu, k.uniform_angles(7), off, 0.0)
    want = distributed.slab_bounds(grid, geom, world)
    got = (C.c_int * (world + 1))()
    g, ge = grid._c(), geom._c()
    assert k.load_library().kct_slab_bounds(C.byref(g), C.byref(ge), world, got) == 0
    assert list(got) == list(want)


def test_native_slab_bounds_rejects_too_many_ranks():
    import ctypes as C
    grid = k.GridSpec((8, 4, 8))
    geom = k.ConeBeamGeometry(100.0, 150.0, 12, 12, 1.0, 1.0, k.uniform_angles(4))
    got = (C.c_int * 6)()
    g, ge = grid._c(), geom._c()
    assert k.load_library().kct_slab_bounds(C.byref(g), C.byref(ge), 5, got) == 2
