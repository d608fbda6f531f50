"""GPU parity of the CUDA projector pair against the reference / oracle.

Bar (BASELINE.json north_star): projections and backprojections within 1e-4
relative L2 of the float64 reference on identical float32 inputs.  Restates
proj/tests/test_projector.cpp properties (adjoint pair, exact transpose,
uniform-volume chords, bit-identical reruns, size checks) on the CUDA path.
"""
import numpy as np
import pytest
import torch

import paper_2509_08574_b200 as k
from oracle import Oracle
from tests._util import (baseline_geometry, geom_from, grid_from, load_golden, rel_l2,
                         tiny_geometry, tiny_grid, to_pkg)

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def ora():
    import oracle
    oracle.build("ora")
    return Oracle("ora")


def projector(grid, geom):
    gs, ge = to_pkg(grid, geom)
    return k.ConeBeamProjector(gs, ge)


@pytest.mark.parametrize("case", ["op_tiny", "op_tiny_odd", "op_c1_small"])
def test_golden_operator_parity(case):
    d = load_golden(case)
    A = projector(grid_from(d), geom_from(d))
    assert rel_l2(A.apply(d["x"]), d["ax"]) < TOL
    assert rel_l2(A.apply_adjoint(d["y"]), d["aty"]) < TOL
    assert rel_l2(A.apply(np.full(A.domain_size(), 2.5)), d["ax_uniform"]) < TOL
    # exact Siddon nnz, up to degenerate corner/edge segments whose length is
    # positive in float64 but rounds to zero in float32 (this case is full of
    # exact corner crossings: 4 mm voxels, 4 mm pitch, axis-aligned views)
    assert abs(A.count_nnz() - int(d["nnz"])) <= max(2, 1e-2 * int(d["nnz"]))


def test_uniform_volume_gives_chords(ora):
    """test_projector.cpp:54-69: A * 2.5 = 2.5 * chord per ray."""
    grid, geom = tiny_grid(6, 6, 6), tiny_geometry(4, 8, 8)
    A = projector(grid, geom)
    got = A.apply(np.full(grid.count, 2.5, dtype=np.float32))
    want = ora.forward(grid, geom, np.full(grid.count, 2.5))
    np.testing.assert_allclose(got, want, rtol=2e-6, atol=2e-6)


def test_exact_transpose_matricised():
    """test_projector.cpp:77-85 on the CUDA pair: dense A from apply() equals dense
    A^T from apply_adjoint() (float32 rounding), non-negative, non-trivial."""
    grid, geom = tiny_grid(), tiny_geometry(3, 6, 5)
    A = projector(grid, geom)
    m, n = grid.count, geom.ray_count
    fwd = np.stack([A.apply(np.eye(m, dtype=np.float32)[j]) for j in range(m)], axis=1)
    adj = np.stack([A.apply_adjoint(np.eye(n, dtype=np.float32)[i]) for i in range(n)], axis=0)
    assert np.abs(fwd - adj).max() <= 1e-6 * np.abs(fwd).max()
    assert fwd.min() >= 0 and fwd.max() > 0
    ref = Oracle("ora")
    dense_ref = np.stack([ref.forward(grid, geom, np.eye(m)[j]) for j in range(m)], axis=1)
    assert np.abs(fwd - dense_ref).max() <= 1e-5 * np.abs(dense_ref).max()
    assert np.array_equal(fwd > 0, adj > 0)


def test_adjoint_identity():
    """test_projector.cpp:71-75 (<Ax,y> = <x,A^T y>), float32 pair."""
    grid, geom = tiny_grid(5, 6, 4), tiny_geometry(7, 9, 8)
    A = projector(grid, geom)
    rng = np.random.default_rng(22)
    for _ in range(5):
        x = rng.uniform(-1, 1, grid.count).astype(np.float32)
        y = rng.uniform(-1, 1, geom.ray_count).astype(np.float32)
        lhs = np.dot(A.apply(x).astype(np.float64), y)
        rhs = np.dot(x.astype(np.float64), A.apply_adjoint(y))
        assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_bit_identical_reruns():
    """test_projector.cpp:100-111."""
    grid, geom = tiny_grid(6, 5, 6), tiny_geometry(5)
    A = projector(grid, geom)
    rng = np.random.default_rng(23)
    x = rng.uniform(-1, 1, grid.count).astype(np.float32)
    y = rng.uniform(-1, 1, geom.ray_count).astype(np.float32)
    ax, aty = A.apply(x), A.apply_adjoint(y)
    for _ in range(3):
        assert np.array_equal(A.apply(x), ax)
        assert np.array_equal(A.apply_adjoint(y), aty)


def test_size_mismatch():
    """test_projector.cpp:143-147."""
    A = projector(tiny_grid(), tiny_geometry(2))
    with pytest.raises(k.ConfigError):
        A.apply(np.zeros(A.domain_size() + 1, dtype=np.float32))


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 45), (3, 12), (4, 6), (5, 9)])
def test_baseline_geometry_parity(ora, cfg, n_angles):
    """Full-size BASELINE volumes/detectors, angle subsets the oracle finishes in seconds."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    rng = np.random.default_rng(cfg)
    # smooth-ish positive volume plus noise, like attenuation maps
    x = rng.uniform(0.0, 0.04, grid.count).astype(np.float32)
    A = projector(grid, geom)
    ax = A.apply(x)
    ref = ora.forward(grid, geom, x)
    assert rel_l2(ax, ref) < TOL
    y = rng.uniform(0.0, 1.0, geom.ray_count).astype(np.float32)
    assert rel_l2(A.apply_adjoint(y), ora.adjoint(grid, geom, y)) < TOL


def test_device_native_matches_host_reference():
    """Native-layout device tensors and reference-layout host arrays agree."""
    import torch
    grid, geom = baseline_geometry(1, n_angles=16)
    A = projector(grid, geom)
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, grid.count).astype(np.float32)
    host = A.apply(x)
    xd = torch.from_numpy(x).cuda()
    xn = A.volume_to_native(xd)
    yn = A.apply(xn)  # native in, native out
    yr = A.proj_from_native(yn)
    assert np.array_equal(yr.cpu().numpy(), host)
    yref_dev = A.apply(xd, layout="reference")
    assert np.array_equal(yref_dev.cpu().numpy(), host)
    back = A.apply_adjoint(yn)
    back_host = A.apply_adjoint(host)
    assert np.array_equal(A.volume_from_native(back).cpu().numpy(), back_host)


@pytest.mark.parametrize("cfg,n_angles", [(1, 8), (3, 2)])
def test_brick_and_gather_adjoints_agree(monkeypatch, cfg, n_angles):
    """The brick-owned transpose and the per-voxel gather compute the same
    segment lengths from the same crossing expressions."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    y = np.random.default_rng(9).uniform(0, 1, geom.ray_count).astype(np.float32)
    brick = projector(grid, geom).apply_adjoint(y)
    monkeypatch.setenv("KCT_ADJOINT", "gather")
    gather = projector(grid, geom).apply_adjoint(y)
    assert rel_l2(brick, gather) < 2e-6


@pytest.mark.parametrize("env", [{"KCT_ADJ_GROUPS": "1"}, {"KCT_ADJ_GROUPS": "5"},
                                 {"KCT_ADJ_SCHED": "static"}])
def test_adjoint_schedule_independent(monkeypatch, ora, env):
    """Angle groups (partial volumes summed in group order) and the brick
    queue change only the summation order: same result to rounding, each
    schedule bit-reproducible."""
    grid, geom = baseline_geometry(1, n_angles=64)
    y = np.random.default_rng(4).uniform(0, 1, geom.ray_count).astype(np.float32)
    A = projector(grid, geom)
    base = A.apply_adjoint(y)
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    B = projector(grid, geom)
    other = B.apply_adjoint(y)
    assert rel_l2(other, base) < 2e-6
    assert np.array_equal(B.apply_adjoint(y), other)
    assert rel_l2(other, ora.adjoint(grid, geom, y)) < TOL


def test_handles_with_different_bricks_coexist(ora):
    """Kernel attributes are per function: a handle created later with shorter
    bricks must not break an earlier handle with taller ones."""
    from tests._util import Grid
    geom = tiny_geometry(4, nu=12, nv=40)
    tall, short = Grid(8, 8, 192, 0.5, 0.5, 0.25), Grid(8, 8, 16, 0.5, 0.5, 0.25)
    A = projector(tall, geom)
    B = projector(short, geom)
    y = np.random.default_rng(5).uniform(0, 1, geom.ray_count).astype(np.float32)
    assert rel_l2(A.apply_adjoint(y), ora.adjoint(tall, geom, y)) < TOL
    assert rel_l2(B.apply_adjoint(y), ora.adjoint(short, geom, y)) < TOL


def test_host_pipeline_is_bitwise(monkeypatch):
    """kct_forward with host buffers runs in angle chunks whose projections
    leave the device while the next chunk is computed: same bits."""
    grid, geom = baseline_geometry(1, n_angles=64)
    x = np.random.default_rng(12).uniform(0, 0.04, grid.count).astype(np.float32)
    piped = projector(grid, geom).apply(x)
    monkeypatch.setenv("KCT_HOST_PIPELINE", "0")
    plain = projector(grid, geom).apply(x)
    assert np.array_equal(piped, plain)


def test_more_than_one_angle_batch(ora):
    """> 1024 angles: several launches accumulate (angle batches in param space)."""
    grid, geom = tiny_grid(6, 5, 6), tiny_geometry(1100)
    rng = np.random.default_rng(31)
    x = rng.uniform(0, 1, grid.count).astype(np.float32)
    y = rng.uniform(0, 1, geom.ray_count).astype(np.float32)
    A = projector(grid, geom)
    assert rel_l2(A.apply(x), ora.forward(grid, geom, x)) < TOL
    assert rel_l2(A.apply_adjoint(y), ora.adjoint(grid, geom, y)) < TOL


def test_sharded_operators_match_full():
    """Angle-shard forward and z- / y-slab adjoints (shard.py, the multi-GPU
    decomposition) reproduce the full operators on the CUDA path."""
    from paper_2509_08574_b200 import shard
    grid, geom = baseline_geometry(1, n_angles=12)
    gs, ge = to_pkg(grid, geom)
    full = k.ConeBeamProjector(gs, ge)
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    y = rng.uniform(0, 1, geom.ray_count).astype(np.float32)
    fwd = full.apply(x).reshape(geom.n_angles, -1)
    adj = full.apply_adjoint(y).reshape(grid.nz, -1)
    for world in (2, 3):
        for r in range(world):
            part = k.ConeBeamProjector(gs, shard.shard_geometry(ge, world, r)).apply(x)
            np.testing.assert_array_equal(part.reshape(-1, fwd.shape[1]),
                                          fwd[shard.angle_indices(geom.n_angles, world, r)])
            z0, z1 = shard.slab_range(grid.nz, world, r)
            blk = k.ConeBeamProjector(shard.slab_grid(gs, world, r), ge).apply_adjoint(y)
            assert rel_l2(blk, adj[z0:z1]) < 1e-6
            y0, y1 = shard.slab_range(grid.ny, world, r)
            blk = k.ConeBeamProjector(shard.slab_grid(gs, world, r, axis="y"), ge).apply_adjoint(y)
            ref = adj.reshape(grid.nz, grid.ny, grid.nx)[:, y0:y1, :]
            assert rel_l2(blk, ref) < 1e-6


def slab_geometry(n_angles=3, nu=12, nv=12):
    """A small geometry inside the slab-lane adjoint's validity range
    (projector.cu brick_rows_slab: z-span over a brick chord < row spacing)."""
    from tests._util import Geometry, Grid, uniform_angles
    return Grid(8, 8, 8, 1.0, 1.0, 1.0), Geometry(100.0, 150.0, nu, nv, 1.0, 1.0,
                                                  uniform_angles(n_angles))


def test_slab_adjoint_exact_transpose(monkeypatch):
    """test_projector.cpp:77-85 on the slab-lane adjoint path: dense A^T from
    apply_adjoint() equals the dense A from apply() (float32 rounding), same
    sparsity."""
    monkeypatch.setenv("KCT_ADJ_SLAB", "force")
    grid, geom = slab_geometry()
    A = projector(grid, geom)
    m, n = grid.count, geom.ray_count
    fwd = np.stack([A.apply(np.eye(m, dtype=np.float32)[j]) for j in range(m)], axis=1)
    adj = np.stack([A.apply_adjoint(np.eye(n, dtype=np.float32)[i]) for i in range(n)], axis=0)
    assert fwd.max() > 0
    assert np.abs(fwd - adj).max() <= 1e-6 * np.abs(fwd).max()
    assert np.array_equal(fwd > 0, adj > 0)


@pytest.mark.parametrize("cfg,n_angles", [(1, 16), (2, 6), (3, 3), (4, 1)])
def test_slab_and_row_adjoints_agree(monkeypatch, ora, cfg, n_angles):
    """The slab-lane deposits and the row-wise deposits compute the same piece
    lengths (summation order differs); both bit-reproducible; BASELINE
    geometries are inside the slab path's validity range."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    y = np.random.default_rng(31).uniform(0, 1, geom.ray_count).astype(np.float32)
    monkeypatch.setenv("KCT_ADJ_SLAB", "force")
    A = projector(grid, geom)
    slab = A.apply_adjoint(y)
    assert np.array_equal(A.apply_adjoint(y), slab)
    monkeypatch.setenv("KCT_ADJ_SLAB", "0")
    row = projector(grid, geom).apply_adjoint(y)
    assert rel_l2(slab, row) < 1e-6
    if cfg <= 2:
        assert rel_l2(slab, ora.adjoint(grid, geom, y)) < TOL


def test_split_upload_forward_is_bitwise(monkeypatch):
    """Host-buffer forward with the split volume upload (row band 0 runs while
    the upper slabs are uploaded): same bits as the plain path, also on a
    second call whose upper slabs differ from the first call's (band 0 never
    reads slabs that are not uploaded yet)."""
    grid, geom = baseline_geometry(3, n_angles=16)
    rng = np.random.default_rng(41)
    x1 = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    x2 = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    A = projector(grid, geom)
    A.apply(x1)
    split = A.apply(x2)
    monkeypatch.setenv("KCT_FWD_SPLIT", "0")
    monkeypatch.setenv("KCT_HOST_PIPELINE", "0")
    plain = projector(grid, geom).apply(x2)
    assert np.array_equal(split, plain)


def test_projector_info_reports_paths():
    """kct_projector_info: BASELINE c3 runs the slab-lane adjoint, z-mirror
    pairs (3 chunks of 32 row pairs per warp: 192 rows) and the split host
    upload of the central slabs; c1 (one row band) has no split; unknown keys
    are ConfigError."""
    A = projector(*baseline_geometry(3, n_angles=16))
    assert A.info("adj_slab") == 1 and A.info("adj_gather") == 0
    assert A.info("mirror") == 1
    # z-mirror brick pairs: lower bricks of 64 slabs tiling z < 0
    assert A.info("adj_mirror") == 1 and A.info("adj_bz") == 64
    assert A.info("fwd_rows_per_warp") == 192
    lo, hi = A.info("fwd_split_lo"), A.info("fwd_split_z")
    assert 0 < lo < 128 < hi < 256 and lo + hi == 256
    assert A.info("adj_walk_entries") > 0
    B = projector(*baseline_geometry(1, n_angles=8))
    assert B.info("adj_slab") == 1 and B.info("fwd_split_z") == 0
    with pytest.raises(k.ConfigError):
        A.info("no_such_key")


def test_host_adjoint_split_upload(monkeypatch):
    """kct_adjoint with host buffers (reference layouts) uploads the projections
    in two angle halves and accumulates the second half's launch onto the
    first: the device result to float rounding, bit-reproducible, and the
    unsplit host path agrees too."""
    import torch
    grid, geom = baseline_geometry(3, n_angles=16)
    A = projector(grid, geom)
    y = np.random.default_rng(43).uniform(0, 1, geom.ray_count).astype(np.float32)
    host = A.apply_adjoint(y)
    assert np.array_equal(A.apply_adjoint(y), host)
    yd = A.proj_to_native(torch.from_numpy(y).cuda())
    dev = A.volume_from_native(A.apply_adjoint(yd)).cpu().numpy()
    assert rel_l2(host, dev) < 1e-6
    monkeypatch.setenv("KCT_ADJ_SPLIT", "0")
    whole = projector(grid, geom).apply_adjoint(y)
    assert np.array_equal(whole, dev)


def test_slab_paths_awkward_geometry(monkeypatch, ora):
    """Slab-lane adjoint and padded forward on awkward sizes: partial bricks in
    x and y, an uneven z split, anisotropic voxels, detector offsets, a row
    count that is not a multiple of 32 and non-uniform angles — against the
    float64 oracle and (adjoint) the row-wise path."""
    from tests._util import Geometry, Grid
    grid = Grid(37, 29, 53, 0.9, 1.1, 1.3)
    angles = np.sort(np.random.default_rng(5).uniform(0, 2 * np.pi, 24))
    geom = Geometry(600.0, 900.0, 61, 75, 1.2, 1.25, angles, 0.7, -0.9)
    rng = np.random.default_rng(6)
    x = rng.uniform(0, 1, grid.count).astype(np.float32)
    y = rng.uniform(0, 1, geom.ray_count).astype(np.float32)
    monkeypatch.setenv("KCT_ADJ_SLAB", "force")
    A = projector(grid, geom)
    assert A.info("adj_slab") == 1
    slab = A.apply_adjoint(y)
    assert rel_l2(slab, ora.adjoint(grid, geom, y)) < TOL
    assert rel_l2(A.apply(x), ora.forward(grid, geom, x)) < TOL
    monkeypatch.setenv("KCT_ADJ_SLAB", "0")
    row = projector(grid, geom).apply_adjoint(y)
    assert rel_l2(slab, row) < 1e-6


def test_out_argument_validation():
    """Caller-supplied outputs must match what the C ABI writes:
    exact size, contiguous float32, same memory kind / device as the input."""
    import torch
    grid, geom = tiny_grid(), tiny_geometry(4)
    gs, ge = to_pkg(grid, geom)
    A = k.ConeBeamProjector(gs, ge)
    x = np.random.default_rng(0).uniform(0, 1, gs.count()).astype(np.float32)
    n = ge.ray_count()
    bad = [np.empty(n - 1, np.float32), np.empty(n, np.float64),
           np.empty(2 * n, np.float32)[::2], torch.empty(n, device="cuda")]
    for out in bad:
        with pytest.raises(k.ConfigError):
            A.apply(x, out=out)
    xd = torch.from_numpy(x).cuda()
    for out in (np.empty(n, np.float32), torch.empty(n, device="cuda", dtype=torch.float64),
                torch.empty(n + 1, device="cuda")):
        with pytest.raises(k.ConfigError):
            A.apply(xd, out=out)
    with pytest.raises(k.ConfigError):
        A.apply_adjoint(np.zeros(n, np.float32), out=np.empty(gs.count() - 1, np.float32))
    with pytest.raises(k.ConfigError):
        A.volume_to_native(xd, out=torch.empty(3, device="cuda"))
    good = np.empty(n, np.float32)
    assert A.apply(x, out=good) is good
    np.testing.assert_array_equal(good, A.apply(x))


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (3, 6), (4, 3)])
@pytest.mark.parametrize("how", ["KCT_ADJ_TABLE=0", "KCT_ADJ_TABLE_MB=1"])
def test_walk_table_fallback(monkeypatch, ora, cfg, n_angles, how):
    """Without the precomputed walk table (disabled, or over the memory budget)
    the adjoint recomputes the walks on the fly (standard bricks: the brick
    pairs stream the table): same parity bar, bit-identical to the standard
    bricks' table path (same walk, same deposits) and within float rounding of
    the brick-pair path."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    y = np.random.default_rng(41).uniform(0, 1, geom.ray_count).astype(np.float32)
    pairs = projector(grid, geom)
    assert pairs.info("adj_walk_entries") > 0 and pairs.info("adj_mirror") == 1
    monkeypatch.setenv("KCT_ADJ_MIRROR", "0")
    with_tab = projector(grid, geom)
    assert with_tab.info("adj_walk_entries") > 0 and with_tab.info("adj_mirror") == 0
    key, val = how.split("=")
    monkeypatch.setenv(key, val)
    monkeypatch.delenv("KCT_ADJ_MIRROR")
    A = projector(grid, geom)
    assert A.info("adj_walk_entries") == 0 and A.info("adj_mirror") == 0
    got = A.apply_adjoint(y)
    assert np.array_equal(got, A.apply_adjoint(y))
    assert np.array_equal(got, with_tab.apply_adjoint(y))
    assert rel_l2(got, pairs.apply_adjoint(y)) < 1e-6
    assert rel_l2(got, ora.adjoint(grid, geom, y)) < TOL


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 8), (3, 4), (4, 2)])
def test_count_nnz_matches_reference(ora, cfg, n_angles):
    """nnz (the roofline's unit) equals the reference traverse_ray's count of
    positive-length segments up to degenerate segments: at the axis-aligned
    views (multiples of 90 degrees) rays run inside voxel planes / through
    voxel edges and the float64 walk produces segments shorter than 1e-6 mm
    (0.38% of the segments of a c2 view at 0 degrees, 1e-5 at 45 degrees,
    oracle trace) that the float32 walk gets as exactly 0.  They carry no
    weight, so the byte model is unaffected (measured: c1 64 views -2.0e-4,
    c2 8 views -1.5e-3); bar 5e-3 of nnz."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    got, want = projector(grid, geom).count_nnz(), ora.count_nnz(grid, geom)
    print(f"\n[nnz c{cfg}/{n_angles} views] gpu {got} reference {want} "
          f"diff {got - want} ({(got - want) / want:.2e})")
    assert abs(got - want) <= max(2, 5e-3 * want)


@pytest.mark.parametrize("n_angles", [8])
def test_c4_slot_conflict_path(ora, n_angles):
    """c4's row spacing can reach one slab, so the adjoint's slot-conflict
    detection is on (adj_slab_detect) — checked against the oracle over several
    views, not one."""
    grid, geom = baseline_geometry(4, n_angles=n_angles)
    y = np.random.default_rng(43).uniform(0, 1, geom.ray_count).astype(np.float32)
    # (brick pairs have no conflicts: primary and mirror rows fill separate
    # bricks; the standard bricks detect them)
    pairs = projector(grid, geom)
    assert pairs.info("adj_mirror") == 1
    assert rel_l2(pairs.apply_adjoint(y), ora.adjoint(grid, geom, y)) < TOL
    import os
    os.environ["KCT_ADJ_MIRROR"] = "0"
    try:
        A = projector(grid, geom)
    finally:
        del os.environ["KCT_ADJ_MIRROR"]
    assert A.info("adj_slab") == 1 and A.info("adj_slab_detect") == 1
    assert rel_l2(A.apply_adjoint(y), ora.adjoint(grid, geom, y)) < TOL


def mirror_geometry(n_angles=5, nu=7, nv=6):
    """z-symmetric tiny geometry: offset_v = 0, nv even, grid centred in z."""
    from oracle import Geometry, uniform_angles
    return Geometry(40.0, 90.0, nu, nv, 1.6, 1.9, uniform_angles(n_angles) + 0.1, 0.7, 0.0)


def test_mirror_pairs_exact_transpose():
    """With z-mirror pairs (fwd_kernel MIR: rows iv / nv-1-iv share one z
    state; the adjoint's per-ray records encode the mirror's) the dense A from
    apply() still equals the dense A^T from apply_adjoint(), same sparsity."""
    grid, geom = tiny_grid(4, 5, 6), mirror_geometry()
    A = projector(grid, geom)
    assert A.info("mirror") == 1
    m, n = grid.count, geom.ray_count
    fwd = np.stack([A.apply(np.eye(m, dtype=np.float32)[j]) for j in range(m)], axis=1)
    adj = np.stack([A.apply_adjoint(np.eye(n, dtype=np.float32)[i]) for i in range(n)], axis=0)
    assert fwd.max() > 0
    assert np.abs(fwd - adj).max() <= 1e-6 * np.abs(fwd).max()
    assert np.array_equal(fwd > 0, adj > 0)
    # the mirror row of every ray carries the primary's lengths, reflected
    fw = fwd.reshape(geom.n_angles, geom.nv, geom.nu, grid.nz, grid.ny, grid.nx)
    np.testing.assert_array_equal(fw, fw[:, ::-1, :, ::-1, :, :])


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 9), (3, 6), (4, 3)])
def test_mirror_pairs_match_unpaired(monkeypatch, ora, cfg, n_angles):
    """Mirror pairs on (BASELINE geometries are z-symmetric) and off
    (KCT_MIRROR=0): both within the parity bar of the oracle and within
    float rounding of each other."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    rng = np.random.default_rng(53)
    x = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    y = rng.uniform(0, 1, geom.ray_count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("mirror") == 1
    monkeypatch.setenv("KCT_MIRROR", "0")
    B = projector(grid, geom)
    assert B.info("mirror") == 0
    ax, bx = A.apply(x), B.apply(x)
    aty, bty = A.apply_adjoint(y), B.apply_adjoint(y)
    assert rel_l2(ax, bx) < 1e-6 and rel_l2(aty, bty) < 1e-6
    assert rel_l2(ax, ora.forward(grid, geom, x)) < TOL
    assert rel_l2(aty, ora.adjoint(grid, geom, y)) < TOL
    assert abs(A.count_nnz() - B.count_nnz()) <= max(2, 1e-4 * B.count_nnz())


def test_mirror_brick_pairs_exact_transpose(monkeypatch):
    """test_projector.cpp:77-85 on the z-mirror brick-pair adjoint
    (adj_mirror_kernel: one classification of the primary rows feeds both
    bricks of a pair): dense A^T equals dense A, same sparsity, and the mirror
    rows carry the primary's lengths reflected."""
    monkeypatch.setenv("KCT_ADJ_SLAB", "force")
    grid, geom = slab_geometry(n_angles=4)
    A = projector(grid, geom)
    assert A.info("mirror") == 1 and A.info("adj_mirror") == 1
    m, n = grid.count, geom.ray_count
    fwd = np.stack([A.apply(np.eye(m, dtype=np.float32)[j]) for j in range(m)], axis=1)
    adj = np.stack([A.apply_adjoint(np.eye(n, dtype=np.float32)[i]) for i in range(n)], axis=0)
    assert fwd.max() > 0
    assert np.abs(fwd - adj).max() <= 1e-6 * np.abs(fwd).max()
    assert np.array_equal(fwd > 0, adj > 0)
    aw = adj.reshape(geom.n_angles, geom.nv, geom.nu, grid.nz, grid.ny, grid.nx)
    np.testing.assert_array_equal(aw, aw[:, ::-1, :, ::-1, :, :])


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 9), (3, 6), (4, 2), (5, 5)])
@pytest.mark.parametrize("bz", ["64", "43", "128"])
def test_mirror_brick_pairs_match_standard_bricks(monkeypatch, ora, cfg, n_angles, bz):
    """Brick pairs (default) against the standard bricks (KCT_ADJ_MIRROR=0) and
    the oracle, at the default and other pair heights (KCT_ADJ_MIR_BZ: 43 ->
    uneven splits, 128 -> four slab chunks); bit-reproducible."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    y = np.random.default_rng(61).uniform(0, 1, geom.ray_count).astype(np.float32)
    monkeypatch.setenv("KCT_ADJ_MIR_BZ", bz)
    A = projector(grid, geom)
    assert A.info("adj_mirror") == 1
    assert A.info("adj_bz") == -(-(grid.nz // 2) // -(-(grid.nz // 2) // int(bz)))
    got = A.apply_adjoint(y)
    assert np.array_equal(got, A.apply_adjoint(y))
    monkeypatch.setenv("KCT_ADJ_MIRROR", "0")
    std = projector(grid, geom).apply_adjoint(y)
    assert rel_l2(got, std) < 1e-6
    if bz == "64":
        assert rel_l2(got, ora.adjoint(grid, geom, y)) < TOL


def test_mirror_brick_pairs_host_and_groups(monkeypatch):
    """The brick pairs' host path (reference layout written by the kernel, z
    levels copied out pairwise) and angle groups give the device result."""
    import torch
    grid, geom = baseline_geometry(3, n_angles=16)
    A = projector(grid, geom)
    assert A.info("adj_mirror") == 1
    y = np.random.default_rng(71).uniform(0, 1, geom.ray_count).astype(np.float32)
    host = A.apply_adjoint(y)
    yd = A.proj_to_native(torch.from_numpy(y).cuda())
    dev = A.volume_from_native(A.apply_adjoint(yd)).cpu().numpy()
    assert rel_l2(host, dev) < 1e-6
    monkeypatch.setenv("KCT_ADJ_GROUPS", "3")
    B = projector(grid, geom)
    assert B.info("adj_groups") == 3
    assert rel_l2(B.apply_adjoint(y), dev) < 1e-6


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 9), (3, 6), (4, 2)])
def test_warp_specialised_pairs_bitwise(monkeypatch, cfg, n_angles):
    """adj_mirror_ws_kernel (producer warp classifies, consumer warp deposits,
    named-barrier handshakes) computes exactly what the one-warp brick-pair
    kernel computes (KCT_ADJ_WS=0): same bits, also on the host path."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    y = np.random.default_rng(81).uniform(0, 1, geom.ray_count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("adj_mirror") == 1 and A.info("adj_ws") == 1
    ws = A.apply_adjoint(y)
    # 2 or 3 producer warps per consumer (picked by timing at creation;
    # forced here): the same entries in the same order, bit-identical
    assert A.info("adj_np") in (2, 3)
    for np_forced in ("2", "3"):
        monkeypatch.setenv("KCT_ADJ_NP", np_forced)
        C = projector(grid, geom)
        assert C.info("adj_np") == int(np_forced)
        assert np.array_equal(ws, C.apply_adjoint(y))
        x_dev = C.apply_adjoint(torch.from_numpy(C.proj_to_native(y) if False else y).cuda(),
                                layout="reference")
        assert np.array_equal(ws, x_dev.cpu().numpy())
    monkeypatch.delenv("KCT_ADJ_NP")
    monkeypatch.setenv("KCT_ADJ_WS", "0")
    B = projector(grid, geom)
    assert B.info("adj_ws") == 0 and B.info("adj_np") == 0
    assert np.array_equal(ws, B.apply_adjoint(y))


def test_mirror_pairs_awkward_geometry(monkeypatch, ora):
    """Brick pairs on awkward sizes: partial 5x5 bricks in x and y, a lower
    half (27 slabs) that is an odd brick height, anisotropic voxels, a detector
    u offset and non-uniform angles (z-mirror: offset_v = 0, nv even) —
    against the oracle, the standard bricks and the one-warp pair kernel."""
    from tests._util import Geometry, Grid
    grid = Grid(37, 29, 54, 0.9, 1.1, 1.3)
    angles = np.sort(np.random.default_rng(7).uniform(0, 2 * np.pi, 24))
    geom = Geometry(600.0, 900.0, 61, 76, 1.2, 1.25, angles, 0.7, 0.0)
    y = np.random.default_rng(8).uniform(0, 1, geom.ray_count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("adj_mirror") == 1 and A.info("adj_ws") == 1 and A.info("adj_bz") == 27
    ws = A.apply_adjoint(y)
    assert rel_l2(ws, ora.adjoint(grid, geom, y)) < TOL
    monkeypatch.setenv("KCT_ADJ_WS", "0")
    assert np.array_equal(projector(grid, geom).apply_adjoint(y), ws)
    monkeypatch.setenv("KCT_ADJ_MIRROR", "0")
    assert rel_l2(projector(grid, geom).apply_adjoint(y), ws) < 1e-6


@pytest.mark.parametrize("parts", ["1", "3", "16"])
def test_host_adjoint_progress_parts(monkeypatch, parts):
    """The host-buffer adjoint copies (z level, y part) blocks out as soon as
    their bricks are final (strided copies of brick rows): any part count
    gives the device result's bits."""
    import torch
    grid, geom = baseline_geometry(3, n_angles=16)
    y = np.random.default_rng(47).uniform(0, 1, geom.ray_count).astype(np.float32)
    monkeypatch.setenv("KCT_ADJ_PARTS", parts)
    A = projector(grid, geom)
    host = A.apply_adjoint(y)
    yd = A.proj_to_native(torch.from_numpy(y).cuda())
    dev = A.volume_from_native(A.apply_adjoint(yd)).cpu().numpy()
    assert rel_l2(host, dev) < 1e-6
    monkeypatch.setenv("KCT_ADJ_SPLIT", "0")
    assert np.array_equal(projector(grid, geom).apply_adjoint(y), dev)


@pytest.mark.parametrize("cfg,n_angles", [(3, 60), (4, 24), (2, 45)])
def test_staged_host_forward_is_bitwise(monkeypatch, cfg, n_angles):
    """kct_forward with host buffers uploads the volume in stage ranges (centre
    out) and runs each row stage once its slabs are in: same bits as the
    device-resident forward, also on a second call whose outer slabs differ
    from the first call's (no stage reads slabs not uploaded yet), and as the
    two-band split path (KCT_FWD_STAGED=0)."""
    import torch
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    rng = np.random.default_rng(51)
    x1 = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    x2 = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("fwd_stages") >= 2
    A.apply(x1)
    staged = A.apply(x2)
    dev = A.proj_from_native(A.apply(A.volume_to_native(torch.from_numpy(x2).cuda()))).cpu().numpy()
    assert np.array_equal(staged, dev)
    # native-layout stages + transpose kernels on the copy stream
    monkeypatch.setenv("KCT_FWD_REFOUT", "0")
    assert np.array_equal(projector(grid, geom).apply(x2), staged)
    monkeypatch.delenv("KCT_FWD_REFOUT")
    # every stage's rows streaming out as the stage ends (opt-in), other stage sizes
    monkeypatch.setenv("KCT_FWD_ROWSTAGES", "1")
    assert np.array_equal(projector(grid, geom).apply(x2), staged)
    for sizes in ("1,1,1,1,1,1", "2,1,3", "1,4"):
        monkeypatch.setenv("KCT_FWD_STAGE_SIZES", sizes)
        assert np.array_equal(projector(grid, geom).apply(x2), staged), sizes
    monkeypatch.delenv("KCT_FWD_ROWSTAGES")
    assert np.array_equal(projector(grid, geom).apply(x2), staged)
    monkeypatch.delenv("KCT_FWD_STAGE_SIZES")
    monkeypatch.setenv("KCT_FWD_STAGED", "0")
    B = projector(grid, geom)
    assert B.info("fwd_stages") == 0
    assert np.array_equal(B.apply(x2), staged)


def test_staged_host_forward_without_mirror_symmetry(monkeypatch):
    """A detector offset in v breaks the z-mirror symmetry: the staged host
    forward then walks single rows (one row band per stage) — same bits as the
    device-resident forward."""
    import torch
    from oracle import Geometry, Grid, uniform_angles
    grid = Grid(128, 128, 128, 0.8, 0.8, 0.8)
    geom = Geometry(1000.0, 1500.0, 192, 200, 0.8, 0.8, uniform_angles(24), 0.0, 3.3)
    gs, ge = to_pkg(grid, geom)
    x = np.random.default_rng(52).uniform(0, 0.04, grid.count).astype(np.float32)
    for rowstages in ("0", "1"):
        monkeypatch.setenv("KCT_FWD_ROWSTAGES", rowstages)
        A = k.ConeBeamProjector(gs, ge)
        assert A.info("mirror") == 0
        host = A.apply(x)
        dev = A.proj_from_native(A.apply(A.volume_to_native(torch.from_numpy(x).cuda()))).cpu().numpy()
        assert np.array_equal(host, dev)


@pytest.mark.parametrize("cfg,n_angles", [(1, 64), (2, 9), (3, 6), (4, 2), (5, 5)])
def test_forward_walk_table_bitwise(monkeypatch, cfg, n_angles):
    """The forward's xy walks from the precomputed walk table (fwd_tab_build:
    the same xy_walk, stored) give the on-the-fly walk's bits
    (KCT_FWD_TABLE=0), device-resident and through the host pipeline."""
    grid, geom = baseline_geometry(cfg, n_angles=n_angles)
    x = np.random.default_rng(57).uniform(0, 0.04, grid.count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("fwd_table_segments") > 0
    tab = A.apply(x)
    monkeypatch.setenv("KCT_FWD_TABLE", "0")
    B = projector(grid, geom)
    assert B.info("fwd_table_segments") == 0
    assert np.array_equal(B.apply(x), tab)


def test_forward_walk_table_awkward(monkeypatch, ora):
    """Walk table on the awkward geometry (partial columns, offsets, odd sizes,
    a non-mirror detector): oracle parity and the on-the-fly walk's bits."""
    from tests._util import Geometry, Grid
    grid = Grid(37, 29, 53, 0.9, 1.1, 1.3)
    angles = np.sort(np.random.default_rng(5).uniform(0, 2 * np.pi, 24))
    geom = Geometry(600.0, 900.0, 61, 75, 1.2, 1.25, angles, 0.7, -0.9)
    x = np.random.default_rng(6).uniform(0, 1, grid.count).astype(np.float32)
    A = projector(grid, geom)
    assert A.info("fwd_table_segments") > 0
    tab = A.apply(x)
    assert rel_l2(tab, ora.forward(grid, geom, x)) < TOL
    monkeypatch.setenv("KCT_FWD_TABLE", "0")
    assert np.array_equal(projector(grid, geom).apply(x), tab)
