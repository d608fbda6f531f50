"""GPU: the angle-sharded multi-process solver (distributed.py + the C ABI
all-reduce hook).  One GPU here: world_size 1 must be bit-identical to the
single-process solve; two ranks sharing cuda:0 over gloo must reproduce the
single-process solve up to the rounding of the partial-volume sums."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2509_08574_b200 as k
from oracle import Grid
from tests._util import recon_geometry, rel_l2, to_pkg

pytestmark = pytest.mark.gpu


def _problem(nz=10):
    grid, geom = Grid(12, 12, nz), recon_geometry(8)
    gs, ge = to_pkg(grid, geom)
    rng = np.random.default_rng(21)
    prior = rng.uniform(0, 1, grid.count).astype(np.float32)
    truth = prior.copy()
    truth[300:360] += 0.5
    b = k.ConeBeamProjector(gs, ge).apply(truth)
    return gs, ge, prior, b


PARAMS = dict(alpha=0.3, outer_iters=2, inner_iters=3, tau=1e-3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    import torch.distributed as dist
    from paper_2509_08574_b200 import distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gs, ge, prior, b = _problem()
    local = distributed.shard_projections(k.ProjectionSet(ge, b), world, rank)
    rep = distributed.irn_piccs_sharded(local, gs, prior, k.RegularizationParams(**PARAMS))
    q.put((rank, np.asarray(rep.volume), rep.objective_history, rep.residual_history))
    dist.barrier()
    dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get() for _ in range(world)]
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_world1_is_bitwise_single_process():
    gs, ge, prior, b = _problem()
    ref = k.irn_piccs(k.ProjectionSet(ge, b), gs, prior, k.RegularizationParams(**PARAMS))
    (_, x, obj, res), = _run(1)
    assert np.array_equal(x, ref.volume)
    np.testing.assert_array_equal(obj, ref.objective_history)


def test_two_ranks_match_single_process():
    gs, ge, prior, b = _problem()
    ref = k.irn_piccs(k.ProjectionSet(ge, b), gs, prior, k.RegularizationParams(**PARAMS))
    outs = _run(2)
    for _, x, obj, res in outs:
        assert rel_l2(x, ref.volume) < 1e-5
        np.testing.assert_allclose(obj, ref.objective_history, rtol=1e-5)
        np.testing.assert_allclose(res, ref.residual_history, rtol=1e-5)
    assert np.array_equal(outs[0][1], outs[1][1])  # replicated state stays identical


# ---- y-slab-sharded solver (kct_set_slab) ------------------------------------
def _rank_slab(rank, world, port, q, fn, nz, params):
    import torch.distributed as dist
    from paper_2509_08574_b200 import distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gs, ge, prior, b = _problem(nz)
    proj = k.ProjectionSet(ge, b)
    truth = prior.copy()
    truth[300:360] += 0.5
    opts = k.ReconOptions(ground_truth=truth)
    if fn == "piccs":
        rep = distributed.irn_piccs_slab(proj, gs, prior, k.RegularizationParams(**params), opts)
    elif fn == "tv":
        rep = distributed.irn_tv_slab(proj, gs, k.RegularizationParams(**params), opts)
    else:
        rep = distributed.cgls_recon_slab(proj, gs, 6, opts)
    q.put((rank, np.asarray(rep.volume), rep.objective_history, rep.residual_history,
           rep.error_history, rep.tau))
    dist.barrier()
    dist.destroy_process_group()


def _run_slab(world, fn, nz=10, params=PARAMS):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_slab, args=(r, world, port, q, fn, nz, params))
          for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get() for _ in range(world)]
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fn", ["piccs", "tv", "cgls"])
def test_y_slab_ranks_match_single_process(world, fn):
    """Volume vectors split in y-slabs with halo planes: the assembled slabs
    and every history match the single-process solve (partial sums only)."""
    from paper_2509_08574_b200 import distributed
    gs, ge, prior, b = _problem()
    proj = k.ProjectionSet(ge, b)
    truth = prior.copy()
    truth[300:360] += 0.5
    opts = k.ReconOptions(ground_truth=truth)
    if fn == "piccs":
        ref = k.irn_piccs(proj, gs, prior, k.RegularizationParams(**PARAMS), opts)
    elif fn == "tv":
        ref = k.irn_tv(proj, gs, k.RegularizationParams(**PARAMS), opts)
    else:
        ref = k.cgls_recon(proj, gs, 6, opts)
    outs = _run_slab(world, fn)
    x = distributed.assemble_y_slabs([o[1] for o in outs], gs)
    assert rel_l2(x, ref.volume) < 1e-5
    for _, _, obj, res, err, tau in outs:
        np.testing.assert_allclose(obj, ref.objective_history, rtol=1e-5)
        np.testing.assert_allclose(res, ref.residual_history, rtol=1e-5)
        np.testing.assert_allclose(err, ref.error_history, rtol=1e-5)


@pytest.mark.parametrize("nz", [8, 10])
def test_y_slab_auto_tau_and_float4_stencils(nz):
    """tau from the prior's global range (gather over the slabs) and, at
    nz % 4 == 0, the float4 stencil kernels with halo planes."""
    from paper_2509_08574_b200 import distributed
    gs, ge, prior, b = _problem(nz)
    params = dict(PARAMS, tau=0.0)
    truth = prior.copy()
    truth[300:360] += 0.5
    ref = k.irn_piccs(k.ProjectionSet(ge, b), gs, prior, k.RegularizationParams(**params),
                      k.ReconOptions(ground_truth=truth))
    outs = _run_slab(2, "piccs", nz, params)
    x = distributed.assemble_y_slabs([o[1] for o in outs], gs)
    assert rel_l2(x, ref.volume) < 1e-5
    for _, _, obj, res, err, tau in outs:
        assert tau == pytest.approx(ref.tau, rel=1e-12)
        np.testing.assert_allclose(obj, ref.objective_history, rtol=1e-5)


# ---- collectives per CGLS iteration (two scalar all-reduces) -------
def _rank_count(rank, world, port, q, mode):
    import torch.distributed as dist
    from paper_2509_08574_b200 import distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = {"scalar": 0, "vector": 0, "p2p": 0}
    real_ar, real_p2p = dist.all_reduce, dist.batch_isend_irecv

    def counting_ar(t, *a, **kw):
        calls["scalar" if t.dtype == torch.float64 and t.numel() <= 8 else "vector"] += 1
        return real_ar(t, *a, **kw)

    def counting_p2p(ops):
        calls["p2p"] += 1
        return real_p2p(ops)
    dist.all_reduce, dist.batch_isend_irecv = counting_ar, counting_p2p
    gs, ge, prior, b = _problem()
    proj = k.ProjectionSet(ge, b)
    res = []
    for inner in (2, 5):
        for key in calls:
            calls[key] = 0
        params = k.RegularizationParams(alpha=0.3, outer_iters=1, inner_iters=inner, tau=1e-3)
        if mode == "slab":
            distributed.irn_piccs_slab(proj, gs, prior, params)
        else:
            local = distributed.shard_projections(proj, world, rank)
            distributed.irn_piccs_sharded(local, gs, prior, params)
        res.append(dict(calls))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["slab", "angles"])
def test_collectives_per_iteration(mode):
    """Per CGLS iteration: 2 packed fp64 scalar all-reduces (||A p||^2 and the
    regulariser norms; ||s||^2, ||r||^2 and the error norm), 1 vector
    all-reduce (slab: partial projections; angles: the partial A^T volume) and,
    in slab mode, 2 neighbour halo exchanges (x and p)."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_count, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get() for _ in range(2)]
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    for _, (c2, c5) in out:
        per = {key: (c5[key] - c2[key]) / 3 for key in c2}
        assert per["scalar"] == 2, per
        assert per["vector"] == 1, per
        assert per["p2p"] == (2 if mode == "slab" else 0), per


# ---- the library's own NCCL communicator (kct_comm_*, ABI 4) -----------------
def _native_rank(q, mode):
    """One rank on cuda:0 with a real NCCL communicator of world size 1 (more
    ranks need more GPUs: NCCL refuses two ranks on one device)."""
    from paper_2509_08574_b200 import distributed
    torch.cuda.set_device(0)
    out = {}
    if mode == "torch":  # bootstrap over torch.distributed's nccl backend
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1)
        comm = distributed.native_comm()
        assert comm is not None and (comm.rank, comm.world) == (0, 1)
    else:  # no torch.distributed at all: explicit id
        comm = distributed.NativeComm(0, 1, distributed.NativeComm.unique_id())
    t = torch.arange(5, dtype=torch.float64, device="cuda")
    comm.all_reduce(t, "sum")
    comm.all_reduce(t, "max")
    f = torch.full((7,), 2.5, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(torch.cuda.Stream()):  # a non-default current stream
        comm.all_reduce(f)
        torch.cuda.current_stream().synchronize()
    out["reduce"] = (t.cpu().numpy(), f.cpu().numpy())
    gs, ge, prior, b = _problem(8)
    proj = k.ProjectionSet(ge, b)
    params = k.RegularizationParams(**dict(PARAMS, tau=0.0))
    ref = k.irn_piccs(proj, gs, prior, params)
    # y-slab mode: the whole volume is rank 0's slab
    A = k.ConeBeamProjector(gs, ge)
    distributed.install_slab(A, 0, 1, 0, gs.dims[1], comm=comm)
    n0 = k.launch_count()
    rep = k.irn_piccs(proj, gs, prior, params, projector=A)
    out["slab"] = (bool(np.array_equal(rep.volume, ref.volume)),
                   bool(np.array_equal(rep.objective_history, ref.objective_history)),
                   bool(rep.tau == ref.tau),
                   k.launch_count() - n0)
    # angle-sharded mode
    A2 = k.ConeBeamProjector(gs, ge)
    distributed.install_allreduce(A2, comm=comm)
    rep2 = k.irn_piccs(proj, gs, prior, params, projector=A2)
    out["angles"] = (bool(np.array_equal(rep2.volume, ref.volume)),
                     bool(np.array_equal(rep2.residual_history, ref.residual_history)))
    if mode == "torch":  # the public entry picks the native communicator by itself
        rep3 = distributed.irn_piccs_slab(proj, gs, prior, params)
        out["auto"] = bool(np.array_equal(rep3.volume, ref.volume))
        import torch.distributed as dist
        dist.destroy_process_group()
    comm.close()
    q.put(out)


@pytest.mark.parametrize("mode", ["explicit", "torch"])
def test_native_nccl_comm_world1(mode):
    """kct_comm_* with NCCL itself (run-time bound): sums and maxima on the
    caller's stream, and slab / angle-sharded solves through the native hooks
    bit-identical to the single-process solve at world size 1."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    p = ctx.Process(target=_native_rank, args=(q, mode))
    p.start()
    while q.empty() and p.is_alive():  # a crashed rank must fail the test, not hang it
        p.join(0.2)
    assert not q.empty(), f"rank exited with {p.exitcode}"
    out = q.get()
    p.join(300)
    assert p.exitcode == 0
    t, f = out["reduce"]
    np.testing.assert_array_equal(t, np.arange(5.0))
    np.testing.assert_array_equal(f, np.full(7, 2.5, np.float32))
    assert out["slab"][:3] == (True, True, True) and out["slab"][3] > 0, out["slab"]
    assert out["angles"] == (True, True), out["angles"]
    if mode == "torch":
        assert out["auto"]


def test_native_comm_argument_errors():
    """ConfigError before any NCCL work: bad rank / world, null id, null handle."""
    import ctypes as C
    lib = k.load_library()
    h = C.c_void_p()
    buf = C.create_string_buffer(128)
    assert lib.kct_comm_create(2, 2, buf, -1, C.byref(h)) == 2
    assert lib.kct_comm_create(0, 0, buf, -1, C.byref(h)) == 2
    assert lib.kct_comm_create(0, 1, None, -1, C.byref(h)) == 2
    assert lib.kct_comm_allreduce(None, None, 0, 0, 0, None) == 2
    assert lib.kct_comm_rank(None) == -1 and lib.kct_comm_world(None) == 0
    gs, ge, prior, b = _problem(8)
    A = k.ConeBeamProjector(gs, ge)
    assert lib.kct_use_comm(A.handle, None) == 0  # NULL: back to single-process
