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
