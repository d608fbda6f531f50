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


def _problem():
    grid, geom = Grid(12, 12, 10), recon_geometry(8)
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
