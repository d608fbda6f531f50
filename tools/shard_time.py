"""Per-rank operator time of the multi-GPU decompositions at c3, run on one
GPU rank by rank (no contention): angle-shard forward, z-slab and y-slab
adjoints.  python tools/shard_time.py [N ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import distributed, shard, synth  # noqa: E402


def t_op(fn, reps=3):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cfg = synth.CONFIGS["c3"]
grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                          synth.angles(cfg.followup_views))
y = torch.rand(geom.ray_count(), device="cuda")
x = torch.rand(grid.count(), device="cuda")
for N in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    tf, tz, ty, tfy, ta = [], [], [], [], []
    for r in range(N):
        Af = k.ConeBeamProjector(grid, shard.shard_geometry(geom, N, r))
        q = torch.empty(Af.range_size(), device="cuda")
        tf.append(t_op(lambda: Af.apply(x, out=q)))
        vb = torch.empty(Af.domain_size(), device="cuda")
        qa = torch.rand(Af.range_size(), device="cuda")
        ta.append(t_op(lambda: Af.apply_adjoint(qa, out=vb)))  # angle-sharded solver's adjoint
        del Af
        # y-slabs balanced by backprojection work (distributed.slab_bounds),
        # as the bench and the slab solver cut them
        yb = distributed.slab_bounds(grid, geom, N)
        for axis, acc in (("z", tz), ("y", ty)):
            g = shard.slab_grid(grid, N, r, axis, yb if axis == "y" else None)
            Ab = k.ConeBeamProjector(g, geom)
            b = torch.empty(Ab.domain_size(), device="cuda")
            acc.append(t_op(lambda: Ab.apply_adjoint(y, out=b)))
            if axis == "y":  # the slab solver's forward: this slab's share of every ray
                xs = torch.rand(Ab.domain_size(), device="cuda")
                qs = torch.empty(Ab.range_size(), device="cuda")
                tfy.append(t_op(lambda: Ab.apply(xs, out=qs)))
            del Ab
    print(f"N={N} fwd max {max(tf):.3f} ms | adj angle-shard max {max(ta):.3f} | adj z-slab max {max(tz):.3f} "
          f"[{' '.join(f'{t:.2f}' for t in tz)}] | adj y-slab max {max(ty):.3f} "
          f"[{' '.join(f'{t:.2f}' for t in ty)}] | fwd y-slab max {max(tfy):.3f}", flush=True)
