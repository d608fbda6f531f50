"""One warm 20-iteration IRN-PICCS at c3 on device-resident data (for ncu launch
lists and host-overhead checks).  python tools/recon_prof.py [--reps 2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import synth  # noqa: E402

reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 2
cfg = synth.CONFIGS["c3"]
grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                          synth.angles(cfg.followup_views))
A = k.ConeBeamProjector(grid, geom)
_, prior, follow = synth.study("c3")
xf = A.volume_to_native(torch.from_numpy(follow).cuda())
b = A.apply(xf)
pr = A.volume_to_native(torch.from_numpy(prior).cuda())
params = k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner)
proj = k.ProjectionSet(geom, b)
for i in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = k.irn_piccs(proj, grid, pr, params, projector=A)
    torch.cuda.synchronize()
    print(f"recon {time.perf_counter() - t:.4f} s  solve_seconds {rep.solve_seconds:.4f}", flush=True)
