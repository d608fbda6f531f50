"""Profiling driver: c3 forward + adjoint on device-resident data (no timing).

    python tools/kprof.py [--cfg c3] [--reps 3]
Used under ncu (one GPU): ncu --set full -k regex:adj_brick -s 1 -c 1 python tools/kprof.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--views", type=int, default=0)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.cfg]
    na = a.views or cfg.followup_views
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                              synth.angles(na))
    A = k.ConeBeamProjector(grid, geom)
    _, prior, _ = synth.study(a.cfg)
    x = A.volume_to_native(torch.from_numpy(prior).cuda())
    q = torch.empty(geom.ray_count(), device="cuda")
    b = torch.empty(grid.count(), device="cuda")
    ev = []
    for _ in range(a.reps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        A.apply(x, out=q)
        e1.record()
        A.apply_adjoint(q, out=b)
        e2.record()
        ev.append((e0, e1, e2))
    torch.cuda.synchronize()
    for e0, e1, e2 in ev:
        print(f"fwd {e0.elapsed_time(e1):.3f} ms  adj {e1.elapsed_time(e2):.3f} ms")


if __name__ == "__main__":
    main()
