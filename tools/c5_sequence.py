"""BASELINE config c5 on one GPU: 256^3 @0.5 mm, 384^2 @0.5 mm, one 360-view
prior, 8 follow-ups x 45 views, needle tip advancing 5 mm per follow-up,
Poisson I0 = 1e5, 15 PICCS iterations (3x5) per follow-up warm-started from
the previous result.  Prints one JSON line: seconds per follow-up (device
resident) and the end-to-end total.

    python tools/c5_sequence.py [--followups 8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import synth  # noqa: E402
from paper_2509_08574_b200.sequence import repeated_scan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--followups", type=int, default=8)
    a = ap.parse_args()
    cfg = synth.CONFIGS["c5"]
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    mk = lambda n: k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch,  # noqa: E731
                                      cfg.pitch, synth.angles(n))
    Ap, Af = k.ConeBeamProjector(grid, mk(cfg.prior_views)), k.ConeBeamProjector(grid, mk(cfg.followup_views))
    table = synth.draw_ellipsoids(cfg, 5)
    prior_img = synth.render(cfg, table)
    tip, d = synth.needle_pose(cfg, 5 + 700)
    t0 = time.perf_counter()
    bp = Ap.apply(Ap.volume_to_native(torch.from_numpy(prior_img).cuda()))
    prior = k.cgls_recon(k.ProjectionSet(Ap.geometry, bp), grid, 20, projector=Ap).volume
    t_prior = time.perf_counter() - t0
    scans, truths = [], []
    for t in range(a.followups):
        img = synth.add_cylinder(cfg, prior_img, tip + 5.0 * t * d, d, 60.0, 1.0, 0.2)
        p = Af.proj_from_native(Af.apply(Af.volume_to_native(torch.from_numpy(img).cuda())))
        b = synth.poisson_log(p.cpu().numpy(), cfg.i0, seed=2000 + t)
        scans.append(Af.proj_to_native(torch.from_numpy(b).cuda()))
        truths.append(img)
    params = k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner)
    repeated_scan(Af, scans[:1], prior, params)  # warm-up (allocation, clocks)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps, secs = repeated_scan(Af, scans, prior, params)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    errs = [float(np.linalg.norm(Af.volume_from_native(r.volume).cpu().numpy() - g) /
                  np.linalg.norm(g)) for r, g in zip(reps, truths)]
    print(json.dumps({"workload": "c5: 256^3, 384^2, 360-view prior, followups x 45 views, 15 "
                                  "PICCS iterations each (3x5) warm-started",
                      "followups": a.followups, "seconds_per_followup": [round(s, 4) for s in secs],
                      "mean_seconds_per_followup": round(float(np.mean(secs)), 4),
                      "total_seconds": round(total, 3), "prior_cgls_seconds": round(t_prior, 3),
                      "rel_error_vs_phantom": [round(e, 4) for e in errs],
                      "taus": [r.tau for r in reps]}))


if __name__ == "__main__":
    main()
