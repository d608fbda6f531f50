"""Where the reconstruction error of a BASELINE config comes from (c4 shows
0.52 relative error vs the follow-up phantom, c3 0.12): the prior CGLS
alone, the follow-up solve with the computed prior vs a perfect prior, and
more iterations.  Prints one JSON line per variant.

    python tools/convergence_diag.py --cfg c4
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


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c4")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.cfg]
    dev = torch.device("cuda", 0)
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    geom_p = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                                synth.angles(cfg.prior_views))
    geom_f = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                                synth.angles(cfg.followup_views))
    _, prior, follow = synth.study(a.cfg)
    Ap = k.ConeBeamProjector(grid, geom_p)
    bp = Ap.apply(Ap.volume_to_native(torch.from_numpy(prior).to(dev)))
    out = {"cfg": a.cfg}
    priors = {}
    for it in (20, 60):
        t0 = time.perf_counter()
        rep = k.cgls_recon(k.ProjectionSet(geom_p, bp), grid, it, projector=Ap)
        torch.cuda.synchronize()
        x = Ap.volume_from_native(rep.volume).cpu().numpy()
        priors[it] = x
        out[f"prior_cgls{it}_rel_err"] = round(rel(x, prior), 4)
        out[f"prior_cgls{it}_s"] = round(time.perf_counter() - t0, 2)
    del Ap, bp
    torch.cuda.empty_cache()
    Af = k.ConeBeamProjector(grid, geom_f)
    pf = Af.proj_from_native(Af.apply(Af.volume_to_native(torch.from_numpy(follow).to(dev))))
    b = synth.poisson_log(pf.cpu().numpy(), cfg.i0, seed=synth.noise_seed(a.cfg))
    b_n = Af.proj_to_native(torch.from_numpy(b).to(dev))
    proj = k.ProjectionSet(geom_f, b_n)
    gt = Af.volume_to_native(torch.from_numpy(follow).to(dev))
    out["followup_vs_prior_phantom_rel"] = round(rel(follow, prior), 4)
    runs = [("cgls20 prior", priors[20], cfg.outer, cfg.inner),
            ("cgls60 prior", priors[60], cfg.outer, cfg.inner),
            ("perfect prior", prior, cfg.outer, cfg.inner),
            ("cgls20 prior, 4x iterations", priors[20], 4 * cfg.outer, cfg.inner)]
    for name, pr, outer, inner in runs:
        pn = Af.volume_to_native(torch.from_numpy(np.ascontiguousarray(pr)).to(dev))
        rep = k.irn_piccs(proj, grid, pn, k.RegularizationParams(alpha=cfg.alpha,
                                                                 outer_iters=outer,
                                                                 inner_iters=inner),
                          k.ReconOptions(ground_truth=gt), projector=Af)
        eh = rep.error_history
        out[f"piccs[{name}] {outer}x{inner}"] = {
            "rel_err_final": round(float(eh[-1]), 4),
            "rel_err_per_cycle": [round(float(eh[i - 1]), 4) for i in rep.outer_boundaries],
            "objective": [float(f"{v:.6e}") for v in rep.objective_history]}
    # the regulariser weight and the noise: alpha sweep and a noiseless scan
    pn = Af.volume_to_native(torch.from_numpy(np.ascontiguousarray(priors[20])).to(dev))
    for alpha in (2.0, 8.0):
        rep = k.irn_piccs(proj, grid, pn, k.RegularizationParams(alpha=alpha, outer_iters=cfg.outer,
                                                                 inner_iters=cfg.inner),
                          k.ReconOptions(ground_truth=gt), projector=Af)
        out[f"piccs alpha={alpha}"] = round(float(rep.error_history[-1]), 4)
    proj0 = k.ProjectionSet(geom_f, Af.proj_to_native(pf))
    rep = k.irn_piccs(proj0, grid, pn, k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer,
                                                              inner_iters=cfg.inner),
                      k.ReconOptions(ground_truth=gt), projector=Af)
    out["piccs noiseless scan"] = round(float(rep.error_history[-1]), 4)
    # plain CGLS of the follow-up (no prior) for scale
    rep = k.cgls_recon(proj, grid, cfg.outer * cfg.inner, k.ReconOptions(ground_truth=gt),
                       projector=Af)
    out["followup_cgls_rel_err"] = round(float(rep.error_history[-1]), 4)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
