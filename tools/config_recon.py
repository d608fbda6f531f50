"""A BASELINE config end to end on the device: prior (20-iteration CGLS of the
noiseless prior scan), follow-up scan with Poisson noise, then the config's
PICCS (c2-c4) or CGLS (c1) solve.  Prints one JSON line with the timings.

    python tools/config_recon.py --cfg c4
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/config_recon.py --cfg c4    # y-slab-sharded solves, max over ranks
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c4")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev_i = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    shared = ws > torch.cuda.device_count()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if shared else "nccl", **({} if shared else {"device_id": dev}))

    def sync():
        torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()

    def red(vals, op):
        if ws == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else dev)
        torch.distributed.all_reduce(t, op=op)
        return t.tolist()

    cfg, prior_img, follow = synth.study(a.cfg)
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    mk = lambda n: k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch,  # noqa: E731
                                      cfg.pitch, synth.angles(n))
    gp, gf = mk(cfg.prior_views), mk(cfg.followup_views)
    t0 = time.perf_counter()
    Ap, Af = k.ConeBeamProjector(grid, gp), k.ConeBeamProjector(grid, gf)
    if ws > 1:
        from paper_2509_08574_b200 import distributed
        Ap_s, j0, j1 = distributed.slab_projector(grid, gp, ws, rank)
        Af_s, _, _ = distributed.slab_projector(grid, gf, ws, rank)
    else:
        Ap_s, Af_s, j0, j1 = Ap, Af, 0, cfg.n
    sync()
    t_setup = time.perf_counter() - t0
    # prior: 20-iteration CGLS of the noiseless prior scan
    bp = Ap.apply(Ap.volume_to_native(torch.from_numpy(prior_img).to(dev)))
    sync()
    t0 = time.perf_counter()
    prior_rep = k.cgls_recon(k.ProjectionSet(gp, bp), Ap_s.grid, 20, projector=Ap_s)
    sync()
    t_prior = time.perf_counter() - t0
    del bp
    pf = Af.proj_from_native(Af.apply(Af.volume_to_native(torch.from_numpy(follow).to(dev))))
    b = synth.poisson_log(pf.cpu().numpy(), cfg.i0, seed=1000 + int(a.cfg[1])) if cfg.i0 else \
        pf.cpu().numpy()
    proj = k.ProjectionSet(gf, Af.proj_to_native(torch.from_numpy(b).to(dev)))
    truth = follow.reshape(cfg.n, cfg.n, cfg.n)[:, j0:j1, :].reshape(-1)
    times = []
    for _ in range(a.reps + 1):
        sync()
        t0 = time.perf_counter()
        if a.cfg == "c1":
            rep = k.cgls_recon(proj, Af_s.grid, cfg.iters, projector=Af_s)
        else:
            params = k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer,
                                            inner_iters=cfg.inner)
            rep = k.irn_piccs(proj, Af_s.grid, prior_rep.volume, params, projector=Af_s)
        sync()
        times.append(time.perf_counter() - t0)
    x = Af_s.volume_from_native(rep.volume).cpu().numpy().astype(np.float64)
    e2, g2 = red([float(np.sum((x - truth) ** 2)), float(np.sum(truth.astype(np.float64) ** 2))],
                 torch.distributed.ReduceOp.SUM if ws > 1 else None)
    t_solve = red([float(np.median(times[1:]))], torch.distributed.ReduceOp.MAX if ws > 1 else None)[0]
    t_prior = red([t_prior], torch.distributed.ReduceOp.MAX if ws > 1 else None)[0]
    if rank == 0:
        print(json.dumps({
            "cfg": a.cfg, "n_gpus": ws,
            "parallelism": "y-slab-sharded state" if ws > 1 else "single GPU",
            **({"shared_devices": "functional check: more ranks than GPUs"} if shared else {}),
            "volume": f"{cfg.n}^3 @ {cfg.voxel} mm", "detector": f"{cfg.det}^2 @ {cfg.pitch} mm",
            "prior_views": cfg.prior_views, "followup_views": cfg.followup_views,
            "solve": "cgls" if a.cfg == "c1" else f"irn_piccs {cfg.outer}x{cfg.inner}",
            "solve_seconds": round(t_solve, 4), "prior_cgls20_seconds": round(t_prior, 3),
            "setup_seconds": round(t_setup, 3),
            "rel_error_vs_followup_phantom": round(float(np.sqrt(e2 / g2)), 5),
            "objective_history": [float(v) for v in rep.objective_history]}), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
