"""BASELINE config c5: 256^3 @0.5 mm, 384^2 @0.5 mm, one 360-view prior,
8 follow-ups x 45 views, needle tip advancing 5 mm per follow-up, Poisson
I0 = 1e5, 15 PICCS iterations (3x5) per follow-up warm-started from the
previous result.  Prints one JSON line: seconds per follow-up (device
resident) and the end-to-end total.

    python tools/c5_sequence.py [--followups 8]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/c5_sequence.py          # N GPUs: y-slab-sharded prior CGLS and
                                      # follow-up solves (distributed.py),
                                      # times = max over ranks
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
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev_i = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    shared = ws > torch.cuda.device_count()
    if ws > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def rmax(v):
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def rsum(vals):
        if ws == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else dev)
        torch.distributed.all_reduce(t)
        return t.tolist()

    def sync():
        torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()

    cfg = synth.CONFIGS["c5"]
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    mk = lambda n: k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch,  # noqa: E731
                                      cfg.pitch, synth.angles(n))
    gp, gf = mk(cfg.prior_views), mk(cfg.followup_views)
    Ap, Af = k.ConeBeamProjector(grid, gp), k.ConeBeamProjector(grid, gf)
    if ws > 1:
        from paper_2509_08574_b200 import distributed
        Ap_s, j0, j1 = distributed.slab_projector(grid, gp, ws, rank)
        Af_s, _, _ = distributed.slab_projector(grid, gf, ws, rank)
    else:
        Ap_s, Af_s, j0, j1 = Ap, Af, 0, grid.dims[1]
    table = synth.draw_ellipsoids(cfg, 5)
    prior_img = synth.render(cfg, table)
    tip, d = synth.needle_pose(cfg, 5 + 700)
    sync()
    t0 = time.perf_counter()
    bp = Ap.apply(Ap.volume_to_native(torch.from_numpy(prior_img).to(dev)))
    prior = k.cgls_recon(k.ProjectionSet(gp, bp), Ap_s.grid, 20, projector=Ap_s).volume
    sync()
    t_prior = rmax(time.perf_counter() - t0)
    scans, truths = [], []
    for t in range(a.followups):
        img = synth.add_cylinder(cfg, prior_img, tip + 5.0 * t * d, d, 60.0, 1.0, 0.2)
        p = Af.proj_from_native(Af.apply(Af.volume_to_native(torch.from_numpy(img).to(dev))))
        b = synth.poisson_log(p.cpu().numpy(), cfg.i0, seed=2000 + t)
        scans.append(Af.proj_to_native(torch.from_numpy(b).to(dev)))
        truths.append(img.reshape(cfg.n, cfg.n, cfg.n)[:, j0:j1, :].reshape(-1))  # y-slab
    params = k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner)
    repeated_scan(Af_s, scans[:1], prior, params)  # warm-up (allocation, clocks)
    sync()
    t0 = time.perf_counter()
    reps, secs = repeated_scan(Af_s, scans, prior, params)
    sync()
    total = rmax(time.perf_counter() - t0)
    secs = [rmax(s) for s in secs]
    errs = []
    for r, g in zip(reps, truths):
        x = Af_s.volume_from_native(r.volume).cpu().numpy().astype(np.float64)
        e2, g2 = rsum([float(np.sum((x - g) ** 2)), float(np.sum(g.astype(np.float64) ** 2))])
        errs.append(float(np.sqrt(e2 / g2)))
    if rank == 0:
        print(json.dumps({"workload": "c5: 256^3, 384^2, 360-view prior, followups x 45 views, "
                                      "15 PICCS iterations each (3x5) warm-started",
                          "n_gpus": ws,
                          "parallelism": "y-slab-sharded state" if ws > 1 else "single GPU",
                          **({"shared_devices": "functional check: more ranks than GPUs"}
                             if shared else {}),
                          "followups": a.followups,
                          "seconds_per_followup": [round(s, 4) for s in secs],
                          "mean_seconds_per_followup": round(float(np.mean(secs)), 4),
                          "median_seconds_per_followup": round(float(np.median(secs)), 4),
                          "total_seconds": round(total, 3), "prior_cgls_seconds": round(t_prior, 3),
                          "rel_error_vs_phantom": [round(e, 4) for e in errs],
                          "taus": [r.tau for r in reps]}), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
