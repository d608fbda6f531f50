"""Where the host-buffer (e2e) step's time goes at c3: kct_forward and
kct_adjoint with pinned host buffers in the reference layouts, the same
operators device-resident, and plain pinned copies of the step's buffers.
Median of --reps after one warm-up; wall clock around each synchronous call.

    python tools/e2e_time.py [--cfg c3] [--reps 10]
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


def med(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return round(1e3 * float(np.median(ts)), 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.cfg]
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                              synth.angles(cfg.followup_views))
    A = k.ConeBeamProjector(grid, geom)
    dev = torch.device("cuda", 0)
    _, prior, _ = synth.study(a.cfg)
    M, N = grid.count(), geom.ray_count()
    vol_h = torch.from_numpy(prior).pin_memory()
    proj_h = torch.empty(N).pin_memory()
    back_h = torch.empty(M).pin_memory()
    y_h = torch.rand(N).pin_memory()
    vol_d = torch.empty(M, device=dev)
    proj_d = torch.empty(N, device=dev)
    x = A.volume_to_native(vol_h.to(dev))
    yd = A.proj_to_native(y_h.to(dev))
    out = {"cfg": a.cfg, "M_bytes": 4 * M, "N_bytes": 4 * N}
    out["fwd_host_ms"] = med(lambda: A.apply(vol_h.numpy(), out=proj_h.numpy()), a.reps)
    out["adj_host_ms"] = med(lambda: A.apply_adjoint(y_h.numpy(), out=back_h.numpy()), a.reps)
    out["fwd_dev_ms"] = med(lambda: A.apply(x), a.reps)
    out["adj_dev_ms"] = med(lambda: A.apply_adjoint(yd), a.reps)
    out["h2d_vol_ms"] = med(lambda: vol_d.copy_(vol_h, non_blocking=True), a.reps)
    out["d2h_vol_ms"] = med(lambda: back_h.copy_(vol_d, non_blocking=True), a.reps)
    out["h2d_proj_ms"] = med(lambda: proj_d.copy_(y_h, non_blocking=True), a.reps)
    out["d2h_proj_ms"] = med(lambda: proj_h.copy_(proj_d, non_blocking=True), a.reps)
    for key in ("h2d_vol", "d2h_vol"):
        out[key + "_gbs"] = round(4 * M / out[key + "_ms"] / 1e6, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
