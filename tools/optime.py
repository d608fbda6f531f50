"""Operator timing on device-resident data: forward / adjoint kernel ms,
GUPS and the fraction of the HBM roofline (SURVEY §8d byte model), median of
--reps launches with an L2 flush before each (CUDA events).

    python tools/optime.py --cfg c3 [--reps 10] [--views 60]
Environment switches of the library (KCT_MIRROR=0, KCT_FWD_C=..., ...) apply.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import synth  # noqa: E402

PEAK = 6542.7


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--views", type=int, default=0)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.cfg]
    na = a.views or cfg.followup_views
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                              synth.angles(na))
    A = k.ConeBeamProjector(grid, geom)
    dev = torch.device("cuda", 0)
    _, prior, _ = synth.study(a.cfg)
    x = A.volume_to_native(torch.from_numpy(prior).to(dev))
    y = torch.rand(geom.ray_count(), device=dev, generator=torch.Generator(dev).manual_seed(7))
    q = torch.empty(geom.ray_count(), device=dev)
    v = torch.empty(grid.count(), device=dev)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    nnz = A.count_nnz()
    M, N = grid.count(), geom.ray_count()
    res = {}
    for name, fn in (("forward", lambda: A.apply(x, out=q)), ("adjoint", lambda: A.apply_adjoint(y, out=v))):
        fn()
        ts = []
        for r in range(a.reps):
            flush.fill_(float(r))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        byts = 4.0 * nnz + 4.0 * (N if name == "forward" else M)
        res[name] = {"ms": round(ms, 4), "gups": round(M * na / ms / 1e6, 1),
                     "frac": round(byts / (ms * 1e-3) / 1e9 / PEAK, 4)}
    res["fwd+adj GUPS"] = round(2 * M * na / (res["forward"]["ms"] + res["adjoint"]["ms"]) / 1e6, 1)
    res["cfg"] = a.cfg
    res["views"] = na
    res["mirror"] = A.info("mirror")
    res["tag"] = a.tag
    res["checksum"] = [float(q.double().sum()), float(v.double().sum())]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
