"""Time FDK at a BASELINE config (device-resident projections).  python tools/fdk_time.py [c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_08574_b200 as k  # noqa: E402
from paper_2509_08574_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
geom = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                          synth.angles(cfg.followup_views))
A = k.ConeBeamProjector(grid, geom)
q = torch.rand(geom.ray_count(), device="cuda")
out = torch.empty(grid.count(), device="cuda")
A.fdk(q, out=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    A.fdk(q, out=out)
e1.record()
torch.cuda.synchronize()
print(f"fdk {e0.elapsed_time(e1) / 5:.3f} ms")
