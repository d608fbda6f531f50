"""GPU: the repeated-scan driver (c5 semantics) against a chain of reference
IRN-PICCS calls warm-started with the previous result (oracle)."""
import numpy as np
import pytest

import paper_2509_08574_b200 as k
from oracle import KIND_PICCS, Grid, Oracle
from paper_2509_08574_b200.sequence import repeated_scan
from tests._util import recon_geometry, rel_l2, to_pkg

pytestmark = pytest.mark.gpu


def test_repeated_scan_matches_warm_started_reference_chain():
    import oracle
    oracle.build("ora")
    ora = Oracle("ora")
    grid, geom = Grid(10, 10, 8), recon_geometry(8)
    gs, ge = to_pkg(grid, geom)
    rng = np.random.default_rng(5)
    prior = rng.uniform(0, 1, grid.count).astype(np.float32)
    A = k.ConeBeamProjector(gs, ge)
    scans, truths = [], []
    for t in range(3):
        truth = prior.copy()
        truth[100 + 30 * t: 140 + 30 * t] += 0.5
        truths.append(truth)
        scans.append(A.apply(truth))
    params = k.RegularizationParams(alpha=0.3, outer_iters=2, inner_iters=3)
    reps, secs = repeated_scan(A, scans, prior, params)
    assert len(secs) == 3 and all(s > 0 for s in secs)
    x = None
    for t in range(3):
        x, r = ora.irn(grid, geom, KIND_PICCS, scans[t].astype(np.float64), prior,
                       dict(alpha=0.3, outer_iters=2, inner_iters=3), x0=x)
        assert rel_l2(reps[t].volume, x) < 1e-3
        # tau comes from the (slightly different) previous iterate: not bitwise
        assert reps[t].tau == pytest.approx(r["tau"], rel=1e-4)
