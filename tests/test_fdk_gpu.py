"""GPU parity of the FDK reconstruction (fdk.hpp:50-139)
against the reference's own output (golden) and the oracle at c1 geometry."""
import numpy as np
import pytest

import paper_2509_08574_b200 as k
from oracle import Oracle
from tests._util import baseline_geometry, geom_from, grid_from, load_golden, rel_l2, to_pkg

pytestmark = pytest.mark.gpu


def test_fdk_golden():
    d = load_golden("fdk_small")
    gs, ge = to_pkg(grid_from(d), geom_from(d))
    vol = k.fdk(k.ProjectionSet(ge, d["proj"]), gs)
    assert rel_l2(vol, d["fdk"]) < 1e-4


def test_fdk_c1_vs_oracle():
    import oracle
    oracle.build("ora")
    ora = Oracle("ora")
    grid, geom = baseline_geometry(1)
    gs, ge = to_pkg(grid, geom)
    rng = np.random.default_rng(8)
    x = rng.uniform(0, 0.04, grid.count).astype(np.float32)
    A = k.ConeBeamProjector(gs, ge)
    p = A.apply(x)
    assert rel_l2(A.fdk(p), ora.fdk(grid, geom, p)) < 1e-4


def test_fdk_needs_two_angles():
    grid, geom = baseline_geometry(1, n_angles=1)
    gs, ge = to_pkg(grid, geom)
    with pytest.raises(k.ConfigError):
        k.ConeBeamProjector(gs, ge).fdk(np.zeros(ge.ray_count(), dtype=np.float32))


@pytest.mark.parametrize("nu", [1024, 2048, 4100])
def test_fdk_wide_detector(nu):
    """detectors wider than one 32-row shared-memory tile (33 nu
    floats > 227 KB from nu ~ 1760) filter with fewer rows per CTA; same
    result as the oracle on projections of a random volume (nu = 1024: the
    32-row path on the same kind of data)."""
    import oracle
    from oracle import Geometry, Grid, uniform_angles
    oracle.build("ora")
    ora = Oracle("ora")
    grid = Grid(48, 48, 8, 1.0, 1.0, 1.0)
    geom = Geometry(1000.0, 1500.0, nu, 12, 100.0 / nu, 1.0, uniform_angles(16))
    gs, ge = to_pkg(grid, geom)
    A = k.ConeBeamProjector(gs, ge)
    x = np.random.default_rng(9).uniform(0, 0.04, gs.count()).astype(np.float32)
    p = A.apply(x)
    err = rel_l2(A.fdk(p), ora.fdk(grid, geom, p))
    print(f"\n[fdk nu={nu}] rel err {err:.2e}")
    assert err < 1e-4
