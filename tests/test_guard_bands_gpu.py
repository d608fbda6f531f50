"""GPU: guard bands around every caller buffer.  Inputs and outputs are views
into larger allocations whose margins hold a canary pattern; after the
operator, FDK and solver calls (device-native and device-reference layouts,
awkward sizes that are no multiple of any tile) the margins must be untouched
and the inputs unchanged — an out-of-bounds store of a kernel into a caller
buffer's neighbourhood shows up here (compute-sanitizer is not available on
this GPU pool)."""
import numpy as np
import pytest
import torch

import paper_2509_08574_b200 as k
from tests._util import to_pkg
from oracle import Geometry, Grid, uniform_angles

pytestmark = pytest.mark.gpu
PAD = 4096  # floats on each side
CANARY = -12345.678


class Banded:
    """`n` floats in the middle of a canary-filled allocation."""

    def __init__(self, n, fill=None):
        self.buf = torch.full((n + 2 * PAD,), CANARY, dtype=torch.float32, device="cuda")
        self.view = self.buf[PAD:PAD + n]
        if fill is not None:
            self.view.copy_(fill)
        else:
            self.view.zero_()

    def intact(self):
        torch.cuda.synchronize()
        return bool((self.buf[:PAD] == CANARY).all()) and bool((self.buf[-PAD:] == CANARY).all())


@pytest.mark.parametrize("dims,nu,nv,na", [((37, 29, 41), 53, 47, 5), ((64, 64, 64), 96, 96, 6),
                                           ((20, 24, 132), 40, 150, 3)])
@pytest.mark.parametrize("layout", ["native", "reference"])
def test_guard_bands(dims, nu, nv, na, layout):
    grid = Grid(*dims, 1.0, 1.1, 0.9)
    geom = Geometry(400.0, 600.0, nu, nv, 1.3, 1.2, uniform_angles(na))
    gs, ge = to_pkg(grid, geom)
    A = k.ConeBeamProjector(gs, ge)
    m, n = A.domain_size(), A.range_size()
    g = torch.Generator(device="cuda").manual_seed(3)
    x = Banded(m, torch.rand(m, device="cuda", generator=g) * 0.03)
    y = Banded(n, torch.rand(n, device="cuda", generator=g))
    x_keep, y_keep = x.view.clone(), y.view.clone()
    ax, aty, rec = Banded(n), Banded(m), Banded(m)
    A.apply(x.view, out=ax.view, layout=layout)
    A.apply_adjoint(y.view, out=aty.view, layout=layout)
    A.fdk(y.view, out=rec.view, layout=layout)
    for b in (x, y, ax, aty, rec):
        assert b.intact()
    assert torch.equal(x.view, x_keep) and torch.equal(y.view, y_keep)
    assert float(ax.view.abs().sum()) > 0 and float(aty.view.abs().sum()) > 0
    # solvers: b, prior, x0, ground truth in; volume out
    params = k.RegularizationParams(alpha=0.3, outer_iters=2, inner_iters=2)
    out = Banded(m)
    prior = Banded(m, x.view * 0.9)
    rep = k.irn_piccs(k.ProjectionSet(ge, ax.view), gs, prior.view, params,
                      k.ReconOptions(initial=prior.view, ground_truth=x.view), projector=A,
                      layout=layout, out=out.view)
    assert np.all(np.isfinite(rep.residual_history))
    out2 = Banded(m)
    k.cgls_recon(k.ProjectionSet(ge, ax.view), gs, 3, projector=A, layout=layout, out=out2.view)
    for b in (x, ax, prior, out, out2):
        assert b.intact()
    assert torch.equal(x.view, x_keep)
