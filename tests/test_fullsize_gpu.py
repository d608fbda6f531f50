"""GPU: size-independent properties of A / A^T at the FULL BASELINE sizes
(every view of c2 / c3 / c4), where the CPU oracle is too slow to run:

  * A 1 = the analytic chord of every ray through the volume box (slab clip
    of projector.hpp:70-82 evaluated in float64 numpy) — the row sums of A;
  * sum(A 1) = sum(A^T 1) (both are the sum of all matrix entries: a checksum
    of checksums), non-negativity;
  * <A x, y> = <x, A^T y> (test_projector.cpp:71-75) with float64 dot products;
  * linearity A (a x1 + b x2) = a A x1 + b A x2.
Together with the exact-transpose and oracle parity tests on angle subsets
(test_projector_gpu.py) these pin the operator pair at the sizes the bench runs.
"""
import numpy as np
import pytest
import torch

import paper_2509_08574_b200 as k
from tests._util import baseline_geometry, to_pkg

pytestmark = pytest.mark.gpu


def box_chords(grid, geom):
    """Length of every ray's intersection with the volume box, float64,
    reference order iu + nu * (iv + nv * ia) (source_position /
    detector_pixel_center: projector.hpp:24-39; slab clip :70-82)."""
    ang = np.asarray(geom.angles, dtype=np.float64)
    c, s = np.cos(ang)[:, None, None], np.sin(ang)[:, None, None]
    du = ((np.arange(geom.nu) + 0.5 - geom.nu / 2.0) * geom.pu + geom.offset_u)[None, None, :]
    dv = ((np.arange(geom.nv) + 0.5 - geom.nv / 2.0) * geom.pv + geom.offset_v)[None, :, None]
    src = [geom.dso * c, geom.dso * s, np.zeros_like(c)]
    back = -(geom.dsd - geom.dso)
    dst = [back * c - du * s, back * s + du * c, dv + 0.0 * c]
    lo = [grid.ox, grid.oy, grid.oz]
    hi = [grid.ox + grid.nx * grid.sx, grid.oy + grid.ny * grid.sy, grid.oz + grid.nz * grid.sz]
    shape = (len(ang), geom.nv, geom.nu)
    t0, t1 = np.zeros(shape), np.ones(shape)
    length2 = np.zeros(shape)
    for a in range(3):
        d = np.broadcast_to(dst[a] - src[a], shape)
        length2 = length2 + d * d
        with np.errstate(divide="ignore", invalid="ignore"):
            ta = (lo[a] - src[a]) / d
            tb = (hi[a] - src[a]) / d
        par = d == 0
        inside = np.broadcast_to((src[a] >= lo[a]) & (src[a] <= hi[a]), shape)
        tmin = np.where(par, np.where(inside, -np.inf, np.inf), np.minimum(ta, tb))
        tmax = np.where(par, np.where(inside, np.inf, -np.inf), np.maximum(ta, tb))
        t0, t1 = np.maximum(t0, tmin), np.minimum(t1, tmax)
    return (np.clip(t1 - t0, 0.0, None) * np.sqrt(length2)).reshape(-1)


def dot64(a, b):
    return float(torch.dot(a.double(), b.double()))


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_full_size_operator_properties(cfg):
    grid, geom = baseline_geometry(cfg)  # every view of the follow-up scan
    gs, ge = to_pkg(grid, geom)
    A = k.ConeBeamProjector(gs, ge)
    m, n = A.domain_size(), A.range_size()
    dev = torch.device("cuda")
    ones_v = torch.ones(m, dtype=torch.float32, device=dev)
    ones_p = torch.ones(n, dtype=torch.float32, device=dev)
    # row sums of A: the box chord of every ray
    a1 = A.apply(ones_v)  # native layouts throughout (device-resident calls)
    chords = box_chords(grid, geom)
    got = A.proj_from_native(a1).cpu().numpy().astype(np.float64)
    err = np.linalg.norm(got - chords) / np.linalg.norm(chords)
    worst = np.abs(got - chords).max()
    print(f"c{cfg}: ||A 1 - chords|| / ||chords|| = {err:.2e}, max abs {worst:.2e} mm")
    assert err < 1e-5  # float32 sums of up to ~500 segments; the bar is 1e-4
    # worst rays: near-axis-aligned views, where up to 512 equal float32
    # addends round the same way (systematic, <= 0.5 ulp of the running sum each)
    assert worst < 1e-5 * chords.max()
    assert np.array_equal(got > 0, chords > 1e-4 * grid.sx) or \
        np.mean((got > 0) != (chords > 0)) < 1e-5  # grazing rays only
    # column sums, and the checksum of checksums
    at1 = A.apply_adjoint(ones_p)
    assert float(a1.min()) >= 0.0 and float(at1.min()) >= 0.0
    total_f, total_b = float(a1.double().sum()), float(at1.double().sum())
    print(f"c{cfg}: sum(A 1) = {total_f:.9e}, sum(A^T 1) = {total_b:.9e}")
    assert abs(total_f - total_b) <= 1e-5 * total_f
    assert abs(total_f - float(chords.sum())) <= 1e-5 * total_f
    # adjoint identity with float64 dot products
    g = torch.Generator(device=dev).manual_seed(cfg)
    x = torch.rand(m, dtype=torch.float32, device=dev, generator=g) * 0.04
    y = torch.rand(n, dtype=torch.float32, device=dev, generator=g)
    ax, aty = A.apply(x), A.apply_adjoint(y)
    lhs, rhs = dot64(ax, y), dot64(x, aty)
    print(f"c{cfg}: <Ax,y> = {lhs:.9e}, <x,A^T y> = {rhs:.9e}")
    assert abs(lhs - rhs) <= 1e-6 * abs(lhs)
    # linearity
    x2 = torch.rand(m, dtype=torch.float32, device=dev, generator=g) * 0.04
    lin = A.apply(0.75 * x + 2.0 * x2)
    ref = 0.75 * ax.double() + 2.0 * A.apply(x2).double()
    rel = float((lin.double() - ref).norm() / ref.norm())
    assert rel < 1e-5
    # bit-identical reruns at full size (no atomics on the data path)
    assert torch.equal(A.apply(x), ax) and torch.equal(A.apply_adjoint(y), aty)
