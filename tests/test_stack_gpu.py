"""GPU parity of the device-resident generic CGLS over caller-assembled stacks
(kct_cgls_stack: krylov.hpp:59-127 on linear_map.hpp:159-216 StackedMaps).

Bar as for the drivers: iterates within 1e-3 relative L2 of the float64
reference (measured 1e-6..1e-5).  Golden vectors come from the reference's own
kryct::cgls on kryct::StackedMap (tests/golden/make_golden.py stack_case).
"""
import numpy as np
import pytest

import paper_2509_08574_b200 as k
from oracle import Oracle
from tests._util import baseline_geometry, geom_from, grid_from, load_golden, rel_l2, to_pkg

pytestmark = pytest.mark.gpu
RTOL = 1e-3


@pytest.fixture(scope="module")
def ora():
    import oracle
    oracle.build("ora")
    return Oracle("ora")


@pytest.fixture(scope="module")
def small():
    d = load_golden("stack_small")
    gs, ge = to_pkg(grid_from(d), geom_from(d))
    return d, gs, ge, k.ConeBeamProjector(gs, ge)


def _stacks(d, A, conv=lambda a: a):
    D = k.DiffOperator(A.grid.dims)
    m = A.domain_size()
    sa = k.stack_maps([
        k.ScaledBlock(1.0, A),
        k.ScaledBlock(0.3, k.compose(k.DiagonalMap(conv(d["w1"])), D)),
        k.ScaledBlock(0.4, k.compose(k.DiagonalMap(conv(d["w2"])), D)),
        k.ScaledBlock(0.2, k.compose(k.DiagonalMap(conv(d["wi"])), k.IdentityMap(m))),
    ])
    sb = k.stack_maps([k.ScaledBlock(0.7, k.compose(k.DiagonalMap(conv(d["wp"])), A)),
                       k.ScaledBlock(0.5, D)])
    return sa, sb


def test_stack_golden_host(small):
    d, gs, ge, A = small
    sa, sb = _stacks(d, A)
    assert sa.range_size() == d["rhs_a"].size and sa.domain_size() == A.domain_size()
    ra = k.cgls(sa, d["rhs_a"], None, k.KrylovConfig(max_iters=6))
    assert rel_l2(ra.x, d["xa"]) < RTOL
    np.testing.assert_allclose(ra.trace.residual_norms, d["res_a"], rtol=RTOL)
    assert ra.trace.iterations == 6 and not ra.trace.converged and not ra.trace.breakdown
    assert len(ra.trace.wall_times) == 6 and np.all(np.diff(ra.trace.wall_times) > 0)
    rb = k.cgls(sb, d["rhs_b"], d["prior"], k.KrylovConfig(max_iters=12, tolerance=2e-2))
    assert rel_l2(rb.x, d["xb"]) < RTOL
    assert rb.trace.iterations == int(d["iters_b"]) and rb.trace.converged == bool(d["converged_b"])
    np.testing.assert_allclose(rb.trace.residual_norms, d["res_b"], rtol=RTOL)
    print(f"stack A {rel_l2(ra.x, d['xa']):.2e}  stack B {rel_l2(rb.x, d['xb']):.2e}")


def test_stack_device_tensors_match_host(small):
    """CUDA tensors in the reference layout take the same path without host copies."""
    import torch
    d, gs, ge, A = small
    dev = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).cuda()  # noqa: E731
    sa_h, _ = _stacks(d, A)
    sa_d, _ = _stacks(d, A, dev)
    rh = k.cgls(sa_h, d["rhs_a"], None, k.KrylovConfig(max_iters=6))
    rd = k.cgls(sa_d, dev(d["rhs_a"]), None, k.KrylovConfig(max_iters=6), layout="reference")
    assert np.array_equal(rd.x.cpu().numpy(), rh.x)
    # native layout: convert the pieces with the projector's own converters
    m, n = A.domain_size(), A.range_size()
    nat_v = lambda a: A.volume_to_native(dev(a))  # noqa: E731
    nat3 = lambda a: torch.cat([nat_v(a[c * m:(c + 1) * m]) for c in range(3)])  # noqa: E731
    D = k.DiffOperator(gs.dims)
    sn = k.stack_maps([k.ScaledBlock(1.0, A),
                       k.ScaledBlock(0.3, k.compose(k.DiagonalMap(nat3(d["w1"])), D)),
                       k.ScaledBlock(0.4, k.compose(k.DiagonalMap(nat3(d["w2"])), D)),
                       k.ScaledBlock(0.2, k.compose(k.DiagonalMap(nat_v(d["wi"])), k.IdentityMap(m)))])
    rhs = d["rhs_a"]
    rhs_n = torch.cat([A.proj_to_native(dev(rhs[:n])), nat3(rhs[n:n + 3 * m]),
                       nat3(rhs[n + 3 * m:n + 6 * m]), nat_v(rhs[n + 6 * m:])])
    rn = k.cgls(sn, rhs_n, None, k.KrylovConfig(max_iters=6))  # device default: native
    assert np.array_equal(A.volume_from_native(rn.x).cpu().numpy(), rh.x)


def test_single_block_is_cgls_recon(small):
    """cgls(A, b, 0) is what cgls_recon runs (recon.hpp:274-307)."""
    d, gs, ge, A = small
    r = k.cgls(A, d["b"], None, k.KrylovConfig(max_iters=8))
    rep = k.cgls_recon(k.ProjectionSet(ge, d["b"]), gs, 8, projector=A)
    assert rel_l2(r.x, rep.volume) < 1e-5
    np.testing.assert_allclose(r.trace.residual_norms, rep.residual_history, rtol=1e-5)


def test_stack_reproduces_irn_cycle(small, ora):
    """One outer cycle of irn_piccs == cgls on the caller-assembled reweighted
    stack (recon.hpp:195-232): the fused implicit-residual engine and the
    materialised generic engine agree."""
    d, gs, ge, A = small
    grid = grid_from(d)
    dims, m = (grid.nx, grid.ny, grid.nz), grid.count
    tau, a, lam = 1e-3, 0.3, 0.3
    w1 = ora.tv_weights(ora.diff(dims, np.zeros(m)), tau)
    w2 = ora.tv_weights(ora.diff(dims, -d["prior"].astype(np.float64)), tau)
    rhs = np.concatenate([d["b"], np.zeros(3 * m), lam * w2 * ora.diff(dims, d["prior"])])
    D = k.DiffOperator(dims)
    st = k.stack_maps([(1.0, A), (a, k.compose(k.DiagonalMap(w1), D)),
                       (lam, k.compose(k.DiagonalMap(w2), D))])
    r = k.cgls(st, rhs, None, k.KrylovConfig(max_iters=4))
    rep = k.irn_piccs(k.ProjectionSet(ge, d["b"]), gs, d["prior"],
                      k.RegularizationParams(alpha=a, tau=tau, outer_iters=1, inner_iters=4), projector=A)
    assert rel_l2(r.x, rep.volume) < 1e-4
    np.testing.assert_allclose(r.trace.residual_norms, rep.residual_history, rtol=1e-4)


def test_stack_hook_order(small):
    """test_krylov.cpp:120-135: the hook sees iterations 1..n with the iterate."""
    d, gs, ge, A = small
    sa, _ = _stacks(d, A)
    seen = []
    r = k.cgls(sa, d["rhs_a"], None, k.KrylovConfig(max_iters=5, hook=lambda it, x: seen.append((it, x.copy()))))
    assert [it for it, _ in seen] == [1, 2, 3, 4, 5]
    assert np.array_equal(seen[-1][1], r.x)


def test_zero_rhs_converges_at_start(small):
    """krylov.hpp:76-79: gamma == 0 -> converged, no iterations, x = x0."""
    d, gs, ge, A = small
    r = k.cgls(A, np.zeros(A.range_size(), np.float32), None, k.KrylovConfig(max_iters=5))
    assert r.trace.converged and r.trace.iterations == 0 and not np.any(r.x)


def test_stack_errors(small):
    d, gs, ge, A = small
    D = k.DiffOperator(gs.dims)
    with pytest.raises(k.ConfigError):   # cgls: rhs size mismatch (krylov.hpp:61)
        k.cgls(k.stack_maps([(1.0, A), (0.5, D)]), d["b"], None)
    with pytest.raises(k.ConfigError):   # x0 size mismatch (:62)
        k.cgls(A, d["b"], np.zeros(3, np.float32))
    with pytest.raises(k.ConfigError):   # no projector block: nothing owns the device
        k.cgls(k.stack_maps([(1.0, D)]), np.zeros(D.range_size(), np.float32), None)
    with pytest.raises(k.ConfigError):   # compose: size mismatch (linear_map.hpp:117-118)
        k.compose(k.DiagonalMap(np.ones(5)), D)
    with pytest.raises(k.ConfigError):   # stack: empty (linear_map.hpp:165)
        k.stack_maps([])
    with pytest.raises(k.ConfigError):
        k.cgls(k.stack_maps([(1.0, A), (1.0, k.DiffOperator((3, 3, 3)))]), d["b"], None)
    with pytest.raises(k.SolverError):   # krylov.hpp:75
        bad = d["b"].copy()
        # the central ray of the first view crosses the volume, so A^T r is
        # non-finite (a corner ray that misses it would leave gamma finite,
        # in the reference too)
        bad[(ge.nv // 2) * ge.nu + ge.nu // 2] = np.inf
        k.cgls(A, bad, None, k.KrylovConfig(max_iters=2))


def test_stack_c1_geometry(ora):
    """Config-size run: c1 (64^3, 30 views) reweighted TV stack, 10 iterations,
    against the float64 oracle."""
    grid, geom = baseline_geometry(1)
    gs, ge = to_pkg(grid, geom)
    A = k.ConeBeamProjector(gs, ge)
    rng = np.random.default_rng(11)
    m = grid.count
    dims = (grid.nx, grid.ny, grid.nz)
    z, y, x = np.meshgrid(*(np.linspace(-1, 1, n) for n in dims[::-1]), indexing="ij")
    truth = (0.02 * ((x * x + y * y + z * z) < 0.5) + 0.01 * ((x - 0.2) ** 2 + y * y < 0.05)).reshape(-1)
    truth = truth.astype(np.float32)
    b = A.apply(truth)
    b = (b + 0.01 * b.max() * rng.standard_normal(b.size)).astype(np.float32)
    xr = (truth + 0.001 * rng.standard_normal(m)).astype(np.float32)
    w = ora.tv_weights(ora.diff(dims, xr), 1e-4).astype(np.float32)
    rhs = np.concatenate([b, np.zeros(3 * m, np.float32)])
    st = k.stack_maps([(1.0, A), (0.5, k.compose(k.DiagonalMap(w), k.DiffOperator(dims)))])
    r = k.cgls(st, rhs, None, k.KrylovConfig(max_iters=10))
    xo, to = ora.cgls_stack(grid, geom, [(0, 1.0, None), (1, 0.5, w)], rhs, 10)
    e = rel_l2(r.x, xo)
    print(f"c1 stack cgls: iterate {e:.2e}")
    assert e < RTOL
    np.testing.assert_allclose(r.trace.residual_norms, to["residual_history"], rtol=RTOL)
