"""CPU: pin the oracle (our plain-C restatement) against the reference.

The golden fixtures were produced by the unmodified reference code
(tests/golden/make_golden.py -> oracle/_ref).  When the compiled reference is
present (it travels with the repo snapshot) it is also compared directly.
Property checks restate the reference's own unit tests
(proj/tests/test_projector.cpp, test_diffreg.cpp, test_recon.cpp).
"""
import math
import os

import numpy as np
import pytest

from oracle import KIND_PICCS, KIND_PIPLE, KIND_TV, LIBS, Geometry, Grid, Oracle, uniform_angles
from tests._util import geom_from, grid_from, load_golden, recon_geometry, rel_l2, tiny_geometry, tiny_grid

HAVE_REF = os.path.exists(LIBS["ref"][0])


@pytest.fixture(scope="module")
def ora():
    import oracle
    oracle.build("ora")
    return Oracle("ora")


@pytest.mark.parametrize("case", ["op_tiny", "op_tiny_odd", "op_c1_small"])
def test_operator_golden(ora, case):
    d = load_golden(case)
    grid, geom = grid_from(d), geom_from(d)
    np.testing.assert_allclose(ora.forward(grid, geom, d["x"]), d["ax"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ora.adjoint(grid, geom, d["y"]), d["aty"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ora.forward(grid, geom, np.full(grid.count, 2.5)), d["ax_uniform"],
                               rtol=0, atol=1e-12)
    assert ora.count_nnz(grid, geom) == int(d["nnz"])


def test_recon_golden(ora):
    d = load_golden("recon_small")
    grid, geom = grid_from(d), geom_from(d)
    x, r = ora.cgls_recon(grid, geom, d["b"], 8, ground_truth=d["truth"])
    assert rel_l2(x, d["cgls_x"]) < 1e-12
    np.testing.assert_allclose(r["residual_history"], d["cgls_res"], rtol=1e-12)
    np.testing.assert_allclose(r["error_history"], d["cgls_err"], rtol=1e-12)
    p = dict(alpha=0.3, outer_iters=3, inner_iters=4, tau=1e-3)
    for kind, tag in ((KIND_TV, "tv"), (KIND_PIPLE, "piple"), (KIND_PICCS, "piccs")):
        x, r = ora.irn(grid, geom, kind, d["b"], d["prior"], p, ground_truth=d["truth"])
        assert rel_l2(x, d[f"{tag}_x"]) < 1e-12, tag
        np.testing.assert_allclose(r["objective_history"], d[f"{tag}_obj"], rtol=1e-12)
        np.testing.assert_allclose(r["residual_history"], d[f"{tag}_res"], rtol=1e-12)
        np.testing.assert_allclose(r["error_history"], d[f"{tag}_err"], rtol=1e-12)
    x, r = ora.irn(grid, geom, KIND_PICCS, d["b"], d["prior"],
                   {"alpha": 0.2, "lambda": 0.4, "outer_iters": 2, "inner_iters": 5},
                   ground_truth=d["truth"])
    assert r["tau"] == pytest.approx(float(d["piccs_auto_tau"]), rel=1e-15)
    assert rel_l2(x, d["piccs_auto_x"]) < 1e-12


def _stack_blocks(d):
    a = [(0, 1.0, None), (1, 0.3, d["w1"]), (1, 0.4, d["w2"]), (2, 0.2, d["wi"])]
    b = [(0, 0.7, d["wp"]), (1, 0.5, None)]
    return a, b


def test_stack_cgls_golden(ora):
    """cgls (krylov.hpp:59-127) over caller-assembled StackedMaps
    (linear_map.hpp:159-216): the restatement against the reference's own run."""
    d = load_golden("stack_small")
    grid, geom = grid_from(d), geom_from(d)
    blk_a, blk_b = _stack_blocks(d)
    xa, ta = ora.cgls_stack(grid, geom, blk_a, d["rhs_a"], 6)
    assert rel_l2(xa, d["xa"]) < 1e-12
    np.testing.assert_allclose(ta["residual_history"], d["res_a"], rtol=1e-12)
    xb, tb = ora.cgls_stack(grid, geom, blk_b, d["rhs_b"], 12, x0=d["prior"], tol=2e-2)
    assert rel_l2(xb, d["xb"]) < 1e-12
    np.testing.assert_allclose(tb["residual_history"], d["res_b"], rtol=1e-12)
    assert tb["iterations"] == int(d["iters_b"]) and tb["converged"] == bool(d["converged_b"])


def test_stack_cgls_reduces_to_irn_cycle(ora):
    """One outer cycle of irn_piccs is cgls on [A; a W1 D; l W2 D] with the rhs
    [b; 0; l W2 D x_p] (recon.hpp:195-232) — the stack API reproduces it."""
    d = load_golden("recon_small")
    grid, geom = grid_from(d), geom_from(d)
    dims, m = (grid.nx, grid.ny, grid.nz), grid.count
    tau, a, lam = 1e-3, 0.3, 0.3
    w1 = ora.tv_weights(ora.diff(dims, np.zeros(m)), tau)
    w2 = ora.tv_weights(ora.diff(dims, -d["prior"]), tau)
    rhs = np.concatenate([d["b"], np.zeros(3 * m), lam * w2 * ora.diff(dims, d["prior"])])
    x, _ = ora.cgls_stack(grid, geom, [(0, 1.0, None), (1, a, w1), (1, lam, w2)], rhs, 4)
    xi, _ = ora.irn(grid, geom, KIND_PICCS, d["b"], d["prior"],
                    dict(alpha=a, outer_iters=1, inner_iters=4, tau=tau))
    assert rel_l2(x, xi) < 1e-12


def test_stack_errors(ora):
    d = load_golden("stack_small")
    grid, geom = grid_from(d), geom_from(d)
    with pytest.raises(Exception):
        ora.cgls_stack(grid, geom, [(7, 1.0, None)], np.zeros(geom.ray_count), 2)


def test_fdk_golden(ora):
    """fdk.hpp:50-139 restated (radix-2 FFT ramp filter) reproduces the reference."""
    d = load_golden("fdk_small")
    np.testing.assert_allclose(ora.fdk(grid_from(d), geom_from(d), d["proj"]), d["fdk"],
                               rtol=0, atol=1e-12)


@pytest.mark.skipif(not HAVE_REF, reason="reference not compiled (make -C oracle ref)")
def test_oracle_equals_reference_c1():
    """Our restatement reproduces the reference bit for bit at c1 geometry."""
    from tests._util import baseline_geometry
    ora, ref = Oracle("ora"), Oracle("ref")
    grid, geom = baseline_geometry(1, n_angles=8)
    x = np.random.default_rng(5).uniform(0, 1, grid.count).astype(np.float32)
    a, b = ora.forward(grid, geom, x), ref.forward(grid, geom, x)
    assert np.array_equal(a, b)
    y = b.astype(np.float32)
    assert rel_l2(ora.adjoint(grid, geom, y), ref.adjoint(grid, geom, y)) < 1e-14


# ---- properties restated from the reference's own unit tests ----------------
def test_axis_aligned_ray_unit_lengths(ora):
    """test_projector.cpp:7-15."""
    grid = Grid(16, 8, 8, 1.0, 2.0, 2.0)
    vox, lens, _ = ora.trace_ray(grid, [-100, 0.3, 0.4], [100, 0.3, 0.4])
    assert len(vox) == 16
    np.testing.assert_allclose(lens, 1.0, atol=1e-12)
    assert np.all(np.diff(vox.astype(np.int64)) == 1)


def test_lengths_sum_to_chord(ora):
    """test_projector.cpp:17-31."""
    grid = Grid(7, 9, 11, 1.2, 0.7, 1.0)
    rng = np.random.default_rng(21)
    for _ in range(200):
        t = rng.uniform(0, 2 * math.pi)
        src = [40 * math.cos(t), 40 * math.sin(t), rng.uniform(-6, 6) * 0.5]
        dst = [rng.uniform(-6, 6) * 0.2, rng.uniform(-6, 6) * 0.2, rng.uniform(-6, 6) * 0.4]
        vox, lens, (t0, t1) = ora.trace_ray(grid, src, dst)
        chord = (t1 - t0) * np.linalg.norm(np.subtract(dst, src))
        assert abs(lens.sum() - chord) < 1e-9
        assert np.all(lens > 0)


def test_missing_rays(ora):
    """test_projector.cpp:33-39."""
    grid = Grid(8, 8, 8)
    assert len(ora.trace_ray(grid, [-20, 30, 0], [20, 30, 0])[0]) == 0
    assert len(ora.trace_ray(grid, [-20, 0, 9], [20, 0, 9])[0]) == 0
    assert len(ora.trace_ray(grid, [-20, 4.0, 0], [20, 4.0, 0])[0]) == 0


def test_exact_transpose_tiny(ora):
    """test_projector.cpp:77-85: dense matricisations agree to 1e-14, A >= 0."""
    grid, geom = tiny_grid(), tiny_geometry(3, 6, 5)
    m, n = grid.count, geom.ray_count
    fwd = np.stack([ora.forward(grid, geom, np.eye(m)[j]) for j in range(m)], axis=1)
    adj = np.stack([ora.adjoint(grid, geom, np.eye(n)[i]) for i in range(n)], axis=0)
    assert np.abs(fwd - adj).max() < 1e-14
    assert fwd.min() >= 0 and fwd.max() > 0


def test_diff_kronecker(ora):
    """test_diffreg.cpp:29-48."""
    nx, ny, nz = 4, 3, 2
    m = nx * ny * nz

    def d1(n):
        a = np.zeros((n, n))
        for i in range(n - 1):
            a[i, i], a[i, i + 1] = -1, 1
        return a

    want = np.vstack([np.kron(np.eye(nz), np.kron(np.eye(ny), d1(nx))),
                      np.kron(np.eye(nz), np.kron(d1(ny), np.eye(nx))),
                      np.kron(d1(nz), np.kron(np.eye(ny), np.eye(nx)))])
    got = np.stack([ora.diff((nx, ny, nz), np.eye(m)[j]) for j in range(m)], axis=1)
    gotT = np.stack([ora.diff_adjoint((nx, ny, nz), np.eye(3 * m)[i]) for i in range(3 * m)], axis=0)
    assert np.array_equal(got, want) and np.array_equal(gotT, want)


def test_tv_weights_formula(ora):
    """test_diffreg.cpp:98-113 and :170-184."""
    rng = np.random.default_rng(34)
    x = rng.uniform(-1, 1, 64)
    g = ora.diff((4, 4, 4), x)
    w = ora.tv_weights(g, 1e-4)
    mag2 = g[:64] ** 2 + g[64:128] ** 2 + g[128:] ** 2
    np.testing.assert_allclose(w[:64], (mag2 + 1e-8) ** -0.25, rtol=1e-12)
    assert np.array_equal(w[:64], w[64:128]) and np.array_equal(w[:64], w[128:])
    w0 = ora.tv_weights(ora.diff((4, 4, 4), x - x), 1e-4)
    np.testing.assert_allclose(w0, 1 / math.sqrt(1e-4), rtol=1e-12)


def test_resolve_tau_cases(ora):
    """test_recon.cpp:72-86."""
    assert ora.resolve_tau(0.5) == 0.5
    assert ora.resolve_tau(0.5, [1.0, 9.0]) == 0.5
    assert ora.resolve_tau(0.0) == 1e-4
    assert ora.resolve_tau(-3.0) == 1e-4
    assert ora.resolve_tau(0.0, [0.25, 1.0, 2.25]) == pytest.approx(2e-4, rel=1e-12)
    assert ora.resolve_tau(0.0, [0.7] * 10) == 1e-4
    assert ora.resolve_tau(0.0, [0.0, 1e-6]) == 1e-8


def test_lambda_zero_collapses_to_tv(ora):
    """test_recon.cpp:238-275 (bitwise)."""
    grid, geom = Grid(7, 7, 7), recon_geometry(5)
    rng = np.random.default_rng(1)
    truth = rng.uniform(0, 1, grid.count)
    b = ora.forward(grid, geom, truth)
    p = dict(alpha=0.25, lambda_=0.0, outer_iters=3, inner_iters=5)
    x_tv, _ = ora.irn(grid, geom, KIND_TV, b, None, p)
    x_pc, _ = ora.irn(grid, geom, KIND_PICCS, b, 0.9 * truth, p)
    x_pl, _ = ora.irn(grid, geom, KIND_PIPLE, b, 0.9 * truth, p)
    assert np.array_equal(x_tv, x_pc) and np.array_equal(x_tv, x_pl)


def test_uniform_volume_row_sums_are_box_chords():
    """A 1 = the ray's chord through the volume box (test_projector.cpp:54-69):
    the oracle's Siddon sums against the closed-form slab clip used by the
    full-size GPU property test (tests/test_fullsize_gpu.py)."""
    from tests._util import baseline_geometry, tiny_geometry, tiny_grid
    from oracle import build
    from tests.test_fullsize_gpu import box_chords
    build("ora")
    ora = Oracle("ora")
    for grid, geom in [(tiny_grid(6, 5, 7), tiny_geometry(5, 8, 9)), baseline_geometry(1, 3)]:
        want = ora.forward(grid, geom, np.ones(grid.count))
        got = box_chords(grid, geom)
        assert np.abs(got - want).max() < 1e-10
