"""GPU: IRN-PICCS at the BASELINE configs' own sizes and inputs against the
UNMODIFIED reference (oracle/_ref: the reference headers compiled in place).

North-star bar: reconstructions after a fixed iteration count within 1e-3
relative L2 of the reference iterate, on the same seeded inputs.  The inputs
are the configs' seeded studies (synth.scan_inputs): prior image = 20-iteration
CGLS of a noiseless 360-view scan of the prior phantom, follow-up readings with
Poisson noise; identical float32 b / prior / initial go to both solvers.

Both control flows of the device solver are checked:
* "reuse" (default): a warm start continues the data residual of the previous
  cycle's CGLS recurrence;
* "restart" (kct_set_option "solver_restart" = 1): the reference's own flow —
  r = b - A x and A^T r recomputed at every CGLS start (krylov.hpp:68-75) and
  a fresh A x for every objective (recon.hpp:189, :238).

The reference solve runs once per config on all host cores (c3: the metric's
own config, 4x5 iterations, alpha = lambda = 0.5, tau auto).
"""
import os
import time

import numpy as np
import pytest

import paper_2509_08574_b200 as k
from paper_2509_08574_b200 import synth
from oracle import KIND_PICCS, Geometry, Grid, Oracle, LIBS
from tests._util import rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
RTOL = 1e-3

needs_ref = pytest.mark.skipif(not os.path.exists(LIBS["ref"][0]),
                               reason="oracle/_ref not built (make -C oracle ref)")


def _ora_grid_geom(grid, geom):
    g = Grid(*grid.dims, *grid.spacing, *grid.origin)
    ge = Geometry(geom.dso, geom.dsd, geom.nu, geom.nv, geom.pu, geom.pv, geom.angles,
                  geom.offset_u, geom.offset_v)
    return g, ge


def _reference(inp, params, x0=None):
    ref = Oracle("ref")
    ref.set_threads(os.cpu_count() or 1)
    g, ge = _ora_grid_geom(inp["grid"], inp["geom"])
    t0 = time.perf_counter()
    x, rep = ref.irn(g, ge, KIND_PICCS, inp["b"].astype(np.float64),
                     inp["prior"].astype(np.float64), params, x0=x0,
                     ground_truth=inp["follow"])
    rep["wall"] = time.perf_counter() - t0
    return x, rep


def _gpu(inp, params, restart, x0=None):
    A = inp["projector"]
    A.set_option("solver_restart", 1 if restart else 0)
    try:
        rep = k.irn_piccs(k.ProjectionSet(inp["geom"], inp["b"]), inp["grid"], inp["prior"],
                          k.RegularizationParams(alpha=params["alpha"],
                                                 outer_iters=params["outer_iters"],
                                                 inner_iters=params["inner_iters"]),
                          k.ReconOptions(initial=x0, ground_truth=inp["follow"]), projector=A)
    finally:
        A.set_option("solver_restart", 0)
    return rep


def _compare(name, rep, x_ref, r_ref):
    ex = rel_l2(rep.volume, x_ref)
    eo = float(np.max(np.abs(rep.objective_history / r_ref["objective_history"] - 1)))
    er = float(np.max(np.abs(rep.residual_history / r_ref["residual_history"] - 1)))
    ee = float(np.max(np.abs(rep.error_history / r_ref["error_history"] - 1)))
    print(f"\n[{name}] iterate rel-L2 {ex:.3e}  objective {eo:.3e}  residual {er:.3e}  "
          f"error history {ee:.3e}  tau {rep.tau:.6e} / {r_ref['tau']:.6e}  "
          f"rel error vs phantom {rep.error_history[-1]:.4f}  "
          f"(reference {r_ref['wall']:.1f} s on {os.cpu_count()} threads, "
          f"GPU {rep.solve_seconds:.3f} s)")
    assert ex < RTOL, (name, ex)
    assert eo < RTOL, (name, eo)
    assert er < RTOL, (name, er)
    assert ee < RTOL, (name, ee)
    assert rep.tau == pytest.approx(r_ref["tau"], rel=1e-6)
    assert list(rep.outer_boundaries) == list(r_ref["outer_boundaries"])
    return ex


def _params(cfg):
    return dict(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner)


@needs_ref
@pytest.mark.parametrize("cfg_name", ["c2", "c3"])
def test_piccs_config_parity(cfg_name):
    """c2 (128^3, 45 views, I0 1e5) and c3 (256^3, 60 views, I0 5e4), 4x5 PICCS."""
    inp = synth.scan_inputs(cfg_name)
    p = _params(inp["cfg"])
    x_ref, r_ref = _reference(inp, p)
    for restart in (False, True):
        rep = _gpu(inp, p, restart)
        _compare(f"{cfg_name} {'restart' if restart else 'reuse'}", rep, x_ref, r_ref)


@needs_ref
def test_c5_warm_started_followup_parity():
    """c5 (256^3, 45 views, I0 1e5): the second follow-up, 3x5 PICCS warm-started
    (ReconOptions.initial, recon.hpp:157; tau from the initial image :161-162)
    from the GPU's first follow-up result; both solvers get the same initial."""
    inp0 = synth.scan_inputs("c5", followup_step=0)
    p = _params(inp0["cfg"])
    first = _gpu(inp0, p, False, x0=inp0["prior"])
    x0 = np.asarray(first.volume, dtype=np.float32)
    inp = synth.scan_inputs("c5", followup_step=1)
    x_ref, r_ref = _reference(inp, p, x0=x0)
    for restart in (False, True):
        rep = _gpu(inp, p, restart, x0=x0)
        _compare(f"c5 step 1 {'restart' if restart else 'reuse'}", rep, x_ref, r_ref)
