"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference kryct code (oracle/_ref/libkryct_ref.so, compiled
from /root/reference/proj/include by oracle/Makefile) on small seeded inputs
and stores inputs + float64 outputs as .npz.  Inputs are float32-representable
so the CUDA path (float32 boundary) sees bit-identical data.

    make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import (KIND_PICCS, KIND_PIPLE, KIND_TV, Geometry, Grid, Oracle,  # noqa: E402
                    uniform_angles)

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def tiny_geometry(n_angles=8, nu=10, nv=9):
    """oracle_helpers.hpp:97-108."""
    return Geometry(40.0, 90.0, nu, nv, 1.6, 1.9, uniform_angles(n_angles), 0.7, -0.5)


def recon_geometry(n_angles, nu=16, nv=16):
    """test_recon.cpp:16-25."""
    return Geometry(30.0, 60.0, nu, nv, 2.0, 2.0, uniform_angles(n_angles))


def sphere(grid, radius=0.6, value=1.0):
    """phantoms.hpp:176-183 shape on normalised coordinates (voxel centres)."""
    x = -1 + 2 * (np.arange(grid.nx) + 0.5) / grid.nx
    y = -1 + 2 * (np.arange(grid.ny) + 0.5) / grid.ny
    z = -1 + 2 * (np.arange(grid.nz) + 0.5) / grid.nz
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return np.where(X * X + Y * Y + Z * Z <= radius * radius, value, 0.0).reshape(-1)


def grid_dict(g):
    return dict(grid=np.array([g.nx, g.ny, g.nz, g.sx, g.sy, g.sz, g.ox, g.oy, g.oz]))


def geom_dict(g):
    return dict(geom=np.array([g.dso, g.dsd, g.nu, g.nv, g.pu, g.pv, g.offset_u, g.offset_v]),
                angles=g.angles)


def op_case(ref, name, grid, geom, seed):
    rng = np.random.default_rng(seed)
    x = f32(rng.uniform(-1, 1, grid.count))
    y = f32(rng.uniform(-1, 1, geom.ray_count))
    ax = ref.forward(grid, geom, x)
    aty = ref.adjoint(grid, geom, y)
    ones = ref.forward(grid, geom, np.full(grid.count, 2.5))
    nnz = ref.count_nnz(grid, geom)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x=x, y=y, ax=ax, aty=aty,
                        ax_uniform=ones, nnz=nnz, **grid_dict(grid), **geom_dict(geom))


def recon_case(ref, name, grid, geom, seed):
    rng = np.random.default_rng(seed)
    truth = f32(sphere(grid, 0.6, 0.8) + 0.05 * rng.uniform(0, 1, grid.count))
    prior = f32(0.9 * truth)
    b = f32(ref.forward(grid, geom, truth) + 0.01 * rng.standard_normal(geom.ray_count))
    res = {}
    x, r = ref.cgls_recon(grid, geom, b, 8, ground_truth=truth)
    res["cgls_x"], res["cgls_res"], res["cgls_err"] = x, r["residual_history"], r["error_history"]
    p = dict(alpha=0.3, outer_iters=3, inner_iters=4, tau=1e-3)
    for kind, tag in ((KIND_TV, "tv"), (KIND_PIPLE, "piple"), (KIND_PICCS, "piccs")):
        x, r = ref.irn(grid, geom, kind, b, prior, p, ground_truth=truth)
        res[f"{tag}_x"] = x
        res[f"{tag}_obj"] = r["objective_history"]
        res[f"{tag}_res"] = r["residual_history"]
        res[f"{tag}_err"] = r["error_history"]
    # auto tau from the prior, lambda != alpha
    x, r = ref.irn(grid, geom, KIND_PICCS, b, prior,
                   dict(alpha=0.2, lambda_=0.4, outer_iters=2, inner_iters=5), ground_truth=truth)
    res["piccs_auto_x"], res["piccs_auto_obj"], res["piccs_auto_tau"] = x, r["objective_history"], r["tau"]
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), truth=truth, prior=prior, b=b, **res,
                        **grid_dict(grid), **geom_dict(geom))


def fdk_case(ref, name, grid, geom, seed):
    """fdk.hpp:50-139 on a projected ellipsoid phantom."""
    rng = np.random.default_rng(seed)
    truth = f32(sphere(grid, 0.55, 0.02) + 0.005 * rng.uniform(0, 1, grid.count))
    proj = f32(ref.forward(grid, geom, truth))
    vol = ref.fdk(grid, geom, proj)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), truth=truth, proj=proj, fdk=vol,
                        **grid_dict(grid), **geom_dict(geom))


def stack_inputs(ref, grid, geom, seed):
    """Two caller-assembled stacks (linear_map.hpp:159-216) on the recon_small problem:
    A = [A; 0.3 W1 D; 0.4 W2 D; 0.2 Wi I] from zero (the reweighted PICCS system of
    recon.hpp:195-221 plus a weighted identity block), B = [0.7 Wp A; 0.5 D] warm-started
    with a tolerance.  Returns float32-representable inputs."""
    rng = np.random.default_rng(seed)
    m, n = grid.count, geom.ray_count
    dims = (grid.nx, grid.ny, grid.nz)
    truth = f32(sphere(grid, 0.6, 0.8) + 0.05 * rng.uniform(0, 1, m))
    prior = f32(0.9 * truth)
    b = f32(ref.forward(grid, geom, truth) + 0.01 * rng.standard_normal(n))
    xr = f32(truth + 0.02 * rng.standard_normal(m))
    w1 = f32(ref.tv_weights(ref.diff(dims, xr), 1e-2))
    w2 = f32(ref.tv_weights(ref.diff(dims, xr - prior), 1e-2))
    wi = f32(rng.uniform(0.5, 1.5, m))
    wp = f32(rng.uniform(0.5, 1.5, n))
    rhs_a = np.concatenate([b, np.zeros(3 * m), f32(0.4 * w2 * ref.diff(dims, prior)),
                            f32(0.2 * wi * prior)])
    rhs_b = np.concatenate([f32(0.7 * wp * b), np.zeros(3 * m)])
    return dict(truth=truth, prior=prior, b=b, w1=w1, w2=w2, wi=wi, wp=wp, rhs_a=rhs_a, rhs_b=rhs_b)


def stack_blocks(d):
    a = [(0, 1.0, None), (1, 0.3, d["w1"]), (1, 0.4, d["w2"]), (2, 0.2, d["wi"])]
    b = [(0, 0.7, d["wp"]), (1, 0.5, None)]
    return a, b


def stack_case(ref, name, grid, geom, seed):
    """cgls (krylov.hpp:59-127) over caller-assembled StackedMaps, by the reference."""
    d = stack_inputs(ref, grid, geom, seed)
    blk_a, blk_b = stack_blocks(d)
    xa, ta = ref.cgls_stack(grid, geom, blk_a, d["rhs_a"], 6)
    xb, tb = ref.cgls_stack(grid, geom, blk_b, d["rhs_b"], 12, x0=d["prior"], tol=2e-2)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d, xa=xa, res_a=ta["residual_history"],
                        xb=xb, res_b=tb["residual_history"], iters_b=tb["iterations"],
                        converged_b=tb["converged"], **grid_dict(grid), **geom_dict(geom))


def main():
    ref = Oracle("ref")
    if len(sys.argv) > 1 and sys.argv[1] == "stack":   # add the stack fixture only
        stack_case(ref, "stack_small", Grid(8, 8, 8), recon_geometry(6), 106)
        return
    op_case(ref, "op_tiny", Grid(4, 4, 4, 1.0, 1.1, 0.9), tiny_geometry(8, 10, 9), 101)
    op_case(ref, "op_tiny_odd", Grid(5, 6, 4, 1.0, 1.1, 0.9), tiny_geometry(7, 9, 8), 102)
    op_case(ref, "op_c1_small", Grid(16, 16, 16, 4.0, 4.0, 4.0),
            Geometry(1000.0, 1500.0, 24, 24, 4.0, 4.0, uniform_angles(16)), 103)
    recon_case(ref, "recon_small", Grid(8, 8, 8), recon_geometry(6), 104)
    stack_case(ref, "stack_small", Grid(8, 8, 8), recon_geometry(6), 106)
    fdk_case(ref, "fdk_small", Grid(24, 24, 16, 2.0, 2.0, 2.0),
             Geometry(1000.0, 1500.0, 48, 32, 2.0, 2.0, uniform_angles(36), 0.5, -0.7), 105)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
