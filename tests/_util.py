"""Shared test helpers: golden fixtures, geometry converters, metrics."""
import os

import numpy as np

from oracle import Geometry, Grid, uniform_angles

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def grid_from(d):
    g = d["grid"]
    return Grid(int(g[0]), int(g[1]), int(g[2]), *map(float, g[3:9]))


def geom_from(d):
    g = d["geom"]
    return Geometry(float(g[0]), float(g[1]), int(g[2]), int(g[3]), float(g[4]), float(g[5]),
                    d["angles"], float(g[6]), float(g[7]))


def to_pkg(grid, geom):
    """oracle Grid/Geometry -> package GridSpec/ConeBeamGeometry."""
    import paper_2509_08574_b200 as k
    gs = k.GridSpec((grid.nx, grid.ny, grid.nz), (grid.sx, grid.sy, grid.sz),
                    (grid.ox, grid.oy, grid.oz))
    ge = k.ConeBeamGeometry(geom.dso, geom.dsd, geom.nu, geom.nv, geom.pu, geom.pv, geom.angles,
                            geom.offset_u, geom.offset_v)
    return gs, ge


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def tiny_geometry(n_angles=8, nu=10, nv=9):
    """oracle_helpers.hpp:97-108."""
    return Geometry(40.0, 90.0, nu, nv, 1.6, 1.9, uniform_angles(n_angles), 0.7, -0.5)


def tiny_grid(nx=4, ny=4, nz=4):
    """oracle_helpers.hpp:110-112."""
    return Grid(nx, ny, nz, 1.0, 1.1, 0.9)


def recon_geometry(n_angles, nu=16, nv=16):
    """test_recon.cpp:16-25."""
    return Geometry(30.0, 60.0, nu, nv, 2.0, 2.0, uniform_angles(n_angles))


def baseline_geometry(cfg, n_angles=None):
    """BASELINE.json configs c1..c5 (DSO 1000, DSD 1500)."""
    vol = {1: (64, 1.0), 2: (128, 0.8), 3: (256, 0.5), 4: (512, 0.25), 5: (256, 0.5)}[cfg]
    det = {1: (96, 1.0), 2: (192, 0.8), 3: (384, 0.5), 4: (768, 0.4), 5: (384, 0.5)}[cfg]
    na = n_angles or {1: 64, 2: 45, 3: 60, 4: 90, 5: 45}[cfg]
    grid = Grid(vol[0], vol[0], vol[0], vol[1], vol[1], vol[1])
    geom = Geometry(1000.0, 1500.0, det[0], det[0], det[1], det[1], uniform_angles(na))
    return grid, geom
