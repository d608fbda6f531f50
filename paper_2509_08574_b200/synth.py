"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference's paper data (TIGRE head, clinical thorax scans) are not
available, and the reference's own phantoms are [0,1]-clamped normalised
shapes (phantoms.hpp:43-69) that cannot express the BASELINE configs, so the
configs are restated here: seeded random ellipsoids in mm with
additive attenuation in /mm (clipped >= 0, no upper clamp), z-rotation only,
evaluated at voxel centres; follow-up inserts (sphere, needle cylinder, grown
ellipsoid); Poisson transmission noise  counts ~ Poisson(I0 exp(-p)),
b = -ln(max(counts, 1) / I0).  Everything is float32 in the reference layout
(x-fastest volumes, u-fastest projections).  Pinned choices are recorded in
``CONFIGS`` and in DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int            # volume n^3
    voxel: float      # mm
    det: int          # detector det^2
    pitch: float      # mm
    n_ellipsoids: int
    prior_views: int
    followup_views: int
    i0: float         # Poisson I0 of the follow-up (0 = noiseless)
    iters: int        # PICCS (or CGLS for c1) iterations
    outer: int
    inner: int
    alpha: float = 0.5


DSO, DSD = 1000.0, 1500.0
CONFIGS = {
    "c1": Config("c1", 64, 1.0, 96, 1.0, 10, 64, 64, 0.0, 20, 1, 20),
    "c2": Config("c2", 128, 0.8, 192, 0.8, 15, 360, 45, 1e5, 20, 4, 5),
    "c3": Config("c3", 256, 0.5, 384, 0.5, 20, 360, 60, 5e4, 20, 4, 5),
    "c4": Config("c4", 512, 0.25, 768, 0.4, 30, 720, 90, 1e5, 30, 6, 5),
    "c5": Config("c5", 256, 0.5, 384, 0.5, 20, 360, 45, 1e5, 15, 3, 5),
}


def angles(n: int) -> np.ndarray:
    """experiment.hpp:89-94."""
    return 2.0 * np.pi * np.arange(n, dtype=np.float64) / float(n)


def _centres(n, voxel):
    return (np.arange(n, dtype=np.float64) + 0.5 - 0.5 * n) * voxel


def draw_ellipsoids(cfg: Config, seed: int):
    """Ellipsoid table [value, a, b, c, x0, y0, z0, phi] in mm / radians."""
    rng = np.random.Generator(np.random.PCG64(seed))
    fov = cfg.n * cfg.voxel
    scale = fov / 64.0
    rows = []
    for _ in range(cfg.n_ellipsoids):
        a, b, c = rng.uniform(4.0, 28.0, 3) * (scale if cfg.name != "c1" else 1.0)
        x0, y0, z0 = rng.uniform(-0.3, 0.3, 3) * fov
        phi = rng.uniform(0.0, np.pi)
        val = rng.uniform(0.005, 0.04)
        rows.append([val, a, b, c, x0, y0, z0, phi])
    return np.array(rows)


def render(cfg: Config, table, vol=None) -> np.ndarray:
    """Additive ellipsoids at voxel centres; returns float32 x-fastest (nz, ny, nx)."""
    n = cfg.n
    xs = _centres(n, cfg.voxel)
    acc = np.zeros((n, n, n), dtype=np.float64) if vol is None else vol.astype(np.float64).reshape(n, n, n)
    for val, a, b, c, x0, y0, z0, phi in table:
        r = max(a, b, c)
        sl = [np.nonzero(np.abs(xs - q) <= r + cfg.voxel)[0] for q in (z0, y0, x0)]
        if any(len(s) == 0 for s in sl):
            continue
        zk, yj, xi = [slice(s[0], s[-1] + 1) for s in sl]
        Z, Y, X = np.meshgrid(xs[zk] - z0, xs[yj] - y0, xs[xi] - x0, indexing="ij")
        cp, sp = np.cos(phi), np.sin(phi)
        qx = cp * X + sp * Y
        qy = -sp * X + cp * Y
        inside = (qx / a) ** 2 + (qy / b) ** 2 + (Z / c) ** 2 <= 1.0
        acc[zk, yj, xi] += val * inside
    np.maximum(acc, 0.0, out=acc)
    return acc.astype(np.float32).reshape(-1)


def add_sphere(cfg: Config, vol, centre, radius, value):
    n = cfg.n
    xs = _centres(n, cfg.voxel)
    Z, Y, X = np.meshgrid(xs - centre[2], xs - centre[1], xs - centre[0], indexing="ij")
    out = vol.reshape(n, n, n).astype(np.float64)
    out += value * (X * X + Y * Y + Z * Z <= radius * radius)
    return np.maximum(out, 0).astype(np.float32).reshape(-1)


def add_cylinder(cfg: Config, vol, tip, direction, length, radius, value):
    """Needle: segment from tip - length*dir to tip, radius r, additive value."""
    n = cfg.n
    xs = _centres(n, cfg.voxel)
    d = np.asarray(direction, dtype=np.float64)
    d /= np.linalg.norm(d)
    base = np.asarray(tip, dtype=np.float64) - length * d
    Z, Y, X = np.meshgrid(xs, xs, xs, indexing="ij")
    px, py, pz = X - base[0], Y - base[1], Z - base[2]
    t = px * d[0] + py * d[1] + pz * d[2]
    r2 = px * px + py * py + pz * pz - t * t
    inside = (t >= 0) & (t <= length) & (r2 <= radius * radius)
    out = vol.reshape(n, n, n).astype(np.float64)
    out += value * inside
    return np.maximum(out, 0).astype(np.float32).reshape(-1)


def poisson_log(p: np.ndarray, i0: float, seed: int) -> np.ndarray:
    """counts ~ Poisson(I0 exp(-p)); b = -ln(max(counts, 1) / I0)."""
    if i0 <= 0:
        return p.astype(np.float32)
    rng = np.random.Generator(np.random.PCG64(seed))
    counts = rng.poisson(i0 * np.exp(-p.astype(np.float64)))
    return (-np.log(np.maximum(counts, 1) / i0)).astype(np.float32)


def needle_pose(cfg: Config, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    fov = cfg.n * cfg.voxel
    tip = rng.uniform(-0.1, 0.1, 3) * fov
    d = rng.normal(size=3)
    d[2] *= 0.3
    return tip, d / np.linalg.norm(d)


def study(cfg_name: str, seed: int | None = None, followup_step: int = 0):
    """Prior phantom and follow-up phantom of a BASELINE config (float32, x-fastest).

    c2: + sphere r U(3,8) mm, +0.01/mm;  c3/c5: + needle r 1 mm, L 60 mm, 0.2/mm
    (c5: tip advanced 5 mm per follow-up step along its axis);
    c4: one ellipsoid's semi-axes x1.15 (local growth).
    """
    cfg = CONFIGS[cfg_name]
    seed = int(cfg_name[1]) if seed is None else seed
    table = draw_ellipsoids(cfg, seed)
    prior = render(cfg, table)
    rng = np.random.Generator(np.random.PCG64(seed + 500))
    if cfg_name == "c1":
        follow = prior
    elif cfg_name == "c2":
        centre = rng.uniform(-0.25, 0.25, 3) * cfg.n * cfg.voxel
        follow = add_sphere(cfg, prior, centre, rng.uniform(3.0, 8.0), 0.01)
    elif cfg_name in ("c3", "c5"):
        tip, d = needle_pose(cfg, seed + 700)
        tip = tip + 5.0 * followup_step * d
        follow = add_cylinder(cfg, prior, tip, d, 60.0, 1.0, 0.2)
    else:
        grown = table.copy()
        grown[0, 1:4] *= 1.15
        follow = render(cfg, grown)
    return cfg, prior, follow


def noise_seed(cfg_name: str, followup_step: int = 0) -> int:
    """Poisson seed of a follow-up scan: 1000 + config id (+ 10 * step for c5)."""
    return 1000 + int(cfg_name[1]) + 10 * followup_step


def scan_inputs(cfg_name: str, followup_step: int = 0, prior_iters: int = 20, device: int = 0,
                n_followup_views: int | None = None):
    """The inputs of a BASELINE config's follow-up solve, made on the GPU.

    * prior image: ``prior_iters``-iteration CGLS (``cgls_recon``) of a
      noiseless ``prior_views`` scan of the prior phantom (SURVEY §8d pins);
    * follow-up readings b: forward projection of the follow-up phantom at
      ``followup_views`` (or ``n_followup_views``) angles, Poisson noise at the
      config's I0, seed ``noise_seed``.
    Returns a dict of host float32 arrays in the reference layouts (x-fastest
    volumes, u-fastest projections) plus the package grid / geometries, so the
    identical values can be fed to the GPU solver and to the CPU reference."""
    import torch
    from . import ConeBeamGeometry, ConeBeamProjector, GridSpec, ProjectionSet, cgls_recon
    cfg = CONFIGS[cfg_name]
    dev = torch.device("cuda", device)
    grid = GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    nf = n_followup_views or cfg.followup_views
    geom_p = ConeBeamGeometry(DSO, DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                              angles(cfg.prior_views))
    geom_f = ConeBeamGeometry(DSO, DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch, angles(nf))
    _, prior, follow = study(cfg_name, followup_step=followup_step)
    Ap = ConeBeamProjector(grid, geom_p, device=device)
    xp = Ap.volume_to_native(torch.from_numpy(prior).to(dev))
    prior_rec = cgls_recon(ProjectionSet(geom_p, Ap.apply(xp)), grid, prior_iters, projector=Ap)
    prior_rec = Ap.volume_from_native(prior_rec.volume).cpu().numpy()
    del Ap, xp
    Af = ConeBeamProjector(grid, geom_f, device=device)
    xf = Af.volume_to_native(torch.from_numpy(follow).to(dev))
    pf = Af.proj_from_native(Af.apply(xf)).cpu().numpy()
    b = poisson_log(pf, cfg.i0, seed=noise_seed(cfg_name, followup_step))
    torch.cuda.synchronize(dev)
    return dict(cfg=cfg, grid=grid, geom=geom_f, projector=Af, prior_phantom=prior,
                follow=follow, prior=prior_rec.astype(np.float32), b=b)
