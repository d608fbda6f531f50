"""Multi-GPU decomposition of the projector pair (one process per GPU).

Rays are independent in A x (projector.hpp:192-193) and voxels are
independent in the voxel-owned A^T y, so the operator pair shards without any
reduction: rank r projects the angle subset r::world of the full volume, and
backprojects its slab of the volume from all angles.  Slab
boundaries are grid planes, so the slab grid's Siddon segments are the full
grid's segments inside the slab: the slab adjoint equals the slab of the full
adjoint (to float rounding of the re-based plane coefficients).  Slabs can be
cut along z (contiguous in the reference layout) or y (contiguous in the
native z-fastest layout, and the brick adjoint keeps full-height bricks: the
bench's choice, tools/shard_time.py).  These helpers are pure host logic (tested on CPU with gloo);
the CUDA operators are built per rank from the returned geometry / grid.
"""
from __future__ import annotations

import numpy as np

from . import ConeBeamGeometry, GridSpec  # noqa: F401  (circular-safe: defined first)


def angle_indices(n_angles: int, world: int, rank: int) -> np.ndarray:
    """Angles owned by `rank` for the forward projection (round robin)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return np.arange(n_angles)[rank::world]


def slab_range(nz: int, world: int, rank: int) -> tuple[int, int]:
    """[z0, z1) slab of `rank` along an axis of nz planes (balanced,
    contiguous, covers 0..nz)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def coverage_weights(grid: GridSpec, geom: ConeBeamGeometry, axis: str = "y") -> np.ndarray:
    """Per plane along `axis` ("x" or "y"): the number of (voxel column, angle)
    pairs whose voxel-column centre projects onto the detector's u extent —
    the backprojection work of the plane (voxels outside the field of view of
    some angles, e.g. the corners of a cube inscribing it, are crossed by
    fewer rays)."""
    nx, ny, _ = grid.dims
    x = grid.origin[0] + (np.arange(nx) + 0.5) * grid.spacing[0]
    y = grid.origin[1] + (np.arange(ny) + 0.5) * grid.spacing[1]
    X, Y = np.meshgrid(x, y, indexing="xy")  # [ny, nx]
    half = 0.5 * geom.nu * geom.pu
    w = np.zeros((ny, nx))
    for t in np.asarray(geom.angles, dtype=np.float64):
        c, s = np.cos(t), np.sin(t)
        den = geom.dso - (X * c + Y * s)
        u = geom.dsd * (-X * s + Y * c) / np.where(den > 0, den, np.inf) - geom.offset_u
        w += (np.abs(u) <= half) & (den > 0)
    return w.sum(axis=1) if axis == "y" else w.sum(axis=0)


def balanced_bounds(weights: np.ndarray, world: int, quantum: int = 4) -> list[int]:
    """world + 1 plane boundaries splitting `weights` into contiguous slabs of
    about equal total weight, interior boundaries on multiples of `quantum`
    (whole 4-plane adjoint bricks) when that leaves every slab non-empty."""
    n = len(weights)
    if world > n:
        raise ValueError("more ranks than slabs")
    cum = np.concatenate([[0.0], np.cumsum(np.maximum(weights, 0) + 1e-9)])
    bounds = [0]
    for r in range(1, world):
        j = int(np.searchsorted(cum, cum[-1] * r / world))
        q = int(round(j / quantum)) * quantum if n >= quantum * world else j
        bounds.append(min(max(q, bounds[-1] + 1), n - (world - r)))
    bounds.append(n)
    return bounds


def shard_geometry(geom: ConeBeamGeometry, world: int, rank: int) -> ConeBeamGeometry:
    idx = angle_indices(geom.n_angles(), world, rank)
    return ConeBeamGeometry(geom.dso, geom.dsd, geom.nu, geom.nv, geom.pu, geom.pv,
                            geom.angles[idx], geom.offset_u, geom.offset_v)


def slab_grid(grid: GridSpec, world: int, rank: int, axis: str = "z",
              bounds: list[int] | None = None) -> GridSpec:
    """The grid of `rank`'s slab along `axis` ("z": contiguous in the
    reference layout; "y": contiguous in the native z-fastest layout);
    `bounds` (world + 1 plane indices, e.g. balanced_bounds) overrides the
    even split."""
    ax = {"x": 0, "y": 1, "z": 2}[axis]
    a0, a1 = (bounds[rank], bounds[rank + 1]) if bounds else slab_range(grid.dims[ax], world, rank)
    if a1 <= a0:
        raise ValueError("more ranks than slabs")
    dims = list(grid.dims)
    origin = list(grid.origin)
    dims[ax] = a1 - a0
    origin[ax] = grid.origin[ax] + a0 * grid.spacing[ax]
    return GridSpec(tuple(dims), grid.spacing, tuple(origin))
