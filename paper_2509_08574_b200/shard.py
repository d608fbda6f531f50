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


def shard_geometry(geom: ConeBeamGeometry, world: int, rank: int) -> ConeBeamGeometry:
    idx = angle_indices(geom.n_angles(), world, rank)
    return ConeBeamGeometry(geom.dso, geom.dsd, geom.nu, geom.nv, geom.pu, geom.pv,
                            geom.angles[idx], geom.offset_u, geom.offset_v)


def slab_grid(grid: GridSpec, world: int, rank: int, axis: str = "z") -> GridSpec:
    """The grid of `rank`'s slab along `axis` ("z": contiguous in the
    reference layout; "y": contiguous in the native z-fastest layout)."""
    ax = {"x": 0, "y": 1, "z": 2}[axis]
    a0, a1 = slab_range(grid.dims[ax], world, rank)
    if a1 <= a0:
        raise ValueError("more ranks than slabs")
    dims = list(grid.dims)
    origin = list(grid.origin)
    dims[ax] = a1 - a0
    origin[ax] = grid.origin[ax] + a0 * grid.spacing[ax]
    return GridSpec(tuple(dims), grid.spacing, tuple(origin))
