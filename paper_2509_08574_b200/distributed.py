"""Multi-process (one process per GPU) IRN / CGLS solves.

Angle-sharded data parallelism: rank r holds the projection angles r::world
(`shard.angle_indices`) and its readings; the volume-domain CGLS state is
replicated.  Each iteration runs the forward and the adjoint over the local
angles only and sums, over the ranks, the partial adjoint volume and the
projection-domain reductions (||A p||^2, ||r0||^2, the objective's data term)
— NCCL all-reduces over NVLink when torch.distributed runs the nccl backend.
The regulariser terms are computed redundantly (identical on every rank).
The collective is injected through the C ABI hook `kct_set_allreduce`
(include/kct.h); the library itself stays free of any communication runtime.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import (ConeBeamProjector, ProjectionSet, ReconReport, _check, cgls_recon, irn_piccs,
               irn_piple, irn_tv, load_library, shard)

_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)


class _DeviceBuffer:
    """Zero-copy view of a raw device pointer (CUDA array interface)."""

    def __init__(self, ptr: int, count: int, dtype: int):
        self.__cuda_array_interface__ = {"shape": (int(count),),
                                         "typestr": "<f4" if dtype == 0 else "<f8",
                                         "data": (int(ptr), False), "version": 3}


def install_allreduce(projector: ConeBeamProjector, group=None) -> None:
    """Put `projector` in angle-sharded mode, summing over `group` (torch.distributed)."""
    import torch
    import torch.distributed as dist
    lib = load_library()
    device = torch.device("cuda", torch.cuda.current_device())

    def hook(ctx, buf, count, dtype, stream):
        try:
            t = torch.as_tensor(_DeviceBuffer(buf, count, dtype), device=device)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception:  # surfaced as KCT_ERR_CUDA by the library
            return 1

    cb = _HOOK(hook)
    projector._allreduce_hook = cb  # keep the trampoline alive with the handle
    lib.kct_set_allreduce.argtypes = [C.c_void_p, _HOOK, C.c_void_p]
    lib.kct_set_allreduce.restype = C.c_int
    _check(lib.kct_set_allreduce(projector.handle, cb, None))


def shard_projections(proj: ProjectionSet, world: int, rank: int) -> ProjectionSet:
    """This rank's angles r::world of a full projection set (host arrays)."""
    g = proj.geometry
    idx = shard.angle_indices(g.n_angles(), world, rank)
    data = np.asarray(proj.data).reshape(g.n_angles(), -1)[idx].reshape(-1)
    return ProjectionSet(shard.shard_geometry(g, world, rank), np.ascontiguousarray(data))


def sharded_projector(proj_local: ProjectionSet, grid, group=None, device=None):
    A = ConeBeamProjector(grid, proj_local.geometry, device)
    install_allreduce(A, group)
    return A


def irn_piccs_sharded(proj_local, grid, prior, params=None, opts=None, group=None,
                      layout=None) -> ReconReport:
    """irn_piccs (recon.hpp:267-270) with this rank's angles `proj_local`."""
    A = sharded_projector(proj_local, grid, group)
    return irn_piccs(proj_local, grid, prior, params, opts, projector=A, layout=layout)


def irn_tv_sharded(proj_local, grid, params=None, opts=None, group=None, layout=None):
    A = sharded_projector(proj_local, grid, group)
    return irn_tv(proj_local, grid, params, opts, projector=A, layout=layout)


def irn_piple_sharded(proj_local, grid, prior, params=None, opts=None, group=None, layout=None):
    A = sharded_projector(proj_local, grid, group)
    return irn_piple(proj_local, grid, prior, params, opts, projector=A, layout=layout)


def cgls_recon_sharded(proj_local, grid, iters, opts=None, tolerance=0.0, group=None,
                       layout=None):
    A = sharded_projector(proj_local, grid, group)
    return cgls_recon(proj_local, grid, iters, opts, tolerance, projector=A, layout=layout)
