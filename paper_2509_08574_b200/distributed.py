"""Multi-process (one process per GPU) IRN / CGLS solves.

Angle-sharded data parallelism: rank r holds the projection angles r::world
(`shard.angle_indices`) and its readings; the volume-domain CGLS state is
replicated.  Each iteration runs the forward and the adjoint over the local
angles only and sums, over the ranks, the partial adjoint volume and the
projection-domain reductions (||A p||^2, ||r0||^2, the objective's data term)
— NCCL all-reduces over NVLink when torch.distributed runs the nccl backend.
The regulariser terms are computed redundantly (identical on every rank).
The collectives reach the solver through the C ABI hooks `kct_set_allreduce`
/ `kct_set_slab` (include/kct.h).  Under torch's nccl backend they are served
by the library's own NCCL communicator (`NativeComm`, `kct_comm_*`: NCCL bound
at run time, collectives enqueued on the solver's stream without a Python
trampoline); under gloo (the CPU-side multi-rank tests) or with
KCT_NATIVE_COMM=0 by torch.distributed callbacks.

y-slab-sharded mode (SURVEY §8e's volume-partitioned variant, `*_slab`):
rank r holds the y planes [j0, j1) of every volume vector (one halo plane on
each side, exchanged through the `kct_set_slab` hook) and all projections;
each iteration sums the partial forward projections (N floats) and the
volume-domain reductions over the ranks.  Per iteration it moves N floats +
4 halo planes instead of M floats, and the regulariser stencils are split
across the ranks instead of computed redundantly — the better partition when
M > N (c4: 134 M voxels, 53 M rays).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import (ConeBeamProjector, ProjectionSet, ReconReport, _check, cgls_recon, irn_piccs,
               irn_piple, irn_tv, load_library, shard)

_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
_HALO = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                    C.c_size_t, C.c_void_p)


class _DeviceBuffer:
    """Zero-copy view of a raw device pointer (CUDA array interface)."""

    def __init__(self, ptr: int, count: int, dtype: int):
        self.__cuda_array_interface__ = {"shape": (int(count),),
                                         "typestr": "<f4" if dtype == 0 else "<f8",
                                         "data": (int(ptr), False), "version": 3}


def _on_stream(stream, device):
    """Context making the library's CUDA stream (a raw handle; None / 0: the
    legacy default stream, which is torch's default stream) torch's current
    stream for a hook's collectives, so they are ordered after the kernels that
    produced the buffer and before the library's next kernels, whatever stream
    the caller has made current."""
    import torch
    if not stream:
        return torch.cuda.stream(torch.cuda.default_stream(device))
    return torch.cuda.stream(torch.cuda.ExternalStream(stream, device=device))


class NativeComm:
    """The library's own NCCL communicator (`kct_comm_*`, include/kct.h): the
    solver's sums and halo exchanges become ncclAllReduce / grouped ncclSend +
    ncclRecv enqueued on the solver's stream by the library itself — no Python
    trampoline and no host synchronisation per collective.  Join with an
    explicit (rank, world, id) or bootstrap over a torch.distributed group
    (`NativeComm.from_group`: rank 0's unique id is broadcast as an object)."""

    def __init__(self, rank: int, world: int, uid: bytes, device: int | None = None):
        lib = load_library()
        if len(uid) != ID_BYTES:
            raise ValueError(f"unique id must be {ID_BYTES} bytes")
        if device is None:  # torch's current device, named explicitly
            import torch
            device = torch.cuda.current_device()
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), ID_BYTES)
        _check(lib.kct_comm_create(int(rank), int(world), buf, int(device), C.byref(h)))
        self.handle, self.rank, self.world = h, int(rank), int(world)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(ID_BYTES)
        _check(load_library().kct_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_group(cls, group=None) -> "NativeComm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0 if group is None else dist.get_global_rank(group, 0),
                                   group=group)
        return cls(rank, world, box[0])

    def all_reduce(self, tensor, op: str = "sum", stream=None) -> None:
        """In-place sum / max of a contiguous float32 / float64 CUDA tensor."""
        import torch
        dt = {torch.float32: 0, torch.float64: 1}[tensor.dtype]
        assert tensor.is_cuda and tensor.is_contiguous()
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        _check(load_library().kct_comm_allreduce(self.handle, tensor.data_ptr(), tensor.numel(), dt,
                                                 {"sum": 0, "max": 1}[op], s))

    def close(self) -> None:
        if self.handle:
            load_library().kct_comm_destroy(self.handle)
            self.handle = None


ID_BYTES = 128  # KCT_COMM_ID_BYTES
_native_comms: dict = {}


def native_comm(group=None):
    """The cached NativeComm of `group`, or None when the solves should go
    through the torch.distributed hooks: any backend but nccl (the gloo tests),
    or KCT_NATIVE_COMM=0."""
    import os

    import torch.distributed as dist
    if os.environ.get("KCT_NATIVE_COMM", "1") == "0" or dist.get_backend(group) != "nccl":
        return None
    key = id(group) if group is not None else None
    if key not in _native_comms:
        _native_comms[key] = NativeComm.from_group(group)
    return _native_comms[key]


def install_allreduce(projector: ConeBeamProjector, group=None, comm=None) -> None:
    """Put `projector` in angle-sharded mode, summing over `group`: through
    the library's NCCL communicator (`comm`, or the group's `native_comm`) when
    there is one, else through a torch.distributed all-reduce hook."""
    import torch
    import torch.distributed as dist
    lib = load_library()
    comm = comm if comm is not None else native_comm(group)
    if comm is not None:
        _check(lib.kct_use_comm(projector.handle, comm.handle))
        projector._comm = comm  # keep the communicator alive with the handle
        return
    device = torch.device("cuda", torch.cuda.current_device())

    def hook(ctx, buf, count, dtype, stream):
        try:
            t = torch.as_tensor(_DeviceBuffer(buf, count, dtype), device=device)
            # stream-ordered with the library's stream (NCCL waits for the
            # kernels that produced `buf`, the library's next kernels wait
            # for the sum)
            with _on_stream(stream, device):
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


# ---------------------------------------------------------------------------
# y-slab-sharded solves
# ---------------------------------------------------------------------------
def install_slab(projector: ConeBeamProjector, rank: int, world: int, j0: int, ny_global: int,
                 group=None, comm=None) -> None:
    """Put `projector` (built on this rank's y-slab grid) in slab mode: the
    all-reduce hook plus a neighbour exchange of boundary y planes (P2P
    send / recv with ranks r - 1 and r + 1) — both by the library's NCCL
    communicator when there is one (`comm` / `native_comm(group)`), else by
    torch.distributed hooks (CPU staging under gloo)."""
    import torch
    import torch.distributed as dist
    lib = load_library()
    comm = comm if comm is not None else native_comm(group)
    if comm is not None:
        if (comm.rank, comm.world) != (rank, world):
            raise ValueError("communicator rank / world differ from the slab's")
        _check(lib.kct_use_comm_slab(projector.handle, comm.handle, j0, ny_global))
        projector._comm = comm
        return
    install_allreduce(projector, group)
    device = torch.device("cuda", torch.cuda.current_device())
    cpu = dist.get_backend(group) == "gloo"

    def halo(ctx, lo_plane, hi_plane, lo_halo, hi_halo, count, stream):
        try:
            with _on_stream(stream, device):
                return _halo(lo_plane, hi_plane, lo_halo, hi_halo, count)
        except Exception:  # surfaced as KCT_ERR_CUDA by the library
            return 1

    def peer(r):  # group rank -> global rank (P2P ops address global ranks)
        return r if group is None else dist.get_global_rank(group, r)

    def _halo(lo_plane, hi_plane, lo_halo, hi_halo, count):
        """Neighbour exchange: send the first / last interior plane to rank - 1 /
        rank + 1 and receive theirs into the halos (P2P, O(1) traffic per rank)."""
        try:
            ops, recv = [], []
            buf = lambda p: torch.as_tensor(_DeviceBuffer(p, count, 0), device=device)  # noqa: E731
            for nb, plane, halo in ((rank - 1, lo_plane, lo_halo), (rank + 1, hi_plane, hi_halo)):
                if not 0 <= nb < world:
                    continue
                send = buf(plane)
                dst = buf(halo)
                if cpu:
                    send, tmp = send.cpu(), torch.empty(count, dtype=torch.float32)
                else:
                    tmp = dst
                ops.append(dist.P2POp(dist.isend, send, peer(nb), group))
                ops.append(dist.P2POp(dist.irecv, tmp, peer(nb), group))
                recv.append((dst, tmp))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for dst, tmp in recv:
                if tmp is not dst:
                    dst.copy_(tmp)
            return 0
        except Exception:  # surfaced as KCT_ERR_CUDA by the library
            return 1

    cb = _HALO(halo)
    projector._halo_hook = cb
    lib.kct_set_slab.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _HALO, C.c_void_p]
    lib.kct_set_slab.restype = C.c_int
    _check(lib.kct_set_slab(projector.handle, rank, world, j0, ny_global, cb, None))


def slab_bounds(grid, geometry, world: int) -> list:
    """y-slab boundaries of all ranks, balanced by backprojection work
    (shard.coverage_weights of a full circle of 64 views with this system's
    source, detector and offsets — not of the scan's own angles, so every scan
    of one system (prior and follow-ups) gets the same slabs); the same on
    every rank."""
    from . import ConeBeamGeometry
    circle = ConeBeamGeometry(geometry.dso, geometry.dsd, geometry.nu, geometry.nv, geometry.pu,
                              geometry.pv, 2.0 * np.pi * np.arange(64) / 64, geometry.offset_u,
                              geometry.offset_v)
    return shard.balanced_bounds(shard.coverage_weights(grid, circle, "y"), world)


def slab_projector(grid, geometry, world: int, rank: int, group=None, device=None):
    """This rank's projector on its (work-balanced) y-slab of `grid`, in slab
    mode; returns (projector, j0, j1)."""
    bounds = slab_bounds(grid, geometry, world)
    j0, j1 = bounds[rank], bounds[rank + 1]
    A = ConeBeamProjector(shard.slab_grid(grid, world, rank, "y", bounds), geometry, device)
    install_slab(A, rank, world, j0, grid.dims[1], group)
    return A, j0, j1


def y_slab(volume, grid, j0: int, j1: int):
    """Planes [j0, j1) of a reference-layout (x-fastest) host volume."""
    nx, ny, nz = grid.dims
    return np.ascontiguousarray(np.asarray(volume).reshape(nz, ny, nx)[:, j0:j1, :].reshape(-1))


def assemble_y_slabs(slabs, grid):
    """Reference-layout volume from the ranks' y-slabs (in rank order)."""
    nx, ny, nz = grid.dims
    return np.concatenate([np.asarray(s).reshape(nz, -1, nx) for s in slabs], axis=1).reshape(-1)


def _slab_opts(opts, grid, j0, j1):
    from . import ReconOptions
    if opts is None:
        return None
    return ReconOptions(
        initial=None if opts.initial is None else y_slab(opts.initial, grid, j0, j1),
        ground_truth=None if opts.ground_truth is None else y_slab(opts.ground_truth, grid, j0, j1))


def irn_piccs_slab(proj, grid, prior, params=None, opts=None, group=None) -> ReconReport:
    """irn_piccs (recon.hpp:267-270), y-slab sharded.  `proj`: all projections
    (host arrays); `prior`, `opts` volumes: full reference-layout host arrays.
    The report's volume is this rank's y-slab (reference layout of the slab
    grid; `assemble_y_slabs` joins them)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    A, j0, j1 = slab_projector(grid, proj.geometry, world, rank, group)
    g = A.grid
    return irn_piccs(proj, g, y_slab(prior, grid, j0, j1), params, _slab_opts(opts, grid, j0, j1),
                     projector=A)


def irn_tv_slab(proj, grid, params=None, opts=None, group=None) -> ReconReport:
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    A, j0, j1 = slab_projector(grid, proj.geometry, world, rank, group)
    g = A.grid
    return irn_tv(proj, g, params, _slab_opts(opts, grid, j0, j1), projector=A)


def cgls_recon_slab(proj, grid, iters, opts=None, tolerance=0.0, group=None) -> ReconReport:
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    A, j0, j1 = slab_projector(grid, proj.geometry, world, rank, group)
    g = A.grid
    return cgls_recon(proj, g, iters, _slab_opts(opts, grid, j0, j1), tolerance, projector=A)
