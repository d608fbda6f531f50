"""B200-native PICCS-Krylov CBCT core (drop-in for the kryct hot path).

Python mirror of the reference's C++ solver API over the C ABI of
``libkct.so`` (``include/kct.h``).  Names, argument meaning and errors follow
the reference (paths relative to /root/reference/proj/include/kryct/):

* ``GridSpec`` (types.hpp:56-80), ``ConeBeamGeometry`` (types.hpp:138-161),
  ``ProjectionSet`` (types.hpp:165-187)
* ``ConeBeamProjector`` with ``apply`` / ``apply_adjoint`` (projector.hpp:264-291)
* ``cgls_recon`` (recon.hpp:312-315), ``irn_tv`` / ``irn_piple`` / ``irn_piccs``
  (recon.hpp:252-270), ``RegularizationParams`` (recon.hpp:37-55),
  ``ReconOptions`` (recon.hpp:68-72), ``ReconReport`` (recon.hpp:74-83)
* ``ConfigError`` / ``SolverError`` (types.hpp:16-26)

Arrays are numpy (host) or torch CUDA tensors (device).  Host arrays use the
reference layouts (volumes x-fastest, projections u-fastest).  Device tensors
default to the native layouts (volume z-fastest, projections v-fastest; see
``kct.h``); pass ``layout="reference"`` to use the reference's.  There is no
CPU fallback: every call runs the CUDA library, and loading fails loudly when
it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _build

__all__ = [
    "ConfigError", "SolverError", "KctError", "GridSpec", "ConeBeamGeometry", "ProjectionSet",
    "ConeBeamProjector", "RegularizationParams", "ReconOptions", "ReconReport", "cgls_recon",
    "irn_tv", "irn_piple", "irn_piccs", "fdk", "resolve_tau", "uniform_angles", "load_library",
    "subsample_indices", "subsample_angles", "LIB_PATH", "shard",
    "DiffOperator", "IdentityMap", "DiagonalMap", "ComposedMap", "compose", "ScaledBlock",
    "StackedMap", "stack_maps", "KrylovConfig", "SolveTrace", "SolveResult", "cgls",
]

LIB_PATH = os.environ.get("KCT_LIB_PATH", _build.LIB)
MEM_HOST, MEM_DEVICE = 0, 1
LAYOUT_REFERENCE, LAYOUT_NATIVE = 0, 1
KIND_TV, KIND_PIPLE, KIND_PICCS = 0, 1, 2


class KctError(RuntimeError):
    code = 1


class ConfigError(KctError):
    """types.hpp:16-19."""
    code = 2


class SolverError(KctError):
    """types.hpp:23-26."""
    code = 3


class CudaError(KctError):
    code = 4


_ERRORS = {2: ConfigError, 3: SolverError, 4: CudaError}


class _Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("sx", C.c_double), ("sy", C.c_double), ("sz", C.c_double),
                ("ox", C.c_double), ("oy", C.c_double), ("oz", C.c_double)]


class _Geom(C.Structure):
    _fields_ = [("dso", C.c_double), ("dsd", C.c_double), ("nu", C.c_int), ("nv", C.c_int),
                ("pu", C.c_double), ("pv", C.c_double),
                ("offset_u", C.c_double), ("offset_v", C.c_double),
                ("n_angles", C.c_int), ("angles", C.POINTER(C.c_double))]


class _Reg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("tau", C.c_double),
                ("outer_iters", C.c_size_t), ("inner_iters", C.c_size_t),
                ("inner_tolerance", C.c_double), ("warm_start", C.c_int)]


class _StackBlock(C.Structure):
    _fields_ = [("map", C.c_int), ("scale", C.c_double), ("weights", C.c_void_p)]


class _Report(C.Structure):
    _fields_ = [("objective_history", C.POINTER(C.c_double)), ("objective_count", C.c_size_t),
                ("residual_history", C.POINTER(C.c_double)), ("residual_count", C.c_size_t),
                ("error_history", C.POINTER(C.c_double)), ("error_count", C.c_size_t),
                ("outer_boundaries", C.POINTER(C.c_uint64)), ("outer_count", C.c_size_t),
                ("outer_seconds", C.POINTER(C.c_double)),
                ("solve_seconds", C.c_double), ("tau", C.c_double),
                ("converged", C.c_int), ("breakdown", C.c_int),
                ("wall_times", C.POINTER(C.c_double)), ("wall_count", C.c_size_t)]


# kct_iterate_hook(ctx, iteration, x, m)
_ITER_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.POINTER(C.c_float), C.c_size_t)

# Every symbol include/kct.h declares, with its ctypes signature.
_P = C.c_void_p
_SIGS = {
    "kct_last_error": ([], C.c_char_p),
    "kct_abi_version": ([], C.c_int),
    "kct_launch_count": ([], C.c_ulonglong),
    "kct_host_alloc": ([C.c_size_t, C.POINTER(_P)], C.c_int),
    "kct_host_free": ([_P], C.c_int),
    "kct_set_slab": ([_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),  # typed by distributed.install_slab
    "kct_projector_create": ([C.POINTER(_Grid), C.POINTER(_Geom), C.c_int, C.POINTER(_P)], C.c_int),
    "kct_projector_destroy": ([_P], C.c_int),
    "kct_projector_sizes": ([_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)], C.c_int),
    "kct_forward": ([_P, _P, _P, C.c_int, C.c_int, _P], C.c_int),
    "kct_adjoint": ([_P, _P, _P, C.c_int, C.c_int, _P], C.c_int),
    "kct_forward_f64": ([_P, _P, _P], C.c_int),
    "kct_adjoint_f64": ([_P, _P, _P], C.c_int),
    "kct_count_nnz": ([_P, C.POINTER(C.c_uint64), _P], C.c_int),
    "kct_projector_info": ([_P, C.c_char_p, C.POINTER(C.c_double)], C.c_int),
    "kct_volume_to_native": ([_P, _P, _P, _P], C.c_int),
    "kct_volume_from_native": ([_P, _P, _P, _P], C.c_int),
    "kct_proj_to_native": ([_P, _P, _P, _P], C.c_int),
    "kct_proj_from_native": ([_P, _P, _P, _P], C.c_int),
    "kct_cgls_recon": ([_P, _P, C.c_size_t, _P, _P, C.c_double, _P, C.POINTER(_Report), C.c_int,
                        C.c_int, _P], C.c_int),
    "kct_cgls_stack": ([_P, C.POINTER(_StackBlock), C.c_size_t, _P, _P, C.c_size_t, C.c_double, _P,
                        C.POINTER(_Report), C.c_int, C.c_int, _P], C.c_int),
    "kct_irn": ([_P, C.c_int, _P, _P, _P, _P, C.POINTER(_Reg), _P, C.POINTER(_Report), C.c_int,
                 C.c_int, _P], C.c_int),
    "kct_irn_piccs": ([_P, _P, _P, _P, _P, C.POINTER(_Reg), _P, C.POINTER(_Report), C.c_int,
                       C.c_int, _P], C.c_int),
    "kct_resolve_tau": ([C.c_double, _P, C.c_size_t], C.c_double),
    "kct_set_allreduce": ([_P, _P, _P], C.c_int),  # typed by distributed.install_allreduce
    "kct_comm_unique_id": ([_P], C.c_int),
    "kct_comm_create": ([C.c_int, C.c_int, _P, C.c_int, C.POINTER(_P)], C.c_int),
    "kct_comm_destroy": ([_P], C.c_int),
    "kct_comm_rank": ([_P], C.c_int),
    "kct_comm_world": ([_P], C.c_int),
    "kct_comm_allreduce": ([_P, _P, C.c_size_t, C.c_int, C.c_int, _P], C.c_int),
    "kct_comm_allreduce_host": ([_P, _P, C.c_size_t, C.c_int, C.c_int], C.c_int),
    "kct_use_comm": ([_P, _P], C.c_int),
    "kct_use_comm_slab": ([_P, _P, C.c_int, C.c_int], C.c_int),
    "kct_slab_bounds": ([C.POINTER(_Grid), C.POINTER(_Geom), C.c_int, C.POINTER(C.c_int)], C.c_int),
    "kct_fdk": ([_P, _P, _P, C.c_int, C.c_int, _P], C.c_int),
    "kct_set_option": ([_P, C.c_char_p, C.c_double], C.c_int),
    "kct_set_iterate_hook": ([_P, _ITER_HOOK, _P], C.c_int),
}

_lib = None


def load_library(build: bool = True):
    """Load (building in-tree first if stale) the CUDA library.  Raises if absent."""
    global _lib
    if _lib is None:
        if build and LIB_PATH == _build.LIB:
            try:
                _build.build()
            except Exception:  # no nvcc on this host: the prebuilt .so must exist
                if not os.path.exists(LIB_PATH):
                    raise
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"CUDA library not built: {LIB_PATH}")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def launch_count() -> int:
    """Kernels the CUDA library has launched in this process (kct_launch_count)."""
    return int(load_library().kct_launch_count())


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.kct_last_error().decode()
        raise _ERRORS.get(rc, KctError)(msg)


# ---------------------------------------------------------------------------
# domain types
# ---------------------------------------------------------------------------
@dataclass
class GridSpec:
    """GridSpec (types.hpp:56-80): dims, spacing [mm], origin (min corner)."""
    dims: tuple
    spacing: tuple = (1.0, 1.0, 1.0)
    origin: tuple | None = None

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        self.spacing = tuple(float(s) for s in self.spacing)
        if self.origin is None:  # GridSpec::centered (types.hpp:62-65)
            self.origin = tuple(-0.5 * d * s for d, s in zip(self.dims, self.spacing))
        self.origin = tuple(float(o) for o in self.origin)

    @staticmethod
    def centered(dims, spacing=(1.0, 1.0, 1.0)) -> "GridSpec":
        return GridSpec(dims, spacing)

    def count(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def _c(self) -> _Grid:
        return _Grid(*self.dims, *self.spacing, *self.origin)


@dataclass
class ConeBeamGeometry:
    """ConeBeamGeometry (types.hpp:138-161); detector = (nu, nv, pu, pv)."""
    dso: float
    dsd: float
    nu: int
    nv: int
    pu: float
    pv: float
    angles: np.ndarray
    offset_u: float = 0.0
    offset_v: float = 0.0

    def __post_init__(self):
        self.angles = np.ascontiguousarray(np.asarray(self.angles, dtype=np.float64).reshape(-1))

    def n_angles(self) -> int:
        return int(self.angles.size)

    def rays_per_angle(self) -> int:
        return self.nu * self.nv

    def ray_count(self) -> int:
        return self.rays_per_angle() * self.n_angles()

    def _c(self) -> _Geom:
        return _Geom(self.dso, self.dsd, self.nu, self.nv, self.pu, self.pv, self.offset_u,
                     self.offset_v, self.n_angles(),
                     self.angles.ctypes.data_as(C.POINTER(C.c_double)))


@dataclass
class ProjectionSet:
    """ProjectionSet (types.hpp:165-187): geometry + u-fastest readings."""
    geometry: ConeBeamGeometry
    data: object = None

    def __post_init__(self):
        if self.data is None:
            self.data = np.zeros(self.geometry.ray_count(), dtype=np.float32)


def uniform_angles(n: int) -> np.ndarray:
    """experiment.hpp:89-94."""
    return 2.0 * np.pi * np.arange(n, dtype=np.float64) / float(n)


def subsample_indices(n: int, n_keep: int) -> list:
    """projector.hpp:300-305."""
    if n_keep < 1 or n_keep > n:
        raise ConfigError("subsample: need 1 <= n_keep <= n_angles")
    return [i * n // n_keep for i in range(n_keep)]


def subsample_angles(full: ProjectionSet, n_keep: int) -> ProjectionSet:
    """projector.hpp:307-318 (host arrays)."""
    keep = subsample_indices(full.geometry.n_angles(), n_keep)
    g = full.geometry
    geom = ConeBeamGeometry(g.dso, g.dsd, g.nu, g.nv, g.pu, g.pv, g.angles[keep], g.offset_u,
                            g.offset_v)
    per = g.rays_per_angle()
    data = np.asarray(full.data).reshape(-1, per)[keep].reshape(-1)
    return ProjectionSet(geom, np.ascontiguousarray(data))


@dataclass
class RegularizationParams:
    """recon.hpp:37-55."""
    alpha: float = 0.05
    lambda_: float = -1.0
    tau: float = 0.0
    outer_iters: int = 4
    inner_iters: int = 25
    inner_tolerance: float = 0.0
    warm_start: bool = True

    def resolved_lambda(self) -> float:
        return self.alpha if self.lambda_ < 0.0 else self.lambda_

    def _c(self) -> _Reg:
        return _Reg(self.alpha, self.lambda_, self.tau, self.outer_iters, self.inner_iters,
                    self.inner_tolerance, 1 if self.warm_start else 0)


@dataclass
class ReconOptions:
    """recon.hpp:68-72.  ``hook(iteration, x)`` is the reference's IterateHook
    (krylov.hpp:22-23): called after every inner iteration (1-based, across
    outer cycles) with a float32 copy of the iterate in the reference layout.
    It is an opt-in device->host copy per iteration (kct_set_iterate_hook,
    overlapped with the solve on a side stream); the error history against
    ``ground_truth`` is computed on the device and needs no hook."""
    initial: object = None
    ground_truth: object = None
    hook: object = None


@dataclass
class ReconReport:
    """recon.hpp:74-83 (+ the resolved tau and the CGLS breakdown flag)."""
    volume: object
    objective_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    error_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    outer_boundaries: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    outer_seconds: np.ndarray = field(default_factory=lambda: np.zeros(0))
    solve_seconds: float = 0.0
    converged: bool = False
    tau: float = 0.0
    breakdown: bool = False
    wall_times: np.ndarray = field(default_factory=lambda: np.zeros(0))  # SolveTrace (krylov.hpp:40)


# ---------------------------------------------------------------------------
# array plumbing: numpy (host) or torch CUDA tensors (device)
# ---------------------------------------------------------------------------
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class _Arg:
    """A float32 buffer handed to the C ABI."""

    def __init__(self, a, n, name):
        self.keep = None
        if _is_torch(a):
            import torch
            if not a.is_cuda:
                a = a.detach().cpu().numpy()
            else:
                if a.dtype != torch.float32 or not a.is_contiguous():
                    raise ConfigError(f"{name}: device tensors must be contiguous float32")
                if a.numel() != n:
                    raise ConfigError(f"{name}: expected {n} values, got {a.numel()}")
                self.mem, self.ptr, self.keep = MEM_DEVICE, a.data_ptr(), a
                return
        arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
        if arr.size != n:
            raise ConfigError(f"{name}: expected {n} values, got {arr.size}")
        self.mem, self.ptr, self.keep = MEM_HOST, arr.ctypes.data, arr


def _stream_of(mem, device_index):
    if mem != MEM_DEVICE:
        return None
    import torch
    return torch.cuda.current_stream(device_index).cuda_stream


def _layout_code(layout, mem) -> int:
    if layout is None:
        return LAYOUT_REFERENCE if mem == MEM_HOST else LAYOUT_NATIVE
    return {"reference": LAYOUT_REFERENCE, "native": LAYOUT_NATIVE}[layout]


def _alloc_like(arg: _Arg, n: int):
    if arg.mem == MEM_DEVICE:
        import torch
        return torch.empty(n, dtype=torch.float32, device=arg.keep.device)
    return np.empty(n, dtype=np.float32)


def _ptr(out):
    return out.data_ptr() if _is_torch(out) else out.ctypes.data


def _check_out(out, like: "_Arg", n: int, name: str = "out"):
    """A caller-supplied output buffer must be what the C ABI will write: n
    contiguous float32 values in the same memory kind (and device) as the
    input — the library writes through the raw pointer (the reference checks
    the output span's size, linear_map.hpp:52-57)."""
    if _is_torch(out):
        import torch
        if not out.is_cuda:
            raise ConfigError(f"{name}: CPU tensors are not accepted as outputs (use numpy)")
        if like.mem != MEM_DEVICE:
            raise ConfigError(f"{name}: device output for host input")
        if out.device != like.keep.device:
            raise ConfigError(f"{name}: output on {out.device}, input on {like.keep.device}")
        if out.dtype != torch.float32 or not out.is_contiguous():
            raise ConfigError(f"{name}: must be a contiguous float32 tensor")
        if out.numel() != n:
            raise ConfigError(f"{name}: expected {n} values, got {out.numel()}")
        return out
    if not isinstance(out, np.ndarray):
        raise ConfigError(f"{name}: expected a numpy array or a CUDA tensor")
    if like.mem != MEM_HOST:
        raise ConfigError(f"{name}: host output for device input")
    if out.dtype != np.float32 or not out.flags.c_contiguous or not out.flags.writeable:
        raise ConfigError(f"{name}: must be a writeable C-contiguous float32 array")
    if out.size != n:
        raise ConfigError(f"{name}: expected {n} values, got {out.size}")
    return out


# ---------------------------------------------------------------------------
# operator
# ---------------------------------------------------------------------------
class ConeBeamProjector:
    """ConeBeamProjector (projector.hpp:264-291) on one CUDA device."""

    def __init__(self, grid: GridSpec, geometry: ConeBeamGeometry, device: int | None = None):
        lib = load_library()
        self.grid, self.geometry = grid, geometry
        self._h = C.c_void_p()
        g, ge = grid._c(), geometry._c()
        _check(lib.kct_projector_create(C.byref(g), C.byref(ge), -1 if device is None else device,
                                        C.byref(self._h)))
        self.device = device

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.kct_projector_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def domain_size(self) -> int:
        return self.grid.count()

    def range_size(self) -> int:
        return self.geometry.ray_count()

    def _dev_index(self, arg):
        return arg.keep.device.index if arg.mem == MEM_DEVICE else None

    def apply(self, x, out=None, layout=None):
        """y = A x (project_forward, projector.hpp:194-204)."""
        xa = _Arg(x, self.domain_size(), "forward: volume")
        y = _check_out(out, xa, self.range_size()) if out is not None else _alloc_like(xa, self.range_size())
        _check(_lib.kct_forward(self._h, xa.ptr, _ptr(y), xa.mem, _layout_code(layout, xa.mem),
                                _stream_of(xa.mem, self._dev_index(xa))))
        return y

    def apply_adjoint(self, y, out=None, layout=None):
        """x = A^T y (project_adjoint, projector.hpp:226-261)."""
        ya = _Arg(y, self.range_size(), "adjoint: projections")
        x = _check_out(out, ya, self.domain_size()) if out is not None else _alloc_like(ya, self.domain_size())
        _check(_lib.kct_adjoint(self._h, ya.ptr, _ptr(x), ya.mem, _layout_code(layout, ya.mem),
                                _stream_of(ya.mem, self._dev_index(ya))))
        return x

    def fdk(self, proj, out=None, layout=None):
        """FDK reconstruction (fdk.hpp:50-139) of a full-circle scan on this geometry."""
        pa = _Arg(proj, self.range_size(), "fdk: projections")
        x = _check_out(out, pa, self.domain_size()) if out is not None else _alloc_like(pa, self.domain_size())
        _check(_lib.kct_fdk(self._h, pa.ptr, _ptr(x), pa.mem, _layout_code(layout, pa.mem),
                            _stream_of(pa.mem, self._dev_index(pa))))
        return x

    def count_nnz(self) -> int:
        n = C.c_uint64()
        _check(_lib.kct_count_nnz(self._h, C.byref(n), None))
        return int(n.value)

    def set_option(self, key: str, value) -> None:
        """Solver option of this handle (kct_set_option): "solver_restart" = 1
        runs the reference's control flow at every CGLS start (fresh
        r = b - A x and A^T r, krylov.hpp:68-75; fresh A x for each objective)."""
        _check(_lib.kct_set_option(self._h, key.encode(), float(value)))

    def info(self, key: str) -> float:
        """Which code path the handle runs (kct_projector_info): adj_slab,
        adj_bz, adj_groups, fwd_split_z, solver_restart, ..."""
        v = C.c_double()
        _check(_lib.kct_projector_info(self._h, key.encode(), C.byref(v)))
        return v.value

    # layout conversions of device tensors
    def volume_to_native(self, ref, out=None):
        import torch
        a = _Arg(ref, self.domain_size(), "volume_to_native")
        if a.mem != MEM_DEVICE:
            raise ConfigError("volume_to_native: expects a CUDA tensor")
        out = _check_out(out, a, self.domain_size()) if out is not None else torch.empty_like(ref)
        _check(_lib.kct_volume_to_native(self._h, ref.data_ptr(), out.data_ptr(),
                                         torch.cuda.current_stream(ref.device).cuda_stream))
        return out

    def volume_from_native(self, nat, out=None):
        import torch
        a = _Arg(nat, self.domain_size(), "volume_from_native")
        if a.mem != MEM_DEVICE:
            raise ConfigError("volume_from_native: expects a CUDA tensor")
        out = _check_out(out, a, self.domain_size()) if out is not None else torch.empty_like(nat)
        _check(_lib.kct_volume_from_native(self._h, nat.data_ptr(), out.data_ptr(),
                                           torch.cuda.current_stream(nat.device).cuda_stream))
        return out

    def proj_to_native(self, ref, out=None):
        import torch
        a = _Arg(ref, self.range_size(), "proj_to_native")
        if a.mem != MEM_DEVICE:
            raise ConfigError("proj_to_native: expects a CUDA tensor")
        out = _check_out(out, a, self.range_size()) if out is not None else torch.empty_like(ref)
        _check(_lib.kct_proj_to_native(self._h, ref.data_ptr(), out.data_ptr(),
                                       torch.cuda.current_stream(ref.device).cuda_stream))
        return out

    def proj_from_native(self, nat, out=None):
        import torch
        a = _Arg(nat, self.range_size(), "proj_from_native")
        if a.mem != MEM_DEVICE:
            raise ConfigError("proj_from_native: expects a CUDA tensor")
        out = _check_out(out, a, self.range_size()) if out is not None else torch.empty_like(nat)
        _check(_lib.kct_proj_from_native(self._h, nat.data_ptr(), out.data_ptr(),
                                         torch.cuda.current_stream(nat.device).cuda_stream))
        return out


# ---------------------------------------------------------------------------
# solvers
# ---------------------------------------------------------------------------
def _report_buffers(n_obj, n_res, n_outer):
    bufs = dict(obj=np.zeros(max(n_obj, 1)), res=np.zeros(max(n_res, 1)),
                err=np.zeros(max(n_res, 1)), bnd=np.zeros(max(n_outer, 1), dtype=np.uint64),
                sec=np.zeros(max(n_outer, 1)), wall=np.zeros(max(n_res, 1)))
    rep = _Report()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rep.objective_history = dp(bufs["obj"])
    rep.residual_history = dp(bufs["res"])
    rep.error_history = dp(bufs["err"])
    rep.outer_boundaries = bufs["bnd"].ctypes.data_as(C.POINTER(C.c_uint64))
    rep.outer_seconds = dp(bufs["sec"])
    rep.wall_times = dp(bufs["wall"])
    return rep, bufs


def _unpack(rep, bufs, volume) -> ReconReport:
    return ReconReport(volume=volume,
                       objective_history=bufs["obj"][:rep.objective_count].copy(),
                       residual_history=bufs["res"][:rep.residual_count].copy(),
                       error_history=bufs["err"][:rep.error_count].copy(),
                       outer_boundaries=bufs["bnd"][:rep.outer_count].astype(np.int64),
                       outer_seconds=bufs["sec"][:rep.outer_count].copy(),
                       solve_seconds=rep.solve_seconds, converged=bool(rep.converged),
                       tau=rep.tau, breakdown=bool(rep.breakdown),
                       wall_times=bufs["wall"][:rep.wall_count].copy())


class _HookInstall:
    """ReconOptions.hook installed on the handle for one solve (kct_set_iterate_hook)."""

    def __init__(self, A, hook):
        self.A, self.hook, self.cb, self.err = A, hook, None, None

    def __enter__(self):
        if self.hook is not None:
            def tramp(ctx, it, x, m):
                if self.err is not None:
                    return
                try:
                    self.hook(int(it), np.ctypeslib.as_array(x, shape=(int(m),)).copy())
                except BaseException as e:  # re-raised after the solve
                    self.err = e
            self.cb = _ITER_HOOK(tramp)
            _check(_lib.kct_set_iterate_hook(self.A.handle, self.cb, None))
        return self

    def __exit__(self, *exc):
        if self.cb is not None:
            _lib.kct_set_iterate_hook(self.A.handle, _ITER_HOOK(), None)
            self.cb = None
        if self.err is not None and exc[0] is None:
            raise self.err
        return False


def _projector_for(proj: ProjectionSet, grid: GridSpec, projector):
    if projector is not None:
        return projector
    return ConeBeamProjector(grid, proj.geometry)


def _same_mem(args):
    mems = {a.mem for a in args if a is not None}
    if len(mems) > 1:
        raise ConfigError("all arrays must be host arrays or all device tensors")
    return mems.pop() if mems else MEM_HOST


def _out_for(arg: _Arg, m: int, out):
    """The caller's output buffer (e.g. pinned host memory) or a new one."""
    if out is None:
        return _alloc_like(arg, m)
    return _check_out(out, arg, m)


def cgls_recon(proj: ProjectionSet, grid: GridSpec, iters: int, opts: ReconOptions | None = None,
               tolerance: float = 0.0, projector: ConeBeamProjector | None = None,
               layout=None, out=None) -> ReconReport:
    """Unregularised least squares from zero (recon.hpp:312-315).  `out`: an
    optional caller buffer for the volume (same memory kind as the data)."""
    opts = opts or ReconOptions()
    A = _projector_for(proj, grid, projector)
    m, n = A.domain_size(), A.range_size()
    b = _Arg(proj.data, n, "projections")
    x0 = _Arg(opts.initial, m, "initial") if opts.initial is not None else None
    gt = _Arg(opts.ground_truth, m, "ground truth") if opts.ground_truth is not None else None
    mem = _same_mem([b, x0, gt])
    out = _out_for(b, m, out)
    rep, bufs = _report_buffers(iters, iters, 1)
    with _HookInstall(A, opts.hook):
        _check(_lib.kct_cgls_recon(A.handle, b.ptr, int(iters), x0.ptr if x0 else None,
                                   gt.ptr if gt else None, float(tolerance), _ptr(out),
                                   C.byref(rep), mem, _layout_code(layout, mem),
                                   _stream_of(mem, b.keep.device.index if mem == MEM_DEVICE else None)))
    return _unpack(rep, bufs, out)


# ---------------------------------------------------------------------------
# caller-assembled stacks: the LinearMap algebra (linear_map.hpp) as block
# descriptors, solved on the device by kct_cgls_stack
# ---------------------------------------------------------------------------
MAP_PROJECTOR, MAP_DIFF, MAP_IDENTITY = 0, 1, 2


class DiffOperator:
    """DiffOperator (diffreg.hpp:20-81): forward differences [dx; dy; dz], 3M values."""

    def __init__(self, dims):
        self.dims = tuple(int(d) for d in dims)
        if min(self.dims) < 1:
            raise ConfigError("diff operator: dims must be positive")

    def domain_size(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def range_size(self) -> int:
        return 3 * self.domain_size()


class IdentityMap:
    """IdentityMap (linear_map.hpp:59-80)."""

    def __init__(self, n: int):
        self.n = int(n)

    def domain_size(self) -> int:
        return self.n

    def range_size(self) -> int:
        return self.n


class DiagonalMap:
    """DiagonalMap (linear_map.hpp:82-106): multiplication by diag(weights)."""

    def __init__(self, weights):
        self.weights = weights

    def domain_size(self) -> int:
        w = self.weights
        return int(w.numel()) if _is_torch(w) else int(np.asarray(w).size)

    range_size = domain_size


class ComposedMap:
    """ComposedMap (linear_map.hpp:108-150): outer after inner."""

    def __init__(self, outer, inner):
        if outer is None or inner is None:
            raise ConfigError("compose: null operand")
        if outer.domain_size() != inner.range_size():
            raise ConfigError("compose: inner range must match outer domain")
        self.outer, self.inner = outer, inner

    def domain_size(self) -> int:
        return self.inner.domain_size()

    def range_size(self) -> int:
        return self.outer.range_size()


def compose(outer, inner) -> ComposedMap:
    return ComposedMap(outer, inner)


@dataclass
class ScaledBlock:
    """linear_map.hpp:152-157."""
    scale: float = 1.0
    map: object = None


class StackedMap:
    """StackedMap (linear_map.hpp:159-216): [c1 A1; c2 A2; ...] over one domain."""

    def __init__(self, blocks):
        self.blocks = [b if isinstance(b, ScaledBlock) else ScaledBlock(*b) for b in blocks]
        if not self.blocks:
            raise ConfigError("stack: needs at least one block")
        if any(b.map is None for b in self.blocks):
            raise ConfigError("stack: null block")
        self._domain = self.blocks[0].map.domain_size()
        if any(b.map.domain_size() != self._domain for b in self.blocks):
            raise ConfigError("stack: all blocks must share the domain")

    def domain_size(self) -> int:
        return self._domain

    def range_size(self) -> int:
        return sum(b.map.range_size() for b in self.blocks)

    def block_count(self) -> int:
        return len(self.blocks)


def stack_maps(blocks) -> StackedMap:
    return StackedMap(blocks)


@dataclass
class KrylovConfig:
    """krylov.hpp:25-33."""
    max_iters: int = 100
    tolerance: float = 0.0
    hook: object = None


@dataclass
class SolveTrace:
    """krylov.hpp:35-41."""
    iterations: int = 0
    converged: bool = False
    breakdown: bool = False
    residual_norms: np.ndarray = field(default_factory=lambda: np.zeros(0))
    wall_times: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class SolveResult:
    """krylov.hpp:43-46."""
    x: object = None
    trace: SolveTrace = field(default_factory=SolveTrace)


def _flatten_stack(A):
    """A LinearMap expression -> (projector, [(map code, scale, weights | None)]).
    Accepted shapes (what recon.hpp:211-221 assembles, and plain maps): a
    ConeBeamProjector / DiffOperator / IdentityMap, compose(DiagonalMap, one
    of those), or a StackedMap of such blocks with exactly one projector
    handle among them.  Anything else is a ConfigError: there is no CPU path."""
    blocks = A.blocks if isinstance(A, StackedMap) else [ScaledBlock(1.0, A)]
    projector, out = None, []
    for blk in blocks:
        mp, w = blk.map, None
        if isinstance(mp, ComposedMap) and isinstance(mp.outer, DiagonalMap):
            w, mp = mp.outer.weights, mp.inner
        if isinstance(mp, ConeBeamProjector):
            if projector is not None and projector is not mp:
                raise ConfigError("stack: blocks must share one projector handle")
            projector, code = mp, MAP_PROJECTOR
        elif isinstance(mp, DiffOperator):
            code = MAP_DIFF
        elif isinstance(mp, IdentityMap):
            code = MAP_IDENTITY
        else:
            raise ConfigError(f"stack: unsupported block {type(mp).__name__} "
                              "(projector, DiffOperator, IdentityMap, optionally under a DiagonalMap)")
        out.append((code, float(blk.scale), w, mp))
    if projector is None:
        raise ConfigError("stack: needs a ConeBeamProjector block (it owns the device)")
    m = projector.domain_size()
    for code, _, _, mp in out:
        if code == MAP_DIFF and (mp.domain_size() != m or tuple(mp.dims) != tuple(projector.grid.dims)):
            raise ConfigError("stack: DiffOperator dims must match the projector grid")
        if mp.domain_size() != m:
            raise ConfigError("stack: all blocks must share the domain")
    return projector, out


def cgls(A, b, x0=None, cfg: KrylovConfig | None = None, layout=None, out=None) -> SolveResult:
    """cgls (krylov.hpp:59-127) over a caller-assembled stack, device-resident
    (kct_cgls_stack).  `b` is the concatenated right-hand side (block order),
    `x0` the start (None = zeros); numpy arrays or CUDA tensors, all of one kind."""
    cfg = cfg or KrylovConfig()
    P, blocks = _flatten_stack(A)
    m, n = P.domain_size(), P.range_size()
    lens = [n if c == MAP_PROJECTOR else (3 * m if c == MAP_DIFF else m) for c, _, _, _ in blocks]
    if (b.numel() if _is_torch(b) else np.asarray(b).size) != sum(lens):
        raise ConfigError("cgls: rhs size mismatch")
    bb = _Arg(b, sum(lens), "rhs")
    xx = _Arg(x0, m, "x0") if x0 is not None else None
    ws = [_Arg(w, ln, "weights") if w is not None else None for (_, _, w, _), ln in zip(blocks, lens)]
    mem = _same_mem([bb, xx] + ws)
    out = _out_for(bb, m, out)
    arr = (_StackBlock * len(blocks))()
    for i, ((code, scale, _, _), w) in enumerate(zip(blocks, ws)):
        arr[i].map, arr[i].scale, arr[i].weights = code, scale, (w.ptr if w else None)
    iters = int(cfg.max_iters)
    rep, bufs = _report_buffers(1, iters, 1)
    with _HookInstall(P, cfg.hook):
        _check(_lib.kct_cgls_stack(P.handle, arr, len(blocks), bb.ptr, xx.ptr if xx else None, iters,
                                   float(cfg.tolerance), _ptr(out), C.byref(rep), mem,
                                   _layout_code(layout, mem),
                                   _stream_of(mem, bb.keep.device.index if mem == MEM_DEVICE else None)))
    return SolveResult(x=out, trace=SolveTrace(
        iterations=int(rep.residual_count), converged=bool(rep.converged),
        breakdown=bool(rep.breakdown), residual_norms=bufs["res"][:rep.residual_count].copy(),
        wall_times=bufs["wall"][:rep.wall_count].copy()))


def _irn(kind, proj, grid, prior, params, opts, projector, layout, out=None):
    params = params or RegularizationParams()
    opts = opts or ReconOptions()
    A = _projector_for(proj, grid, projector)
    m, n = A.domain_size(), A.range_size()
    b = _Arg(proj.data, n, "projections")
    pr = _Arg(prior, m, "prior") if prior is not None else None
    x0 = _Arg(opts.initial, m, "initial") if opts.initial is not None else None
    gt = _Arg(opts.ground_truth, m, "ground truth") if opts.ground_truth is not None else None
    mem = _same_mem([b, pr, x0, gt])
    out = _out_for(b, m, out)
    o, i = int(params.outer_iters), int(params.inner_iters)
    rep, bufs = _report_buffers(o + 1, o * i, o)
    p = params._c()
    with _HookInstall(A, opts.hook):
        _check(_lib.kct_irn(A.handle, kind, b.ptr, pr.ptr if pr else None, x0.ptr if x0 else None,
                            gt.ptr if gt else None, C.byref(p), _ptr(out), C.byref(rep), mem,
                            _layout_code(layout, mem),
                            _stream_of(mem, b.keep.device.index if mem == MEM_DEVICE else None)))
    return _unpack(rep, bufs, out)


def irn_tv(proj, grid, params=None, opts=None, projector=None, layout=None,
           out=None) -> ReconReport:
    """recon.hpp:252-255."""
    return _irn(KIND_TV, proj, grid, None, params, opts, projector, layout, out)


def irn_piple(proj, grid, prior, params=None, opts=None, projector=None, layout=None, out=None):
    """recon.hpp:260-263."""
    return _irn(KIND_PIPLE, proj, grid, prior, params, opts, projector, layout, out)


def irn_piccs(proj, grid, prior, params=None, opts=None, projector=None, layout=None, out=None):
    """recon.hpp:267-270 — the north-star entry point.  `out`: optional caller
    buffer for the volume (e.g. pinned host memory for fast copies)."""
    return _irn(KIND_PICCS, proj, grid, prior, params, opts, projector, layout, out)


def fdk(proj: ProjectionSet, grid: GridSpec, projector: ConeBeamProjector | None = None,
        layout=None):
    """fdk (fdk.hpp:50-139)."""
    A = _projector_for(proj, grid, projector)
    return A.fdk(proj.data, layout=layout)


def resolve_tau(tau: float, reference=None) -> float:
    """recon.hpp:60-66."""
    lib = load_library()
    if reference is None:
        return float(lib.kct_resolve_tau(tau, None, 0))
    r = np.ascontiguousarray(np.asarray(reference, dtype=np.float32).reshape(-1))
    return float(lib.kct_resolve_tau(tau, r.ctypes.data, r.size))


from . import shard  # noqa: E402  (depends on the types above)
