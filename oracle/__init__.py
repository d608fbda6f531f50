"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

* ``Oracle("ora")`` loads ``oracle/libkct_oracle.so``: our plain-C float64
  restatement of the reference hot path (``oracle/kct_oracle.c``).
* ``Oracle("ref")`` loads ``oracle/_ref/libkryct_ref.so``: the UNMODIFIED
  reference headers compiled in place (``oracle/Makefile``), i.e. the
  reference's own code path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package; the product library never links or calls it.
Arrays use the reference layouts (volumes x-fastest, projections u-fastest).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ora": (os.path.join(HERE, "libkct_oracle.so"), "ora_"),
    "ref": (os.path.join(HERE, "_ref", "libkryct_ref.so"), "ref_"),
}


class KctGrid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("sx", C.c_double), ("sy", C.c_double), ("sz", C.c_double),
                ("ox", C.c_double), ("oy", C.c_double), ("oz", C.c_double)]


class KctGeometry(C.Structure):
    _fields_ = [("dso", C.c_double), ("dsd", C.c_double), ("nu", C.c_int), ("nv", C.c_int),
                ("pu", C.c_double), ("pv", C.c_double),
                ("offset_u", C.c_double), ("offset_v", C.c_double),
                ("n_angles", C.c_int), ("angles", C.POINTER(C.c_double))]


class KctRegParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("tau", C.c_double),
                ("outer_iters", C.c_size_t), ("inner_iters", C.c_size_t),
                ("inner_tolerance", C.c_double), ("warm_start", C.c_int)]


class KctReport(C.Structure):
    _fields_ = [("objective_history", C.POINTER(C.c_double)), ("objective_count", C.c_size_t),
                ("residual_history", C.POINTER(C.c_double)), ("residual_count", C.c_size_t),
                ("error_history", C.POINTER(C.c_double)), ("error_count", C.c_size_t),
                ("outer_boundaries", C.POINTER(C.c_uint64)), ("outer_count", C.c_size_t),
                ("outer_seconds", C.POINTER(C.c_double)),
                ("solve_seconds", C.c_double), ("tau", C.c_double),
                ("converged", C.c_int), ("breakdown", C.c_int),
                ("wall_times", C.POINTER(C.c_double)), ("wall_count", C.c_size_t)]


@dataclass
class Grid:
    """GridSpec (types.hpp:56-80)."""
    nx: int
    ny: int
    nz: int
    sx: float = 1.0
    sy: float = 1.0
    sz: float = 1.0
    ox: float | None = None
    oy: float | None = None
    oz: float | None = None

    def __post_init__(self):  # GridSpec::centered (types.hpp:62-65) when origin omitted
        if self.ox is None:
            self.ox = -0.5 * self.nx * self.sx
        if self.oy is None:
            self.oy = -0.5 * self.ny * self.sy
        if self.oz is None:
            self.oz = -0.5 * self.nz * self.sz

    @property
    def count(self) -> int:
        return self.nx * self.ny * self.nz

    def c(self) -> KctGrid:
        return KctGrid(self.nx, self.ny, self.nz, self.sx, self.sy, self.sz,
                       self.ox, self.oy, self.oz)


@dataclass
class Geometry:
    """ConeBeamGeometry (types.hpp:138-161)."""
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
        self.angles = np.ascontiguousarray(np.asarray(self.angles, dtype=np.float64))

    @property
    def n_angles(self) -> int:
        return int(self.angles.size)

    @property
    def ray_count(self) -> int:
        return self.nu * self.nv * self.n_angles

    def c(self) -> KctGeometry:
        return KctGeometry(self.dso, self.dsd, self.nu, self.nv, self.pu, self.pv,
                           self.offset_u, self.offset_v, self.n_angles,
                           self.angles.ctypes.data_as(C.POINTER(C.c_double)))


def uniform_angles(n: int) -> np.ndarray:
    """experiment.hpp:89-94: 2*pi*i/n."""
    return 2.0 * np.pi * np.arange(n, dtype=np.float64) / float(n)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(kind: str = "ora") -> None:
    target = [] if kind == "ora" else ["ref"]
    subprocess.run(["make", "-s", "-C", HERE] + target, check=True)


class Oracle:
    def __init__(self, kind: str = "ora"):
        path, pre = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle {'' if kind == 'ora' else 'ref'})")
        self.kind = kind
        lib = C.CDLL(path)
        self.lib = lib
        self.pre = pre
        g = lambda n: getattr(lib, pre + n)  # noqa: E731
        self._last_error = g("last_error")
        self._last_error.restype = C.c_char_p
        self._set_threads = g("set_threads")
        self._set_threads.argtypes = [C.c_int]
        P = C.POINTER
        gp, gg = P(KctGrid), P(KctGeometry)
        self._fwd = g("forward"); self._fwd.argtypes = [gp, gg, P(C.c_double), P(C.c_double)]
        self._adj = g("adjoint"); self._adj.argtypes = [gp, gg, P(C.c_double), P(C.c_double)]
        self._nnz = g("count_nnz"); self._nnz.argtypes = [gp, gg]; self._nnz.restype = C.c_uint64
        self._trace = g("trace_ray")
        self._trace.argtypes = [gp, P(C.c_double), P(C.c_double), P(C.c_uint64), P(C.c_double),
                                C.c_size_t, P(C.c_double)]
        self._trace.restype = C.c_size_t
        self._diff = g("diff"); self._diff.argtypes = [C.c_int] * 3 + [P(C.c_double)] * 2
        self._diffT = g("diff_adjoint"); self._diffT.argtypes = [C.c_int] * 3 + [P(C.c_double)] * 2
        self._tvw = g("tv_weights")
        self._tvw.argtypes = [P(C.c_double), C.c_size_t, C.c_double, P(C.c_double)]
        self._stv = g("smoothed_tv"); self._stv.argtypes = [P(C.c_double), C.c_size_t, C.c_double]
        self._stv.restype = C.c_double
        self._tau = g("resolve_tau"); self._tau.argtypes = [C.c_double, P(C.c_double), C.c_size_t]
        self._tau.restype = C.c_double
        self._obj = g("objective")
        self._obj.argtypes = [gp, gg, C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                              C.c_double, C.c_double, C.c_double]
        self._obj.restype = C.c_double
        self._fdk = g("fdk"); self._fdk.argtypes = [gp, gg, P(C.c_double), P(C.c_double)]
        self._cgls = g("cgls_recon")
        self._cgls.argtypes = [gp, gg, P(C.c_double), C.c_size_t, P(C.c_double), P(C.c_double),
                               C.c_double, P(C.c_double), P(KctReport)]
        self._cgls_stack = g("cgls_stack")
        self._cgls_stack.argtypes = [gp, gg, C.c_size_t, P(C.c_int), P(C.c_double),
                                     P(P(C.c_double)), P(C.c_double), P(C.c_double), C.c_size_t,
                                     C.c_double, P(C.c_double), P(C.c_size_t), P(C.c_int), P(C.c_int)]
        self._irn = g("irn")
        self._irn.argtypes = [gp, gg, C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                              P(C.c_double), P(KctRegParams), P(C.c_double), P(KctReport)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._last_error().decode())

    def set_threads(self, n: int) -> None:
        self._set_threads(int(n))

    @staticmethod
    def _f64(a, n=None):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
        if n is not None and a.size != n:
            raise ValueError(f"expected {n} values, got {a.size}")
        return a

    def forward(self, grid: Grid, geom: Geometry, vol) -> np.ndarray:
        v = self._f64(vol, grid.count)
        out = np.zeros(geom.ray_count)
        gc, ge = grid.c(), geom.c()
        self._check(self._fwd(C.byref(gc), C.byref(ge), _dp(v), _dp(out)))
        return out

    def adjoint(self, grid: Grid, geom: Geometry, proj) -> np.ndarray:
        p = self._f64(proj, geom.ray_count)
        out = np.zeros(grid.count)
        gc, ge = grid.c(), geom.c()
        self._check(self._adj(C.byref(gc), C.byref(ge), _dp(p), _dp(out)))
        return out

    def fdk(self, grid: Grid, geom: Geometry, proj) -> np.ndarray:
        p = self._f64(proj, geom.ray_count)
        out = np.zeros(grid.count)
        gc, ge = grid.c(), geom.c()
        self._check(self._fdk(C.byref(gc), C.byref(ge), _dp(p), _dp(out)))
        return out

    def count_nnz(self, grid: Grid, geom: Geometry) -> int:
        gc, ge = grid.c(), geom.c()
        return int(self._nnz(C.byref(gc), C.byref(ge)))

    def trace_ray(self, grid: Grid, src, dst, cap: int = 1 << 16):
        s, d = self._f64(src, 3), self._f64(dst, 3)
        vox = np.zeros(cap, dtype=np.uint64)
        lens = np.zeros(cap)
        t = np.zeros(2)
        gc = grid.c()
        n = self._trace(C.byref(gc), _dp(s), _dp(d), vox.ctypes.data_as(C.POINTER(C.c_uint64)),
                        _dp(lens), cap, _dp(t))
        return vox[:n].copy(), lens[:n].copy(), (float(t[0]), float(t[1]))

    def diff(self, dims, x) -> np.ndarray:
        nx, ny, nz = dims
        v = self._f64(x, nx * ny * nz)
        out = np.zeros(3 * v.size)
        self._diff(nx, ny, nz, _dp(v), _dp(out))
        return out

    def diff_adjoint(self, dims, y) -> np.ndarray:
        nx, ny, nz = dims
        v = self._f64(y, 3 * nx * ny * nz)
        out = np.zeros(nx * ny * nz)
        self._diffT(nx, ny, nz, _dp(v), _dp(out))
        return out

    def tv_weights(self, grad, tau: float) -> np.ndarray:
        g = self._f64(grad)
        out = np.zeros(g.size)
        self._check(self._tvw(_dp(g), g.size // 3, tau, _dp(out)))
        return out

    def smoothed_tv(self, grad, tau: float) -> float:
        g = self._f64(grad)
        return float(self._stv(_dp(g), g.size // 3, tau))

    def resolve_tau(self, tau: float, ref=None) -> float:
        r = self._f64(ref) if ref is not None else None
        return float(self._tau(tau, _dp(r), 0 if r is None else r.size))

    def objective(self, grid, geom, kind, b, x, prior, alpha, lam, tau) -> float:
        bb, xx = self._f64(b, geom.ray_count), self._f64(x, grid.count)
        pp = self._f64(prior, grid.count) if prior is not None else None
        gc, ge = grid.c(), geom.c()
        return float(self._obj(C.byref(gc), C.byref(ge), kind, _dp(bb), _dp(xx), _dp(pp),
                               alpha, lam, tau))

    @staticmethod
    def _report(n_obj, n_res, n_outer):
        bufs = dict(obj=np.zeros(max(n_obj, 1)), res=np.zeros(max(n_res, 1)),
                    err=np.zeros(max(n_res, 1)), bnd=np.zeros(max(n_outer, 1), dtype=np.uint64),
                    sec=np.zeros(max(n_outer, 1)))
        rep = KctReport()
        rep.objective_history = _dp(bufs["obj"])
        rep.residual_history = _dp(bufs["res"])
        rep.error_history = _dp(bufs["err"])
        rep.outer_boundaries = bufs["bnd"].ctypes.data_as(C.POINTER(C.c_uint64))
        rep.outer_seconds = _dp(bufs["sec"])
        return rep, bufs

    @staticmethod
    def _unpack(rep, bufs):
        return dict(objective_history=bufs["obj"][:rep.objective_count].copy(),
                    residual_history=bufs["res"][:rep.residual_count].copy(),
                    error_history=bufs["err"][:rep.error_count].copy(),
                    outer_boundaries=bufs["bnd"][:rep.outer_count].astype(np.int64),
                    outer_seconds=bufs["sec"][:rep.outer_count].copy(),
                    solve_seconds=rep.solve_seconds, tau=rep.tau,
                    converged=bool(rep.converged), breakdown=bool(rep.breakdown))

    def cgls_recon(self, grid, geom, b, iters, x0=None, ground_truth=None, tol=0.0):
        bb = self._f64(b, geom.ray_count)
        x0a = self._f64(x0, grid.count) if x0 is not None else None
        gta = self._f64(ground_truth, grid.count) if ground_truth is not None else None
        out = np.zeros(grid.count)
        rep, bufs = self._report(iters, iters, 1)
        gc, ge = grid.c(), geom.c()
        self._check(self._cgls(C.byref(gc), C.byref(ge), _dp(bb), iters, _dp(x0a), _dp(gta),
                               tol, _dp(out), C.byref(rep)))
        return out, self._unpack(rep, bufs)

    def cgls_stack(self, grid, geom, blocks, b, iters, x0=None, tol=0.0):
        """cgls (krylov.hpp:59-127) on a caller-assembled StackedMap
        (linear_map.hpp:159-216).  blocks: [(map, scale, weights | None), ...] with map
        0 projector / 1 DiffOperator / 2 IdentityMap.  Returns (x, info dict)."""
        m, n = grid.count, geom.ray_count
        lens = [n if mp == 0 else (3 * m if mp == 1 else m) for mp, _, _ in blocks]
        bb = self._f64(b, sum(lens))
        nb = len(blocks)
        maps = (C.c_int * nb)(*[int(mp) for mp, _, _ in blocks])
        scales = (C.c_double * nb)(*[float(sc) for _, sc, _ in blocks])
        keep = [None if w is None else self._f64(w, ln) for (_, _, w), ln in zip(blocks, lens)]
        wts = (C.POINTER(C.c_double) * nb)(*[
            C.cast(None, C.POINTER(C.c_double)) if w is None else _dp(w) for w in keep])
        x = np.zeros(m) if x0 is None else self._f64(x0, m).copy()
        res = np.zeros(max(int(iters), 1))
        its, conv, brk = C.c_size_t(0), C.c_int(0), C.c_int(0)
        gc, ge = grid.c(), geom.c()
        self._check(self._cgls_stack(C.byref(gc), C.byref(ge), nb, maps, scales, wts, _dp(bb), _dp(x),
                                     int(iters), float(tol), _dp(res), C.byref(its), C.byref(conv),
                                     C.byref(brk)))
        return x, dict(iterations=its.value, converged=bool(conv.value), breakdown=bool(brk.value),
                       residual_history=res[:its.value].copy())

    def irn(self, grid, geom, kind, b, prior, params: dict, x0=None, ground_truth=None):
        bb = self._f64(b, geom.ray_count)
        pr = self._f64(prior, grid.count) if prior is not None else None
        x0a = self._f64(x0, grid.count) if x0 is not None else None
        gta = self._f64(ground_truth, grid.count) if ground_truth is not None else None
        p = KctRegParams(params.get("alpha", 0.05), params.get("lambda", params.get("lambda_", -1.0)),
                         params.get("tau", 0.0), params.get("outer_iters", 4),
                         params.get("inner_iters", 25), params.get("inner_tolerance", 0.0),
                         int(params.get("warm_start", True)))
        out = np.zeros(grid.count)
        rep, bufs = self._report(p.outer_iters + 1, p.outer_iters * p.inner_iters, p.outer_iters)
        gc, ge = grid.c(), geom.c()
        self._check(self._irn(C.byref(gc), C.byref(ge), kind, _dp(bb), _dp(pr), _dp(x0a),
                              _dp(gta), C.byref(p), _dp(out), C.byref(rep)))
        return out, self._unpack(rep, bufs)


KIND_TV, KIND_PIPLE, KIND_PICCS = 0, 1, 2
