#!/usr/bin/env python
"""Benchmark of the PICCS-Krylov CBCT hot path (BASELINE.json metric).

metric: "fwd+back-proj GUPS; seconds per 20-iter PICCS-Krylov recon at 256^3".
One step = one forward projection A x plus one backprojection A^T y of the
c3 workload (256^3 volume at 0.5 mm, 384^2 detector at 0.5 mm, 60 views),
inputs resident in HBM; value = 2 * M * n_angles * steps / time  [GUPS].
The line also carries the 20-iteration IRN-PICCS reconstruction time at c3
("recon"), the end-to-end numbers through the C ABI with host buffers ("e2e"),
the roofline of the dominant kernel and the reference CPU baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N > 1 runs under torchrun: rank r projects angles r::N (forward) and
backprojects z-slab r of the volume from all angles (no data-path collective;
inputs are resident), the device time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_TAG = "fwd+back-proj GUPS; seconds per 20-iter PICCS-Krylov recon at 256^3"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # NVML (~ms per query: many samples even in a short timed region),
        # else nvidia-smi
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active"
                                                          for b in bits])
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU code (oracle/_ref) on host cores
# ---------------------------------------------------------------------------
def _ref_oracle(threads: int = 0):
    """The unmodified reference compiled in place (oracle/_ref), else the C port."""
    import oracle
    from oracle import Oracle
    if not os.path.exists(oracle.LIBS["ref"][0]):
        try:
            oracle.build("ref")
        except Exception:
            pass
    kind = "reference" if os.path.exists(oracle.LIBS["ref"][0]) else "port"
    if kind == "port":
        oracle.build("ora")
    o = Oracle("ref" if kind == "reference" else "ora")
    nthreads = threads or os.cpu_count() or 1
    o.set_threads(nthreads)
    return o, kind, nthreads


def host_info() -> dict:
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model or "unknown"}


def _c3_ora(n_views: int):
    from oracle import Geometry, Grid
    from paper_2509_08574_b200 import synth
    cfg = synth.CONFIGS["c3"]
    sel = synth.angles(cfg.followup_views)
    if n_views < cfg.followup_views:
        sel = sel[:: max(1, cfg.followup_views // n_views)][:n_views]
    grid = Grid(cfg.n, cfg.n, cfg.n, cfg.voxel, cfg.voxel, cfg.voxel)
    geom = Geometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch, sel)
    return cfg, grid, geom


def cpu_reference_gups(n_views: int, repeats: int, warmup: int = 1, threads: int = 0):
    """fwd+adj GUPS of the unmodified reference (oracle/_ref) on the c3 geometry
    (all 60 views, or an evenly spaced sample of n_views)."""
    from paper_2509_08574_b200 import synth
    o, kind, nthreads = _ref_oracle(threads)
    cfg, grid, geom = _c3_ora(n_views)
    _, prior, _ = synth.study("c3")
    x = prior.astype(np.float64)
    times = []
    for r in range(warmup + repeats):
        t0 = time.perf_counter()
        y = o.forward(grid, geom, x)
        o.adjoint(grid, geom, y)
        dt = time.perf_counter() - t0
        if r >= warmup:
            times.append(dt)
    m = cfg.n ** 3
    nv = geom.n_angles
    total = sum(times)
    return {"value": 2.0 * m * nv * repeats / total / 1e9, "unit": "GUPS", "cores": nthreads,
            "kind": kind, "views": nv,
            "sample": f"c3 256^3/384^2, {nv} of {cfg.followup_views} views, A x + A^T y "
                      f"(project_forward + project_adjoint, float64), {repeats} timed after "
                      f"{warmup} warm-up",
            "seconds_per_step": total / repeats, "all_seconds": [round(t, 3) for t in times]}


def cpu_reference_recon(threads: int = 0) -> dict:
    """ReconReport.solve_seconds (recon.hpp:243-244) of the reference's own
    irn_piccs (recon.hpp:267-270) at c3: 4x5 iterations, alpha = lambda = 0.5,
    tau auto; b = the reference's forward projection of the follow-up phantom
    (60 views) with Poisson noise I0 = 5e4; prior = the prior phantom (the
    solve's cost does not depend on the values; no GPU on this path)."""
    from oracle import KIND_PICCS
    from paper_2509_08574_b200 import synth
    o, kind, nthreads = _ref_oracle(threads)
    cfg, grid, geom = _c3_ora(60)
    _, prior, follow = synth.study("c3")
    b = synth.poisson_log(o.forward(grid, geom, follow.astype(np.float64)), cfg.i0,
                          seed=synth.noise_seed("c3"))
    t0 = time.perf_counter()
    _, rep = o.irn(grid, geom, KIND_PICCS, b.astype(np.float64), prior.astype(np.float64),
                   dict(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner))
    wall = time.perf_counter() - t0
    return {"seconds_per_recon": round(rep["solve_seconds"], 3), "wall_seconds": round(wall, 3),
            "outer_seconds": [round(v, 3) for v in rep["outer_seconds"]],
            "iterations": cfg.outer * cfg.inner, "outer_x_inner": f"{cfg.outer}x{cfg.inner}",
            "threads": nthreads, "kind": kind,
            "what": "irn_piccs c3 (256^3, 384^2, 60 views), ReconReport.solve_seconds"}


def cpu_reference_cgls_c1(threads: int) -> dict:
    """ReconReport.solve_seconds of the reference's cgls_recon (recon.hpp:312-315),
    BASELINE config 1: 64^3, 96^2, 64 views, 20 iterations from zero, noiseless."""
    from oracle import Geometry, Grid
    from paper_2509_08574_b200 import synth
    o, kind, nthreads = _ref_oracle(threads)
    cfg = synth.CONFIGS["c1"]
    grid = Grid(cfg.n, cfg.n, cfg.n, cfg.voxel, cfg.voxel, cfg.voxel)
    geom = Geometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                    synth.angles(cfg.followup_views))
    _, prior, _ = synth.study("c1")
    b = o.forward(grid, geom, prior.astype(np.float64))
    o.cgls_recon(grid, geom, b, 2)  # warm-up (first OpenMP call)
    _, rep = o.cgls_recon(grid, geom, b, cfg.iters)
    return {"seconds": round(rep["solve_seconds"], 3), "threads": nthreads, "kind": kind}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    # the whole c3 scan per step (same workload as our arm) unless K is large:
    # then an evenly spaced angle sample keeps the run within a few minutes
    views = 60 if steps <= 20 else max(4, 60 * 20 // steps)
    res = cpu_reference_gups(views, steps, warmup)
    value = res["value"]
    line = {"impl": "reference", "metric": M_TAG, "value": round(value, 5), "unit": "GUPS",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": round(1e3 * res["seconds_per_step"], 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c3: A x + A^T y, 256^3 @0.5mm, 384^2 @0.5mm, 60 views, "
                                   "DSO 1000 / DSD 1500",
                       "views_per_step": res["views"], "same_config": res["views"] == 60},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": round(value, 5), "unit": "GUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "host": host_info(), "all_seconds": res["all_seconds"]}
    if not args.skip_recon:
        line["recon"] = cpu_reference_recon()
        line["cgls_c1"] = {"all_threads": cpu_reference_cgls_c1(0),
                           "one_thread": cpu_reference_cgls_c1(1)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_2509_08574_b200 as k
    from paper_2509_08574_b200 import synth

    ws, rank, local = dist_env()
    ndev = torch.cuda.device_count()
    # one process per GPU; if fewer GPUs than ranks (functional check only),
    # ranks share devices and synchronise over gloo (host barriers only)
    shared = ws > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS["c3"]
    M = cfg.n ** 3
    na = cfg.followup_views
    geom_all = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                                  synth.angles(na))
    grid = k.GridSpec((cfg.n,) * 3, (cfg.voxel,) * 3)
    log(f"[bench] rank {rank}/{ws}: generating c3 phantoms")
    _, prior, follow = synth.study("c3")

    # sharding (paper_2509_08574_b200/shard.py): forward over angles r::ws,
    # adjoint over y-slab r from all angles (contiguous in the native layout;
    # keeps the bricks full height: 74% vs 58% efficiency for z-slabs at 8
    # ranks, tools/shard_time.py); no data-path collective
    from paper_2509_08574_b200 import shard
    my_angles = shard.angle_indices(na, ws, rank)
    geom_f = shard.shard_geometry(geom_all, ws, rank)
    from paper_2509_08574_b200 import distributed as _dist
    grid_b = shard.slab_grid(grid, ws, rank, "y", _dist.slab_bounds(grid, geom_all, ws))
    A_f = k.ConeBeamProjector(grid, geom_f, device=local)
    A_b = A_f if ws == 1 else k.ConeBeamProjector(grid_b, geom_all, device=local)
    nnz_f = A_f.count_nnz()
    nnz_b = nnz_f if ws == 1 else A_b.count_nnz()
    Nf = geom_f.ray_count()
    Nb = geom_all.ray_count()
    Mb = grid_b.count()

    x_host = torch.from_numpy(prior).to(dev)
    x = A_f.volume_to_native(x_host)
    q = torch.empty(Nf, dtype=torch.float32, device=dev)
    y = torch.rand(Nb, dtype=torch.float32, device=dev, generator=torch.Generator(dev).manual_seed(7))
    back = torch.empty(Mb, dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream(dev)

    def step():
        A_f.apply(x, out=q)
        A_b.apply_adjoint(y, out=back)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = k.launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 between timed steps (not timed)
            e0, e1, e2 = ev[i]
            e0.record(stream)
            A_f.apply(x, out=q)
            e1.record(stream)
            A_b.apply_adjoint(y, out=back)
            e2.record(stream)
        torch.cuda.synchronize(dev)
    launches = k.launch_count() - launches0  # kernels of libkct.so in the timed region
    t_f = [a.elapsed_time(b) * 1e-3 for a, b, _ in ev]
    t_b = [b.elapsed_time(c) * 1e-3 for _, b, c in ev]
    t_tot = sum(t_f) + sum(t_b)
    if ws > 1:
        tt = torch.tensor([t_tot], device="cpu" if shared else dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_tot = float(tt.item())
    gups = 2.0 * M * na * args.steps / t_tot / 1e9
    mean_f, mean_b = float(np.mean(t_f)), float(np.mean(t_b))

    # roofline of the dominant kernel (SURVEY §8d byte model, per launch)
    peak, peak_src = measured_peak()
    bytes_f = 4.0 * nnz_f + 4.0 * Nf
    bytes_b = 4.0 * nnz_b + 4.0 * Mb
    adj_kernel = ("adj_mirror_ws_kernel" if A_b.info("adj_ws") else "adj_mirror_kernel") \
        if A_b.info("adj_mirror") else "adj_brick_kernel"
    if mean_b >= mean_f:
        dom = (f"adjoint ({adj_kernel})", bytes_b, mean_b)
    else:
        dom = ("forward (fwd_kernel)", bytes_f, mean_f)
    achieved = dom[1] / dom[2] / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(adj_kernel if "adj" in dom[0] else "fwd_kernel")
        except Exception:
            traffic = None

    out = {"metric": M_TAG, "value": round(gups, 3), "unit": "GUPS", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(1e3 * t_tot / args.steps, 4), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded 20-ellipsoid c3 phantom, resident in HBM)",
           "config": {"workload": "c3: A x + A^T y, 256^3 @0.5mm, 384^2 @0.5mm, 60 views, "
                                  "DSO 1000 / DSD 1500",
                      "M": M, "n_angles": na, "nnz": nnz_f if ws == 1 else None,
                      "l2": "flushed (256 MiB write) between timed steps, flush not timed",
                      "parallelism": f"angles/y-slabs x{ws}" if ws > 1 else "single GPU",
                      **({"shared_devices": "functional check: more ranks than GPUs"} if shared else {})},
           "kernels_ms": {"forward": round(1e3 * mean_f, 4), "adjoint": round(1e3 * mean_b, 4)},
           "gups_forward": round(M * len(my_angles) / mean_f / 1e9, 3),
           "gups_adjoint": round(Mb * na / mean_b / 1e9, 3),
           "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": round(achieved, 1),
                        "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                        "traffic": traffic, "peak_source": peak_src,
                        "algorithmic_bytes_per_launch": dom[1],
                        "byte_model": "4*nnz + 4*N (A x) / 4*nnz + 4*M (A^T y), nnz = exact "
                                      "Siddon intersections counted on device"},
           "gpu_launches": launches, "clocks": clk.summary(),
           "launches_per_step": {"forward": "pad_kernel + fwd_kernel",
                                 "adjoint": (f"adj_weight_mir_kernel + {adj_kernel}"
                                             if "mirror" in adj_kernel else
                                             "adj_weight_kernel + adj_brick_kernel")
                                 + " (+ adj_group_sum when angle groups > 1)"},
           # which code paths the handles run (kct_projector_info)
           "paths": {key: A_b.info(key) for key in ("adj_slab", "adj_mirror", "adj_ws", "adj_np", "adj_bz",
                                                      "adj_groups", "adj_walk_entries")}
           | {key: A_f.info(key) for key in ("fwd_rows_per_warp", "fwd_bands", "fwd_split_z")}}

    # ---- FDK (fdk.hpp:50-139) of the c3 follow-up geometry, device resident ----
    if rank == 0 and ws == 1 and not args.skip_fdk:
        fdk_out = torch.empty(M, dtype=torch.float32, device=dev)
        A_f.fdk(q, out=fdk_out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            A_f.fdk(q, out=fdk_out)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        out["fdk_ms"] = round(e0.elapsed_time(e1) / 3, 4)

    # ---- end to end through the C ABI with host buffers (reference layouts) ----
    # every rank: its forward (host volume in, host projections out) and its
    # adjoint (host projections in, host volume slab out); whole-job rate over
    # the slowest rank
    if not args.skip_e2e:
        vol_h = torch.from_numpy(prior).pin_memory().numpy()
        proj_h = torch.empty(Nf, dtype=torch.float32).pin_memory().numpy()
        yb_h = proj_h if ws == 1 else y.cpu().pin_memory().numpy()
        back_h = torch.empty(Mb, dtype=torch.float32).pin_memory().numpy()

        def e2e_step():
            A_f.apply(vol_h, out=proj_h)
            A_b.apply_adjoint(yb_h, out=back_h)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        te = time.perf_counter() - t0
        if ws > 1:
            tt = torch.tensor([te], device="cpu" if shared else dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e_gups = 2.0 * M * na * args.steps / te / 1e9
        out["e2e"] = {"value": round(e2e_gups, 3), "unit": "GUPS",
                      "h2d_bytes_per_step": 4 * (M + (Nf if ws == 1 else Nb)),
                      "d2h_bytes_per_step": 4 * (Nf + Mb),
                      "ms_per_step": round(1e3 * te / args.steps, 3),
                      "path": "kct_forward + kct_adjoint, pinned host, reference layouts"
                              + ("" if ws == 1 else "; bytes per rank, time = slowest rank")}

    # ---- 20-iteration IRN-PICCS at c3 (the metric's second half) --------------
    if not args.skip_recon:
        rec = run_recon(k, synth, cfg, grid, prior, follow, dev, args, ws, rank, shared)
        if rank == 0:
            out["recon"] = rec
            if ws == 1:
                shim = run_shim()
                if shim is not None:
                    out["recon"]["cpp_dropin"] = shim

    if rank == 0 and not args.skip_cpu:
        try:
            out["cpu_baseline"] = {kk: v for kk, v in cpu_reference_gups(60, 2).items()
                                   if kk in ("value", "unit", "cores", "kind", "sample")}
            out["cpu_baseline"]["host"] = host_info()
        except Exception as e:  # report, do not fail the bench
            out["cpu_baseline"] = {"value": None, "error": str(e)}
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_shim():
    """The C++ drop-in (include/kryct_b200.hpp: kryct_b200::irn_piccs with the
    reference's signature and double buffers) in a fresh process at c3:
    handle creation (CUDA context, walk tables, workspace) and the first call
    reported apart from the cached calls (build/bench_shim, tests/cpp/bench_shim.cpp)."""
    exe = os.path.join(ROOT, "build", "bench_shim")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {
            "error": (r.stderr or r.stdout)[-300:]}
    except Exception as e:  # report, do not fail the bench
        return {"error": str(e)}


def run_recon(k, synth, cfg, grid, prior, follow, dev, args, ws=1, rank=0, shared=False):
    """20-iteration IRN-PICCS at c3.  With ws > 1 (distributed.py) either every
    rank holds y planes [j0, j1) of the volume vectors and all projections
    (--recon-split yslab: partial-projection and scalar all-reduces, halo
    planes) or the angles r::ws (angles: partial-volume and scalar
    all-reduces); the reported time is the max over ranks."""
    import torch
    na_p, na_f = cfg.prior_views, cfg.followup_views
    geom_p = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                                synth.angles(na_p))
    geom_f = k.ConeBeamGeometry(synth.DSO, synth.DSD, cfg.det, cfg.det, cfg.pitch, cfg.pitch,
                                synth.angles(na_f))
    Ap = k.ConeBeamProjector(grid, geom_p)
    Af = k.ConeBeamProjector(grid, geom_f)
    t0 = time.perf_counter()
    # prior: 360-view noiseless scan of the prior phantom, 20-iteration CGLS (pinned)
    xp_n = Ap.volume_to_native(torch.from_numpy(prior).to(dev))
    bp_n = Ap.apply(xp_n)
    prior_rec = k.cgls_recon(k.ProjectionSet(geom_p, bp_n), grid, 20, projector=Ap).volume
    # follow-up: 60 views, Poisson I0 = 5e4 on the transmission
    xf_n = Af.volume_to_native(torch.from_numpy(follow).to(dev))
    pf = Af.proj_from_native(Af.apply(xf_n)).cpu().numpy()
    b = synth.poisson_log(pf, cfg.i0, seed=1003)
    del Ap, xp_n, bp_n, xf_n
    slab = ws > 1 and args.recon_split == "yslab"
    grid_s, prior_s, follow_s = grid, prior_rec, follow
    if slab:
        # y-slab-sharded state (distributed.irn_piccs_slab): this rank's volume
        # planes [j0, j1) with halos, all projections, partial-projection sums
        from paper_2509_08574_b200 import distributed, shard
        proj_h = k.ProjectionSet(geom_f, b)
        A, j0, j1 = distributed.slab_projector(grid, geom_f, ws, rank)
        grid_s = A.grid
        plane = grid.dims[0] * grid.dims[2]
        prior_s = prior_rec[j0 * plane:j1 * plane].contiguous()  # native y-slab
        follow_s = distributed.y_slab(follow, grid, j0, j1)
    elif ws > 1:
        from paper_2509_08574_b200 import distributed
        proj_h = distributed.shard_projections(k.ProjectionSet(geom_f, b), ws, rank)
        A = distributed.sharded_projector(proj_h, grid)
    else:
        proj_h = k.ProjectionSet(geom_f, b)
        A = Af
    b_n = A.proj_to_native(torch.from_numpy(np.asarray(proj_h.data)).to(dev))
    torch.cuda.synchronize(dev)
    setup = time.perf_counter() - t0
    params = k.RegularizationParams(alpha=cfg.alpha, outer_iters=cfg.outer, inner_iters=cfg.inner)
    proj = k.ProjectionSet(proj_h.geometry, b_n)

    def rsum(vals, op="sum"):
        if ws == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else dev)
        torch.distributed.all_reduce(
            t, op=torch.distributed.ReduceOp.SUM if op == "sum" else torch.distributed.ReduceOp.MAX)
        return t.tolist()

    def timed(fn):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        r = fn()
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t
        if ws > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        return r, dt

    reps = []
    rep = None
    for i in range(args.recon_warmup + args.recon_steps):
        rep, dt = timed(lambda: k.irn_piccs(proj, grid_s, prior_s, params, projector=A))
        if i >= args.recon_warmup:
            reps.append(dt)
    x_ref = A.volume_from_native(rep.volume).cpu().numpy()
    e2, f2 = rsum([float(np.sum((x_ref.astype(np.float64) - follow_s) ** 2)),
                   float(np.sum(np.asarray(follow_s, dtype=np.float64) ** 2))])
    rel = float(np.sqrt(e2 / f2))
    # end to end: host float32 arrays in the reference layouts through kct_irn_piccs
    # (pinned host buffers; one untimed warm-up of the host-buffer path)
    prior_h = A.volume_from_native(prior_s).cpu().pin_memory().numpy()
    b_h = torch.from_numpy(np.ascontiguousarray(proj_h.data, dtype=np.float32)).pin_memory().numpy()
    proj_hp = k.ProjectionSet(proj_h.geometry, b_h)
    x_h = torch.empty(grid_s.count(), dtype=torch.float32).pin_memory().numpy()
    k.irn_piccs(proj_hp, grid_s, prior_h, params, projector=A, out=x_h)
    rep_h, e2e = timed(lambda: k.irn_piccs(proj_hp, grid_s, prior_h, params, projector=A,
                                           out=x_h))
    same = rsum([float(np.abs(rep_h.volume - x_ref).max())], op="max")[0]
    return {"seconds_per_recon": round(float(np.median(reps)), 4),
            "all_seconds": [round(r, 4) for r in reps],
            "solve_seconds_reported": round(rep.solve_seconds, 4),
            "e2e_seconds": round(e2e, 4),
            "e2e_h2d_bytes": 4 * (2 * grid_s.count() + proj_h.geometry.ray_count()),
            "e2e_d2h_bytes": 4 * grid_s.count(), "e2e_max_abs_diff_vs_device_run": same,
            "iterations": cfg.outer * cfg.inner, "outer_x_inner": f"{cfg.outer}x{cfg.inner}",
            "alpha": cfg.alpha, "lambda": cfg.alpha, "tau": rep.tau,
            "objective_history": [float(v) for v in rep.objective_history],
            "rel_error_vs_followup_phantom": round(rel, 5),
            "prior": "20-iter CGLS of a 360-view noiseless scan (computed on device, untimed)",
            "parallelism": (f"y-slab-sharded x{ws}: partial-projection + scalar all-reduces, "
                            "halo planes" if slab else
                            f"angle-sharded x{ws}: partial-volume + scalar all-reduces"
                            if ws > 1 else "single GPU"),
            "collectives": (None if ws == 1 else
                            "library NCCL communicator (kct_comm_*: ncclAllReduce / ncclSend+Recv "
                            "on the solver's stream)" if getattr(A, "_comm", None) is not None
                            else "torch.distributed hooks"),
            "setup_seconds_untimed": round(setup, 2),
            "reference_cpu": "the --impl reference line's recon.seconds_per_recon (same box, "
                             "all host cores); tests/test_config_parity_gpu.py measured 151.9 s "
                             "on 16 threads (profiles/r02_config_parity.log)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--recon-steps", type=int, default=3)
    ap.add_argument("--recon-warmup", type=int, default=1)
    ap.add_argument("--skip-recon", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-fdk", action="store_true")
    ap.add_argument("--recon-split", default="yslab", choices=["yslab", "angles"],
                    help="multi-GPU PICCS decomposition (N > 1)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the ranks ourselves (torchrun, rendezvous
        # on 127.0.0.1) with NCCL's communicator logging on, so the rank count
        # of every communicator is visible in the log; rank 0 prints the line
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        log(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}")
        sys.exit(subprocess.call(cmd, env=env))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
