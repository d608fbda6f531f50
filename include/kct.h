/*
 * kct.h — C ABI of the B200-native PICCS-Krylov CBCT core.
 *
 * Drop-in boundary for the hot path of the reference library `kryct`
 * (header-only C++20, /root/reference/proj/include/kryct).  Every entry point
 * below replaces one reference interface; the replaced symbol is cited as
 * file:line next to it.  Plain C: POD structs, raw pointers, sizes and status
 * codes — no C++ or torch types cross this boundary.
 *
 * Data layouts (KCT_LAYOUT_REFERENCE is what the reference uses):
 *   volume       x-fastest  idx = i + nx*(j + ny*k)          types.hpp:86-88
 *   projections  u-fastest  idx = iu + nu*(iv + nv*ia)       types.hpp:163-164
 * KCT_LAYOUT_NATIVE is the device-internal layout the kernels run on:
 *   volume       z-fastest  idx = k + nz*(i + nx*j)
 *   projections  v-fastest  idx = iv + nv*(iu + nu*ia)
 * Values cross the boundary as float32 (the reference promotes float32 files
 * to double, io.hpp:48-49); reductions and solver scalars are float64.
 *
 * Status codes mirror the reference's error taxonomy and CLI exit codes
 * (types.hpp:16-26, tools/kryct.cpp:120-128):
 *   KCT_OK 0, KCT_ERR_INTERNAL 1, KCT_ERR_CONFIG 2 (ConfigError),
 *   KCT_ERR_SOLVER 3 (SolverError), KCT_ERR_CUDA 4 (device failure).
 * kct_last_error() returns the message of the last failure on this thread.
 *
 * Threading: a projector handle is bound to one device and is stream-ordered;
 * calls on one handle must not run concurrently.  All functions synchronise
 * the given stream before returning when any pointer is KCT_MEM_HOST.
 */
#ifndef KCT_H
#define KCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KCT_ABI_VERSION 4

enum kct_status {
    KCT_OK = 0,
    KCT_ERR_INTERNAL = 1,
    KCT_ERR_CONFIG = 2,
    KCT_ERR_SOLVER = 3,
    KCT_ERR_CUDA = 4
};

enum kct_mem { KCT_MEM_HOST = 0, KCT_MEM_DEVICE = 1 };
enum kct_layout { KCT_LAYOUT_REFERENCE = 0, KCT_LAYOUT_NATIVE = 1 };
enum kct_kind { KCT_KIND_TV = 0, KCT_KIND_PIPLE = 1, KCT_KIND_PICCS = 2 };
/* Row-block maps of a caller-assembled stack (kct_cgls_stack). */
enum kct_map {
    KCT_MAP_PROJECTOR = 0, /* the handle's cone-beam projector, range N (projector.hpp:264-291) */
    KCT_MAP_DIFF = 1,      /* DiffOperator, range 3M [dx; dy; dz] (diffreg.hpp:20-81) */
    KCT_MAP_IDENTITY = 2   /* IdentityMap, range M (linear_map.hpp:59-80) */
};

/* GridSpec (types.hpp:56-80): dims, spacing [mm], origin = min corner of voxel (0,0,0). */
typedef struct kct_grid {
    int nx, ny, nz;
    double sx, sy, sz;
    double ox, oy, oz;
} kct_grid;

/* ConeBeamGeometry (types.hpp:138-161) + DetectorSpec (types.hpp:125-130).
 * `angles` (radians, n_angles entries) is copied at handle creation. */
typedef struct kct_geometry {
    double dso, dsd;
    int nu, nv;
    double pu, pv;
    double offset_u, offset_v;
    int n_angles;
    const double* angles;
} kct_geometry;

/* RegularizationParams (recon.hpp:37-55).  lambda < 0 means "use alpha";
 * tau <= 0 resolves from the dynamic range (recon.hpp:60-66). */
typedef struct kct_reg_params {
    double alpha;
    double lambda;
    double tau;
    size_t outer_iters;
    size_t inner_iters;
    double inner_tolerance;
    int warm_start;
} kct_reg_params;

/* ReconReport (recon.hpp:74-83).  The caller owns every array; any pointer may
 * be NULL to skip that history.  Required capacities:
 *   objective_history  outer_iters + 1   (irn_*; cgls_recon: iters)
 *   residual_history   outer_iters * inner_iters   (cgls_recon: iters)
 *   error_history      same as residual_history (needs ground_truth)
 *   outer_boundaries   outer_iters       (cgls_recon: 1)
 *   outer_seconds      outer_iters       (cgls_recon: 1)
 * The *_count fields are written by the solver. */
typedef struct kct_report {
    double* objective_history;  size_t objective_count;
    double* residual_history;   size_t residual_count;
    double* error_history;      size_t error_count;
    uint64_t* outer_boundaries; size_t outer_count;
    double* outer_seconds;
    double solve_seconds;
    double tau;        /* resolved smoothing parameter (irn_*) */
    int converged;
    int breakdown;
    /* SolveTrace::wall_times (krylov.hpp:40, :115): seconds since the solve
     * started, one per inner iteration (device event timeline); capacity as
     * residual_history; NULL skips it.  (ABI 2) */
    double* wall_times;         size_t wall_count;
} kct_report;

typedef struct kct_projector kct_projector;

/* ---- library ---------------------------------------------------------- */
const char* kct_last_error(void);
int kct_abi_version(void);
/* Number of CUDA kernels the library has launched in this process (all
 * handles, all devices) — lets a caller verify which work ran on the GPU. */
unsigned long long kct_launch_count(void);
/* Page-locked host staging memory (cudaMallocHost): host buffers passed with
 * KCT_MEM_HOST that live here are copied asynchronously at full PCIe rate
 * and overlap the kernels.  No reference counterpart: the C++ shim
 * (kryct_b200.hpp) converts the reference's double spans into such buffers. */
int kct_host_alloc(size_t bytes, void** out);
int kct_host_free(void* ptr);

/* ---- operator: ConeBeamProjector (projector.hpp:264-291) --------------- */
/* ctor: validate grid + geometry, reject a source inside the volume
 * (projector.hpp:269-274, :162-168).  device < 0 means the current device. */
int kct_projector_create(const kct_grid* grid, const kct_geometry* geom, int device,
                         kct_projector** out);
int kct_projector_destroy(kct_projector* h);
/* domain_size() / range_size() (projector.hpp:276-277) */
int kct_projector_sizes(const kct_projector* h, size_t* domain, size_t* range);
/* y = A x  — project_forward (projector.hpp:194-204).  vol: M floats, proj: N floats. */
int kct_forward(kct_projector* h, const float* vol, float* proj, int mem, int layout,
                void* stream);
/* x = A^T y — project_adjoint (projector.hpp:226-261); overwrites vol. */
int kct_adjoint(kct_projector* h, const float* proj, float* vol, int mem, int layout,
                void* stream);
/* float64 host spans, reference layouts: LinearMap::apply / apply_adjoint
 * (linear_map.hpp:33-36) for the C++ shim; values are rounded to float32. */
int kct_forward_f64(kct_projector* h, const double* vol, double* proj);
int kct_adjoint_f64(kct_projector* h, const double* proj, double* vol);
/* Exact Siddon intersection count nnz (number of (ray, voxel) pairs with
 * positive length) — the algorithmic-bytes unit of the roofline. */
int kct_count_nnz(kct_projector* h, uint64_t* nnz, void* stream);
/* Which code paths this handle runs (no reference counterpart; evidence for
 * tests and benchmarks).  key: "adj_slab" (1: slab-lane adjoint deposits),
 * "adj_slab_detect", "adj_bz" (brick height), "adj_np" (producer warps per consumer of the
 * warp-specialised adjoint, 0: another kernel), "adj_stride" (row-wise pass
 * stride S), "adj_groups" (angle groups), "adj_gather", "adj_walk_entries",
 * "fwd_rows_per_warp", "fwd_bands", "fwd_split_z" / "fwd_split_lo" (host
 * forward split upload: slabs [lo, z) first, z = 0: off), "mirror" (1: z-mirror
 * ray pairs, rows iv / nv-1-iv), "solver_restart".  Unknown key: ConfigError. */
int kct_projector_info(const kct_projector* h, const char* key, double* value);
/* Layout conversion on device (reference <-> native), stream-ordered. */
int kct_volume_to_native(const kct_projector* h, const float* ref, float* native, void* stream);
int kct_volume_from_native(const kct_projector* h, const float* native, float* ref, void* stream);
int kct_proj_to_native(const kct_projector* h, const float* ref, float* native, void* stream);
int kct_proj_from_native(const kct_projector* h, const float* native, float* ref, void* stream);

/* Feldkamp-Davis-Kress reconstruction — fdk (fdk.hpp:50-139): cosine
 * weighting, Ram-Lak ramp filter, distance-weighted bilinear backprojection.
 * Needs >= 2 angles over a full circle (short scans are not compensated). */
int kct_fdk(kct_projector* h, const float* proj, float* vol, int mem, int layout, void* stream);

/* ---- solver options and the per-iteration hook ------------------------- */
/* Options of the solvers run on this handle (value as double):
 *   "solver_restart" 1: the reference's control flow at every CGLS start —
 *       recompute r = b - A x and A^T r (krylov.hpp:68-75) — and a fresh A x
 *       for every objective evaluation (recon.hpp:189, :238).  0 (default):
 *       a warm start continues the data residual the previous cycle's CGLS
 *       recurrence ended on and its A^T r (one forward and
 *       one adjoint projection less per outer cycle).  The environment
 *       variable KCT_SOLVER_RESTART=1 sets the default for new handles.
 * Unknown key: ConfigError.  kct_projector_info reads options back. */
int kct_set_option(kct_projector* h, const char* key, double value);

/* IterateHook (krylov.hpp:22-23; ReconOptions::hook recon.hpp:68-72, called
 * at recon.hpp:223-228 / :291-295): after every inner CGLS iteration the
 * solver copies the iterate to pinned host memory on a side stream and calls
 * fn(ctx, iteration, x, m) from a CUDA host callback (iteration is 1-based and
 * runs across outer cycles, as the reference's global_iter; x is float32 in
 * the reference layout, valid only during the call; m = domain size of the
 * handle — a y-slab handle passes its slab).  Calls arrive in iteration order
 * and all have returned when the solver returns.  The callback must not call
 * CUDA or this library.  fn = NULL removes the hook (no copies at all). */
typedef void (*kct_iterate_hook)(void* ctx, size_t iteration, const float* x, size_t m);
int kct_set_iterate_hook(kct_projector* h, kct_iterate_hook fn, void* ctx);

/* ---- multi-process solves ------------------------------------------------ */
/* Collective hook: sum `count` elements (dtype 0 = float32, 1 = float64) of
 * the device buffer `buf` over all ranks, in place, ordered on `stream`;
 * return 0 on success.  Installing a hook puts the handle in angle-sharded
 * mode: its geometry holds this rank's projection angles, solver inputs `b`
 * are this rank's readings, the volume-domain state is replicated, and the
 * solvers sum A^T partial volumes and projection-domain reductions over the
 * ranks (the "partial-volume reductions and Krylov scalar all-reduces" of the
 * north star).  NULL restores single-process mode. */
typedef int (*kct_allreduce_fn)(void* ctx, void* buf, size_t count, int dtype, void* stream);
int kct_set_allreduce(kct_projector* h, kct_allreduce_fn fn, void* ctx);

/* y-slab-sharded solves (the volume-partitioned variant).  The
 * handle's grid is planes [j0, j0 + ny) of a grid with ny_global y planes
 * (e.g. shard.slab_grid(..., axis="y")); every rank holds all projections.
 * The solver then keeps its volume vectors slab-local with one halo plane on
 * each side, sums the partial forward projections and the volume-domain
 * reductions with the all-reduce hook (kct_set_allreduce, required), and
 * exchanges halo planes through `fn`: send this rank's first / last interior
 * y plane (lo_plane / hi_plane, `count` floats each) and receive the
 * neighbouring ranks' adjacent planes into lo_halo (from rank - 1) /
 * hi_halo (from rank + 1); buffers without a neighbour are left untouched.
 * fn = NULL leaves slab mode.  Not part of the reference (the reference is
 * single-process). */
typedef int (*kct_halo_fn)(void* ctx, const void* lo_plane, const void* hi_plane, void* lo_halo,
                           void* hi_halo, size_t count, void* stream);
int kct_set_slab(kct_projector* h, int rank, int world, int j0, int ny_global, kct_halo_fn fn,
                 void* ctx);

/* Library-owned NCCL communicator (ABI 4): the two hooks above served by
 * NCCL itself — ncclAllReduce for the sums, one grouped ncclSend / ncclRecv
 * pair per neighbour for the halo planes — enqueued on the solver's stream
 * with no host synchronisation and no callback into the caller's runtime, so
 * a C++ host (kryct_b200.hpp) runs multi-GPU solves without Python.  One
 * process per GPU; NCCL is bound at run time (the libnccl.so.2 already loaded
 * in the process, else the system's; KCT_NCCL_LIB overrides), the library
 * itself does not link it.  Not part of the reference (single-process,
 * OpenMP only: projector.hpp:178-181).
 *   kct_comm_unique_id  fill `id` (KCT_COMM_ID_BYTES) on one rank; the caller
 *                       distributes it (file, MPI, torch.distributed, ...)
 *   kct_comm_create     join as `rank` of `world` on CUDA device `device`, which
 *                       becomes the calling thread's current device (< 0: stay
 *                       on the current device); collective over the ranks
 *   kct_comm_allreduce  in-place sum (dtype 0 = float32, 1 = float64) or,
 *                       op = 1, maximum, of a device buffer over the ranks
 *   kct_comm_allreduce_host  the same for a host buffer, staged through a
 *                       temporary device buffer (joining the ranks' result
 *                       slabs once per solve; not for the iteration path)
 *   kct_use_comm        kct_set_allreduce with the communicator's all-reduce
 *                       (angle-sharded mode); comm = NULL: single-process
 *   kct_use_comm_slab   kct_set_allreduce + kct_set_slab (rank and world from
 *                       the communicator) with the communicator's exchange */
#define KCT_COMM_ID_BYTES 128
typedef struct kct_comm kct_comm;
int kct_comm_unique_id(void* id);
int kct_comm_create(int rank, int world, const void* id, int device, kct_comm** out);
int kct_comm_destroy(kct_comm* c);
int kct_comm_rank(const kct_comm* c);
int kct_comm_world(const kct_comm* c);
int kct_comm_allreduce(kct_comm* c, void* buf, size_t count, int dtype, int op, void* stream);
int kct_comm_allreduce_host(kct_comm* c, void* buf, size_t count, int dtype, int op);
int kct_use_comm(kct_projector* h, kct_comm* c);
int kct_use_comm_slab(kct_projector* h, kct_comm* c, int j0, int ny_global);

/* Work-balanced y-slab boundaries for `world` ranks (world + 1 ints, bounds[0]
 * = 0, bounds[world] = ny): contiguous y-plane ranges of about equal
 * backprojection work — the number of (voxel column, angle) pairs of a plane
 * that project onto the detector's u extent, counted over a full circle of 64
 * views of this system so that every scan of one system gets the same slabs —
 * interior boundaries on multiples of 4 planes (whole adjoint bricks).  Host
 * arithmetic only. */
int kct_slab_bounds(const kct_grid* grid, const kct_geometry* geom, int world, int* bounds);

/* ---- solvers ---------------------------------------------------------- */
/* cgls_recon (recon.hpp:312-315 -> baseline_solve :274-307 -> cgls krylov.hpp:59-127).
 * b: N floats, x0: M floats or NULL (zeros), ground_truth: M or NULL,
 * x_out: M floats.  All arrays share `mem` and `layout`. */
int kct_cgls_recon(kct_projector* h, const float* b, size_t iters, const float* x0,
                   const float* ground_truth, double tolerance, float* x_out,
                   kct_report* report, int mem, int layout, void* stream);

/* irn_tv / irn_piple / irn_piccs (recon.hpp:252-270 -> irn_solve :169-247).
 * prior: M floats (ignored for KCT_KIND_TV, may be NULL then). */
int kct_irn(kct_projector* h, int kind, const float* b, const float* prior, const float* x0,
            const float* ground_truth, const kct_reg_params* params, float* x_out,
            kct_report* report, int mem, int layout, void* stream);

/* Convenience wrapper with the irn_piccs signature (recon.hpp:267-270). */
int kct_irn_piccs(kct_projector* h, const float* b, const float* prior, const float* x0,
                  const float* ground_truth, const kct_reg_params* params, float* x_out,
                  kct_report* report, int mem, int layout, void* stream);

/* One row block of a vertically stacked system (ScaledBlock, linear_map.hpp:152-157):
 * scale * diag(weights) * map.  `weights` is the DiagonalMap a caller composes
 * on the left of the map (compose(DiagonalMap(w), map), linear_map.hpp:82-150;
 * recon.hpp:211-217 builds the reweighted TV blocks this way); range-sized,
 * same mem / layout as the other arrays; NULL = no diagonal.  (ABI 3) */
typedef struct kct_stack_block {
    int map;      /* enum kct_map */
    double scale;
    const float* weights;
} kct_stack_block;

/* cgls(const LinearMap&, b, x0, KrylovConfig) (krylov.hpp:59-127) on a
 * caller-assembled StackedMap (linear_map.hpp:159-216), device-resident: the
 * iteration vectors never leave the GPU (the alternative, driving the
 * reference's own cgls through kct_forward_f64 / kct_adjoint_f64, pays two
 * PCIe copies and two float64 conversions per operator application).
 * b: the concatenated right-hand side, block by block (N / 3M / M floats);
 * x0: M floats or NULL (zeros); x_out: M floats.  Volume-shaped pieces (x0,
 * x_out, each of a DIFF block's three components, IDENTITY blocks, and the
 * weights of those blocks) use `layout`'s volume order, PROJECTOR blocks its
 * projection order.  report: residual_history / wall_times (capacity
 * max_iters), residual_count = SolveTrace::iterations, converged, breakdown.
 * The per-iteration hook (kct_set_iterate_hook) is served as in the drivers.
 * Single-process only (KCT_ERR_CONFIG in the sharded solver modes). */
int kct_cgls_stack(kct_projector* h, const kct_stack_block* blocks, size_t n_blocks,
                   const float* b, const float* x0, size_t max_iters, double tolerance,
                   float* x_out, kct_report* report, int mem, int layout, void* stream);

/* resolve_tau (recon.hpp:60-66) over a float32 host array (NULL/0 = empty). */
double kct_resolve_tau(double tau, const float* reference, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* KCT_H */
