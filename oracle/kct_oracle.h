/*
 * kct_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, float64 restatement of the reference kryct hot path, used as the
 * parity checker for the CUDA library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  It is never part of the
 * product path.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/kryct/).
 *
 * Layouts are the reference's: volumes x-fastest, projections u-fastest.
 */
#ifndef KCT_ORACLE_H
#define KCT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/kct.h"

#ifdef __cplusplus
extern "C" {
#endif

/* 0 ok, 2 config error (message via ora_last_error) */
const char* ora_last_error(void);
void ora_set_threads(int n);

/* projector.hpp:24-39 */
void ora_source_position(const kct_geometry* g, int ia, double out[3]);
void ora_detector_pixel_center(const kct_geometry* g, int ia, int iu, int iv, double out[3]);

/* projector.hpp:53-131 — materialised ray (trace_ray :149-157).  Writes up to
 * cap visits; returns the number of visits (may exceed cap).  t_io[2] gets
 * [t_entry, t_exit]. */
size_t ora_trace_ray(const kct_grid* grid, const double src[3], const double dst[3],
                     uint64_t* voxels, double* lengths, size_t cap, double t_io[2]);

/* projector.hpp:194-204 / :226-261 */
int ora_forward(const kct_grid* grid, const kct_geometry* g, const double* vol, double* proj);
int ora_adjoint(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol);
uint64_t ora_count_nnz(const kct_grid* grid, const kct_geometry* g);

/* diffreg.hpp:34-76, :118-156 */
void ora_diff(int nx, int ny, int nz, const double* x, double* out3m);
void ora_diff_adjoint(int nx, int ny, int nz, const double* y3m, double* out);
int ora_tv_weights(const double* grad3m, size_t m, double tau, double* w3m);
double ora_smoothed_tv(const double* grad3m, size_t m, double tau);

/* recon.hpp:60-66 */
double ora_resolve_tau(double tau, const double* ref, size_t n);

/* recon.hpp:312-315 (cgls_recon) and recon.hpp:169-247 (irn_solve) with
 * krylov.hpp:59-127 (cgls) inside.  Histories follow kct_report. */
int ora_cgls_recon(const kct_grid* grid, const kct_geometry* g, const double* b, size_t iters,
                   const double* x0, const double* ground_truth, double tol, double* x_out,
                   kct_report* rep);
/* cgls (krylov.hpp:59-127) on a caller-assembled StackedMap (linear_map.hpp:159-216):
 * block i = scales[i] * diag(weights[i]) * map(maps[i]) (enum kct_map; weights[i] NULL = none).
 * x: in x0, out solution (M); b: concatenated rhs; res_hist capacity max_iters. */
int ora_cgls_stack(const kct_grid* grid, const kct_geometry* g, size_t n_blocks, const int* maps,
                   const double* scales, const double* const* weights, const double* b, double* x,
                   size_t max_iters, double tol, double* res_hist, size_t* iterations,
                   int* converged, int* breakdown);

int ora_irn(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
            const double* prior, const double* x0, const double* ground_truth,
            const kct_reg_params* p, double* x_out, kct_report* rep);

/* fdk.hpp:50-139 (FFT ramp filter detail/fft.hpp:23-49) */
int ora_fdk(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol);

/* recon.hpp:93-120 */
double ora_objective(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
                     const double* x, const double* prior, double alpha, double lambda,
                     double tau);

#ifdef __cplusplus
}
#endif
#endif
