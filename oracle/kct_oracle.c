/*
 * kct_oracle.c — TEST INFRASTRUCTURE ONLY (see kct_oracle.h).
 *
 * Plain-C float64 restatement of the reference kryct algorithms on the
 * PICCS-Krylov hot path.  It is the checker the CUDA library is compared to;
 * it is pinned in turn against the reference itself (oracle/_ref, built from
 * the reference headers by oracle/Makefile) through tests/golden fixtures.
 * Paths in citations are relative to /root/reference/proj/include/kryct/.
 */
#include "kct_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[256];
static int g_threads = 0;

const char* ora_last_error(void) { return g_err; }
void ora_set_threads(int n) { g_threads = n; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int nthreads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- validation: types.hpp:72-77, :152-160; projector.hpp:162-168 ---- */
static int validate(const kct_grid* grid, const kct_geometry* g) {
    if (grid->nx < 1 || grid->ny < 1 || grid->nz < 1) return fail(2, "grid dims must be positive");
    if (!(grid->sx > 0) || !(grid->sy > 0) || !(grid->sz > 0))
        return fail(2, "voxel spacing must be strictly positive");
    if (!(g->dso > 0.0) || !(g->dsd > g->dso)) return fail(2, "geometry requires dsd > dso > 0");
    if (g->nu < 1 || g->nv < 1) return fail(2, "detector must have at least one pixel per axis");
    if (!(g->pu > 0) || !(g->pv > 0)) return fail(2, "detector pixel pitch must be positive");
    if (g->n_angles < 1) return fail(2, "geometry requires at least one angle");
    const double hi[3] = {grid->ox + grid->nx * grid->sx, grid->oy + grid->ny * grid->sy,
                          grid->oz + grid->nz * grid->sz};
    for (int ia = 0; ia < g->n_angles; ++ia) {
        double s[3];
        ora_source_position(g, ia, s);
        if (s[0] > grid->ox && s[0] < hi[0] && s[1] > grid->oy && s[1] < hi[1] &&
            s[2] > grid->oz && s[2] < hi[2])
            return fail(2, "source position lies inside the volume");
    }
    return 0;
}

/* projector.hpp:24-27 */
void ora_source_position(const kct_geometry* g, int ia, double out[3]) {
    const double t = g->angles[ia];
    out[0] = g->dso * cos(t);
    out[1] = g->dso * sin(t);
    out[2] = 0.0;
}

/* projector.hpp:30-39 */
void ora_detector_pixel_center(const kct_geometry* g, int ia, int iu, int iv, double out[3]) {
    const double t = g->angles[ia];
    const double c = cos(t), s = sin(t);
    const double cx = -(g->dsd - g->dso) * c, cy = -(g->dsd - g->dso) * s;
    const double du = (iu + 0.5 - 0.5 * g->nu) * g->pu + g->offset_u;
    const double dv = (iv + 0.5 - 0.5 * g->nv) * g->pv + g->offset_v;
    out[0] = cx + du * -s;
    out[1] = cy + du * c;
    out[2] = dv;
}

/* ---- Siddon traversal: projector.hpp:53-131 --------------------------- */
enum { V_FWD = 0, V_ADJ = 1, V_COUNT = 2, V_TRACE = 3 };

typedef struct {
    int mode;
    const double* vol; /* V_FWD */
    double acc;
    double* out;       /* V_ADJ */
    double w;
    uint64_t count;    /* V_COUNT / V_TRACE */
    uint64_t* tv;
    double* tl;
    size_t cap;
} visitor;

static inline void visit(visitor* v, size_t lin, double len) {
    switch (v->mode) {
    case V_FWD: v->acc += len * v->vol[lin]; break;
    case V_ADJ: v->out[lin] += len * v->w; break;
    case V_TRACE:
        if (v->count < v->cap) {
            v->tv[v->count] = lin;
            v->tl[v->count] = len;
        }
        /* fallthrough */
    default: v->count++; break;
    }
}

static void traverse(const kct_grid* grid, const double src[3], const double dst[3], visitor* vis,
                     double t_io[2]) {
    const double bmin[3] = {grid->ox, grid->oy, grid->oz};
    const double sp[3] = {grid->sx, grid->sy, grid->sz};
    const int n[3] = {grid->nx, grid->ny, grid->nz};
    const double bmax[3] = {bmin[0] + n[0] * sp[0], bmin[1] + n[1] * sp[1],
                            bmin[2] + n[2] * sp[2]};
    const double d[3] = {dst[0] - src[0], dst[1] - src[1], dst[2] - src[2]};
    const double ray_len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (t_io) t_io[0] = t_io[1] = 0.0;
    if (ray_len == 0.0) return;

    double t0 = 0.0, t1 = 1.0; /* slab clip :70-82 */
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0) {
            double ta = (bmin[a] - src[a]) / d[a];
            double tb = (bmax[a] - src[a]) / d[a];
            if (ta > tb) { double tt = ta; ta = tb; tb = tt; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        } else if (src[a] <= bmin[a] || src[a] >= bmax[a]) {
            return;
        }
    }
    if (!(t0 < t1)) return;

    int idx[3], step[3]; /* entry voxel :93-110 */
    double t_next[3], t_delta[3];
    const size_t stride[3] = {1, (size_t)n[0], (size_t)n[0] * (size_t)n[1]};
    for (int a = 0; a < 3; ++a) {
        const double p = src[a] + t0 * d[a];
        int i = (int)floor((p - bmin[a]) / sp[a]);
        idx[a] = i < 0 ? 0 : (i > n[a] - 1 ? n[a] - 1 : i);
        if (d[a] > 0.0) {
            step[a] = 1;
            t_delta[a] = sp[a] / d[a];
            t_next[a] = (bmin[a] + (idx[a] + 1) * sp[a] - src[a]) / d[a];
        } else if (d[a] < 0.0) {
            step[a] = -1;
            t_delta[a] = -sp[a] / d[a];
            t_next[a] = (bmin[a] + idx[a] * sp[a] - src[a]) / d[a];
        } else {
            step[a] = 0;
            t_delta[a] = INFINITY;
            t_next[a] = INFINITY;
        }
    }
    if (t_io) { t_io[0] = t0; t_io[1] = t1; }
    size_t lin = idx[0] * stride[0] + idx[1] * stride[1] + idx[2] * stride[2];
    double t = t0;
    for (;;) { /* incremental walk :116-129 */
        int m = 0;
        if (t_next[1] < t_next[m]) m = 1;
        if (t_next[2] < t_next[m]) m = 2;
        const double t_stop = t_next[m] < t1 ? t_next[m] : t1;
        const double len = (t_stop - t) * ray_len;
        if (len > 0.0) visit(vis, lin, len);
        if (t_next[m] >= t1) break;
        t = t_next[m];
        idx[m] += step[m];
        if (idx[m] < 0 || idx[m] >= n[m]) break;
        lin = step[m] > 0 ? lin + stride[m] : lin - stride[m];
        t_next[m] += t_delta[m];
    }
}

size_t ora_trace_ray(const kct_grid* grid, const double src[3], const double dst[3],
                     uint64_t* voxels, double* lengths, size_t cap, double t_io[2]) {
    visitor v = {0};
    v.mode = V_TRACE;
    v.tv = voxels;
    v.tl = lengths;
    v.cap = cap;
    traverse(grid, src, dst, &v, t_io);
    return (size_t)v.count;
}

/* project_forward_angle / project_forward: projector.hpp:173-204 */
int ora_forward(const kct_grid* grid, const kct_geometry* g, const double* vol, double* proj) {
    int rc = validate(grid, g);
    if (rc) return rc;
    const int nu = g->nu, nv = g->nv;
    const long total = (long)g->n_angles * nv;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads())
    for (long r = 0; r < total; ++r) {
        const int ia = (int)(r / nv), iv = (int)(r % nv);
        double src[3], dst[3];
        ora_source_position(g, ia, src);
        for (int iu = 0; iu < nu; ++iu) {
            ora_detector_pixel_center(g, ia, iu, iv, dst);
            visitor v = {0};
            v.mode = V_FWD;
            v.vol = vol;
            traverse(grid, src, dst, &v, NULL);
            proj[(size_t)iu + (size_t)nu * ((size_t)iv + (size_t)nv * ia)] = v.acc;
        }
    }
    return 0;
}

/* project_adjoint_angle_accumulate / project_adjoint: projector.hpp:207-261.
 * Deterministic for a fixed thread count: angle blocks accumulate into
 * private buffers that are reduced in fixed order (as the reference does). */
int ora_adjoint(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol) {
    int rc = validate(grid, g);
    if (rc) return rc;
    const size_t m = (size_t)grid->nx * grid->ny * grid->nz;
    const int nu = g->nu, nv = g->nv, na = g->n_angles;
    int nt = nthreads();
    const size_t budget = (size_t)4 << 30; /* cap private buffers at 4 GiB */
    if ((size_t)nt * m * sizeof(double) > budget) nt = (int)(budget / (m * sizeof(double)));
    if (nt < 1) nt = 1;
    if (nt > na) nt = na;
    memset(vol, 0, m * sizeof(double));
    double* part = nt > 1 ? (double*)calloc((size_t)nt * m, sizeof(double)) : NULL;
    if (nt > 1 && !part) nt = 1;
#pragma omp parallel num_threads(nt)
    {
#ifdef _OPENMP
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
        double* mine = nt > 1 ? part + (size_t)tid * m : vol;
#pragma omp for schedule(static)
        for (int ia = 0; ia < na; ++ia) {
            double src[3], dst[3];
            ora_source_position(g, ia, src);
            for (int iv = 0; iv < nv; ++iv)
                for (int iu = 0; iu < nu; ++iu) {
                    const double w = proj[(size_t)iu + (size_t)nu * ((size_t)iv + (size_t)nv * ia)];
                    if (w == 0.0) continue;
                    ora_detector_pixel_center(g, ia, iu, iv, dst);
                    visitor v = {0};
                    v.mode = V_ADJ;
                    v.out = mine;
                    v.w = w;
                    traverse(grid, src, dst, &v, NULL);
                }
        }
    }
    if (nt > 1) {
        for (int t = 0; t < nt; ++t) {
            const double* p = part + (size_t)t * m;
            for (size_t i = 0; i < m; ++i) vol[i] += 1.0 * p[i];
        }
        free(part);
    }
    return 0;
}

uint64_t ora_count_nnz(const kct_grid* grid, const kct_geometry* g) {
    if (validate(grid, g)) return 0;
    const int nu = g->nu, nv = g->nv;
    const long total = (long)g->n_angles * nv;
    uint64_t sum = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : sum) num_threads(nthreads())
    for (long r = 0; r < total; ++r) {
        const int ia = (int)(r / nv), iv = (int)(r % nv);
        double src[3], dst[3];
        ora_source_position(g, ia, src);
        for (int iu = 0; iu < nu; ++iu) {
            ora_detector_pixel_center(g, ia, iu, iv, dst);
            visitor v = {0};
            v.mode = V_COUNT;
            traverse(grid, src, dst, &v, NULL);
            sum += v.count;
        }
    }
    return sum;
}

/* ---- difference operator and weights: diffreg.hpp --------------------- */
/* DiffOperator::apply :34-49 */
void ora_diff(int nx, int ny, int nz, const double* x, double* out) {
    const size_t m = (size_t)nx * ny * nz, sy = (size_t)nx, sz = (size_t)nx * ny;
    size_t v = 0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i, ++v) {
                out[v] = i + 1 < nx ? x[v + 1] - x[v] : 0.0;
                out[m + v] = j + 1 < ny ? x[v + sy] - x[v] : 0.0;
                out[2 * m + v] = k + 1 < nz ? x[v + sz] - x[v] : 0.0;
            }
}

/* DiffOperator::apply_adjoint :51-76 */
void ora_diff_adjoint(int nx, int ny, int nz, const double* y, double* out) {
    const size_t m = (size_t)nx * ny * nz, sy = (size_t)nx, sz = (size_t)nx * ny;
    memset(out, 0, m * sizeof(double));
    size_t v = 0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i, ++v) {
                if (i + 1 < nx) { out[v] -= y[v]; out[v + 1] += y[v]; }
                if (j + 1 < ny) { out[v] -= y[m + v]; out[v + sy] += y[m + v]; }
                if (k + 1 < nz) { out[v] -= y[2 * m + v]; out[v + sz] += y[2 * m + v]; }
            }
}

/* tv_weights :142-156 */
int ora_tv_weights(const double* g, size_t m, double tau, double* w) {
    if (!(tau > 0.0)) return fail(2, "reweighting requires tau > 0");
    for (size_t v = 0; v < m; ++v) {
        const double m2 = g[v] * g[v] + g[m + v] * g[m + v] + g[2 * m + v] * g[2 * m + v];
        const double wv = 1.0 / sqrt(sqrt(m2 + tau * tau));
        w[v] = wv;
        w[m + v] = wv;
        w[2 * m + v] = wv;
    }
    return 0;
}

/* smoothed_tv :118-126 */
double ora_smoothed_tv(const double* g, size_t m, double tau) {
    double s = 0.0;
    for (size_t v = 0; v < m; ++v)
        s += sqrt(g[v] * g[v] + g[m + v] * g[m + v] + g[2 * m + v] * g[2 * m + v] + tau * tau);
    return s;
}

/* resolve_tau: recon.hpp:60-66 */
double ora_resolve_tau(double tau, const double* ref, size_t n) {
    if (tau > 0.0) return tau;
    if (!ref || n == 0) return 1e-4;
    double lo = ref[0], hi = ref[0];
    for (size_t i = 1; i < n; ++i) {
        if (ref[i] < lo) lo = ref[i];
        if (ref[i] > hi) hi = ref[i];
    }
    const double range = hi - lo;
    return range > 0.0 ? (1e-4 * range > 1e-8 ? 1e-4 * range : 1e-8) : 1e-4;
}

/* ---- vector kernels: vector_ops.hpp:15-45 (sequential, left to right) -- */
static double dot(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static void axpy(double c, const double* x, double* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] += c * x[i];
}

/* ---- stacked operator: linear_map.hpp:84-216 ------------------------- */
typedef struct {
    const kct_grid* grid;
    const kct_geometry* g;
    size_t m, n;
    double alpha, lambda;
    const double* w1; /* 3M, NULL = block absent */
    const double* w2; /* 3M (piccs) */
    int identity;     /* piple: lambda*I block */
    double* tmp3;     /* 3M scratch */
    double* tmpm;     /* M scratch */
    /* caller-assembled stack (ora_cgls_stack): nblk > 0 replaces the fixed layout above */
    size_t nblk;
    const int* maps;            /* enum kct_map */
    const double* scales;       /* ScaledBlock::scale */
    const double* const* wts;   /* DiagonalMap composed on the left, NULL = none */
    double* tmpn;               /* N scratch */
} stack_op;

static size_t block_len(const stack_op* s, size_t i) {
    return s->maps[i] == KCT_MAP_PROJECTOR ? s->n : (s->maps[i] == KCT_MAP_DIFF ? 3 * s->m : s->m);
}

static size_t stack_range(const stack_op* s) {
    if (s->nblk) {
        size_t t = 0;
        for (size_t i = 0; i < s->nblk; ++i) t += block_len(s, i);
        return t;
    }
    size_t r = s->n;
    if (s->w1) r += 3 * s->m;
    if (s->identity) r += s->m;
    else if (s->w2) r += 3 * s->m;
    return r;
}

static void scale(double c, double* x, size_t n) {
    for (size_t i = 0; i < n; ++i) x[i] *= c;
}

/* StackedMap::apply :185-193 over caller blocks; a weighted block is
 * ComposedMap(DiagonalMap(w), map) (:82-150): map first, then diag(w) */
static void gstack_apply(const stack_op* s, const double* x, double* out) {
    const kct_grid* gr = s->grid;
    size_t off = 0;
    for (size_t b = 0; b < s->nblk; ++b) {
        const size_t len = block_len(s, b);
        double* o = out + off;
        if (s->maps[b] == KCT_MAP_PROJECTOR) ora_forward(gr, s->g, x, o);
        else if (s->maps[b] == KCT_MAP_DIFF) ora_diff(gr->nx, gr->ny, gr->nz, x, o);
        else for (size_t i = 0; i < len; ++i) o[i] = x[i];
        if (s->wts[b]) for (size_t i = 0; i < len; ++i) o[i] = s->wts[b][i] * o[i];
        if (s->scales[b] != 1.0) scale(s->scales[b], o, len);
        off += len;
    }
}

/* StackedMap::apply_adjoint :195-205 */
static void gstack_adjoint(const stack_op* s, const double* y, double* out) {
    const kct_grid* gr = s->grid;
    memset(out, 0, s->m * sizeof(double));
    size_t off = 0;
    for (size_t b = 0; b < s->nblk; ++b) {
        const size_t len = block_len(s, b);
        const double* in = y + off;
        if (s->wts[b]) {
            double* t = s->maps[b] == KCT_MAP_PROJECTOR ? s->tmpn : s->tmp3;
            for (size_t i = 0; i < len; ++i) t[i] = s->wts[b][i] * in[i];
            in = t;
        }
        if (s->maps[b] == KCT_MAP_PROJECTOR) ora_adjoint(gr, s->g, in, s->tmpm);
        else if (s->maps[b] == KCT_MAP_DIFF) ora_diff_adjoint(gr->nx, gr->ny, gr->nz, in, s->tmpm);
        else memcpy(s->tmpm, in, len * sizeof(double));
        axpy(s->scales[b], s->tmpm, out, s->m);
        off += len;
    }
}

/* StackedMap::apply :185-193 with ComposedMap(DiagonalMap, D) blocks */
static void stack_apply(const stack_op* s, const double* x, double* out) {
    if (s->nblk) { gstack_apply(s, x, out); return; }
    const kct_grid* gr = s->grid;
    ora_forward(gr, s->g, x, out);
    size_t off = s->n;
    if (s->w1) {
        ora_diff(gr->nx, gr->ny, gr->nz, x, s->tmp3);
        for (size_t i = 0; i < 3 * s->m; ++i) out[off + i] = s->w1[i] * s->tmp3[i];
        if (s->alpha != 1.0) scale(s->alpha, out + off, 3 * s->m);
        off += 3 * s->m;
    }
    if (s->identity) {
        for (size_t i = 0; i < s->m; ++i) out[off + i] = x[i];
        if (s->lambda != 1.0) scale(s->lambda, out + off, s->m);
    } else if (s->w2) {
        ora_diff(gr->nx, gr->ny, gr->nz, x, s->tmp3);
        for (size_t i = 0; i < 3 * s->m; ++i) out[off + i] = s->w2[i] * s->tmp3[i];
        if (s->lambda != 1.0) scale(s->lambda, out + off, 3 * s->m);
    }
}

/* StackedMap::apply_adjoint :195-205 */
static void stack_adjoint(const stack_op* s, const double* y, double* out) {
    if (s->nblk) { gstack_adjoint(s, y, out); return; }
    const kct_grid* gr = s->grid;
    memset(out, 0, s->m * sizeof(double));
    ora_adjoint(gr, s->g, y, s->tmpm);
    axpy(1.0, s->tmpm, out, s->m);
    size_t off = s->n;
    if (s->w1) {
        for (size_t i = 0; i < 3 * s->m; ++i) s->tmp3[i] = s->w1[i] * y[off + i];
        ora_diff_adjoint(gr->nx, gr->ny, gr->nz, s->tmp3, s->tmpm);
        axpy(s->alpha, s->tmpm, out, s->m);
        off += 3 * s->m;
    }
    if (s->identity) {
        axpy(s->lambda, y + off, out, s->m);
    } else if (s->w2) {
        for (size_t i = 0; i < 3 * s->m; ++i) s->tmp3[i] = s->w2[i] * y[off + i];
        ora_diff_adjoint(gr->nx, gr->ny, gr->nz, s->tmp3, s->tmpm);
        axpy(s->lambda, s->tmpm, out, s->m);
    }
}

/* ---- cgls: krylov.hpp:59-127 ----------------------------------------- */
typedef struct {
    size_t iterations;
    int converged, breakdown;
    double* res_hist; /* appended */
    size_t res_count;
    const double* gt;
    double* err_hist;
    size_t err_count;
} cgls_trace;

static double rel_error_span(const double* x, const double* ref, size_t n) { /* recon.hpp:124-132 */
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = x[i] - ref[i];
        num += d * d;
        den += ref[i] * ref[i];
    }
    return den > 0.0 ? sqrt(num / den) : sqrt(num);
}

static int cgls(const stack_op* A, const double* b, double* x, size_t max_iters, double tol,
                cgls_trace* tr) {
    const size_t dom = A->m, rng = stack_range(A);
    double* r = (double*)malloc(rng * sizeof(double));
    double* q = (double*)malloc(rng * sizeof(double));
    double* s = (double*)malloc(dom * sizeof(double));
    double* p = (double*)malloc(dom * sizeof(double));
    int rc = 0;
    stack_apply(A, x, r);
    for (size_t i = 0; i < rng; ++i) r[i] = b[i] - r[i];
    stack_adjoint(A, r, s);
    double gamma = dot(s, s, dom);
    if (!isfinite(gamma)) { rc = fail(3, "cgls: non-finite normal residual"); goto out; }
    if (gamma == 0.0) { tr->converged = 1; goto out; }
    double stop_tol = 0.0;
    if (tol > 0.0) {
        double ref2 = gamma;
        int nonzero = 0;
        for (size_t i = 0; i < dom; ++i)
            if (x[i] != 0.0) { nonzero = 1; break; }
        if (nonzero) {
            double* sb = (double*)malloc(dom * sizeof(double));
            stack_adjoint(A, b, sb);
            ref2 = dot(sb, sb, dom);
            free(sb);
        }
        stop_tol = tol * sqrt(ref2);
        if (sqrt(gamma) <= stop_tol) { tr->converged = 1; goto out; }
    }
    memcpy(p, s, dom * sizeof(double));
    for (size_t it = 1; it <= max_iters; ++it) {
        stack_apply(A, p, q);
        const double delta = dot(q, q, rng);
        if (!isfinite(delta)) { rc = fail(3, "cgls: non-finite iterate"); goto out; }
        if (delta == 0.0) { tr->breakdown = 1; break; }
        const double a = gamma / delta;
        axpy(a, p, x, dom);
        axpy(-a, q, r, rng);
        stack_adjoint(A, r, s);
        const double gamma_next = dot(s, s, dom);
        if (!isfinite(gamma_next)) { rc = fail(3, "cgls: non-finite iterate"); goto out; }
        tr->iterations = it;
        if (tr->res_hist) tr->res_hist[tr->res_count] = sqrt(dot(r, r, rng));
        tr->res_count++;
        if (tr->gt) {
            if (tr->err_hist) tr->err_hist[tr->err_count] = rel_error_span(x, tr->gt, dom);
            tr->err_count++;
        }
        if (sqrt(gamma_next) <= stop_tol) { tr->converged = 1; break; }
        const double beta = gamma_next / gamma;
        gamma = gamma_next;
        for (size_t i = 0; i < dom; ++i) p[i] = s[i] + beta * p[i];
    }
out:
    free(r); free(q); free(s); free(p);
    return rc;
}

/* cgls (krylov.hpp:59-127) on a caller-assembled StackedMap (linear_map.hpp:159-216).
 * x: in = x0, out = the solution; res_hist: capacity max_iters. */
int ora_cgls_stack(const kct_grid* grid, const kct_geometry* g, size_t n_blocks, const int* maps,
                   const double* scales, const double* const* weights, const double* b, double* x,
                   size_t max_iters, double tol, double* res_hist, size_t* iterations,
                   int* converged, int* breakdown) {
    int rc = validate(grid, g);
    if (rc) return rc;
    if (n_blocks == 0) return fail(2, "stack: needs at least one block");
    for (size_t i = 0; i < n_blocks; ++i)
        if (maps[i] != KCT_MAP_PROJECTOR && maps[i] != KCT_MAP_DIFF && maps[i] != KCT_MAP_IDENTITY)
            return fail(2, "stack: unknown block map");
    stack_op A = {0};
    A.grid = grid;
    A.g = g;
    A.m = (size_t)grid->nx * grid->ny * grid->nz;
    A.n = (size_t)g->n_angles * g->nu * g->nv;
    A.nblk = n_blocks;
    A.maps = maps;
    A.scales = scales;
    A.wts = weights;
    A.tmp3 = (double*)malloc(3 * A.m * sizeof(double));
    A.tmpm = (double*)malloc(A.m * sizeof(double));
    A.tmpn = (double*)malloc(A.n * sizeof(double));
    cgls_trace tr = {0};
    tr.res_hist = res_hist;
    rc = cgls(&A, b, x, max_iters, tol, &tr);
    if (iterations) *iterations = tr.iterations;
    if (converged) *converged = tr.converged;
    if (breakdown) *breakdown = tr.breakdown;
    free(A.tmp3); free(A.tmpm); free(A.tmpn);
    return rc;
}

/* evaluate_objective: recon.hpp:93-120 */
double ora_objective(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
                     const double* x, const double* prior, double alpha, double lambda,
                     double tau) {
    const size_t m = (size_t)grid->nx * grid->ny * grid->nz;
    const size_t n = (size_t)g->nu * g->nv * g->n_angles;
    double* ax = (double*)malloc(n * sizeof(double));
    double* gr = (double*)malloc(3 * m * sizeof(double));
    ora_forward(grid, g, x, ax);
    double obj = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = ax[i] - b[i];
        obj += d * d;
    }
    if (alpha != 0.0) {
        ora_diff(grid->nx, grid->ny, grid->nz, x, gr);
        obj += 2.0 * alpha * alpha * ora_smoothed_tv(gr, m, tau);
    }
    if (kind == KCT_KIND_PIPLE && lambda != 0.0) {
        double q = 0.0;
        for (size_t i = 0; i < m; ++i) {
            const double d = x[i] - prior[i];
            q += d * d;
        }
        obj += lambda * lambda * q;
    } else if (kind == KCT_KIND_PICCS && lambda != 0.0) {
        double* diff = (double*)malloc(m * sizeof(double));
        for (size_t i = 0; i < m; ++i) diff[i] = x[i] - prior[i];
        ora_diff(grid->nx, grid->ny, grid->nz, diff, gr);
        obj += 2.0 * lambda * lambda * ora_smoothed_tv(gr, m, tau);
        free(diff);
    }
    free(ax);
    free(gr);
    return obj;
}

static void rep_reset(kct_report* rep) {
    if (!rep) return;
    rep->objective_count = rep->residual_count = rep->error_count = rep->outer_count = 0;
    rep->solve_seconds = 0.0;
    rep->converged = rep->breakdown = 0;
}

/* cgls_recon / baseline_solve: recon.hpp:274-315 */
int ora_cgls_recon(const kct_grid* grid, const kct_geometry* g, const double* b, size_t iters,
                   const double* x0, const double* gt, double tol, double* x_out,
                   kct_report* rep) {
    int rc = validate(grid, g);
    if (rc) return rc;
    if (iters < 1) return fail(2, "reconstruction needs at least one iteration");
    const size_t m = (size_t)grid->nx * grid->ny * grid->nz;
    stack_op A = {grid, g, m, (size_t)g->nu * g->nv * g->n_angles, 1.0, 0.0, NULL, NULL, 0,
                  NULL, (double*)malloc(m * sizeof(double))};
    if (x0) memcpy(x_out, x0, m * sizeof(double));
    else memset(x_out, 0, m * sizeof(double));
    rep_reset(rep);
    cgls_trace tr = {0};
    tr.res_hist = rep ? rep->residual_history : NULL;
    tr.gt = gt;
    tr.err_hist = rep ? rep->error_history : NULL;
    const double t0 = now_s();
    rc = cgls(&A, b, x_out, iters, tol, &tr);
    free(A.tmpm);
    if (rc) return rc;
    if (rep) {
        rep->solve_seconds = now_s() - t0;
        rep->residual_count = tr.res_count;
        rep->error_count = tr.err_count;
        if (rep->objective_history)
            for (size_t i = 0; i < tr.res_count; ++i)
                rep->objective_history[i] = tr.res_hist[i] * tr.res_hist[i];
        rep->objective_count = tr.res_count;
        if (rep->outer_boundaries) rep->outer_boundaries[0] = tr.res_count;
        if (rep->outer_seconds) rep->outer_seconds[0] = rep->solve_seconds;
        rep->outer_count = 1;
        rep->converged = tr.converged;
        rep->breakdown = tr.breakdown;
    }
    return 0;
}

/* irn_solve: recon.hpp:141-247 */
int ora_irn(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
            const double* prior, const double* x0, const double* gt, const kct_reg_params* p,
            double* x_out, kct_report* rep) {
    int rc = validate(grid, g);
    if (rc) return rc;
    if (p->outer_iters < 1 || p->inner_iters < 1)
        return fail(2, "reconstruction needs at least one outer and one inner iteration");
    if (p->alpha < 0.0) return fail(2, "alpha must be non-negative");
    if (!isfinite(p->alpha) || !isfinite(p->lambda) || !isfinite(p->tau))
        return fail(2, "regularisation parameters must be finite");
    const double alpha = p->alpha;
    const double lambda = p->lambda < 0.0 ? alpha : p->lambda;
    const size_t m = (size_t)grid->nx * grid->ny * grid->nz;
    const size_t n = (size_t)g->nu * g->nv * g->n_angles;
    if (kind != KCT_KIND_TV && !prior) return fail(2, "prior volume required");
    const double* tau_ref = x0 ? x0 : ((kind != KCT_KIND_TV && lambda != 0.0) ? prior : NULL);
    const double tau = ora_resolve_tau(p->tau, tau_ref, tau_ref ? m : 0);
    const double* pr = kind == KCT_KIND_TV ? NULL : prior;

    if (x0) memcpy(x_out, x0, m * sizeof(double));
    else memset(x_out, 0, m * sizeof(double));
    rep_reset(rep);
    if (rep) rep->tau = tau;

    double* w1 = (double*)malloc(3 * m * sizeof(double));
    double* w2 = (double*)malloc(3 * m * sizeof(double));
    double* tmp3 = (double*)malloc(3 * m * sizeof(double));
    double* tmpm = (double*)malloc(m * sizeof(double));
    double* rhs = (double*)malloc((n + 6 * m) * sizeof(double));
    double* start = (double*)malloc(m * sizeof(double));

    const double t_start = now_s();
    double obj = ora_objective(grid, g, kind, b, x_out, pr, alpha, lambda, tau);
    if (rep && rep->objective_history) rep->objective_history[0] = obj;
    size_t n_obj = 1, n_res = 0, n_err = 0;
    for (size_t cycle = 0; cycle < p->outer_iters; ++cycle) {
        const double t_cycle = now_s();
        stack_op A = {grid, g, m, n, alpha, lambda, NULL, NULL, 0, tmp3, tmpm};
        memcpy(rhs, b, n * sizeof(double));
        size_t off = n;
        if (alpha != 0.0) {
            ora_diff(grid->nx, grid->ny, grid->nz, x_out, tmp3);
            ora_tv_weights(tmp3, m, tau, w1);
            A.w1 = w1;
            memset(rhs + off, 0, 3 * m * sizeof(double));
            off += 3 * m;
        }
        if (kind == KCT_KIND_PIPLE && lambda != 0.0) {
            A.identity = 1;
            for (size_t i = 0; i < m; ++i) rhs[off + i] = lambda * pr[i];
        } else if (kind == KCT_KIND_PICCS && lambda != 0.0) {
            for (size_t i = 0; i < m; ++i) tmpm[i] = x_out[i] - pr[i];
            ora_diff(grid->nx, grid->ny, grid->nz, tmpm, tmp3);
            ora_tv_weights(tmp3, m, tau, w2);
            A.w2 = w2;
            ora_diff(grid->nx, grid->ny, grid->nz, pr, tmp3);
            for (size_t i = 0; i < 3 * m; ++i) rhs[off + i] = lambda * (w2[i] * tmp3[i]);
        }
        if (p->warm_start) memcpy(start, x_out, m * sizeof(double));
        else memset(start, 0, m * sizeof(double));
        cgls_trace tr = {0};
        tr.res_hist = rep && rep->residual_history ? rep->residual_history + n_res : NULL;
        tr.gt = gt;
        tr.err_hist = rep && rep->error_history ? rep->error_history + n_err : NULL;
        rc = cgls(&A, rhs, start, p->inner_iters, p->inner_tolerance, &tr);
        if (rc) break;
        memcpy(x_out, start, m * sizeof(double));
        n_res += tr.res_count;
        n_err += tr.err_count;
        if (rep) {
            rep->converged = tr.converged;
            rep->breakdown = tr.breakdown;
            if (rep->outer_boundaries) rep->outer_boundaries[cycle] = n_res;
        }
        obj = ora_objective(grid, g, kind, b, x_out, pr, alpha, lambda, tau);
        if (rep && rep->objective_history) rep->objective_history[n_obj] = obj;
        n_obj++;
        if (rep && rep->outer_seconds) rep->outer_seconds[cycle] = now_s() - t_cycle;
        if (rep) rep->outer_count = cycle + 1;
    }
    if (rep) {
        rep->solve_seconds = now_s() - t_start;
        rep->objective_count = n_obj;
        rep->residual_count = n_res;
        rep->error_count = n_err;
    }
    free(w1); free(w2); free(tmp3); free(tmpm); free(rhs); free(start);
    return rc;
}

/* ---- FDK: fdk.hpp:50-139 with detail/fft.hpp:23-49 -------------------- */
typedef struct { double re, im; } cpx;

static void fft_inplace(cpx* a, size_t n, int inverse) { /* fft.hpp:23-49 */
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { cpx t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const double ang = (inverse ? 2.0 : -2.0) * M_PI / (double)len;
        const cpx wl = {cos(ang), sin(ang)};
        for (size_t i = 0; i < n; i += len) {
            cpx w = {1.0, 0.0};
            for (size_t k = 0; k < len / 2; ++k) {
                const cpx u = a[i + k], x = a[i + k + len / 2];
                const cpx v = {x.re * w.re - x.im * w.im, x.re * w.im + x.im * w.re};
                a[i + k] = (cpx){u.re + v.re, u.im + v.im};
                a[i + k + len / 2] = (cpx){u.re - v.re, u.im - v.im};
                const cpx nw = {w.re * wl.re - w.im * wl.im, w.re * wl.im + w.im * wl.re};
                w = nw;
            }
        }
    }
    if (inverse)
        for (size_t i = 0; i < n; ++i) { a[i].re /= (double)n; a[i].im /= (double)n; }
}

int ora_fdk(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol) {
    int rc = validate(grid, g);
    if (rc) return rc;
    if (g->n_angles < 2) return fail(2, "fdk needs at least two projection angles");
    const int nu = g->nu, nv = g->nv, na = g->n_angles;
    const size_t per = (size_t)nu * nv;
    const double mag = g->dso / g->dsd;
    const double du = g->pu * mag, dv = g->pv * mag;
    const double u0 = (0.5 - 0.5 * nu) * du + g->offset_u * mag;
    const double v0 = (0.5 - 0.5 * nv) * dv + g->offset_v * mag;
    size_t pad = 1;
    while (pad < 2 * (size_t)nu) pad <<= 1;
    cpx* ramp = (cpx*)calloc(pad, sizeof(cpx)); /* ramlak_response fdk.hpp:30-42 */
    const double inv = 1.0 / (du * du);
    ramp[0].re = 0.25 * inv;
    for (size_t k = 1; k < pad / 2; k += 2) {
        const double v = -inv / (M_PI * M_PI * (double)k * (double)k);
        ramp[k].re = v;
        ramp[pad - k].re = v;
    }
    fft_inplace(ramp, pad, 0);
    double* filtered = (double*)malloc((size_t)na * per * sizeof(double));
#pragma omp parallel num_threads(nthreads())
    {
        cpx* row = (cpx*)malloc(pad * sizeof(cpx));
#pragma omp for schedule(static)
        for (long r = 0; r < (long)na * nv; ++r) {
            const int ia = (int)(r / nv), iv = (int)(r % nv);
            const double v = v0 + iv * dv;
            memset(row, 0, pad * sizeof(cpx));
            const size_t base = ia * per + (size_t)iv * nu;
            for (int iu = 0; iu < nu; ++iu) {
                const double u = u0 + iu * du;
                const double cosw = g->dso / sqrt(g->dso * g->dso + u * u + v * v);
                row[iu].re = proj[base + iu] * cosw;
            }
            fft_inplace(row, pad, 0);
            for (size_t i = 0; i < pad; ++i) {
                const cpx a = row[i], b = ramp[i];
                row[i] = (cpx){a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
            }
            fft_inplace(row, pad, 1);
            for (int iu = 0; iu < nu; ++iu) filtered[base + iu] = row[iu].re * du;
        }
        free(row);
    }
    const double scale = 0.5 * (2.0 * M_PI / (double)na);
#pragma omp parallel for schedule(static) num_threads(nthreads())
    for (int k = 0; k < grid->nz; ++k) {
        const double z = grid->oz + (k + 0.5) * grid->sz;
        for (int j = 0; j < grid->ny; ++j) {
            const double y = grid->oy + (j + 0.5) * grid->sy;
            for (int i = 0; i < grid->nx; ++i) {
                const double x = grid->ox + (i + 0.5) * grid->sx;
                double acc = 0.0;
                for (int ia = 0; ia < na; ++ia) {
                    const double c = cos(g->angles[ia]), s = sin(g->angles[ia]);
                    const double ss = x * c + y * s, t = -x * s + y * c;
                    const double L = g->dso - ss;
                    if (L <= 1e-6 * g->dso) continue;
                    const double u = t * g->dso / L, v = z * g->dso / L;
                    const double fu = (u - u0) / du, fv = (v - v0) / dv;
                    const int ju = (int)floor(fu), jv = (int)floor(fv);
                    if (ju < -1 || ju > nu - 1 || jv < -1 || jv > nv - 1) continue;
                    const double au = fu - ju, av = fv - jv;
                    const double* f = filtered + (size_t)ia * per;
#define S_(uu, vv) (((uu) < 0 || (uu) >= nu || (vv) < 0 || (vv) >= nv) ? 0.0 : f[(size_t)(vv) * nu + (uu)])
                    const double val = (1.0 - au) * (1.0 - av) * S_(ju, jv) + au * (1.0 - av) * S_(ju + 1, jv) +
                                       (1.0 - au) * av * S_(ju, jv + 1) + au * av * S_(ju + 1, jv + 1);
#undef S_
                    acc += (g->dso * g->dso) / (L * L) * val;
                }
                vol[(size_t)i + (size_t)grid->nx * ((size_t)j + (size_t)grid->ny * k)] = scale * acc;
            }
        }
    }
    free(ramp);
    free(filtered);
    return 0;
}
