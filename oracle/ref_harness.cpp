// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shims around the UNMODIFIED reference library (header-only
// kryct, compiled from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libkryct_ref.so).  It gives tests and bench.py's reference arm
// the reference's own double-precision code path behind the same C signatures
// as kct_oracle.h (prefix ref_ instead of ora_).  Only the hot-path headers
// are included (io.hpp / experiment.hpp need a vendor/ tree that is absent).
#include <kryct/diffreg.hpp>
#include <kryct/fdk.hpp>
#include <kryct/krylov.hpp>
#include <kryct/linear_map.hpp>
#include <kryct/projector.hpp>
#include <kryct/recon.hpp>
#include <kryct/types.hpp>
#include <kryct/vector_ops.hpp>

#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/kct.h"

namespace {

thread_local std::string g_err;

kryct::GridSpec to_grid(const kct_grid* g) {
    kryct::GridSpec s;
    s.dims = {g->nx, g->ny, g->nz};
    s.spacing = {g->sx, g->sy, g->sz};
    s.origin = {g->ox, g->oy, g->oz};
    return s;
}

kryct::ConeBeamGeometry to_geom(const kct_geometry* g) {
    kryct::ConeBeamGeometry c;
    c.dso = g->dso;
    c.dsd = g->dsd;
    c.detector = {g->nu, g->nv, g->pu, g->pv};
    c.offset_u = g->offset_u;
    c.offset_v = g->offset_v;
    c.angles.assign(g->angles, g->angles + g->n_angles);
    return c;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const kryct::ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const kryct::SolverError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void fill_report(const kryct::ReconReport& r, kct_report* rep) {
    if (!rep) return;
    rep->objective_count = r.objective_history.size();
    rep->residual_count = r.residual_history.size();
    rep->error_count = r.error_history.size();
    rep->outer_count = r.outer_boundaries.size();
    if (rep->objective_history)
        std::memcpy(rep->objective_history, r.objective_history.data(),
                    r.objective_history.size() * sizeof(double));
    if (rep->residual_history)
        std::memcpy(rep->residual_history, r.residual_history.data(),
                    r.residual_history.size() * sizeof(double));
    if (rep->error_history)
        std::memcpy(rep->error_history, r.error_history.data(),
                    r.error_history.size() * sizeof(double));
    if (rep->outer_boundaries)
        for (std::size_t i = 0; i < r.outer_boundaries.size(); ++i)
            rep->outer_boundaries[i] = r.outer_boundaries[i];
    if (rep->outer_seconds)
        std::memcpy(rep->outer_seconds, r.outer_seconds.data(),
                    r.outer_seconds.size() * sizeof(double));
    rep->solve_seconds = r.solve_seconds;
    rep->converged = r.converged ? 1 : 0;
    rep->breakdown = 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ConeBeamProjector ctor + apply / apply_adjoint (projector.hpp:264-291)
int ref_forward(const kct_grid* grid, const kct_geometry* g, const double* vol, double* proj) {
    return guarded([&] {
        kryct::ConeBeamProjector a(to_grid(grid), to_geom(g));
        a.apply(std::span<const double>(vol, a.domain_size()),
                std::span<double>(proj, a.range_size()));
    });
}

int ref_adjoint(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol) {
    return guarded([&] {
        kryct::ConeBeamProjector a(to_grid(grid), to_geom(g));
        a.apply_adjoint(std::span<const double>(proj, a.range_size()),
                        std::span<double>(vol, a.domain_size()));
    });
}

// traverse_ray visit count (projector.hpp:53-131) summed over all rays.
uint64_t ref_count_nnz(const kct_grid* grid, const kct_geometry* g) {
    uint64_t total = 0;
    guarded([&] {
        const auto gs = to_grid(grid);
        const auto geom = to_geom(g);
        const int nu = geom.detector.nu, nv = geom.detector.nv;
        const long rows = static_cast<long>(geom.n_angles()) * nv;
        uint64_t sum = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : sum)
        for (long r = 0; r < rows; ++r) {
            const std::size_t ia = static_cast<std::size_t>(r / nv);
            const int iv = static_cast<int>(r % nv);
            const auto src = kryct::source_position(geom, ia);
            for (int iu = 0; iu < nu; ++iu) {
                uint64_t c = 0;
                kryct::traverse_ray(src, kryct::detector_pixel_center(geom, ia, iu, iv), gs,
                                    [&](std::size_t, double) { ++c; });
                sum += c;
            }
        }
        total = sum;
    });
    return total;
}

size_t ref_trace_ray(const kct_grid* grid, const double src[3], const double dst[3],
                     uint64_t* voxels, double* lengths, size_t cap, double t_io[2]) {
    const auto p = kryct::trace_ray({src[0], src[1], src[2]}, {dst[0], dst[1], dst[2]},
                                    to_grid(grid));
    for (std::size_t i = 0; i < p.voxels.size() && i < cap; ++i) {
        voxels[i] = p.voxels[i];
        lengths[i] = p.lengths[i];
    }
    if (t_io) {
        t_io[0] = p.t_entry;
        t_io[1] = p.t_exit;
    }
    return p.voxels.size();
}

// DiffOperator (diffreg.hpp:20-84), tv_weights (:142-156), smoothed_tv (:118-126)
void ref_diff(int nx, int ny, int nz, const double* x, double* out3m) {
    kryct::DiffOperator d({nx, ny, nz});
    d.apply(std::span<const double>(x, d.domain_size()),
            std::span<double>(out3m, d.range_size()));
}

void ref_diff_adjoint(int nx, int ny, int nz, const double* y3m, double* out) {
    kryct::DiffOperator d({nx, ny, nz});
    d.apply_adjoint(std::span<const double>(y3m, d.range_size()),
                    std::span<double>(out, d.domain_size()));
}

int ref_tv_weights(const double* grad3m, size_t m, double tau, double* w3m) {
    return guarded([&] {
        const auto w = kryct::tv_weights(std::span<const double>(grad3m, 3 * m), tau);
        std::memcpy(w3m, w.data(), w.size() * sizeof(double));
    });
}

double ref_smoothed_tv(const double* grad3m, size_t m, double tau) {
    return kryct::smoothed_tv(std::span<const double>(grad3m, 3 * m), tau);
}

double ref_resolve_tau(double tau, const double* ref, size_t n) {
    return kryct::resolve_tau(tau, std::span<const double>(ref, ref ? n : 0));
}

double ref_objective(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
                     const double* x, const double* prior, double alpha, double lambda,
                     double tau) {
    double obj = 0.0;
    guarded([&] {
        kryct::ConeBeamProjector a(to_grid(grid), to_geom(g));
        const std::size_t m = a.domain_size();
        obj = kryct::evaluate_objective(
            static_cast<kryct::ObjectiveKind>(kind), a,
            std::span<const double>(b, a.range_size()), std::span<const double>(x, m),
            std::span<const double>(prior, prior ? m : 0), a.grid().dims, alpha, lambda, tau);
    });
    return obj;
}

// fdk (fdk.hpp:50-139)
int ref_fdk(const kct_grid* grid, const kct_geometry* g, const double* proj, double* vol) {
    return guarded([&] {
        kryct::ProjectionSet p(to_geom(g));
        std::memcpy(p.data.data(), proj, p.data.size() * sizeof(double));
        const auto v = kryct::fdk(p, to_grid(grid));
        std::memcpy(vol, v.data.data(), v.data.size() * sizeof(double));
    });
}

// cgls_recon (recon.hpp:312-315)
int ref_cgls_recon(const kct_grid* grid, const kct_geometry* g, const double* b, size_t iters,
                   const double* x0, const double* gt, double tol, double* x_out,
                   kct_report* rep) {
    return guarded([&] {
        kryct::ProjectionSet proj(to_geom(g));
        std::memcpy(proj.data.data(), b, proj.data.size() * sizeof(double));
        const auto gs = to_grid(grid);
        const std::size_t m = gs.dims.count();
        kryct::Volume init(gs), truth(gs);
        kryct::ReconOptions opts;
        if (x0) {
            std::memcpy(init.data.data(), x0, m * sizeof(double));
            opts.initial = &init;
        }
        if (gt) {
            std::memcpy(truth.data.data(), gt, m * sizeof(double));
            opts.ground_truth = &truth;
        }
        const auto r = kryct::cgls_recon(proj, gs, iters, opts, tol);
        std::memcpy(x_out, r.volume.data.data(), m * sizeof(double));
        fill_report(r, rep);
    });
}

// irn_tv / irn_piple / irn_piccs (recon.hpp:252-270)
int ref_irn(const kct_grid* grid, const kct_geometry* g, int kind, const double* b,
            const double* prior, const double* x0, const double* gt, const kct_reg_params* p,
            double* x_out, kct_report* rep) {
    return guarded([&] {
        kryct::ProjectionSet proj(to_geom(g));
        std::memcpy(proj.data.data(), b, proj.data.size() * sizeof(double));
        const auto gs = to_grid(grid);
        const std::size_t m = gs.dims.count();
        kryct::Volume init(gs), truth(gs), pri(gs);
        kryct::ReconOptions opts;
        if (x0) {
            std::memcpy(init.data.data(), x0, m * sizeof(double));
            opts.initial = &init;
        }
        if (gt) {
            std::memcpy(truth.data.data(), gt, m * sizeof(double));
            opts.ground_truth = &truth;
        }
        if (prior) std::memcpy(pri.data.data(), prior, m * sizeof(double));
        kryct::RegularizationParams rp;
        rp.alpha = p->alpha;
        rp.lambda = p->lambda;
        rp.tau = p->tau;
        rp.outer_iters = p->outer_iters;
        rp.inner_iters = p->inner_iters;
        rp.inner_tolerance = p->inner_tolerance;
        rp.warm_start = p->warm_start != 0;
        kryct::ReconReport r;
        if (kind == KCT_KIND_TV) r = kryct::irn_tv(proj, gs, rp, opts);
        else if (kind == KCT_KIND_PIPLE) r = kryct::irn_piple(proj, gs, pri, rp, opts);
        else r = kryct::irn_piccs(proj, gs, pri, rp, opts);
        std::memcpy(x_out, r.volume.data.data(), m * sizeof(double));
        fill_report(r, rep);
        if (rep) rep->tau = kryct::resolve_tau(
            rp.tau, x0 ? std::span<const double>(init.data)
                       : ((kind != KCT_KIND_TV && rp.resolved_lambda() != 0.0)
                              ? std::span<const double>(pri.data)
                              : std::span<const double>()));
    });
}

// cgls (krylov.hpp:59-127) on a StackedMap the caller assembles (linear_map.hpp:159-216):
// block i = ScaledBlock{scales[i], compose(DiagonalMap(weights[i]), map_i)} (plain map_i
// without weights), map_i the reference's ConeBeamProjector / DiffOperator / IdentityMap.
int ref_cgls_stack(const kct_grid* grid, const kct_geometry* g, size_t n_blocks, const int* maps,
                   const double* scales, const double* const* weights, const double* b, double* x,
                   size_t max_iters, double tol, double* res_hist, size_t* iterations,
                   int* converged, int* breakdown) {
    return guarded([&] {
        const auto gs = to_grid(grid);
        const auto ge = to_geom(g);
        const std::size_t m = gs.dims.count();
        std::vector<kryct::ScaledBlock> blocks;
        for (size_t i = 0; i < n_blocks; ++i) {
            std::shared_ptr<const kryct::LinearMap> map;
            if (maps[i] == KCT_MAP_PROJECTOR) map = std::make_shared<kryct::ConeBeamProjector>(gs, ge);
            else if (maps[i] == KCT_MAP_DIFF) map = kryct::make_diff(gs.dims);
            else if (maps[i] == KCT_MAP_IDENTITY) map = std::make_shared<kryct::IdentityMap>(m);
            else throw kryct::ConfigError("stack: unknown block map");
            if (weights[i]) {
                std::vector<double> w(weights[i], weights[i] + map->range_size());
                map = kryct::compose(std::make_shared<kryct::DiagonalMap>(std::move(w)), map);
            }
            blocks.push_back({scales[i], map});
        }
        const auto A = kryct::stack_maps(std::move(blocks));
        kryct::KrylovConfig cfg;
        cfg.max_iters = max_iters;
        cfg.tolerance = tol;
        const auto r = kryct::cgls(*A, std::span<const double>(b, A->range_size()),
                                   std::span<const double>(x, m), cfg);
        std::memcpy(x, r.x.data(), m * sizeof(double));
        if (res_hist)
            for (size_t i = 0; i < r.trace.residual_norms.size(); ++i) res_hist[i] = r.trace.residual_norms[i];
        if (iterations) *iterations = r.trace.iterations;
        if (converged) *converged = r.trace.converged ? 1 : 0;
        if (breakdown) *breakdown = r.trace.breakdown ? 1 : 0;
    });
}

}  // extern "C"
