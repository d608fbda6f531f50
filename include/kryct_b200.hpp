// kryct_b200.hpp — C++ drop-in shim: the reference kryct API on the B200
// library (libkct.so, C ABI in kct.h).
//
// Include this after the reference headers.  It provides, with the reference
// signatures and error behaviour (ConfigError / SolverError):
//   kryct_b200::GpuConeBeamProjector : kryct::LinearMap   (projector.hpp:264-291)
//   kryct_b200::cgls_recon(proj, grid, iters, opts, tol)   (recon.hpp:312-315)
//   kryct_b200::irn_tv / irn_piple / irn_piccs             (recon.hpp:252-270)
//   kryct_b200::cgls(A, b, x0, cfg)                        (krylov.hpp:59-127)
//     device-resident CGLS over a caller-assembled kryct::StackedMap whose
//     blocks are a GpuConeBeamProjector, kryct::DiffOperator or
//     kryct::IdentityMap, each optionally under compose(DiagonalMap, .) —
//     the stacks recon.hpp:211-221 assembles (kct_cgls_stack)
//   kryct_b200::Communicator + the same drivers with a communicator first:
//     one process per GPU, y-slab-sharded solves over the library's own NCCL
//     communicator (kct_comm_*; no reference counterpart)
// so existing callers switch by namespace, and the reference's own generic
// solvers (kryct::cgls, kryct::StackedMap, ...) can drive the GPU operator.
// Values cross the boundary as float32 (the reference reads float32 files,
// io.hpp:48-49); the solvers reduce in float64 on the device.
// ReconOptions::hook (the reference's per-iteration IterateHook) is served as
// an opt-in device->host copy of every iterate (kct_set_iterate_hook): the
// copy overlaps the solve on a side stream and the hook runs on a CUDA host
// callback thread, in iteration order, all calls done before the solver
// returns.  The error history against ground_truth needs no hook (device).
//
// Handle cache: a projector handle owns device tables (the adjoint walk
// table: 339 MB at 256^3 / 60 views) and a solver workspace, whose creation
// costs milliseconds of kernels and allocations.  The reference builds its
// CPU projector per call (recon.hpp:155, :282), which is cheap there; here the
// drivers keep the last KRYCT_B200_CACHE (default 2, 0 = off) handles keyed by
// (grid, geometry) and reuse them.  A handle in use by one call is not handed
// to a concurrent call (that call builds its own).
#pragma once

#include <kryct/diffreg.hpp>
#include <kryct/krylov.hpp>
#include <kryct/linear_map.hpp>
#include <kryct/recon.hpp>
#include <kryct/types.hpp>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <future>
#include <list>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "kct.h"

namespace kryct_b200 {

namespace detail {

inline void check(int rc) {
    if (rc == KCT_OK) return;
    const std::string msg = kct_last_error();
    if (rc == KCT_ERR_CONFIG) throw kryct::ConfigError(msg);
    if (rc == KCT_ERR_SOLVER) throw kryct::SolverError(msg);
    throw std::runtime_error("kct: " + msg);
}

inline kct_grid to_grid(const kryct::GridSpec& g) {
    return kct_grid{g.dims.nx,   g.dims.ny,   g.dims.nz,   g.spacing.x, g.spacing.y,
                    g.spacing.z, g.origin.x, g.origin.y, g.origin.z};
}

inline kct_geometry to_geom(const kryct::ConeBeamGeometry& g) {
    return kct_geometry{g.dso,      g.dsd,      g.detector.nu,
                        g.detector.nv, g.detector.pu, g.detector.pv,
                        g.offset_u, g.offset_v, static_cast<int>(g.angles.size()),
                        g.angles.data()};
}

inline std::vector<float> to_f32(std::span<const double> v) {
    return std::vector<float>(v.begin(), v.end());
}

// Page-locked float staging buffers (kct_host_alloc) per slot, grown on
// demand and kept for the process: the solver's host copies then run
// asynchronously at full PCIe rate.  Conversions double <-> float run on all
// OpenMP threads when the caller compiles with OpenMP (as the reference does).
struct Pinned {
    std::mutex mu;
    float* ptr[4] = {nullptr, nullptr, nullptr, nullptr};
    std::size_t cap[4] = {0, 0, 0, 0};
    float* get(int slot, std::size_t n) {
        if (cap[slot] < n) {
            if (ptr[slot]) kct_host_free(ptr[slot]);
            ptr[slot] = nullptr;
            cap[slot] = 0;
            void* p = nullptr;
            if (kct_host_alloc(n * sizeof(float), &p) != KCT_OK) return nullptr;
            ptr[slot] = static_cast<float*>(p);
            cap[slot] = n;
        }
        return ptr[slot];
    }
};
inline Pinned& pinned() {
    // never destroyed: its buffers belong to the CUDA context, which may be
    // gone by the time static destructors run at process exit (the page-locked
    // memory goes with the process)
    static Pinned* const p = new Pinned;
    return *p;
}

// double -> float; returns false if any value is not finite (the caller
// throws the reference's ConfigError: types.hpp Volume/ProjectionSet::validate)
inline bool to_f32(std::span<const double> v, float* out) {
    const std::ptrdiff_t n = static_cast<std::ptrdiff_t>(v.size());
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (std::ptrdiff_t i = 0; i < n; ++i) {
        bad |= std::isfinite(v[i]) ? 0 : 1;
        out[i] = static_cast<float>(v[i]);
    }
    return bad == 0;
}

struct Handle {
    kct_projector* h = nullptr;
    ~Handle() {
        if (h) kct_projector_destroy(h);
    }
};

}  // namespace detail

// The operator lives in an inner namespace so that an unqualified
// `cgls(gpu_projector, ...)` in caller code (argument-dependent lookup) keeps
// resolving to kryct::cgls alone, not also to kryct_b200::cgls below.
namespace ops {

/// ConeBeamProjector on one CUDA device (projector.hpp:264-291).
class GpuConeBeamProjector final : public kryct::LinearMap {
  public:
    using kryct::LinearMap::apply;
    using kryct::LinearMap::apply_adjoint;

    GpuConeBeamProjector(kryct::GridSpec grid, kryct::ConeBeamGeometry geometry, int device = -1)
        : grid_(grid), geom_(std::move(geometry)), h_(std::make_shared<detail::Handle>()) {
        const kct_grid g = detail::to_grid(grid_);
        const kct_geometry ge = detail::to_geom(geom_);
        detail::check(kct_projector_create(&g, &ge, device, &h_->h));
    }

    std::size_t domain_size() const override { return grid_.dims.count(); }
    std::size_t range_size() const override { return geom_.ray_count(); }
    const kryct::GridSpec& grid() const { return grid_; }
    const kryct::ConeBeamGeometry& geometry() const { return geom_; }
    kct_projector* handle() const { return h_->h; }

    void apply(std::span<const double> x, std::span<double> out) const override {
        check_domain(x.size());
        check_range(out.size());
        if (!staged(x, out, true)) detail::check(kct_forward_f64(h_->h, x.data(), out.data()));
    }
    void apply_adjoint(std::span<const double> y, std::span<double> out) const override {
        check_range(y.size());
        check_domain(out.size());
        if (!staged(y, out, false)) detail::check(kct_adjoint_f64(h_->h, y.data(), out.data()));
    }

  private:
    // through the page-locked float staging slots (the host pipelines of
    // kct_forward / kct_adjoint then overlap their copies with the kernels);
    // false when another call holds the slots
    bool staged(std::span<const double> in, std::span<double> out, bool fwd) const {
        std::unique_lock<std::mutex> lk(detail::pinned().mu, std::try_to_lock);
        if (!lk.owns_lock()) return false;
        float* fi = detail::pinned().get(1, in.size());
        float* fo = detail::pinned().get(0, out.size());
        if (!fi || !fo) return false;
        detail::to_f32(in, fi);
        detail::check(fwd ? kct_forward(h_->h, fi, fo, KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr)
                          : kct_adjoint(h_->h, fi, fo, KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr));
        const std::ptrdiff_t n = static_cast<std::ptrdiff_t>(out.size());
        double* o = out.data();
#pragma omp parallel for schedule(static)
        for (std::ptrdiff_t i = 0; i < n; ++i) o[i] = fo[i];
        return true;
    }

    kryct::GridSpec grid_;
    kryct::ConeBeamGeometry geom_;
    std::shared_ptr<detail::Handle> h_;
};

}  // namespace ops
using ops::GpuConeBeamProjector;

namespace detail {

// ---- handle cache keyed by (grid, geometry) ---------------------------------
struct CacheKey {
    kryct::GridSpec grid;
    kryct::ConeBeamGeometry geom;
    bool operator==(const CacheKey& o) const {
        const auto& a = grid;
        const auto& b = o.grid;
        return a.dims == b.dims && a.spacing.x == b.spacing.x && a.spacing.y == b.spacing.y &&
               a.spacing.z == b.spacing.z && a.origin.x == b.origin.x &&
               a.origin.y == b.origin.y && a.origin.z == b.origin.z && geom.dso == o.geom.dso &&
               geom.dsd == o.geom.dsd && geom.detector.nu == o.geom.detector.nu &&
               geom.detector.nv == o.geom.detector.nv && geom.detector.pu == o.geom.detector.pu &&
               geom.detector.pv == o.geom.detector.pv && geom.offset_u == o.geom.offset_u &&
               geom.offset_v == o.geom.offset_v && geom.angles == o.geom.angles;
    }
};

struct HandleCache {
    std::mutex mu;
    std::list<std::pair<CacheKey, std::shared_ptr<GpuConeBeamProjector>>> idle;  // MRU first
    std::size_t capacity() const {
        const char* e = std::getenv("KRYCT_B200_CACHE");
        return e ? static_cast<std::size_t>(std::strtoul(e, nullptr, 10)) : 2;
    }
    // check a handle out (removed from the cache while in use)
    std::shared_ptr<GpuConeBeamProjector> acquire(const kryct::GridSpec& g,
                                                  const kryct::ConeBeamGeometry& ge) {
        {
            std::lock_guard<std::mutex> lk(mu);
            const CacheKey key{g, ge};
            for (auto it = idle.begin(); it != idle.end(); ++it)
                if (it->first == key) {
                    auto h = it->second;
                    idle.erase(it);
                    return h;
                }
        }
        return std::make_shared<GpuConeBeamProjector>(g, ge);
    }
    void release(std::shared_ptr<GpuConeBeamProjector> h) {
        const std::size_t cap = capacity();
        if (cap == 0) return;
        std::lock_guard<std::mutex> lk(mu);
        idle.emplace_front(CacheKey{h->grid(), h->geometry()}, std::move(h));
        while (idle.size() > cap) idle.pop_back();
    }
    void clear() {
        std::lock_guard<std::mutex> lk(mu);
        idle.clear();
    }
};

inline HandleCache& handle_cache() {
    // never destroyed (see pinned()): cached handles are released by
    // clear_handle_cache() or with the process, never by a static destructor
    // racing the CUDA runtime's own teardown
    static HandleCache* const c = new HandleCache;
    return *c;
}

struct CheckedOut {
    std::shared_ptr<GpuConeBeamProjector> h;
    CheckedOut(const kryct::GridSpec& g, const kryct::ConeBeamGeometry& ge)
        : h(handle_cache().acquire(g, ge)) {}
    ~CheckedOut() {
        kct_set_iterate_hook(h->handle(), nullptr, nullptr);
        handle_cache().release(std::move(h));
    }
};

// IterateHook trampoline: float32 reference-layout iterate -> span<const double>.
// An exception thrown by the hook stops further calls and is rethrown by the
// solver entry point once the solve has returned.
struct HookCtx {
    const kryct::IterateHook* hook;
    std::exception_ptr err;
    std::vector<double> xd;
};

inline void hook_trampoline(void* ctx, std::size_t it, const float* x, std::size_t m) {
    auto& c = *static_cast<HookCtx*>(ctx);
    if (c.err) return;
    try {
        c.xd.assign(x, x + m);
        (*c.hook)(it, c.xd);
    } catch (...) {
        c.err = std::current_exception();
    }
}

inline kryct::ReconReport run(int kind, const kryct::ProjectionSet& proj,
                              const kryct::GridSpec& grid, const kryct::Volume* prior,
                              const kryct::RegularizationParams* params, std::size_t iters,
                              double tol, const kryct::ReconOptions& opts) {
    // ProjectionSet::validate (types.hpp:180-186) with the finiteness scan
    // fused into the conversion below
    proj.geometry.validate();
    if (proj.data.size() != proj.geometry.ray_count())
        throw kryct::ConfigError("projection data length does not match geometry");
    grid.validate();
    CheckedOut co(grid, proj.geometry);
    const GpuConeBeamProjector& A = *co.h;
    HookCtx hc{&opts.hook, nullptr, {}};
    if (opts.hook) check(kct_set_iterate_hook(A.handle(), hook_trampoline, &hc));
    const std::size_t m = grid.dims.count();
    // the large buffers go through the page-locked staging slots (one caller
    // at a time holds them; a concurrent call falls back to plain vectors)
    std::unique_lock<std::mutex> plk(pinned().mu, std::try_to_lock);
    std::vector<float> b_v, pr_v, x_v;
    float* b = plk.owns_lock() ? pinned().get(0, proj.data.size()) : nullptr;
    float* pr_p = nullptr;
    float* x = plk.owns_lock() ? pinned().get(2, m) : nullptr;
    if (!b) b = (b_v.resize(proj.data.size()), b_v.data());
    if (!x) x = (x_v.resize(m), x_v.data());
    if (!to_f32(proj.data, b)) throw kryct::ConfigError("projections contain non-finite values");
    // the result's double vector is allocated (and its pages touched) by a
    // helper thread while the device solves
    auto result = std::async(std::launch::async, [m] { return std::vector<double>(m); });
    std::vector<float> x0, gt;
    if (prior) {
        if (!(prior->dims == grid.dims))
            throw kryct::ConfigError("prior volume does not match the reconstruction grid");
        pr_p = plk.owns_lock() ? pinned().get(1, m) : nullptr;
        if (!pr_p) pr_p = (pr_v.resize(m), pr_v.data());
        if (!to_f32(prior->data, pr_p)) throw kryct::ConfigError("volume contains non-finite values");
    }
    if (opts.initial) {
        if (!(opts.initial->dims == grid.dims))
            throw kryct::ConfigError("initial volume does not match the reconstruction grid");
        x0 = to_f32(opts.initial->data);
    }
    if (opts.ground_truth) {
        if (!(opts.ground_truth->dims == grid.dims))
            throw kryct::ConfigError("ground truth does not match the reconstruction grid");
        gt = to_f32(opts.ground_truth->data);
    }
    const std::size_t outer = params ? params->outer_iters : 1;
    const std::size_t inner = params ? params->inner_iters : iters;
    std::vector<double> obj(outer * inner + outer + 1), res(outer * inner), err(outer * inner),
        secs(outer + 1);
    std::vector<uint64_t> bnd(outer + 1);
    kct_report rep{};
    rep.objective_history = obj.data();
    rep.residual_history = res.data();
    rep.error_history = err.data();
    rep.outer_boundaries = bnd.data();
    rep.outer_seconds = secs.data();
    const float* px0 = x0.empty() ? nullptr : x0.data();
    const float* pgt = gt.empty() ? nullptr : gt.data();
    if (params) {
        const kct_reg_params p{params->alpha,       params->lambda,          params->tau,
                               params->outer_iters, params->inner_iters,    params->inner_tolerance,
                               params->warm_start ? 1 : 0};
        check(kct_irn(A.handle(), kind, b, pr_p, px0, pgt, &p, x, &rep, KCT_MEM_HOST,
                      KCT_LAYOUT_REFERENCE, nullptr));
    } else {
        check(kct_cgls_recon(A.handle(), b, iters, px0, pgt, tol, x, &rep, KCT_MEM_HOST,
                             KCT_LAYOUT_REFERENCE, nullptr));
    }
    kryct::ReconReport r;
    r.volume.dims = grid.dims;
    r.volume.spacing = grid.spacing;
    r.volume.origin = grid.origin;
    r.volume.data = result.get();
    {
        double* dst = r.volume.data.data();
        const std::ptrdiff_t mm = static_cast<std::ptrdiff_t>(m);
#pragma omp parallel for schedule(static)
        for (std::ptrdiff_t i = 0; i < mm; ++i) dst[i] = x[i];
    }
    r.objective_history.assign(obj.begin(), obj.begin() + rep.objective_count);
    r.residual_history.assign(res.begin(), res.begin() + rep.residual_count);
    r.error_history.assign(err.begin(), err.begin() + rep.error_count);
    for (std::size_t i = 0; i < rep.outer_count; ++i) {
        r.outer_boundaries.push_back(bnd[i]);
        r.outer_seconds.push_back(secs[i]);
    }
    r.solve_seconds = rep.solve_seconds;
    r.converged = rep.converged != 0;
    if (hc.err) std::rethrow_exception(hc.err);
    return r;
}

}  // namespace detail

namespace detail {

// kryct::ComposedMap keeps its operands private and has no accessors
// (linear_map.hpp:146-149).  Reading them through an explicit template
// instantiation (which may name private members) lets the drop-in take the
// caller's unmodified compose(DiagonalMap, map) blocks; a maintainer adopting
// the shim would add outer() / inner() accessors instead.
template <class Tag, typename Tag::type Member>
struct MemberOf {
    friend typename Tag::type member_ptr(Tag) { return Member; }
};
struct ComposedOuter {
    using type = std::shared_ptr<const kryct::LinearMap> kryct::ComposedMap::*;
    friend type member_ptr(ComposedOuter);
};
struct ComposedInner {
    using type = std::shared_ptr<const kryct::LinearMap> kryct::ComposedMap::*;
    friend type member_ptr(ComposedInner);
};
template struct MemberOf<ComposedOuter, &kryct::ComposedMap::outer_>;
template struct MemberOf<ComposedInner, &kryct::ComposedMap::inner_>;

struct FlatBlock {
    int map;
    double scale;
    const std::vector<double>* weights;  // nullptr = no diagonal
    std::size_t len;
};

// One block: [DiagonalMap o] {GpuConeBeamProjector | DiffOperator | IdentityMap}
inline FlatBlock flatten_block(const kryct::LinearMap& m, double scale,
                               const GpuConeBeamProjector*& projector) {
    const kryct::LinearMap* map = &m;
    const std::vector<double>* w = nullptr;
    if (const auto* cm = dynamic_cast<const kryct::ComposedMap*>(map)) {
        const auto& outer = cm->*member_ptr(ComposedOuter{});
        const auto& inner = cm->*member_ptr(ComposedInner{});
        const auto* dm = dynamic_cast<const kryct::DiagonalMap*>(outer.get());
        if (!dm) throw kryct::ConfigError("kryct_b200::cgls: a composed block must be DiagonalMap o map");
        w = &dm->weights();
        map = inner.get();
    }
    int code;
    if (const auto* gp = dynamic_cast<const GpuConeBeamProjector*>(map)) {
        if (projector && projector->handle() != gp->handle())
            throw kryct::ConfigError("kryct_b200::cgls: blocks must share one projector");
        projector = gp;
        code = KCT_MAP_PROJECTOR;
    } else if (dynamic_cast<const kryct::DiffOperator*>(map)) {
        code = KCT_MAP_DIFF;
    } else if (dynamic_cast<const kryct::IdentityMap*>(map)) {
        code = KCT_MAP_IDENTITY;
    } else {
        throw kryct::ConfigError(
            "kryct_b200::cgls: unsupported block (GpuConeBeamProjector, DiffOperator or IdentityMap, "
            "optionally under a DiagonalMap; other maps: kryct::cgls drives the GPU operator)");
    }
    return FlatBlock{code, scale, w, map->range_size()};
}

}  // namespace detail

/// krylov.hpp:59-127 — cgls on a caller-assembled stack with every iteration
/// vector resident on the device.  Same signature, error behaviour and trace
/// as kryct::cgls; values cross the boundary as float32.
inline kryct::SolveResult cgls(const kryct::LinearMap& A, std::span<const double> b,
                               std::span<const double> x0, const kryct::KrylovConfig& cfg = {}) {
    if (b.size() != A.range_size()) throw kryct::ConfigError("cgls: rhs size mismatch");
    if (x0.size() != A.domain_size()) throw kryct::ConfigError("cgls: x0 size mismatch");
    const GpuConeBeamProjector* P = nullptr;
    std::vector<detail::FlatBlock> flat;
    if (const auto* st = dynamic_cast<const kryct::StackedMap*>(&A)) {
        for (std::size_t i = 0; i < st->block_count(); ++i)
            flat.push_back(detail::flatten_block(*st->block(i).map, st->block(i).scale, P));
    } else {
        flat.push_back(detail::flatten_block(A, 1.0, P));
    }
    if (!P) throw kryct::ConfigError("kryct_b200::cgls: the stack needs a GpuConeBeamProjector block");
    const std::size_t m = P->domain_size();
    for (const auto& f : flat) {
        const std::size_t want =
            f.map == KCT_MAP_PROJECTOR ? P->range_size() : (f.map == KCT_MAP_DIFF ? 3 * m : m);
        if (f.len != want) throw kryct::ConfigError("kryct_b200::cgls: block size does not match the grid");
    }
    // DiffOperator dims must be the projector grid's (its range alone does not say so)
    if (const auto* st = dynamic_cast<const kryct::StackedMap*>(&A))
        for (std::size_t i = 0; i < st->block_count(); ++i) {
            const kryct::LinearMap* mp = st->block(i).map.get();
            if (const auto* cm = dynamic_cast<const kryct::ComposedMap*>(mp))
                mp = (cm->*member_ptr(detail::ComposedInner{})).get();
            if (const auto* d = dynamic_cast<const kryct::DiffOperator*>(mp))
                if (!(d->dims() == P->grid().dims))
                    throw kryct::ConfigError("kryct_b200::cgls: DiffOperator dims do not match the grid");
        }

    std::vector<float> bf(b.size()), xf(m), out(m);
    detail::to_f32(b, bf.data());  // non-finite data surfaces as SolverError from the device (krylov.hpp:75)
    detail::to_f32(x0, xf.data());
    std::vector<std::vector<float>> wf(flat.size());
    std::vector<kct_stack_block> blocks(flat.size());
    for (std::size_t i = 0; i < flat.size(); ++i) {
        if (flat[i].weights) {
            wf[i].resize(flat[i].weights->size());
            detail::to_f32(*flat[i].weights, wf[i].data());
        }
        blocks[i] = kct_stack_block{flat[i].map, flat[i].scale, flat[i].weights ? wf[i].data() : nullptr};
    }
    bool x_zero = true;
    for (double v : x0) x_zero = x_zero && v == 0.0;
    detail::HookCtx hc{&cfg.hook, nullptr, {}};
    struct HookGuard {
        kct_projector* h;
        ~HookGuard() { kct_set_iterate_hook(h, nullptr, nullptr); }
    } guard{P->handle()};
    if (cfg.hook) detail::check(kct_set_iterate_hook(P->handle(), detail::hook_trampoline, &hc));
    const std::size_t cap = cfg.max_iters > 0 ? cfg.max_iters : 1;
    std::vector<double> res(cap), wall(cap);
    kct_report rep{};
    rep.residual_history = res.data();
    rep.wall_times = wall.data();
    detail::check(kct_cgls_stack(P->handle(), blocks.data(), blocks.size(), bf.data(),
                                 x_zero ? nullptr : xf.data(), cfg.max_iters, cfg.tolerance, out.data(),
                                 &rep, KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr));
    if (hc.err) std::rethrow_exception(hc.err);
    kryct::SolveResult r;
    r.x.assign(out.begin(), out.end());
    r.trace.iterations = rep.residual_count;
    r.trace.converged = rep.converged != 0;
    r.trace.breakdown = rep.breakdown != 0;
    r.trace.residual_norms.assign(res.begin(), res.begin() + rep.residual_count);
    r.trace.wall_times.assign(wall.begin(), wall.begin() + rep.wall_count);
    return r;
}

/// Drop the cached projector handles (frees their device memory).
inline void clear_handle_cache() { detail::handle_cache().clear(); }

/// recon.hpp:312-315
inline kryct::ReconReport cgls_recon(const kryct::ProjectionSet& proj, const kryct::GridSpec& grid,
                                     std::size_t iters, const kryct::ReconOptions& opts = {},
                                     double tolerance = 0.0) {
    return detail::run(KCT_KIND_TV, proj, grid, nullptr, nullptr, iters, tolerance, opts);
}

/// recon.hpp:252-255
inline kryct::ReconReport irn_tv(const kryct::ProjectionSet& proj, const kryct::GridSpec& grid,
                                 const kryct::RegularizationParams& params,
                                 const kryct::ReconOptions& opts = {}) {
    return detail::run(KCT_KIND_TV, proj, grid, nullptr, &params, 0, 0.0, opts);
}

/// recon.hpp:260-263
inline kryct::ReconReport irn_piple(const kryct::ProjectionSet& proj, const kryct::GridSpec& grid,
                                    const kryct::Volume& prior,
                                    const kryct::RegularizationParams& params,
                                    const kryct::ReconOptions& opts = {}) {
    return detail::run(KCT_KIND_PIPLE, proj, grid, &prior, &params, 0, 0.0, opts);
}

/// recon.hpp:267-270 — the north-star entry point.
inline kryct::ReconReport irn_piccs(const kryct::ProjectionSet& proj, const kryct::GridSpec& grid,
                                    const kryct::Volume& prior,
                                    const kryct::RegularizationParams& params,
                                    const kryct::ReconOptions& opts = {}) {
    return detail::run(KCT_KIND_PICCS, proj, grid, &prior, &params, 0, 0.0, opts);
}

// ---- multi-GPU: one process per GPU, y-slab-sharded solves ------------------
// The reference is single-process (OpenMP only, projector.hpp:178-181); these
// entry points are the B200 library's scale-out of the same solvers (SURVEY
// §8e: volume vectors partitioned in slabs, NCCL over NVLink for the partial
// projections, the halo planes and the Krylov scalars).  Every rank calls
// with the SAME arguments (all projections, full-size prior / initial /
// ground truth) and gets the same report; the library's own NCCL
// communicator (kct_comm_*) carries the collectives, no MPI or Python needed.

/// RAII handle of the library's NCCL communicator.
class Communicator {
  public:
    using Id = std::array<unsigned char, KCT_COMM_ID_BYTES>;
    static Id unique_id() {
        Id id{};
        detail::check(kct_comm_unique_id(id.data()));
        return id;
    }
    /// Join as `rank` of `world` (collective); `device` >= 0 becomes the
    /// calling thread's CUDA device.
    Communicator(int rank, int world, const Id& id, int device = -1) {
        kct_comm* c = nullptr;
        detail::check(kct_comm_create(rank, world, id.data(), device, &c));
        c_ = std::shared_ptr<kct_comm>(c, [](kct_comm* p) { kct_comm_destroy(p); });
    }
    /// From a launcher's environment (torchrun / mpirun / srun): rank = RANK |
    /// OMPI_COMM_WORLD_RANK | PMI_RANK | SLURM_PROCID, world = WORLD_SIZE | ...,
    /// device = LOCAL_RANK | OMPI_COMM_WORLD_LOCAL_RANK | SLURM_LOCALID (else
    /// rank).  The unique id travels through `id_file` (default
    /// $KCT_COMM_ID_FILE; a path on a file system all ranks see, fresh per
    /// job): rank 0 writes it atomically and removes it once every rank has
    /// joined, the others poll for it ($KCT_COMM_TIMEOUT seconds, default 120).
    static Communicator from_env(std::string id_file = {}) {
        auto env_int = [](std::initializer_list<const char*> names, int dflt) {
            for (const char* n : names)
                if (const char* v = std::getenv(n)) return std::atoi(v);
            return dflt;
        };
        const int rank = env_int({"RANK", "OMPI_COMM_WORLD_RANK", "PMI_RANK", "SLURM_PROCID"}, 0);
        const int world = env_int({"WORLD_SIZE", "OMPI_COMM_WORLD_SIZE", "PMI_SIZE", "SLURM_NTASKS"}, 1);
        const int device =
            env_int({"LOCAL_RANK", "OMPI_COMM_WORLD_LOCAL_RANK", "SLURM_LOCALID"}, rank);
        if (id_file.empty())
            if (const char* f = std::getenv("KCT_COMM_ID_FILE")) id_file = f;
        Id id{};
        if (world > 1 && id_file.empty())
            throw kryct::ConfigError("Communicator::from_env: no id file (KCT_COMM_ID_FILE)");
        if (rank == 0) {
            id = unique_id();
            if (world > 1) {
                const std::string tmp = id_file + ".tmp";
                std::FILE* f = std::fopen(tmp.c_str(), "wb");
                if (!f || std::fwrite(id.data(), 1, id.size(), f) != id.size())
                    throw kryct::ConfigError("Communicator: cannot write " + tmp);
                std::fclose(f);
                if (std::rename(tmp.c_str(), id_file.c_str()) != 0)
                    throw kryct::ConfigError("Communicator: cannot create " + id_file);
            }
        } else {
            const char* t = std::getenv("KCT_COMM_TIMEOUT");
            const double limit = t ? std::atof(t) : 120.0;
            const auto t0 = std::chrono::steady_clock::now();
            for (;;) {
                if (std::FILE* f = std::fopen(id_file.c_str(), "rb")) {
                    const std::size_t n = std::fread(id.data(), 1, id.size(), f);
                    std::fclose(f);
                    if (n == id.size()) break;
                }
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
                    throw kryct::ConfigError("Communicator: timed out waiting for " + id_file);
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
        }
        Communicator c(rank, world, id, device);
        if (rank == 0 && world > 1) std::remove(id_file.c_str());  // every rank has joined
        return c;
    }
    int rank() const { return kct_comm_rank(c_.get()); }
    int world() const { return kct_comm_world(c_.get()); }
    kct_comm* handle() const { return c_.get(); }
    /// In-place sum (or maximum) of a host array over the ranks.
    void all_reduce(std::span<double> v, bool max = false) const {
        detail::check(kct_comm_allreduce_host(c_.get(), v.data(), v.size(), 1, max ? 1 : 0));
    }

  private:
    std::shared_ptr<kct_comm> c_;
};

/// This rank's y-plane range [j0, j1) of `grid` (kct_slab_bounds: balanced by
/// backprojection work, the same on every rank and for every scan of a system).
inline std::pair<int, int> slab_range(const Communicator& comm, const kryct::GridSpec& grid,
                                      const kryct::ConeBeamGeometry& geom) {
    std::vector<int> bounds(static_cast<std::size_t>(comm.world()) + 1);
    const kct_grid g = detail::to_grid(grid);
    const kct_geometry ge = detail::to_geom(geom);
    detail::check(kct_slab_bounds(&g, &ge, comm.world(), bounds.data()));
    return {bounds[comm.rank()], bounds[comm.rank() + 1]};
}

namespace detail {

// planes [j0, j1) of a reference-layout (x-fastest) volume, as float32
inline std::vector<float> y_slab_f32(std::span<const double> v, const kryct::Dims3& d, int j0,
                                     int j1, const char* what) {
    const std::size_t nx = d.nx, ny = d.ny, nz = d.nz, sy = static_cast<std::size_t>(j1 - j0);
    std::vector<float> out(nx * sy * nz);
    bool ok = true;
    for (std::size_t k = 0; k < nz; ++k)
        for (std::size_t j = 0; j < sy; ++j) {
            const double* src = v.data() + nx * (j0 + j + ny * k);
            float* dst = out.data() + nx * (j + sy * k);
            for (std::size_t i = 0; i < nx; ++i) {
                ok = ok && std::isfinite(src[i]);
                dst[i] = static_cast<float>(src[i]);
            }
        }
    if (!ok) throw kryct::ConfigError(std::string(what) + " contains non-finite values");
    return out;
}

inline kryct::ReconReport run_slab(const Communicator& comm, int kind,
                                   const kryct::ProjectionSet& proj, const kryct::GridSpec& grid,
                                   const kryct::Volume* prior,
                                   const kryct::RegularizationParams* params, std::size_t iters,
                                   double tol, const kryct::ReconOptions& opts) {
    proj.geometry.validate();
    if (proj.data.size() != proj.geometry.ray_count())
        throw kryct::ConfigError("projection data length does not match geometry");
    grid.validate();
    if (opts.hook)
        throw kryct::ConfigError("ReconOptions::hook is not served by the slab-sharded solves "
                                 "(each rank holds a slab of the iterate)");
    const auto [j0, j1] = slab_range(comm, grid, proj.geometry);
    kryct::GridSpec sg = grid;
    sg.dims.ny = j1 - j0;
    sg.origin.y = grid.origin.y + j0 * grid.spacing.y;
    CheckedOut co(sg, proj.geometry);
    const GpuConeBeamProjector& A = *co.h;
    check(kct_use_comm_slab(A.handle(), comm.handle(), j0, grid.dims.ny));
    struct Leave {  // a cached handle goes back in single-process mode
        kct_projector* h;
        ~Leave() { kct_use_comm_slab(h, nullptr, 0, 0); }
    } leave{A.handle()};
    std::vector<float> b(proj.data.size());
    if (!to_f32(proj.data, b.data()))
        throw kryct::ConfigError("projections contain non-finite values");
    auto slab_of = [&](const kryct::Volume& v, const char* what) {
        if (!(v.dims == grid.dims))
            throw kryct::ConfigError(std::string(what) + " does not match the reconstruction grid");
        return y_slab_f32(v.data, grid.dims, j0, j1, what);
    };
    std::vector<float> pr, x0, gt;
    if (prior) pr = slab_of(*prior, "prior volume");
    if (opts.initial) x0 = slab_of(*opts.initial, "initial volume");
    if (opts.ground_truth) gt = slab_of(*opts.ground_truth, "ground truth");
    const std::size_t ms = sg.dims.count(), m = grid.dims.count();
    std::vector<float> x(ms);
    const std::size_t outer = params ? params->outer_iters : 1;
    const std::size_t inner = params ? params->inner_iters : iters;
    std::vector<double> obj(outer * inner + outer + 1), res(outer * inner), err(outer * inner),
        secs(outer + 1);
    std::vector<uint64_t> bnd(outer + 1);
    kct_report rep{};
    rep.objective_history = obj.data();
    rep.residual_history = res.data();
    rep.error_history = err.data();
    rep.outer_boundaries = bnd.data();
    rep.outer_seconds = secs.data();
    const float* ppr = pr.empty() ? nullptr : pr.data();
    const float* px0 = x0.empty() ? nullptr : x0.data();
    const float* pgt = gt.empty() ? nullptr : gt.data();
    if (params) {
        const kct_reg_params p{params->alpha,       params->lambda,       params->tau,
                               params->outer_iters, params->inner_iters, params->inner_tolerance,
                               params->warm_start ? 1 : 0};
        check(kct_irn(A.handle(), kind, b.data(), ppr, px0, pgt, &p, x.data(), &rep, KCT_MEM_HOST,
                      KCT_LAYOUT_REFERENCE, nullptr));
    } else {
        check(kct_cgls_recon(A.handle(), b.data(), iters, px0, pgt, tol, x.data(), &rep,
                             KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr));
    }
    // join the slabs: every rank places its planes in a zero volume; the sum
    // over the ranks (x + 0 + ... + 0, exact) is the whole iterate everywhere
    std::vector<float> full(comm.world() > 1 ? m : 0);
    const float* whole = x.data();
    if (comm.world() > 1) {
        const std::size_t nx = grid.dims.nx, ny = grid.dims.ny, nz = grid.dims.nz,
                          sy = static_cast<std::size_t>(j1 - j0);
        for (std::size_t k = 0; k < nz; ++k)
            for (std::size_t j = 0; j < sy; ++j)
                std::copy_n(x.data() + nx * (j + sy * k), nx, full.data() + nx * (j0 + j + ny * k));
        check(kct_comm_allreduce_host(comm.handle(), full.data(), m, 0, 0));
        whole = full.data();
    }
    kryct::ReconReport r;
    r.volume.dims = grid.dims;
    r.volume.spacing = grid.spacing;
    r.volume.origin = grid.origin;
    r.volume.data.assign(whole, whole + m);
    r.objective_history.assign(obj.begin(), obj.begin() + rep.objective_count);
    r.residual_history.assign(res.begin(), res.begin() + rep.residual_count);
    r.error_history.assign(err.begin(), err.begin() + rep.error_count);
    for (std::size_t i = 0; i < rep.outer_count; ++i) {
        r.outer_boundaries.push_back(bnd[i]);
        r.outer_seconds.push_back(secs[i]);
    }
    r.solve_seconds = rep.solve_seconds;
    r.converged = rep.converged != 0;
    return r;
}

}  // namespace detail

/// cgls_recon (recon.hpp:312-315) over the communicator's GPUs.
inline kryct::ReconReport cgls_recon(const Communicator& comm, const kryct::ProjectionSet& proj,
                                     const kryct::GridSpec& grid, std::size_t iters,
                                     const kryct::ReconOptions& opts = {}, double tolerance = 0.0) {
    return detail::run_slab(comm, KCT_KIND_TV, proj, grid, nullptr, nullptr, iters, tolerance, opts);
}
/// irn_tv (recon.hpp:252-255) over the communicator's GPUs.
inline kryct::ReconReport irn_tv(const Communicator& comm, const kryct::ProjectionSet& proj,
                                 const kryct::GridSpec& grid,
                                 const kryct::RegularizationParams& params,
                                 const kryct::ReconOptions& opts = {}) {
    return detail::run_slab(comm, KCT_KIND_TV, proj, grid, nullptr, &params, 0, 0.0, opts);
}
/// irn_piple (recon.hpp:260-263) over the communicator's GPUs.
inline kryct::ReconReport irn_piple(const Communicator& comm, const kryct::ProjectionSet& proj,
                                    const kryct::GridSpec& grid, const kryct::Volume& prior,
                                    const kryct::RegularizationParams& params,
                                    const kryct::ReconOptions& opts = {}) {
    return detail::run_slab(comm, KCT_KIND_PIPLE, proj, grid, &prior, &params, 0, 0.0, opts);
}
/// irn_piccs (recon.hpp:267-270) over the communicator's GPUs.
inline kryct::ReconReport irn_piccs(const Communicator& comm, const kryct::ProjectionSet& proj,
                                    const kryct::GridSpec& grid, const kryct::Volume& prior,
                                    const kryct::RegularizationParams& params,
                                    const kryct::ReconOptions& opts = {}) {
    return detail::run_slab(comm, KCT_KIND_PICCS, proj, grid, &prior, &params, 0, 0.0, opts);
}

}  // namespace kryct_b200
