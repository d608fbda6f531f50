// TEST INFRASTRUCTURE: the C++ drop-in shim (include/kryct_b200.hpp) against
// the unmodified reference.  Compiled against /root/reference headers by
// oracle/Makefile (target `shim`) into oracle/_ref/test_shim; run on a GPU box by
// tests/test_shim_gpu.py.  Exit code 0 = all checks passed.
#include <kryct/diffreg.hpp>
#include <kryct/krylov.hpp>
#include <kryct/projector.hpp>
#include <kryct/recon.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <random>
#include <stdexcept>

#include "kryct_b200.hpp"

using namespace kryct;

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}

static int fails = 0;
static void expect(bool ok, const char* what, double v) {
    std::printf("%-52s %s (%.3e)\n", what, ok ? "ok" : "FAIL", v);
    if (!ok) ++fails;
}

int main() {
    GridSpec grid = GridSpec::centered({32, 32, 24}, {2.0, 2.0, 2.0});
    ConeBeamGeometry g;
    g.dso = 1000.0;
    g.dsd = 1500.0;
    g.detector = {48, 40, 2.0, 2.0};
    for (int i = 0; i < 24; ++i) g.angles.push_back(2.0 * std::numbers::pi * i / 24.0);
    std::mt19937 rng(7);
    std::uniform_real_distribution<float> u(0.f, 0.04f);
    std::vector<double> x(grid.dims.count()), y(g.ray_count());
    for (auto& v : x) v = u(rng);
    for (auto& v : y) v = u(rng);

    ConeBeamProjector ref(grid, g);
    kryct_b200::GpuConeBeamProjector gpu(grid, g);
    expect(rel(gpu.apply(x), ref.apply(x)) < 1e-4, "GpuConeBeamProjector::apply vs reference",
           rel(gpu.apply(x), ref.apply(x)));
    expect(rel(gpu.apply_adjoint(y), ref.apply_adjoint(y)) < 1e-4,
           "GpuConeBeamProjector::apply_adjoint vs reference",
           rel(gpu.apply_adjoint(y), ref.apply_adjoint(y)));

    // the reference's own cgls driving the GPU operator
    const auto b = ref.apply(x);
    std::vector<double> bf(b.begin(), b.end());
    for (auto& v : bf) v = static_cast<float>(v);
    const std::vector<double> x0(grid.dims.count(), 0.0);
    const auto r_ref = cgls(ref, bf, x0, {.max_iters = 10});
    const auto r_gpu = cgls(gpu, bf, x0, {.max_iters = 10});
    expect(rel(r_gpu.x, r_ref.x) < 1e-3, "kryct::cgls(GpuConeBeamProjector) vs reference",
           rel(r_gpu.x, r_ref.x));

    // device-resident cgls over a caller-assembled stack (krylov.hpp:59-127 on
    // linear_map.hpp:159-216): the reweighted system recon.hpp:211-221 builds,
    // assembled with the reference's own compose / DiagonalMap / stack_maps
    {
        auto gpu_sp = std::make_shared<kryct_b200::GpuConeBeamProjector>(grid, g);
        auto ref_sp = std::make_shared<ConeBeamProjector>(grid, g);
        auto D = make_diff(grid.dims);
        const auto w1 = tv_weights(D->apply(x), 1e-3);
        std::vector<double> xs(x.size());
        for (size_t i = 0; i < x.size(); ++i) xs[i] = static_cast<float>(0.1 * x[i]);
        auto w2 = tv_weights(D->apply(xs), 1e-3);
        std::vector<double> w1f(w1.size()), w2f(w2.size()), wi(x.size());
        for (size_t i = 0; i < w1.size(); ++i) w1f[i] = static_cast<float>(w1[i]);
        for (size_t i = 0; i < w2.size(); ++i) w2f[i] = static_cast<float>(w2[i]);
        for (size_t i = 0; i < wi.size(); ++i) wi[i] = static_cast<float>(0.5 + 10.0 * x[i]);
        auto mk = [&](std::shared_ptr<const LinearMap> A) {
            return stack_maps({{1.0, A},
                               {0.01, compose(std::make_shared<DiagonalMap>(w1f), D)},
                               {0.02, compose(std::make_shared<DiagonalMap>(w2f), D)},
                               {0.05, compose(std::make_shared<DiagonalMap>(wi),
                                              std::make_shared<IdentityMap>(x.size()))}});
        };
        const auto S_gpu = mk(gpu_sp);
        const auto S_ref = mk(ref_sp);
        std::vector<double> rhs(S_ref->range_size(), 0.0);
        std::copy(bf.begin(), bf.end(), rhs.begin());
        for (size_t i = 0; i < x.size(); ++i)
            rhs[S_ref->block_offset(3) + i] = static_cast<float>(0.05 * wi[i] * 0.9 * x[i]);
        const auto s_ref = cgls(*S_ref, rhs, x0, {.max_iters = 8});
        std::vector<size_t> seen;
        KrylovConfig kc;
        kc.max_iters = 8;
        kc.hook = [&](std::size_t it, std::span<const double>) { seen.push_back(it); };
        const auto s_gpu = kryct_b200::cgls(*S_gpu, rhs, x0, kc);
        expect(rel(s_gpu.x, s_ref.x) < 1e-3, "kryct_b200::cgls(stack) vs kryct::cgls(stack)",
               rel(s_gpu.x, s_ref.x));
        expect(s_gpu.trace.iterations == s_ref.trace.iterations &&
                   rel(s_gpu.trace.residual_norms, s_ref.trace.residual_norms) < 1e-3,
               "stack cgls: residual norms", rel(s_gpu.trace.residual_norms, s_ref.trace.residual_norms));
        expect(seen.size() == 8 && seen.front() == 1 && seen.back() == 8 &&
                   s_gpu.trace.wall_times.size() == 8,
               "stack cgls: hook order + wall_times", (double)seen.size());
        // warm start with a tolerance (krylov.hpp:81-96)
        const auto t_ref = cgls(*S_ref, rhs, xs, {.max_iters = 30, .tolerance = 0.05});
        const auto t_gpu = kryct_b200::cgls(*S_gpu, rhs, xs, {.max_iters = 30, .tolerance = 0.05});
        expect(t_gpu.trace.converged == t_ref.trace.converged &&
                   t_gpu.trace.iterations == t_ref.trace.iterations && rel(t_gpu.x, t_ref.x) < 1e-3,
               "stack cgls: warm start + tolerance", rel(t_gpu.x, t_ref.x));
        bool bad_rhs = false, bad_map = false;
        try {
            kryct_b200::cgls(*S_gpu, bf, x0, {.max_iters = 2});
        } catch (const ConfigError&) {
            bad_rhs = true;
        }
        try {   // a CPU projector block is not something the device solver can run
            kryct_b200::cgls(*S_ref, rhs, x0, {.max_iters = 2});
        } catch (const ConfigError&) {
            bad_map = true;
        }
        expect(bad_rhs && bad_map, "stack cgls: ConfigError on size / unsupported block", 0.0);
    }

    // solver entry points with the reference signatures
    ProjectionSet proj(g);
    proj.data = bf;
    Volume prior(grid);
    for (size_t i = 0; i < x.size(); ++i) prior.data[i] = static_cast<float>(0.9 * x[i]);
    RegularizationParams p;
    p.alpha = 0.5;
    p.outer_iters = 2;
    p.inner_iters = 4;
    const auto a_ref = irn_piccs(proj, grid, prior, p);
    const auto a_gpu = kryct_b200::irn_piccs(proj, grid, prior, p);
    expect(rel(a_gpu.volume.data, a_ref.volume.data) < 1e-3, "kryct_b200::irn_piccs vs irn_piccs",
           rel(a_gpu.volume.data, a_ref.volume.data));
    expect(a_gpu.objective_history.size() == a_ref.objective_history.size() &&
               rel(a_gpu.objective_history, a_ref.objective_history) < 1e-3,
           "objective history", rel(a_gpu.objective_history, a_ref.objective_history));
    expect(a_gpu.outer_boundaries == a_ref.outer_boundaries, "outer boundaries", 0.0);
    const auto c_ref = cgls_recon(proj, grid, 8);
    const auto c_gpu = kryct_b200::cgls_recon(proj, grid, 8);
    expect(rel(c_gpu.volume.data, c_ref.volume.data) < 1e-3, "kryct_b200::cgls_recon vs cgls_recon",
           rel(c_gpu.volume.data, c_ref.volume.data));

    // ReconOptions::hook: every inner iterate, in order, numbered across the
    // outer cycles (recon.hpp:223-228; the reference's test_krylov.cpp:120-135)
    {
        std::vector<std::size_t> seen_ref, seen_gpu;
        std::vector<std::vector<double>> it_ref, it_gpu;
        ReconOptions o_ref, o_gpu;
        o_ref.hook = [&](std::size_t it, std::span<const double> xi) {
            seen_ref.push_back(it);
            it_ref.emplace_back(xi.begin(), xi.end());
        };
        o_gpu.hook = [&](std::size_t it, std::span<const double> xi) {
            seen_gpu.push_back(it);
            it_gpu.emplace_back(xi.begin(), xi.end());
        };
        irn_piccs(proj, grid, prior, p, o_ref);
        const auto h_gpu = kryct_b200::irn_piccs(proj, grid, prior, p, o_gpu);
        bool order = seen_gpu == seen_ref && seen_gpu.size() == 8;
        for (std::size_t i = 0; i < seen_gpu.size(); ++i) order = order && seen_gpu[i] == i + 1;
        expect(order, "hook: iterations 1..8 in order, as the reference", (double)seen_gpu.size());
        double worst = 0.0;
        for (std::size_t i = 0; i < it_gpu.size() && i < it_ref.size(); ++i)
            worst = std::max(worst, rel(it_gpu[i], it_ref[i]));
        expect(worst < 1e-3 && it_gpu.size() == it_ref.size(), "hook: iterates vs reference", worst);
        expect(it_gpu.back() == h_gpu.volume.data, "hook: last iterate == result volume", 0.0);
        // cached handle: a repeated call is bit-identical
        const auto again = kryct_b200::irn_piccs(proj, grid, prior, p);
        expect(again.volume.data == h_gpu.volume.data, "cached handle: repeated call bitwise", 0.0);
        // a throwing hook surfaces after the solve
        ReconOptions o_bad;
        o_bad.hook = [](std::size_t it, std::span<const double>) {
            if (it == 2) throw std::runtime_error("hook failure");
        };
        bool hook_threw = false;
        try {
            kryct_b200::cgls_recon(proj, grid, 4, o_bad);
        } catch (const std::runtime_error&) {
            hook_threw = true;
        }
        expect(hook_threw, "hook exception propagates to the caller", 0.0);
    }

    // multi-GPU entry points on the library's own NCCL communicator, world
    // size 1 (one GPU here; NCCL refuses two ranks on one device): the
    // y-slab-sharded drivers reduce to the single-process solves bit for bit
    {
        kryct_b200::Communicator comm(0, 1, kryct_b200::Communicator::unique_id());
        expect(comm.rank() == 0 && comm.world() == 1, "Communicator: rank 0 of 1", 0.0);
        const auto range = kryct_b200::slab_range(comm, grid, g);
        expect(range.first == 0 && range.second == grid.dims.ny, "slab_range: whole grid", 0.0);
        std::vector<double> v{1.0, 2.5, -3.0};
        comm.all_reduce(v);
        comm.all_reduce(v, true);
        expect(v == std::vector<double>{1.0, 2.5, -3.0}, "Communicator::all_reduce (sum, max)", 0.0);
        const auto s_gpu = kryct_b200::irn_piccs(comm, proj, grid, prior, p);
        expect(s_gpu.volume.data == a_gpu.volume.data, "irn_piccs(comm, ...) == irn_piccs(...) bitwise",
               rel(s_gpu.volume.data, a_gpu.volume.data));
        expect(s_gpu.objective_history == a_gpu.objective_history, "slab objective history bitwise", 0.0);
        const auto sc = kryct_b200::cgls_recon(comm, proj, grid, 8);
        expect(sc.volume.data == c_gpu.volume.data, "cgls_recon(comm, ...) bitwise", 0.0);
        // from_env with the launcher's variables of a 1-rank job
        setenv("RANK", "0", 1);
        setenv("WORLD_SIZE", "1", 1);
        setenv("LOCAL_RANK", "0", 1);
        auto env_comm = kryct_b200::Communicator::from_env();
        expect(env_comm.world() == 1, "Communicator::from_env", 0.0);
        // a handle that served a slab solve goes back to the cache single-process
        const auto after = kryct_b200::irn_piccs(proj, grid, prior, p);
        expect(after.volume.data == a_gpu.volume.data, "cached handle after a slab solve", 0.0);
        bool rejected = false;
        try {
            ReconOptions o;
            o.hook = [](std::size_t, std::span<const double>) {};
            kryct_b200::cgls_recon(comm, proj, grid, 2, o);
        } catch (const ConfigError&) {
            rejected = true;
        }
        expect(rejected, "slab solves reject ReconOptions::hook (ConfigError)", 0.0);
    }

    // error taxonomy (test_projector.cpp:113-120)
    bool threw = false;
    try {
        ConeBeamGeometry tiny = g;
        tiny.dso = 40.0;
        tiny.dsd = 90.0;
        kryct_b200::GpuConeBeamProjector bad(GridSpec::centered({32, 32, 32}, {10, 10, 10}), tiny);
    } catch (const ConfigError&) {
        threw = true;
    }
    expect(threw, "source inside the volume -> ConfigError", 0.0);
    std::printf(fails ? "FAILED %d\n" : "ALL OK\n", fails);
    return fails ? 1 : 0;
}
