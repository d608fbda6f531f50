// MEASUREMENT TOOL (not a test): the C++ drop-in's real per-call cost in a
// fresh process.  The reference's own types and call (kryct::ProjectionSet of
// doubles, kryct_b200::irn_piccs with the reference signature), BASELINE c3
// (256^3 @ 0.5 mm, 384^2 @ 0.5 mm, 60 views), 4x5 PICCS, alpha = 0.5: the
// first call (handle creation: walk tables, workspace), then cached calls.
// Built by tools/Makefile into build/bench_shim (reference headers at build time); run by
// bench.py; prints one JSON line.
#include <kryct/recon.hpp>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <numbers>

#include "kryct_b200.hpp"

using namespace kryct;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

int main() {
    const int n = 256, det = 384, views = 60;
    GridSpec grid = GridSpec::centered({n, n, n}, {0.5, 0.5, 0.5});
    ConeBeamGeometry g;
    g.dso = 1000.0;
    g.dsd = 1500.0;
    g.detector = {det, det, 0.5, 0.5};
    for (int i = 0; i < views; ++i) g.angles.push_back(2.0 * std::numbers::pi * i / views);
    // a smooth synthetic object (two ellipsoids) and its projections
    std::vector<double> x(grid.dims.count());
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const double u = (i + 0.5) / n - 0.5, v = (j + 0.5) / n - 0.5, w = (k + 0.5) / n - 0.5;
                double a = (u * u + v * v) / 0.16 + w * w / 0.2 < 1.0 ? 0.02 : 0.0;
                a += ((u - 0.1) * (u - 0.1) + v * v + w * w) / 0.01 < 1.0 ? 0.01 : 0.0;
                x[(size_t)i + n * ((size_t)j + (size_t)n * k)] = a;
            }
    const auto t0 = clk::now();
    kryct_b200::GpuConeBeamProjector A(grid, g);  // includes CUDA context start-up
    const auto t1 = clk::now();
    kryct_b200::GpuConeBeamProjector A2(grid, g);  // a second handle: tables + workspace only
    const auto t2 = clk::now();
    ProjectionSet proj(g);
    proj.data = A.apply(x);
    Volume prior(grid);
    for (size_t i = 0; i < x.size(); ++i) prior.data[i] = 0.95 * x[i];
    RegularizationParams p;
    p.alpha = 0.5;
    p.outer_iters = 4;
    p.inner_iters = 5;
    kryct_b200::clear_handle_cache();
    const auto t3 = clk::now();
    const auto r1 = kryct_b200::irn_piccs(proj, grid, prior, p);  // builds its cached handle
    const auto t4 = clk::now();
    double best = 1e30, solve = 0.0;
    for (int r = 0; r < 3; ++r) {
        const auto a = clk::now();
        const auto rr = kryct_b200::irn_piccs(proj, grid, prior, p);
        const auto b = clk::now();
        if (secs(a, b) < best) {
            best = secs(a, b);
            solve = rr.solve_seconds;
        }
    }
    // the library's own host-buffer path (C ABI, page-locked float buffers):
    // what the shim adds on top is the double <-> float conversion, the
    // validation and the result allocation
    double cabi = 1e30;
    {
        const std::size_t M = grid.dims.count(), N = g.ray_count();
        void *pb = nullptr, *pp = nullptr, *px = nullptr;
        kct_host_alloc(N * sizeof(float), &pb);
        kct_host_alloc(M * sizeof(float), &pp);
        kct_host_alloc(M * sizeof(float), &px);
        float *fb = static_cast<float*>(pb), *fp = static_cast<float*>(pp);
        for (std::size_t i = 0; i < N; ++i) fb[i] = (float)proj.data[i];
        for (std::size_t i = 0; i < M; ++i) fp[i] = (float)prior.data[i];
        const kct_reg_params kp{0.5, 0.5, 0.0, 4, 5, 0.0, 1};
        for (int r = 0; r < 3; ++r) {
            kct_report rep{};
            const auto a = clk::now();
            kct_irn_piccs(A.handle(), fb, fp, nullptr, nullptr, &kp, static_cast<float*>(px), &rep,
                          KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr);
            cabi = std::min(cabi, secs(a, clk::now()));
        }
        kct_host_free(pb);
        kct_host_free(pp);
        kct_host_free(px);
    }
    std::printf("{\"what\": \"kryct_b200::irn_piccs (reference signature, double buffers), c3 4x5, "
                "fresh process\", \"first_handle_with_context_s\": %.4f, \"handle_create_s\": %.4f, "
                "\"first_call_s\": %.4f, \"cached_call_s\": %.4f, \"cached_solve_seconds\": %.4f, "
                "\"first_call_solve_seconds\": %.4f, \"c_abi_pinned_float_call_s\": %.4f, "
                "\"iterations\": %zu}\n",
                secs(t0, t1), secs(t1, t2), secs(t3, t4), best, solve, r1.solve_seconds, cabi,
                r1.residual_history.size());
    return 0;
}
