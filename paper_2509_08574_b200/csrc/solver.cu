// solver.cu — device-resident CGLS on the stacked IRN systems.
//
// The reference solves, per outer cycle (recon.hpp:192-242),
//     min || [A; a*W1*D; l*W2*D] x - [b; 0; l*W2*D*x_p] ||        (PICCS)
// with cgls (krylov.hpp:59-127) on materialised stacked vectors of length
// N + 6M.  In exact arithmetic the regulariser blocks of the CGLS residual are
// always  r1 = -a*W1*D*x  and  r2 = -l*W2*D*(x - x_p)  (block 2 of the rhs is
// 0, block 3 is l*W2*D*x_p, and x moves by the same steps as r), so this
// implementation keeps only the projection block r0 (length N) on the
// recurrence and evaluates the regulariser blocks from x and p in fused
// stencil kernels:
//     A~^T r   = A^T r0 - a^2 D^T W1^2 D x - l^2 D^T W2^2 D (x - x_p)
//     ||A~ p||^2 = ||A p||^2 + a^2 ||W1 D p||^2 + l^2 ||W2 D p||^2
//     ||r||^2  = ||r0||^2 + a^2 ||W1 D x||^2 + l^2 ||W2 D (x - x_p)||^2
// PIPLE's l*I block works the same way with D -> I, W2 -> 1.  Vectors are
// float32; every reduction is float64, deterministic (fixed grid, per-block
// partials, fixed-order final sum), as the reference's sequential double
// reductions are (vector_ops.hpp:3-5).  The CGLS scalars (gamma, delta, a,
// beta) live on the device so the host never waits inside a cycle.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <initializer_list>
#include <string>
#include <vector>

#include <cuda.h>

#include "solver.cuh"

namespace kct {

namespace {

constexpr int kGrid = 148 * 8;  // fixed grid -> deterministic partial sums
constexpr int kBlock = 256;
constexpr int kSlots = 8;

struct Ctl {
    double gamma, a, beta, stop_tol;
    double r2, e2, gt2, ref2;
    double alpha2, lambda2;
    double tv1, tv2, data;
    int stop, converged, breakdown, error;
    int iters, x_nonzero, pad0, pad1;
};

enum ScalarMode {
    S_DATA = 0,    // data = sum slot0
    S_TV = 1,      // tv1 = slot1, tv2 = slot2
    S_INIT = 2,    // gamma = slot0 (reset flags, tolerance)
    S_DELTA = 3,   // delta = slot0 + a2*slot1 + l2*slot2 -> a
    S_GAMMA = 4,   // gamma' = slot0; residual from r2(slot4), reg slot1/2; err slot5
    S_REF = 5,     // ref2 = slot0, x_nonzero = slot3 > 0
    S_GT2 = 6,     // gt2 = slot0
    S_OBJ = 7,     // obj_out[idx] = data + ...
};

// Regulariser configuration shared by the stencil kernels.
struct RegCfg {
    int nx, ny, nz;  // this rank's grid (the whole grid unless y-slab sharded)
    int j0, nyg;     // y-slab: global index of local plane 0, global plane count
    int use_w1;      // a != 0: TV block present
    int mode2;       // 0 none, 1 PICCS (W2 D block), 2 PIPLE (I block)
    float alpha2, lambda2;
    float tau2;
};

__device__ __forceinline__ void decode(size_t v, const RegCfg& c, int& k, int& i, int& j) {
    const unsigned p = (unsigned)(v / (unsigned)c.nz);
    k = (int)(v - (size_t)p * c.nz);
    i = (int)(p % (unsigned)c.nx);
    j = (int)(p / (unsigned)c.nx);
}

// forward differences of f at v (zero at the far face, diffreg.hpp:34-49)
__device__ __forceinline__ void fdiff(const float* __restrict__ f, size_t v, int k, int i, int j,
                                      const RegCfg& c, size_t si, size_t sj, float fv, float& gx,
                                      float& gy, float& gz) {
    gx = i + 1 < c.nx ? f[v + si] - fv : 0.f;
    gy = j + c.j0 + 1 < c.nyg ? f[v + sj] - fv : 0.f;
    gz = k + 1 < c.nz ? f[v + 1] - fv : 0.f;
}

__device__ __forceinline__ void write_partials(double* part, int slot, double v, double* sm) {
    const double t = block_sum(v, sm);
    if (threadIdx.x == 0) part[slot * kGrid + blockIdx.x] = t;
}

// ---- weights + smoothed-TV sums (tv_weights diffreg.hpp:142-156; ----------
// smoothed_tv :118-126; the PIPLE quadratic of recon.hpp:107-114) ----------
// w = r^(-1/2) with r = sqrt(|grad|^2 + tau^2): r by the IEEE square root (it
// also enters the smoothed-TV sums), w by rsqrtf (<= 2 ulp; a second square
// root and a division measured 94 vs 73 us per launch of the issue-bound
// tile kernel at c3) — the same expression in all three weight kernels.
__global__ void __launch_bounds__(kBlock) k_weights(const float* __restrict__ x,
                                                    const float* __restrict__ xp,
                                                    float* __restrict__ w1, float* __restrict__ w2,
                                                    RegCfg c, int write_w, double* part) {
    __shared__ double sm[32];
    const size_t m = (size_t)c.nx * c.ny * c.nz, si = c.nz, sj = (size_t)c.nz * c.nx;
    double t1 = 0.0, t2 = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < m;
         v += (size_t)gridDim.x * blockDim.x) {
        int k, i, j;
        decode(v, c, k, i, j);
        const float xv = x[v];
        if (c.use_w1) {
            float gx, gy, gz;
            fdiff(x, v, k, i, j, c, si, sj, xv, gx, gy, gz);
            const float m2 = gx * gx + gy * gy + gz * gz + c.tau2;
            const float r = sqrtf(m2);
            t1 += (double)r;
            if (write_w) w1[v] = rsqrtf(r);
        }
        if (c.mode2 == 1) {
            const float dv = xv - xp[v];
            const float gx = i + 1 < c.nx ? (x[v + si] - xp[v + si]) - dv : 0.f;
            const float gy = j + c.j0 + 1 < c.nyg ? (x[v + sj] - xp[v + sj]) - dv : 0.f;
            const float gz = k + 1 < c.nz ? (x[v + 1] - xp[v + 1]) - dv : 0.f;
            const float r = sqrtf(gx * gx + gy * gy + gz * gz + c.tau2);
            t2 += (double)r;
            if (write_w) w2[v] = rsqrtf(r);
        } else if (c.mode2 == 2) {
            const double d = (double)xv - (double)xp[v];
            t2 += d * d;
        }
    }
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// ---- r = b - q (q == nullptr: r = b); slot0 = ||r||^2 ---------------------
__global__ void __launch_bounds__(kBlock) k_resid(const float* __restrict__ b,
                                                  const float* __restrict__ q,
                                                  float* __restrict__ r, size_t n, double* part,
                                                  int slot) {
    __shared__ double sm[32];
    double t = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const float rv = q ? b[v] - q[v] : b[v];
        if (r) r[v] = rv;
        t += (double)rv * (double)rv;
    }
    write_partials(part, slot, t, sm);
}

// ---- s = A^T r0 - a^2 D^T W1^2 D x - l^2 D^T W2^2 D (x - x_p) --------------
// slot0 = ||s||^2, slot1 = ||W1 D x||^2, slot2 = ||W2 D (x-x_p)||^2 (or ||x-x_p||^2)
// x == nullptr means x = 0 (the right-hand-side adjoint for the tolerance ref).
__global__ void __launch_bounds__(kBlock) k_reggrad(const float* __restrict__ sA,
                                                    const float* __restrict__ x,
                                                    const float* __restrict__ xp,
                                                    const float* __restrict__ w1,
                                                    const float* __restrict__ w2,
                                                    float* __restrict__ s, RegCfg c, double* part) {
    __shared__ double sm[32];
    const size_t m = (size_t)c.nx * c.ny * c.nz, si = c.nz, sj = (size_t)c.nz * c.nx;
    double ts = 0.0, t1 = 0.0, t2 = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < m;
         v += (size_t)gridDim.x * blockDim.x) {
        int k, i, j;
        decode(v, c, k, i, j);
        float sv = sA[v];
        const float xv = x ? x[v] : 0.f;
        if (c.use_w1 && x) {
            float gx, gy, gz;
            fdiff(x, v, k, i, j, c, si, sj, xv, gx, gy, gz);
            const float wv = w1[v], wv2 = wv * wv;
            float g = -wv2 * (gx + gy + gz);
            if (i > 0) { const float w = w1[v - si]; g += w * w * (xv - x[v - si]); }
            if (j + c.j0 > 0) { const float w = w1[v - sj]; g += w * w * (xv - x[v - sj]); }
            if (k > 0) { const float w = w1[v - 1]; g += w * w * (xv - x[v - 1]); }
            sv -= c.alpha2 * g;
            t1 += (double)(wv2 * (gx * gx + gy * gy + gz * gz));
        }
        if (c.mode2 == 1) {
            auto d = [&](size_t u) { return (x ? x[u] : 0.f) - xp[u]; };
            const float dv = d(v);
            const float gx = i + 1 < c.nx ? d(v + si) - dv : 0.f;
            const float gy = j + c.j0 + 1 < c.nyg ? d(v + sj) - dv : 0.f;
            const float gz = k + 1 < c.nz ? d(v + 1) - dv : 0.f;
            const float wv = w2[v], wv2 = wv * wv;
            float g = -wv2 * (gx + gy + gz);
            if (i > 0) { const float w = w2[v - si]; g += w * w * (dv - d(v - si)); }
            if (j + c.j0 > 0) { const float w = w2[v - sj]; g += w * w * (dv - d(v - sj)); }
            if (k > 0) { const float w = w2[v - 1]; g += w * w * (dv - d(v - 1)); }
            sv -= c.lambda2 * g;
            t2 += (double)(wv2 * (gx * gx + gy * gy + gz * gz));
        } else if (c.mode2 == 2) {
            const float dv = xv - xp[v];
            sv -= c.lambda2 * dv;
            t2 += (double)dv * (double)dv;
        }
        s[v] = sv;
        ts += (double)sv * (double)sv;
    }
    write_partials(part, 0, ts, sm);
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// ---- float4 versions of the three stencil kernels (nz % 4 == 0) ----------
// A lane owns 4 consecutive slabs of one voxel column (one float4); the k-1 /
// k+4 neighbours come from the adjacent lanes by shuffle (lanes 0 / 31 load
// them), the i / j neighbours are float4 loads — 4x fewer load instructions
// and all of a lane's loads independent, so the (L2 / DRAM latency bound)
// scalar kernels become bandwidth bound.  Same arithmetic per voxel as the
// scalar kernels; the partial sums add the 4 voxels of a lane in k order.
#ifndef KCT_STENCIL_MINB
#define KCT_STENCIL_MINB 4  // k_reggrad4: cap registers at 64 (2x the warps of the uncapped 118)
#endif
struct Nb4 {
    float f[6];           // f[0] = slab k-1, f[1..4] = slabs k..k+3, f[5] = slab k+4
    float4 ip, im, jp, jm;  // columns i+1, i-1, j+1, j-1 (0 outside the grid)
};

__device__ __forceinline__ float4 ld4(const float* __restrict__ f, size_t v) {
    return __ldg(reinterpret_cast<const float4*>(f + v));
}
__device__ __forceinline__ float q4(const float4& a, int q) {
    return q == 0 ? a.x : (q == 1 ? a.y : (q == 2 ? a.z : a.w));
}

// All lanes must call (shuffles); `ok` false lanes pass v = 0 and get zeros.
template <bool MINUS_I, bool MINUS_J>
__device__ __forceinline__ void load_nb(const float* __restrict__ f, size_t v, int k, int i, int j,
                                        const RegCfg& c, bool ok, int lane, Nb4& n) {
    const size_t si = c.nz, sj = (size_t)c.nz * c.nx;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 a = (ok && f) ? ld4(f, v) : z4;
    n.f[1] = a.x; n.f[2] = a.y; n.f[3] = a.z; n.f[4] = a.w;
    const float up = __shfl_up_sync(0xffffffffu, a.w, 1);
    const float dn = __shfl_down_sync(0xffffffffu, a.x, 1);
    n.f[0] = (ok && f && k > 0) ? (lane > 0 ? up : f[v - 1]) : 0.f;
    n.f[5] = (ok && f && k + 4 < c.nz) ? (lane < 31 ? dn : f[v + 4]) : 0.f;
    n.ip = (ok && f && i + 1 < c.nx) ? ld4(f, v + si) : z4;
    n.jp = (ok && f && j + c.j0 + 1 < c.nyg) ? ld4(f, v + sj) : z4;
    n.im = (MINUS_I && ok && f && i > 0) ? ld4(f, v - si) : z4;
    n.jm = (MINUS_J && ok && f && j + c.j0 > 0) ? ld4(f, v - sj) : z4;
}

__device__ __forceinline__ void decode4(size_t base, int lane, size_t m4, const RegCfg& c, bool& ok,
                                        size_t& v, int& k, int& i, int& j) {
    const size_t e = base + lane;
    ok = e < m4;
    v = ok ? 4 * e : 0;
    decode(v, c, k, i, j);
}

__global__ void __launch_bounds__(kBlock) k_weights4(const float* __restrict__ x,
                                                     const float* __restrict__ xp,
                                                     float* __restrict__ w1, float* __restrict__ w2,
                                                     RegCfg c, int write_w, double* part) {
    __shared__ double sm[32];
    const int lane = threadIdx.x & 31;
    const size_t m4 = (size_t)c.nx * c.ny * c.nz / 4, stride = (size_t)gridDim.x * blockDim.x;
    double t1 = 0.0, t2 = 0.0;
    for (size_t base = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); base < m4;
         base += stride) {
        bool ok;
        size_t v;
        int k, i, j;
        decode4(base, lane, m4, c, ok, v, k, i, j);
        Nb4 X, P;
        load_nb<false, false>(x, v, k, i, j, c, ok, lane, X);
        if (c.mode2) load_nb<false, false>(xp, v, k, i, j, c, ok, lane, P);
        float o1[4], o2[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float xv = X.f[q + 1];
            if (c.use_w1) {
                const float gx = i + 1 < c.nx ? q4(X.ip, q) - xv : 0.f;
                const float gy = j + c.j0 + 1 < c.nyg ? q4(X.jp, q) - xv : 0.f;
                const float gz = k + q + 1 < c.nz ? X.f[q + 2] - xv : 0.f;
                const float r = sqrtf(gx * gx + gy * gy + gz * gz + c.tau2);
                if (ok) t1 += (double)r;
                o1[q] = rsqrtf(r);
            }
            if (c.mode2 == 1) {
                const float dv = xv - P.f[q + 1];
                const float gx = i + 1 < c.nx ? (q4(X.ip, q) - q4(P.ip, q)) - dv : 0.f;
                const float gy = j + c.j0 + 1 < c.nyg ? (q4(X.jp, q) - q4(P.jp, q)) - dv : 0.f;
                const float gz = k + q + 1 < c.nz ? (X.f[q + 2] - P.f[q + 2]) - dv : 0.f;
                const float r = sqrtf(gx * gx + gy * gy + gz * gz + c.tau2);
                if (ok) t2 += (double)r;
                o2[q] = rsqrtf(r);
            } else if (c.mode2 == 2) {
                const double d = (double)xv - (double)P.f[q + 1];
                if (ok) t2 += d * d;
            }
        }
        if (ok && write_w) {
            if (c.use_w1) *reinterpret_cast<float4*>(w1 + v) = make_float4(o1[0], o1[1], o1[2], o1[3]);
            if (c.mode2 == 1) *reinterpret_cast<float4*>(w2 + v) = make_float4(o2[0], o2[1], o2[2], o2[3]);
        }
    }
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// D^T W^2 D f at the 4 voxels of a lane, from f's and w's neighbourhoods
__device__ __forceinline__ void dtwd(const Nb4& F, const Nb4& W, int k, int i, int j,
                                     const RegCfg& c, float g[4], float g2[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float fv = F.f[q + 1];
        const float gx = i + 1 < c.nx ? q4(F.ip, q) - fv : 0.f;
        const float gy = j + c.j0 + 1 < c.nyg ? q4(F.jp, q) - fv : 0.f;
        const float gz = k + q + 1 < c.nz ? F.f[q + 2] - fv : 0.f;
        const float wv = W.f[q + 1], wv2 = wv * wv;
        float t = -wv2 * (gx + gy + gz);
        if (i > 0) { const float w = q4(W.im, q); t += w * w * (fv - q4(F.im, q)); }
        if (j + c.j0 > 0) { const float w = q4(W.jm, q); t += w * w * (fv - q4(F.jm, q)); }
        if (k + q > 0) { const float w = W.f[q]; t += w * w * (fv - F.f[q]); }
        g[q] = t;
        g2[q] = wv2 * (gx * gx + gy * gy + gz * gz);
    }
}

__device__ __forceinline__ void nb_sub(Nb4& a, const Nb4& b) {
#pragma unroll
    for (int q = 0; q < 6; ++q) a.f[q] -= b.f[q];
    a.ip.x -= b.ip.x; a.ip.y -= b.ip.y; a.ip.z -= b.ip.z; a.ip.w -= b.ip.w;
    a.im.x -= b.im.x; a.im.y -= b.im.y; a.im.z -= b.im.z; a.im.w -= b.im.w;
    a.jp.x -= b.jp.x; a.jp.y -= b.jp.y; a.jp.z -= b.jp.z; a.jp.w -= b.jp.w;
    a.jm.x -= b.jm.x; a.jm.y -= b.jm.y; a.jm.z -= b.jm.z; a.jm.w -= b.jm.w;
}

__global__ void __launch_bounds__(kBlock, KCT_STENCIL_MINB) k_reggrad4(const float* __restrict__ sA,
                                                     const float* __restrict__ x,
                                                     const float* __restrict__ xp,
                                                     const float* __restrict__ w1,
                                                     const float* __restrict__ w2,
                                                     float* __restrict__ s, RegCfg c, double* part) {
    __shared__ double sm[32];
    const int lane = threadIdx.x & 31;
    const size_t m4 = (size_t)c.nx * c.ny * c.nz / 4, stride = (size_t)gridDim.x * blockDim.x;
    double ts = 0.0, t1 = 0.0, t2 = 0.0;
    for (size_t base = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); base < m4;
         base += stride) {
        bool ok;
        size_t v;
        int k, i, j;
        decode4(base, lane, m4, c, ok, v, k, i, j);
        const float4 a = ok ? ld4(sA, v) : make_float4(0.f, 0.f, 0.f, 0.f);
        float sv[4] = {a.x, a.y, a.z, a.w};
        float g[4], gg[4];
        Nb4 X, W;
        if (c.use_w1 && x) {
            load_nb<true, true>(x, v, k, i, j, c, ok, lane, X);
            load_nb<true, true>(w1, v, k, i, j, c, ok, lane, W);
            dtwd(X, W, k, i, j, c, g, gg);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                sv[q] -= c.alpha2 * g[q];
                if (ok) t1 += (double)gg[q];
            }
        }
        if (c.mode2 == 1) {
            Nb4 D, P;
            load_nb<true, true>(x, v, k, i, j, c, ok, lane, D);  // x == nullptr -> zeros
            load_nb<true, true>(xp, v, k, i, j, c, ok, lane, P);
            nb_sub(D, P);
            load_nb<true, true>(w2, v, k, i, j, c, ok, lane, W);
            dtwd(D, W, k, i, j, c, g, gg);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                sv[q] -= c.lambda2 * g[q];
                if (ok) t2 += (double)gg[q];
            }
        } else if (c.mode2 == 2) {
            const float4 xv = (ok && x) ? ld4(x, v) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 pv = ok ? ld4(xp, v) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float dv = q4(xv, q) - q4(pv, q);
                sv[q] -= c.lambda2 * dv;
                if (ok) t2 += (double)dv * (double)dv;
            }
        }
        if (ok) {
            *reinterpret_cast<float4*>(s + v) = make_float4(sv[0], sv[1], sv[2], sv[3]);
#pragma unroll
            for (int q = 0; q < 4; ++q) ts += (double)sv[q] * (double)sv[q];
        }
    }
    write_partials(part, 0, ts, sm);
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// a thread's 4-slab quad of a field with its k-1 / k+4 neighbours
struct Q4 {
    float4 c;      // slabs k .. k+3
    float km, kp;  // slab k-1, slab k+4
};
__device__ __forceinline__ float4 sub4(float4 a, float4 b) {
    return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
// D^T W^2 D of the quad F (neighbours fip, fim, fjp, fjm) with weights W
// (centre, i-1, j-1, k-1): dtwd's arithmetic
__device__ __forceinline__ void dtwd_m(const Q4& F, float4 fip, float4 fim, float4 fjp, float4 fjm,
                                       const Q4& W, float4 wim, float4 wjm, int k, bool hasip,
                                       bool hasim, bool hasjp, bool hasjm, int nz, float g[4],
                                       float g2[4]) {
    const float f[6] = {F.km, F.c.x, F.c.y, F.c.z, F.c.w, F.kp};
    const float w[5] = {W.km, W.c.x, W.c.y, W.c.z, W.c.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float fv = f[q + 1];
        const float gx = hasip ? q4(fip, q) - fv : 0.f;
        const float gy = hasjp ? q4(fjp, q) - fv : 0.f;
        const float gz = k + q + 1 < nz ? f[q + 2] - fv : 0.f;
        const float wv = w[q + 1], wv2 = wv * wv;
        float t = -wv2 * (gx + gy + gz);
        if (hasim) { const float ww = q4(wim, q); t += ww * ww * (fv - q4(fim, q)); }
        if (hasjm) { const float ww = q4(wjm, q); t += ww * ww * (fv - q4(fjm, q)); }
        if (k + q > 0) { const float ww = w[q]; t += ww * ww * (fv - f[q]); }
        g[q] = t;
        g2[q] = wv2 * (gx * gx + gy * gy + gz * gz);
    }
}

// ---- k_reggrad4 on TMA tiles (PICCS / TV, x != nullptr) ------------------
// A CTA takes tiles of 64 slabs x 8 x-columns x 4 y-rows; the halo'd tiles of
// x, x_p, W1, W2 (72 x 10 x 6 floats each: slabs k0-4 .. k0+67, columns
// i0-1 .. i0+8, rows j0-1 .. j0+4) arrive in shared memory by four TMA
// tensor loads (cp.async.bulk.tensor.3d, zero fill outside the volume /
// slab, completion on an mbarrier), so every voxel value is read from DRAM
// about once and all the stencil's neighbour reads are shared-memory loads.
// Per voxel the arithmetic of k_reggrad4 (dtwd); the CTA's partial sums add
// in (tile, thread, quad) order: deterministic.
#ifndef KCT_TMA_TY
#define KCT_TMA_TY 2
#endif
constexpr int kTZ = 64, kTX = 8, kTY = KCT_TMA_TY;          // voxels per tile
constexpr int kBZ = kTZ + 8, kBX = kTX + 2, kBY = kTY + 2;  // TMA box (z padded to 16 B)
constexpr int kTile = kBZ * kBX * kBY;                      // floats per tensor tile
constexpr int kStages = 2;  // tile buffers: the next tile's loads overlap this tile's math

__device__ __forceinline__ void tma_load3(float* dst, const CUtensorMap* tm, int z, int x, int y,
                                          unsigned mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(reinterpret_cast<unsigned long long>(tm)),
        "r"(z), "r"(x), "r"(y), "r"(mbar)
        : "memory");
}

__global__ void __launch_bounds__(kBlock, 2) k_reggrad4t(
    const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_xp,
    const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_w2,
    const float* __restrict__ sA, float* __restrict__ s, RegCfg c, int yoff, double* part) {
    extern __shared__ __align__(1024) float tsm[];  // [kStages][4][kTile]
    __shared__ __align__(8) unsigned long long mbar_s[kStages];
    __shared__ double red[32];
    const bool w1on = c.use_w1, m2 = c.mode2 == 1, m3 = c.mode2 == 2;
    const int ntz = (c.nz + kTZ - 1) / kTZ, ntx = (c.nx + kTX - 1) / kTX, nty = (c.ny + kTY - 1) / kTY;
    const int ntiles = ntz * ntx * nty;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&mbar_s[st]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned bytes = (unsigned)(kTile * sizeof(float)) * ((w1on || m2 || m3 ? 1u : 0u) +
                                                                 (m2 || m3 ? 1u : 0u) +
                                                                 (w1on ? 1u : 0u) + (m2 ? 1u : 0u));
    // thread 0: this CTA's n-th tile into stage n % kStages
    auto issue = [&](int tile, int n) {
        const int tz = tile % ntz, rest = tile / ntz, txi = rest % ntx, tyi = rest / ntx;
        const int k0 = tz * kTZ, i0 = txi * kTX, j0 = tyi * kTY;
        float* const T = tsm + (size_t)(n % kStages) * 4 * kTile;
        const unsigned mbar = (unsigned)__cvta_generic_to_shared(&mbar_s[n % kStages]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                     : "memory");
        // tensor coordinates (z, x, y); y shifted by the slab's halo plane
        if (w1on || m2 || m3) tma_load3(T, &tm_x, k0 - 4, i0 - 1, j0 - 1 + yoff, mbar);
        if (m2 || m3) tma_load3(T + kTile, &tm_xp, k0 - 4, i0 - 1, j0 - 1 + yoff, mbar);
        if (w1on) tma_load3(T + 2 * kTile, &tm_w1, k0 - 4, i0 - 1, j0 - 1 + yoff, mbar);
        if (m2) tma_load3(T + 3 * kTile, &tm_w2, k0 - 4, i0 - 1, j0 - 1 + yoff, mbar);
    };
    // thread -> z quad (16 per 64 slabs) x column (8) x rows (kTY / 2 each)
    constexpr int RPT = kTY * kTX * (kTZ / 4) / kBlock;  // quads (rows) per thread
    const int qz = threadIdx.x & 15, col = threadIdx.x >> 4;
    const int tx = col & 7, ty0 = (col >> 3) * RPT;
    const size_t si = c.nz;
    double ts = 0.0, t1 = 0.0, t2 = 0.0;
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    int n = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
        if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, n + 1);
        const int tz = tile % ntz, rest = tile / ntz, txi = rest % ntx, tyi = rest / ntx;
        const int k0 = tz * kTZ, i0 = txi * kTX, j0 = tyi * kTY;
        const float* const TX = tsm + (size_t)(n % kStages) * 4 * kTile;
        const float* const TP = TX + kTile;
        const float* const T1 = TX + 2 * kTile;
        const float* const T2 = TX + 3 * kTile;
        // wait for this tile (use n / kStages of its stage's mbarrier)
        asm volatile(
            "{\n\t.reg .pred done;\n"
            "TMAWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
            "@!done bra TMAWAIT_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(&mbar_s[n % kStages])),
            "r"((unsigned)((n / kStages) & 1))
            : "memory");
        const int k = k0 + 4 * qz, i = i0 + tx;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int ty = ty0 + r, j = j0 + ty;
            const bool ok = k < c.nz && i < c.nx && j < c.ny;
            // tile offset of the quad: slab kk = 4 + 4 qz, column tx + 1, row ty + 1
            const int o = ((ty + 1) * kBX + (tx + 1)) * kBZ + 4 + 4 * qz;
            const size_t v = ok ? (size_t)k + si * ((size_t)i + (size_t)c.nx * j) : 0;
            const float4 a = ok ? __ldg(reinterpret_cast<const float4*>(sA + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
            float sv[4] = {a.x, a.y, a.z, a.w};
            const int jg = j + c.j0;
            const bool hasip = i + 1 < c.nx, hasim = i > 0, hasjp = jg + 1 < c.nyg, hasjm = jg > 0;
            auto ld4s = [&](const float* T, int off) { return *reinterpret_cast<const float4*>(T + off); };
            float g[4], gg[4];
            if (w1on) {
                Q4 X, W;
                X.c = ld4s(TX, o);
                X.km = TX[o - 1];
                X.kp = TX[o + 4];
                W.c = ld4s(T1, o);
                W.km = T1[o - 1];
                dtwd_m(X, ld4s(TX, o + kBZ), ld4s(TX, o - kBZ), ld4s(TX, o + kBZ * kBX),
                       ld4s(TX, o - kBZ * kBX), W, ld4s(T1, o - kBZ), ld4s(T1, o - kBZ * kBX), k,
                       hasip, hasim, hasjp, hasjm, c.nz, g, gg);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sv[q] -= c.alpha2 * g[q];
                    if (ok) t1 += (double)gg[q];
                }
            }
            if (m2) {
                auto d4 = [&](int off) { return sub4(ld4s(TX, off), ld4s(TP, off)); };
                Q4 D, W;
                D.c = d4(o);
                D.km = TX[o - 1] - TP[o - 1];
                D.kp = TX[o + 4] - TP[o + 4];
                W.c = ld4s(T2, o);
                W.km = T2[o - 1];
                dtwd_m(D, d4(o + kBZ), d4(o - kBZ), d4(o + kBZ * kBX), d4(o - kBZ * kBX), W,
                       ld4s(T2, o - kBZ), ld4s(T2, o - kBZ * kBX), k, hasip, hasim, hasjp, hasjm,
                       c.nz, g, gg);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sv[q] -= c.lambda2 * g[q];
                    if (ok) t2 += (double)gg[q];
                }
            } else if (m3) {
                const float4 xv = ld4s(TX, o), pv = ld4s(TP, o);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float dv = q4(xv, q) - q4(pv, q);
                    sv[q] -= c.lambda2 * dv;
                    if (ok) t2 += (double)dv * (double)dv;
                }
            }
            if (ok) {
                *reinterpret_cast<float4*>(s + v) = make_float4(sv[0], sv[1], sv[2], sv[3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) ts += (double)sv[q] * (double)sv[q];
            }
        }
        __syncthreads();  // this stage is free for the tile after next
    }
    write_partials(part, 0, ts, red);
    write_partials(part, 1, t1, red);
    write_partials(part, 2, t2, red);
}

// ---- k_reggrad4m: the same stencil on a y-marching TMA ring ---------------
// k_reggrad4t reloads every tile's halo (72 x 10 x 4 floats for 64 x 8 x 2
// voxels: 2.8x the voxels in L2 -> shared traffic, and the 16-byte z halos
// cost a whole DRAM sector each: 446 MB read per launch for 335 MB of
// operands).  Here a CTA owns a contiguous range of the flattened (column
// tile, y) rows — a column tile is the WHOLE z extent (up to 256 slabs; no z
// halo at all, the volume faces are the stencil's own boundary rules) x mx
// x-columns — and marches along y: every step loads ONE row plane (zbox x
// (mx + 2) floats per tensor, one cp.async.bulk.tensor.3d box {zbox, mx + 2,
// 1} each) into a ring of kMR slots and computes the row whose three planes
// (y - 1, y, y + 1) are resident, so a plane is loaded once per CTA and the
// halo costs (mx + 2) / mx in x plus two planes per run.  kMR - 3 planes are
// in flight ahead of the one being waited for.  kMarch CTAs (one per SM, 512
// threads) carry the work; the other blocks of the fixed partial-sum grid
// write zero partials.  Per voxel the arithmetic of k_reggrad4 (dtwd);
// partial sums in (row, thread, quad) order.
constexpr int kMR = 5;           // ring slots
constexpr int kMarch = 148;      // CTAs that carry work (fixed: deterministic sums)
constexpr int kMBlock = 512;     // threads per march CTA
constexpr int kMZ = 248;         // z tile when nz > 256 (box = tile + 8 <= 256)
constexpr int kMPlaneMax = 2560; // floats per tensor row plane (10 KB)
static_assert(kMarch <= kGrid, "march CTAs within the partial-sum grid");

struct MarchCfg {
    int zt;     // z extent of a column tile (multiple of 4)
    int zbox;   // TMA box z extent (zt + 2 zo)
    int zo;     // z halo on each side (0: the tile is the whole z extent)
    int nzq;    // z quads per tile
    int mx;     // x columns per tile
    int ntz, ntx;
    int plane;  // floats per tensor row plane in shared memory (128-byte multiple)
};

inline MarchCfg march_cfg(const RegCfg& c) {
    MarchCfg m{};
    if (c.nz <= 256) {
        m.ntz = 1;
        m.zt = c.nz;
        m.zo = 0;
    } else {
        m.ntz = (c.nz + kMZ - 1) / kMZ;
        m.zt = (((c.nz + m.ntz - 1) / m.ntz) + 3) & ~3;
        m.zo = 4;
    }
    m.zbox = m.zt + 2 * m.zo;
    m.nzq = m.zt / 4;
    m.mx = std::max(1, std::min({kMBlock / m.nzq, kMPlaneMax / m.zbox - 2, 254}));
    m.ntx = (c.nx + m.mx - 1) / m.mx;
    m.plane = (m.zbox * (m.mx + 2) + 31) & ~31;
    return m;
}

// Walks the row planes a CTA loads, run by run: the CTA's rows [g0, g1) of
// the flattened (column tile, y) space split into runs inside one column
// tile; a run [ja, jb) loads planes ja - 1 .. jb.
struct MarchRuns {
    long g, g1;   // next unvisited flattened row / end of the CTA's range
    int ny;
    int col, j, jb;  // current run: column tile, next plane, last plane (inclusive)
    bool done;
    __device__ void init(long g0, long g1_, int ny_) {
        g = g0; g1 = g1_; ny = ny_;
        done = g0 >= g1_;
        if (!done) start();
    }
    __device__ void start() {
        col = (int)(g / ny);
        const int ja = (int)(g - (long)col * ny);
        const long left = g1 - g;
        jb = (int)(left < (long)(ny - ja) ? ja + left : ny);
        j = ja - 1;
        g += jb - ja;
    }
    // advance past plane j of the current run
    __device__ void next() {
        if (++j > jb) {
            if (g >= g1) done = true;
            else start();
        }
    }
};

__global__ void __launch_bounds__(kMBlock, 1) k_reggrad4m(
    const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_xp,
    const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_w2,
    const float* __restrict__ sA, float* __restrict__ s, RegCfg c, MarchCfg mc, int yoff,
    double* part) {
    extern __shared__ __align__(1024) float tsm[];  // [kMR][4][mc.plane]
    __shared__ __align__(8) unsigned long long mbar_s[kMR];
    __shared__ double red[32];
    double ts = 0.0, t1 = 0.0, t2 = 0.0;
    if (blockIdx.x < kMarch) {
        const bool w1on = c.use_w1, m2 = c.mode2 == 1, m3 = c.mode2 == 2;
        const int ntz = mc.ntz, P = mc.plane, ZB = mc.zbox;
        const long total = (long)ntz * mc.ntx * c.ny;
        const long g0 = total * blockIdx.x / kMarch, g1 = total * (blockIdx.x + 1) / kMarch;
        if (threadIdx.x == 0) {
            for (int st = 0; st < kMR; ++st)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(&mbar_s[st]))
                             : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        const unsigned bytes = (unsigned)(ZB * (mc.mx + 2) * sizeof(float)) *  // the boxes, not the padded planes
                               ((w1on || m2 || m3 ? 1u : 0u) + (m2 || m3 ? 1u : 0u) +
                                (w1on ? 1u : 0u) + (m2 ? 1u : 0u));
        MarchRuns ld;  // thread 0: the planes still to load
        int issued = 0;
        ld.init(g0, g1, c.ny);
        auto issue = [&]() {
            const int tz = ld.col % ntz, txi = ld.col / ntz;
            float* const T = tsm + (size_t)(issued % kMR) * 4 * P;
            const unsigned mbar = (unsigned)__cvta_generic_to_shared(&mbar_s[issued % kMR]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                         : "memory");
            const int z = tz * mc.zt - mc.zo, x = txi * mc.mx - 1, y = ld.j + yoff;
            if (w1on || m2 || m3) tma_load3(T, &tm_x, z, x, y, mbar);
            if (m2 || m3) tma_load3(T + P, &tm_xp, z, x, y, mbar);
            if (w1on) tma_load3(T + 2 * P, &tm_w1, z, x, y, mbar);
            if (m2) tma_load3(T + 3 * P, &tm_w2, z, x, y, mbar);
            ++issued;
            ld.next();
        };
        auto wait = [&](int n) {
            asm volatile(
                "{\n\t.reg .pred done;\n"
                "MARCHWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
                "@!done bra MARCHWAIT_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(&mbar_s[n % kMR])),
                "r"((unsigned)((n / kMR) & 1))
                : "memory");
        };
        if (threadIdx.x == 0)
            while (issued < kMR && !ld.done) issue();
        const int qz = threadIdx.x % mc.nzq, tx = threadIdx.x / mc.nzq;
        const bool mine = tx < mc.mx;
        const int o = (tx + 1) * ZB + mc.zo + 4 * qz;
        const size_t si = c.nz;
        MarchRuns cr;  // all threads: the runs being computed
        cr.init(g0, g1, c.ny);
        int n = 0;  // load index of the current run's first plane (ja - 1)
        while (!cr.done) {
            const int col = cr.col, ja = cr.j + 1, jb = cr.jb;
            const int tz = col % ntz, txi = col / ntz;
            const int k = tz * mc.zt + 4 * qz, i = txi * mc.mx + tx;
            const bool ok = mine && k < c.nz && k < (tz + 1) * mc.zt && i < c.nx;
            const bool hasip = i + 1 < c.nx, hasim = i > 0;
            wait(n);
            wait(n + 1);
            for (int j = ja; j < jb; ++j) {
                const int nn = n + 2 + (j - ja);  // load index of plane j + 1
                wait(nn);
                if (ok) {
                    const float* const Tm = tsm + (size_t)((nn - 2) % kMR) * 4 * P;
                    const float* const Tc = tsm + (size_t)((nn - 1) % kMR) * 4 * P;
                    const float* const Tp = tsm + (size_t)(nn % kMR) * 4 * P;
                    const size_t v = (size_t)k + si * ((size_t)i + (size_t)c.nx * j);
                    const float4 a = __ldg(reinterpret_cast<const float4*>(sA + v));
                    float sv[4] = {a.x, a.y, a.z, a.w};
                    const int jg = j + c.j0;
                    const bool hasjp = jg + 1 < c.nyg, hasjm = jg > 0;
                    auto ld4s = [&](const float* T, int off) { return *reinterpret_cast<const float4*>(T + off); };
                    float g[4], gg[4];
                    if (w1on) {
                        const float* const T1 = Tc + 2 * P;
                        Q4 X, W;
                        X.c = ld4s(Tc, o);
                        X.km = Tc[o - 1];
                        X.kp = Tc[o + 4];
                        W.c = ld4s(T1, o);
                        W.km = T1[o - 1];
                        dtwd_m(X, ld4s(Tc, o + ZB), ld4s(Tc, o - ZB), ld4s(Tp, o), ld4s(Tm, o), W,
                               ld4s(T1, o - ZB), ld4s(Tm + 2 * P, o), k, hasip, hasim, hasjp, hasjm,
                               c.nz, g, gg);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            sv[q] -= c.alpha2 * g[q];
                            t1 += (double)gg[q];
                        }
                    }
                    if (m2) {
                        const float* const T2 = Tc + 3 * P;
                        auto d4 = [&](const float* T, int off) { return sub4(ld4s(T, off), ld4s(T + P, off)); };
                        Q4 D, W;
                        D.c = d4(Tc, o);
                        D.km = Tc[o - 1] - Tc[P + o - 1];
                        D.kp = Tc[o + 4] - Tc[P + o + 4];
                        W.c = ld4s(T2, o);
                        W.km = T2[o - 1];
                        dtwd_m(D, d4(Tc, o + ZB), d4(Tc, o - ZB), d4(Tp, o), d4(Tm, o), W,
                               ld4s(T2, o - ZB), ld4s(Tm + 3 * P, o), k, hasip, hasim, hasjp, hasjm,
                               c.nz, g, gg);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            sv[q] -= c.lambda2 * g[q];
                            t2 += (double)gg[q];
                        }
                    } else if (m3) {
                        const float4 xv = ld4s(Tc, o), pv = ld4s(Tc + P, o);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float dv = q4(xv, q) - q4(pv, q);
                            sv[q] -= c.lambda2 * dv;
                            t2 += (double)dv * (double)dv;
                        }
                    }
                    *reinterpret_cast<float4*>(s + v) = make_float4(sv[0], sv[1], sv[2], sv[3]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) ts += (double)sv[q] * (double)sv[q];
                }
                __syncthreads();  // plane j - 1's slot is free
                // planes up to (next needed) + kMR - 3 may be in flight
                const int next_needed = j + 1 < jb ? nn + 1 : nn + 3;
                if (threadIdx.x == 0)
                    while (issued < next_needed + kMR - 2 && !ld.done) issue();
            }
            n += jb - ja + 2;
            cr.j = cr.jb;  // the run is consumed
            cr.next();
        }
    }
    write_partials(part, 0, ts, red);
    write_partials(part, 1, t1, red);
    write_partials(part, 2, t2, red);
}

#ifndef KCT_TMA_MINB2
#define KCT_TMA_MINB2 4  // 3 -> 4 CTAs per SM: k_weights4t 70 -> 68 us, k_normq4t unchanged (58 us)
#endif
// ---- k_weights4 / k_normq4 on TMA tiles ---------------------------------
// The same tiles and two-stage pipeline as k_reggrad4t for the forward-
// difference stencils: k_weights4t reads tiles of x and x_p (TV weights,
// smoothed-TV sums), k_normq4t tiles of p (||W1 D p||^2, ||W2 D p||^2) with
// W1 / W2 read directly (each voxel once).  Per voxel the arithmetic of
// k_weights4 / k_normq4.
template <class Body>
__device__ __forceinline__ void tma_tiles(const CUtensorMap* tmA, const CUtensorMap* tmB, int ntile_maps,
                                          const RegCfg& c, int yoff, float* tsm,
                                          unsigned long long* mbar_s, Body&& body) {
    const int ntz = (c.nz + kTZ - 1) / kTZ, ntx = (c.nx + kTX - 1) / kTX, nty = (c.ny + kTY - 1) / kTY;
    const int ntiles = ntz * ntx * nty;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&mbar_s[st]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned bytes = (unsigned)(kTile * sizeof(float)) * (unsigned)ntile_maps;
    auto issue = [&](int tile, int n) {
        const int tz = tile % ntz, rest = tile / ntz, txi = rest % ntx, tyi = rest / ntx;
        float* const T = tsm + (size_t)(n % kStages) * 2 * kTile;
        const unsigned mbar = (unsigned)__cvta_generic_to_shared(&mbar_s[n % kStages]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                     : "memory");
        tma_load3(T, tmA, tz * kTZ - 4, txi * kTX - 1, tyi * kTY - 1 + yoff, mbar);
        if (ntile_maps > 1) tma_load3(T + kTile, tmB, tz * kTZ - 4, txi * kTX - 1, tyi * kTY - 1 + yoff, mbar);
    };
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    int n = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
        if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, n + 1);
        asm volatile(
            "{\n\t.reg .pred done;\n"
            "TMAWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
            "@!done bra TMAWAIT_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(&mbar_s[n % kStages])),
            "r"((unsigned)((n / kStages) & 1))
            : "memory");
        const int tz = tile % ntz, rest = tile / ntz, txi = rest % ntx, tyi = rest / ntx;
        const float* const T = tsm + (size_t)(n % kStages) * 2 * kTile;
        // thread -> z quad x column x row (one quad per thread and tile)
        const int qz = threadIdx.x & 15, col = threadIdx.x >> 4;
        const int tx = col & 7, ty = col >> 3;
        const int k = tz * kTZ + 4 * qz, i = txi * kTX + tx, j = tyi * kTY + ty;
        const int o = ((ty + 1) * kBX + (tx + 1)) * kBZ + 4 + 4 * qz;
        body(T, T + kTile, o, k, i, j, k < c.nz && i < c.nx && j < c.ny);
        __syncthreads();
    }
}
static_assert(kTY * kTX * (kTZ / 4) == kBlock, "one quad per thread and tile");

__global__ void __launch_bounds__(kBlock, KCT_TMA_MINB2) k_weights4t(const __grid_constant__ CUtensorMap tm_x,
                                                         const __grid_constant__ CUtensorMap tm_xp,
                                                         float* __restrict__ w1, float* __restrict__ w2,
                                                         RegCfg c, int yoff, int write_w, double* part) {
    extern __shared__ __align__(1024) float tsm[];  // [kStages][2][kTile]
    __shared__ __align__(8) unsigned long long mbar_s[kStages];
    __shared__ double red[32];
    const size_t si = c.nz;
    double t1 = 0.0, t2 = 0.0;
    const bool m2 = c.mode2 == 1, m3 = c.mode2 == 2;
    tma_tiles(&tm_x, &tm_xp, m2 || m3 ? 2 : 1, c, yoff, tsm, mbar_s,
              [&](const float* TX, const float* TP, int o, int k, int i, int j, bool ok) {
        const int jg = j + c.j0;
        const bool hasip = i + 1 < c.nx, hasjp = jg + 1 < c.nyg;
        const float4 xc = *reinterpret_cast<const float4*>(TX + o);
        const float4 xip = *reinterpret_cast<const float4*>(TX + o + kBZ);
        const float4 xjp = *reinterpret_cast<const float4*>(TX + o + kBZ * kBX);
        const float xf[5] = {xc.x, xc.y, xc.z, xc.w, TX[o + 4]};
        float o1[4], o2[4];
        float4 pc = make_float4(0.f, 0.f, 0.f, 0.f), pip = pc, pjp = pc;
        float pk4 = 0.f;
        if (m2 || m3) {
            pc = *reinterpret_cast<const float4*>(TP + o);
            pip = *reinterpret_cast<const float4*>(TP + o + kBZ);
            pjp = *reinterpret_cast<const float4*>(TP + o + kBZ * kBX);
            pk4 = TP[o + 4];
        }
        const float pf[5] = {pc.x, pc.y, pc.z, pc.w, pk4};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float xv = xf[q];
            if (c.use_w1) {
                const float gx = hasip ? q4(xip, q) - xv : 0.f;
                const float gy = hasjp ? q4(xjp, q) - xv : 0.f;
                const float gz = k + q + 1 < c.nz ? xf[q + 1] - xv : 0.f;
                const float r = sqrtf(gx * gx + gy * gy + gz * gz + c.tau2);
                if (ok) t1 += (double)r;
                o1[q] = rsqrtf(r);
            }
            if (m2) {
                const float dv = xv - pf[q];
                const float gx = hasip ? (q4(xip, q) - q4(pip, q)) - dv : 0.f;
                const float gy = hasjp ? (q4(xjp, q) - q4(pjp, q)) - dv : 0.f;
                const float gz = k + q + 1 < c.nz ? (xf[q + 1] - pf[q + 1]) - dv : 0.f;
                const float r = sqrtf(gx * gx + gy * gy + gz * gz + c.tau2);
                if (ok) t2 += (double)r;
                o2[q] = rsqrtf(r);
            } else if (m3) {
                const double d = (double)xv - (double)pf[q];
                if (ok) t2 += d * d;
            }
        }
        if (ok && write_w) {
            const size_t v = (size_t)k + si * ((size_t)i + (size_t)c.nx * j);
            if (c.use_w1) *reinterpret_cast<float4*>(w1 + v) = make_float4(o1[0], o1[1], o1[2], o1[3]);
            if (m2) *reinterpret_cast<float4*>(w2 + v) = make_float4(o2[0], o2[1], o2[2], o2[3]);
        }
    });
    write_partials(part, 1, t1, red);
    write_partials(part, 2, t2, red);
}

__global__ void __launch_bounds__(kBlock, KCT_TMA_MINB2) k_normq4t(const float* __restrict__ q, size_t n,
                                                       const __grid_constant__ CUtensorMap tm_p,
                                                       const float* __restrict__ pv0,
                                                       const float* __restrict__ w1,
                                                       const float* __restrict__ w2, RegCfg c,
                                                       int yoff, const Ctl* ctl, double* part) {
    if (ctl->stop) return;
    extern __shared__ __align__(1024) float tsm[];
    __shared__ __align__(8) unsigned long long mbar_s[kStages];
    __shared__ double red[32];
    double tq = 0.0, t1 = 0.0, t2 = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    // ||q||^2 with float4 loads (four values per thread and step, k order)
    {
        const size_t n4 = n / 4;
        const float4* q4p = reinterpret_cast<const float4*>(q);
        for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n4; v += stride) {
            const float4 a = __ldg(q4p + v);
            tq += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
        }
        for (size_t v = 4 * n4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n; v += stride) {
            const double qv = q[v];
            tq += qv * qv;
        }
    }
    const size_t si = c.nz;
    tma_tiles(&tm_p, &tm_p, 1, c, yoff, tsm, mbar_s,
              [&](const float* TPn, const float*, int o, int k, int i, int j, bool ok) {
        const int jg = j + c.j0;
        const bool hasip = i + 1 < c.nx, hasjp = jg + 1 < c.nyg;
        const float4 pc = *reinterpret_cast<const float4*>(TPn + o);
        const float4 pip = *reinterpret_cast<const float4*>(TPn + o + kBZ);
        const float4 pjp = *reinterpret_cast<const float4*>(TPn + o + kBZ * kBX);
        const float pf[5] = {pc.x, pc.y, pc.z, pc.w, TPn[o + 4]};
        const size_t v = ok ? (size_t)k + si * ((size_t)i + (size_t)c.nx * j) : 0;
        const float4 a1 = (ok && c.use_w1) ? __ldg(reinterpret_cast<const float4*>(w1 + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 a2 = (ok && c.mode2 == 1) ? __ldg(reinterpret_cast<const float4*>(w2 + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const float pvv = pf[qq];
            if (c.mode2 == 2 && ok) t2 += (double)pvv * (double)pvv;
            if (c.use_w1 || c.mode2 == 1) {
                const float gx = hasip ? q4(pip, qq) - pvv : 0.f;
                const float gy = hasjp ? q4(pjp, qq) - pvv : 0.f;
                const float gz = k + qq + 1 < c.nz ? pf[qq + 1] - pvv : 0.f;
                const float g2 = gx * gx + gy * gy + gz * gz;
                if (c.use_w1 && ok) { const float w = q4(a1, qq); t1 += (double)(w * w * g2); }
                if (c.mode2 == 1 && ok) { const float w = q4(a2, qq); t2 += (double)(w * w * g2); }
            }
        }
    });
    (void)pv0;
    write_partials(part, 0, tq, red);
    write_partials(part, 1, t1, red);
    write_partials(part, 2, t2, red);
}

__global__ void __launch_bounds__(kBlock) k_normq4(const float* __restrict__ q, size_t n,
                                                   const float* __restrict__ p,
                                                   const float* __restrict__ w1,
                                                   const float* __restrict__ w2, RegCfg c,
                                                   const Ctl* ctl, double* part) {
    if (ctl->stop) return;
    __shared__ double sm[32];
    const int lane = threadIdx.x & 31;
    double tq = 0.0, t1 = 0.0, t2 = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        const double qv = q[v];
        tq += qv * qv;
    }
    if (c.use_w1 || c.mode2) {
        const size_t m4 = (size_t)c.nx * c.ny * c.nz / 4;
        for (size_t base = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); base < m4;
             base += stride) {
            bool ok;
            size_t v;
            int k, i, j;
            decode4(base, lane, m4, c, ok, v, k, i, j);
            Nb4 Pn;
            load_nb<false, false>(p, v, k, i, j, c, ok, lane, Pn);
            const float4 a1 = (ok && c.use_w1) ? ld4(w1, v) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 a2 = (ok && c.mode2 == 1) ? ld4(w2, v) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const float pv = Pn.f[qq + 1];
                if (c.mode2 == 2 && ok) t2 += (double)pv * (double)pv;
                if (c.use_w1 || c.mode2 == 1) {
                    const float gx = i + 1 < c.nx ? q4(Pn.ip, qq) - pv : 0.f;
                    const float gy = j + c.j0 + 1 < c.nyg ? q4(Pn.jp, qq) - pv : 0.f;
                    const float gz = k + qq + 1 < c.nz ? Pn.f[qq + 2] - pv : 0.f;
                    const float g2 = gx * gx + gy * gy + gz * gz;
                    if (c.use_w1 && ok) { const float w = q4(a1, qq); t1 += (double)(w * w * g2); }
                    if (c.mode2 == 1 && ok) { const float w = q4(a2, qq); t2 += (double)(w * w * g2); }
                }
            }
        }
    }
    write_partials(part, 0, tq, sm);
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// ---- slot0 = ||q||^2 (N); slot1 = ||W1 D p||^2, slot2 = ||W2 D p||^2 (M) ---
__global__ void __launch_bounds__(kBlock) k_normq(const float* __restrict__ q, size_t n,
                                                  const float* __restrict__ p,
                                                  const float* __restrict__ w1,
                                                  const float* __restrict__ w2, RegCfg c,
                                                  const Ctl* ctl, double* part) {
    if (ctl->stop) return;
    __shared__ double sm[32];
    double tq = 0.0, t1 = 0.0, t2 = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        const double qv = q[v];
        tq += qv * qv;
    }
    if (c.use_w1 || c.mode2) {
        const size_t m = (size_t)c.nx * c.ny * c.nz, si = c.nz, sj = (size_t)c.nz * c.nx;
        for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < m; v += stride) {
            int k, i, j;
            decode(v, c, k, i, j);
            const float pv = p[v];
            if (c.mode2 == 2) t2 += (double)pv * (double)pv;
            if (c.use_w1 || c.mode2 == 1) {
                float gx, gy, gz;
                fdiff(p, v, k, i, j, c, si, sj, pv, gx, gy, gz);
                const float g2 = gx * gx + gy * gy + gz * gz;
                if (c.use_w1) { const float w = w1[v]; t1 += (double)(w * w * g2); }
                if (c.mode2 == 1) { const float w = w2[v]; t2 += (double)(w * w * g2); }
            }
        }
    }
    write_partials(part, 0, tq, sm);
    write_partials(part, 1, t1, sm);
    write_partials(part, 2, t2, sm);
}

// ---- x += a p ; r0 -= a q ; slot4 = ||r0||^2, slot5 = ||x - gt||^2 ---------
__device__ __forceinline__ bool aligned16(const void* a, const void* b, const void* c = nullptr) {
    return ((reinterpret_cast<size_t>(a) | reinterpret_cast<size_t>(b) | reinterpret_cast<size_t>(c)) & 15) == 0;
}

__global__ void __launch_bounds__(kBlock) k_update_xr(float* __restrict__ x,
                                                      const float* __restrict__ p, size_t m,
                                                      float* __restrict__ r,
                                                      const float* __restrict__ q, size_t n,
                                                      const float* __restrict__ gt,
                                                      const Ctl* ctl, double* part) {
    if (ctl->stop) return;
    __shared__ double sm[32];
    const float a = (float)ctl->a;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    double tr = 0.0, te = 0.0;
    // four values per thread and step when the buffers allow 16-byte accesses
    const size_t m4 = aligned16(x, p, gt) ? m / 4 : 0, n4 = aligned16(r, q) ? n / 4 : 0;
    for (size_t v = t0; v < m4; v += stride) {
        const float4 pv = __ldg(reinterpret_cast<const float4*>(p) + v);
        float4 xv = reinterpret_cast<float4*>(x)[v];
        xv.x = fmaf(a, pv.x, xv.x);
        xv.y = fmaf(a, pv.y, xv.y);
        xv.z = fmaf(a, pv.z, xv.z);
        xv.w = fmaf(a, pv.w, xv.w);
        reinterpret_cast<float4*>(x)[v] = xv;
        if (gt) {
            const float4 g = __ldg(reinterpret_cast<const float4*>(gt) + v);
            const double d0 = (double)xv.x - (double)g.x, d1 = (double)xv.y - (double)g.y,
                         d2 = (double)xv.z - (double)g.z, d3 = (double)xv.w - (double)g.w;
            te += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
        }
    }
    for (size_t v = 4 * m4 + t0; v < m; v += stride) {
        const float xv = fmaf(a, p[v], x[v]);
        x[v] = xv;
        if (gt) { const double d = (double)xv - (double)gt[v]; te += d * d; }
    }
    for (size_t v = t0; v < n4; v += stride) {
        const float4 qv = __ldg(reinterpret_cast<const float4*>(q) + v);
        float4 rv = reinterpret_cast<float4*>(r)[v];
        rv.x = fmaf(-a, qv.x, rv.x);
        rv.y = fmaf(-a, qv.y, rv.y);
        rv.z = fmaf(-a, qv.z, rv.z);
        rv.w = fmaf(-a, qv.w, rv.w);
        reinterpret_cast<float4*>(r)[v] = rv;
        tr += (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
    }
    for (size_t v = 4 * n4 + t0; v < n; v += stride) {
        const float rv = fmaf(-a, q[v], r[v]);
        r[v] = rv;
        tr += (double)rv * (double)rv;
    }
    write_partials(part, 4, tr, sm);
    write_partials(part, 5, te, sm);
}
__global__ void __launch_bounds__(kBlock) k_update_p(float* __restrict__ p,
                                                     const float* __restrict__ s, size_t m,
                                                     const Ctl* ctl, int init) {
    if (ctl->stop) return;
    const float beta = (float)ctl->beta;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t m4 = aligned16(p, s) ? m / 4 : 0;
    for (size_t v = t0; v < m4; v += stride) {
        const float4 sv = __ldg(reinterpret_cast<const float4*>(s) + v);
        float4 pv = sv;
        if (!init) {
            pv = reinterpret_cast<float4*>(p)[v];
            pv.x = fmaf(beta, pv.x, sv.x);
            pv.y = fmaf(beta, pv.y, sv.y);
            pv.z = fmaf(beta, pv.z, sv.z);
            pv.w = fmaf(beta, pv.w, sv.w);
        }
        reinterpret_cast<float4*>(p)[v] = pv;
    }
    for (size_t v = 4 * m4 + t0; v < m; v += stride) p[v] = init ? s[v] : fmaf(beta, p[v], s[v]);
}

// ---- misc reductions -------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_stats(const float* __restrict__ f, size_t n,
                                                  double* part) {
    // slot0 = sum f^2, slot3 = count(f != 0), slot6 = min, slot7 = max
    __shared__ double sm[32];
    double t = 0.0, nz = 0.0;
    float lo = __builtin_huge_valf(), hi = -__builtin_huge_valf();
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const float fv = f[v];
        t += (double)fv * (double)fv;
        nz += fv != 0.f ? 1.0 : 0.0;
        lo = fminf(lo, fv);
        hi = fmaxf(hi, fv);
    }
    write_partials(part, 0, t, sm);
    write_partials(part, 3, nz, sm);
    // min / max: reuse the block reduction tree on warp-level min/max
    __shared__ float smin[32], smax[32];
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_down_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_down_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = lo; smax[threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fminf(lo, smin[w]); hi = fmaxf(hi, smax[w]); }
        part[6 * kGrid + blockIdx.x] = lo;
        part[7 * kGrid + blockIdx.x] = hi;
    }
}


// One-block scalar step: reduces the partials of the preceding kernel(s) in a
// fixed order and runs the CGLS scalar recurrence (krylov.hpp:68-125).
__global__ void __launch_bounds__(kBlock) k_scalar(Ctl* ctl, const double* part, int mode,
                                                   double tol, double* res_hist, double* err_hist,
                                                   double* obj_out, int obj_kind) {
    // the slots a mode needs, one warp per slot, all at once (fixed order:
    // lane l adds partials l, l + 32, ..., then the shuffle tree)
    __shared__ double ss[8];
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const bool m12 = mode == S_TV || mode == S_DELTA || mode == S_GAMMA;
        const bool need = warp == 0 || ((warp == 1 || warp == 2) && m12) ||
                          (warp == 3 && mode == S_REF) || ((warp == 4 || warp == 5) && mode == S_GAMMA);
        if (warp < 6) {
            double t = 0.0;
            if (need)
                for (int b = lane; b < kGrid; b += 32) t += part[warp * kGrid + b];
            t = warp_sum(t);
            if (lane == 0) ss[warp] = t;
        }
        __syncthreads();
    }
    const double s0 = ss[0], s1 = ss[1], s2 = ss[2], s3 = ss[3], s4 = ss[4], s5 = ss[5];
    if (threadIdx.x != 0) return;
    Ctl& c = *ctl;
    switch (mode) {
    case S_DATA: c.data = s0; break;
    case S_TV: c.tv1 = s1; c.tv2 = s2; break;
    case S_GT2: c.gt2 = s0; break;
    case S_REF:
        c.ref2 = s0;
        break;
    case S_INIT: {
        c.stop = c.converged = c.breakdown = c.error = 0;
        c.iters = 0;
        c.gamma = s0;
        if (!isfinite(s0)) { c.error = 1; c.stop = 1; break; }
        if (s0 == 0.0) { c.converged = 1; c.stop = 1; break; }
        c.stop_tol = 0.0;
        if (tol > 0.0) {
            const double ref2 = c.x_nonzero ? c.ref2 : s0;
            c.stop_tol = tol * sqrt(ref2);
            if (sqrt(s0) <= c.stop_tol) { c.converged = 1; c.stop = 1; }
        }
        break;
    }
    case S_DELTA: {
        if (c.stop) break;
        const double delta = s0 + c.alpha2 * s1 + c.lambda2 * s2;
        if (!isfinite(delta)) { c.error = 2; c.stop = 1; break; }
        if (delta == 0.0) { c.breakdown = 1; c.stop = 1; break; }
        c.a = c.gamma / delta;
        break;
    }
    case S_GAMMA: {
        if (c.stop) break;
        const double g = s0;
        if (!isfinite(g)) { c.error = 2; c.stop = 1; break; }
        c.r2 = s4;
        const double res2 = s4 + c.alpha2 * s1 + c.lambda2 * s2;
        if (res_hist) res_hist[c.iters] = sqrt(res2);
        if (err_hist) err_hist[c.iters] = c.gt2 > 0.0 ? sqrt(s5 / c.gt2) : sqrt(s5);
        c.iters += 1;
        if (sqrt(g) <= c.stop_tol) { c.converged = 1; c.stop = 1; break; }
        c.beta = g / c.gamma;
        c.gamma = g;
        break;
    }
    case S_OBJ: {
        // recon.hpp:93-120; obj_kind: 0 tv, 1 piple, 2 piccs; alpha2/lambda2 as doubles
        double obj = c.data;
        if (c.alpha2 != 0.0) obj += 2.0 * c.alpha2 * c.tv1;
        if (obj_kind == KCT_KIND_PIPLE && c.lambda2 != 0.0) obj += c.lambda2 * c.tv2;
        if (obj_kind == KCT_KIND_PICCS && c.lambda2 != 0.0) obj += 2.0 * c.lambda2 * c.tv2;
        *obj_out = obj;
        break;
    }
    }
}

__global__ void k_minmax_final(const double* part, double* out) {
    __shared__ double slo[kBlock], shi[kBlock];
    double lo = INFINITY, hi = -INFINITY;
    for (int b = threadIdx.x; b < kGrid; b += blockDim.x) {
        lo = fmin(lo, part[6 * kGrid + b]);
        hi = fmax(hi, part[7 * kGrid + b]);
    }
    slo[threadIdx.x] = lo;
    shi[threadIdx.x] = hi;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < (int)blockDim.x; ++t) { lo = fmin(lo, slo[t]); hi = fmax(hi, shi[t]); }
        out[0] = lo;
        out[1] = hi;
    }
}

// ---- workspace -----------------------------------------------------------------
struct Workspace {
    size_t m = 0, n = 0;
    size_t halo = 0;  // y-slab mode: floats of one y plane kept on each side of volume vectors
    float *b = nullptr, *r = nullptr, *q = nullptr;
    float *x = nullptr, *p = nullptr, *s = nullptr, *prior = nullptr, *w1 = nullptr,
          *w2 = nullptr, *gt = nullptr;
    float* atr = nullptr;  // A^T r of the current residual (before the regulariser terms)
    double* part = nullptr;
    Ctl* ctl = nullptr;
    double* hist = nullptr;  // [2][cap]: residual, error
    double* obj = nullptr;   // [cap_obj]
    double* scal = nullptr;  // misc scalars
    double* gath = nullptr;  // y-slab mode: [2 * world] gather-by-sum buffer
    double* red = nullptr;   // multi-process: packed fp64 slots of one all-reduce
    size_t cap = 0, cap_obj = 0;
    float* stack = nullptr;  // kct_cgls_stack: r | q | weights of the caller's stack
    size_t stack_cap = 0;
    std::vector<void*> allocs;
    // per-iteration hook: reference-layout device copy of x, pinned host copy,
    // side stream, events (x copied / host copy done)
    float* hook_dev = nullptr;
    float* hook_host = nullptr;
    int* hook_stop = nullptr;      // pinned copy of the CGLS stop flag at the copy
    int* hook_stop_dev = nullptr;  // its snapshot on the solver stream
    cudaStream_t hook_stream = nullptr;
    cudaEvent_t hook_ev_x = nullptr, hook_ev_done = nullptr;
    // wall_times: one event at the solve start + one per inner iteration
    std::vector<cudaEvent_t> wall_ev;

    ~Workspace() {
        if (hook_stream) cudaStreamSynchronize(hook_stream);
        for (void* ptr : allocs) cudaFree(ptr);
        for (void* ptr : {(void*)hist, (void*)obj, (void*)stack}) cudaFree(ptr);
        if (hook_host) cudaFreeHost(hook_host);
        if (hook_stop) cudaFreeHost(hook_stop);
        if (hook_stream) cudaStreamDestroy(hook_stream);
        for (cudaEvent_t e : {hook_ev_x, hook_ev_done})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : wall_ev) cudaEventDestroy(e);
    }
};

template <class T>
void ensure(Workspace& w, T*& ptr, size_t n) {
    if (!ptr) {
        KCT_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
        w.allocs.push_back(ptr);
    }
}

// volume vectors: `halo` floats (one y plane) of zeros before and after
void ensure_vol(Workspace& w, float*& ptr) {
    if (!ptr) {
        float* base = nullptr;
        const size_t tot = w.m + 2 * w.halo;
        KCT_CUDA(cudaMalloc(&base, tot * sizeof(float)));
        KCT_CUDA(cudaMemset(base, 0, tot * sizeof(float)));
        w.allocs.push_back(base);
        ptr = base + w.halo;
    }
}

Workspace& workspace(Projector& P, size_t hist_cap, size_t obj_cap) {
    auto ws = std::static_pointer_cast<Workspace>(P.workspace);
    if (!ws) {
        ws = std::make_shared<Workspace>();
        ws->m = P.domain_size();
        ws->n = P.range_size();
        ws->halo = P.slab_mode() ? (size_t)P.grid().nx * P.grid().nz : 0;
        P.workspace = ws;
    }
    Workspace& w = *ws;
    const size_t n = w.n;
    ensure(w, w.b, n); ensure(w, w.r, n); ensure(w, w.q, n);
    ensure_vol(w, w.x); ensure_vol(w, w.p); ensure_vol(w, w.s); ensure_vol(w, w.atr);
    ensure(w, w.part, (size_t)kSlots * kGrid);
    ensure(w, w.ctl, 1);
    ensure(w, w.scal, 8);
    if (P.slab_mode()) ensure(w, w.gath, (size_t)2 * P.slab_world);
    if (P.comm_fn) ensure(w, w.red, (size_t)kSlots);
    if (P.hook_fn && !w.hook_dev) {
        ensure(w, w.hook_dev, w.m);
        ensure(w, w.hook_stop_dev, 1);
        KCT_CUDA(cudaMallocHost(&w.hook_host, w.m * sizeof(float)));
        KCT_CUDA(cudaMallocHost(&w.hook_stop, sizeof(int)));
        KCT_CUDA(cudaStreamCreateWithFlags(&w.hook_stream, cudaStreamNonBlocking));
        KCT_CUDA(cudaEventCreateWithFlags(&w.hook_ev_x, cudaEventDisableTiming));
        KCT_CUDA(cudaEventCreateWithFlags(&w.hook_ev_done, cudaEventDisableTiming));
    }
    while (w.wall_ev.size() < hist_cap + 1) {
        cudaEvent_t e;
        KCT_CUDA(cudaEventCreate(&e));
        w.wall_ev.push_back(e);
    }
    if (w.cap < hist_cap) {
        cudaFree(w.hist);
        w.hist = nullptr;
        KCT_CUDA(cudaMalloc(&w.hist, 2 * hist_cap * sizeof(double)));
        w.cap = hist_cap;
    }
    if (w.cap_obj < obj_cap) {
        cudaFree(w.obj);
        w.obj = nullptr;
        KCT_CUDA(cudaMalloc(&w.obj, obj_cap * sizeof(double)));
        w.cap_obj = obj_cap;
    }
    return w;
}

// Copy an input (host/device, reference/native layout) into a native device buffer.
void load(Projector& P, float* dst, const float* src, size_t n, bool is_vol, int mem, int layout,
          cudaStream_t s) {
    if (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) {
        KCT_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
        return;
    }
    const float* nat = stage_in(P, src, n, is_vol, mem, layout, is_vol ? 0 : 1, 2, s);
    KCT_CUDA(cudaMemcpyAsync(dst, nat, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
}

void launch_scalar(Workspace& w, int mode, cudaStream_t s, double tol = 0.0,
                   double* res = nullptr, double* err = nullptr, double* obj = nullptr,
                   int kind = 0) {
    k_scalar<<<1, kBlock, 0, s>>>(w.ctl, w.part, mode, tol, res, err, obj, kind);
    KCT_LAUNCHED();
}

#define KCT_LAUNCH(kernel, ...)                                \
    do {                                                       \
        kernel<<<kGrid, kBlock, 0, stream>>>(__VA_ARGS__);     \
        KCT_LAUNCHED();                          \
    } while (0)


__global__ void k_set_nonzero(Ctl* ctl, const double* part) {
    __shared__ double sm[32];
    double t = 0.0;
    for (int b = threadIdx.x; b < kGrid; b += blockDim.x) t += part[3 * kGrid + b];
    t = block_sum(t, sm);
    if (threadIdx.x == 0) ctl->x_nonzero = t > 0.0 ? 1 : 0;
}

// Fold the block partials of each listed slot (fixed order) into red[idx],
// so one all-reduce of `count` doubles carries every slot of a phase across
// the ranks; k_unpack writes the sums back as the slots' only partials.
struct SlotList {
    int n;
    int slot[kSlots];
};

__global__ void k_fold(double* part, SlotList sl, double* red) {
    __shared__ double sm[32];
    for (int q = 0; q < sl.n; ++q) {
        double* row = part + sl.slot[q] * kGrid;
        double t = 0.0;
        for (int b = threadIdx.x; b < kGrid; b += blockDim.x) t += row[b];
        t = block_sum(t, sm);
        __syncthreads();
        if (threadIdx.x == 0) red[q] = t;
    }
}

__global__ void k_unpack(double* part, SlotList sl, const double* red) {
    for (int q = 0; q < sl.n; ++q) {
        double* row = part + sl.slot[q] * kGrid;
        for (int b = threadIdx.x; b < kGrid; b += blockDim.x) row[b] = b == 0 ? red[q] : 0.0;
    }
}

// Host trampoline of the per-iteration hook (cudaLaunchHostFunc on the side stream).
// The iteration number counts the calls actually made (the reference's
// global_iter, recon.hpp:223-228): an iteration of a stopped CGLS (breakdown,
// tolerance reached) changes nothing and, as in the reference, has no call.
struct HookCall {
    kct_iterate_hook fn;
    void* ctx;
    size_t* counter;
    const int* stopped;
    const float* x;
    size_t m;
};

void CUDART_CB hook_trampoline(void* arg) {
    const HookCall* c = static_cast<const HookCall*>(arg);
    if (*c->stopped) return;
    c->fn(c->ctx, ++*c->counter, c->x, c->m);
}

// cuTensorMapEncodeTiled (driver API), resolved at run time through the
// runtime's entry-point query (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 3D tensor map of a native-layout volume vector (z, x, y[+ halo planes]) with
// the k_reggrad4t box
bool volume_tmap(CUtensorMap& tm, const float* v, const RegCfg& rc, size_t halo, int bz = kBZ,
                 int bx = kBX, int by = kBY) {
    const EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const int hy = halo ? 1 : 0;
    const cuuint64_t dims[3] = {(cuuint64_t)rc.nz, (cuuint64_t)rc.nx, (cuuint64_t)(rc.ny + 2 * hy)};
    const cuuint64_t strides[2] = {(cuuint64_t)rc.nz * sizeof(float),
                                   (cuuint64_t)rc.nz * rc.nx * sizeof(float)};
    const cuuint32_t box[3] = {(cuuint32_t)bz, (cuuint32_t)bx, (cuuint32_t)by};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(v - halo), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Engine {
    Projector& P;
    Workspace& w;
    cudaStream_t stream;
    RegCfg rc{};
    int kind = KCT_KIND_TV;
    // w.r == b - A w.x and w.atr == A^T w.r (set by start / iterate; cleared
    // when x is replaced)
    bool r_current = false;

    // Multi-process modes (no-ops in a single process):
    //  * angle-sharded (kct_set_allreduce): rank-local rays; sum the partial
    //    A^T volumes and the projection-domain reductions;
    //  * y-slab-sharded (kct_set_slab): rank-local volume slab with halo
    //    planes; sum the partial forward projections and the volume-domain
    //    reductions, exchange halos after every update of a stencil operand.
    bool slab() const { return P.slab_mode(); }
    // the reference's control flow at every CGLS start (kct_set_option "solver_restart")
    bool restart = false;
    // per-iteration hook state (P.hook_fn): 1-based global iteration counter
    size_t hook_iter = 0;
    std::deque<HookCall>* hook_calls = nullptr;  // stable addresses for the host callbacks
    // wall_times: events recorded so far (index 0 = solve start)
    size_t n_wall = 0;
    // scalar all-reduces issued (evidence for the per-iteration collective count)
    size_t n_scalar_reduce = 0;

    void allreduce(void* buf, size_t count, int dtype, const char* what) {
        if (P.comm_fn(P.comm_ctx, buf, count, dtype, stream) != 0)
            throw CudaError(std::string("allreduce hook failed (") + what + ")");
    }
    // one all-reduce of all listed slots (fixed order)
    void reduce_slots(std::initializer_list<int> slots) {
        if (!P.comm_fn || slots.size() == 0) return;
        SlotList sl{};
        for (int slot : slots) sl.slot[sl.n++] = slot;
        k_fold<<<1, kBlock, 0, stream>>>(w.part, sl, w.red);
        KCT_LAUNCHED();
        allreduce(w.red, (size_t)sl.n, 1, "scalars");
        ++n_scalar_reduce;
        k_unpack<<<1, kBlock, 0, stream>>>(w.part, sl, w.red);
        KCT_LAUNCHED();
    }
    void proj_slots(std::initializer_list<int> slots) { if (!slab()) reduce_slots(slots); }
    void vol_slots(std::initializer_list<int> slots) { if (slab()) reduce_slots(slots); }
    void forward(const float* v, float* q) {
        P.forward(v, q, stream);
        if (slab()) allreduce(q, w.n, 0, "projections");
    }
    void adjoint(const float* y, float* v) {
        P.adjoint(y, v, stream);
        if (!slab() && P.comm_fn) allreduce(v, w.m, 0, "volume");
    }
    void halo(float* v) {
        if (!slab() || !v) return;
        const size_t pl = w.halo;
        const size_t ny = (size_t)P.grid().ny;
        if (P.halo_fn(P.halo_ctx, v, v + (ny - 1) * pl, v - pl, v + ny * pl, pl, stream) != 0)
            throw CudaError("halo exchange hook failed");
    }

    // weights (optional) and smoothed-TV / quadratic sums of the objective at w.x
    void weights(bool write) {
        if (!rc.use_w1 && !rc.mode2) {
            KCT_CUDA(cudaMemsetAsync(w.part + 1 * kGrid, 0, 2 * kGrid * sizeof(double), stream));
        } else {
            if (weights_tma(write)) {
            } else if (use4()) KCT_LAUNCH(k_weights4, w.x, w.prior, w.w1, w.w2, rc, write ? 1 : 0, w.part);
            else KCT_LAUNCH(k_weights, w.x, w.prior, w.w1, w.w2, rc, write ? 1 : 0, w.part);
            vol_slots({1, 2});
            if (write) {
                if (rc.use_w1) halo(w.w1);
                if (rc.mode2 == 1) halo(w.w2);
            }
        }
        launch_scalar(w, S_TV, stream);
    }

    // objective(x) (recon.hpp:93-120) into w.obj[idx]; the TV sums must be current
    void objective(bool x_is_zero, int idx) {
        if (x_is_zero) {
            KCT_LAUNCH(k_resid, w.b, nullptr, nullptr, w.n, w.part, 0);
        } else if (r_current && !restart) {
            KCT_LAUNCH(k_stats, w.r, w.n, w.part);  // ||r||^2, r = b - A x (CGLS recurrence)
        } else {
            forward(w.x, w.q);
            KCT_LAUNCH(k_resid, w.b, w.q, nullptr, w.n, w.part, 0);
        }
        proj_slots({0});
        launch_scalar(w, S_DATA, stream);
        launch_scalar(w, S_OBJ, stream, 0.0, nullptr, nullptr, w.obj + idx, kind);
    }

    // CGLS start (krylov.hpp:66-96) from w.x.  When obj_idx >= 0 the data term
    // ||b - A x||^2 of this residual also completes objective[obj_idx].
    void start(bool x_is_zero, double tol, int obj_idx) {
        if (tol > 0.0 && !x_is_zero) {
            // ||A~^T b~||^2, the tolerance reference of a warm start (krylov.hpp:81-88)
            KCT_LAUNCH(k_stats, w.x, w.m, w.part);
            vol_slots({3});
            k_set_nonzero<<<1, kBlock, 0, stream>>>(w.ctl, w.part);
            KCT_LAUNCHED();
            adjoint(w.b, w.p);
            reggrad(w.p, w.p, nullptr);
            launch_scalar(w, S_REF, stream);
        } else {
            KCT_CUDA(cudaMemsetAsync(&w.ctl->x_nonzero, 0, sizeof(int), stream));
        }
        // A warm start from the x the previous cycle's iterations ended on
        // reuses their data residual r = b - A x (the CGLS recurrence keeps it
        // up to rounding) and its A^T r: the stacked system changes between
        // cycles only in the regulariser blocks, whose residual parts are
        // evaluated from x anyway (section 4 of DESIGN.md) — one forward and one
        // adjoint projection less per cycle.
        const bool reuse = r_current && !x_is_zero && !restart;
        if (x_is_zero) {
            KCT_LAUNCH(k_resid, w.b, nullptr, w.r, w.n, w.part, 0);
        } else if (reuse) {
            KCT_LAUNCH(k_stats, w.r, w.n, w.part);
        } else {
            forward(w.x, w.q);
            KCT_LAUNCH(k_resid, w.b, w.q, w.r, w.n, w.part, 0);
        }
        proj_slots({0});
        if (obj_idx >= 0) {
            launch_scalar(w, S_DATA, stream);
            launch_scalar(w, S_OBJ, stream, 0.0, nullptr, nullptr, w.obj + obj_idx, kind);
        }
        if (!reuse) adjoint(w.r, w.atr);
        reggrad(w.atr, w.s, x_is_zero ? nullptr : w.x);
        launch_scalar(w, S_INIT, stream, tol);
        KCT_LAUNCH(k_update_p, w.p, w.s, w.m, w.ctl, 1);
        halo(w.p);
        r_current = true;
    }

    // float4 stencil kernels when the slab count allows (KCT_SCALAR_STENCILS=1: scalar)
    bool use4() const {
        const char* e = std::getenv("KCT_SCALAR_STENCILS");
        return rc.nz % 4 == 0 && !(e && e[0] == '1');
    }

    // out <- in - regulariser gradient (in == out allowed), norms into slots 0..2
    // (with_err: slot 5 of the preceding k_update_xr joins the same all-reduce)
    // k_reggrad4t: x present, nz a multiple of 4, the volume at least one
    // tile deep (KCT_TMA_STENCIL=0: the grid-stride kernel)
    bool reggrad_tma(const float* in, float* out, const float* xv) {
        const char* e = std::getenv("KCT_TMA_STENCIL");
        if ((e && e[0] == '0') || !use4() || !xv || rc.nz < kTZ || rc.nx < kTX || rc.ny < kTY)
            return false;
        CUtensorMap tx, tp, t1, t2;
        const float* xp = w.prior ? w.prior : xv;
        const float* w1 = w.w1 ? w.w1 : xv;
        const float* w2 = w.w2 ? w.w2 : xv;
        // KCT_TMA_MARCH=1: the y-marching ring (measured at c3: same time as the
        // tiles, 108.9 vs 107.3 us, with 412 instead of 446 MB of DRAM reads —
        // both kernels are issue-bound, not traffic-bound)
        const char* me = std::getenv("KCT_TMA_MARCH");
        const MarchCfg mc = march_cfg(rc);
        if (me && me[0] == '1' && volume_tmap(tx, xv, rc, w.halo, mc.zbox, mc.mx + 2, 1) &&
            volume_tmap(tp, xp, rc, w.halo, mc.zbox, mc.mx + 2, 1) &&
            volume_tmap(t1, w1, rc, w.halo, mc.zbox, mc.mx + 2, 1) &&
            volume_tmap(t2, w2, rc, w.halo, mc.zbox, mc.mx + 2, 1)) {
            const int smem = kMR * 4 * mc.plane * (int)sizeof(float);
            KCT_CUDA(cudaFuncSetAttribute(k_reggrad4m, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_reggrad4m<<<kGrid, kMBlock, smem, stream>>>(tx, tp, t1, t2, in, out, rc, mc, w.halo ? 1 : 0,
                                                         w.part);
            KCT_LAUNCHED();
            return true;
        }
        if (!volume_tmap(tx, xv, rc, w.halo) || !volume_tmap(tp, xp, rc, w.halo) ||
            !volume_tmap(t1, w1, rc, w.halo) || !volume_tmap(t2, w2, rc, w.halo))
            return false;
        const int smem = kStages * 4 * kTile * (int)sizeof(float);
        KCT_CUDA(cudaFuncSetAttribute(k_reggrad4t, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_reggrad4t<<<kGrid, kBlock, smem, stream>>>(tx, tp, t1, t2, in, out, rc, w.halo ? 1 : 0, w.part);
        KCT_LAUNCHED();
        return true;
    }

    bool tma_ok() const {
        const char* e = std::getenv("KCT_TMA_STENCIL");
        return !(e && e[0] == '0') && use4() && rc.nz >= kTZ && rc.nx >= kTX && rc.ny >= kTY &&
               encode_tiled();
    }
    bool weights_tma(bool write) {
        if (!tma_ok() || !w.x) return false;
        CUtensorMap tx, tp;
        if (!volume_tmap(tx, w.x, rc, w.halo) ||
            !volume_tmap(tp, w.prior ? w.prior : w.x, rc, w.halo))
            return false;
        const int smem = kStages * 2 * kTile * (int)sizeof(float);
        KCT_CUDA(cudaFuncSetAttribute(k_weights4t, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_weights4t<<<kGrid, kBlock, smem, stream>>>(tx, tp, w.w1, w.w2, rc, w.halo ? 1 : 0,
                                                    write ? 1 : 0, w.part);
        KCT_LAUNCHED();
        return true;
    }
    bool normq_tma() {
        if (!tma_ok() || !(rc.use_w1 || rc.mode2)) return false;
        CUtensorMap tp;
        if (!volume_tmap(tp, w.p, rc, w.halo)) return false;
        const int smem = kStages * 2 * kTile * (int)sizeof(float);
        KCT_CUDA(cudaFuncSetAttribute(k_normq4t, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_normq4t<<<kGrid, kBlock, smem, stream>>>(w.q, w.n, tp, w.p, w.w1, w.w2, rc, w.halo ? 1 : 0,
                                                  w.ctl, w.part);
        KCT_LAUNCHED();
        return true;
    }

    void reggrad(const float* in, float* out, const float* xv, bool with_err = false) {
        if (reggrad_tma(in, out, xv)) {
        } else if (use4()) KCT_LAUNCH(k_reggrad4, in, xv, w.prior, w.w1, w.w2, out, rc, w.part);
        else KCT_LAUNCH(k_reggrad, in, xv, w.prior, w.w1, w.w2, out, rc, w.part);
        if (with_err) vol_slots({0, 1, 2, 5});
        else vol_slots({0, 1, 2});
    }

    // One CGLS iteration (krylov.hpp:98-125).
    void iterate(double* res, double* err, bool with_gt) {
        forward(w.p, w.q);
        if (normq_tma()) {
        } else if (use4()) KCT_LAUNCH(k_normq4, w.q, w.n, w.p, w.w1, w.w2, rc, w.ctl, w.part);
        else KCT_LAUNCH(k_normq, w.q, w.n, w.p, w.w1, w.w2, rc, w.ctl, w.part);
        proj_slots({0});
        vol_slots({1, 2});
        launch_scalar(w, S_DELTA, stream);
        KCT_LAUNCH(k_update_xr, w.x, w.p, w.m, w.r, w.q, w.n, with_gt ? w.gt : nullptr, w.ctl,
                   w.part);
        proj_slots({4});
        halo(w.x);
        hook_copy();
        adjoint(w.r, w.atr);
        reggrad(w.atr, w.s, w.x, with_gt);  // + slot 5 (||x - gt||^2) in slab mode
        launch_scalar(w, S_GAMMA, stream, 0.0, res, err);
        KCT_LAUNCH(k_update_p, w.p, w.s, w.m, w.ctl, 0);
        halo(w.p);
        if (n_wall < w.wall_ev.size()) KCT_CUDA(cudaEventRecord(w.wall_ev[n_wall++], stream));
    }

    // solve start on the device timeline (wall_times reference point)
    void mark_start() {
        n_wall = 0;
        KCT_CUDA(cudaEventRecord(w.wall_ev[n_wall++], stream));
    }
    // seconds since the start event of the iterations recorded (synchronises)
    size_t wall_times(double* out) {
        if (n_wall < 2) return 0;
        KCT_CUDA(cudaEventSynchronize(w.wall_ev[n_wall - 1]));
        for (size_t i = 1; i < n_wall; ++i) {
            float ms = 0.f;
            KCT_CUDA(cudaEventElapsedTime(&ms, w.wall_ev[0], w.wall_ev[i]));
            if (out) out[i - 1] = 1e-3 * ms;
        }
        return n_wall - 1;
    }

    // IterateHook (krylov.hpp:116): x (reference layout) -> pinned host on the
    // side stream, then the caller's callback; the main stream only waits
    // for the previous iteration's copy before it overwrites the device copy.
    // A stopped solve (tolerance / breakdown) skips the call, as the
    // reference's loop exits before its hook.
    void hook_copy() {
        if (!P.hook_fn || !hook_calls) return;
        KCT_CUDA(cudaStreamWaitEvent(stream, w.hook_ev_done, 0));
        P.vol_from_native(w.x, w.hook_dev, stream);
        KCT_CUDA(cudaMemcpyAsync(w.hook_stop_dev, &w.ctl->stop, sizeof(int),
                                 cudaMemcpyDeviceToDevice, stream));
        KCT_CUDA(cudaEventRecord(w.hook_ev_x, stream));
        KCT_CUDA(cudaStreamWaitEvent(w.hook_stream, w.hook_ev_x, 0));
        KCT_CUDA(cudaMemcpyAsync(w.hook_host, w.hook_dev, w.m * sizeof(float),
                                 cudaMemcpyDeviceToHost, w.hook_stream));
        KCT_CUDA(cudaMemcpyAsync(w.hook_stop, w.hook_stop_dev, sizeof(int),
                                 cudaMemcpyDeviceToHost, w.hook_stream));
        KCT_CUDA(cudaEventRecord(w.hook_ev_done, w.hook_stream));
        hook_calls->push_back(HookCall{P.hook_fn, P.hook_ctx, &hook_iter, w.hook_stop, w.hook_host, w.m});
        KCT_CUDA(cudaLaunchHostFunc(w.hook_stream, hook_trampoline, &hook_calls->back()));
    }
    void hook_drain() {
        if (w.hook_stream) KCT_CUDA(cudaStreamSynchronize(w.hook_stream));
    }

    void ground_truth_norm() {
        KCT_LAUNCH(k_stats, w.gt, w.m, w.part);
        vol_slots({0});
        launch_scalar(w, S_GT2, stream);
    }
};

Ctl read_ctl(Workspace& w, cudaStream_t s) {
    Ctl c;
    KCT_CUDA(cudaMemcpyAsync(&c, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    KCT_CUDA(cudaStreamSynchronize(s));
    return c;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

void init_ctl(Workspace& w, double alpha2, double lambda2, cudaStream_t s) {
    Ctl c{};
    c.alpha2 = alpha2;
    c.lambda2 = lambda2;
    KCT_CUDA(cudaMemcpyAsync(w.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, s));
}

void throw_solver(const Ctl& c) {
    if (c.error == 1) throw SolverError("cgls: non-finite normal residual");
    if (c.error) throw SolverError("cgls: non-finite iterate");
}

// device (min, max) of a native buffer -> resolve_tau semantics (recon.hpp:60-66)
double device_tau(Projector& P, Workspace& w, const float* ref, size_t n, double tau,
                  cudaStream_t stream) {
    if (tau > 0.0) return tau;
    if (!ref || n == 0) return 1e-4;
    KCT_LAUNCH(k_stats, ref, n, w.part);
    k_minmax_final<<<1, kBlock, 0, stream>>>(w.part, w.scal);
    KCT_LAUNCHED();
    double mm[2];
    if (P.slab_mode()) {
        // global (min, max) over the slabs: gather by sum into [2 * world]
        const int W = P.slab_world;
        KCT_CUDA(cudaMemsetAsync(w.gath, 0, 2 * W * sizeof(double), stream));
        KCT_CUDA(cudaMemcpyAsync(w.gath + 2 * P.slab_rank, w.scal, 2 * sizeof(double),
                                 cudaMemcpyDeviceToDevice, stream));
        if (P.comm_fn(P.comm_ctx, w.gath, 2 * W, 1, stream) != 0)
            throw CudaError("allreduce hook failed (tau)");
        std::vector<double> g(2 * W);
        KCT_CUDA(cudaMemcpyAsync(g.data(), w.gath, 2 * W * sizeof(double), cudaMemcpyDeviceToHost,
                                 stream));
        KCT_CUDA(cudaStreamSynchronize(stream));
        mm[0] = g[0];
        mm[1] = g[1];
        for (int r = 1; r < W; ++r) {
            mm[0] = std::min(mm[0], g[2 * r]);
            mm[1] = std::max(mm[1], g[2 * r + 1]);
        }
    } else {
        KCT_CUDA(cudaMemcpyAsync(mm, w.scal, sizeof mm, cudaMemcpyDeviceToHost, stream));
        KCT_CUDA(cudaStreamSynchronize(stream));
    }
    const double range = mm[1] - mm[0];
    return range > 0.0 ? std::max(1e-8, 1e-4 * range) : 1e-4;
}

void check_slab(Projector& P) {
    if (P.slab_mode() && !P.comm_fn)
        throw ConfigError("y-slab mode needs the all-reduce hook (kct_set_allreduce)");
}

void set_grid(RegCfg& rc, Projector& P) {
    rc.nx = P.grid().nx;
    rc.ny = P.grid().ny;
    rc.nz = P.grid().nz;
    rc.j0 = P.slab_mode() ? P.slab_j0 : 0;
    rc.nyg = P.slab_mode() ? P.slab_nyg : rc.ny;
}

void copy_hist(double* dst, const double* src, size_t n, cudaStream_t s) {
    if (dst && n) KCT_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, s));
}

void reset_report(kct_report* rep) {
    if (!rep) return;
    rep->objective_count = rep->residual_count = rep->error_count = rep->outer_count = 0;
    rep->wall_count = 0;
    rep->solve_seconds = 0.0;
    rep->tau = 0.0;
    rep->converged = rep->breakdown = 0;
}

// Drains the hook stream when a solve ends (normally or by exception), so
// no host callback outlives the call list it points into.
struct HookScope {
    Engine& e;
    std::deque<HookCall> calls;
    explicit HookScope(Engine& en) : e(en) { e.hook_calls = &calls; }
    ~HookScope() {
        if (e.w.hook_stream) cudaStreamSynchronize(e.w.hook_stream);
        e.hook_calls = nullptr;
    }
};

void write_wall(Engine& e, kct_report* rep) {
    if (!rep) return;
    rep->wall_count = e.wall_times(rep->wall_times);
}

}  // namespace

double resolve_tau(double tau, const float* ref, size_t n) {
    if (tau > 0.0) return tau;
    if (!ref || n == 0) return 1e-4;
    float lo = ref[0], hi = ref[0];
    for (size_t i = 1; i < n; ++i) {
        lo = std::min(lo, ref[i]);
        hi = std::max(hi, ref[i]);
    }
    const double range = (double)hi - (double)lo;
    return range > 0.0 ? std::max(1e-8, 1e-4 * range) : 1e-4;
}

// cgls_recon / baseline_solve (recon.hpp:274-315)
void cgls_recon(Projector& P, const float* b, size_t iters, const float* x0, const float* gt,
                double tol, float* x_out, kct_report* rep, int mem, int layout,
                cudaStream_t stream) {
    if (!b || !x_out) throw ConfigError("cgls_recon: null buffer");
    if (iters < 1) throw ConfigError("reconstruction needs at least one iteration");
    reset_report(rep);
    check_slab(P);
    Workspace& w = workspace(P, iters, 1);
    if (gt) ensure_vol(w, w.gt);
    load(P, w.b, b, w.n, false, mem, layout, stream);
    if (x0) load(P, w.x, x0, w.m, true, mem, layout, stream);
    else KCT_CUDA(cudaMemsetAsync(w.x, 0, w.m * sizeof(float), stream));
    if (gt) load(P, w.gt, gt, w.m, true, mem, layout, stream);
    init_ctl(w, 0.0, 0.0, stream);
    Engine e{P, w, stream};
    e.restart = P.solver_restart;
    set_grid(e.rc, P);
    e.halo(w.x);
    if (gt) e.ground_truth_norm();
    KCT_CUDA(cudaStreamSynchronize(stream));

    HookScope hooks(e);
    const double t0 = now_s();
    e.mark_start();
    e.start(x0 == nullptr, tol, -1);
    for (size_t it = 0; it < iters; ++it) e.iterate(w.hist, w.hist + w.cap, gt != nullptr);
    const Ctl c = read_ctl(w, stream);
    const double secs = now_s() - t0;
    e.hook_drain();
    throw_solver(c);
    stage_out(P, w.x, x_out, w.m, true, mem, layout, 2, stream);
    if (rep) {
        const size_t n = (size_t)c.iters;
        copy_hist(rep->residual_history, w.hist, n, stream);
        if (gt) copy_hist(rep->error_history, w.hist + w.cap, n, stream);
        KCT_CUDA(cudaStreamSynchronize(stream));
        rep->residual_count = n;
        rep->error_count = gt ? n : 0;
        if (rep->objective_history && rep->residual_history)
            for (size_t i = 0; i < n; ++i)
                rep->objective_history[i] = rep->residual_history[i] * rep->residual_history[i];
        rep->objective_count = n;
        if (rep->outer_boundaries) rep->outer_boundaries[0] = n;
        if (rep->outer_seconds) rep->outer_seconds[0] = secs;
        rep->outer_count = 1;
        rep->solve_seconds = secs;
        rep->converged = c.converged;
        rep->breakdown = c.breakdown;
        write_wall(e, rep);
        if (rep->wall_count > n) rep->wall_count = n;
    }
    KCT_CUDA(cudaStreamSynchronize(stream));
}

// irn_setup + irn_solve (recon.hpp:141-247)
void irn_solve(Projector& P, int kind, const float* b, const float* prior, const float* x0,
               const float* gt, const kct_reg_params& p, float* x_out, kct_report* rep, int mem,
               int layout, cudaStream_t stream) {
    if (kind != KCT_KIND_TV && kind != KCT_KIND_PIPLE && kind != KCT_KIND_PICCS)
        throw ConfigError("unknown reconstruction kind");
    if (!b || !x_out) throw ConfigError("irn: null buffer");
    if (p.outer_iters < 1 || p.inner_iters < 1)
        throw ConfigError("reconstruction needs at least one outer and one inner iteration");
    if (p.alpha < 0.0) throw ConfigError("alpha must be non-negative");
    if (!std::isfinite(p.alpha) || !std::isfinite(p.lambda) || !std::isfinite(p.tau))
        throw ConfigError("regularisation parameters must be finite");
    if (kind != KCT_KIND_TV && !prior) throw ConfigError("prior volume required");
    const double alpha = p.alpha;
    const double lambda = p.lambda < 0.0 ? alpha : p.lambda;
    const size_t outer = p.outer_iters, inner = p.inner_iters;
    reset_report(rep);
    check_slab(P);

    Workspace& w = workspace(P, outer * inner, outer + 1);
    const bool use_prior = kind != KCT_KIND_TV;
    if (use_prior) ensure_vol(w, w.prior);
    if (alpha != 0.0) ensure_vol(w, w.w1);
    if (kind == KCT_KIND_PICCS && lambda != 0.0) ensure_vol(w, w.w2);
    if (gt) ensure_vol(w, w.gt);
    load(P, w.b, b, w.n, false, mem, layout, stream);
    if (use_prior) load(P, w.prior, prior, w.m, true, mem, layout, stream);
    if (x0) load(P, w.x, x0, w.m, true, mem, layout, stream);
    else KCT_CUDA(cudaMemsetAsync(w.x, 0, w.m * sizeof(float), stream));
    if (gt) load(P, w.gt, gt, w.m, true, mem, layout, stream);

    // tau from the initial image, else the prior when the prior term is active
    const float* tau_ref = x0 ? w.x : ((use_prior && lambda != 0.0) ? w.prior : nullptr);
    const double tau = device_tau(P, w, tau_ref, w.m, p.tau, stream);

    Engine e{P, w, stream};
    e.kind = kind;
    e.restart = P.solver_restart;
    set_grid(e.rc, P);
    e.halo(w.x);
    if (use_prior) e.halo(w.prior);
    e.rc.use_w1 = alpha != 0.0;
    e.rc.mode2 = lambda == 0.0 ? 0 : (kind == KCT_KIND_PICCS ? 1 : (kind == KCT_KIND_PIPLE ? 2 : 0));
    e.rc.alpha2 = (float)(alpha * alpha);
    e.rc.lambda2 = (float)(lambda * lambda);
    e.rc.tau2 = (float)(tau * tau);
    init_ctl(w, alpha * alpha, e.rc.mode2 ? lambda * lambda : 0.0, stream);
    if (gt) e.ground_truth_norm();
    KCT_CUDA(cudaStreamSynchronize(stream));

    std::vector<uint64_t> bounds;
    std::vector<double> secs;
    size_t n_res = 0;
    bool x_zero = x0 == nullptr;
    int converged = 0, breakdown = 0;
    HookScope hooks(e);
    const double t_start = now_s();
    e.mark_start();
    std::vector<size_t> wall_keep;  // event indices of the iterations that ran
    for (size_t cycle = 0; cycle < outer; ++cycle) {
        NvtxRange nvtx("irn outer cycle");  // (host enqueue; the device runs behind)
        const double t_cycle = now_s();
        e.weights(true);
        if (p.warm_start) {
            e.start(x_zero, p.inner_tolerance, (int)cycle);
        } else {
            if (cycle == 0) e.objective(x_zero, 0);
            KCT_CUDA(cudaMemsetAsync(w.x, 0, w.m * sizeof(float), stream));
            e.r_current = false;
            e.halo(w.x);
            e.start(true, p.inner_tolerance, -1);
        }
        x_zero = false;
        for (size_t it = 0; it < inner; ++it)
            e.iterate(w.hist + n_res, w.hist + w.cap + n_res, gt != nullptr);
        if (!p.warm_start) {
            e.weights(false);
            e.objective(false, (int)cycle + 1);
        }
        const Ctl c = read_ctl(w, stream);
        e.hook_drain();
        throw_solver(c);
        for (size_t i = 0; i < (size_t)c.iters; ++i) wall_keep.push_back(e.n_wall - inner + i);
        n_res += (size_t)c.iters;
        converged = c.converged;
        breakdown = c.breakdown;
        bounds.push_back(n_res);
        secs.push_back(now_s() - t_cycle);
    }
    if (p.warm_start) {
        e.weights(false);
        e.objective(false, (int)outer);
    }
    KCT_CUDA(cudaStreamSynchronize(stream));
    const double solve = now_s() - t_start;
    stage_out(P, w.x, x_out, w.m, true, mem, layout, 2, stream);
    if (rep) {
        copy_hist(rep->objective_history, w.obj, outer + 1, stream);
        copy_hist(rep->residual_history, w.hist, n_res, stream);
        if (gt) copy_hist(rep->error_history, w.hist + w.cap, n_res, stream);
        rep->objective_count = outer + 1;
        rep->residual_count = n_res;
        rep->error_count = gt ? n_res : 0;
        rep->outer_count = outer;
        for (size_t c = 0; c < outer; ++c) {
            if (rep->outer_boundaries) rep->outer_boundaries[c] = bounds[c];
            if (rep->outer_seconds) rep->outer_seconds[c] = secs[c];
        }
        rep->solve_seconds = solve;
        rep->tau = tau;
        rep->converged = converged;
        rep->breakdown = breakdown;
        // wall_times of the iterations that ran (a cycle stopped early keeps its first c.iters)
        std::vector<double> all(e.n_wall > 0 ? e.n_wall - 1 : 0);
        e.wall_times(all.data());
        rep->wall_count = 0;
        for (size_t idx : wall_keep)
            if (idx >= 1 && idx - 1 < all.size()) {
                if (rep->wall_times) rep->wall_times[rep->wall_count] = all[idx - 1];
                ++rep->wall_count;
            }
    }
    KCT_CUDA(cudaStreamSynchronize(stream));
}

// ---- caller-assembled stacks -------------------------------------------------
// cgls (krylov.hpp:59-127) over a StackedMap (linear_map.hpp:159-216) whose row
// blocks are scale * diag(w) * {projector, DiffOperator, IdentityMap}, all
// vectors resident on the device in the native layouts (a volume-shaped piece
// is z-fastest, a DIFF block [dx; dy; dz] of three such pieces).  Unlike the
// IRN drivers above, the regulariser residual blocks are materialised (the
// caller's right-hand side is arbitrary), so this is the reference's algorithm
// vector for vector: float32 storage, fp64 fixed-order reductions.
namespace {

// partial sums accumulate over the kernels of one phase (same block index,
// stream order: deterministic)
__device__ __forceinline__ void add_partials(double* part, int slot, double v, double* sm,
                                             int acc) {
    const double t = block_sum(v, sm);
    if (threadIdx.x == 0) {
        double* dst = part + slot * kGrid + blockIdx.x;
        *dst = acc ? *dst + t : t;
    }
}

// q = c * w .* (D p)  (diffreg.hpp:34-49); slot0 (+)= ||q||^2
__global__ void __launch_bounds__(kBlock) k_stack_diff(const float* __restrict__ p,
                                                       const float* __restrict__ w, float c,
                                                       float* __restrict__ q, RegCfg g,
                                                       double* part, int acc) {
    __shared__ double sm[32];
    const size_t m = (size_t)g.nx * g.ny * g.nz, si = g.nz, sj = (size_t)g.nz * g.nx;
    double t = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < m;
         v += (size_t)gridDim.x * blockDim.x) {
        int k, i, j;
        decode(v, g, k, i, j);
        float gx, gy, gz;
        fdiff(p, v, k, i, j, g, si, sj, p[v], gx, gy, gz);
        if (w) { gx *= w[v]; gy *= w[m + v]; gz *= w[2 * m + v]; }
        gx *= c; gy *= c; gz *= c;
        q[v] = gx; q[m + v] = gy; q[2 * m + v] = gz;
        t += (double)gx * gx + (double)gy * gy + (double)gz * gz;
    }
    add_partials(part, 0, t, sm, acc);
}

// s (+)= c * D^T (w .* r)  (diffreg.hpp:51-76, as a gather: one owner per voxel)
__global__ void __launch_bounds__(kBlock) k_stack_diff_adj(const float* __restrict__ r,
                                                           const float* __restrict__ w, float c,
                                                           float* __restrict__ s, RegCfg g,
                                                           int acc) {
    const size_t m = (size_t)g.nx * g.ny * g.nz, si = g.nz, sj = (size_t)g.nz * g.nx;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < m;
         v += (size_t)gridDim.x * blockDim.x) {
        int k, i, j;
        decode(v, g, k, i, j);
        auto y = [&](size_t u) { return w ? r[u] * w[u] : r[u]; };
        float a = 0.f;
        if (i + 1 < g.nx) a -= y(v);
        if (i > 0) a += y(v - si);
        if (j + 1 < g.ny) a -= y(m + v);
        if (j > 0) a += y(m + v - sj);
        if (k + 1 < g.nz) a -= y(2 * m + v);
        if (k > 0) a += y(2 * m + v - 1);
        s[v] = acc ? fmaf(c, a, s[v]) : c * a;
    }
}

// q = c * w .* src (src == q allowed: the projector block after its forward;
// src = p: an identity block); slot0 (+)= ||q||^2
__global__ void __launch_bounds__(kBlock) k_stack_scale(const float* src, const float* __restrict__ w,
                                                        float c, float* q, size_t n, double* part,
                                                        int acc) {
    __shared__ double sm[32];
    double t = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        float a = src[v];
        if (w) a *= w[v];
        a *= c;
        q[v] = a;
        t += (double)a * a;
    }
    add_partials(part, 0, t, sm, acc);
}

// s (+)= c * w .* r
__global__ void __launch_bounds__(kBlock) k_stack_axpy(const float* __restrict__ r,
                                                       const float* __restrict__ w, float c,
                                                       float* s, size_t n, int acc) {
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const float a = w ? r[v] * w[v] : r[v];
        s[v] = acc ? fmaf(c, a, s[v]) : c * a;
    }
}

// r -= q; slot0 = ||r||^2
__global__ void __launch_bounds__(kBlock) k_stack_sub(float* __restrict__ r,
                                                      const float* __restrict__ q, size_t n,
                                                      double* part) {
    __shared__ double sm[32];
    double t = 0.0;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const float rv = r[v] - q[v];
        r[v] = rv;
        t += (double)rv * rv;
    }
    write_partials(part, 0, t, sm);
}

struct StackBlock {
    int map;
    float scale;
    size_t off, len;          // position in the concatenated range
    const float* w = nullptr;  // device, native layout (nullptr: no diagonal)
};

struct Stack {
    Projector& P;
    Workspace& w;
    cudaStream_t stream;
    RegCfg rc{};
    std::vector<StackBlock> blocks;
    size_t range = 0;

    // q = A v  (StackedMap::apply, linear_map.hpp:185-193); slot0 = ||q||^2
    void apply(const float* v, float* q) {
        int acc = 0;
        for (const StackBlock& b : blocks) {
            float* qb = q + b.off;
            switch (b.map) {
            case KCT_MAP_PROJECTOR:
                P.forward(v, qb, stream);
                KCT_LAUNCH(k_stack_scale, qb, b.w, b.scale, qb, b.len, w.part, acc);
                break;
            case KCT_MAP_DIFF:
                KCT_LAUNCH(k_stack_diff, v, b.w, b.scale, qb, rc, w.part, acc);
                break;
            default:
                KCT_LAUNCH(k_stack_scale, v, b.w, b.scale, qb, b.len, w.part, acc);
            }
            acc = 1;
        }
    }

    // s = A^T y  (StackedMap::apply_adjoint, linear_map.hpp:195-205); slot0 = ||s||^2
    void adjoint(const float* y, float* s) {
        int acc = 0;
        for (const StackBlock& b : blocks) {
            const float* yb = y + b.off;
            switch (b.map) {
            case KCT_MAP_PROJECTOR: {
                const float* in = yb;
                if (b.w) {  // diag(w) first (ComposedMap::apply_adjoint, linear_map.hpp:134-140)
                    KCT_LAUNCH(k_stack_axpy, yb, b.w, 1.f, w.q, b.len, 0);
                    in = w.q;
                }
                if (!acc && b.scale == 1.f) {
                    P.adjoint(in, s, stream);
                } else {
                    P.adjoint(in, w.atr, stream);
                    KCT_LAUNCH(k_stack_axpy, w.atr, nullptr, b.scale, s, w.m, acc);
                }
                break;
            }
            case KCT_MAP_DIFF:
                KCT_LAUNCH(k_stack_diff_adj, yb, b.w, b.scale, s, rc, acc);
                break;
            default:
                KCT_LAUNCH(k_stack_axpy, yb, b.w, b.scale, s, b.len, acc);
            }
            acc = 1;
        }
        KCT_LAUNCH(k_stats, s, w.m, w.part);
    }
};

}  // namespace

void cgls_stack(Projector& P, const kct_stack_block* blocks, size_t n_blocks, const float* b,
                const float* x0, size_t iters, double tol, float* x_out, kct_report* rep, int mem,
                int layout, cudaStream_t stream) {
    if (!blocks || n_blocks == 0) throw ConfigError("stack: needs at least one block");
    if (!b || !x_out) throw ConfigError("cgls: null buffer");
    if (P.slab_mode() || P.comm_fn)
        throw ConfigError("kct_cgls_stack runs in a single process (sharded modes are set)");
    reset_report(rep);
    Workspace& w = workspace(P, std::max<size_t>(iters, 1), 1);
    Stack st{P, w, stream};
    set_grid(st.rc, P);
    size_t n_weights = 0;
    for (size_t i = 0; i < n_blocks; ++i) {
        StackBlock sb;
        sb.map = blocks[i].map;
        if (sb.map != KCT_MAP_PROJECTOR && sb.map != KCT_MAP_DIFF && sb.map != KCT_MAP_IDENTITY)
            throw ConfigError("stack: unknown block map");
        if (!std::isfinite(blocks[i].scale)) throw ConfigError("stack: block scale must be finite");
        sb.scale = (float)blocks[i].scale;
        sb.len = sb.map == KCT_MAP_PROJECTOR ? w.n : (sb.map == KCT_MAP_DIFF ? 3 * w.m : w.m);
        sb.off = st.range;
        st.range += sb.len;
        if (blocks[i].weights) n_weights += sb.len;
        st.blocks.push_back(sb);
    }
    const size_t R = st.range;
    const size_t need = 2 * R + n_weights;
    if (w.stack_cap < need) {
        cudaFree(w.stack);
        w.stack = nullptr;
        w.stack_cap = 0;
        KCT_CUDA(cudaMalloc(&w.stack, need * sizeof(float)));
        w.stack_cap = need;
    }
    float* r = w.stack;
    float* q = r + R;
    float* wts = q + R;
    // the right-hand side goes straight into r; volume-shaped pieces one by one
    auto load_block = [&](float* dst, const float* src, const StackBlock& sb) {
        if (sb.map == KCT_MAP_PROJECTOR) {
            load(P, dst, src, sb.len, false, mem, layout, stream);
        } else {
            for (size_t c = 0; c < sb.len / w.m; ++c)
                load(P, dst + c * w.m, src + c * w.m, w.m, true, mem, layout, stream);
        }
    };
    for (size_t i = 0; i < n_blocks; ++i) {
        StackBlock& sb = st.blocks[i];
        load_block(r + sb.off, b + sb.off, sb);
        if (blocks[i].weights) {
            load_block(wts, blocks[i].weights, sb);
            sb.w = wts;
            wts += sb.len;
        }
    }
    if (x0) load(P, w.x, x0, w.m, true, mem, layout, stream);
    else KCT_CUDA(cudaMemsetAsync(w.x, 0, w.m * sizeof(float), stream));
    KCT_CUDA(cudaMemsetAsync(w.part, 0, (size_t)kSlots * kGrid * sizeof(double), stream));
    init_ctl(w, 0.0, 0.0, stream);
    Engine e{P, w, stream};  // hook copies and the wall-time events
    set_grid(e.rc, P);
    KCT_CUDA(cudaStreamSynchronize(stream));

    HookScope hooks(e);
    const double t0 = now_s();
    e.mark_start();
    // krylov.hpp:66-96
    if (tol > 0.0 && x0) {
        KCT_LAUNCH(k_stats, w.x, w.m, w.part);
        k_set_nonzero<<<1, kBlock, 0, stream>>>(w.ctl, w.part);
        KCT_LAUNCHED();
        st.adjoint(r, w.p);  // A^T b, the tolerance reference of a warm start (:81-88)
        launch_scalar(w, S_REF, stream);
    }
    if (x0) {
        st.apply(w.x, q);
        KCT_LAUNCH(k_stack_sub, r, q, R, w.part);
    }
    st.adjoint(r, w.s);
    launch_scalar(w, S_INIT, stream, tol);
    KCT_LAUNCH(k_update_p, w.p, w.s, w.m, w.ctl, 1);
    Ctl c{};
    bool stopped = false;
    if (tol > 0.0) stopped = (c = read_ctl(w, stream)).stop != 0;
    // krylov.hpp:98-125
    for (size_t it = 0; it < iters && !stopped; ++it) {
        st.apply(w.p, q);
        launch_scalar(w, S_DELTA, stream);
        KCT_LAUNCH(k_update_xr, w.x, w.p, w.m, r, q, R, nullptr, w.ctl, w.part);
        e.hook_copy();
        st.adjoint(r, w.s);
        launch_scalar(w, S_GAMMA, stream, 0.0, w.hist, nullptr);
        KCT_LAUNCH(k_update_p, w.p, w.s, w.m, w.ctl, 0);
        if (e.n_wall < w.wall_ev.size()) KCT_CUDA(cudaEventRecord(w.wall_ev[e.n_wall++], stream));
        // an early stop (tolerance) is noticed within a few iterations
        if (tol > 0.0 && (it & 3) == 3) stopped = (c = read_ctl(w, stream)).stop != 0;
    }
    c = read_ctl(w, stream);
    const double secs = now_s() - t0;
    e.hook_drain();
    throw_solver(c);
    stage_out(P, w.x, x_out, w.m, true, mem, layout, 2, stream);
    if (rep) {
        const size_t n = (size_t)c.iters;
        copy_hist(rep->residual_history, w.hist, n, stream);
        KCT_CUDA(cudaStreamSynchronize(stream));
        rep->residual_count = n;
        rep->solve_seconds = secs;
        rep->converged = c.converged;
        rep->breakdown = c.breakdown;
        write_wall(e, rep);
        if (rep->wall_count > n) rep->wall_count = n;
    }
    KCT_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace kct
