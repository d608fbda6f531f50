// fdk.cu — Feldkamp-Davis-Kress filtered backprojection (reference fdk.hpp:50-139).
//
// Used by the reference to build priors and to calibrate alpha
// (experiment.hpp:372-385, :440-449); SURVEY §8(f) item 4.  Three stages as in
// the reference: cosine weighting, row-wise Ram-Lak ramp filter, and
// distance-weighted bilinear voxel-driven backprojection.  The reference
// filters with a radix-2 FFT on rows zero-padded to >= 2*nu, which is exactly
// the linear convolution with the spatial Ram-Lak kernel
//     h(0) = 1/(4 du^2),  h(odd d) = -1/(pi^2 d^2 du^2),  h(even d != 0) = 0
// (every tap |d| < nu <= pad/2), so the filter here is that direct
// convolution, evaluated from a shared-memory tile of 32 detector rows.
#include <algorithm>
#include <cmath>

#include "projector.cuh"

namespace kct {

namespace {

struct FdkGeom {
    int nu, nv, na;
    int nx, ny, nz;
    double dso, du, dv, u0, v0;  // virtual detector through the axis (fdk.hpp:59-63)
    double ox, oy, oz, sx, sy, sz;
    float scale;                 // 0.5 * 2 pi / na (fdk.hpp:96-97)
};

// Stage 1+2 (fdk.hpp:65-86): one CTA = one angle x R detector rows; the
// cosine-weighted rows are staged in shared memory ([nu][R]), a lane takes row
// lane % R of output column phase lane / R, warps stride over the output
// columns.  R = 32 while the tile fits (nu <= ~1700 columns at 227 KB), fewer
// rows per CTA for wider detectors (R = 1 reaches nu ~ 19000; the reference's
// FFT filter has no width limit).  Input / output in the native v-fastest layout.
template <int R>
__global__ void __launch_bounds__(256) k_fdk_filter(const float* __restrict__ proj,
                                                    float* __restrict__ out, FdkGeom f) {
    constexpr int CP = 32 / R;              // column phases per warp
    extern __shared__ double smd[];
    double* h = smd;                                      // [nu] kernel taps by distance
    float* tile = reinterpret_cast<float*>(smd + f.nu);  // [nu][R]
    const int a = blockIdx.y, iv0 = blockIdx.x * R;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int row = lane % R, cph = lane / R;
    const int iv = iv0 + row;
    const bool row_ok = iv < f.nv;
    const float* pa = proj + (size_t)a * f.nu * f.nv;
    const double v = f.v0 + iv * f.dv;
    for (int iu = warp * CP + cph; iu < f.nu; iu += nwarp * CP) {
        float w = 0.f;
        if (row_ok) {
            const double u = f.u0 + iu * f.du;
            const double cosw = f.dso / sqrt(f.dso * f.dso + u * u + v * v);
            w = (float)(pa[(size_t)iu * f.nv + iv] * cosw);
        }
        tile[iu * R + row] = w;
    }
    const double inv = 1.0 / (f.du * f.du);
    for (int d = threadIdx.x; d < f.nu; d += blockDim.x)
        h[d] = d == 0 ? 0.25 * inv : ((d & 1) ? -inv / (M_PI * M_PI * (double)d * (double)d) : 0.0);
    __syncthreads();
    float* po = out + (size_t)a * f.nu * f.nv;
    for (int iu = warp * CP + cph; iu < f.nu; iu += nwarp * CP) {
        // float64 taps and sum: the ramp filter of a smooth row is a small
        // residual of large cancelling terms (float32 sums lose ~1e-4 relative
        // at a few thousand columns; the reference filters in float64)
        double acc = h[0] * tile[iu * R + row];
        // odd distances only: iu' = iu -/+ 1, 3, 5, ...
        for (int d = 1; d <= iu; d += 2) acc = fma(h[d], (double)tile[(iu - d) * R + row], acc);
        for (int d = 1; iu + d < f.nu; d += 2) acc = fma(h[d], (double)tile[(iu + d) * R + row], acc);
        if (row_ok) po[(size_t)iu * f.nv + iv] = (float)(acc * f.du);
    }
}

template <int R>
void launch_fdk_filter(const float* proj, float* filt, const FdkGeom& f, cudaStream_t s) {
    const size_t smem = (size_t)f.nu * R * sizeof(float) + (size_t)f.nu * sizeof(double);
    KCT_CUDA(cudaFuncSetAttribute(k_fdk_filter<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 g1((f.nv + R - 1) / R, f.na);
    k_fdk_filter<R><<<g1, 256, smem, s>>>(proj, filt, f);
    KCT_LAUNCHED();
}

// Stage 3 (fdk.hpp:88-138): a warp owns 32*KZ consecutive slabs of one voxel
// column (native z-fastest layout), lane = slab k = kbase + lane + 32 q.  The
// per-(column, angle) projection (u coordinate, magnification, distance
// weight) is warp-uniform; per slab only the v coordinate changes, so the
// detector reads of a warp are consecutive rows of one or two detector
// columns (coalesced).  Float32 positions: |error| ~1e-5 pixel, far inside the
// 1e-4 bar, with the bilinear interpolation continuous across pixel and
// detector edges.  Each voxel sums its own angle loop (deterministic).
constexpr int kFdkKZ = 4;
__global__ void __launch_bounds__(256) k_fdk_backproject(const float* __restrict__ filt,
                                                         float* __restrict__ vol, FdkGeom f,
                                                         AngleBatch ab, int a0, int nab,
                                                         int accumulate) {
    const int lane = threadIdx.x & 31;
    const size_t wid = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const int kchunks = (f.nz + 32 * kFdkKZ - 1) / (32 * kFdkKZ);
    const size_t col = wid / kchunks;
    if (col >= (size_t)f.nx * f.ny) return;
    const int kbase = (int)(wid - col * kchunks) * 32 * kFdkKZ + lane;
    const int i = (int)(col % f.nx), j = (int)(col / f.nx);
    const float x = (float)(f.ox + (i + 0.5) * f.sx), y = (float)(f.oy + (j + 0.5) * f.sy);
    const float dso = (float)f.dso;
    const float inv_du = (float)(1.0 / f.du), inv_dv = (float)(1.0 / f.dv);
    const float u0 = (float)f.u0, v0 = (float)f.v0;
    float zq[kFdkKZ], acc[kFdkKZ];
#pragma unroll
    for (int q = 0; q < kFdkKZ; ++q) {
        zq[q] = (float)(f.oz + (kbase + 32 * q + 0.5) * f.sz);
        acc[q] = 0.f;
    }
    for (int a = 0; a < nab; ++a) {
        const float c = ab.cs[a].x, s = ab.cs[a].y;
        const float ss = fmaf(x, c, y * s), t = fmaf(-x, s, y * c);
        const float L = dso - ss;
        if (!(L > 1e-6f * dso)) continue;
        const float mag = __fdiv_rn(dso, L);
        const float fu = (t * mag - u0) * inv_du;
        const int ju = (int)floorf(fu);
        if (ju < -1 || ju > f.nu - 1) continue;
        const float au = fu - (float)ju;
        const float wgt = mag * mag;
        const float* fa = filt + (size_t)(a0 + a) * f.nu * f.nv;
        const float* c0 = ju >= 0 ? fa + (size_t)ju * f.nv : nullptr;
        const float* c1 = ju + 1 < f.nu ? fa + (size_t)(ju + 1) * f.nv : nullptr;
#pragma unroll
        for (int q = 0; q < kFdkKZ; ++q) {
            const float fv = (zq[q] * mag - v0) * inv_dv;
            const int jv = (int)floorf(fv);
            if (jv < -1 || jv > f.nv - 1) continue;
            const float av = fv - (float)jv;
            const bool r0 = jv >= 0, r1 = jv + 1 < f.nv;
            const float s00 = (c0 && r0) ? __ldg(c0 + jv) : 0.f;
            const float s01 = (c0 && r1) ? __ldg(c0 + jv + 1) : 0.f;
            const float s10 = (c1 && r0) ? __ldg(c1 + jv) : 0.f;
            const float s11 = (c1 && r1) ? __ldg(c1 + jv + 1) : 0.f;
            const float val = (1.f - au) * ((1.f - av) * s00 + av * s01) +
                              au * ((1.f - av) * s10 + av * s11);
            acc[q] = fmaf(wgt, val, acc[q]);
        }
    }
    float* o = vol + col * f.nz;
#pragma unroll
    for (int q = 0; q < kFdkKZ; ++q) {
        const int k = kbase + 32 * q;
        if (k < f.nz) {
            const float r = f.scale * acc[q];
            o[k] = accumulate ? o[k] + r : r;
        }
    }
}

}  // namespace

void Projector::fdk(const float* proj, float* vol, float* filt, cudaStream_t s) const {
    if (dg_.na < 2) throw ConfigError("fdk needs at least two projection angles");
    FdkGeom f;
    f.nu = dg_.nu; f.nv = dg_.nv; f.na = dg_.na;
    f.nx = grid_.nx; f.ny = grid_.ny; f.nz = grid_.nz;
    const double mag = dso_d_ / dsd_d_;
    f.dso = dso_d_;
    f.du = pu_d_ * mag;
    f.dv = pv_d_ * mag;
    f.u0 = (0.5 - 0.5 * f.nu) * f.du + offu_d_ * mag;
    f.v0 = (0.5 - 0.5 * f.nv) * f.dv + offv_d_ * mag;
    f.ox = grid_.ox; f.oy = grid_.oy; f.oz = grid_.oz;
    f.sx = grid_.sx; f.sy = grid_.sy; f.sz = grid_.sz;
    f.scale = (float)(0.5 * (2.0 * M_PI / (double)f.na));
    // rows per filter CTA: the most that fit the shared-memory tile
    int smem_max = 0;
    KCT_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device_));
    const auto fits = [&](int R) {
        return (size_t)f.nu * R * sizeof(float) + (size_t)f.nu * sizeof(double) <= (size_t)smem_max;
    };
    if (fits(32)) launch_fdk_filter<32>(proj, filt, f, s);
    else if (fits(16)) launch_fdk_filter<16>(proj, filt, f, s);
    else if (fits(8)) launch_fdk_filter<8>(proj, filt, f, s);
    else if (fits(4)) launch_fdk_filter<4>(proj, filt, f, s);
    else if (fits(2)) launch_fdk_filter<2>(proj, filt, f, s);
    else if (fits(1)) launch_fdk_filter<1>(proj, filt, f, s);
    else throw ConfigError("fdk: detector too wide for the shared-memory row filter");
    AngleBatch ab;
    const size_t warps = (size_t)f.nx * f.ny * ((f.nz + 32 * kFdkKZ - 1) / (32 * kFdkKZ));
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    for (int a0 = 0; a0 < f.na; a0 += kMaxAnglesPerLaunch) {
        const int nab = std::min(kMaxAnglesPerLaunch, f.na - a0);
        for (int q = 0; q < nab; ++q) ab.cs[q] = cs_[a0 + q];
        k_fdk_backproject<<<blocks, 256, 0, s>>>(filt, vol, f, ab, a0, nab, a0 > 0 ? 1 : 0);
        KCT_LAUNCHED();
    }
}

}  // namespace kct
