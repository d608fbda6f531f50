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

// Stage 1+2 (fdk.hpp:65-86): one CTA = one angle x 32 detector rows; the
// cosine-weighted rows are staged in shared memory, lane = row, warps stride
// over the output columns.  Input / output in the native v-fastest layout.
__global__ void __launch_bounds__(256) k_fdk_filter(const float* __restrict__ proj,
                                                    float* __restrict__ out, FdkGeom f) {
    extern __shared__ float sm[];
    float* tile = sm;                       // [nu][32]
    float* h = sm + (size_t)f.nu * 32;      // [nu] kernel taps by distance
    const int a = blockIdx.y, iv0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int iv = iv0 + lane;
    const bool row_ok = iv < f.nv;
    const float* pa = proj + (size_t)a * f.nu * f.nv;
    const double v = f.v0 + iv * f.dv;
    for (int iu = warp; iu < f.nu; iu += nwarp) {
        float w = 0.f;
        if (row_ok) {
            const double u = f.u0 + iu * f.du;
            const double cosw = f.dso / sqrt(f.dso * f.dso + u * u + v * v);
            w = (float)(pa[(size_t)iu * f.nv + iv] * cosw);
        }
        tile[iu * 32 + lane] = w;
    }
    const double inv = 1.0 / (f.du * f.du);
    for (int d = threadIdx.x; d < f.nu; d += blockDim.x)
        h[d] = d == 0 ? (float)(0.25 * inv)
                      : ((d & 1) ? (float)(-inv / (M_PI * M_PI * (double)d * (double)d)) : 0.f);
    __syncthreads();
    float* po = out + (size_t)a * f.nu * f.nv;
    for (int iu = warp; iu < f.nu; iu += nwarp) {
        float acc = h[0] * tile[iu * 32 + lane];
        // odd distances only: iu' = iu -/+ 1, 3, 5, ...
        for (int d = 1; d <= iu; d += 2) acc = fmaf(h[d], tile[(iu - d) * 32 + lane], acc);
        for (int d = 1; iu + d < f.nu; d += 2) acc = fmaf(h[d], tile[(iu + d) * 32 + lane], acc);
        if (row_ok) po[(size_t)iu * f.nv + iv] = (float)(acc * f.du);
    }
}

// Stage 3 (fdk.hpp:88-138): one thread per voxel (native z-fastest layout, a
// warp = 32 consecutive slabs of one voxel column), each voxel sums its own
// angle loop (deterministic).
__global__ void __launch_bounds__(256) k_fdk_backproject(const float* __restrict__ filt,
                                                         float* __restrict__ vol, FdkGeom f,
                                                         AngleBatch ab, int a0, int nab,
                                                         int accumulate) {
    const size_t m = (size_t)f.nx * f.ny * f.nz;
    const size_t vidx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (vidx >= m) return;
    const int k = (int)(vidx % f.nz);
    const int p = (int)(vidx / f.nz);
    const int i = p % f.nx, j = p / f.nx;
    const double x = f.ox + (i + 0.5) * f.sx, y = f.oy + (j + 0.5) * f.sy;
    const double z = f.oz + (k + 0.5) * f.sz;
    float acc = 0.f;
    for (int q = 0; q < nab; ++q) {
        const double c = ab.cs[q].x, s = ab.cs[q].y;
        const double ss = x * c + y * s, t = -x * s + y * c;
        const double L = f.dso - ss;
        if (L <= 1e-6 * f.dso) continue;
        const double fu = (t * f.dso / L - f.u0) / f.du;
        const double fv = (z * f.dso / L - f.v0) / f.dv;
        const int ju = (int)floor(fu), jv = (int)floor(fv);
        if (ju < -1 || ju > f.nu - 1 || jv < -1 || jv > f.nv - 1) continue;
        const float au = (float)(fu - ju), av = (float)(fv - jv);
        const float* fa = filt + (size_t)(a0 + q) * f.nu * f.nv;
        auto sample = [&](int uu, int vv) -> float {
            return (uu < 0 || uu >= f.nu || vv < 0 || vv >= f.nv) ? 0.f
                                                                   : __ldg(fa + (size_t)uu * f.nv + vv);
        };
        const float val = (1.f - au) * (1.f - av) * sample(ju, jv) + au * (1.f - av) * sample(ju + 1, jv) +
                          (1.f - au) * av * sample(ju, jv + 1) + au * av * sample(ju + 1, jv + 1);
        acc = fmaf((float)((f.dso * f.dso) / (L * L)), val, acc);
    }
    const float r = f.scale * acc;
    vol[vidx] = accumulate ? vol[vidx] + r : r;
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
    const size_t smem = ((size_t)f.nu * 32 + f.nu) * sizeof(float);
    KCT_CUDA(cudaFuncSetAttribute(k_fdk_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 g1((f.nv + 31) / 32, f.na);
    k_fdk_filter<<<g1, 256, smem, s>>>(proj, filt, f);
    KCT_CUDA(cudaGetLastError());
    AngleBatch ab;
    const size_t m = domain_size();
    const unsigned blocks = (unsigned)((m + 255) / 256);
    for (int a0 = 0; a0 < f.na; a0 += kMaxAnglesPerLaunch) {
        const int nab = std::min(kMaxAnglesPerLaunch, f.na - a0);
        for (int q = 0; q < nab; ++q) ab.cs[q] = cs_[a0 + q];
        k_fdk_backproject<<<blocks, 256, 0, s>>>(filt, vol, f, ab, a0, nab, a0 > 0 ? 1 : 0);
        KCT_CUDA(cudaGetLastError());
    }
}

}  // namespace kct
