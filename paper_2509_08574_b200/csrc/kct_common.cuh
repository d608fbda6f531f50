// kct_common.cuh — shared device/host definitions of the B200 CBCT core.
//
// Internal (native) layouts, chosen for the 2D+1 structure of the flat-panel
// circular geometry (projector.hpp:24-39: u ⊥ z, source at z = 0, so a ray's
// xy path depends only on the detector column iu and its z slope only on the
// row iv):
//   volume       z-fastest   idx = k + nz*(i + nx*j)
//   projections  v-fastest   idx = iv + nv*(iu + nu*ia)
// A warp of 32 consecutive detector rows then reads 32 nearly consecutive k
// of one voxel column, and a warp of 32 consecutive k gathers 32 nearly
// consecutive rows of one detector column: both directions are coalesced.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/kct.h"

namespace kct {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define KCT_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::kct::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// NVTX range around a library phase (header-only NVTX v3: free unless a
// profiler such as Nsight Systems injects its tool library).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Every kernel launch of the library is counted (kct_launch_count): evidence
// of which work ran on the device, read by bench.py around its timed region.
void note_launch();
#define KCT_LAUNCHED()                          \
    do {                                        \
        ::kct::note_launch();                   \
        KCT_CUDA(cudaGetLastError());           \
    } while (0)

// Per (angle, detector column) parameters of the shared xy ray path, computed
// on the host in double and stored as float.  w is the signed xy distance
// along the column's unit direction, measured from the foot point R of the
// rotation axis on the ray (re-basing at R keeps |w| <~ FOV, which is what
// makes float32 crossings accurate; a [0,1] parametrisation over the full
// source-detector segment is not).
//   x-plane n is crossed at  w = (float)fma(n, dx, bx)   (float64: a ray nearly
//   parallel to the planes has |bx|, |dx| >> |w|), y-plane n likewise
//   [w_in, w_out]  clip of the ray against the volume's xy box and t in [0,1]
//   continuous z index at w_in of detector row dv (float64, split as k0 + f0):
//           kz_in = fma(dv, g_in, -kz0),  k0 = floor(kz_in),  f0 = kz_in - k0
//   z-plane P is crossed at  w = fmaf((P - k0) - f0, inv_dv * inv_h1, w_in)
//   3D length = dw * sqrt(1 + (dv * inv_l)^2)
// Forward and adjoint evaluate exactly these expressions, so every segment
// endpoint is bit-identical between A and A^T.
struct __align__(16) ColParams {
    double bx, dx, by, dy;
    float w_in, w_out, inv_h1, inv_l;
    double g_in;
    int i0, j0;  // entry voxel (valid when w_in < w_out)
};

__device__ __forceinline__ float xcross(const ColParams& c, int n) {
    return __double2float_rn(fma((double)n, c.dx, c.bx));
}
__device__ __forceinline__ float ycross(const ColParams& c, int n) {
    return __double2float_rn(fma((double)n, c.dy, c.by));
}
// z-plane P crossing of a row with z state (k0, f0) and inverse slope imk
__device__ __forceinline__ float zcross(int P, int k0, float f0, float imk, float w_in) {
    return __fmaf_rn(__fsub_rn((float)(P - k0), f0), imk, w_in);
}

// Per detector row: dv in float64 and float32 and 1/dv (inf at dv == 0), the
// row's z slope data, packed for one 16-byte load.
struct __align__(16) RowTab {
    double dvd;
    float dv, invdv;
};
__device__ __forceinline__ RowTab ld_row(const RowTab* __restrict__ rows, int iv) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(rows) + iv);
    RowTab r;
    r.dvd = t.x;
    const float2 f = *reinterpret_cast<const float2*>(&t.y);
    r.dv = f.x;
    r.invdv = f.y;
    return r;
}

constexpr int kMaxAnglesPerLaunch = 1024;

// Per-angle cos/sin, passed by value in the kernel parameter space (constant
// bank), batched by kMaxAnglesPerLaunch.
struct AngleBatch {
    float2 cs[kMaxAnglesPerLaunch];
};

struct DevGeom {
    int nx, ny, nz;
    int nu, nv, na;
    float ox, oy, sx, sy;  // xy box
    float kz0;             // oz / sz
    double kz0d;
    float dso, dsd;
    float pu, off_u;       // fu = (du - off_u)/pu + nu/2 - 1/2
    float pv, dv0;         // dv(iv) = fmaf(iv, pv, dv0)
    int full_footprint;    // 1: some voxel square is not fully in front of a source
    int fwd_bands;         // forward row bands (32*C rows each) in this launch
    int fwd_band0;         // first row band of this launch
    int fwd_row0;          // row (mirror: row pair) of band 0's first lane (staged host forward)
    int mirror;            // 1: z-mirror geometry, rows iv / nv-1-iv walked as pairs (fwd_kernel MIR)
    int out_ref;           // 1: the forward writes the reference layout [a][iv][iu] (staged host forward)
};

// ---- deterministic fp64 block reduction ----------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Sums `v` over the block (blockDim.x multiple of 32, <= 1024) in a fixed
// order; the result is valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* smem32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) smem32[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        r = lane < nw ? smem32[lane] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

}  // namespace kct
