// projector.cu — Siddon forward projector (ray-driven, 2D+1) and its exact
// transpose (brick-owned, deterministic) for sm_100a.
//
// Reference semantics: projector.hpp:53-131 (traverse_ray), :173-204
// (project_forward), :207-261 (project_adjoint).  The intersection lengths are
// the reference's exact Siddon lengths; only rounding differs (float32 values,
// float64 host geometry and plane crossings).  Forward and adjoint evaluate
// every ray-voxel segment endpoint with the same expressions (ColParams,
// xcross/ycross/zcross in kct_common.cuh), so A^T is the transpose of A up to
// the rounding of the final products and sums.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <climits>
#include <limits>
#include <string>

#include <cuda.h>

#include "projector.cuh"

namespace kct {

namespace {

constexpr float kInf = __builtin_huge_valf();
constexpr unsigned kFull = 0xffffffffu;

// ----------------------------------------------------------------------------
// Forward projector.  One warp = one detector column iu of one angle, C row
// chunks of 32 (lane + 32c).  The xy Siddon walk of the column is shared by
// all its rows (the "2D" part, warp-uniform); every lane carries the z state
// of its C rays (the "+1" part): current slab k, next z-plane crossing wz.
// A CTA holds 4 adjacent columns of the same angle and row band so their
// overlapping voxel columns are served from L1.
// ----------------------------------------------------------------------------
#ifndef KCT_FWD_MINB
#define KCT_FWD_MINB 8  // 64 registers, 8 CTAs of 4 warps per SM (re-swept with the walk table and row
                        // pairs: 6 / 8 / 9 / 10 / 12 -> c3 1.709 / 1.666 / 1.672 / 1.728 / 2.121 ms, c4 11.55 /
                        // 10.81 / 10.61 / 10.78 ms, c2 0.187 / 0.173 / 0.179 ms; 9 and up spill)
#endif
#ifndef KCT_FWD_WARPS
#define KCT_FWD_WARPS 4  // adjacent detector columns per CTA (shared voxel columns in L1)
#endif
constexpr int kFwdWarps = KCT_FWD_WARPS;
#ifndef KCT_VPAD_ALIGN
#define KCT_VPAD_ALIGN 0
#endif
// padded forward volume: slab 0 of a column at offset kVOff, column stride
// vpad_stride(nz) (zero slabs at -1 and nz)
constexpr int kVOff = KCT_VPAD_ALIGN ? 16 : 1;
__host__ __device__ constexpr int vpad_stride(int nz) {
    return KCT_VPAD_ALIGN ? (kVOff + nz + 1 + 31) / 32 * 32 : nz + 2;  // (aligned: measured +-0)
}
// Host pipeline: angle chunks [cb[c], cb[c + 1]) whose finished columns a
// counted forward launch adds to count[c].
struct FwdChunks {
    unsigned* count;
    int n;
    int cb[9];
};
static_assert(Projector::kPipeChunks <= 8, "FwdChunks holds at most 8 pipeline chunks");

// The xy Siddon walk of one (angle, column) through the padded volume's
// voxel columns: seg(wa, wb, col) for every segment [wa, wb] of voxel column
// col = (i + nx j) * vpad_stride(nz), in ray order (projector.hpp:116-129
// restricted to the x / y planes).  Shared by the forward and its walk table.
template <class F>
__device__ __forceinline__ void xy_walk(const ColParams& cp, const DevGeom& g, F&& seg) {
    const int nx = g.nx, ny = g.ny;
    int i = cp.i0, j = cp.j0;
    const int stx = cp.dx > 0.0 ? 1 : -1, sty = cp.dy > 0.0 ? 1 : -1;
    int px = cp.dx > 0.0 ? i + 1 : i;
    int py = cp.dy > 0.0 ? j + 1 : j;
    float wnx = cp.dx != 0.0 ? xcross(cp, px) : kInf;
    float wny = cp.dy != 0.0 ? ycross(cp, py) : kInf;
    float wcur = cp.w_in;
    for (;;) {
        const bool stepx = wnx <= wny;
        const float wnext = stepx ? wnx : wny;
        const float wb = fmaxf(fminf(wnext, cp.w_out), wcur);
        // the column's slab 0 in the padded volume (zero slabs at -1 and nz:
        // slabs k in [-1, nz] need no range check; 32-bit element index)
        seg(wcur, wb, (i + nx * j) * vpad_stride(g.nz));
        if (wnext >= cp.w_out) break;
        wcur = fmaxf(wnext, wcur);
        if (stepx) {
            i += stx;
            if ((unsigned)i >= (unsigned)nx) break;
            px += stx;
            wnx = xcross(cp, px);
        } else {
            j += sty;
            if ((unsigned)j >= (unsigned)ny) break;
            py += sty;
            wny = ycross(cp, py);
        }
    }
}

// Forward walk table (TAB): per (angle, column) the segments of xy_walk as
// {bits of wb, col}, segment s of column (a, iu) at seg[off[a nu + iu] + s]
// (a segment starts where the previous one ends; the first at w_in).
}  // namespace
struct FwdTab {
    const unsigned* off;
    const int2* seg;
};
namespace {

// FILL = false: segment counts per column into cnt; true: write them at off.
template <bool FILL>
__global__ void __launch_bounds__(128) fwd_tab_build(const ColParams* __restrict__ cols, DevGeom g,
                                                     unsigned* __restrict__ cnt,
                                                     const unsigned* __restrict__ off,
                                                     int2* __restrict__ seg) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= (size_t)g.na * g.nu) return;
    const ColParams cp = cols[t];
    unsigned n = 0;
    if (cp.w_in < cp.w_out) {
        int2* o = FILL ? seg + off[t] : nullptr;
        xy_walk(cp, g, [&](float, float wb, int col) {
            if (FILL) o[n] = make_int2(__float_as_int(wb), col);
            ++n;
        });
    }
    if (!FILL) cnt[t] = n;
}

// vol: slab 0 of voxel column 0 of the padded native volume (column stride
// nz + 2, zero slabs at -1 and nz; Projector::pad_volume).
//
// MIR (z-mirror pairs; Projector::mirror_): in a z-symmetric geometry
// (offset_v = 0, nv even, grid centred in z) detector rows iv and nv-1-iv
// are reflections of each other in the plane z = 0, and so are slabs k and
// nz-1-k.  A lane then walks ray pair p — the primary row nv/2-1-p (dv < 0)
// and its mirror nv/2+p — with ONE z state: the mirror ray is defined to
// cross plane nz-P exactly where the primary crosses plane P (the same float
// values; the adjoint's per-ray records encode the mirror's z state so that
// its zcross gives these values, adj_weight_kernel), so per xy segment and per
// z crossing one test serves two rays, which load slabs k and nz-1-k.  Pairs
// are numbered from the centre plane outwards (band 0: the rows nearest z = 0).
template <int C, bool COUNT, bool DONE = false, bool MIR = false, bool TAB = false, bool REF = false>
__global__ void __launch_bounds__(kFwdWarps * 32, KCT_FWD_MINB) fwd_kernel(const float* __restrict__ vol,
                                                  float* __restrict__ out,
                                                  const ColParams* __restrict__ cols,
                                                  const float* __restrict__ dvtab,
                                                  const float* __restrict__ invdv,
                                                  const double* __restrict__ dvd, DevGeom g,
                                                  const int* __restrict__ order,
                                                  FwdChunks done, FwdTab tab) {
    // blocks are dispatched in index order; `order` maps them to (angle, row
    // band, column quad) items longest-chord first, so the last wave holds
    // the shortest rays (no long tail, notably with few angles per GPU)
    const int nq = (g.nu + kFwdWarps - 1) / kFwdWarps;
    const int item = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
    const int quad = item % nq, rest = item / nq;
    const int band = g.fwd_band0 + rest % g.fwd_bands, a = rest / g.fwd_bands;
    const int lane = threadIdx.x & 31;
    const int iu = quad * kFwdWarps + (threadIdx.x >> 5);
    if (iu >= g.nu) return;
    const ColParams cp = cols[(size_t)a * g.nu + iu];
    const int iv0 = g.fwd_row0 + band * (32 * C) + lane;  // row (MIR: pair) of chunk 0
    const int nz = g.nz;
    const int nrows = MIR ? g.nv / 2 : g.nv;

    // per ray: slab k, next crossing wz of plane P (kept as pk = P - k0),
    // remaining crossings nrem of planes inside [0, nz]
    float acc[C], accm[C], wz[C], fz[C], imk[C], dvv[C];
    int k[C], kstep[C], pk[C], nrem[C];
    bool hit = false;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int p = iv0 + 32 * c;
        const int iv = MIR ? g.nv / 2 - 1 - p : p;  // MIR: the primary (dv < 0)
        acc[c] = 0.f;
        accm[c] = 0.f;
        const bool row_ok = p < nrows;
        const float dv = row_ok ? dvtab[iv] : 0.f;
        dvv[c] = dv;
        // z index at w_in in float64, split into integer + fraction
        const double kzd = fma(row_ok ? dvd[iv] : 0.0, cp.g_in, -g.kz0d);
        const double fl = floor(kzd);
        const int k0 = (int)fmax(fmin(fl, 1.0e9), -1.0e9);
        fz[c] = (float)(kzd - fl);
        imk[c] = row_ok ? __fmul_rn(invdv[iv], cp.inv_h1) : 0.f;
        int kk = min(max(k0, -1), nz);
        const int ks = MIR ? -1 : (dv > 0.f ? 1 : -1);
        kstep[c] = ks;
        const int P = ks > 0 ? kk + 1 : kk;
        int n = ks > 0 ? nz - kk : kk + 1;  // planes P, P+ks, ... inside [0, nz]
        if (!row_ok || dv == 0.f) n = 0;
        if (!row_ok) kk = MIR ? nz : -1;  // reads the zero pads, never crosses
        k[c] = kk;
        pk[c] = P - k0;
        nrem[c] = max(n, 0);
        wz[c] = nrem[c] > 0 ? __fmaf_rn(__fsub_rn((float)pk[c], fz[c]), imk[c], cp.w_in) : kInf;
        // a ray meets the volume iff it starts inside the z range or its first
        // plane crossing (the entry plane) comes before the xy exit
        hit = hit || (row_ok && (unsigned)kk < (unsigned)nz) || wz[c] < cp.w_out;
    }

    // rows that all pass above / below the volume (detector overhang, c4)
    // skip the walk: their line integrals are 0
    if (cp.w_in < cp.w_out && __any_sync(kFull, hit)) {
        // one xy segment [wcur, wb] of padded voxel column col, all rows
        auto segment = [&](float wcur, float wb, int col) {
            const int colm = col + nz - 1;  // MIR: slab nz-1-k at colm - k
            float v[C], vm[C], wa[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                wa[c] = wcur;
                v[c] = COUNT ? ((unsigned)k[c] < (unsigned)nz ? 1.f : 0.f) : __ldg(vol + (col + k[c]));
                if (MIR) vm[c] = COUNT ? v[c] : __ldg(vol + (colm - k[c]));
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (wz[c] < wb) {  // this ray crosses z-plane(s) inside the segment
                    do {
                        const float len = wz[c] - wa[c];
                        if (COUNT) {
                            acc[c] += (len > 0.f && v[c] != 0.f) ? 1.f : 0.f;
                        } else {
                            acc[c] = __fmaf_rn(len, v[c], acc[c]);
                            if (MIR) accm[c] = __fmaf_rn(len, vm[c], accm[c]);
                        }
                        wa[c] = wz[c];
                        k[c] += kstep[c];
                        v[c] = COUNT ? ((unsigned)k[c] < (unsigned)nz ? 1.f : 0.f) : __ldg(vol + (col + k[c]));
                        if (MIR && !COUNT) vm[c] = __ldg(vol + (colm - k[c]));
                        pk[c] += kstep[c];
                        nrem[c] -= 1;
                        wz[c] = nrem[c] > 0
                                    ? __fmaf_rn(__fsub_rn((float)pk[c], fz[c]), imk[c], cp.w_in)
                                    : kInf;
                    } while (wz[c] < wb);
                }
                const float len = wb - wa[c];
                if (COUNT) {
                    acc[c] += (len > 0.f && v[c] != 0.f) ? 1.f : 0.f;
                } else {
                    acc[c] = __fmaf_rn(len, v[c], acc[c]);
                    if (MIR) accm[c] = __fmaf_rn(len, vm[c], accm[c]);
                }
            }
        };
        if (TAB) {
            // the column's walk from the table (fwd_tab_build: the segments
            // xy_walk produces), 32 segments per coalesced load, broadcast
            const unsigned s0 = tab.off[(size_t)a * g.nu + iu], s1 = tab.off[(size_t)a * g.nu + iu + 1];
            float wcur = cp.w_in;
            for (unsigned sb = s0; sb < s1; sb += 32) {
                const int2 e = sb + lane < s1 ? __ldg(tab.seg + sb + lane) : make_int2(0, 0);
                const int ns = (int)min(32u, s1 - sb);
                for (int t = 0; t < ns; ++t) {
                    const float wb = __int_as_float(__shfl_sync(kFull, e.x, t));
                    segment(wcur, wb, __shfl_sync(kFull, e.y, t));
                    wcur = wb;
                }
            }
        } else {
            xy_walk(cp, g, segment);
        }
    }

    // native layout [a][iu][iv] (a warp's rows are contiguous), or — REF, the
    // staged host forward — the reference layout [a][iv][iu] directly: the
    // strided stores merge in L2 (the projections fit) and the copy stream
    // needs no transpose kernel, which had to squeeze in between the forward's
    // blocks (a template flag: as a run-time flag it cost the device-resident
    // forward 1.6-2%)
    float* o = REF ? out + (size_t)a * g.nu * g.nv + iu : out + ((size_t)a * g.nu + iu) * g.nv;
    const size_t os = REF ? (size_t)g.nu : 1;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int p = iv0 + 32 * c;
        if (p < nrows) {
            const int iv = MIR ? g.nv / 2 - 1 - p : p;
            if (COUNT) {
                o[iv * os] = acc[c];
                if (MIR) o[(g.nv - 1 - iv) * os] = acc[c];  // the mirror's pieces are the primary's
            } else {
                // the mirror's 3D length factor is the primary's (dv(nv-1-iv) = -dv(iv))
                const float q = dvv[c] * cp.inv_l;
                const float f = __fsqrt_rn(__fmaf_rn(q, q, 1.f));
                o[iv * os] = acc[c] * f;
                if (MIR) o[(g.nv - 1 - iv) * os] = accm[c] * f;
            }
        }
    }
    if (DONE) {  // host pipeline: this column of this band of angle a is out
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            int ck = 0;
            while (ck + 1 < done.n && a >= done.cb[ck + 1]) ++ck;
            atomicAdd(done.count + ck, 1u);
        }
    }
}

// Detector-column footprint of an axis-aligned xy rectangle at one angle:
// the columns whose ray passes the rectangle's interior (projected corners,
// widened by eps pixels).
__device__ __forceinline__ void footprint(const DevGeom& g, float cth, float sth, float X0, float X1,
                                          float Y0, float Y1, int& lo, int& hi) {
    lo = 0;
    hi = g.nu - 1;
    const float l00 = g.dso - X0 * cth - Y0 * sth, l01 = g.dso - X0 * cth - Y1 * sth;
    const float l10 = g.dso - X1 * cth - Y0 * sth, l11 = g.dso - X1 * cth - Y1 * sth;
    const float lmin = fminf(fminf(l00, l01), fminf(l10, l11));
    if (g.full_footprint && !(lmin > 0.f)) return;
    const float lx0 = -X0 * sth, lx1 = -X1 * sth, ly0 = Y0 * cth, ly1 = Y1 * cth;
    const float u00 = (lx0 + ly0) / l00, u01 = (lx0 + ly1) / l01;
    const float u10 = (lx1 + ly0) / l10, u11 = (lx1 + ly1) / l11;
    const float umin = fminf(fminf(u00, u01), fminf(u10, u11)) * g.dsd;
    const float umax = fmaxf(fmaxf(u00, u01), fmaxf(u10, u11)) * g.dsd;
    const float off = 0.5f * g.nu - 0.5f;
    constexpr float eps = 1e-3f;
    lo = max(0, (int)ceilf((umin - g.off_u) / g.pu + off - eps));
    hi = min(g.nu - 1, (int)floorf((umax - g.off_u) / g.pu + off + eps));
}

// ----------------------------------------------------------------------------
// Adjoint, brick-owned exact transpose.
//
// Each warp owns a brick of BX x BY voxel columns x bz slabs, accumulated in
// shared memory; the 4 warps of a CTA own 4 bricks stacked in z over the same
// voxel columns, so they share the detector-column footprint and the xy walks.
// For every angle the CTA takes the footprint columns in batches of 4: warp w
// replays the forward's xy walk of column (batch + w) through the brick
// (segment list in shared memory), then every warp deposits the rows that
// cross its own slabs: C rows per lane, rows of one pass S apart so that no
// two lanes can touch the same voxel (S * dkz_min > 1 + span_max, derived on
// the host).  Each deposit is len * F * y of one ray-voxel piece —
// the same segment endpoints the forward computes.  Every voxel is owned by
// one warp and its contributions are added in a fixed (angle, column, pass,
// row group, segment, piece) order: deterministic, no atomics, exactly A^T.
// ----------------------------------------------------------------------------
// Brick shape: 5x5 voxel columns (x 64-slab pairs with the warp-specialised
// z-mirror kernel; measured against 4x4, 6x5, 6x6, 8x4, 4x8 at c1-c5,
// DESIGN.md §3).  The slab-lane condition bounds the xy size: a row's z-span
// over the brick's chord must stay below the row spacing (c4: 6x6 is the
// largest square that passes, 7x6 fails at c3).
#ifndef KCT_BX
#define KCT_BX 5
#define KCT_BY 5
#endif
#ifndef KCT_ADJ_WARPS
#define KCT_ADJ_WARPS 1  // one-warp CTAs: the warp's shared-memory base is CTA-uniform (uniform registers)
#endif
constexpr int BX = KCT_BX, BY = KCT_BY;
constexpr int kAdjWarps = KCT_ADJ_WARPS;
constexpr int kMaxSeg = 16;  // (BX - 1) + (BY - 1) interior crossings + 1 (+ slack)
constexpr int kMaxBz = 512 * 16 / (BX * BY);  // brick smem stays below 227 KB per CTA

struct __align__(16) Seg {
    float wa, wb;
    int ij;  // (i - I0) + BX * (j - J0)
    int pad;
};

}  // namespace

struct BrickCfg {
    int bz;  // slabs per brick (<= kMaxBz)
    int S;   // row stride of a pass
    int nbx, nby, nbz;
    int ngrp;      // angle groups: work item = (brick, group of the batch's angles)
    int slab;      // slab-lane deposits (brick_rows_slab): 0 off, 1 on, 2 on with slot-conflict detection
    size_t gstride;  // floats between the partial volumes of groups 1.. (group 0 -> out)
    int out_ref;     // 1: write `out` in the reference layout (x fastest) ...
    unsigned* level_done;  // ... and count finished bricks per (z level, y part) (adjoint_host_ref)
    int nparts;            // y parts per z level of those counters (brick row bj -> bj * nparts / nby)
    int mirror;      // 1: z-mirror brick pairs (adj_mirror_kernel): bricks tile the lower half
                     //    z < 0 (slabs [0, nz/2)), rows iv < nv/2
};

namespace {

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float lds_f(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f(unsigned a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
}
__device__ __forceinline__ float4 lds_f4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f4(unsigned a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ void sts_f2(unsigned a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y));
}

// z state of one detector row inside a brick: the forward's per-ray state
// (k0, f0, imk) restricted to the brick's slab planes [K0, kend].  wz is the
// next z-plane crossing, wz2 the one after it when that lies beyond the
// entry's chord (then the row crosses at most once more inside the entry and
// the crossing takes the short path), else -inf (general path).
struct RowZ {
    int k, kstep, k0;
    float f0, imk, wz, wz2, yf;
};

// The per-(angle, column) values the row z-state needs (a ColParams subset;
// carried in the walk-table entries so the adjoint never loads ColParams).
struct RowCol {
    float w_in, inv_h1;
    double g_in;
};
__device__ __forceinline__ RowCol row_col(const ColParams& cp) {
    RowCol r;
    r.w_in = cp.w_in;
    r.inv_h1 = cp.inv_h1;
    r.g_in = cp.g_in;
    return r;
}

// Per-ray adjoint record, written once per application by adj_weight_kernel
// (native layout, one float4 per ray): x = y * sqrt(1 + (dv inv_l)^2) (the
// forward's 3D length factor), y = f0, z = imk, w = bits of 4 k0 + kstep + 1
// — the forward's z state of the ray (fwd_kernel: k0, f0, imk), so the
// per-(row, brick) set-up is one 16-byte load instead of a float64 split.
__device__ __forceinline__ void row_init(RowZ& r, bool on, int iv, float w_in, float lo, float hi,
                                         float h1, int K0, int kend,
                                         const float4* __restrict__ rec, const DevGeom& g) {
    if (!on) {
        r.k = K0 - 1;
        r.kstep = 0;
        r.k0 = 0;
        r.f0 = 0.f;
        r.imk = 0.f;
        r.wz = kInf;
        r.wz2 = kInf;
        r.yf = 0.f;
        return;
    }
    const float4 q = __ldg(rec + iv);
    r.yf = q.x;
    r.f0 = q.y;
    r.imk = q.z;
    const int code = __float_as_int(q.w);
    const int k0 = code >> 2, sg = (code & 3) - 1;
    r.k0 = k0;
    r.kstep = sg;
    // slab at lo: last plane crossed strictly before lo (forward semantics);
    // the float estimate (dv from the row index) is corrected with the exact
    // crossing expression
    const float dvh = __fmul_rn(__fmaf_rn((float)iv, g.pv, g.dv0), h1);
    int k = k0 + __float2int_rd(__fmaf_rn(lo - w_in, dvh, r.f0));
    if (sg == 0) {
        r.wz = kInf;
        r.wz2 = kInf;
        r.k = min(max(k0, K0 - 1), kend);
        return;
    }
    // the ray's slab at w_in: k0, or k0 - 1 for a z-mirror record (f0 <= 0,
    // adj_weight_kernel); the walk never returns behind it
    const int kin = r.f0 < 0.f ? k0 - 1 : k0;
    k = sg > 0 ? max(k, kin) : min(k, kin);
    int pn = sg > 0 ? k + 1 : k;      // next plane
    const int pp = sg > 0 ? k : k + 1;  // plane crossed entering slab k
    float zn = zcross(pn, k0, r.f0, r.imk, w_in);
    const float zp = k != kin ? zcross(pp, k0, r.f0, r.imk, w_in) : -kInf;
    if (!(zp < lo && !(zn < lo))) {
        // z(lo) within rounding of a plane: search
        if (sg > 0) {
            while (k > kin && !(zcross(k, k0, r.f0, r.imk, w_in) < lo)) --k;
            while (zcross(k + 1, k0, r.f0, r.imk, w_in) < lo) ++k;
            pn = k + 1;
        } else {
            while (k < k0 && !(zcross(k + 1, k0, r.f0, r.imk, w_in) < lo)) ++k;
            while (zcross(k, k0, r.f0, r.imk, w_in) < lo) --k;
            pn = k;
        }
        zn = zcross(pn, k0, r.f0, r.imk, w_in);
    }
    // rows entering the brick from below / above start in a guard slab and
    // cross the brick's first plane next
    const int kc = sg > 0 ? max(k, K0 - 1) : min(k, kend);
    const int pc = sg > 0 ? kc + 1 : kc;
    r.wz = (pc >= K0 && pc <= kend) ? (kc == k ? zn : zcross(pc, k0, r.f0, r.imk, w_in)) : kInf;
    const int pc2 = pc + sg;
    const float z2 = (pc >= K0 && pc <= kend && pc2 >= K0 && pc2 <= kend)
                         ? zcross(pc2, k0, r.f0, r.imk, w_in)
                         : kInf;
    r.wz2 = z2 < hi ? -kInf : z2;
    r.k = min(max(kc, K0 - 1), kend);
}

// Deposit one row's pieces of one xy segment: [wa, min(wb, wz)] into slab k,
// then (rarely) the pieces after each z-plane crossing inside the segment.
// r.k stays within [K0 - 1, kend]; the two guard slabs of every column
// (K0 - 1 and kend) absorb the pieces outside the brick, so no range checks.
__device__ __forceinline__ void row_segment(RowZ& r, const Seg& sg, unsigned colbase, int K0,
                                            int kend, float w_in) {
    const bool cr = r.wz < sg.wb;
    const float wm = cr ? r.wz : sg.wb;
    const unsigned a = colbase + 4u * (unsigned)r.k;
    sts_f(a, __fmaf_rn(wm - sg.wa, r.yf, lds_f(a)));
    if (cr) {
        if (!(r.wz2 < sg.wb)) {
            // the row's last crossing inside this entry: [wz, wb] into the
            // next slab (the general path below computes the same values:
            // the next crossing wz2 lies beyond wb)
            r.k += r.kstep;
            const unsigned b = colbase + 4u * (unsigned)r.k;
            sts_f(b, __fmaf_rn(sg.wb - r.wz, r.yf, lds_f(b)));
            r.wz = r.wz2;
        } else {
            float wa = r.wz;
            for (;;) {
                r.k += r.kstep;
                const int P = r.kstep > 0 ? r.k + 1 : r.k;
                r.wz = (P >= K0 && P <= kend) ? zcross(P, r.k0, r.f0, r.imk, w_in) : kInf;
                const float we = fminf(r.wz, sg.wb);
                const unsigned b = colbase + 4u * (unsigned)r.k;
                sts_f(b, __fmaf_rn(we - wa, r.yf, lds_f(b)));
                if (!(r.wz < sg.wb)) break;
                wa = r.wz;
            }
        }
    }
}

// ---- the xy part of one (brick, detector column): chord, row range, walk ----
// Fills bnd[0..nseg] (segment boundaries, shared memory) and, for lanes
// < nseg, the segment's voxel column `ij` = (i - I0) + BX (j - J0).  Returns
// nseg, 0 when the column's rays miss the brick.  Used on the fly by the
// adjoint and by the walk-table builder (bit-identical entries).
struct BrickGeo {
    int I0, J0, K0, bxn, byn, bzn;
    int rmax;  // last detector row that can cross the brick (z-mirror pairs: nv/2 - 1)
};

__device__ __forceinline__ int brick_walk(const ColParams& cp, const DevGeom& g, const BrickGeo& B,
                                          int lane, float* bnd, int* axis, float& lo_out,
                                          int& rlo_out, int& rhi_out, int& ij_out) {
    const int I0 = B.I0, J0 = B.J0, bxn = B.bxn, byn = B.byn;
    // chord of the column's xy line through the brick
    float lo = cp.w_in, hi = cp.w_out;
    if (cp.dx != 0.0) {
        const float e0 = xcross(cp, I0), e1 = xcross(cp, I0 + bxn);
        lo = fmaxf(lo, fminf(e0, e1));
        hi = fminf(hi, fmaxf(e0, e1));
    } else if (cp.i0 < I0 || cp.i0 >= I0 + bxn) {
        return 0;
    }
    if (cp.dy != 0.0) {
        const float e0 = ycross(cp, J0), e1 = ycross(cp, J0 + byn);
        lo = fmaxf(lo, fminf(e0, e1));
        hi = fminf(hi, fmaxf(e0, e1));
    } else if (cp.j0 < J0 || cp.j0 >= J0 + byn) {
        return 0;
    }
    if (!(lo < hi)) return 0;
    // rows whose z-span over [lo, hi] meets slabs [K0, K0 + bzn]
    // (approximate reciprocals: the row range carries a 1e-3-row margin >>
    // their 2^-22 relative error)
    const float h1 = rcp_approx(cp.inv_h1);
    const float gin = (float)cp.g_in;
    const float Glo = gin + (lo - cp.w_in) * h1, Ghi = gin + (hi - cp.w_in) * h1;
    const float rGlo = rcp_approx(Glo), rGhi = rcp_approx(Ghi);
    const float n0 = (float)B.K0 + g.kz0, n1 = n0 + (float)B.bzn;
    const float dlo = n0 * (n0 >= 0.f ? rGhi : rGlo);
    const float dhi = n1 * (n1 >= 0.f ? rGlo : rGhi);
    const float rpv = 1.f / g.pv;
    const int rlo = max(0, (int)ceilf((dlo - g.dv0) * rpv - 1e-3f));
    const int rhi = min(B.rmax, (int)floorf((dhi - g.dv0) * rpv + 1e-3f));
    if (rlo > rhi) return 0;

    // lane-parallel walk: lanes 0..7 take the interior x planes, 8..15 the y planes
    const bool xl = lane < 8;
    const int pl = xl ? lane : lane - 8;
    const unsigned below = (1u << lane) - 1u;
    float v = kInf;
    bool has = false;
    if (xl && pl < bxn - 1 && cp.dx != 0.0) {
        v = xcross(cp, I0 + 1 + pl);
        has = true;
    } else if (!xl && lane < 16 && pl < byn - 1 && cp.dy != 0.0) {
        v = ycross(cp, J0 + 1 + pl);
        has = true;
    }
    const unsigned mbefore = __ballot_sync(kFull, has && v <= lo);
    const bool valid = has && v > lo && v < hi;
    const unsigned mval = __ballot_sync(kFull, valid);
    const int cbx = __popc(mbefore & 0xffu), cby = __popc(mbefore & 0xff00u);
    const int stx = cp.dx > 0.0 ? 1 : -1, sty = cp.dy > 0.0 ? 1 : -1;
    const int ie = cp.dx == 0.0 ? cp.i0 : (stx > 0 ? I0 + cbx : I0 + bxn - 1 - cbx);
    const int je = cp.dy == 0.0 ? cp.j0 : (sty > 0 ? J0 + cby : J0 + byn - 1 - cby);
    // rank along the ray: own-axis predecessors (plane order) + other-axis
    // crossings before it (x first at ties, as the forward's walk)
    const unsigned own = xl ? (mval & 0xffu) : (mval & 0xff00u);
    int rank = (xl ? stx : sty) > 0 ? __popc(own & below) : __popc(own & ~below & ~(1u << lane));
    const unsigned other = xl ? (mval >> 8) & 0xffu : mval & 0xffu;
#pragma unroll
    for (int t = 0; t < (BX > BY ? BX : BY) - 1; ++t) {
        const float ov = __shfl_sync(kFull, v, xl ? 8 + t : t);
        rank += (((other >> t) & 1u) && (xl ? ov < v : ov <= v)) ? 1 : 0;
    }
    const int nval = __popc(mval);
    if (valid) {
        bnd[rank + 1] = v;
        axis[rank] = xl ? 1 : 0;
    }
    if (lane == 0) {
        bnd[0] = lo;
        bnd[nval + 1] = hi;
    }
    __syncwarp();
    const unsigned mx = __ballot_sync(kFull, lane < nval && axis[lane]);
    const int nxb = __popc(mx & below);
    ij_out = (ie + stx * nxb - I0) + BX * (je + sty * (lane - nxb) - J0);
    lo_out = lo;
    rlo_out = rlo;
    rhi_out = rhi;
    return nval + 1;
}

// ---- the rows of one (brick, detector column) ----
// The n rows go in Sp = max(S, ceil(n / 32)) residue classes of rows Sp apart
// (one lane per row: no two lanes of a class touch the same voxel, since
// Sp * dkz_min > 1 + span_max), two classes at a time: lane l takes rows
// base + Sp l (c = 0) and base + 1 + Sp l (c = 1), deposited by separate
// warp-converged instructions (__syncwarp between them), so only the rows of
// one class need the spacing.  An odd last class runs alone.
template <int C>
__device__ __forceinline__ void row_chunks(const Seg* segs, int nseg, const RowCol& cp, float lo,
                                           float hi, float h1, int base, int rhi, int Sp, int K0,
                                           int kend, int lane, const float4* __restrict__ rec,
                                           const DevGeom& g) {
    RowZ r[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int iv = base + c + Sp * lane;
        row_init(r[c], iv <= rhi, iv, cp.w_in, lo, hi, h1, K0, kend, rec, g);
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
        const Seg sg = segs[sgi];
        row_segment(r[0], sg, (unsigned)sg.ij, K0, kend, cp.w_in);
        if (C == 2) {
            __syncwarp();
            row_segment(r[C - 1], sg, (unsigned)sg.ij, K0, kend, cp.w_in);
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void brick_rows(const Seg* segs, int nseg, const RowCol& cp, float lo,
                                           int rlo, int rhi, int S, int K0, int kend, int lane,
                                           const float4* __restrict__ rec, const DevGeom& g) {
    const float h1 = rcp_approx(cp.inv_h1);
    const float hi = segs[nseg - 1].wb;
    const int Sp = max(S, (rhi - rlo + 32) >> 5);
    int q = 0;
    for (; q + 1 < Sp; q += 2)
        row_chunks<2>(segs, nseg, cp, lo, hi, h1, rlo + q, rhi, Sp, K0, kend, lane, rec, g);
    if (q < Sp) row_chunks<1>(segs, nseg, cp, lo, hi, h1, rlo + q, rhi, Sp, K0, kend, lane, rec, g);
}

// ---- slab-lane deposits (the common case) ----
// When a row's z-span over a brick chord is below one slab and below the row
// spacing, and rows two apart are more than one slab apart (host-checked:
// Projector::adj_slab_), every row of an entry either stays in one slab over
// the whole chord ("simple") or crosses exactly one z-plane, and a slab is
// left / entered by at most one row.  The rows of the entry are classified
// once (lanes = consecutive rows) into per-slab tables — H[k]: the sum of the
// simple rows' weights, Xb[k]: (crossing, weight) of the row leaving slab k,
// Xa[k]: the row entering it — and the deposits run with lanes = slabs:
//   acc[ij][k] += (wb - wa) H[k] + (clamp(Xb.w) - wa) Xb.y + (wb - clamp(Xa.w)) Xa.y
// with clamp(w) = min(max(w, wa), wb): per segment exactly the forward's piece
// lengths ([wa, wz] / [wz, wb] in the crossing segment, 0 or wb - wa
// elsewhere).  Each row's crossing is the forward's zcross of one of the two
// planes bounding its slab at the chord's midpoint.  A detected slot conflict
// (not expected under the host condition) returns false and the entry takes
// the row-wise path.  Fixed summation order: deterministic.
constexpr int kSlabChunks = 4;  // slab table slots (bz + 2) <= 32 * kSlabChunks

// floats of one warp's shared memory in adj_brick_kernel (16-byte multiple)
// (the accumulators padded to a 16-byte multiple: Seg / float4 tables follow)
__host__ __device__ constexpr int adj_acc_floats(int bz) { return (BX * BY * (bz + 2) + 3) & ~3; }
__host__ __device__ constexpr int adj_warp_floats(int bz) {
    return (adj_acc_floats(bz) + 4 * kMaxSeg + 2 * (kMaxSeg + 2) + 5 * (bz + 2) + 3) & ~3;
}

// Row classification of one entry into the slab tables: tH[j] = H (4 B),
// tX[j] = {Xb.w, Xb.y, Xa.w, Xa.y} (16 B), slot j = slab K0 - 1 + j, j < NS;
// all-zero on entry (cleared by slab_deposits).  Simple rows add
// their weight to H; a crossing row leaving slab kb / entering ka at wc
// writes Xb[kb] and Xa[ka] (one writer per slot: row z-intervals are
// disjoint).  Returns false when two rows could claim one slot (only
// possible for a falling and a rising row around dv = 0 when the row spacing
// can reach one slab: detect = true).
__device__ __forceinline__ bool slab_classify(const float4* __restrict__ p, float4 q, int nrows,
                                              int rlo, float lo, float hi, float w_in, float h1,
                                              int K0, int NS, int lane, bool detect,
                                              const DevGeom& g, unsigned tH, unsigned tX) {
    const float mid = 0.5f * (lo + hi) - w_in;
    const unsigned tH0 = tH + 4u * (unsigned)(1 - K0), tX0 = tX + 16u * (unsigned)(1 - K0);
    const int km = K0 - 1;
    p += lane;
    float ivf = (float)(rlo + lane);
    bool bad = false;
    unsigned prev_fall = 0u;
    for (int b = lane; b < nrows + lane; b += 32) {
        const float4 qc = q;
        p += 32;
        if (b + 32 < nrows) q = __ldg(p);  // next chunk
        const bool valid = b < nrows;
        const int code = __float_as_int(qc.w);
        const int k0 = code >> 2, ks = (code & 3) - 1;
        const float dvh = __fmul_rn(__fmaf_rn(ivf, g.pv, g.dv0), h1);
        ivf += 32.f;
        int k = k0 + __float2int_rd(__fmaf_rn(mid, dvh, qc.y));
        k = ks != 0 ? k : k0;
        const float z1 = zcross(k, k0, qc.y, qc.z, w_in);
        const float z2 = zcross(k + 1, k0, qc.y, qc.z, w_in);
        const float wen = fminf(z1, z2), wlv = fmaxf(z1, z2);
        const bool enter = ks != 0 && wen > lo;
        const bool leave = ks != 0 && wlv < hi;
        const bool cx = valid && (enter || leave);
        const float yf = qc.x;
        // H: rows two apart never share a slab; two parity passes (a run of
        // two rows adds in the same order either way: 0 + a + b)
        const bool hw = valid && !cx && (unsigned)(k - km) < (unsigned)NS;
        const unsigned ha = tH0 + 4u * (unsigned)k;
        if (hw && !(lane & 1)) sts_f(ha, lds_f(ha) + yf);
        __syncwarp();
        if (hw && (lane & 1)) sts_f(ha, lds_f(ha) + yf);
        if (cx) {
            const int kb = enter ? k - ks : k, ka = enter ? k : k + ks;
            const float wc = enter ? wen : wlv;
            if ((unsigned)(kb - km) < (unsigned)NS) sts_f2(tX0 + 16u * (unsigned)kb, make_float2(wc, yf));
            if ((unsigned)(ka - km) < (unsigned)NS) sts_f2(tX0 + 16u * (unsigned)ka + 8u, make_float2(wc, yf));
        }
        if (detect) {
            const unsigned fall = __ballot_sync(kFull, cx && ks < 0);
            const unsigned pf = ((fall << 1) | prev_fall) >> lane;
            bad |= cx && ks > 0 && (pf & 1u);
            prev_fall = fall >> 31;
        }
        __syncwarp();
    }
    return !(detect && __any_sync(kFull, bad));
}

// Deposits of one entry with lanes = slabs (slot j = lane + 32 r; slots past
// the brick deposit 0 into the upper guard slab); clears the tables.
template <int RC>
__device__ __forceinline__ void slab_deposits(const Seg* segs, int nseg, int K0, int NS, int lane,
                                              unsigned tH, unsigned tX) {
    float H[RC], bw[RC], by[RC], aw[RC], ay[RC];
    unsigned off[RC];
    bool xs[RC];
#pragma unroll
    for (int r = 0; r < RC; ++r) {
        const int j = lane + 32 * r;
        float h = 0.f;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < NS) {
            h = lds_f(tH + 4u * j);
            x = lds_f4(tX + 16u * j);
            sts_f(tH + 4u * j, 0.f);
            sts_f4(tX + 16u * j, make_float4(0.f, 0.f, 0.f, 0.f));
        }
        H[r] = h;
        bw[r] = x.x;
        by[r] = x.y;
        aw[r] = x.z;
        ay[r] = x.w;
        off[r] = 4u * (unsigned)(K0 - 1 + min(j, NS - 1));
        xs[r] = __any_sync(kFull, x.y != 0.f || x.w != 0.f);
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
        const Seg sg = segs[sgi];
        const float d = sg.wb - sg.wa;
        // the chunks' slabs are distinct: all loads first, then the stores
        float v[RC];
#pragma unroll
        for (int r = 0; r < RC; ++r) v[r] = lds_f((unsigned)sg.ij + off[r]);
#pragma unroll
        for (int r = 0; r < RC; ++r) {
            float dep;
            if (xs[r]) {
                const float cb = fminf(fmaxf(bw[r], sg.wa), sg.wb);
                const float ca = fminf(fmaxf(aw[r], sg.wa), sg.wb);
                dep = __fmaf_rn(d, H[r], __fmaf_rn(cb - sg.wa, by[r], (sg.wb - ca) * ay[r]));
            } else {
                dep = __fmul_rn(d, H[r]);
            }
            v[r] += dep;
        }
#pragma unroll
        for (int r = 0; r < RC; ++r) sts_f((unsigned)sg.ij + off[r], v[r]);
    }
    __syncwarp();
}

// The slab-lane path for one entry (q: the first row chunk's records,
// prefetched by the caller); false: take the row-wise path (the tables are
// left clean either way).
__device__ __forceinline__ bool brick_rows_slab(const Seg* segs, int nseg, float w_in, float inv_h1,
                                                float lo, float hi, int rlo, int rhi, int K0,
                                                int kend, int lane, bool detect,
                                                const float4* __restrict__ rec, float4 q,
                                                const DevGeom& g, unsigned tH, unsigned tX) {
    const int NS = kend - K0 + 2;
    if (!slab_classify(rec + rlo, q, rhi - rlo + 1, rlo, lo, hi, w_in, rcp_approx(inv_h1), K0, NS,
                       lane, detect, g, tH, tX)) {
        for (int j = lane; j < NS; j += 32) {
            sts_f(tH + 4u * j, 0.f);
            sts_f4(tX + 16u * j, make_float4(0.f, 0.f, 0.f, 0.f));
        }
        __syncwarp();
        return false;
    }
    switch ((NS + 31) >> 5) {
    case 1: slab_deposits<1>(segs, nseg, K0, NS, lane, tH, tX); break;
    case 2: slab_deposits<2>(segs, nseg, K0, NS, lane, tH, tX); break;
    case 3: slab_deposits<3>(segs, nseg, K0, NS, lane, tH, tX); break;
    default: slab_deposits<4>(segs, nseg, K0, NS, lane, tH, tX); break;
    }
    return true;
}

// ---- walk table: the xy part of every (brick, angle, column), built once per
// projector (geometry-only) and streamed by the adjoint instead of recomputed
// for every application.  64 bytes per entry. ----
// kEW 32-bit words per entry: segment boundaries (kNB words), segment voxel
// columns (one byte each, kNB / 4 words; the last byte holds nseg), then
// angle | column << 16, rlo | rhi << 16, and the RowCol values.  64 bytes for
// bricks with <= 7 segments (4x4), 128 bytes for <= 15 (8x4, 8x8).
constexpr int kEW = BX + BY - 1 <= 7 ? 16 : 32;
constexpr int kNB = kEW / 2;
constexpr int kTabMaxSeg = kNB - 1;
struct alignas(4 * kEW) WalkEntry {
    float bnd[kNB];          // segment boundaries, lo = bnd[0] .. hi = bnd[nseg]
    unsigned char ij[kNB];   // per segment: (i - I0) + BX (j - J0); ij[kNB - 1] = nseg
    unsigned roff;           // first ray of the column: (angle * nu + column) * nv (global)
    unsigned short rlo, rhi; // detector rows crossing the brick
    RowCol rc;               // the column's row z-state inputs
};
static_assert(sizeof(WalkEntry) == 4 * kEW, "WalkEntry layout");
constexpr bool kTabOk = BX + BY - 1 <= kTabMaxSeg && BX * BY <= 256;

__device__ __forceinline__ BrickGeo brick_geo(int brick, const BrickCfg& bc, const DevGeom& g) {
    const int bi = brick % bc.nbx, bj = (brick / bc.nbx) % bc.nby, bk = brick / (bc.nbx * bc.nby);
    BrickGeo B;
    B.I0 = bi * BX;
    B.J0 = bj * BY;
    B.K0 = bk * bc.bz;
    B.bxn = min(BX, g.nx - B.I0);
    B.byn = min(BY, g.ny - B.J0);
    B.bzn = min(bc.bz, (bc.mirror ? g.nz / 2 : g.nz) - B.K0);
    B.rmax = bc.mirror ? g.nv / 2 - 1 : g.nv - 1;
    return B;
}

// counter of a finished brick in adjoint_host_ref: (z level, y part)
__device__ __forceinline__ int progress_slot(int brick, const BrickCfg& bc) {
    const int plane = bc.nbx * bc.nby, bj = (brick / bc.nbx) % bc.nby;
    return (brick / plane) * bc.nparts + bj * bc.nparts / bc.nby;
}

// FILL = false: count entries per (brick, angle) into off[b (na + 1) + a];
// FILL = true: write them from off[] (exclusive prefix sums).  One warp per brick.
template <bool FILL>
__global__ void __launch_bounds__(128) adj_walk_build(const ColParams* __restrict__ cols,
                                                      const float2* __restrict__ cs, DevGeom g,
                                                      BrickCfg bc,
                                                      unsigned long long* __restrict__ off,
                                                      WalkEntry* __restrict__ tab) {
    __shared__ float sbnd[4][kMaxSeg + 2];
    __shared__ int saxis[4][kMaxSeg + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int brick = blockIdx.x * 4 + warp;
    if (brick >= bc.nbx * bc.nby * bc.nbz) return;
    const BrickGeo B = brick_geo(brick, bc, g);
    const float X0 = g.ox + B.I0 * g.sx, X1 = g.ox + (B.I0 + B.bxn) * g.sx;
    const float Y0 = g.oy + B.J0 * g.sy, Y1 = g.oy + (B.J0 + B.byn) * g.sy;
    unsigned long long* ob = off + (size_t)brick * (g.na + 1);
    for (int ia = 0; ia < g.na; ++ia) {
        int iu_lo, iu_hi;
        footprint(g, cs[ia].x, cs[ia].y, X0, X1, Y0, Y1, iu_lo, iu_hi);
        unsigned long long e = FILL ? ob[ia] : 0ull;
        for (int iu = iu_lo; iu <= iu_hi; ++iu) {
            const ColParams cp = cols[(size_t)ia * g.nu + iu];
            float lo;
            int rlo, rhi, ij;
            const int nseg = brick_walk(cp, g, B, lane, sbnd[warp], saxis[warp], lo, rlo, rhi, ij);
            if (nseg == 0) continue;
            if (FILL) {
                WalkEntry* E = tab + e;
                if (lane <= nseg) E->bnd[lane] = sbnd[warp][lane];
                if (lane < nseg) E->ij[lane] = (unsigned char)ij;
                if (lane == 0) {
                    E->ij[kNB - 1] = (unsigned char)nseg;
                    E->roff = ((unsigned)ia * (unsigned)g.nu + (unsigned)iu) * (unsigned)g.nv;
                    E->rlo = (unsigned short)rlo;
                    E->rhi = (unsigned short)rhi;
                    E->rc = row_col(cp);
                }
            }
            ++e;
            __syncwarp();
        }
        if (!FILL && lane == 0) ob[ia] = e;
    }
}

#ifndef KCT_ADJ_MINB
#define KCT_ADJ_MINB (22 / KCT_ADJ_WARPS)  // register target 93 (80 used; measured 1.5% faster than 24 / 85)
#endif
// TAB: the xy walks come from the walk table (tab, off) instead of being
// recomputed; identical values either way.
template <bool TAB>
__global__ void __launch_bounds__(kAdjWarps * 32, KCT_ADJ_MINB) adj_brick_kernel(
    const float4* __restrict__ rec, float* __restrict__ out, const ColParams* __restrict__ cols,
    DevGeom g, BrickCfg bc, const float2* __restrict__ csb, int a0, int nab, int accumulate,
    const int* __restrict__ order, int* queue, float* __restrict__ out_part,
    const WalkEntry* __restrict__ tab, const unsigned long long* __restrict__ off) {
    extern __shared__ float sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nbricks = bc.nbx * bc.nby * bc.nbz;
    const int BZ = bc.bz;
    const int nu = g.nu, nv = g.nv;
    // per-warp shared layout (adj_warp_floats): acc[BX*BY][BZ + 2] (slab k at
    // k - K0 + 1; two guard slabs) | segs[kMaxSeg] | bnd[kMaxSeg + 2] |
    // axis[kMaxSeg + 2] | slab tables tX[BZ + 2] (float4), tH[BZ + 2] (float)
    const int CS = BZ + 2;
    const int wfloats = adj_warp_floats(BZ);
    float* acc = sm + warp * wfloats;
    const int ACCF = adj_acc_floats(BZ);
    Seg* segs = reinterpret_cast<Seg*>(acc + ACCF);
    float* bnd = acc + ACCF + 4 * kMaxSeg;
    int* axis = reinterpret_cast<int*>(bnd + kMaxSeg + 2);
    const unsigned acc_s = (unsigned)__cvta_generic_to_shared(acc);
    const unsigned tX = acc_s + 4u * (unsigned)(ACCF + 4 * kMaxSeg + 2 * (kMaxSeg + 2));
    const unsigned tH = tX + 16u * (unsigned)CS;
    const int S = bc.S;

    // Bricks are handed out to warps by a queue (heaviest first, `order`), so
    // the uneven per-brick work does not leave a partial last wave; without a
    // queue every warp takes one brick.  Each brick is still computed by one
    // warp in a fixed order: the result does not depend on the schedule.
    // Small problems have too few bricks to fill the GPU: the angles of the
    // batch are then split into ngrp groups, group g accumulating into its own
    // partial volume (g = 0: `out`), summed in group order afterwards.
    const int nitems = nbricks * bc.ngrp;
    int ticket = queue ? 0 : blockIdx.x * kAdjWarps + warp;
    for (;;) {
    int item;
    if (queue) {
        int tk = 0;
        if (lane == 0) tk = atomicAdd(queue, 1);
        tk = __shfl_sync(kFull, tk, 0);
        if (tk >= nitems) break;
        item = tk;
    } else {
        if (ticket >= nitems) break;
        item = ticket;
        ticket = nitems;
    }
    const int grp = item % bc.ngrp;
    const int brick = queue ? order[item / bc.ngrp] : item / bc.ngrp;
    const int a_lo = (int)((long long)nab * grp / bc.ngrp);
    const int a_hi = (int)((long long)nab * (grp + 1) / bc.ngrp);
    float* const dst = grp == 0 ? out : out_part + (size_t)(grp - 1) * bc.gstride;
    const int acc_in = grp == 0 ? accumulate : 0;
    const BrickGeo B = brick_geo(brick, bc, g);
    const int K0 = B.K0, kend = B.K0 + B.bzn;
    for (int q = lane; q < BX * BY * CS; q += 32) acc[q] = 0.f;
    if (bc.slab)
        for (int j = lane; j < CS; j += 32) {
            sts_f(tH + 4u * j, 0.f);
            sts_f4(tX + 16u * j, make_float4(0.f, 0.f, 0.f, 0.f));
        }
    __syncwarp();
    // byte address of slab 0 of voxel column ij (so that slab k sits at + 4k)
    const unsigned seg_base = acc_s + 4u * (unsigned)(1 - K0);

    if (TAB) {
        const unsigned long long* ob = off + (size_t)brick * (g.na + 1);
        const unsigned long long e0 = ob[a0 + a_lo], e1 = ob[a0 + a_hi];
        const unsigned* tw = reinterpret_cast<const unsigned*>(tab);
        // lanes 0..kEW-1 hold one entry; two entries ahead are in flight, and
        // the next entry's first row chunk of records is fetched while the
        // current one's rows run
        constexpr int M = kNB + kNB / 4;  // first meta word
        auto ld_entry = [&](unsigned long long e) {
            return (e < e1 && lane < kEW) ? __ldg(tw + e * kEW + lane) : 0u;
        };
        // records of this angle batch start at ray a0 * nu * nv
        const unsigned boff = (unsigned)a0 * (unsigned)nu * (unsigned)nv;
        auto first_chunk = [&](unsigned we, unsigned long long e) {
            const unsigned ro = __shfl_sync(kFull, we, M), r = __shfl_sync(kFull, we, M + 1);
            const int rl = (int)(r & 0xffffu), n = (int)(r >> 16) - rl + 1;
            return (e < e1 && bc.slab && lane < n) ? __ldg(rec + (ro - boff + (unsigned)(rl + lane)))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        unsigned w = ld_entry(e0), w1 = ld_entry(e0 + 1);
        float4 q = first_chunk(w, e0);
        for (unsigned long long e = e0; e < e1; ++e) {
            const unsigned ijw1 = __shfl_sync(kFull, w, M - 1);
            const int nseg = (int)(ijw1 >> 24);
            const unsigned rr = __shfl_sync(kFull, w, M + 1);
            const float wa = __uint_as_float(__shfl_sync(kFull, w, lane & (kNB - 1)));
            const float wb = __uint_as_float(__shfl_sync(kFull, w, (lane + 1) & (kNB - 1)));
            const unsigned ijw = __shfl_sync(kFull, w, kNB + ((lane >> 2) & (kNB / 4 - 1)));
            const float lo = __uint_as_float(__shfl_sync(kFull, w, 0));
            const float hi = __uint_as_float(__shfl_sync(kFull, w, nseg & (kNB - 1)));
            const unsigned ro = __shfl_sync(kFull, w, M);
            const float w_in = __uint_as_float(__shfl_sync(kFull, w, M + 2));
            const float inv_h1 = __uint_as_float(__shfl_sync(kFull, w, M + 3));
            if (lane < nseg) {
                const unsigned ij = (ijw >> (8 * (lane & 3))) & 0xffu;
                Seg sg;
                sg.wa = wa;
                sg.wb = wb;
                sg.ij = (int)(seg_base + 4u * ij * (unsigned)CS);
                sg.pad = 0;
                segs[lane] = sg;
            }
            const unsigned w2 = ld_entry(e + 2);
            const float4 q1 = first_chunk(w1, e + 1);
            __syncwarp();
            const int rlo = (int)(rr & 0xffffu), rhi = (int)(rr >> 16);
            const float4* rc = rec + (ro - boff);
            if (!(bc.slab && brick_rows_slab(segs, nseg, w_in, inv_h1, lo, hi, rlo, rhi, K0, kend,
                                             lane, bc.slab > 1, rc, q, g, tH, tX))) {
                RowCol rcp;
                rcp.w_in = w_in;
                rcp.inv_h1 = inv_h1;
                rcp.g_in = __hiloint2double((int)__shfl_sync(kFull, w, M + 5),
                                            (int)__shfl_sync(kFull, w, M + 4));
                brick_rows(segs, nseg, rcp, lo, rlo, rhi, S, K0, kend, lane, rc, g);
            }
            __syncwarp();
            w = w1;
            w1 = w2;
            q = q1;
        }
    } else {
        const float X0 = g.ox + B.I0 * g.sx, X1 = g.ox + (B.I0 + B.bxn) * g.sx;
        const float Y0 = g.oy + B.J0 * g.sy, Y1 = g.oy + (B.J0 + B.byn) * g.sy;
        for (int ia = a_lo; ia < a_hi; ++ia) {
            int iu_lo, iu_hi;
            const float2 csa = __ldg(csb + ia);
            footprint(g, csa.x, csa.y, X0, X1, Y0, Y1, iu_lo, iu_hi);
            const ColParams* colp = cols + (size_t)ia * nu;
            const float4* yb = rec + (size_t)ia * nu * nv;
            for (int iu = iu_lo; iu <= iu_hi; ++iu) {
                const ColParams cp = colp[iu];
                float lo;
                int rlo, rhi, ij;
                const int nseg = brick_walk(cp, g, B, lane, bnd, axis, lo, rlo, rhi, ij);
                if (nseg == 0) continue;
                if (lane < nseg) {
                    Seg sg;
                    sg.wa = bnd[lane];
                    sg.wb = bnd[lane + 1];
                    sg.ij = (int)(seg_base + 4u * (unsigned)(ij * CS));
                    sg.pad = 0;
                    segs[lane] = sg;
                }
                __syncwarp();
                const RowCol rcp = row_col(cp);
                const float4* ry = yb + (size_t)iu * nv;
                const float4 q = lane <= rhi - rlo ? __ldg(ry + rlo + lane)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                if (!(bc.slab && brick_rows_slab(segs, nseg, cp.w_in, cp.inv_h1, lo, bnd[nseg],
                                                 rlo, rhi, K0, kend, lane, bc.slab > 1, ry, q, g,
                                                 tH, tX)))
                    brick_rows(segs, nseg, rcp, lo, rlo, rhi, S, K0, kend, lane,
                               yb + (size_t)iu * nv, g);
                __syncwarp();
            }
        }
    }
    if (!bc.out_ref) {
        // write the brick (coalesced runs of bzn slabs per voxel column)
        for (int c = 0; c < B.bxn * B.byn; ++c) {
            const int ci = c % B.bxn, cj = c / B.bxn;
            float* o = dst + ((size_t)(B.I0 + ci) + (size_t)g.nx * (B.J0 + cj)) * g.nz + K0;
            const float* a = acc + (ci + BX * cj) * CS + 1;
            for (int kk = lane; kk < B.bzn; kk += 32) o[kk] = acc_in ? o[kk] + a[kk] : a[kk];
        }
        __syncwarp();
    } else {
        // reference layout (x fastest): lanes over the brick's voxel columns
        // (runs of BX floats in x), then slabs; the z level's counter tells
        // the host copy stream when the level's slabs are final
        const int ncol = BX * BY;
        for (int t = lane; t < ncol * B.bzn; t += 32) {
            const int c = t % ncol, kk = t / ncol;
            const int ci = c % BX, cj = c / BX;
            if (ci < B.bxn && cj < B.byn) {
                float* o = dst + (size_t)(B.I0 + ci) +
                           (size_t)g.nx * ((size_t)(B.J0 + cj) + (size_t)g.ny * (K0 + kk));
                *o = acc_in ? *o + acc[c * CS + 1 + kk] : acc[c * CS + 1 + kk];
            }
        }
        if (bc.level_done) {
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(bc.level_done + progress_slot(brick, bc), 1u);
        }
    }
    }
}

// ----------------------------------------------------------------------------
// Adjoint, z-mirror brick pairs (the path every BASELINE geometry takes).
//
// In a z-mirror geometry (DevGeom::mirror, fwd_kernel MIR: offset_v = 0, nv
// even, grid centred in z, here also nz even) detector row nv-1-iv is the
// reflection of row iv in the plane z = 0 and slab nz-1-k that of slab k; the
// mirror ray crosses plane nz-P exactly where the primary crosses plane P (the
// same float values).  A work item is a pair of bricks: L = an xy brick's
// voxel columns x slabs [K0, K0 + bzn) of the lower half (z < 0) and its
// reflection U = slabs [nz - K0 - bzn, nz - K0).  Only primary rows (dv < 0,
// iv < nv/2) cross L and exactly their mirrors cross U, so one classification
// of the primary rows (slab_classify's, ks = -1) serves both bricks — each
// slab slot holds the primary's and the mirror's weight — and one pass of the
// slab lanes over the segments updates both bricks (U kept with its slabs in
// slot order: slot j = slab nz-1-(K0 + j)).  Deposits are slab_deposits'
// expressions in the same order: per voxel the result is the brick kernel's.
// Per (entry, row) the fixed and the classification work are shared by two
// rays; slots are the brick's own slabs (no guard slabs: a simple row outside
// the brick deposits nothing into it).
// Shared memory per warp (floats): accL[BX*BY][bz] | accU[BX*BY][bz] |
// segs[kMaxSeg] (float4: wa, wb, L column index) | tX[bz + 1] (float4:
// crossing w, primary weight, mirror weight, 0 of the row leaving slot j
// downwards, i.e. entering slot j - 1: primary rows all fall) | tH[bz] (float2).
// ----------------------------------------------------------------------------
constexpr int kMirMaxBz = 32 * kSlabChunks;
__host__ __device__ constexpr int adj_mir_floats(int bz) {
    return 2 * BX * BY * ((bz + 1) & ~1) + 4 * kMaxSeg + 4 * (((bz + 1) & ~1) + 2) + 2 * ((bz + 1) & ~1);
}

// Classification of the primary rows rlo.. (nrows; records p and the
// mirrors' weights pm, both from row rlo on) into the
// slot tables; q / ym: the first chunk's record and mirror weight.  Slot j =
// slab K0 + j, j < NS; tables all-zero on entry.
__device__ __forceinline__ void mir_classify(const float4* __restrict__ p,
                                             const float* __restrict__ pm, float4 q, float ym,
                                             int nrows, int rlo, float lo, float hi, float w_in,
                                             float h1, int K0, int NS, int lane, const DevGeom& g,
                                             float2* tH, float4* tX, int xodd) {
    const float mid = 0.5f * (lo + hi) - w_in;
    tH -= K0;  // slot of slab k at tH[k]
    p += lane;
    pm += lane;
    float ivf = (float)(rlo + lane);
    for (int b = lane; b < nrows + lane; b += 32) {
        const float4 qc = q;
        const float ymc = ym;
        p += 32;
        pm += 32;
        if (b + 32 < nrows) {  // next chunk
            q = __ldg(p);
            ym = __ldg(pm);
        }
        const bool valid = b < nrows;
        const int k0 = __float_as_int(qc.w) >> 2;  // primary rows: kstep -1
        const float dvh = __fmul_rn(__fmaf_rn(ivf, g.pv, g.dv0), h1);
        ivf += 32.f;
        const int k = k0 + __float2int_rd(__fmaf_rn(mid, dvh, qc.y));
        const float z1 = zcross(k, k0, qc.y, qc.z, w_in);
        const float z2 = zcross(k + 1, k0, qc.y, qc.z, w_in);
        const float wen = fminf(z1, z2), wlv = fmaxf(z1, z2);
        const bool enter = wen > lo;
        const bool leave = wlv < hi;
        const bool cx = valid && (enter || leave);
        // H: rows two apart never share a slab (two parity passes)
        const bool hw = valid && !cx && (unsigned)(k - K0) < (unsigned)NS;
        if (hw && !(lane & 1)) {
            const float2 h = tH[k];
            tH[k] = make_float2(h.x + qc.x, h.y + ymc);
        }
        __syncwarp();
        if (hw && (lane & 1)) {
            const float2 h = tH[k];
            tH[k] = make_float2(h.x + qc.x, h.y + ymc);
        }
        // the slab left: entering slab k from above (k + 1) or leaving it
        // (slot NS: the row entering the brick's top slab from above)
        const int kb = enter ? k + 1 : k;
        const int sb = kb - K0;  // slot: even ones at tX[s / 2], odd ones at tX[xodd + s / 2]
        if (cx && (unsigned)sb <= (unsigned)NS)
            tX[(sb & 1) * xodd + (sb >> 1)] = make_float4(enter ? wen : wlv, qc.x, ymc, 0.f);
        __syncwarp();
    }
}

// Deposits of one entry into both bricks.  Lane l takes the slot pair
// j = 2 l + 64 r, j + 1; the accumulators hold per voxel column CS slots of
// float2 {L, U}, so a lane's pair is one float4 (one shared load and store per
// segment and pair).  segs[s] = {wa, wb, float4 index of the column}.  Per
// voxel the pieces are added in one fixed order:
//   v + (wb - clamp(Xa.w)) Xa.y + (clamp(Xb.w) - wa) Xb.y + (wb - wa) H
// (Xb = tX[j]: the row leaving slot j; Xa = tX[j + 1]: the row entering it).
// Clears the tables.
#ifndef KCT_MIR_PCLEAR
#define KCT_MIR_PCLEAR 0  // 1: the producers clear a table buffer before refilling it (measured slower:
                          // c3 1.96 -> 2.02 ms, c4 13.2 -> 13.8 ms; the consumer clears only the live slots)
#endif
#ifndef KCT_MIR_UNROLL
#define KCT_MIR_UNROLL 2  // c3 adjoint with 3 producers: 2.04 (1) / 1.96 (2) / 1.98 (3) / 2.20 ms (4)
#endif
template <int RC, bool CLR = true>
__device__ __forceinline__ void mir_deposits(float4* acc, const float4* segs, int nseg, int NS,
                                             int lane, float2* tH, float4* tX, int xodd) {
    float4 h[RC], xA[RC], xB[RC], xC[RC];
    bool xs[RC], on[RC];
    float4* const tH4 = reinterpret_cast<float4*>(tH);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < RC; ++r) {
        const int j = 2 * lane + 64 * r;
        on[r] = j < NS;
        h[r] = xA[r] = xB[r] = xC[r] = z4;
        if (on[r]) {
            h[r] = tH4[lane + 32 * r];  // {hL, hU} of slots j, j + 1
            xA[r] = tX[lane + 32 * r];             // slot j (even slots: conflict-free rows)
            xB[r] = tX[xodd + lane + 32 * r];      // slot j + 1
            xC[r] = tX[lane + 1 + 32 * r];         // slot j + 2
        }
        xs[r] = __any_sync(kFull, xA[r].y != 0.f || xA[r].z != 0.f || xB[r].y != 0.f ||
                                      xB[r].z != 0.f || xC[r].y != 0.f || xC[r].z != 0.f);
    }
    // clear the tables (after every lane's reads: slot j + 2 is the next lane's)
    if (CLR) {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < RC; ++r)
            if (on[r]) {
                tH4[lane + 32 * r] = z4;
                tX[lane + 32 * r] = z4;
                tX[xodd + lane + 32 * r] = z4;
            }
        if (lane == 0) tX[(NS & 1) * xodd + (NS >> 1)] = z4;
    }
    int sgi = 0;
#if KCT_MIR_UNROLL > 1
    // KCT_MIR_UNROLL segments per step: an entry's segments lie in distinct
    // voxel columns (the xy walk never revisits one), so the later segments'
    // accumulator loads need not wait for the earlier ones' stores
    constexpr int U = KCT_MIR_UNROLL;
    for (; sgi + U <= nseg; sgi += U) {
        float4 sg[U];
        float4* a[U];
        float4 v[U][RC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            sg[u] = segs[sgi + u];
            a[u] = acc + (__float_as_int(sg[u].z) + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < RC; ++r) v[u][r] = on[r] ? a[u][32 * r] : z4;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float wa = sg[u].x, wb = sg[u].y;
            const float d = wb - wa;
#pragma unroll
            for (int r = 0; r < RC; ++r) {
                float4& w = v[u][r];
                if (xs[r]) {
                    const float cA = fminf(fmaxf(xA[r].x, wa), wb);
                    const float cB = fminf(fmaxf(xB[r].x, wa), wb);
                    const float cC = fminf(fmaxf(xC[r].x, wa), wb);
                    const float tbA = cA - wa, taA = wb - cB, tbB = cB - wa, taB = wb - cC;
                    w.x = __fmaf_rn(d, h[r].x, __fmaf_rn(tbA, xA[r].y, __fmaf_rn(taA, xB[r].y, w.x)));
                    w.y = __fmaf_rn(d, h[r].y, __fmaf_rn(tbA, xA[r].z, __fmaf_rn(taA, xB[r].z, w.y)));
                    w.z = __fmaf_rn(d, h[r].z, __fmaf_rn(tbB, xB[r].y, __fmaf_rn(taB, xC[r].y, w.z)));
                    w.w = __fmaf_rn(d, h[r].w, __fmaf_rn(tbB, xB[r].z, __fmaf_rn(taB, xC[r].z, w.w)));
                } else {
                    w.x = __fmaf_rn(d, h[r].x, w.x);
                    w.y = __fmaf_rn(d, h[r].y, w.y);
                    w.z = __fmaf_rn(d, h[r].z, w.z);
                    w.w = __fmaf_rn(d, h[r].w, w.w);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < RC; ++r)
                if (on[r]) a[u][32 * r] = v[u][r];
    }
#endif
    for (; sgi < nseg; ++sgi) {
        const float4 sg = segs[sgi];
        const float wa = sg.x, wb = sg.y;
        float4* const a = acc + (__float_as_int(sg.z) + lane);
        const float d = wb - wa;
        float4 v[RC];
#pragma unroll
        for (int r = 0; r < RC; ++r) v[r] = on[r] ? a[32 * r] : z4;
#pragma unroll
        for (int r = 0; r < RC; ++r) {
            if (xs[r]) {
                const float cA = fminf(fmaxf(xA[r].x, wa), wb);
                const float cB = fminf(fmaxf(xB[r].x, wa), wb);
                const float cC = fminf(fmaxf(xC[r].x, wa), wb);
                const float tbA = cA - wa, taA = wb - cB, tbB = cB - wa, taB = wb - cC;
                v[r].x = __fmaf_rn(d, h[r].x, __fmaf_rn(tbA, xA[r].y, __fmaf_rn(taA, xB[r].y, v[r].x)));
                v[r].y = __fmaf_rn(d, h[r].y, __fmaf_rn(tbA, xA[r].z, __fmaf_rn(taA, xB[r].z, v[r].y)));
                v[r].z = __fmaf_rn(d, h[r].z, __fmaf_rn(tbB, xB[r].y, __fmaf_rn(taB, xC[r].y, v[r].z)));
                v[r].w = __fmaf_rn(d, h[r].w, __fmaf_rn(tbB, xB[r].z, __fmaf_rn(taB, xC[r].z, v[r].w)));
            } else {
                v[r].x = __fmaf_rn(d, h[r].x, v[r].x);
                v[r].y = __fmaf_rn(d, h[r].y, v[r].y);
                v[r].z = __fmaf_rn(d, h[r].z, v[r].z);
                v[r].w = __fmaf_rn(d, h[r].w, v[r].w);
            }
        }
#pragma unroll
        for (int r = 0; r < RC; ++r)
            if (on[r]) a[32 * r] = v[r];
    }
    __syncwarp();
}

// Zero one table buffer (tX: CS + 1 float4, tH: CS float2).
__device__ __forceinline__ void mir_clear(float2* tH, float4* tX, int CS, int lane) {
    for (int j = lane; j <= CS; j += 32) {
        tX[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < CS) tH[j] = make_float2(0.f, 0.f);
    }
    __syncwarp();
}

// mir_deposits for NC consumer warps of the warp-specialised kernel:
// consumer c0 owns the voxel columns ij with ij % NC == c0 and takes the
// segments in them (so consumers never touch one column, even when one runs
// an entry ahead of another, and each column's deposits keep entry order);
// the tables are read only (the producer clears a buffer before refilling
// it).  Same arithmetic per voxel.
template <int RC>
__device__ __forceinline__ void mir_deposits_nc(float4* acc, const float4* segs, int nseg, int NS,
                                                int lane, const float2* tH, const float4* tX,
                                                int xodd, int c0, int NC) {
    float4 h[RC], xA[RC], xB[RC], xC[RC];
    bool xs[RC], on[RC];
    const float4* const tH4 = reinterpret_cast<const float4*>(tH);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < RC; ++r) {
        const int j = 2 * lane + 64 * r;
        on[r] = j < NS;
        h[r] = xA[r] = xB[r] = xC[r] = z4;
        if (on[r]) {
            h[r] = tH4[lane + 32 * r];
            xA[r] = tX[lane + 32 * r];
            xB[r] = tX[xodd + lane + 32 * r];
            xC[r] = tX[lane + 1 + 32 * r];
        }
        xs[r] = __any_sync(kFull, xA[r].y != 0.f || xA[r].z != 0.f || xB[r].y != 0.f ||
                                      xB[r].z != 0.f || xC[r].y != 0.f || xC[r].z != 0.f);
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
        const float4 sg = segs[sgi];
        if (__float_as_int(sg.w) % NC != c0) continue;
        const float wa = sg.x, wb = sg.y;
        float4* const a = acc + (__float_as_int(sg.z) + lane);
        const float d = wb - wa;
        float4 v[RC];
#pragma unroll
        for (int r = 0; r < RC; ++r) v[r] = on[r] ? a[32 * r] : z4;
#pragma unroll
        for (int r = 0; r < RC; ++r) {
            if (xs[r]) {
                const float cA = fminf(fmaxf(xA[r].x, wa), wb);
                const float cB = fminf(fmaxf(xB[r].x, wa), wb);
                const float cC = fminf(fmaxf(xC[r].x, wa), wb);
                const float tbA = cA - wa, taA = wb - cB, tbB = cB - wa, taB = wb - cC;
                v[r].x = __fmaf_rn(d, h[r].x, __fmaf_rn(tbA, xA[r].y, __fmaf_rn(taA, xB[r].y, v[r].x)));
                v[r].y = __fmaf_rn(d, h[r].y, __fmaf_rn(tbA, xA[r].z, __fmaf_rn(taA, xB[r].z, v[r].y)));
                v[r].z = __fmaf_rn(d, h[r].z, __fmaf_rn(tbB, xB[r].y, __fmaf_rn(taB, xC[r].y, v[r].z)));
                v[r].w = __fmaf_rn(d, h[r].w, __fmaf_rn(tbB, xB[r].z, __fmaf_rn(taB, xC[r].z, v[r].w)));
            } else {
                v[r].x = __fmaf_rn(d, h[r].x, v[r].x);
                v[r].y = __fmaf_rn(d, h[r].y, v[r].y);
                v[r].z = __fmaf_rn(d, h[r].z, v[r].z);
                v[r].w = __fmaf_rn(d, h[r].w, v[r].w);
            }
        }
#pragma unroll
        for (int r = 0; r < RC; ++r)
            if (on[r]) a[32 * r] = v[r];
    }
    __syncwarp();
}

#ifndef KCT_MIR_MINB
#define KCT_MIR_MINB 20  // 11 KB of shared memory per warp at 64-slab bricks: <= 20 warps per SM
#endif
// CSC: the brick height as a compile-time constant (shared-memory offsets
// become immediates), 0: bc.bz at run time.
template <int CSC>
__global__ void __launch_bounds__(32, KCT_MIR_MINB) adj_mirror_kernel(
    const float4* __restrict__ rec, const float* __restrict__ ymw, float* __restrict__ out,
    DevGeom g, BrickCfg bc, int a0, int nab, int accumulate, const int* __restrict__ order,
    int* queue, float* __restrict__ out_part, const WalkEntry* __restrict__ tab,
    const unsigned long long* __restrict__ off) {
    // rec / ymw: adj_weight_mir_kernel's records of the primary rows and the
    // mirror rows' weights, [column][p], p < nv/2 (primary row p, mirror row nv-1-p)
    extern __shared__ float4 sm4[];
    float* const sm = reinterpret_cast<float*>(sm4);
    const int lane = threadIdx.x & 31;
    const int nbricks = bc.nbx * bc.nby * bc.nbz;
    const int CS = CSC ? CSC : (bc.bz + 1) & ~1;  // slots per voxel column (even)
    const int nu = g.nu, nv = g.nv, nz = g.nz;
    // acc: [BX * BY voxel columns][CS slots] of float2 {L, U}
    float2* const acc = reinterpret_cast<float2*>(sm);
    float4* const segs = reinterpret_cast<float4*>(sm + 2 * BX * BY * CS);
    float4* const tX = segs + kMaxSeg;
    float2* const tH = reinterpret_cast<float2*>(tX + CS + 1);
    const int nitems = nbricks * bc.ngrp;
    int ticket = queue ? 0 : blockIdx.x;
    for (;;) {
        int item;
        if (queue) {
            int tk = 0;
            if (lane == 0) tk = atomicAdd(queue, 1);
            tk = __shfl_sync(kFull, tk, 0);
            if (tk >= nitems) break;
            item = tk;
        } else {
            if (ticket >= nitems) break;
            item = ticket;
            ticket = nitems;
        }
        const int grp = item % bc.ngrp;
        const int brick = queue ? order[item / bc.ngrp] : item / bc.ngrp;
        const int a_lo = (int)((long long)nab * grp / bc.ngrp);
        const int a_hi = (int)((long long)nab * (grp + 1) / bc.ngrp);
        float* const dst = grp == 0 ? out : out_part + (size_t)(grp - 1) * bc.gstride;
        const int acc_in = grp == 0 ? accumulate : 0;
        const BrickGeo B = brick_geo(brick, bc, g);
        const int K0 = B.K0, NS = B.bzn;
        for (int q = lane; q < BX * BY * CS / 2; q += 32) sm4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = lane; j < CS; j += 32) {
            tH[j] = make_float2(0.f, 0.f);
            tX[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (lane == 0) tX[CS] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();

        const unsigned long long* ob = off + (size_t)brick * (g.na + 1);
        const unsigned long long e0 = ob[a0 + a_lo], e1 = ob[a0 + a_hi];
        const unsigned* tw = reinterpret_cast<const unsigned*>(tab);
        constexpr int M = kNB + kNB / 4;  // first meta word
        auto ld_entry = [&](unsigned long long e) {
            return (e < e1 && lane < kEW) ? __ldg(tw + e * kEW + lane) : 0u;
        };
        const unsigned boff = (unsigned)a0 * (unsigned)nu * (unsigned)nv;
        // the first row chunk's records (and mirror weights) of entry e
        auto first_chunk = [&](unsigned we, unsigned long long e, float& ymo) {
            const unsigned ro = __shfl_sync(kFull, we, M), r = __shfl_sync(kFull, we, M + 1);
            const int rl = (int)(r & 0xffffu), n = (int)(r >> 16) - rl + 1;
            const bool ok = e < e1 && lane < n;
            const unsigned idx = ((ro - boff) >> 1) + (unsigned)(rl + lane);
            ymo = ok ? __ldg(ymw + idx) : 0.f;
            return ok ? __ldg(rec + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        unsigned w = ld_entry(e0), w1 = ld_entry(e0 + 1);
        float ym;
        float4 q = first_chunk(w, e0, ym);
        for (unsigned long long e = e0; e < e1; ++e) {
            const unsigned ijw1 = __shfl_sync(kFull, w, M - 1);
            const int nseg = (int)(ijw1 >> 24);
            const unsigned rr = __shfl_sync(kFull, w, M + 1);
            const float wa = __uint_as_float(__shfl_sync(kFull, w, lane & (kNB - 1)));
            const float wb = __uint_as_float(__shfl_sync(kFull, w, (lane + 1) & (kNB - 1)));
            const unsigned ijw = __shfl_sync(kFull, w, kNB + ((lane >> 2) & (kNB / 4 - 1)));
            const float lo = __uint_as_float(__shfl_sync(kFull, w, 0));
            const float hi = __uint_as_float(__shfl_sync(kFull, w, nseg & (kNB - 1)));
            const unsigned ro = __shfl_sync(kFull, w, M);
            const float w_in = __uint_as_float(__shfl_sync(kFull, w, M + 2));
            const float inv_h1 = __uint_as_float(__shfl_sync(kFull, w, M + 3));
            if (lane < nseg) {
                const int ij = (int)((ijw >> (8 * (lane & 3))) & 0xffu);
                segs[lane] = make_float4(wa, wb, __int_as_float(ij * (CS / 2)), 0.f);
            }
            const unsigned w2 = ld_entry(e + 2);
            float ym1;
            const float4 q1 = first_chunk(w1, e + 1, ym1);
            __syncwarp();
            const int rlo = (int)(rr & 0xffffu), rhi = (int)(rr >> 16);
            const unsigned cb = ((ro - boff) >> 1) + (unsigned)rlo;
            mir_classify(rec + cb, ymw + cb, q, ym, rhi - rlo + 1, rlo, lo, hi, w_in,
                         rcp_approx(inv_h1), K0, NS, lane, g, tH, tX, CS / 2 + 1);
            if (NS > 64)  // (NS <= kMirMaxBz = 128)
                mir_deposits<2>(sm4, segs, nseg, NS, lane, tH, tX, CS / 2 + 1);
            else
                mir_deposits<1>(sm4, segs, nseg, NS, lane, tH, tX, CS / 2 + 1);
            w = w1;
            w1 = w2;
            q = q1;
            ym = ym1;
        }
        if (!bc.out_ref) {
            // coalesced runs of the bricks' slabs per voxel column (U reversed)
            for (int c = 0; c < B.bxn * B.byn; ++c) {
                const int ci = c % B.bxn, cj = c / B.bxn;
                float* o = dst + ((size_t)(B.I0 + ci) + (size_t)g.nx * (B.J0 + cj)) * nz;
                const float2* ac = acc + (ci + BX * cj) * CS;
                for (int kk = lane; kk < NS; kk += 32) {
                    const float2 v = ac[kk];
                    float* oL = o + K0 + kk;
                    float* oU = o + (nz - 1 - K0 - kk);
                    *oL = acc_in ? *oL + v.x : v.x;
                    *oU = acc_in ? *oU + v.y : v.y;
                }
            }
            __syncwarp();
        } else {
            // reference layout (x fastest), lanes over the voxel columns then slabs
            const int ncol = BX * BY;
            for (int t = lane; t < ncol * NS; t += 32) {
                const int c = t % ncol, kk = t / ncol;
                const int ci = c % BX, cj = c / BX;
                if (ci < B.bxn && cj < B.byn) {
                    const size_t xy = (size_t)(B.I0 + ci) + (size_t)g.nx * (B.J0 + cj);
                    const size_t plane = (size_t)g.nx * g.ny;
                    float* oL = dst + xy + plane * (size_t)(K0 + kk);
                    float* oU = dst + xy + plane * (size_t)(nz - 1 - K0 - kk);
                    const float2 v = acc[c * CS + kk];
                    *oL = acc_in ? *oL + v.x : v.x;
                    *oU = acc_in ? *oU + v.y : v.y;
                }
            }
            if (bc.level_done) {
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(bc.level_done + progress_slot(brick, bc), 1u);
            }
        }
    }
}

// ---- warp-specialised brick pairs (adj_mirror_ws_kernel) ----
// Two warps per brick pair: warp 0 (producer) decodes the walk-table entries
// and classifies their rows into one of two table buffers, warp 1 (consumer)
// runs the deposits of the previous entry from the other buffer into the
// shared accumulators (and writes the bricks out).  Handshakes are shared-
// memory mbarriers (full[b]: producer arrives, consumer waits; empty[b]: the
// reverse), the queue ticket is handed over at a CTA barrier per item.  Same classification,
// same deposits, same order as adj_mirror_kernel: bit-identical results; the
// point is twice the warps per shared accumulator (the one-warp kernel is
// held to 20 warps per SM by its 11 KB of shared memory).
// shared-memory mbarriers (count 32: every lane of the signalling warp arrives)
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(a)
                 : "memory");
}
// Waiting warps poll: 29% of the kernel's issued warp instructions at c3 are
// SYNCS / NANOSLEEP / BRA of these loops (ncu source page).  They do not cost
// time: test_wait + a fixed __nanosleep of 20 / 50 / 100 / 200 ns between polls
// (KCT_MBAR_SLEEP_NS > 0) measured 2.073 / 2.072 / 2.064 / 2.069 ms against
// 2.053 ms for try_wait with a suspend hint — the working warps are latency-
// bound, not short of issue slots.
#ifndef KCT_MBAR_SLEEP_NS
#define KCT_MBAR_SLEEP_NS 0
#endif
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
#if KCT_MBAR_SLEEP_NS > 0
    // poll, then sleep a fixed time between polls (plain nanosleep: no wake-up
    // on unrelated barrier traffic)
    for (;;) {
        unsigned done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) break;
        __nanosleep(KCT_MBAR_SLEEP_NS);
    }
#else
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1, %2;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep (no spinning) until the phase flips
        : "memory");
#endif
}

// one table buffer: segs[kMaxSeg] | tX[CS + 1] | tH[CS] (float2) | meta (nseg)
__host__ __device__ constexpr int mir_buf_floats(int cs) {
    return 4 * kMaxSeg + 4 * (cs + 1) + 2 * cs + 4;
}
// accumulators | 2 NP buffers | item slots [2] + 4 NP mbarriers (8 B each)
__host__ __device__ constexpr int adj_mir_ws_floats(int bz, int np) {
    return 2 * BX * BY * ((bz + 1) & ~1) + 2 * np * mir_buf_floats((bz + 1) & ~1) + 4 + 8 * np;
}

#ifndef KCT_MIR_WARPS
#define KCT_MIR_WARPS 32  // resident warps per SM the register allocation aims at (64 registers; 28 / 36 / 40:
                          // 72 / 56 / 48 registers, c3 2.06 / 2.03 / 2.31 ms against 1.96 ms)
#endif
#ifndef KCT_MIR_NC
#define KCT_MIR_NC 1  // consumer warps (deposits; 2 / 3 measured slower: 2.51 / 3.14 ms at c3)
#endif
// NP producer warps take the entries of an item in turn (global entry g ->
// producer g % NP), each into its own two buffers (g % (2 NP)) which it
// clears before refilling; the NC consumer warps deposit every entry in
// entry order, consumer c the segments in its voxel columns (ij % NC == c),
// and share the bricks' clear and write-out (a named barrier between the
// consumers orders them around the deposits).
template <int CSC, int NP, int NC>
__global__ void __launch_bounds__(32 * (NP + NC), KCT_MIR_WARPS / (NP + NC)) adj_mirror_ws_kernel(
    const float4* __restrict__ rec, const float* __restrict__ ymw, float* __restrict__ out,
    DevGeom g, BrickCfg bc, int a0, int nab, int accumulate, const int* __restrict__ order,
    int* queue, float* __restrict__ out_part, const WalkEntry* __restrict__ tab,
    const unsigned long long* __restrict__ off) {
    constexpr int NB = 2 * NP;  // table buffers
    extern __shared__ float4 sm4[];
    float* const sm = reinterpret_cast<float*>(sm4);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const bool producer = warp < NP;
    const int cw = warp - NP;  // consumer index (>= 0)
    const int nbricks = bc.nbx * bc.nby * bc.nbz;
    const int CS = CSC ? CSC : (bc.bz + 1) & ~1;
    const int nu = g.nu, nv = g.nv, nz = g.nz;
    float2* const acc = reinterpret_cast<float2*>(sm);
    float* const bufbase = sm + 2 * BX * BY * CS;
    auto consumers_sync = [&]() {  // named barrier 1: the NC consumer warps
        if (NC > 1) asm volatile("bar.sync 1, %0;" ::"n"(32 * NC) : "memory");
        else __syncwarp();
    };
    const int BF = mir_buf_floats(CS);
    int* const s_item = reinterpret_cast<int*>(bufbase + NB * BF);  // [2]
    // mbarriers full[0..NB), empty[0..NB) (8-byte aligned)
    const unsigned mb = (unsigned)__cvta_generic_to_shared(bufbase + NB * BF + 4);
    auto full_of = [&](int b) { return mb + 8u * (unsigned)b; };
    auto empty_of = [&](int b) { return mb + 8u * (unsigned)(NB + b); };
    auto segs_of = [&](int b) { return reinterpret_cast<float4*>(bufbase + b * BF); };
    auto tX_of = [&](int b) { return segs_of(b) + kMaxSeg; };
    auto tH_of = [&](int b) { return reinterpret_cast<float2*>(tX_of(b) + CS + 1); };
    auto meta_of = [&](int b) { return reinterpret_cast<int*>(tH_of(b) + CS); };
    const int nitems = nbricks * bc.ngrp;
    if (producer) {  // tables start zeroed
        for (int b = warp; b < NB; b += NP)
            for (int j = lane; j <= CS; j += 32) {
                tX_of(b)[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (j < CS) tH_of(b)[j] = make_float2(0.f, 0.f);
            }
        // full[b]: the producer's 32 lanes arrive; empty[b]: every consumer's
        if (warp == 0 && lane < 2 * NB) mbar_init(mb + 8u * (unsigned)lane, lane < NB ? 32 : 32 * NC);
    }
    __syncthreads();
    unsigned gcount = 0;  // entries of earlier items (entry g: buffer g % NB)
    int ip = 0;
    for (;;) {
        if (threadIdx.x == 0) s_item[ip] = atomicAdd(queue, 1);
        __syncthreads();
        const int item = s_item[ip];
        ip ^= 1;
        if (item >= nitems) break;
        const int grp = item % bc.ngrp;
        const int brick = order[item / bc.ngrp];
        const int a_lo = (int)((long long)nab * grp / bc.ngrp);
        const int a_hi = (int)((long long)nab * (grp + 1) / bc.ngrp);
        const BrickGeo B = brick_geo(brick, bc, g);
        const int K0 = B.K0, NS = B.bzn;
        const unsigned long long* ob = off + (size_t)brick * (g.na + 1);
        const unsigned long long e0 = ob[a0 + a_lo], e1 = ob[a0 + a_hi];
        if (producer) {
            const unsigned* tw = reinterpret_cast<const unsigned*>(tab);
            constexpr int M = kNB + kNB / 4;
            auto ld_entry = [&](unsigned long long e) {
                return (e < e1 && lane < kEW) ? __ldg(tw + e * kEW + lane) : 0u;
            };
            const unsigned boff = (unsigned)a0 * (unsigned)nu * (unsigned)nv;
            auto first_chunk = [&](unsigned we, unsigned long long e, float& ymo) {
                const unsigned ro = __shfl_sync(kFull, we, M), r = __shfl_sync(kFull, we, M + 1);
                const int rl = (int)(r & 0xffffu), n = (int)(r >> 16) - rl + 1;
                const bool ok = e < e1 && lane < n;
                const unsigned idx = ((ro - boff) >> 1) + (unsigned)(rl + lane);
                ymo = ok ? __ldg(ymw + idx) : 0.f;
                return ok ? __ldg(rec + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
            };
            // this warp's entries: e0 + d, d = (warp - gcount) mod NP, step NP
            const unsigned long long es = e0 + (unsigned)((warp - (int)(gcount % NP) + NP) % NP);
            unsigned w = ld_entry(es), w1 = ld_entry(es + NP);
            float ym;
            float4 q = first_chunk(w, es, ym);
            for (unsigned long long e = es; e < e1; e += NP) {
                const unsigned gi = gcount + (unsigned)(e - e0);
                const int b = (int)(gi % NB);
                // the consumer is done with b (its use gi / NB - 1)
                if (gi >= (unsigned)NB) {
                    mbar_wait(empty_of(b), (gi / NB - 1u) & 1u);
                    if (NC > 1 || KCT_MIR_PCLEAR) mir_clear(tH_of(b), tX_of(b), CS, lane);
                }
                float4* const segs = segs_of(b);
                const unsigned ijw1 = __shfl_sync(kFull, w, M - 1);
                const int nseg = (int)(ijw1 >> 24);
                const unsigned rr = __shfl_sync(kFull, w, M + 1);
                const float wa = __uint_as_float(__shfl_sync(kFull, w, lane & (kNB - 1)));
                const float wb = __uint_as_float(__shfl_sync(kFull, w, (lane + 1) & (kNB - 1)));
                const unsigned ijw = __shfl_sync(kFull, w, kNB + ((lane >> 2) & (kNB / 4 - 1)));
                const float lo = __uint_as_float(__shfl_sync(kFull, w, 0));
                const float hi = __uint_as_float(__shfl_sync(kFull, w, nseg & (kNB - 1)));
                const unsigned ro = __shfl_sync(kFull, w, M);
                const float w_in = __uint_as_float(__shfl_sync(kFull, w, M + 2));
                const float inv_h1 = __uint_as_float(__shfl_sync(kFull, w, M + 3));
                if (lane < nseg) {
                    const int ij = (int)((ijw >> (8 * (lane & 3))) & 0xffu);
                    segs[lane] = make_float4(wa, wb, __int_as_float(ij * (CS / 2)), __int_as_float(ij));
                }
                if (lane == 0) *meta_of(b) = nseg;
                const unsigned w2 = ld_entry(e + 2 * NP);
                float ym1;
                const float4 q1 = first_chunk(w1, e + NP, ym1);
                const int rlo = (int)(rr & 0xffffu), rhi = (int)(rr >> 16);
                const unsigned cb = ((ro - boff) >> 1) + (unsigned)rlo;
                mir_classify(rec + cb, ymw + cb, q, ym, rhi - rlo + 1, rlo, lo, hi, w_in,
                             rcp_approx(inv_h1), K0, NS, lane, g, tH_of(b), tX_of(b), CS / 2 + 1);
                mbar_arrive(full_of(b));  // release: the tables / segments written above
                w = w1;
                w1 = w2;
                q = q1;
                ym = ym1;
            }
        } else {
            for (int q = lane + 32 * cw; q < BX * BY * CS / 2; q += 32 * NC)
                sm4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            consumers_sync();
            for (unsigned long long e = e0; e < e1; ++e) {
                const unsigned gi = gcount + (unsigned)(e - e0);
                const int b = (int)(gi % NB);
                mbar_wait(full_of(b), (gi / NB) & 1u);
                const int nseg = *meta_of(b);
                if (NC > 1) {
                    if (CSC ? CSC > 64 : NS > 64)
                        mir_deposits_nc<2>(sm4, segs_of(b), nseg, NS, lane, tH_of(b), tX_of(b), CS / 2 + 1, cw, NC);
                    else
                        mir_deposits_nc<1>(sm4, segs_of(b), nseg, NS, lane, tH_of(b), tX_of(b), CS / 2 + 1, cw, NC);
                } else {
                    if (CSC ? CSC > 64 : NS > 64)
                        mir_deposits<2, !KCT_MIR_PCLEAR>(sm4, segs_of(b), nseg, NS, lane, tH_of(b), tX_of(b), CS / 2 + 1);
                    else
                        mir_deposits<1, !KCT_MIR_PCLEAR>(sm4, segs_of(b), nseg, NS, lane, tH_of(b), tX_of(b), CS / 2 + 1);
                }
                mbar_arrive(empty_of(b));
            }
            consumers_sync();  // every consumer's deposits are in before the write-out
            float* const dst = grp == 0 ? out : out_part + (size_t)(grp - 1) * bc.gstride;
            const int acc_in = grp == 0 ? accumulate : 0;
            if (!bc.out_ref) {
                for (int c = cw; c < B.bxn * B.byn; c += NC) {
                    const int ci = c % B.bxn, cj = c / B.bxn;
                    float* o = dst + ((size_t)(B.I0 + ci) + (size_t)g.nx * (B.J0 + cj)) * nz;
                    const float2* ac = acc + (ci + BX * cj) * CS;
                    for (int kk = lane; kk < NS; kk += 32) {
                        const float2 v = ac[kk];
                        float* oL = o + K0 + kk;
                        float* oU = o + (nz - 1 - K0 - kk);
                        *oL = acc_in ? *oL + v.x : v.x;
                        *oU = acc_in ? *oU + v.y : v.y;
                    }
                }
            } else {
                const int ncol = BX * BY;
                for (int t = lane + 32 * cw; t < ncol * NS; t += 32 * NC) {
                    const int c = t % ncol, kk = t / ncol;
                    const int ci = c % BX, cj = c / BX;
                    if (ci < B.bxn && cj < B.byn) {
                        const size_t xy = (size_t)(B.I0 + ci) + (size_t)g.nx * (B.J0 + cj);
                        const size_t plane = (size_t)g.nx * g.ny;
                        float* oL = dst + xy + plane * (size_t)(K0 + kk);
                        float* oU = dst + xy + plane * (size_t)(nz - 1 - K0 - kk);
                        const float2 v = acc[c * CS + kk];
                        *oL = acc_in ? *oL + v.x : v.x;
                        *oU = acc_in ? *oU + v.y : v.y;
                    }
                }
                if (bc.level_done) {
                    __threadfence();
                    consumers_sync();
                    if (cw == 0 && lane == 0) atomicAdd(bc.level_done + progress_slot(brick, bc), 1u);
                }
            }
            __syncwarp();
        }
        gcount += (unsigned)(e1 - e0);
    }
}

// The warp-specialised kernel by (brick height, producer warps): handles pick
// 2 or 3 producers per consumer at creation (Projector::tune_adjoint).
using AdjWsFn = void (*)(const float4*, const float*, float*, DevGeom, BrickCfg, int, int, int,
                         const int*, int*, float*, const WalkEntry*, const unsigned long long*);
static AdjWsFn adj_ws_fn(int bz, int np) {
    if (np == 1)
        return bz == 64 ? adj_mirror_ws_kernel<64, 1, KCT_MIR_NC>
               : bz == 32 ? adj_mirror_ws_kernel<32, 1, KCT_MIR_NC> : adj_mirror_ws_kernel<0, 1, KCT_MIR_NC>;
    if (np == 3)
        return bz == 64 ? adj_mirror_ws_kernel<64, 3, KCT_MIR_NC>
               : bz == 32 ? adj_mirror_ws_kernel<32, 3, KCT_MIR_NC> : adj_mirror_ws_kernel<0, 3, KCT_MIR_NC>;
    return bz == 64 ? adj_mirror_ws_kernel<64, 2, KCT_MIR_NC>
           : bz == 32 ? adj_mirror_ws_kernel<32, 2, KCT_MIR_NC> : adj_mirror_ws_kernel<0, 2, KCT_MIR_NC>;
}

// ----------------------------------------------------------------------------
// Adjoint, per-voxel gather (alternative; KCT_ADJOINT=gather).  One warp = one
// voxel column (i,j), lane owns voxels k = kbase + lane + 32c.  For each angle
// and footprint column the chord is computed from the voxel's own planes and
// every candidate row's overlap with slab k from the shared crossing
// expressions.  Slower than the brick kernel; kept as an independent check.
// ----------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(128) adj_gather_kernel(const float* __restrict__ proj,
                                                         float* __restrict__ out,
                                                         const ColParams* __restrict__ cols,
                                                         const float* __restrict__ dvtab,
                                                         const float* __restrict__ invdv,
                                                         const double* __restrict__ dvd,
                                                         DevGeom g, AngleBatch ab, int nab,
                                                         int accumulate) {
    const int lane = threadIdx.x & 31;
    const int colid = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (colid >= g.nx * g.ny) return;
    const int i = colid % g.nx, j = colid / g.nx;
    const int kbase = blockIdx.y * (32 * K) + lane;
    const int nz = g.nz, nu = g.nu, nv = g.nv;
    const float X0 = g.ox + i * g.sx, X1 = g.ox + (i + 1) * g.sx;
    const float Y0 = g.oy + j * g.sy, Y1 = g.oy + (j + 1) * g.sy;
    const float rpv = 1.f / g.pv;
    float acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.f;
    for (int ia = 0; ia < nab; ++ia) {
        int iu_lo, iu_hi;
        footprint(g, ab.cs[ia].x, ab.cs[ia].y, X0, X1, Y0, Y1, iu_lo, iu_hi);
        for (int iu = iu_lo; iu <= iu_hi; ++iu) {
            const ColParams cp = cols[(size_t)ia * nu + iu];
            float lo = cp.w_in, hi = cp.w_out;
            if (cp.dx != 0.0) {
                const float e0 = xcross(cp, i), e1 = xcross(cp, i + 1);
                lo = fmaxf(lo, fminf(e0, e1));
                hi = fminf(hi, fmaxf(e0, e1));
            } else if (i != cp.i0) {
                continue;
            }
            if (cp.dy != 0.0) {
                const float e0 = ycross(cp, j), e1 = ycross(cp, j + 1);
                lo = fmaxf(lo, fminf(e0, e1));
                hi = fminf(hi, fmaxf(e0, e1));
            } else if (j != cp.j0) {
                continue;
            }
            if (!(lo < hi)) continue;
            const float h1 = 1.f / cp.inv_h1;
            const float gin = (float)cp.g_in;
            const float rGa = 1.f / (gin + (lo - cp.w_in) * h1);
            const float rGb = 1.f / (gin + (hi - cp.w_in) * h1);
            const float* py = proj + ((size_t)ia * nu + iu) * nv;
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const int k = kbase + 32 * c;
                if (k >= nz) continue;
                const float n0 = (float)k + g.kz0, n1 = n0 + 1.f;
                const float dlo = n0 * (n0 >= 0.f ? rGb : rGa);
                const float dhi = n1 * (n1 >= 0.f ? rGa : rGb);
                const int rlo = max(0, (int)ceilf((dlo - g.dv0) * rpv - 1e-3f));
                const int rhi = min(nv - 1, (int)floorf((dhi - g.dv0) * rpv + 1e-3f));
                for (int iv = rlo; iv <= rhi; ++iv) {
                    const float dv = dvtab[iv];
                    // z-mirror rows: the primary's z state, planes reflected
                    // (the forward's MIR definition, fwd_kernel)
                    const bool mir = g.mirror && iv >= nv / 2;
                    const int ivp = mir ? nv - 1 - iv : iv;
                    const double kzd = fma(dvd[ivp], cp.g_in, -g.kz0d);
                    const double fl = floor(kzd);
                    const int k0 = (int)fmax(fmin(fl, 1.0e9), -1.0e9);
                    const float f0 = (float)(kzd - fl);
                    float zlo, zhi;
                    if (dv != 0.f) {
                        const float imk = __fmul_rn(invdv[ivp], cp.inv_h1);
                        const int kp = mir ? nz - 1 - k : k;  // the primary's slab
                        const float w0 = zcross(kp, k0, f0, imk, cp.w_in);
                        const float w1 = zcross(kp + 1, k0, f0, imk, cp.w_in);
                        zlo = fminf(w0, w1);
                        zhi = fmaxf(w0, w1);
                    } else {
                        if (k0 != k) continue;
                        zlo = -kInf;
                        zhi = kInf;
                    }
                    const float len = fminf(hi, zhi) - fmaxf(lo, zlo);
                    if (len > 0.f) {
                        const float q = dv * cp.inv_l;
                        const float f = __fsqrt_rn(__fmaf_rn(q, q, 1.f));
                        acc[c] = __fmaf_rn(len, __ldg(py + iv) * f, acc[c]);
                    }
                }
            }
        }
    }
    float* o = out + (size_t)colid * nz;
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const int k = kbase + 32 * c;
        if (k < nz) o[k] = accumulate ? o[k] + acc[c] : acc[c];
    }
}

// Batched 2D transpose: in[b][r][c] -> out[b][c][r].
__global__ void transpose_kernel(const float* __restrict__ in, float* __restrict__ out, int R,
                                 int Cc, int ldo) {
    __shared__ float tile[32][33];
    const size_t boff = (size_t)blockIdx.z * R * Cc;
    const size_t ooff = (size_t)blockIdx.z * ldo * Cc;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int r = r0 + dy, c = c0 + threadIdx.x;
        if (r < R && c < Cc) tile[dy][threadIdx.x] = in[boff + (size_t)r * Cc + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int c = c0 + dy, r = r0 + threadIdx.x;
        if (r < R && c < Cc) out[ooff + (size_t)c * ldo + r] = tile[threadIdx.x][dy];
    }
}

// Sub-block transpose with leading dimensions and batch strides:
// in[b * bsi + r * ldi + c] -> out[b * bso + c * ldo + r], r < R, c < Cc.
__global__ void transpose_sub_kernel(const float* __restrict__ in, float* __restrict__ out, int R,
                                     int Cc, int ldi, int ldo, size_t bsi, size_t bso) {
    __shared__ float tile[32][33];
    const size_t boff = (size_t)blockIdx.z * bsi, ooff = (size_t)blockIdx.z * bso;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int r = r0 + dy, c = c0 + threadIdx.x;
        if (r < R && c < Cc) tile[dy][threadIdx.x] = in[boff + (size_t)r * ldi + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int c = c0 + dy, r = r0 + threadIdx.x;
        if (r < R && c < Cc) out[ooff + (size_t)c * ldo + r] = tile[threadIdx.x][dy];
    }
}

// in[b][r][c] -> out[b][c][r] (row stride of out: ldo >= R)
void launch_transpose(const float* in, float* out, int B, int R, int Cc, cudaStream_t s,
                      int ldo = 0) {
    dim3 grid((Cc + 31) / 32, (R + 31) / 32, B);
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, out, R, Cc, ldo ? ldo : R);
    KCT_LAUNCHED();
}

}  // namespace

// ---- validation ---------------------------------------------------------------
void validate_geometry(const kct_grid& grid, const kct_geometry& g) {
    if (grid.nx < 1 || grid.ny < 1 || grid.nz < 1) throw ConfigError("grid dims must be positive");
    if (!(grid.sx > 0.0) || !(grid.sy > 0.0) || !(grid.sz > 0.0))
        throw ConfigError("voxel spacing must be strictly positive");
    if (!(g.dso > 0.0) || !(g.dsd > g.dso)) throw ConfigError("geometry requires dsd > dso > 0");
    if (g.nu < 1 || g.nv < 1) throw ConfigError("detector must have at least one pixel per axis");
    if (!(g.pu > 0.0) || !(g.pv > 0.0)) throw ConfigError("detector pixel pitch must be positive");
    if (g.n_angles < 1 || g.angles == nullptr)
        throw ConfigError("geometry requires at least one angle");
    const double hx = grid.ox + grid.nx * grid.sx, hy = grid.oy + grid.ny * grid.sy,
                 hz = grid.oz + grid.nz * grid.sz;
    for (int ia = 0; ia < g.n_angles; ++ia) {
        const double t = g.angles[ia];
        const double sx = g.dso * std::cos(t), sy = g.dso * std::sin(t), sz = 0.0;
        if (sx > grid.ox && sx < hx && sy > grid.oy && sy < hy && sz > grid.oz && sz < hz)
            throw ConfigError("source position lies inside the volume");
    }
    // The forward indexes the padded volume (column stride vpad_stride(nz)) and
    // the walk table the rays ((angle * nu + column) * nv) with 32-bit integers.
    const double mpad = (double)grid.nx * grid.ny * vpad_stride(grid.nz);
    if (mpad > 2147483647.0) throw ConfigError("volume too large for 32-bit voxel indexing");
    const double rays = (double)g.nu * g.nv * g.n_angles;
    if (rays > 4294967295.0) throw ConfigError("too many rays for 32-bit ray indexing");
}

// ---- host-side tables ---------------------------------------------------------
Projector::Projector(const kct_grid& grid, const kct_geometry& geom, int device)
    : grid_(grid) {
    validate_geometry(grid, geom);
    if (device >= 0) KCT_CUDA(cudaSetDevice(device));
    KCT_CUDA(cudaGetDevice(&device_));
    m_ = (size_t)grid.nx * grid.ny * grid.nz;
    n_ = (size_t)geom.nu * geom.nv * geom.n_angles;
    dso_d_ = geom.dso;
    dsd_d_ = geom.dsd;
    pu_d_ = geom.pu;
    pv_d_ = geom.pv;
    offu_d_ = geom.offset_u;
    offv_d_ = geom.offset_v;
    const char* rs = std::getenv("KCT_SOLVER_RESTART");
    solver_restart = rs && rs[0] == '1';
    const char* mode = std::getenv("KCT_ADJOINT");
    adj_gather_ = mode && std::string(mode) == "gather";
    build_tables(geom);
    // padded native volume of the forward (zero slabs at -1 and nz)
    KCT_CUDA(cudaMalloc(&d_vpad_, (size_t)grid.nx * grid.ny * vpad_stride(grid.nz) * sizeof(float)));
    KCT_CUDA(cudaMemset(d_vpad_, 0, (size_t)grid.nx * grid.ny * vpad_stride(grid.nz) * sizeof(float)));
}

Projector::~Projector() {
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(device_);
    workspace.reset();
    cudaFree(d_cols_);
    cudaFree(d_dv_);
    cudaFree(d_invdv_);
    cudaFree(d_dvd_);
    cudaFree(d_rows_);
    cudaFree(d_border_);
    cudaFree(d_forder_);
    cudaFree(d_fpipe_);
    cudaFree(d_flo_);
    cudaFree(d_fcnt_all_);
    cudaFree(d_fcnt_hi_);
    cudaFree(d_fdone_);
    cudaFree(d_vpad_);
    cudaFree(d_cs_);
    cudaFree(d_fhi_);
    cudaFree(d_fstage_);
    cudaFree(d_ftab_off_);
    cudaFree(d_ftab_);
    if (pipe_stream_) {
        for (auto e : pipe_ev_) cudaEventDestroy(e);
        cudaEventDestroy(up_ev_);
        cudaStreamDestroy(pipe_stream_);
    }
    cudaFree(d_queue_);
    cudaFree(d_part_);
    cudaFree(d_yw_);
    cudaFree(d_tab_);
    cudaFree(d_off_);
    cudaFree(d_level_);
    for (auto* p : scratch_) cudaFree(p);
    if (cur >= 0) cudaSetDevice(cur);
}

float* Projector::scratch(int slot, size_t n) {
    if (scratch_n_[slot] < n) {
        cudaFree(scratch_[slot]);
        scratch_[slot] = nullptr;
        KCT_CUDA(cudaMalloc(&scratch_[slot], n * sizeof(float)));
        scratch_n_[slot] = n;
    }
    return scratch_[slot];
}

void Projector::build_tables(const kct_geometry& geom) {
    const int nx = grid_.nx, ny = grid_.ny, nz = grid_.nz;
    const int nu = geom.nu, nv = geom.nv, na = geom.n_angles;
    dg_.nx = nx; dg_.ny = ny; dg_.nz = nz;
    dg_.nu = nu; dg_.nv = nv; dg_.na = na;
    dg_.ox = (float)grid_.ox; dg_.oy = (float)grid_.oy;
    dg_.sx = (float)grid_.sx; dg_.sy = (float)grid_.sy;
    dg_.kz0 = (float)(grid_.oz / grid_.sz);
    dg_.kz0d = grid_.oz / grid_.sz;
    dg_.dso = (float)geom.dso; dg_.dsd = (float)geom.dsd;
    dg_.pu = (float)geom.pu; dg_.off_u = (float)geom.offset_u;
    dg_.pv = (float)geom.pv;
    dg_.dv0 = (float)((0.5 - 0.5 * nv) * geom.pv + geom.offset_v);
    // z-mirror geometry (fwd_kernel MIR): the source is at z = 0 (projector.hpp:24-27);
    // with offset_v = 0 and nv even, rows iv and nv-1-iv have dv of opposite
    // sign (exactly), and a grid centred in z maps slab k onto nz-1-k
    {
        const char* me = std::getenv("KCT_MIRROR");
        mirror_ = geom.offset_v == 0.0 && nv % 2 == 0 &&
                  std::abs(grid_.oz / grid_.sz + 0.5 * nz) < 1e-9 && !(me && me[0] == '0');
        dg_.mirror = mirror_ ? 1 : 0;
    }

    // detector rows: dv(iv) (projector.hpp:36) — the ray's z at the detector
    std::vector<float> dv(nv), invdv(nv);
    std::vector<double> dvd(nv);
    double dv_max = 0.0;
    for (int iv = 0; iv < nv; ++iv) {
        const double d = (iv + 0.5 - 0.5 * nv) * geom.pv + geom.offset_v;
        dvd[iv] = d;
        dv[iv] = (float)d;
        dv_max = std::max(dv_max, std::abs(d));
        invdv[iv] = dv[iv] != 0.f ? (float)(1.0 / (double)dv[iv])
                                  : std::numeric_limits<float>::infinity();
    }

    const double ox = grid_.ox, oy = grid_.oy, sx = grid_.sx, sy = grid_.sy, sz = grid_.sz;
    const double hx = ox + nx * sx, hy = oy + ny * sy;
    std::vector<ColParams> cols((size_t)na * nu);
    cs_.resize(na);
    bool full_fp = false;
    double r_max = 0.0;  // farthest xy corner of the volume from the axis
    for (double X : {ox, hx})
        for (double Y : {oy, hy}) r_max = std::max(r_max, std::hypot(X, Y));
    double L_min = std::numeric_limits<double>::infinity(), L_max = 0.0;
    for (int a = 0; a < na; ++a) {
        const double t = geom.angles[a];
        const double c = std::cos(t), s = std::sin(t);
        cs_[a] = make_float2((float)c, (float)s);
        const double Sx = geom.dso * c, Sy = geom.dso * s;
        // a voxel square behind the source plane breaks the corner-projection footprint
        for (double X : {ox, hx})
            for (double Y : {oy, hy})
                if (geom.dso - (X * c + Y * s) <= 1e-6 * geom.dso) full_fp = true;
        for (int iu = 0; iu < nu; ++iu) {
            ColParams& cp = cols[(size_t)a * nu + iu];
            const double du = (iu + 0.5 - 0.5 * nu) * geom.pu + geom.offset_u;
            // pixel centre minus source, xy part (projector.hpp:30-39)
            const double dx = -geom.dsd * c - du * s;
            const double dy = -geom.dsd * s + du * c;
            const double L = std::hypot(dx, dy);
            L_min = std::min(L_min, L);
            L_max = std::max(L_max, L);
            const double ex = dx / L, ey = dy / L;
            const double w0 = -(Sx * ex + Sy * ey);  // foot point of the axis
            const double Rx = Sx + w0 * ex, Ry = Sy + w0 * ey;
            cp.bx = ex != 0.0 ? (ox - Rx) / ex : 0.0;
            cp.dx = ex != 0.0 ? sx / ex : 0.0;
            cp.by = ey != 0.0 ? (oy - Ry) / ey : 0.0;
            cp.dy = ey != 0.0 ? sy / ey : 0.0;
            cp.inv_h1 = (float)(L * sz);
            cp.inv_l = (float)(1.0 / L);
            // clip: t in [0,1] and the xy box, evaluated with the same
            // expressions the kernels use for plane crossings
            auto xc = [&](int n) { return (float)std::fma((double)n, cp.dx, cp.bx); };
            auto yc = [&](int n) { return (float)std::fma((double)n, cp.dy, cp.by); };
            float lo = (float)(-w0), hi = (float)(L - w0);
            bool miss = false;
            if (cp.dx != 0.0) {
                const float e0 = xc(0), e1 = xc(nx);
                lo = std::max(lo, std::min(e0, e1));
                hi = std::min(hi, std::max(e0, e1));
            } else if (Sx <= ox || Sx >= hx) {
                miss = true;
            }
            if (cp.dy != 0.0) {
                const float e0 = yc(0), e1 = yc(ny);
                lo = std::max(lo, std::min(e0, e1));
                hi = std::min(hi, std::max(e0, e1));
            } else if (Sy <= oy || Sy >= hy) {
                miss = true;
            }
            if (miss || !(lo < hi)) {
                cp.w_in = 1.f;
                cp.w_out = 0.f;
                cp.g_in = 0.0;
                cp.i0 = cp.j0 = 0;
                continue;
            }
            cp.w_in = lo;
            cp.w_out = hi;
            cp.g_in = (w0 + (double)lo) / (L * sz);
            // entry voxel (projector.hpp:93-98): floor at the entry point, clamped
            const double px = Rx + (double)lo * ex, py = Ry + (double)lo * ey;
            const int ii = (int)std::floor((px - ox) / sx), jj = (int)std::floor((py - oy) / sy);
            cp.i0 = std::clamp(ii, 0, nx - 1);
            cp.j0 = std::clamp(jj, 0, ny - 1);
        }
    }
    dg_.full_footprint = full_fp ? 1 : 0;

    // forward launch shape: rows (mirror: row pairs) per warp = 32*C, C <= 3
    // (C = 4 costs registers and occupancy: c4 with 12 chunks, 3 bands of 4
    // 12.59 ms, 4 bands of 3 11.56 ms, 6 bands of 2 12.33 ms; KCT_FWD_C: up to 4)
    const int chunks = ((mirror_ ? nv / 2 : nv) + 31) / 32;
    int cmax = 3;
    if (const char* e = std::getenv("KCT_FWD_C")) cmax = std::clamp(std::atoi(e), 1, 4);
    fwd_bands_ = (chunks + cmax - 1) / cmax;
    fwd_c_ = (chunks + fwd_bands_ - 1) / fwd_bands_;
    dg_.fwd_bands = fwd_bands_;
    // forward block order: (angle, band, column quad) items by decreasing
    // xy chord of the quad (ray length ~ work), stable
    {
        const int nq = (nu + kFwdWarps - 1) / kFwdWarps;
        const size_t nitems = (size_t)nq * fwd_bands_ * na;
        std::vector<std::pair<float, int>> key(nitems);
        // bands in turn, longest chords first within a band: the volume's z
        // range a band's rays touch stays in L2 (c4: 24.0 -> 20.6 ms; c3 +-0)
        const char* fob = std::getenv("KCT_FWD_ORDER");
        const bool band_major = !(fob && std::string(fob) == "chord");
        for (size_t t = 0; t < nitems; ++t) {
            const int quad = (int)(t % nq), a = (int)(t / ((size_t)nq * fwd_bands_));
            float len = 0.f;
            for (int w = 0; w < kFwdWarps && quad * kFwdWarps + w < nu; ++w) {
                const ColParams& cp = cols[(size_t)a * nu + quad * kFwdWarps + w];
                len += std::max(0.f, cp.w_out - cp.w_in);
            }
            key[t] = {-len, (int)t};
            if (band_major) {  // bands in turn: each band's z range of the volume stays in L2
                const int band = (int)((t / nq) % fwd_bands_);
                key[t].first = (float)band * 1e9f - len;
            }
        }
        std::stable_sort(key.begin(), key.end());
        std::vector<int> order(nitems);
        for (size_t t = 0; t < nitems; ++t) order[t] = key[t].second;
        const char* fo = std::getenv("KCT_FWD_ORDER");
        if (!(fo && std::string(fo) == "0")) {
            KCT_CUDA(cudaMalloc(&d_forder_, nitems * sizeof(int)));
            KCT_CUDA(cudaMemcpy(d_forder_, order.data(), nitems * sizeof(int), cudaMemcpyHostToDevice));
            // the same order restricted to each host-path pipeline chunk of angles
            // (items re-indexed relative to the chunk's first angle)
            pipe_chunks_ = na >= 4 * kPipeMinAngles ? kPipeChunks : 1;
            if (pipe_chunks_ > 1) {
                std::vector<int> pord;
                pipe_off_.assign(pipe_chunks_ + 1, 0);
                const size_t per_angle = (size_t)nq * fwd_bands_;
                for (int c = 0; c < pipe_chunks_; ++c) {
                    const int a0 = pipe_angle(c), a1 = pipe_angle(c + 1);
                    pipe_off_[c] = (int)pord.size();
                    for (size_t t = 0; t < nitems; ++t) {
                        const int it = key[t].second;
                        const int a = (int)(it / per_angle);
                        if (a >= a0 && a < a1) pord.push_back(it - (int)(a0 * per_angle));
                    }
                }
                pipe_off_[pipe_chunks_] = (int)pord.size();
                KCT_CUDA(cudaMalloc(&d_fpipe_, pord.size() * sizeof(int)));
                KCT_CUDA(cudaMemcpy(d_fpipe_, pord.data(), pord.size() * sizeof(int),
                                    cudaMemcpyHostToDevice));
                // the same items chunk-major for the single counted launch of
                // the host pipeline (forward_counted): all bands, and bands 1..
                {
                    const int B = fwd_bands_;
                    std::vector<int> all, hi;
                    for (int c = 0; c < pipe_chunks_; ++c) {
                        const int a0 = pipe_angle(c), a1 = pipe_angle(c + 1);
                        for (size_t t = 0; t < nitems; ++t) {
                            const int it = key[t].second;
                            const int quad = it % nq, band = (it / nq) % B, a = it / (nq * B);
                            if (a < a0 || a >= a1) continue;
                            all.push_back(it);
                            if (band > 0) hi.push_back(quad + nq * ((band - 1) + (B - 1) * a));
                        }
                    }
                    KCT_CUDA(cudaMalloc(&d_fcnt_all_, all.size() * sizeof(int)));
                    KCT_CUDA(cudaMemcpy(d_fcnt_all_, all.data(), all.size() * sizeof(int),
                                        cudaMemcpyHostToDevice));
                    if (!hi.empty()) {
                        KCT_CUDA(cudaMalloc(&d_fcnt_hi_, hi.size() * sizeof(int)));
                        KCT_CUDA(cudaMemcpy(d_fcnt_hi_, hi.data(), hi.size() * sizeof(int),
                                            cudaMemcpyHostToDevice));
                    }
                    KCT_CUDA(cudaMalloc(&d_fdone_, (size_t)pipe_chunks_ * sizeof(unsigned)));
                }
                // split upload of a host volume: the rays of row band 0 stay
                // below slab Z (largest continuous z index over every column's
                // clip, row band 0's top row; + 2 slabs of margin), so band 0
                // can run once slabs [0, Z) are on the device.  Mirror pairs:
                // band 0 holds the rows nearest z = 0 and stays inside slabs
                // [nz - Z, Z).
                double kmax = -1e30;
                const int r1 = std::min(nv, (mirror_ ? nv / 2 : 0) + 32 * fwd_c_) - 1;
                for (const ColParams& cp : cols) {
                    if (!(cp.w_in < cp.w_out)) continue;
                    const double Gin = cp.g_in, Gout = cp.g_in + (double)(cp.w_out - cp.w_in) / cp.inv_h1;
                    kmax = std::max(kmax, std::max(dvd[r1] * Gin, dvd[r1] * Gout) - grid_.oz / grid_.sz);
                }
                const int Z = std::min((int)std::floor(kmax) + 3, nz);
                const int Zlo = mirror_ ? std::max(0, nz - Z) : 0;
                const char* sp = std::getenv("KCT_FWD_SPLIT");
                if (fwd_bands_ >= 2 && Z - Zlo >= 1 && Z - Zlo <= (nz * 6) / 10 &&
                    !(sp && sp[0] == '0')) {
                    fwd_split_z_ = Z;
                    fwd_split_lo_ = Zlo;
                    std::vector<int> lo, hi;
                    const int B = fwd_bands_;
                    for (size_t t = 0; t < nitems; ++t) {
                        const int it = key[t].second;
                        const int quad = it % nq, band = (it / nq) % B, a = it / (nq * B);
                        if (band == 0) lo.push_back(quad + nq * a);
                    }
                    fhi_off_.assign(pipe_chunks_ + 1, 0);
                    for (int c = 0; c < pipe_chunks_; ++c) {
                        const int a0 = pipe_angle(c), a1 = pipe_angle(c + 1);
                        fhi_off_[c] = (int)hi.size();
                        for (size_t t = 0; t < nitems; ++t) {
                            const int it = key[t].second;
                            const int quad = it % nq, band = (it / nq) % B, a = it / (nq * B);
                            if (band > 0 && a >= a0 && a < a1)
                                hi.push_back(quad + nq * ((band - 1) + (B - 1) * (a - a0)));
                        }
                    }
                    fhi_off_[pipe_chunks_] = (int)hi.size();
                    KCT_CUDA(cudaMalloc(&d_flo_, lo.size() * sizeof(int)));
                    KCT_CUDA(cudaMemcpy(d_flo_, lo.data(), lo.size() * sizeof(int), cudaMemcpyHostToDevice));
                    KCT_CUDA(cudaMalloc(&d_fhi_, hi.size() * sizeof(int)));
                    KCT_CUDA(cudaMemcpy(d_fhi_, hi.data(), hi.size() * sizeof(int), cudaMemcpyHostToDevice));
                }
            }
        }
    }
    // staged host forward (forward_host_staged): row stages of 1, 2, 3, 4, 4,
    // ... chunks of 32 rows (z-mirror: row pairs) from z = 0 outwards; stage s
    // runs once the slabs its rays reach are uploaded (centre out), so the
    // upload of the outer slabs overlaps the inner rows' projection
    if (pipe_chunks_ > 1) {
        const char* se = std::getenv("KCT_FWD_STAGED");
        // KCT_FWD_ROWSTAGES=1: every stage's rows leave the device as soon as
        // the stage is done (default: only the last stage streams out, per
        // pipeline chunk of angles).  Measured slower at c3 (2.84 vs 2.66 ms
        // with stages 1,2,3; 3.06 ms with six one-chunk stages): a stage of C
        // row chunks shares one xy walk between C rows per lane, so small
        // stages redo the walk — the kernels of 1,1,1,1,1,1 sum to 2.29 ms
        // against 1.71 ms in one launch.
        // Tall detectors (more than 6 row chunks; c4: 12) do take it: their
        // outermost stage mostly misses the volume and ends at once, so the
        // angle-chunk scheme leaves the whole download exposed (c4 host
        // forward 22.1 ms; row stages of 1,2,3,4,2 chunks 20.0 ms, of
        // 2,3,3,2,2 chunks 18.7 ms — a short first stage to start early,
        // 3-chunk stages in the middle, short ones last for a short tail).
        const char* rs = std::getenv("KCT_FWD_ROWSTAGES");
        fwd_rowstages_ = rs && rs[0] == '1';
        const bool rows_auto = !rs && ((mirror_ ? nv / 2 : nv) + 31) / 32 > 6;
        const int rows = mirror_ ? nv / 2 : nv, T = (rows + 31) / 32;
        std::vector<int> sizes;
        if (const char* ss = std::getenv("KCT_FWD_STAGE_SIZES")) {  // e.g. "2,4" (sweeps)
            int t = 0;
            for (const char* c = ss; *c && t < T;) {
                const int v = std::clamp(std::atoi(c), 1, 4);
                sizes.push_back(std::min(v, T - t));
                t += sizes.back();
                while (*c && *c != ',') ++c;
                if (*c == ',') ++c;
            }
            while (t < T) sizes.push_back(std::min(4, T - t)), t += sizes.back();
        } else {
            if (rows_auto) {
                std::vector<int> cand = {2};
                int rem = T - 6;
                for (; rem >= 3; rem -= 3) cand.push_back(3);
                if (rem > 0) cand.push_back(rem);
                cand.push_back(2);
                cand.push_back(2);
                if ((int)cand.size() <= kPipeChunks) {
                    sizes = cand;
                    fwd_rowstages_ = true;
                }
            }
            const bool have = !sizes.empty();
            for (int t = 0, c = 1; !have && t < T; c = std::min(c + 1, 4)) {
                sizes.push_back(std::min(c, T - t));
                t += sizes.back();
            }
        }
        auto zrange = [&](int r_end, int& lo, int& hi) {  // slabs of rows (pairs) [0, r_end)
            const int r1 = std::min(nv, (mirror_ ? nv / 2 : 0) + r_end) - 1;
            double kmax = -1e30;
            for (const ColParams& cp : cols) {
                if (!(cp.w_in < cp.w_out)) continue;
                const double Gin = cp.g_in, Gout = cp.g_in + (double)(cp.w_out - cp.w_in) / cp.inv_h1;
                kmax = std::max(kmax, std::max(dvd[r1] * Gin, dvd[r1] * Gout) - grid_.oz / grid_.sz);
            }
            hi = std::clamp((int)std::floor(kmax) + 3, 1, nz);
            lo = mirror_ ? std::max(0, nz - hi) : 0;
        };
        int lo0 = 0, hi0 = nz;
        if (sizes.size() >= 2) zrange(32 * sizes[0], lo0, hi0);
        if (sizes.size() >= 2 && hi0 - lo0 <= (nz * 6) / 10 && !(se && se[0] == '0')) {
            const int nq = (nu + kFwdWarps - 1) / kFwdWarps;
            std::vector<float> chord((size_t)nq * na, 0.f);
            for (int a = 0; a < na; ++a)
                for (int iu = 0; iu < nu; ++iu) {
                    const ColParams& cp = cols[(size_t)a * nu + iu];
                    chord[(size_t)a * nq + iu / kFwdWarps] += std::max(0.f, cp.w_out - cp.w_in);
                }
            std::vector<int> orders;
            int row0 = 0;
            for (size_t st = 0; st < sizes.size(); ++st) {
                const bool last = st + 1 == sizes.size();
                FwdStage f{};
                f.row0 = row0;
                f.C = sizes[st];
                row0 += 32 * f.C;
                if (last) { f.z_lo = 0; f.z_hi = nz; }
                else zrange(row0, f.z_lo, f.z_hi);
                if (!fstages_.empty()) {  // cumulative ranges
                    f.z_lo = std::min(f.z_lo, fstages_.back().z_lo);
                    f.z_hi = std::max(f.z_hi, fstages_.back().z_hi);
                }
                f.order_off = orders.size();
                // items quad + nq * a, longest chords first (last stage: per
                // pipeline chunk of angles, so chunks finish in turn)
                std::vector<std::pair<double, int>> key((size_t)nq * na);
                for (int a = 0; a < na; ++a)
                    for (int qd = 0; qd < nq; ++qd) {
                        int ck = 0;
                        while (last && !fwd_rowstages_ && ck + 1 < pipe_chunks_ && a >= pipe_angle(ck + 1)) ++ck;
                        key[(size_t)a * nq + qd] = {1e9 * ck - chord[(size_t)a * nq + qd], qd + nq * a};
                    }
                std::stable_sort(key.begin(), key.end());
                for (auto& kv : key) orders.push_back(kv.second);
                fstages_.push_back(f);
            }
            KCT_CUDA(cudaMalloc(&d_fstage_, orders.size() * sizeof(int)));
            KCT_CUDA(cudaMemcpy(d_fstage_, orders.data(), orders.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
    }
    const int kc = (nz + 31) / 32;
    adj_k_ = kc <= 1 ? 1 : kc <= 2 ? 2 : kc <= 4 ? 4 : 8;

    // brick adjoint: row stride S so that rows r and r+S of one pass never
    // touch the same slab (S * dkz_min > 1 + span_max).
    const double G_min = std::max(1e-12, (geom.dso - r_max) / (L_max * sz));
    const double dkz_min = geom.pv * G_min;
    const double span_max = dv_max / (L_min * sz) * std::hypot(sx, sy);
    int S = (int)std::ceil((1.0 + span_max) / dkz_min * 1.02 + 1e-9);
    S = std::max(S, 1);
    if (S > 64 || full_fp) adj_gather_ = true;  // degenerate geometry: use the gather kernel
    adj_S_ = S;
    // bricks <= 96 slabs tall, nz split evenly (c3: 3 x 86; measured against
    // 52..192 with the brick queue: shorter bricks pay more per-row z-state
    // initialisations per ray, taller ones cost occupancy and balance)
    {
        const int nbz = (nz + 95) / 96;
        adj_bz_ = (nz + nbz - 1) / nbz;
    }
    if (const char* e = std::getenv("KCT_ADJ_BZ")) adj_bz_ = std::clamp(std::atoi(e), 1, kMaxBz);
    // slab-lane deposits (brick_rows_slab): a row's z-span over a brick chord
    // below one slab and below the row spacing, rows two apart more than one
    // slab apart (c1-c5: spans 0.18-0.58, spacings 0.61-0.97 slabs)
    {
        const double span_brick = dv_max / (L_min * sz) * std::hypot(BX * sx, BY * sy);
        adj_slab_ = span_brick < 0.9 && span_brick < 0.97 * dkz_min && dkz_min > 0.55 &&
                    adj_bz_ + 2 <= 32 * kSlabChunks;
        // a falling and a rising row next to each other (around dv = 0) can
        // claim one crossing slot only if the row spacing can reach one slab
        const double G_max = (geom.dso + r_max) / (L_min * sz);
        adj_slab_detect_ = geom.pv * G_max > 0.98;
        const char* e = std::getenv("KCT_ADJ_SLAB");
        if (e && std::string(e) == "0") adj_slab_ = false;
        if (e && std::string(e) == "force" && !adj_slab_)
            throw ConfigError("KCT_ADJ_SLAB=force: slab-lane adjoint not valid for this geometry");
    }

    KCT_CUDA(cudaMalloc(&d_cols_, cols.size() * sizeof(ColParams)));
    KCT_CUDA(cudaMemcpy(d_cols_, cols.data(), cols.size() * sizeof(ColParams), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_dv_, nv * sizeof(float)));
    KCT_CUDA(cudaMemcpy(d_dv_, dv.data(), nv * sizeof(float), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_invdv_, nv * sizeof(float)));
    KCT_CUDA(cudaMemcpy(d_invdv_, invdv.data(), nv * sizeof(float), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_dvd_, nv * sizeof(double)));
    KCT_CUDA(cudaMemcpy(d_dvd_, dvd.data(), nv * sizeof(double), cudaMemcpyHostToDevice));
    {
        std::vector<RowTab> rt(nv);
        for (int iv = 0; iv < nv; ++iv) rt[iv] = RowTab{dvd[iv], dv[iv], invdv[iv]};
        KCT_CUDA(cudaMalloc(&d_rows_, nv * sizeof(RowTab)));
        KCT_CUDA(cudaMemcpy(d_rows_, rt.data(), nv * sizeof(RowTab), cudaMemcpyHostToDevice));
    }
    // the attribute is per function, not per handle: set it to the largest
    // brick any projector can use, so handles with taller bricks coexist
    const int smem_max = (int)((size_t)kAdjWarps * adj_warp_floats(kMaxBz) * sizeof(float));
    KCT_CUDA(cudaFuncSetAttribute(adj_brick_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    KCT_CUDA(cudaFuncSetAttribute(adj_brick_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    for (auto fn : {adj_mirror_kernel<0>, adj_mirror_kernel<32>, adj_mirror_kernel<64>})
        KCT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(adj_mir_floats(kMirMaxBz) * sizeof(float))));
    for (int np : {1, 2, 3})
        for (int bz : {0, 32, 64})
            KCT_CUDA(cudaFuncSetAttribute(adj_ws_fn(bz, np), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(adj_mir_ws_floats(kMirMaxBz, np) * sizeof(float))));

    // z-mirror brick pairs (adj_mirror_kernel): z-mirror geometry, slab-lane
    // conditions, nz even; bricks of <= 64 slabs tiling the lower half
    // (KCT_ADJ_MIR_BZ: another maximum height, <= 128; KCT_ADJ_MIRROR=0: off)
    {
        const char* e = std::getenv("KCT_ADJ_MIRROR");
        adj_mir_ = mirror_ && adj_slab_ && !adj_gather_ && nz % 2 == 0 && kTabOk &&
                   !(e && e[0] == '0');
        int hmax = 64;
        if (const char* h = std::getenv("KCT_ADJ_MIR_BZ")) hmax = std::clamp(std::atoi(h), 1, kMirMaxBz);
        const int half = nz / 2, nbh = (half + hmax - 1) / std::max(1, hmax);
        adj_mbz_ = std::max(1, (half + nbh - 1) / std::max(1, nbh));
    }

    // y parts per z level whose completion the host path tracks separately
    // (adjoint_host_ref copies a (level, part) out as soon as it is final:
    // the last level's copy is then mostly overlapped too)
    {
        adj_parts_ = 6;  // re-swept with the 1.96 ms kernel: 2 / 4 / 6 / 8 -> host adjoint 2.86 / 2.75 / 2.72 / 2.72 ms
        if (const char* e = std::getenv("KCT_ADJ_PARTS")) adj_parts_ = std::max(1, std::atoi(e));
        adj_parts_ = std::min(adj_parts_, (ny + BY - 1) / BY);
    }

    KCT_CUDA(cudaMalloc(&d_cs_, cs_.size() * sizeof(float2)));
    KCT_CUDA(cudaMemcpy(d_cs_, cs_.data(), cs_.size() * sizeof(float2), cudaMemcpyHostToDevice));
    build_walk_table();
    if (!d_tab_) adj_mir_ = false;  // the pair kernel streams the walk table
    build_fwd_table();

    const BrickCfg bcfg = adj_cfg();
    const long nb = (long)bcfg.nbx * bcfg.nby * bcfg.nbz;
    // angle groups for problems with few bricks (see adj_brick_kernel); a
    // function of the problem size only, so results do not depend on the device
    {
        const int amax = std::min(na, kMaxAnglesPerLaunch);
        // one item per brick once the bricks fill a 148-SM B200 twice (measured:
        // c3's 12288 bricks run 3% faster undivided); otherwise ~4 items per
        // resident warp (c2, slabs of multi-GPU shards, c1); a brick pair
        // counts as two bricks
        constexpr long kWarpSlots = 148 * 32;
        const long nbw = adj_mir_ ? 2 * nb : nb;
        int G = nbw >= 2 * kWarpSlots ? 1 : (int)std::min<long>(16, (4 * kWarpSlots + nbw - 1) / nbw);
        if (const char* e = std::getenv("KCT_ADJ_GROUPS")) G = std::max(1, std::atoi(e));
        G = std::max(1, std::min(G, amax));
        // partial volumes: (G - 1) x M floats, capped at 2 GiB
        while (G > 1 && (size_t)(G - 1) * m_ * sizeof(float) > (2ull << 30)) --G;
        if (adj_gather_) G = 1;
        adj_groups_ = G;
        if (G > 1) KCT_CUDA(cudaMalloc(&d_part_, (size_t)(G - 1) * m_ * sizeof(float)));
    }

    if (!adj_gather_)
        KCT_CUDA(cudaMalloc(&d_yw_, (size_t)std::min(na, kMaxAnglesPerLaunch) * nu * nv * sizeof(float4)));

    // brick queue: persistent grid of resident CTAs, bricks heaviest first
    // (by xy distance of the brick centre from the rotation axis, then by z
    // distance from the mid-plane: central bricks are crossed by the most rays)
    const char* sched = std::getenv("KCT_ADJ_SCHED");
    if (!adj_gather_ && !(sched && std::string(sched) == "static")) {
        const int nbx = bcfg.nbx, nby = bcfg.nby;
        std::vector<std::pair<double, int>> key(nb);
        const char* zo = std::getenv("KCT_ADJ_ORDER");
        const bool z_major = !(zo && std::string(zo) == "radius");
        for (int b = 0; b < (int)nb; ++b) {
            const int bi = b % nbx, bj = (b / nbx) % nby, bk = b / (nbx * nby);
            const double cx = ox + (bi + 0.5) * BX * sx, cy = oy + (bj + 0.5) * BY * sy;
            const double cz = grid_.oz + (bk + 0.5) * bcfg.bz * sz;
            key[b] = {std::hypot(cx, cy) + 1e-3 * std::fabs(cz), b};
            // z levels in turn: the detector rows they read stay in L2 (c4 -1%)
            if (z_major) key[b].first += 1e6 * bk;
        }
        std::vector<std::pair<double, int>> hkey = key;
        std::stable_sort(key.begin(), key.end());
        std::vector<int> order(nb);
        for (int b = 0; b < (int)nb; ++b) order[b] = key[b].second;
        KCT_CUDA(cudaMalloc(&d_border_, 2 * nb * sizeof(int)));
        KCT_CUDA(cudaMemcpy(d_border_, order.data(), nb * sizeof(int), cudaMemcpyHostToDevice));
        // the host path's order: within a level the y parts in turn (it copies
        // a (level, part) out as soon as it is final), heaviest first in a
        // part (measured: costs the kernel itself 3%, so device calls keep
        // the order above)
        for (int b = 0; b < (int)nb; ++b) {
            const int bj = (b / nbx) % nby;
            hkey[b].first += 1e4 * (double)(bj * adj_parts_ / nby);
        }
        std::stable_sort(hkey.begin(), hkey.end());
        for (int b = 0; b < (int)nb; ++b) order[b] = hkey[b].second;
        KCT_CUDA(cudaMemcpy(d_border_ + nb, order.data(), nb * sizeof(int), cudaMemcpyHostToDevice));
        KCT_CUDA(cudaMalloc(&d_queue_, sizeof(int)));
        // warp-specialised brick pairs (adj_mirror_ws_kernel; KCT_ADJ_WS=0: one warp per pair)
        const char* ws = std::getenv("KCT_ADJ_WS");
        adj_ws_ = adj_mir_ && !(ws && ws[0] == '0');
        int per_sm = 0, sms = 0;
        KCT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
        if (adj_ws_) {
            for (int np : {1, 2, 3}) {
                KCT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &per_sm, adj_ws_fn(0, np), 32 * (np + KCT_MIR_NC),
                    (size_t)adj_mir_ws_floats(adj_mbz_, np) * sizeof(float)));
                adj_ctas_np_[np - 1] = std::max(1, per_sm) * std::max(1, sms);
            }
            per_sm = adj_ctas_np_[adj_np_ - 1] / std::max(1, sms);
        } else if (adj_mir_)
            KCT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adj_mirror_kernel<0>, 32,
                                                                   adj_smem_bytes()));
        else
            KCT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adj_brick_kernel<true>,
                                                                   kAdjWarps * 32, adj_smem_bytes()));
        adj_ctas_ = std::max(1, per_sm) * std::max(1, sms);
    }
    tune_adjoint();
}

// Brick configuration of the adjoint (and of its walk table): standard
// bricks of adj_bz_ slabs tiling [0, nz), or (adj_mir_) z-mirror pairs whose
// lower bricks of adj_mbz_ slabs tile [0, nz/2).
BrickCfg Projector::adj_cfg() const {
    BrickCfg bc{};
    bc.mirror = adj_mir_ ? 1 : 0;
    bc.bz = adj_mir_ ? adj_mbz_ : adj_bz_;
    bc.S = adj_S_;
    bc.slab = adj_slab_ ? (adj_slab_detect_ && !adj_mir_ ? 2 : 1) : 0;
    bc.nbx = (dg_.nx + BX - 1) / BX;
    bc.nby = (dg_.ny + BY - 1) / BY;
    const int zext = adj_mir_ ? dg_.nz / 2 : dg_.nz;
    bc.nbz = (zext + bc.bz - 1) / bc.bz;
    bc.ngrp = adj_groups_;
    bc.gstride = m_;
    bc.nparts = adj_parts_;
    return bc;
}

// Walk table (adj_walk_build): the xy part of every (brick, angle, column) of
// the adjoint, 64 bytes each, built once per projector.  Skipped (the adjoint
// then recomputes the walks) when disabled (KCT_ADJ_TABLE=0), when an index
// does not fit the entry, or above the memory budget (KCT_ADJ_TABLE_MB,
// default a quarter of the free device memory).
void Projector::build_walk_table() {
    const char* en = std::getenv("KCT_ADJ_TABLE");
    if (adj_gather_ || !kTabOk || (en && std::string(en) == "0")) return;
    if (dg_.na > 65535 || dg_.nu > 65535 || dg_.nv > 65535) return;
    // budget: a quarter of the free device memory (B200: ~45 GB, enough for
    // c4's 720-view prior, 28 GB), or KCT_ADJ_TABLE_MB
    size_t free_b = 0, total_b = 0;
    KCT_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t budget = free_b / 4;
    if (const char* e = std::getenv("KCT_ADJ_TABLE_MB")) budget = (size_t)std::atoll(e) << 20;
    BrickCfg bc = adj_cfg();
    bc.ngrp = 1;
    const size_t nb = (size_t)bc.nbx * bc.nby * bc.nbz;
    const size_t noff = nb * (dg_.na + 1);
    const float2* d_cs = d_cs_;
    KCT_CUDA(cudaMalloc(&d_off_, noff * sizeof(unsigned long long)));
    const unsigned blocks = (unsigned)((nb + 3) / 4);
    adj_walk_build<false><<<blocks, 128>>>(d_cols_, d_cs, dg_, bc, d_off_, nullptr);
    KCT_LAUNCHED();
    std::vector<unsigned long long> off(noff);
    KCT_CUDA(cudaMemcpy(off.data(), d_off_, noff * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    // per brick: counts per angle -> exclusive prefix over (brick, angle)
    unsigned long long tot = 0;
    for (size_t b = 0; b < nb; ++b) {
        unsigned long long* ob = off.data() + b * (dg_.na + 1);
        for (int a = 0; a < dg_.na; ++a) {
            const unsigned long long c = ob[a];
            ob[a] = tot;
            tot += c;
        }
        ob[dg_.na] = tot;
    }
    if (tot == 0 || tot * sizeof(WalkEntry) > budget) {
        cudaFree(d_off_);
        d_off_ = nullptr;
        return;
    }
    KCT_CUDA(cudaMemcpy(d_off_, off.data(), noff * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_tab_, tot * sizeof(WalkEntry)));
    adj_walk_build<true><<<blocks, 128>>>(d_cols_, d_cs, dg_, bc, d_off_,
                                          static_cast<WalkEntry*>(d_tab_));
    KCT_LAUNCHED();
    KCT_CUDA(cudaDeviceSynchronize());
    tab_entries_ = tot;
}

// Forward walk table (fwd_tab_build): every (angle, column)'s xy segments,
// 8 bytes each (c3: 8.2 M segments = 66 MB), built once per projector; the
// forward then loads 32 segments per coalesced load instead of stepping the
// walk (plane crossings in float64, voxel indices, exits) per segment.
// Skipped (on-the-fly walks) with KCT_FWD_TABLE=0, or above the budget
// KCT_FWD_TABLE_MB (default an eighth of the free device memory).
void Projector::build_fwd_table() {
    const char* en = std::getenv("KCT_FWD_TABLE");
    if (en && en[0] == '0') return;
    const size_t ncol = (size_t)dg_.na * dg_.nu;
    unsigned* cnt = nullptr;
    KCT_CUDA(cudaMalloc(&cnt, ncol * sizeof(unsigned)));
    const unsigned blocks = (unsigned)((ncol + 127) / 128);
    fwd_tab_build<false><<<blocks, 128>>>(d_cols_, dg_, cnt, nullptr, nullptr);
    KCT_LAUNCHED();
    std::vector<unsigned> c(ncol);
    KCT_CUDA(cudaMemcpy(c.data(), cnt, ncol * sizeof(unsigned), cudaMemcpyDeviceToHost));
    cudaFree(cnt);
    std::vector<unsigned> off(ncol + 1);
    unsigned long long tot = 0;
    for (size_t t = 0; t < ncol; ++t) {
        off[t] = (unsigned)tot;
        tot += c[t];
    }
    off[ncol] = (unsigned)tot;
    size_t free_b = 0, total_b = 0;
    KCT_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t budget = free_b / 8;
    if (const char* e = std::getenv("KCT_FWD_TABLE_MB")) budget = (size_t)std::atoll(e) << 20;
    if (tot == 0 || tot >= (1ull << 32) || tot * sizeof(int2) > budget) return;
    KCT_CUDA(cudaMalloc(&d_ftab_off_, (ncol + 1) * sizeof(unsigned)));
    KCT_CUDA(cudaMemcpy(d_ftab_off_, off.data(), (ncol + 1) * sizeof(unsigned), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_ftab_, tot * sizeof(int2)));
    fwd_tab_build<true><<<blocks, 128>>>(d_cols_, dg_, nullptr, d_ftab_off_,
                                         static_cast<int2*>(d_ftab_));
    KCT_LAUNCHED();
    KCT_CUDA(cudaDeviceSynchronize());
    ftab_segs_ = tot;
}

size_t Projector::adj_smem_bytes() const {
    if (adj_ws_) return (size_t)adj_mir_ws_floats(adj_mbz_, adj_np_) * sizeof(float);
    if (adj_mir_) return (size_t)adj_mir_floats(adj_mbz_) * sizeof(float);
    return (size_t)kAdjWarps * adj_warp_floats(adj_bz_) * sizeof(float);
}

// Adjoint per-ray records (row_init): yw = y * sqrt(1 + (dv * inv_l)^2), the
// 3D length factor of each ray (the forward's final scale), applied once per
// ray instead of once per (ray, brick), and the ray's z state (k0, f0, imk)
// evaluated exactly as fwd_kernel does.  Native layout, one thread per ray.
__global__ void __launch_bounds__(256) adj_weight_kernel(const float* __restrict__ y,
                                                         float4* __restrict__ rec,
                                                         const ColParams* __restrict__ cols,
                                                         const RowTab* __restrict__ rows, DevGeom g,
                                                         size_t ncols) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const int nv = g.nv;
    const size_t col = t / (size_t)nv;
    if (col >= ncols) return;
    const int iv = (int)(t - col * (size_t)nv);
    // z-mirror geometry (fwd_kernel MIR): a row of the upper half is the
    // reflection of row nv-1-iv, whose z state it takes, reflected:
    // k0' = nz - k0, f0' = -f0, imk' = -imk, kstep +1 — then zcross(P') is
    // bit-identical to the primary's zcross(nz - P') (the forward's crossings)
    const bool mirror = g.mirror && iv >= nv / 2;
    const RowTab rt = ld_row(rows, mirror ? nv - 1 - iv : iv);
    const float inv_l = cols[col].inv_l, inv_h1 = cols[col].inv_h1;
    const double g_in = cols[col].g_in;
    const float q = rt.dv * inv_l;
    const double kzd = fma(rt.dvd, g_in, -g.kz0d);
    const double fl = floor(kzd);
    const int k0 = (int)fmax(fmin(fl, (double)(1 << 28)), -(double)(1 << 28));
    const int ks = rt.dv > 0.f ? 1 : rt.dv < 0.f ? -1 : 0;
    float4 r;
    r.x = y[t] * __fsqrt_rn(__fmaf_rn(q, q, 1.f));
    const float f0 = (float)(kzd - fl), imk = __fmul_rn(rt.invdv, inv_h1);
    if (mirror) {
        r.y = -f0;
        r.z = -imk;
        r.w = __int_as_float((g.nz - k0) * 4 + 2);
    } else {
        r.y = f0;
        r.z = imk;
        r.w = __int_as_float(k0 * 4 + ks + 1);
    }
    rec[t] = r;
}

// The same records for adj_mirror_kernel, one thread per row pair: the
// primary row p < nv/2's record (float4, [column][p]) and the weight of its
// mirror row nv-1-p (float, [column][p]; its 3D length factor is the
// primary's: dv(nv-1-p) = -dv(p)).
__global__ void __launch_bounds__(256) adj_weight_mir_kernel(const float* __restrict__ y,
                                                             float4* __restrict__ rec,
                                                             float* __restrict__ ymw,
                                                             const ColParams* __restrict__ cols,
                                                             const RowTab* __restrict__ rows,
                                                             DevGeom g, size_t ncols) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const int nh = g.nv / 2;
    const size_t col = t / (size_t)nh;
    if (col >= ncols) return;
    const int p = (int)(t - col * (size_t)nh);
    const RowTab rt = ld_row(rows, p);
    const float inv_l = cols[col].inv_l, inv_h1 = cols[col].inv_h1;
    const double g_in = cols[col].g_in;
    const float q = rt.dv * inv_l;
    const double kzd = fma(rt.dvd, g_in, -g.kz0d);
    const double fl = floor(kzd);
    const int k0 = (int)fmax(fmin(fl, (double)(1 << 28)), -(double)(1 << 28));
    const int ks = rt.dv > 0.f ? 1 : rt.dv < 0.f ? -1 : 0;
    const float f = __fsqrt_rn(__fmaf_rn(q, q, 1.f));
    const float* yc = y + col * (size_t)g.nv;
    float4 r;
    r.x = yc[p] * f;
    r.y = (float)(kzd - fl);
    r.z = __fmul_rn(rt.invdv, inv_h1);
    r.w = __int_as_float(k0 * 4 + ks + 1);
    rec[t] = r;
    ymw[t] = yc[g.nv - 1 - p] * f;
}

// out += part[0] + part[1] + ... (fixed order: deterministic)
__global__ void __launch_bounds__(256) adj_group_sum(float* __restrict__ out,
                                                     const float* __restrict__ part, int nparts,
                                                     size_t m, size_t stride) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m;
         i += (size_t)gridDim.x * blockDim.x) {
        float v = out[i];
        for (int g = 0; g < nparts; ++g) v += part[(size_t)g * stride + i];
        out[i] = v;
    }
}

// ---- launches -----------------------------------------------------------------
template <bool COUNT, bool MIR, bool DONE, bool TAB, bool REF = false>
static void launch_fwd_c(int C, dim3 g1, int th, cudaStream_t s, const float* vol, float* out,
                         const ColParams* cols, const float* dv, const float* invdv,
                         const double* dvd, const DevGeom& gg, const int* order, const FwdChunks& fc,
                         const FwdTab& tab) {
    switch (C) {
    case 1: fwd_kernel<1, COUNT, DONE, MIR, TAB, REF><<<g1, th, 0, s>>>(vol, out, cols, dv, invdv, dvd, gg, order, fc, tab); break;
    case 2: fwd_kernel<2, COUNT, DONE, MIR, TAB, REF><<<g1, th, 0, s>>>(vol, out, cols, dv, invdv, dvd, gg, order, fc, tab); break;
    case 3: fwd_kernel<3, COUNT, DONE, MIR, TAB, REF><<<g1, th, 0, s>>>(vol, out, cols, dv, invdv, dvd, gg, order, fc, tab); break;
    default: fwd_kernel<4, COUNT, DONE, MIR, TAB, REF><<<g1, th, 0, s>>>(vol, out, cols, dv, invdv, dvd, gg, order, fc, tab); break;
    }
    KCT_LAUNCHED();
}

// tab.off == nullptr: walk the columns on the fly; tab.off / cols point at
// the launch's first angle.
template <bool COUNT, bool MIR>
static void launch_fwd_t(int C, int bands, int band0, const float* vol, float* out,
                         const ColParams* cols, const float* dv, const float* invdv,
                         const double* dvd, const DevGeom& g, const int* order, cudaStream_t s,
                         const FwdChunks* done, const FwdTab& tab) {
    // 1D grid over (angle, band, column quad) items
    const unsigned nq = (unsigned)((g.nu + kFwdWarps - 1) / kFwdWarps);
    const dim3 g1(nq * (unsigned)bands * (unsigned)g.na, 1, 1);
    const int th = kFwdWarps * 32;
    DevGeom gg = g;
    gg.fwd_bands = bands;
    gg.fwd_band0 = band0;
    FwdChunks fc{};
    if (done) fc = *done;
    const bool tb = !COUNT && tab.off;
    if (!COUNT && gg.out_ref) {  // staged host forward: reference-layout output
        if (done) {
            if (tb) launch_fwd_c<false, MIR, true, true, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
            else launch_fwd_c<false, MIR, true, false, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
        } else {
            if (tb) launch_fwd_c<false, MIR, false, true, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
            else launch_fwd_c<false, MIR, false, false, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
        }
        return;
    }
    if (!COUNT && done) {  // host pipeline (counted launch)
        if (tb) launch_fwd_c<false, MIR, true, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
        else launch_fwd_c<false, MIR, true, false>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
        return;
    }
    if (tb) launch_fwd_c<false, MIR, false, true>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
    else launch_fwd_c<COUNT, MIR, false, false>(C, g1, th, s, vol, out, cols, dv, invdv, dvd, gg, order, fc, tab);
}

template <bool COUNT>
static void launch_fwd(int C, int bands, int band0, const float* vol, float* out, const ColParams* cols,
                       const float* dv, const float* invdv, const double* dvd, const DevGeom& g,
                       const int* order, cudaStream_t s, const FwdChunks* done = nullptr,
                       const FwdTab& tab = FwdTab{nullptr, nullptr}) {
    if (g.mirror)
        launch_fwd_t<COUNT, true>(C, bands, band0, vol, out, cols, dv, invdv, dvd, g, order, s, done, tab);
    else
        launch_fwd_t<COUNT, false>(C, bands, band0, vol, out, cols, dv, invdv, dvd, g, order, s, done, tab);
}

// the forward walk table from angle a on (none: FwdTab{} -> on-the-fly walks)
FwdTab Projector::ftab(int a) const {
    if (!d_ftab_off_) return FwdTab{nullptr, nullptr};
    return FwdTab{d_ftab_off_ + (size_t)a * dg_.nu, reinterpret_cast<const int2*>(d_ftab_)};
}

void Projector::forward(const float* vol, float* proj, cudaStream_t s) const {
    pad_volume(vol, s);
    forward_padded(proj, 0, dg_.na, s);
}

void Projector::forward_range(const float* vol, float* proj, int a_begin, int a_end,
                              cudaStream_t s) const {
    pad_volume(vol, s);
    forward_padded(proj, a_begin, a_end, s);
}

// Split-upload forward (capi.cu forward_host_pipelined): band 0 (its rays
// stay below slab fwd_split_z_) for all angles, or bands 1.. for angles
// [a_begin, a_end) — with the block orders built for these launches.
void Projector::forward_split_lo(float* proj, cudaStream_t s) const {
    launch_fwd<false>(fwd_c_, 1, 0, d_vpad_ + kVOff, proj, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, d_flo_, s,
                      nullptr, ftab(0));
}
void Projector::forward_split_hi(float* proj, int c, cudaStream_t s) const {
    const int a0 = pipe_angle(c), a1 = pipe_angle(c + 1);
    DevGeom g = dg_;
    g.na = a1 - a0;
    launch_fwd<false>(fwd_c_, fwd_bands_ - 1, 1, d_vpad_ + kVOff, proj + (size_t)a0 * dg_.nu * dg_.nv,
                      d_cols_ + (size_t)a0 * dg_.nu, d_dv_, d_invdv_, d_dvd_, g,
                      d_fhi_ + fhi_off_[c], s, nullptr, ftab(a0));
}
// Host pipeline, one launch: bands band0.. of every angle in chunk-major
// block order, counting finished columns per pipeline chunk into `done`
// (expected counts: fwd_chunk_columns); with the split upload band0 = 1 (band
// 0 ran before), else 0.
void Projector::forward_counted(float* proj, int band0, unsigned* done, cudaStream_t s) const {
    FwdChunks fc{};
    fc.count = done;
    fc.n = pipe_chunks_;
    for (int c = 0; c <= pipe_chunks_; ++c) fc.cb[c] = pipe_angle(c);
    launch_fwd<false>(fwd_c_, fwd_bands_ - band0, band0, d_vpad_ + kVOff, proj, d_cols_, d_dv_,
                      d_invdv_, d_dvd_, dg_, band0 ? d_fcnt_hi_ : d_fcnt_all_, s, &fc, ftab(0));
}
// Stage `stage` of the staged host forward (one band: C chunks from row0),
// counted per pipeline chunk when `done` is set.
void Projector::forward_stage(int stage, float* proj, unsigned* done, cudaStream_t s,
                              bool ref_out) const {
    const FwdStage& f = fstages_[stage];
    DevGeom g = dg_;
    g.fwd_row0 = f.row0;
    g.out_ref = ref_out ? 1 : 0;
    FwdChunks fc{};
    if (done) {
        fc.count = done;
        fc.n = pipe_chunks_;
        for (int c = 0; c <= pipe_chunks_; ++c) fc.cb[c] = pipe_angle(c);
    }
    launch_fwd<false>(f.C, 1, 0, d_vpad_ + kVOff, proj, d_cols_, d_dv_, d_invdv_, d_dvd_, g,
                      d_fstage_ + f.order_off, s, done ? &fc : nullptr, ftab(0));
}

unsigned Projector::fwd_chunk_columns(int c, int band0) const {
    return (unsigned)((pipe_angle(c + 1) - pipe_angle(c)) * dg_.nu * (fwd_bands_ - band0));
}

// reference-layout slabs [z0, z1) straight into the padded native volume
void Projector::vol_to_padded_z(const float* ref, int z0, int z1, cudaStream_t s) const {
    const size_t plane = (size_t)dg_.nx * dg_.ny;
    launch_transpose(ref + (size_t)z0 * plane, d_vpad_ + kVOff + z0, 1, z1 - z0, (int)plane, s,
                     vpad_stride(dg_.nz));
}

// native volume -> padded copy (column stride vpad_stride(nz); the pad slabs
// stay 0): one warp per voxel column, float4 reads when nz % 4 == 0
__global__ void __launch_bounds__(256) pad_kernel(const float* __restrict__ nat,
                                                  float* __restrict__ pad, int nz, int ncols) {
    const int lane = threadIdx.x & 31;
    const int stride = vpad_stride(nz);
    for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < ncols;
         p += (gridDim.x * blockDim.x) >> 5) {
        const float* src = nat + (size_t)p * nz;
        float* dst = pad + (size_t)p * stride + kVOff;
        if ((nz & 3) == 0) {
            for (int q = lane; q < nz / 4; q += 32) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(src) + q);
                dst[4 * q] = v.x;
                dst[4 * q + 1] = v.y;
                dst[4 * q + 2] = v.z;
                dst[4 * q + 3] = v.w;
            }
        } else {
            for (int q = lane; q < nz; q += 32) dst[q] = __ldg(src + q);
        }
    }
}

void Projector::pad_volume(const float* nat, cudaStream_t s) const {
    pad_kernel<<<148 * 16, 256, 0, s>>>(nat, d_vpad_, dg_.nz, dg_.nx * dg_.ny);
    KCT_LAUNCHED();
}

void Projector::forward_padded(float* proj, int a_begin, int a_end, cudaStream_t s) const {
    const int* order = nullptr;
    if (a_begin == 0 && a_end == dg_.na) {
        order = d_forder_;
    } else {
        for (int c = 0; c < pipe_chunks_; ++c)
            if (pipe_angle(c) == a_begin && pipe_angle(c + 1) == a_end && d_fpipe_)
                order = d_fpipe_ + pipe_off_[c];
    }
    DevGeom g = dg_;
    g.na = a_end - a_begin;
    launch_fwd<false>(fwd_c_, fwd_bands_, 0, d_vpad_ + kVOff, proj + (size_t)a_begin * dg_.nu * dg_.nv,
                      d_cols_ + (size_t)a_begin * dg_.nu, d_dv_, d_invdv_, d_dvd_, g, order, s, nullptr,
                      ftab(a_begin));
}

cudaStream_t Projector::pipe_stream() {
    if (!pipe_stream_) {
        // highest priority: the copy stream's small layout-transpose kernels
        // are dispatched ahead of the pending blocks of the long operator
        // kernel on the compute stream, so each chunk's copy starts when the
        // chunk is done (not at the end of the next chunk's launch)
        int lo = 0, hi = 0;
        KCT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        KCT_CUDA(cudaStreamCreateWithPriority(&pipe_stream_, cudaStreamNonBlocking, hi));
        for (auto& e : pipe_ev_) KCT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        KCT_CUDA(cudaEventCreateWithFlags(&up_ev_, cudaEventDisableTiming));
    }
    return pipe_stream_;
}

void Projector::count(float* proj, cudaStream_t s) const {
    launch_fwd<true>(fwd_c_, fwd_bands_, 0, nullptr, proj, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_,
                     d_forder_, s);
}

void Projector::adjoint(const float* proj, float* vol, cudaStream_t s) const {
    adjoint_range(proj, vol, 0, dg_.na, false, s);
}

void Projector::adjoint_range(const float* proj, float* vol, int a_begin, int a_end,
                              bool accumulate, cudaStream_t s) const {
    adjoint_impl(proj, vol, a_begin, a_end, accumulate, false, nullptr, s);
}

void Projector::adjoint_impl(const float* proj, float* vol, int a_begin, int a_end,
                             bool accumulate, bool out_ref, unsigned* level_done,
                             cudaStream_t s) const {
    AngleBatch ab;
    BrickCfg bc = adj_cfg();
    bc.out_ref = out_ref ? 1 : 0;
    bc.level_done = level_done;
    const int nctas = (bc.nbx * bc.nby * bc.nbz * bc.ngrp + kAdjWarps - 1) / kAdjWarps;
    // the host path's brick order (y parts in turn within a z level) when it
    // tracks progress
    const int* border = d_border_ && level_done ? d_border_ + (size_t)bc.nbx * bc.nby * bc.nbz : d_border_;
    const size_t smem = adj_smem_bytes();
    for (int a0 = a_begin; a0 < a_end; a0 += kMaxAnglesPerLaunch) {
        const int nab = std::min(kMaxAnglesPerLaunch, a_end - a0);
        for (int q = 0; q < nab; ++q) ab.cs[q] = cs_[a0 + q];
        const int accum = (a0 > a_begin || accumulate) ? 1 : 0;
        const ColParams* cols = d_cols_ + (size_t)a0 * dg_.nu;
        const float* pr = proj + (size_t)a0 * dg_.nu * dg_.nv;
        const size_t nb = (size_t)nab * dg_.nu * dg_.nv;
        float4* const yrec = reinterpret_cast<float4*>(d_yw_);
        float* const ymw = d_yw_ + 2 * nb;  // after the nb / 2 primary records (adj_mir_)
        if (adj_mir_) {
            adj_weight_mir_kernel<<<(unsigned)((nb / 2 + 255) / 256), 256, 0, s>>>(
                pr, yrec, ymw, cols, d_rows_, dg_, (size_t)nab * dg_.nu);
            KCT_LAUNCHED();
        } else if (!adj_gather_) {
            adj_weight_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(
                pr, yrec, cols, d_rows_, dg_, (size_t)nab * dg_.nu);
            KCT_LAUNCHED();
        }
        if (adj_gather_) {
            const int K = adj_k_;
            dim3 grid((dg_.nx * dg_.ny + 3) / 4, (dg_.nz + 32 * K - 1) / (32 * K), 1);
            switch (K) {
            case 1: adj_gather_kernel<1><<<grid, 128, 0, s>>>(pr, vol, cols, d_dv_, d_invdv_, d_dvd_, dg_, ab, nab, accum); break;
            case 2: adj_gather_kernel<2><<<grid, 128, 0, s>>>(pr, vol, cols, d_dv_, d_invdv_, d_dvd_, dg_, ab, nab, accum); break;
            case 4: adj_gather_kernel<4><<<grid, 128, 0, s>>>(pr, vol, cols, d_dv_, d_invdv_, d_dvd_, dg_, ab, nab, accum); break;
            default: adj_gather_kernel<8><<<grid, 128, 0, s>>>(pr, vol, cols, d_dv_, d_invdv_, d_dvd_, dg_, ab, nab, accum); break;
            }
        } else {
            if (d_queue_) KCT_CUDA(cudaMemsetAsync(d_queue_, 0, sizeof(int), s));
            const unsigned grid = d_queue_ ? std::min(nctas, adj_ws_ ? adj_ctas_np_[adj_np_ - 1] : adj_ctas_)
                                           : nctas;
            if (adj_ws_)
                adj_ws_fn(bc.bz == 64 || bc.bz == 32 ? bc.bz : 0, adj_np_)
                    <<<grid, 32 * (adj_np_ + KCT_MIR_NC), smem, s>>>(
                    yrec, ymw, vol, dg_, bc, a0, nab, accum, border,
                    d_queue_, d_part_, static_cast<const WalkEntry*>(d_tab_), d_off_);
            else if (adj_mir_)
                (bc.bz == 64 ? adj_mirror_kernel<64> : bc.bz == 32 ? adj_mirror_kernel<32> : adj_mirror_kernel<0>)
                    <<<grid, 32, smem, s>>>(
                    yrec, ymw, vol, dg_, bc, a0, nab, accum, border,
                    d_queue_, d_part_, static_cast<const WalkEntry*>(d_tab_), d_off_);
            else if (d_tab_)
                adj_brick_kernel<true><<<grid, kAdjWarps * 32, smem, s>>>(
                    reinterpret_cast<const float4*>(d_yw_), vol, cols, dg_, bc, d_cs_ + a0, a0, nab, accum, border,
                    d_queue_, d_part_, static_cast<const WalkEntry*>(d_tab_), d_off_);
            else
                adj_brick_kernel<false><<<grid, kAdjWarps * 32, smem, s>>>(
                    reinterpret_cast<const float4*>(d_yw_), vol, cols, dg_, bc, d_cs_ + a0, a0, nab, accum, border,
                    d_queue_, d_part_, nullptr, nullptr);
            if (bc.ngrp > 1) {
                KCT_LAUNCHED();
                adj_group_sum<<<1184, 256, 0, s>>>(vol, d_part_, bc.ngrp - 1, m_, m_);
            }
        }
        KCT_LAUNCHED();
    }
}

// Producer warps per consumer of the warp-specialised adjoint: 2 or 3,
// whichever runs this handle's geometry faster (c3: 3 producers 1.96 vs 2.02
// ms, c4: 2 producers 13.2 vs 13.9 ms, c2: 2; one producer is slower
// everywhere: c3 2.55, c4 15.6 ms).  Timed once at creation on the
// first <= 24 angles with non-zero readings (both variants are bit-identical,
// so a noisy choice changes time, never results).  KCT_ADJ_NP=2|3 forces the
// choice, KCT_ADJ_TUNE=0 keeps 2.
void Projector::tune_adjoint() {
    if (!adj_ws_ || !d_queue_) return;
    if (const char* e = std::getenv("KCT_ADJ_NP")) {
        adj_np_ = std::clamp(std::atoi(e), 1, 3);
        return;
    }
    const char* te = std::getenv("KCT_ADJ_TUNE");
    if (te && te[0] == '0') return;
    const int na_t = std::min(dg_.na, 24);
    const size_t n_t = (size_t)na_t * dg_.nu * dg_.nv;
    if ((double)n_t * dg_.nz < 2e8) return;  // small problems: launch-bound either way
    float *y = nullptr, *v = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaMalloc(&y, n_t * sizeof(float)) != cudaSuccess || cudaMalloc(&v, m_ * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(y);
        return;  // no room to tune: keep the default
    }
    KCT_CUDA(cudaMemset(y, 0x3c, n_t * sizeof(float)));  // 0x3c3c3c3c = 0.0115f everywhere
    KCT_CUDA(cudaEventCreate(&e0));
    KCT_CUDA(cudaEventCreate(&e1));
    float best = 0.f;
    int best_np = adj_np_;
    for (int np : {2, 3}) {
        adj_np_ = np;
        adjoint_impl(y, v, 0, na_t, false, false, nullptr, nullptr);  // warm (table in L2 / TLB)
        KCT_CUDA(cudaEventRecord(e0, nullptr));
        for (int r = 0; r < 2; ++r) adjoint_impl(y, v, 0, na_t, false, false, nullptr, nullptr);
        KCT_CUDA(cudaEventRecord(e1, nullptr));
        KCT_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        KCT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (np == 2 || ms < 0.99f * best) {  // 3 producers must win by 1%
            best = ms;
            best_np = np;
        }
    }
    adj_np_ = best_np;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(y);
    cudaFree(v);
}

// cuStreamWaitValue32 (driver API, MemOp v2: supported by default since CUDA
// 11.7), resolved at run time through the runtime's entry-point query.
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value32() {
    static const WaitValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<WaitValue32Fn>(p);
    }();
    return fn;
}

bool Projector::stream_wait_geq(cudaStream_t sc, const unsigned* addr, unsigned value) const {
    if (!wait_value32()) return false;
    return wait_value32()((CUstream)sc, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ) ==
           CUDA_SUCCESS;
}

// Host-buffer adjoint, reference layouts: the projections arrive in two
// angle parts (the second part's upload overlaps the first part's adjoint,
// which the second launch accumulates onto), and the volume leaves the device
// z level by z level: the brick kernel writes the reference layout directly
// (a z level's slabs are contiguous there) and its last launch counts
// finished bricks per level; the copy stream waits on each level's counter
// (cuStreamWaitValue32) and copies the level to the host while the next
// levels are computed.  Same per-brick arithmetic as adjoint() (the two
// launches add the halves' partial sums); false when the configuration does
// not allow it (gather kernel, angle groups, several angle batches, no brick
// queue, no stream-wait support).
bool Projector::adjoint_host_ref(const float* host_proj, float* host, cudaStream_t s) {
    const char* e = std::getenv("KCT_ADJ_PROGRESSIVE");
    if (e && e[0] == '0') return false;
    if (adj_gather_ || adj_groups_ > 1 || dg_.na > kMaxAnglesPerLaunch || !d_queue_ || !wait_value32())
        return false;
    const BrickCfg bcfg = adj_cfg();
    const int nbz = bcfg.nbz, NP = bcfg.nparts, nslots = nbz * NP;
    if (!d_level_) KCT_CUDA(cudaMalloc(&d_level_, (size_t)nslots * sizeof(unsigned)));
    const size_t per = (size_t)dg_.nu * dg_.nv;
    float* tmp = scratch(2, n_);  // reference-layout projections
    float* q = scratch(1, n_);    // native projections
    float* dev = scratch(0, m_);  // reference-layout volume
    cudaStream_t sc = pipe_stream();
    const char* sp = std::getenv("KCT_ADJ_SPLIT");
#ifndef KCT_ADJ_FIRST_PART
// the first launch takes 1 / KCT_ADJ_FIRST_PART of the angles, so that it
// lasts about as long as the rest's upload (round 1, 4 ms kernel: 1/8 best;
// round 2, 2 ms kernel, c3 host adjoint over 1/2 .. 1/12: 3.12 / 2.91 / 2.82 /
// 2.86 / 2.97 / 3.03 ms -> 1/4; end of round 2 -> 1/5, below)
#define KCT_ADJ_FIRST_PART 5  // 1.96 ms kernel, 6 y parts: 1/3 .. 1/8 -> 2.84 / 2.76 / 2.72 / 2.79 / 2.89 ms
#endif
    int first_part = KCT_ADJ_FIRST_PART;
    if (const char* fp = std::getenv("KCT_ADJ_FIRST_PART")) first_part = std::max(1, std::atoi(fp));
    const int H = (dg_.na >= 4 * kPipeMinAngles && !(sp && sp[0] == '0'))
                      ? std::max(1, dg_.na / first_part)
                      : dg_.na;
    const char* tre = std::getenv("KCT_TRACE");
    const bool trace = tre && tre[0] == '1';
    std::vector<std::pair<std::string, cudaEvent_t>> tev;
    cudaEvent_t tr0 = nullptr;
    auto mark = [&](const std::string& name, cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        tev.emplace_back(name, ev);
    };
    if (trace) {
        cudaEventCreate(&tr0);
        cudaEventRecord(tr0, s);
    }
    KCT_CUDA(cudaMemcpyAsync(tmp, host_proj, H * per * sizeof(float), cudaMemcpyHostToDevice, s));
    mark("up0", s);
    KCT_CUDA(cudaMemsetAsync(d_level_, 0, (size_t)nslots * sizeof(unsigned), s));
    KCT_CUDA(cudaEventRecord(pipe_ev_[0], s));  // copy stream: after this call's earlier work
    KCT_CUDA(cudaStreamWaitEvent(sc, pipe_ev_[0], 0));  // and sees the reset counters
    if (H < dg_.na)
        KCT_CUDA(cudaMemcpyAsync(tmp + H * per, host_proj + H * per, (dg_.na - H) * per * sizeof(float),
                                 cudaMemcpyHostToDevice, sc));
    KCT_CUDA(cudaEventRecord(up_ev_, sc));
    mark("up1", sc);
    proj_to_native_range(tmp, q, 0, H, s);
    if (H < dg_.na) {
        adjoint_impl(q, dev, 0, H, false, true, nullptr, s);
        mark("adj0", s);
        KCT_CUDA(cudaStreamWaitEvent(s, up_ev_, 0));
        proj_to_native_range(tmp, q, H, dg_.na, s);
    }
    adjoint_impl(q, dev, H < dg_.na ? H : 0, dg_.na, H < dg_.na, true, d_level_, s);
    mark("adj1", s);
    const size_t plane = (size_t)dg_.nx * dg_.ny;
    // (level L, y part q): brick rows bj with bj * NP / nby == q, i.e. voxel
    // rows [J0, J1) of slabs [k0, k1) (and, with z-mirror pairs, of their
    // reflection): one strided copy per z range
    const int nby = bcfg.nby;
    const size_t zext = adj_mir_ ? dg_.nz / 2 : dg_.nz;
    for (int L = 0; L < nbz; ++L) {
        for (int q = 0; q < NP; ++q) {
            const int bj0 = (q * nby + NP - 1) / NP, bj1 = ((q + 1) * nby + NP - 1) / NP;
            if (bj1 <= bj0) continue;
            const unsigned want = (unsigned)(bcfg.nbx * (bj1 - bj0));
            const CUresult r = wait_value32()((CUstream)sc, (CUdeviceptr)(d_level_ + L * NP + q), want,
                                              CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) {  // fall back: whole volume after the kernel
                KCT_CUDA(cudaStreamSynchronize(s));
                KCT_CUDA(cudaStreamSynchronize(sc));
                KCT_CUDA(cudaMemcpy(host, dev, m_ * sizeof(float), cudaMemcpyDeviceToHost));
                return true;
            }
            const size_t J0 = (size_t)bj0 * BY, J1 = std::min((size_t)dg_.ny, (size_t)bj1 * BY);
            const size_t k0 = (size_t)L * bcfg.bz, k1 = std::min(zext, k0 + bcfg.bz);
            const size_t row0 = J0 * dg_.nx, width = (J1 - J0) * dg_.nx * sizeof(float);
            const size_t pitch = plane * sizeof(float);
            KCT_CUDA(cudaMemcpy2DAsync(host + k0 * plane + row0, pitch, dev + k0 * plane + row0, pitch,
                                       width, k1 - k0, cudaMemcpyDeviceToHost, sc));
            if (adj_mir_) {
                const size_t u0 = dg_.nz - k1;
                KCT_CUDA(cudaMemcpy2DAsync(host + u0 * plane + row0, pitch, dev + u0 * plane + row0,
                                           pitch, width, k1 - k0, cudaMemcpyDeviceToHost, sc));
            }
            mark("L" + std::to_string(L) + "p" + std::to_string(q), sc);
        }
    }
    KCT_CUDA(cudaStreamSynchronize(sc));
    KCT_CUDA(cudaStreamSynchronize(s));
    if (trace) {
        std::string line = "[kct trace] adjoint_host_ref:";
        for (auto& [name, ev] : tev) {
            float ms = 0.f;
            cudaEventSynchronize(ev);
            cudaEventElapsedTime(&ms, tr0, ev);
            char buf[64];
            std::snprintf(buf, sizeof buf, " %s=%.3f", name.c_str(), ms);
            line += buf;
            cudaEventDestroy(ev);
        }
        cudaEventDestroy(tr0);
        std::fprintf(stderr, "%s\n", line.c_str());
    }
    return true;
}

void Projector::vol_to_native(const float* ref, float* nat, cudaStream_t s) const {
    // ref [k][p] (p = i + nx*j) -> native [p][k]
    launch_transpose(ref, nat, 1, dg_.nz, dg_.nx * dg_.ny, s);
}
void Projector::vol_from_native(const float* nat, float* ref, cudaStream_t s) const {
    launch_transpose(nat, ref, 1, dg_.nx * dg_.ny, dg_.nz, s);
}
void Projector::proj_to_native(const float* ref, float* nat, cudaStream_t s) const {
    // ref [a][iv][iu] -> native [a][iu][iv]
    launch_transpose(ref, nat, dg_.na, dg_.nv, dg_.nu, s);
}
void Projector::proj_from_native(const float* nat, float* ref, cudaStream_t s) const {
    launch_transpose(nat, ref, dg_.na, dg_.nu, dg_.nv, s);
}
void Projector::proj_to_native_range(const float* ref, float* nat, int a0, int a1,
                                     cudaStream_t s) const {
    const size_t off = (size_t)a0 * dg_.nu * dg_.nv;
    launch_transpose(ref + off, nat + off, a1 - a0, dg_.nv, dg_.nu, s);
}
// detector rows [v0, v1) of every angle: native [a][iu][iv] -> reference [a][iv][iu]
void Projector::proj_rows_from_native(const float* nat, float* ref, int v0, int v1,
                                      cudaStream_t s) const {
    if (v1 <= v0) return;
    const size_t per = (size_t)dg_.nu * dg_.nv;
    dim3 grid((v1 - v0 + 31) / 32, (dg_.nu + 31) / 32, dg_.na);
    transpose_sub_kernel<<<grid, dim3(32, 8), 0, s>>>(nat + v0, ref + (size_t)v0 * dg_.nu, dg_.nu,
                                                     v1 - v0, dg_.nv, dg_.nu, per, per);
    KCT_LAUNCHED();
}
void Projector::proj_from_native_range(const float* nat, float* ref, int a0, int a1,
                                       cudaStream_t s) const {
    const size_t off = (size_t)a0 * dg_.nu * dg_.nv;
    launch_transpose(nat + off, ref + off, a1 - a0, dg_.nu, dg_.nv, s);
}

}  // namespace kct
