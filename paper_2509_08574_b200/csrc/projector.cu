// projector.cu — Siddon forward projector (ray-driven, 2D+1) and its exact
// transpose (voxel-driven gather) for sm_100a.
//
// Reference semantics: projector.hpp:53-131 (traverse_ray), :173-204
// (project_forward), :207-261 (project_adjoint).  The intersection lengths are
// the reference's exact Siddon lengths; only rounding differs (float32 values,
// float64 host geometry).  Forward and adjoint evaluate every ray-voxel
// segment endpoint with the same float expressions (ColParams, kct_common.cuh)
// so the pair is a transpose up to the rounding of the final products.
#include <algorithm>
#include <cmath>
#include <limits>

#include "projector.cuh"

namespace kct {

namespace {

constexpr float kInf = __builtin_huge_valf();

// ----------------------------------------------------------------------------
// Forward projector.  One warp = one detector column iu of one angle, C row
// chunks of 32 (lane + 32c).  The xy Siddon walk of the column is shared by
// all its rows (the "2D" part, warp-uniform); every lane carries the z state
// of its C rays (the "+1" part): current slab k, next z-plane crossing wz.
// A CTA holds 4 adjacent columns of the same angle and row band so their
// overlapping voxel columns are served from L1.
// ----------------------------------------------------------------------------
template <int C, bool COUNT>
__global__ void __launch_bounds__(128) fwd_kernel(const float* __restrict__ vol,
                                                  float* __restrict__ out,
                                                  const ColParams* __restrict__ cols,
                                                  const float* __restrict__ dvtab,
                                                  const float* __restrict__ invdv,
                                                  const double* __restrict__ dvd, DevGeom g) {
    const int lane = threadIdx.x & 31;
    const int iu = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int a = blockIdx.z;
    if (iu >= g.nu) return;
    const ColParams cp = cols[(size_t)a * g.nu + iu];
    const int iv0 = blockIdx.y * (32 * C) + lane;
    const int nz = g.nz;

    float acc[C], wz[C], fz[C], imk[C], dvv[C];
    int k[C], kstep[C], kz0i[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int iv = iv0 + 32 * c;
        acc[c] = 0.f;
        const bool row_ok = iv < g.nv;
        const float dv = row_ok ? dvtab[iv] : 0.f;
        dvv[c] = dv;
        // z index at w_in in float64, split into integer + fraction
        const double kzd = fma(row_ok ? dvd[iv] : 0.0, cp.g_in, -g.kz0d);
        const double fl = floor(kzd);
        const int k0 = (int)fmax(fmin(fl, 1.0e9), -1.0e9);
        kz0i[c] = k0;
        fz[c] = (float)(kzd - fl);
        imk[c] = row_ok ? __fmul_rn(invdv[iv], cp.inv_h1) : 0.f;
        int kk = min(max(k0, -1), nz);
        kstep[c] = dv > 0.f ? 1 : -1;
        if (!row_ok) kk = -1 - nz;  // never valid, never crosses
        k[c] = kk;
        const int P = dv > 0.f ? kk + 1 : kk;
        wz[c] = (row_ok && dv != 0.f && P >= 0 && P <= nz)
                    ? __fmaf_rn(__fsub_rn((float)(P - k0), fz[c]), imk[c], cp.w_in)
                    : kInf;
    }

    if (cp.w_in < cp.w_out) {
        const int nx = g.nx, ny = g.ny;
        int i = cp.i0, j = cp.j0;
        const int stx = cp.dx > 0.f ? 1 : -1, sty = cp.dy > 0.f ? 1 : -1;
        int px = cp.dx > 0.f ? i + 1 : i;
        int py = cp.dy > 0.f ? j + 1 : j;
        float wnx = cp.dx != 0.f ? __fmaf_rn((float)px, cp.dx, cp.bx) : kInf;
        float wny = cp.dy != 0.f ? __fmaf_rn((float)py, cp.dy, cp.by) : kInf;
        float wcur = cp.w_in;
        for (;;) {
            const bool stepx = wnx <= wny;
            const float wnext = stepx ? wnx : wny;
            const float wb = fmaxf(fminf(wnext, cp.w_out), wcur);
            const int col = (i + nx * j) * nz;
            float v[C], wa[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                wa[c] = wcur;
                v[c] = (unsigned)k[c] < (unsigned)nz ? (COUNT ? 1.f : __ldg(vol + col + k[c])) : 0.f;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (wz[c] < wb) {  // this ray crosses z-plane(s) inside the segment
                    do {
                        const float len = wz[c] - wa[c];
                        if (COUNT) acc[c] += (len > 0.f && v[c] != 0.f) ? 1.f : 0.f;
                        else acc[c] = __fmaf_rn(len, v[c], acc[c]);
                        wa[c] = wz[c];
                        k[c] += kstep[c];
                        const bool ok = (unsigned)k[c] < (unsigned)nz;
                        v[c] = ok ? (COUNT ? 1.f : __ldg(vol + col + k[c])) : 0.f;
                        const int P = kstep[c] > 0 ? k[c] + 1 : k[c];
                        wz[c] = (P >= 0 && P <= nz)
                                    ? __fmaf_rn(__fsub_rn((float)(P - kz0i[c]), fz[c]), imk[c],
                                                cp.w_in)
                                    : kInf;
                    } while (wz[c] < wb);
                }
                const float len = wb - wa[c];
                if (COUNT) acc[c] += (len > 0.f && v[c] != 0.f) ? 1.f : 0.f;
                else acc[c] = __fmaf_rn(len, v[c], acc[c]);
            }
            if (wnext >= cp.w_out) break;
            wcur = fmaxf(wnext, wcur);
            if (stepx) {
                i += stx;
                if ((unsigned)i >= (unsigned)nx) break;
                px += stx;
                wnx = __fmaf_rn((float)px, cp.dx, cp.bx);
            } else {
                j += sty;
                if ((unsigned)j >= (unsigned)ny) break;
                py += sty;
                wny = __fmaf_rn((float)py, cp.dy, cp.by);
            }
        }
    }

    float* o = out + ((size_t)a * g.nu + iu) * g.nv;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int iv = iv0 + 32 * c;
        if (iv < g.nv) {
            if (COUNT) {
                o[iv] = acc[c];
            } else {
                const float q = dvv[c] * cp.inv_l;
                o[iv] = acc[c] * __fsqrt_rn(__fmaf_rn(q, q, 1.f));
            }
        }
    }
}

// ----------------------------------------------------------------------------
// Adjoint (exact transpose), voxel-driven.  One warp = one voxel column (i,j),
// lane owns voxels k = kbase + lane + 32c (c < K).  For each angle the
// detector columns whose rays cross the xy square of (i,j) are found from the
// projected square corners; for each such column the xy chord [wa,wb] is the
// same float expression the forward walk produces, and for every row whose
// z-span over the chord touches slab k the overlap length is gathered from
// the v-fastest projection (consecutive lanes -> consecutive rows).
// ----------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(128) adj_kernel(const float* __restrict__ proj,
                                                  float* __restrict__ out,
                                                  const ColParams* __restrict__ cols,
                                                  const float* __restrict__ dvtab,
                                                  const float* __restrict__ invdv,
                                                  const double* __restrict__ dvd, DevGeom g,
                                                  AngleBatch ab, int a0, int nab, int accumulate) {
    const int lane = threadIdx.x & 31;
    const int colid = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (colid >= g.nx * g.ny) return;
    const int i = colid % g.nx, j = colid / g.nx;
    const int kbase = blockIdx.y * (32 * K) + lane;
    const int nz = g.nz, nu = g.nu, nv = g.nv;

    const float X0 = g.ox + i * g.sx, X1 = g.ox + (i + 1) * g.sx;
    const float Y0 = g.oy + j * g.sy, Y1 = g.oy + (j + 1) * g.sy;
    const float rpv = 1.f / g.pv;
    constexpr float eps = 1e-3f;

    float acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.f;

    for (int ia = 0; ia < nab; ++ia) {
        const int a = a0 + ia;
        const float cth = ab.cs[ia].x, sth = ab.cs[ia].y;
        // footprint: detector columns whose ray passes the square's interior
        int iu_lo = 0, iu_hi = nu - 1;
        {
            const float lx0 = -X0 * sth, lx1 = -X1 * sth, ly0 = Y0 * cth, ly1 = Y1 * cth;
            const float ax0 = X0 * cth, ax1 = X1 * cth, ay0 = Y0 * sth, ay1 = Y1 * sth;
            const float l00 = g.dso - ax0 - ay0, l01 = g.dso - ax0 - ay1;
            const float l10 = g.dso - ax1 - ay0, l11 = g.dso - ax1 - ay1;
            const float lmin = fminf(fminf(l00, l01), fminf(l10, l11));
            if (!g.full_footprint || lmin > 0.f) {
                const float u00 = (lx0 + ly0) / l00, u01 = (lx0 + ly1) / l01;
                const float u10 = (lx1 + ly0) / l10, u11 = (lx1 + ly1) / l11;
                const float umin = fminf(fminf(u00, u01), fminf(u10, u11)) * g.dsd;
                const float umax = fmaxf(fmaxf(u00, u01), fmaxf(u10, u11)) * g.dsd;
                const float off = 0.5f * nu - 0.5f;
                const float flo = (umin - g.off_u) / g.pu + off;
                const float fhi = (umax - g.off_u) / g.pu + off;
                iu_lo = max(0, (int)ceilf(flo - eps));
                iu_hi = min(nu - 1, (int)floorf(fhi + eps));
            }
        }
        for (int iu = iu_lo; iu <= iu_hi; ++iu) {
            const ColParams cp = cols[(size_t)a * nu + iu];
            float lo = cp.w_in, hi = cp.w_out;
            if (cp.dx != 0.f) {
                const float e0 = __fmaf_rn((float)i, cp.dx, cp.bx);
                const float e1 = __fmaf_rn((float)(i + 1), cp.dx, cp.bx);
                lo = fmaxf(lo, fminf(e0, e1));
                hi = fminf(hi, fmaxf(e0, e1));
            } else if (i != cp.i0) {
                continue;
            }
            if (cp.dy != 0.f) {
                const float e0 = __fmaf_rn((float)j, cp.dy, cp.by);
                const float e1 = __fmaf_rn((float)(j + 1), cp.dy, cp.by);
                lo = fmaxf(lo, fminf(e0, e1));
                hi = fminf(hi, fmaxf(e0, e1));
            } else if (j != cp.j0) {
                continue;
            }
            if (!(lo < hi)) continue;
            const float wa = lo, wb = hi;
            // row candidates: z index kz(w) = dv*G(w) - kz0, G increasing in w
            const float h1 = 1.f / cp.inv_h1;
            const float gin = (float)cp.g_in;
            const float Ga = gin + (wa - cp.w_in) * h1;
            const float Gb = gin + (wb - cp.w_in) * h1;
            const float rGa = 1.f / Ga, rGb = 1.f / Gb;
            const float* py = proj + ((size_t)a * nu + iu) * nv;
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const int k = kbase + 32 * c;
                if (k >= nz) continue;
                const float n0 = (float)k + g.kz0, n1 = n0 + 1.f;
                const float dlo = n0 * (n0 >= 0.f ? rGb : rGa);
                const float dhi = n1 * (n1 >= 0.f ? rGa : rGb);
                const int rlo = max(0, (int)ceilf((dlo - g.dv0) * rpv - eps));
                const int rhi = min(nv - 1, (int)floorf((dhi - g.dv0) * rpv + eps));
                for (int iv = rlo; iv <= rhi; ++iv) {
                    const float dv = dvtab[iv];
                    const double kzd = fma(dvd[iv], cp.g_in, -g.kz0d);
                    const double fl = floor(kzd);
                    const int k0 = (int)fmax(fmin(fl, 1.0e9), -1.0e9);
                    const float f0 = (float)(kzd - fl);
                    float zlo, zhi;
                    if (dv != 0.f) {
                        const float imk = __fmul_rn(invdv[iv], cp.inv_h1);
                        const float w0 = __fmaf_rn(__fsub_rn((float)(k - k0), f0), imk, cp.w_in);
                        const float w1 = __fmaf_rn(__fsub_rn((float)(k + 1 - k0), f0), imk, cp.w_in);
                        zlo = fminf(w0, w1);
                        zhi = fmaxf(w0, w1);
                    } else {
                        if (k0 != k) continue;
                        zlo = -kInf;
                        zhi = kInf;
                    }
                    const float len = fminf(wb, zhi) - fmaxf(wa, zlo);
                    if (len > 0.f) {
                        const float q = dv * cp.inv_l;
                        const float f = __fsqrt_rn(__fmaf_rn(q, q, 1.f));
                        acc[c] = __fmaf_rn(len * f, __ldg(py + iv), acc[c]);
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
                                 int Cc) {
    __shared__ float tile[32][33];
    const size_t boff = (size_t)blockIdx.z * R * Cc;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int r = r0 + dy, c = c0 + threadIdx.x;
        if (r < R && c < Cc) tile[dy][threadIdx.x] = in[boff + (size_t)r * Cc + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int c = c0 + dy, r = r0 + threadIdx.x;
        if (r < R && c < Cc) out[boff + (size_t)c * R + r] = tile[threadIdx.x][dy];
    }
}

void launch_transpose(const float* in, float* out, int B, int R, int Cc, cudaStream_t s) {
    dim3 grid((Cc + 31) / 32, (R + 31) / 32, B);
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, out, R, Cc);
    KCT_CUDA(cudaGetLastError());
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
    const double m = (double)grid.nx * grid.ny * grid.nz;
    if (m > 2147483647.0) throw ConfigError("volume too large for 32-bit voxel indexing");
}

// ---- host-side tables ---------------------------------------------------------
Projector::Projector(const kct_grid& grid, const kct_geometry& geom, int device)
    : grid_(grid) {
    validate_geometry(grid, geom);
    if (device >= 0) KCT_CUDA(cudaSetDevice(device));
    KCT_CUDA(cudaGetDevice(&device_));
    m_ = (size_t)grid.nx * grid.ny * grid.nz;
    n_ = (size_t)geom.nu * geom.nv * geom.n_angles;
    build_tables(geom);
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

    // detector rows: dv(iv) (projector.hpp:36) — the ray's z at the detector
    std::vector<float> dv(nv), invdv(nv);
    std::vector<double> dvd(nv);
    for (int iv = 0; iv < nv; ++iv) {
        const double d = (iv + 0.5 - 0.5 * nv) * geom.pv + geom.offset_v;
        dvd[iv] = d;
        dv[iv] = (float)d;
        invdv[iv] = dv[iv] != 0.f ? (float)(1.0 / (double)dv[iv]) : std::numeric_limits<float>::infinity();
    }

    const double ox = grid_.ox, oy = grid_.oy, sx = grid_.sx, sy = grid_.sy, sz = grid_.sz;
    const double hx = ox + nx * sx, hy = oy + ny * sy;
    const float inf = std::numeric_limits<float>::infinity();
    std::vector<ColParams> cols((size_t)na * nu);
    cs_.resize(na);
    bool full_fp = false;
    for (int a = 0; a < na; ++a) {
        const double t = geom.angles[a];
        const double c = std::cos(t), s = std::sin(t);
        cs_[a] = make_float2((float)c, (float)s);
        const double Sx = geom.dso * c, Sy = geom.dso * s;
        // a voxel square behind the source plane breaks the corner-projection footprint
        {
            const double xs[2] = {ox, hx}, ys[2] = {oy, hy};
            for (double X : xs)
                for (double Y : ys)
                    if (geom.dso - (X * c + Y * s) <= 1e-6 * geom.dso) full_fp = true;
        }
        for (int iu = 0; iu < nu; ++iu) {
            ColParams& cp = cols[(size_t)a * nu + iu];
            const double du = (iu + 0.5 - 0.5 * nu) * geom.pu + geom.offset_u;
            // pixel centre minus source, xy part (projector.hpp:30-39)
            const double dx = -geom.dsd * c - du * s;
            const double dy = -geom.dsd * s + du * c;
            const double L = std::hypot(dx, dy);
            const double ex = dx / L, ey = dy / L;
            const double w0 = -(Sx * ex + Sy * ey);  // foot point of the axis
            const double Rx = Sx + w0 * ex, Ry = Sy + w0 * ey;
            cp.bx = ex != 0.0 ? (float)((ox - Rx) / ex) : inf;
            cp.dx = ex != 0.0 ? (float)(sx / ex) : 0.f;
            cp.by = ey != 0.0 ? (float)((oy - Ry) / ey) : inf;
            cp.dy = ey != 0.0 ? (float)(sy / ey) : 0.f;
            cp.inv_h1 = (float)(L * sz);
            cp.inv_l = (float)(1.0 / L);
            // clip: t in [0,1] and the xy box, evaluated with the same float
            // expressions the kernels use for plane crossings
            float lo = (float)(-w0), hi = (float)(L - w0);
            bool miss = false;
            if (cp.dx != 0.f) {
                const float e0 = std::fmaf(0.f, cp.dx, cp.bx), e1 = std::fmaf((float)nx, cp.dx, cp.bx);
                lo = std::max(lo, std::min(e0, e1));
                hi = std::min(hi, std::max(e0, e1));
            } else if (Sx <= ox || Sx >= hx) {
                miss = true;
            }
            if (cp.dy != 0.f) {
                const float e0 = std::fmaf(0.f, cp.dy, cp.by), e1 = std::fmaf((float)ny, cp.dy, cp.by);
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
            int ii = (int)std::floor((px - ox) / sx), jj = (int)std::floor((py - oy) / sy);
            cp.i0 = std::clamp(ii, 0, nx - 1);
            cp.j0 = std::clamp(jj, 0, ny - 1);
        }
    }
    dg_.full_footprint = full_fp ? 1 : 0;

    // launch shapes: forward rows per warp = 32*C, C <= 4; adjoint voxels per lane K
    const int chunks = (nv + 31) / 32;
    fwd_bands_ = (chunks + 3) / 4;
    fwd_c_ = (chunks + fwd_bands_ - 1) / fwd_bands_;
    const int kc = (nz + 31) / 32;
    adj_k_ = kc <= 1 ? 1 : kc <= 2 ? 2 : kc <= 4 ? 4 : 8;

    KCT_CUDA(cudaMalloc(&d_cols_, cols.size() * sizeof(ColParams)));
    KCT_CUDA(cudaMemcpy(d_cols_, cols.data(), cols.size() * sizeof(ColParams), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_dv_, nv * sizeof(float)));
    KCT_CUDA(cudaMemcpy(d_dv_, dv.data(), nv * sizeof(float), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_invdv_, nv * sizeof(float)));
    KCT_CUDA(cudaMemcpy(d_invdv_, invdv.data(), nv * sizeof(float), cudaMemcpyHostToDevice));
    KCT_CUDA(cudaMalloc(&d_dvd_, nv * sizeof(double)));
    KCT_CUDA(cudaMemcpy(d_dvd_, dvd.data(), nv * sizeof(double), cudaMemcpyHostToDevice));
}

// ---- launches -----------------------------------------------------------------
template <bool COUNT>
static void launch_fwd(int C, int bands, const float* vol, float* out, const ColParams* cols,
                       const float* dv, const float* invdv, const double* dvd, const DevGeom& g,
                       cudaStream_t s) {
    dim3 grid((g.nu + 3) / 4, bands, g.na);
    switch (C) {
    case 1: fwd_kernel<1, COUNT><<<grid, 128, 0, s>>>(vol, out, cols, dv, invdv, dvd, g); break;
    case 2: fwd_kernel<2, COUNT><<<grid, 128, 0, s>>>(vol, out, cols, dv, invdv, dvd, g); break;
    case 3: fwd_kernel<3, COUNT><<<grid, 128, 0, s>>>(vol, out, cols, dv, invdv, dvd, g); break;
    default: fwd_kernel<4, COUNT><<<grid, 128, 0, s>>>(vol, out, cols, dv, invdv, dvd, g); break;
    }
    KCT_CUDA(cudaGetLastError());
}

void Projector::forward(const float* vol, float* proj, cudaStream_t s) const {
    launch_fwd<false>(fwd_c_, fwd_bands_, vol, proj, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, s);
}

void Projector::count(float* proj, cudaStream_t s) const {
    launch_fwd<true>(fwd_c_, fwd_bands_, nullptr, proj, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, s);
}

void Projector::adjoint(const float* proj, float* vol, cudaStream_t s) const {
    const int K = adj_k_;
    dim3 grid((dg_.nx * dg_.ny + 3) / 4, (dg_.nz + 32 * K - 1) / (32 * K), 1);
    AngleBatch ab;
    for (int a0 = 0; a0 < dg_.na; a0 += kMaxAnglesPerLaunch) {
        const int nab = std::min(kMaxAnglesPerLaunch, dg_.na - a0);
        for (int q = 0; q < nab; ++q) ab.cs[q] = cs_[a0 + q];
        const int accum = a0 > 0 ? 1 : 0;
        switch (K) {
        case 1: adj_kernel<1><<<grid, 128, 0, s>>>(proj, vol, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, ab, a0, nab, accum); break;
        case 2: adj_kernel<2><<<grid, 128, 0, s>>>(proj, vol, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, ab, a0, nab, accum); break;
        case 4: adj_kernel<4><<<grid, 128, 0, s>>>(proj, vol, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, ab, a0, nab, accum); break;
        default: adj_kernel<8><<<grid, 128, 0, s>>>(proj, vol, d_cols_, d_dv_, d_invdv_, d_dvd_, dg_, ab, a0, nab, accum); break;
        }
        KCT_CUDA(cudaGetLastError());
    }
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

}  // namespace kct
