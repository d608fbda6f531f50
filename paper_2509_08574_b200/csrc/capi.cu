// capi.cu — the C ABI (include/kct.h).  Thin: argument checks, layout and
// host<->device staging, exception -> status-code mapping.  All compute is in
// projector.cu / solver.cu.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "projector.cuh"
#include "solver.cuh"

struct kct_projector {
    kct::Projector* p;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return KCT_OK;
    } catch (const kct::ConfigError& e) {
        g_err = e.what();
        return KCT_ERR_CONFIG;
    } catch (const kct::SolverError& e) {
        g_err = e.what();
        return KCT_ERR_SOLVER;
    } catch (const kct::CudaError& e) {
        g_err = e.what();
        return KCT_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KCT_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return KCT_ERR_INTERNAL;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) KCT_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

kct::Projector& get(kct_projector* h) {
    if (!h || !h->p) throw kct::ConfigError("null projector handle");
    return *h->p;
}

void check_mem_layout(int mem, int layout) {
    if (mem != KCT_MEM_HOST && mem != KCT_MEM_DEVICE) throw kct::ConfigError("invalid mem kind");
    if (layout != KCT_LAYOUT_REFERENCE && layout != KCT_LAYOUT_NATIVE)
        throw kct::ConfigError("invalid layout");
}

__global__ void sum_counts_kernel(const float* __restrict__ c, size_t n, unsigned long long* out) {
    unsigned long long local = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        local += (unsigned long long)c[i];
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

}  // namespace

namespace kct {

// comm.cu's entry points share the status mapping and the last-error slot
int guard_call(const std::function<void()>& f) { return guarded(f); }

std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Stage an input array of `n` floats into a native-layout device buffer.
// Returns a device pointer (either `src` itself or a scratch buffer).
const float* stage_in(Projector& P, const float* src, size_t n, bool is_vol, int mem, int layout,
                      int slot, int tmp_slot, cudaStream_t s) {
    if (!src) return nullptr;
    if (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) return src;
    float* dst = P.scratch(slot, n);
    const float* ref = src;
    if (mem == KCT_MEM_HOST) {
        float* tgt = layout == KCT_LAYOUT_NATIVE ? dst : P.scratch(tmp_slot, n);
        KCT_CUDA(cudaMemcpyAsync(tgt, src, n * sizeof(float), cudaMemcpyHostToDevice, s));
        if (layout == KCT_LAYOUT_NATIVE) return dst;
        ref = tgt;
    }
    if (is_vol) P.vol_to_native(ref, dst, s);
    else P.proj_to_native(ref, dst, s);
    return dst;
}

// Write a native-layout device array `nat` out to `dst` (mem/layout as given).
void stage_out(Projector& P, const float* nat, float* dst, size_t n, bool is_vol, int mem,
               int layout, int tmp_slot, cudaStream_t s) {
    if (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) {
        if (dst != nat) KCT_CUDA(cudaMemcpyAsync(dst, nat, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
        return;
    }
    const float* src = nat;
    if (layout == KCT_LAYOUT_REFERENCE) {
        float* tgt = mem == KCT_MEM_DEVICE ? dst : P.scratch(tmp_slot, n);
        if (is_vol) P.vol_from_native(nat, tgt, s);
        else P.proj_from_native(nat, tgt, s);
        if (mem == KCT_MEM_DEVICE) return;
        src = tgt;
    }
    KCT_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToHost, s));
}

}  // namespace kct

extern "C" {

const char* kct_last_error(void) { return g_err.c_str(); }
int kct_abi_version(void) { return KCT_ABI_VERSION; }

unsigned long long kct_launch_count(void) { return kct::g_launches.load(std::memory_order_relaxed); }

int kct_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) throw kct::ConfigError("null argument");
        *out = nullptr;
        KCT_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    });
}

int kct_host_free(void* ptr) {
    return guarded([&] {
        if (ptr) KCT_CUDA(cudaFreeHost(ptr));
    });
}

int kct_projector_create(const kct_grid* grid, const kct_geometry* geom, int device,
                         kct_projector** out) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_projector_create");
        if (!grid || !geom || !out) throw kct::ConfigError("null argument");
        *out = nullptr;
        auto* h = new kct_projector{nullptr};
        try {
            h->p = new kct::Projector(*grid, *geom, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kct_projector_destroy(kct_projector* h) {
    return guarded([&] {
        if (!h) return;
        delete h->p;
        delete h;
    });
}

int kct_projector_sizes(const kct_projector* h, size_t* domain, size_t* range) {
    return guarded([&] {
        if (!h || !h->p) throw kct::ConfigError("null projector handle");
        if (domain) *domain = h->p->domain_size();
        if (range) *range = h->p->range_size();
    });
}

namespace {

// KCT_TRACE=1: device timeline of the host pipelines (events on both streams,
// printed to stderr after the call; diagnostics only)
struct Trace {
    bool on = false;
    cudaEvent_t t0 = nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    explicit Trace(cudaStream_t s) {
        const char* e = std::getenv("KCT_TRACE");
        on = e && e[0] == '1';
        if (on) {
            cudaEventCreate(&t0);
            cudaEventRecord(t0, s);
        }
    }
    void mark(const std::string& name, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.emplace_back(name, e);
    }
    void dump(const char* what) {
        if (!on) return;
        std::string line = std::string("[kct trace] ") + what + ":";
        for (auto& [name, e] : ev) {
            float ms = 0.f;
            cudaEventSynchronize(e);
            cudaEventElapsedTime(&ms, t0, e);
            char buf[64];
            std::snprintf(buf, sizeof buf, " %s=%.3f", name.c_str(), ms);
            line += buf;
            cudaEventDestroy(e);
        }
        cudaEventDestroy(t0);
        std::fprintf(stderr, "%s\n", line.c_str());
    }
};

// Host-buffer forward, pipelined: the projections of angle chunk c leave the
// device (layout transpose + D2H on the copy stream) while chunk c + 1 is
// computed.  Same kernels and results as the unpipelined path.
// Staged host forward (reference layouts): the volume goes up stage range by
// stage range on the copy stream (slabs [z_lo, z_hi) of stage s, centre out),
// the main stream transposes each range into the padded volume and runs
// stage s's rows as soon as its range is in; the last stage is counted per
// pipeline chunk of angles and each chunk's projections go down as they finish.
bool forward_host_staged(kct::Projector& P, const float* vol, float* proj, cudaStream_t s) {
    const auto& st = P.fwd_stages();
    const int S = (int)st.size();
    if (S < 2 || S > kct::Projector::kPipeChunks || !P.fwd_done()) return false;
    const size_t M = P.domain_size(), N = P.range_size();
    const kct_grid& gr = P.grid();
    const size_t plane = (size_t)gr.nx * gr.ny;
    cudaStream_t sc = P.pipe_stream();
    float* tmp = P.scratch(2, M);
    float* q = P.scratch(1, N);
    float* qr = P.scratch(3, N);
    unsigned* done = P.fwd_done();
    const int K = P.pipe_chunks();
    Trace tr(s);
    KCT_CUDA(cudaMemsetAsync(done, 0, K * sizeof(unsigned), s));
    KCT_CUDA(cudaEventRecord(P.upload_event(), s));  // the copy stream starts after this call's
    KCT_CUDA(cudaStreamWaitEvent(sc, P.upload_event(), 0));  // earlier work and sees the reset
    if (!P.stream_wait_geq(sc, done, 0u)) return false;  // probe: stream memory ops available
    // uploads: the new slabs of each stage (below and above the previous range)
    int lo = st[0].z_lo, hi = st[0].z_lo;
    std::vector<std::pair<int, int>> pieces[kct::Projector::kPipeChunks];
    for (int k = 0; k < S; ++k) {
        if (st[k].z_lo < lo) pieces[k].push_back({st[k].z_lo, lo});
        if (st[k].z_hi > hi) pieces[k].push_back({hi, st[k].z_hi});
        lo = std::min(lo, st[k].z_lo);
        hi = std::max(hi, st[k].z_hi);
        for (auto& pc : pieces[k])
            KCT_CUDA(cudaMemcpyAsync(tmp + pc.first * plane, vol + pc.first * plane,
                                     (size_t)(pc.second - pc.first) * plane * sizeof(float),
                                     cudaMemcpyHostToDevice, sc));
        KCT_CUDA(cudaEventRecord(P.pipe_event(k), sc));
        tr.mark("up" + std::to_string(k), sc);
    }
    const size_t per = N / (size_t)P.n_angles();
    // the stages write the reference layout themselves (KCT_FWD_REFOUT=0: native
    // layout + a transpose kernel per output piece on the copy stream)
    const char* ro = std::getenv("KCT_FWD_REFOUT");
    const bool refout = !(ro && ro[0] == '0');
    if (P.fwd_rowstages()) {
        // every stage's rows (all angles) leave the device as soon as the
        // stage is done: native -> reference transpose of the stage's row
        // band(s) and one strided copy per band on the copy stream, so only
        // the last stage's share of the projections is left when the kernels end
        const int nv = P.dev_geom().nv, nu = P.dev_geom().nu, na = P.n_angles();
        const bool mir = P.mirror();
        for (int k = 0; k < S; ++k) {
            KCT_CUDA(cudaStreamWaitEvent(s, P.pipe_event(k), 0));
            for (auto& pc : pieces[k]) P.vol_to_padded_z(tmp, pc.first, pc.second, s);
            tr.mark("pad" + std::to_string(k), s);
            P.forward_stage(k, refout ? qr : q, nullptr, s, refout);
            tr.mark("stage" + std::to_string(k), s);
            KCT_CUDA(cudaEventRecord(P.pipe_event(k), s));  // (its upload wait is already enqueued)
            KCT_CUDA(cudaStreamWaitEvent(sc, P.pipe_event(k), 0));
            const int r0 = st[k].row0, r1 = st[k].row0 + 32 * st[k].C;
            std::pair<int, int> bands[2];
            int nb = 0;
            if (mir) {  // pairs [r0, r1): rows nv/2 - r1 .. nv/2 - r0 and their mirrors
                const int h = nv / 2;
                if (r0 == 0) bands[nb++] = {std::max(0, h - r1), std::min(nv, h + r1)};
                else {
                    bands[nb++] = {std::max(0, h - r1), h - r0};
                    bands[nb++] = {h + r0, std::min(nv, h + r1)};
                }
            } else {
                bands[nb++] = {r0, std::min(nv, r1)};
            }
            for (int b = 0; b < nb; ++b) {
                const int v0 = bands[b].first, v1 = bands[b].second;
                if (v1 <= v0) continue;
                if (!refout) P.proj_rows_from_native(q, qr, v0, v1, sc);
                KCT_CUDA(cudaMemcpy2DAsync(proj + (size_t)v0 * nu, per * sizeof(float),
                                           qr + (size_t)v0 * nu, per * sizeof(float),
                                           (size_t)(v1 - v0) * nu * sizeof(float), na,
                                           cudaMemcpyDeviceToHost, sc));
            }
            tr.mark("down" + std::to_string(k), sc);
        }
        KCT_CUDA(cudaStreamSynchronize(sc));
        KCT_CUDA(cudaStreamSynchronize(s));
        tr.dump("forward_host_staged (row stages)");
        return true;
    }
    for (int k = 0; k < S; ++k) {
        KCT_CUDA(cudaStreamWaitEvent(s, P.pipe_event(k), 0));
        for (auto& pc : pieces[k]) P.vol_to_padded_z(tmp, pc.first, pc.second, s);
        tr.mark("pad" + std::to_string(k), s);
        P.forward_stage(k, refout ? qr : q, k + 1 == S ? done : nullptr, s, refout);
        tr.mark("stage" + std::to_string(k), s);
    }
    for (int c = 0; c < K; ++c) {
        const int a0 = P.pipe_angle(c), a1 = P.pipe_angle(c + 1);
        if (!P.stream_wait_geq(sc, done + c, (unsigned)((a1 - a0) * P.dev_geom().nu)))
            throw kct::CudaError("forward: stream wait failed");
        if (!refout) P.proj_from_native_range(q, qr, a0, a1, sc);
        KCT_CUDA(cudaMemcpyAsync(proj + a0 * per, qr + a0 * per, (a1 - a0) * per * sizeof(float),
                                 cudaMemcpyDeviceToHost, sc));
        tr.mark("down" + std::to_string(c), sc);
    }
    KCT_CUDA(cudaStreamSynchronize(sc));
    KCT_CUDA(cudaStreamSynchronize(s));
    tr.dump("forward_host_staged");
    return true;
}

void forward_host_pipelined(kct::Projector& P, const float* vol, float* proj, int layout,
                            cudaStream_t s) {
    if (layout == KCT_LAYOUT_REFERENCE && forward_host_staged(P, vol, proj, s)) return;
    const size_t M = P.domain_size(), N = P.range_size();
    cudaStream_t sc = P.pipe_stream();
    // Split upload (reference layout: a z range is contiguous): slabs [Z0, Z)
    // first, row band 0 (whose rays stay inside them: Z0 = 0, or the central
    // slabs with z-mirror pairs) runs while the rest of the volume is uploaded
    // on the copy stream.
    const int Z = layout == KCT_LAYOUT_REFERENCE ? P.fwd_split_z() : 0;
    const int Z0 = Z > 0 ? P.fwd_split_lo() : 0;
    const int nzg = P.grid().nz;
    if (Z > 0) {
        const kct_grid& gr = P.grid();
        const size_t plane = (size_t)gr.nx * gr.ny, lo = (size_t)Z0 * plane, hi = (size_t)Z * plane;
        float* tmp = P.scratch(2, M);
        KCT_CUDA(cudaMemcpyAsync(tmp + lo, vol + lo, (hi - lo) * sizeof(float), cudaMemcpyHostToDevice, s));
        KCT_CUDA(cudaEventRecord(P.upload_event(), s));  // the copy stream starts after this call's
        KCT_CUDA(cudaStreamWaitEvent(sc, P.upload_event(), 0));  // earlier work on s
        if (hi < M)
            KCT_CUDA(cudaMemcpyAsync(tmp + hi, vol + hi, (M - hi) * sizeof(float), cudaMemcpyHostToDevice, sc));
        if (lo > 0) KCT_CUDA(cudaMemcpyAsync(tmp, vol, lo * sizeof(float), cudaMemcpyHostToDevice, sc));
        P.vol_to_padded_z(tmp, Z0, Z, s);
    } else if (layout == KCT_LAYOUT_REFERENCE) {
        float* tmp = P.scratch(2, M);
        KCT_CUDA(cudaMemcpyAsync(tmp, vol, M * sizeof(float), cudaMemcpyHostToDevice, s));
        P.vol_to_padded_z(tmp, 0, P.grid().nz, s);
    } else {
        P.pad_volume(kct::stage_in(P, vol, M, true, KCT_MEM_HOST, layout, 0, 2, s), s);
    }
    float* q = P.scratch(1, N);
    float* qr = layout == KCT_LAYOUT_REFERENCE ? P.scratch(3, N) : nullptr;
    const int K = P.pipe_chunks();
    const size_t per = N / (size_t)P.n_angles();
    // one counted launch (chunk-major blocks, finished columns per chunk):
    // the copy stream waits on each chunk's count (cuStreamWaitValue32)
    // instead of one launch per chunk — no per-chunk launch tails
    const char* ce = std::getenv("KCT_FWD_COUNTED");
    unsigned* done = (ce && ce[0] == '0') ? nullptr : P.fwd_done();
    if (done) {
        KCT_CUDA(cudaMemsetAsync(done, 0, K * sizeof(unsigned), s));
        KCT_CUDA(cudaEventRecord(P.pipe_event(0), s));
    }
    if (Z > 0) {
        P.forward_split_lo(q, s);
        KCT_CUDA(cudaEventRecord(P.upload_event(), sc));
        KCT_CUDA(cudaStreamWaitEvent(s, P.upload_event(), 0));
        if (Z < nzg) P.vol_to_padded_z(P.scratch(2, M), Z, nzg, s);
        if (Z0 > 0) P.vol_to_padded_z(P.scratch(2, M), 0, Z0, s);
    }
    bool counted = false;
    if (done) {
        const int band0 = Z > 0 ? 1 : 0;
        KCT_CUDA(cudaStreamWaitEvent(sc, P.pipe_event(0), 0));  // sees the reset counts
        counted = P.stream_wait_geq(sc, done, 0u);  // probe: stream memory ops available
        if (counted) {
            P.forward_counted(q, band0, done, s);
            for (int c = 0; c < K; ++c) {
                const int a0 = P.pipe_angle(c), a1 = P.pipe_angle(c + 1);
                if (!P.stream_wait_geq(sc, done + c, P.fwd_chunk_columns(c, band0)))
                    throw kct::CudaError("forward: stream wait failed");
                const float* src = q + a0 * per;
                if (qr) {
                    P.proj_from_native_range(q, qr, a0, a1, sc);
                    src = qr + a0 * per;
                }
                KCT_CUDA(cudaMemcpyAsync(proj + a0 * per, src, (a1 - a0) * per * sizeof(float),
                                         cudaMemcpyDeviceToHost, sc));
            }
        }
    }
    for (int c = 0; !counted && c < K; ++c) {
        const int a0 = P.pipe_angle(c), a1 = P.pipe_angle(c + 1);
        if (Z > 0) P.forward_split_hi(q, c, s);
        else P.forward_padded(q, a0, a1, s);
        KCT_CUDA(cudaEventRecord(P.pipe_event(c), s));
        KCT_CUDA(cudaStreamWaitEvent(sc, P.pipe_event(c), 0));
        const float* src = q + a0 * per;
        if (qr) {
            P.proj_from_native_range(q, qr, a0, a1, sc);
            src = qr + a0 * per;
        }
        KCT_CUDA(cudaMemcpyAsync(proj + a0 * per, src, (a1 - a0) * per * sizeof(float),
                                 cudaMemcpyDeviceToHost, sc));
    }
    KCT_CUDA(cudaStreamSynchronize(sc));
    KCT_CUDA(cudaStreamSynchronize(s));
}

// KCT_HOST_PIPELINE=0 turns the forward pipeline off.  (Chunking the adjoint
// the same way to overlap its input copy measured 0.8 ms slower at c3: each
// chunk re-reads and re-writes the whole volume.)
bool pipelined(const kct::Projector& P, int mem) {
    const char* e = std::getenv("KCT_HOST_PIPELINE");
    return mem == KCT_MEM_HOST && P.pipe_chunks() > 1 && !(e && e[0] == '0');
}

}  // namespace

int kct_forward(kct_projector* h, const float* vol, float* proj, int mem, int layout,
                void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_forward");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        if (!vol || !proj) throw kct::ConfigError("forward: null buffer");
        DeviceGuard dg(P.device());
        auto s = static_cast<cudaStream_t>(stream);
        if (pipelined(P, mem)) return forward_host_pipelined(P, vol, proj, layout, s);
        const size_t M = P.domain_size(), N = P.range_size();
        const float* v = kct::stage_in(P, vol, M, true, mem, layout, 0, 2, s);
        float* q = (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) ? proj : P.scratch(1, N);
        P.forward(v, q, s);
        kct::stage_out(P, q, proj, N, false, mem, layout, 2, s);
        if (mem == KCT_MEM_HOST) KCT_CUDA(cudaStreamSynchronize(s));
    });
}

int kct_adjoint(kct_projector* h, const float* proj, float* vol, int mem, int layout,
                void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_adjoint");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        if (!vol || !proj) throw kct::ConfigError("adjoint: null buffer");
        DeviceGuard dg(P.device());
        auto s = static_cast<cudaStream_t>(stream);
        const size_t M = P.domain_size(), N = P.range_size();
        // host buffers, reference layouts: upload in two angle parts, volume out
        // z level by z level while the adjoint runs (Projector::adjoint_host_ref)
        if (mem == KCT_MEM_HOST && layout == KCT_LAYOUT_REFERENCE && P.adjoint_host_ref(proj, vol, s))
            return;
        const float* q = kct::stage_in(P, proj, N, false, mem, layout, 1, 2, s);
        float* v = (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) ? vol : P.scratch(0, M);
        P.adjoint(q, v, s);
        kct::stage_out(P, v, vol, M, true, mem, layout, 2, s);
        if (mem == KCT_MEM_HOST) KCT_CUDA(cudaStreamSynchronize(s));
    });
}

int kct_forward_f64(kct_projector* h, const double* vol, double* proj) {
    return guarded([&] {
        auto& P = get(h);
        if (!vol || !proj) throw kct::ConfigError("forward: null buffer");
        std::vector<float> v(vol, vol + P.domain_size()), q(P.range_size());
        if (kct_forward(h, v.data(), q.data(), KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr))
            throw kct::CudaError(g_err);
        for (size_t i = 0; i < q.size(); ++i) proj[i] = q[i];
    });
}

int kct_adjoint_f64(kct_projector* h, const double* proj, double* vol) {
    return guarded([&] {
        auto& P = get(h);
        if (!vol || !proj) throw kct::ConfigError("adjoint: null buffer");
        std::vector<float> q(proj, proj + P.range_size()), v(P.domain_size());
        if (kct_adjoint(h, q.data(), v.data(), KCT_MEM_HOST, KCT_LAYOUT_REFERENCE, nullptr))
            throw kct::CudaError(g_err);
        for (size_t i = 0; i < v.size(); ++i) vol[i] = v[i];
    });
}

int kct_projector_info(const kct_projector* h, const char* key, double* value) {
    return guarded([&] {
        if (!h || !h->p) throw kct::ConfigError("null projector handle");
        if (!key || !value) throw kct::ConfigError("null argument");
        const kct::Projector& P = *h->p;
        const std::string k(key);
        if (k == "adj_slab") *value = P.adj_slab() ? 1 : 0;
        else if (k == "adj_slab_detect") *value = P.adj_slab_detect() ? 1 : 0;
        else if (k == "adj_bz") *value = P.adj_mirror() ? P.adj_mirror_bz() : P.adj_bz();
        else if (k == "adj_mirror") *value = P.adj_mirror() ? 1 : 0;
        else if (k == "adj_ws") *value = P.adj_ws() ? 1 : 0;
        else if (k == "adj_np") *value = P.adj_ws() ? P.adj_np() : 0;
        else if (k == "adj_stride") *value = P.adj_stride();
        else if (k == "adj_groups") *value = P.adj_groups();
        else if (k == "adj_gather") *value = P.adj_gather() ? 1 : 0;
        else if (k == "adj_walk_entries") *value = (double)P.walk_entries();
        else if (k == "fwd_rows_per_warp") *value = 32 * P.fwd_chunks() * (P.mirror() ? 2 : 1);
        else if (k == "fwd_bands") *value = P.dev_geom().fwd_bands;
        else if (k == "fwd_split_z") *value = P.fwd_split_z();
        else if (k == "fwd_split_lo") *value = P.fwd_split_lo();
        else if (k == "fwd_stages") *value = (double)P.fwd_stages().size();
        else if (k == "fwd_table_segments") *value = (double)P.fwd_table_segments();
        else if (k == "mirror") *value = P.mirror() ? 1 : 0;
        else if (k == "solver_restart") *value = P.solver_restart ? 1 : 0;
        else throw kct::ConfigError("kct_projector_info: unknown key '" + k + "'");
    });
}

int kct_count_nnz(kct_projector* h, uint64_t* nnz, void* stream) {
    return guarded([&] {
        auto& P = get(h);
        if (!nnz) throw kct::ConfigError("null output");
        DeviceGuard dg(P.device());
        auto s = static_cast<cudaStream_t>(stream);
        float* c = P.scratch(1, P.range_size());
        P.count(c, s);
        unsigned long long* d = reinterpret_cast<unsigned long long*>(P.scratch(3, 2));
        KCT_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
        sum_counts_kernel<<<148 * 4, 256, 0, s>>>(c, P.range_size(), d);
        KCT_LAUNCHED();
        unsigned long long r = 0;
        KCT_CUDA(cudaMemcpyAsync(&r, d, sizeof r, cudaMemcpyDeviceToHost, s));
        KCT_CUDA(cudaStreamSynchronize(s));
        *nnz = r;
    });
}

int kct_volume_to_native(const kct_projector* h, const float* ref, float* native, void* stream) {
    return guarded([&] {
        auto& P = get(const_cast<kct_projector*>(h));
        DeviceGuard dg(P.device());
        P.vol_to_native(ref, native, static_cast<cudaStream_t>(stream));
    });
}
int kct_volume_from_native(const kct_projector* h, const float* native, float* ref, void* stream) {
    return guarded([&] {
        auto& P = get(const_cast<kct_projector*>(h));
        DeviceGuard dg(P.device());
        P.vol_from_native(native, ref, static_cast<cudaStream_t>(stream));
    });
}
int kct_proj_to_native(const kct_projector* h, const float* ref, float* native, void* stream) {
    return guarded([&] {
        auto& P = get(const_cast<kct_projector*>(h));
        DeviceGuard dg(P.device());
        P.proj_to_native(ref, native, static_cast<cudaStream_t>(stream));
    });
}
int kct_proj_from_native(const kct_projector* h, const float* native, float* ref, void* stream) {
    return guarded([&] {
        auto& P = get(const_cast<kct_projector*>(h));
        DeviceGuard dg(P.device());
        P.proj_from_native(native, ref, static_cast<cudaStream_t>(stream));
    });
}

int kct_fdk(kct_projector* h, const float* proj, float* vol, int mem, int layout, void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_fdk");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        if (!vol || !proj) throw kct::ConfigError("fdk: null buffer");
        DeviceGuard dg(P.device());
        auto s = static_cast<cudaStream_t>(stream);
        const size_t M = P.domain_size(), N = P.range_size();
        const float* q = kct::stage_in(P, proj, N, false, mem, layout, 1, 2, s);
        float* v = (mem == KCT_MEM_DEVICE && layout == KCT_LAYOUT_NATIVE) ? vol : P.scratch(0, M);
        P.fdk(q, v, P.scratch(3, N), s);
        kct::stage_out(P, v, vol, M, true, mem, layout, 2, s);
        if (mem == KCT_MEM_HOST) KCT_CUDA(cudaStreamSynchronize(s));
    });
}

int kct_set_option(kct_projector* h, const char* key, double value) {
    return guarded([&] {
        auto& P = get(h);
        if (!key) throw kct::ConfigError("null option key");
        const std::string k(key);
        if (k == "solver_restart") {
            if (value != 0.0 && value != 1.0) throw kct::ConfigError("solver_restart must be 0 or 1");
            P.solver_restart = value != 0.0;
        } else {
            throw kct::ConfigError("kct_set_option: unknown key '" + k + "'");
        }
    });
}

int kct_set_iterate_hook(kct_projector* h, kct_iterate_hook fn, void* ctx) {
    return guarded([&] {
        auto& P = get(h);
        P.hook_fn = fn;
        P.hook_ctx = fn ? ctx : nullptr;
    });
}

int kct_set_allreduce(kct_projector* h, kct_allreduce_fn fn, void* ctx) {
    return guarded([&] {
        auto& P = get(h);
        P.comm_fn = fn;
        P.comm_ctx = ctx;
    });
}

int kct_set_slab(kct_projector* h, int rank, int world, int j0, int ny_global, kct_halo_fn fn,
                 void* ctx) {
    return guarded([&] {
        auto& P = get(h);
        if (fn) {
            if (world < 1 || rank < 0 || rank >= world)
                throw kct::ConfigError("slab: rank out of range");
            if (j0 < 0 || ny_global < j0 + P.grid().ny)
                throw kct::ConfigError("slab: plane range outside the global grid");
        }
        P.slab_rank = fn ? rank : -1;
        P.slab_world = fn ? world : 0;
        P.slab_j0 = fn ? j0 : 0;
        P.slab_nyg = fn ? ny_global : 0;
        P.halo_fn = fn;
        P.halo_ctx = ctx;
        P.workspace.reset();  // volume buffers change shape (halo planes)
    });
}

double kct_resolve_tau(double tau, const float* reference, size_t n) {
    return kct::resolve_tau(tau, reference, n);
}

int kct_cgls_recon(kct_projector* h, const float* b, size_t iters, const float* x0,
                   const float* ground_truth, double tolerance, float* x_out,
                   kct_report* report, int mem, int layout, void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_cgls_recon");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        DeviceGuard dg(P.device());
        kct::cgls_recon(P, b, iters, x0, ground_truth, tolerance, x_out, report, mem, layout,
                        static_cast<cudaStream_t>(stream));
    });
}

int kct_cgls_stack(kct_projector* h, const kct_stack_block* blocks, size_t n_blocks,
                   const float* b, const float* x0, size_t max_iters, double tolerance,
                   float* x_out, kct_report* report, int mem, int layout, void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_cgls_stack");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        DeviceGuard dg(P.device());
        kct::cgls_stack(P, blocks, n_blocks, b, x0, max_iters, tolerance, x_out, report, mem,
                        layout, static_cast<cudaStream_t>(stream));
    });
}

int kct_irn(kct_projector* h, int kind, const float* b, const float* prior, const float* x0,
            const float* ground_truth, const kct_reg_params* params, float* x_out,
            kct_report* report, int mem, int layout, void* stream) {
    return guarded([&] {
        kct::NvtxRange nvtx("kct_irn");
        auto& P = get(h);
        check_mem_layout(mem, layout);
        if (!params) throw kct::ConfigError("null params");
        DeviceGuard dg(P.device());
        kct::irn_solve(P, kind, b, prior, x0, ground_truth, *params, x_out, report, mem, layout,
                       static_cast<cudaStream_t>(stream));
    });
}

int kct_irn_piccs(kct_projector* h, const float* b, const float* prior, const float* x0,
                  const float* ground_truth, const kct_reg_params* params, float* x_out,
                  kct_report* report, int mem, int layout, void* stream) {
    return kct_irn(h, KCT_KIND_PICCS, b, prior, x0, ground_truth, params, x_out, report, mem,
                   layout, stream);
}

}  // extern "C"
