// comm.cu — the library-owned NCCL communicator (include/kct.h, ABI 4).
//
// The solvers reach their collectives through two hooks (kct_set_allreduce,
// kct_set_slab).  This file serves both with NCCL itself: every collective is
// enqueued on the solver's stream — no host synchronisation, no callback
// into the caller's runtime — so the CGLS loop stays one asynchronous stream
// of kernels and NCCL operations over NVLink:
//   * sums (Krylov scalars, partial A^T volumes, partial projections of the
//     y-slabs): one ncclAllReduce, in place;
//   * halo planes of the y-slabs: one ncclGroup with a Send / Recv pair per
//     neighbour (rank - 1, rank + 1) — O(1) traffic per rank.
// NCCL is bound at run time with dlopen / dlsym (the copy already loaded in
// the process — torch's, under Python — else libnccl.so.2 from the loader
// path; KCT_NCCL_LIB overrides), so libkct.so carries no link dependency and
// loads on machines without NCCL (single-GPU use).
// The reference has no counterpart (single process, OpenMP: projector.hpp:178-181).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <vector>

#include "kct_common.cuh"

static_assert(NCCL_UNIQUE_ID_BYTES == KCT_COMM_ID_BYTES, "kct.h: KCT_COMM_ID_BYTES");

namespace kct {
int guard_call(const std::function<void()>& f);  // capi.cu
}

namespace {

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

Nccl& nccl() {
    static Nccl api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* lib = nullptr;
        if (const char* path = std::getenv("KCT_NCCL_LIB")) {
            lib = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        } else {
            lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);  // the process's copy
            if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        }
        if (!lib) {
            const char* e = dlerror();
            err = std::string("NCCL not available: ") + (e ? e : "dlopen failed");
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(lib, name);
            if (!p && err.empty()) err = std::string("NCCL symbol missing: ") + name;
            return p;
        };
#define KCT_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(sym(name))
        KCT_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
        KCT_NCCL_SYM(CommInitRank, "ncclCommInitRank");
        KCT_NCCL_SYM(CommDestroy, "ncclCommDestroy");
        KCT_NCCL_SYM(AllReduce, "ncclAllReduce");
        KCT_NCCL_SYM(Send, "ncclSend");
        KCT_NCCL_SYM(Recv, "ncclRecv");
        KCT_NCCL_SYM(GroupStart, "ncclGroupStart");
        KCT_NCCL_SYM(GroupEnd, "ncclGroupEnd");
        KCT_NCCL_SYM(GetErrorString, "ncclGetErrorString");
        KCT_NCCL_SYM(GetVersion, "ncclGetVersion");
#undef KCT_NCCL_SYM
    });
    if (!err.empty()) throw kct::ConfigError(err);
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw kct::CudaError(std::string(what) + ": " + msg);
}

}  // namespace

struct kct_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = -1;
};

namespace {

kct_comm& getc(kct_comm* c) {
    if (!c || !c->comm) throw kct::ConfigError("null communicator");
    return *c;
}

ncclDataType_t dtype_of(int dtype) {
    if (dtype == 0) return ncclFloat32;
    if (dtype == 1) return ncclFloat64;
    throw kct::ConfigError("comm: dtype must be 0 (float32) or 1 (float64)");
}

// kct_allreduce_fn: in-place sum on the solver's stream
int hook_allreduce(void* ctx, void* buf, size_t count, int dtype, void* stream) {
    kct_comm* c = static_cast<kct_comm*>(ctx);
    if (!c || !c->comm || (dtype != 0 && dtype != 1)) return 1;
    if (count == 0) return 0;
    return nccl().AllReduce(buf, buf, count, dtype == 0 ? ncclFloat32 : ncclFloat64, ncclSum,
                            c->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
               ? 0
               : 1;
}

// kct_halo_fn: boundary planes to / from ranks r - 1 and r + 1, one group
int hook_halo(void* ctx, const void* lo_plane, const void* hi_plane, void* lo_halo, void* hi_halo,
              size_t count, void* stream) {
    kct_comm* c = static_cast<kct_comm*>(ctx);
    if (!c || !c->comm) return 1;
    Nccl& n = nccl();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool lo = c->rank > 0, hi = c->rank + 1 < c->world;
    if (!lo && !hi) return 0;
    bool ok = n.GroupStart() == ncclSuccess;
    if (lo) {
        ok = ok && n.Send(lo_plane, count, ncclFloat32, c->rank - 1, c->comm, s) == ncclSuccess;
        ok = ok && n.Recv(lo_halo, count, ncclFloat32, c->rank - 1, c->comm, s) == ncclSuccess;
    }
    if (hi) {
        ok = ok && n.Send(hi_plane, count, ncclFloat32, c->rank + 1, c->comm, s) == ncclSuccess;
        ok = ok && n.Recv(hi_halo, count, ncclFloat32, c->rank + 1, c->comm, s) == ncclSuccess;
    }
    return (n.GroupEnd() == ncclSuccess && ok) ? 0 : 1;
}

}  // namespace

extern "C" {

int kct_comm_unique_id(void* id) {
    return kct::guard_call([&] {
        if (!id) throw kct::ConfigError("comm: null id");
        ncclUniqueId u;
        check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, KCT_COMM_ID_BYTES);
    });
}

int kct_comm_create(int rank, int world, const void* id, int device, kct_comm** out) {
    return kct::guard_call([&] {
        if (!out) throw kct::ConfigError("comm: null output handle");
        *out = nullptr;
        if (!id) throw kct::ConfigError("comm: null id");
        if (world < 1 || rank < 0 || rank >= world) throw kct::ConfigError("comm: rank out of range");
        ncclUniqueId u;
        std::memcpy(&u, id, KCT_COMM_ID_BYTES);
        auto c = new kct_comm;
        c->rank = rank;
        c->world = world;
        try {
            if (device >= 0) KCT_CUDA(cudaSetDevice(device));
            KCT_CUDA(cudaGetDevice(&c->device));
            KCT_CUDA(cudaFree(nullptr));  // the device's primary context exists before NCCL binds to it
            check(nccl().CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int kct_comm_destroy(kct_comm* c) {
    return kct::guard_call([&] {
        if (!c) return;
        if (c->comm) check(nccl().CommDestroy(c->comm), "ncclCommDestroy");
        delete c;
    });
}

int kct_comm_rank(const kct_comm* c) { return c ? c->rank : -1; }
int kct_comm_world(const kct_comm* c) { return c ? c->world : 0; }

int kct_comm_allreduce(kct_comm* c, void* buf, size_t count, int dtype, int op, void* stream) {
    return kct::guard_call([&] {
        kct_comm& k = getc(c);
        if (op != 0 && op != 1) throw kct::ConfigError("comm: op must be 0 (sum) or 1 (max)");
        const ncclDataType_t dt = dtype_of(dtype);
        if (count == 0) return;
        if (!buf) throw kct::ConfigError("comm: null buffer");
        check(nccl().AllReduce(buf, buf, count, dt, op == 0 ? ncclSum : ncclMax, k.comm,
                               static_cast<cudaStream_t>(stream)),
              "ncclAllReduce");
    });
}

int kct_comm_allreduce_host(kct_comm* c, void* buf, size_t count, int dtype, int op) {
    return kct::guard_call([&] {
        kct_comm& k = getc(c);
        if (op != 0 && op != 1) throw kct::ConfigError("comm: op must be 0 (sum) or 1 (max)");
        const ncclDataType_t dt = dtype_of(dtype);
        if (count == 0) return;
        if (!buf) throw kct::ConfigError("comm: null buffer");
        const size_t bytes = count * (dtype == 0 ? sizeof(float) : sizeof(double));
        void* d = nullptr;
        KCT_CUDA(cudaMalloc(&d, bytes));
        try {
            KCT_CUDA(cudaMemcpy(d, buf, bytes, cudaMemcpyHostToDevice));
            check(nccl().AllReduce(d, d, count, dt, op == 0 ? ncclSum : ncclMax, k.comm, nullptr),
                  "ncclAllReduce");
            KCT_CUDA(cudaMemcpy(buf, d, bytes, cudaMemcpyDeviceToHost));
        } catch (...) {
            cudaFree(d);
            throw;
        }
        KCT_CUDA(cudaFree(d));
    });
}

int kct_use_comm(kct_projector* h, kct_comm* c) {
    if (!c) return kct_set_allreduce(h, nullptr, nullptr);
    int rc = kct::guard_call([&] { getc(c); });
    if (rc != KCT_OK) return rc;
    return kct_set_allreduce(h, hook_allreduce, c);
}

int kct_use_comm_slab(kct_projector* h, kct_comm* c, int j0, int ny_global) {
    if (!c) {
        int rc = kct_set_slab(h, 0, 1, 0, 0, nullptr, nullptr);
        return rc != KCT_OK ? rc : kct_set_allreduce(h, nullptr, nullptr);
    }
    int rc = kct::guard_call([&] { getc(c); });
    if (rc != KCT_OK) return rc;
    rc = kct_set_allreduce(h, hook_allreduce, c);
    if (rc != KCT_OK) return rc;
    return kct_set_slab(h, c->rank, c->world, j0, ny_global, hook_halo, c);
}

int kct_slab_bounds(const kct_grid* grid, const kct_geometry* geom, int world, int* bounds) {
    return kct::guard_call([&] {
        if (!grid || !geom || !bounds) throw kct::ConfigError("slab_bounds: null argument");
        const int nx = grid->nx, ny = grid->ny;
        if (nx < 1 || ny < 1) throw kct::ConfigError("slab_bounds: empty grid");
        if (world < 1 || world > ny) throw kct::ConfigError("slab_bounds: more ranks than y planes");
        // backprojection work of every y plane over a full circle of 64 views
        constexpr int kViews = 64, kQuantum = 4;
        const double half = 0.5 * geom->nu * geom->pu;
        std::vector<double> w(ny, 0.0);
        for (int a = 0; a < kViews; ++a) {
            const double t = 2.0 * M_PI * (double)a / (double)kViews;
            const double cs = std::cos(t), sn = std::sin(t);
            for (int j = 0; j < ny; ++j) {
                const double y = grid->oy + (j + 0.5) * grid->sy;
                int cnt = 0;
                for (int i = 0; i < nx; ++i) {
                    const double x = grid->ox + (i + 0.5) * grid->sx;
                    const double den = geom->dso - (x * cs + y * sn);
                    if (!(den > 0)) continue;
                    const double u = geom->dsd * (-x * sn + y * cs) / den - geom->offset_u;
                    cnt += std::fabs(u) <= half;
                }
                w[j] += cnt;
            }
        }
        std::vector<double> cum(ny + 1, 0.0);
        for (int j = 0; j < ny; ++j) cum[j + 1] = cum[j] + (std::max(w[j], 0.0) + 1e-9);
        bounds[0] = 0;
        for (int r = 1; r < world; ++r) {
            const double target = cum[ny] * (double)r / (double)world;
            // first index with cum[index] >= target (numpy.searchsorted, side = left)
            int j = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
            int q = j;
            if (ny >= kQuantum * world) q = (int)std::nearbyint((double)j / kQuantum) * kQuantum;
            q = std::max(q, bounds[r - 1] + 1);
            q = std::min(q, ny - (world - r));
            bounds[r] = q;
        }
        bounds[world] = ny;
    });
}

}  // extern "C"
