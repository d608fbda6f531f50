// projector.cuh — the cone-beam operator pair A / A^T on B200.
//
// Replaces ConeBeamProjector / project_forward / project_adjoint /
// traverse_ray (reference projector.hpp:24-296).  Same model: exact Siddon
// ray-voxel intersection lengths, nearest-voxel piecewise constant, rays from
// the source through every detector pixel centre.
#pragma once

#include <memory>
#include <vector>

#include "kct_common.cuh"

namespace kct {

struct BrickCfg;  // adjoint brick configuration (projector.cu)
struct FwdTab;    // forward walk table view (projector.cu)

class Projector {
  public:
    Projector(const kct_grid& grid, const kct_geometry& geom, int device);
    ~Projector();
    Projector(const Projector&) = delete;
    Projector& operator=(const Projector&) = delete;

    size_t domain_size() const { return m_; }
    size_t range_size() const { return n_; }
    const kct_grid& grid() const { return grid_; }
    const DevGeom& dev_geom() const { return dg_; }
    int device() const { return device_; }
    int n_angles() const { return dg_.na; }

    // Native-layout, device-resident operators (stream-ordered).
    void forward(const float* vol, float* proj, cudaStream_t s) const;
    void adjoint(const float* proj, float* vol, cudaStream_t s) const;
    // Angle sub-ranges [a_begin, a_end) (full-size native buffers; the
    // adjoint adds into `vol` when accumulate).
    void forward_range(const float* vol, float* proj, int a_begin, int a_end,
                       cudaStream_t s) const;
    void adjoint_range(const float* proj, float* vol, int a_begin, int a_end, bool accumulate,
                       cudaStream_t s) const;
    // Adjoint of HOST projections into a HOST volume, reference layouts:
    // uploads in two angle parts, copies the volume out z level by z level
    // while the kernel runs (synchronous).  false: not available for this
    // handle (stage the data and use adjoint()).
    bool adjoint_host_ref(const float* host_proj, float* host, cudaStream_t s);
    // Host-buffer pipeline (capi.cu): angle chunks, a copy stream and events.
#ifndef KCT_PIPE_CHUNKS
#define KCT_PIPE_CHUNKS 6  // host-forward output chunks (counted launch: 6 measured best of 4 / 6 / 8)
#endif
    static constexpr int kPipeChunks = KCT_PIPE_CHUNKS, kPipeMinAngles = 4;
    int pipe_chunks() const { return pipe_chunks_; }
    int pipe_angle(int c) const { return (int)((long long)dg_.na * c / pipe_chunks_); }
    cudaStream_t pipe_stream();
    cudaEvent_t pipe_event(int i) const { return pipe_ev_[i]; }
    cudaEvent_t upload_event() const { return up_ev_; }
    // Split upload of a host volume (forward_host_pipelined): row band 0's
    // rays stay below slab fwd_split_z() (0: no split).
    int fwd_split_z() const { return fwd_split_z_; }
    int fwd_split_lo() const { return fwd_split_lo_; }  // mirror pairs: band 0 needs [lo, z)
    bool mirror() const { return mirror_; }
    void forward_split_lo(float* proj, cudaStream_t s) const;
    void forward_split_hi(float* proj, int chunk, cudaStream_t s) const;
    // The forward reads a padded copy of the native volume (column stride
    // nz + 2, zero slabs at -1 and nz: no per-load range checks).
    void pad_volume(const float* nat, cudaStream_t s) const;
    void vol_to_padded_z(const float* ref, int z0, int z1, cudaStream_t s) const;
    // forward of angles [a_begin, a_end) from the padded volume as it stands
    void forward_padded(float* proj, int a_begin, int a_end, cudaStream_t s) const;
    // Host pipeline: one launch of bands band0.. for all angles, chunk-major,
    // counting finished columns per pipeline chunk (fwd_chunk_columns each)
    // into fwd_done(); false-free: available when pipe_chunks() > 1.
    void forward_counted(float* proj, int band0, unsigned* done, cudaStream_t s) const;
    unsigned fwd_chunk_columns(int chunk, int band0) const;
    unsigned* fwd_done() const { return d_fdone_; }
    // Staged host forward (capi.cu forward_host_staged): stage s covers rows
    // (z-mirror: row pairs) [row0, row0 + 32 C) of every angle, whose rays stay
    // inside slabs [z_lo, z_hi); the volume is uploaded stage range by stage
    // range (centre out) and stage s runs as soon as its slabs are in; the last
    // stage is counted per pipeline chunk (fwd_done(), (a1 - a0) nu columns).
    struct FwdStage {
        int row0, C, z_lo, z_hi;
        size_t order_off;  // its block order in d_fstage_
    };
    const std::vector<FwdStage>& fwd_stages() const { return fstages_; }
    bool fwd_rowstages() const { return fwd_rowstages_; }
    void forward_stage(int stage, float* proj, unsigned* done, cudaStream_t s,
                       bool ref_out = false) const;
    // enqueue on `sc`: wait until *addr >= value (cuStreamWaitValue32); false
    // when stream memory operations are unavailable (nothing enqueued)
    bool stream_wait_geq(cudaStream_t sc, const unsigned* addr, unsigned value) const;
    // Per-ray count of positive-length Siddon segments (as float) into proj.
    void count(float* proj, cudaStream_t s) const;
    // FDK (fdk.hpp:50-139), native layouts; `filt` is N floats of scratch.
    void fdk(const float* proj, float* vol, float* filt, cudaStream_t s) const;

    // Layout conversions (device, stream-ordered).
    void vol_to_native(const float* ref, float* nat, cudaStream_t s) const;
    void vol_from_native(const float* nat, float* ref, cudaStream_t s) const;
    void proj_to_native(const float* ref, float* nat, cudaStream_t s) const;
    void proj_from_native(const float* nat, float* ref, cudaStream_t s) const;
    void proj_to_native_range(const float* ref, float* nat, int a0, int a1, cudaStream_t s) const;
    void proj_from_native_range(const float* nat, float* ref, int a0, int a1, cudaStream_t s) const;
    void proj_rows_from_native(const float* nat, float* ref, int v0, int v1, cudaStream_t s) const;

    // Lazily allocated scratch used by the C-ABI for host / reference-layout calls.
    float* scratch(int slot, size_t n);

    // Solver workspace cached across calls (owned by solver.cu).
    std::shared_ptr<void> workspace;
    // Angle-sharded multi-process mode (kct_set_allreduce).
    kct_allreduce_fn comm_fn = nullptr;
    void* comm_ctx = nullptr;
    // y-slab-sharded multi-process mode (kct_set_slab): this grid is planes
    // [slab_j0, slab_j0 + ny) of a grid with slab_nyg y planes.
    int slab_rank = -1, slab_world = 0, slab_j0 = 0, slab_nyg = 0;
    kct_halo_fn halo_fn = nullptr;
    void* halo_ctx = nullptr;
    bool slab_mode() const { return halo_fn != nullptr; }
    // Solver options (kct_set_option) and the per-iteration hook.
    bool solver_restart = false;  // KCT_SOLVER_RESTART=1 sets it at creation
    kct_iterate_hook hook_fn = nullptr;
    void* hook_ctx = nullptr;

    int fwd_chunks() const { return fwd_c_; }
    int adj_k() const { return adj_k_; }
    int adj_stride() const { return adj_S_; }
    int adj_bz() const { return adj_bz_; }
    bool adj_gather() const { return adj_gather_; }
    bool adj_slab() const { return adj_slab_; }
    bool adj_slab_detect() const { return adj_slab_detect_; }
    bool adj_mirror() const { return adj_mir_; }
    bool adj_ws() const { return adj_ws_; }
    int adj_np() const { return adj_np_; }
    int adj_mirror_bz() const { return adj_mbz_; }
    int adj_groups() const { return adj_groups_; }
    unsigned long long walk_entries() const { return tab_entries_; }
    unsigned long long fwd_table_segments() const { return ftab_segs_; }

  private:
    void build_tables(const kct_geometry& geom);
    size_t adj_smem_bytes() const;
    BrickCfg adj_cfg() const;
    void build_walk_table();
    void tune_adjoint();
    void build_fwd_table();
    FwdTab ftab(int a) const;
    void adjoint_impl(const float* proj, float* vol, int a_begin, int a_end, bool accumulate,
                      bool out_ref, unsigned* level_done, cudaStream_t s) const;

    kct_grid grid_;
    DevGeom dg_{};
    // geometry as given, float64 (FDK weights)
    double dso_d_ = 0, dsd_d_ = 0, pu_d_ = 0, pv_d_ = 0, offu_d_ = 0, offv_d_ = 0;
    int device_ = 0;
    size_t m_ = 0, n_ = 0;
    std::vector<float2> cs_;          // per-angle (cos, sin)
    ColParams* d_cols_ = nullptr;     // [na][nu]
    float* d_dv_ = nullptr;           // [nv] row heights dv(iv)
    float* d_invdv_ = nullptr;        // [nv] 1/dv (inf at dv == 0)
    double* d_dvd_ = nullptr;         // [nv] dv in float64
    RowTab* d_rows_ = nullptr;        // [nv] packed (dvd, dv, 1/dv) for the adjoint
    int fwd_c_ = 4, fwd_bands_ = 1, adj_k_ = 8;
    int adj_S_ = 2, adj_bz_ = 32;
    bool adj_gather_ = false;
    bool adj_slab_ = false;           // slab-lane adjoint deposits valid (brick_rows_slab)
    bool adj_slab_detect_ = false;    // ... with crossing-slot conflict detection
    bool adj_mir_ = false;            // z-mirror brick pairs (adj_mirror_kernel)
    bool adj_ws_ = false;             // ... warp-specialised (adj_mirror_ws_kernel)
    int adj_mbz_ = 64;                // ... slabs per lower brick
    int adj_parts_ = 1;               // y parts per z level of the host path's progress counters
    int* d_border_ = nullptr;         // brick order of the adjoint queue
    int* d_forder_ = nullptr;         // forward block -> item order (longest chords first)
    int* d_fpipe_ = nullptr;          // the same per pipeline chunk (offsets pipe_off_)
    std::vector<int> pipe_off_;
    int pipe_chunks_ = 1;
    cudaStream_t pipe_stream_ = nullptr;
    cudaEvent_t pipe_ev_[kPipeChunks] = {};
    cudaEvent_t up_ev_ = nullptr;
    int fwd_split_z_ = 0, fwd_split_lo_ = 0;
    std::vector<FwdStage> fstages_;   // staged host forward (empty: not used)
    bool fwd_rowstages_ = false;      // ... every stage's rows are copied out as the stage ends (opt-in)
    unsigned* d_ftab_off_ = nullptr;  // forward walk table: segment offsets [angle][column + 1]
    void* d_ftab_ = nullptr;          // ... segments (int2: bits of wb, padded column)
    unsigned long long ftab_segs_ = 0;
    int* d_fstage_ = nullptr;         // block orders of the stages
    bool mirror_ = false;             // z-mirror pairs (fwd_kernel MIR, adj_weight_kernel)
    float* d_vpad_ = nullptr;         // padded native volume read by the forward
    float2* d_cs_ = nullptr;          // per-angle (cos, sin) on the device
    int* d_flo_ = nullptr;            // block order of the split forward's band 0 (all angles)
    int* d_fhi_ = nullptr;            // ... of its bands 1.. per pipeline chunk (offsets fhi_off_)
    std::vector<int> fhi_off_;
    int* d_fcnt_all_ = nullptr;       // chunk-major block orders of forward_counted (all bands,
    int* d_fcnt_hi_ = nullptr;        //   bands 1..)
    unsigned* d_fdone_ = nullptr;     // finished columns per pipeline chunk
    int* d_queue_ = nullptr;          // adjoint brick queue counter
    int adj_ctas_ = 0;                // resident CTAs of the persistent adjoint grid
    int adj_ctas_np_[3] = {0, 0, 0};  // ... of the warp-specialised kernel with 1 / 2 / 3 producers
    int adj_np_ = 2;                  // producer warps per consumer (tune_adjoint)
    int adj_groups_ = 1;              // angle groups of the adjoint (small problems)
    float* d_part_ = nullptr;         // (adj_groups_ - 1) partial volumes
    float* d_yw_ = nullptr;           // adjoint per-ray records (float4, one angle batch)
    void* d_tab_ = nullptr;           // adjoint walk table (WalkEntry, projector.cu)
    unsigned long long* d_off_ = nullptr;  // walk-table offsets [brick][angle + 1]
    unsigned long long tab_entries_ = 0;
    unsigned* d_level_ = nullptr;     // finished bricks per z level (adjoint_host_ref)
    float* scratch_[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t scratch_n_[4] = {0, 0, 0, 0};
};

// Validation mirroring the reference (types.hpp:72-77, :152-160;
// projector.hpp:162-168).  Throws ConfigError.
void validate_geometry(const kct_grid& grid, const kct_geometry& geom);

}  // namespace kct
