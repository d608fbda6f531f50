// solver.cuh — device-resident CGLS and the iteratively reweighted drivers.
//
// Replaces cgls (krylov.hpp:59-127), irn_tv / irn_piple / irn_piccs
// (recon.hpp:169-270), cgls_recon (recon.hpp:274-315), evaluate_objective
// (recon.hpp:93-120), tv_weights (diffreg.hpp:142-156) and the StackedMap /
// ComposedMap / DiagonalMap algebra (linear_map.hpp:84-216) of the stacked
// least-squares system.
#pragma once

#include "projector.cuh"

namespace kct {

double resolve_tau(double tau, const float* host_ref, size_t n);

void cgls_recon(Projector& P, const float* b, size_t iters, const float* x0, const float* gt,
                double tol, float* x_out, kct_report* rep, int mem, int layout, cudaStream_t s);

void irn_solve(Projector& P, int kind, const float* b, const float* prior, const float* x0,
               const float* gt, const kct_reg_params& params, float* x_out, kct_report* rep,
               int mem, int layout, cudaStream_t s);

// cgls over a caller-assembled StackedMap (krylov.hpp:59-127, linear_map.hpp:159-216)
void cgls_stack(Projector& P, const kct_stack_block* blocks, size_t n_blocks, const float* b,
                const float* x0, size_t iters, double tol, float* x_out, kct_report* rep, int mem,
                int layout, cudaStream_t s);

// Staging helpers shared with capi.cu.
const float* stage_in(Projector& P, const float* src, size_t n, bool is_vol, int mem, int layout,
                      int slot, int tmp_slot, cudaStream_t s);
void stage_out(Projector& P, const float* nat, float* dst, size_t n, bool is_vol, int mem,
               int layout, int tmp_slot, cudaStream_t s);

}  // namespace kct
