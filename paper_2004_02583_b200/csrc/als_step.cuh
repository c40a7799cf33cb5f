// Device-side ALS control block and the fused small-LA kernels (als_step.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace tkg {

enum {
  kAlsErrNone = 0,
  kAlsErrRightSingular = 1,
  kAlsErrLeftSingular = 2,
  kAlsErrZeroNorm = 3,
  kAlsErrDegenerate = 4
};

// Lives in mapped pinned memory: written by the kernels, read by the host
// once per batch of sweeps.
struct AlsCtrl {
  int32_t stop;          // any kernel of a later sweep returns immediately
  int32_t iter;          // sweeps completed (report.iterations)
  int32_t status;        // 0 kConverged, 1 kMaxItersReached (als.hpp:25)
  int32_t error;         // kAlsErr*
  int32_t max_iters;
  int32_t history_cap;
  int32_t degenerate_col;  // CholQR: als_init collapse column (1-based), 0 if none
  int32_t pad;
  double norm, norm_sq, prev, eta, residual, achieved, pivot;
};

// norm = sqrt(*sumsq); raises stop + error for a zero norm or (check) a
// collapsed initializer reported by launch_cholqr in ctrl->degenerate_col.
cudaError_t launch_ctrl_init(AlsCtrl* ctrl, const double* sumsq, double eta, int max_iters,
                             int history_cap, int check_degenerate, cudaStream_t st);
// G_L = L^T L, chol with the spd_solve floor, Mt[i][c] = (L G_L^{-1})(i, c)
cudaError_t launch_prep_right(const double* L, uint32_t I, uint32_t r, uint32_t ncp, double* GL,
                              double* cholL, double* Mt, AlsCtrl* ctrl, cudaStream_t st);
// G_R from Gram partials, residual, stop rule, chol(G_R) for the left update
cudaError_t launch_finish_right2(const double* part, int nparts, int rowstride, uint32_t r,
                                 const double* GL, double* GR, double* cholR, AlsCtrl* ctrl,
                                 double* history, cudaStream_t st);
// L = (sum_k part[k]) G_R^{-1}, column-major out
cudaError_t launch_left_solve(const double* part, int nparts, uint32_t ldp, uint32_t I, uint32_t r,
                              const double* cholR, double* L, const AlsCtrl* ctrl, cudaStream_t st);
// One-CTA CholQR2 of Y (partials [k][I][ldp] or column-major with ld ldp);
// Yw: I*r scratch. Sets ctrl->degenerate_col.
cudaError_t launch_cholqr(const double* Y, int nparts, uint64_t ldp, uint32_t I, uint32_t r, double* Yw,
                          double* Q, double* rmat, double* rt, uint32_t ldrt, int check, AlsCtrl* ctrl,
                          cudaStream_t st);

}  // namespace tkg
