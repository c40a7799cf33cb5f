// Device-side ALS control block (als_step.cu); the small dense steps that
// read and update it are in coop.cu.
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

// Lives in device memory: written by the kernels, copied to the host once
// per batch of sweeps.
struct AlsCtrl {
  int32_t stop;          // any kernel of a later sweep returns immediately
  int32_t iter;          // sweeps completed (report.iterations)
  int32_t status;        // 0 kConverged, 1 kMaxItersReached (als.hpp:25)
  int32_t error;         // kAlsErr*
  int32_t max_iters;
  int32_t history_cap;
  int32_t degenerate_col;  // CholQR: als_init collapse column (1-based), 0 if none
  int32_t pad;             // failing Gram column (1-based) of a singular solve
  int32_t trips;           // sweeps begun inside a device-side loop (graph mode guard)
  int32_t pad2;
  double norm, norm_sq, prev, eta, residual, achieved, pivot;
};

// norm = sqrt(*sumsq); raises stop + error for a zero norm or (check) a
// collapsed initializer reported by launch_cholqr in ctrl->degenerate_col.
cudaError_t launch_ctrl_init(AlsCtrl* ctrl, const double* sumsq, double eta, int max_iters,
                             int history_cap, int check_degenerate, cudaStream_t st);
}  // namespace tkg
