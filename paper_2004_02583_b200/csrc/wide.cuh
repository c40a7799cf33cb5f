// Small dense steps for ranks above 64 (wide.cu), used by engine_wide.cpp.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "als_step.cuh"

namespace tkg {

// Cholesky C (lower) and C^T of the n x n Gram G (column-major), spd_solve's
// pivot floor floor_rel * max diag (kernels.cpp:378-393; 0 = positivity
// only). *fail_out: failing column (1-based) or 0. With ctrl and err_code a
// failure raises ctrl->error = err_code and stop (and the kernel is skipped
// once stop is set).
cudaError_t launch_wide_chol(const double* G, uint32_t n, double floor_rel, double* C, double* CT,
                             int32_t* fail_out, AlsCtrl* ctrl, int err_code, cudaStream_t st);
// Per row of X (m rows, x(row, c) = X[row*xr + c*xc]): C y = x, and with
// back also C^T z = y; the result into O[row*or_ + c*oc] (O may alias X).
cudaError_t launch_wide_rowsolve(const double* X, uint64_t m, uint32_t n, uint64_t xr, uint64_t xc, const double* C,
                                 const double* CT, int back, double* O, uint64_t or_, uint64_t oc,
                                 const AlsCtrl* ctrl, int num_sms, cudaStream_t st);
// closed-form residual, history and stop rule (als.cpp:52-55, 136-150)
cudaError_t launch_wide_trace_stop(const double* GL, const double* GR, uint32_t n, AlsCtrl* ctrl, double* history,
                                   cudaStream_t st);
// CholQR2's R = C2^T C1^T (nullable) and ctrl->degenerate_col (fails[0..1]:
// the two factorizations' failing columns; check: als.cpp:74-86 on diag R)
cudaError_t launch_wide_rprod(const double* C2, const double* C1, uint32_t n, double* R, const int32_t* fails,
                              int check, AlsCtrl* ctrl, cudaStream_t st);

}  // namespace tkg
