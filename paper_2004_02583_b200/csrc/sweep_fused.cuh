// One ALS sweep's two contractions from ONE read of the tensor
// (sweep_fused.cu): R = A_(n)^T L' (right update, als.cpp:36-44), R^T R, and
// the left-update sum Y = A_(n) R (als.cpp:46-50). A row of R depends only on
// its own fiber, so a CTA that holds whole fibers in shared memory forms its
// rows of R and at once adds their outer-product contribution to Y. At ranks
// up to 16 both contractions are HBM-bound, so the sweep's
// tensor traffic halves.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace tkg {

struct SweepFusedArgs {
  const double* mt = nullptr;      // L' = L G_L^-1, i-major [K][ncp] (the FC operand)
  uint32_t nc = 0;                 // r
  double* R = nullptr;             // row-major [F][ncp] (fiber j = p*s + jl at row j)
  double* partial = nullptr;       // [grid][K][ncp] left-update partials (the FR layout)
  double* gram_part = nullptr;     // [grid][ncp*ncp] upper tiles of R^T R (the FC-epilogue layout)
  const int32_t* skip = nullptr;   // device flag: return at once when set
};

// Layouts and sizes the fused sweep covers: r <= 16, K <= 256 even, mode-1
// fibers (s == 1) or panels of at least one tile of even length.
bool sweep_fused_ok(const FiberView& v, const double* mt, uint32_t nc, const double* R);
// CTAs launched (= partials written)
int sweep_fused_grid(const FiberView& v, uint32_t nc, int num_sms);
cudaError_t launch_sweep_fused(const FiberView& v, const SweepFusedArgs& a, int num_sms, cudaStream_t st,
                               int* grid_used);

}  // namespace tkg
