// Cooperative small dense steps of the ALS sweep (coop.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "als_step.cuh"

namespace tkg {

struct PrepArgs {
  double* part = nullptr;        // FR partials [nparts][I][ldp] (from_partials; summed
                                 // into slot 0, which then holds L row-major)
  int nparts = 0;
  uint32_t ldp = 0;
  const double* GRinv = nullptr; // r x r
  int from_partials = 0;
  uint32_t I = 0, r = 0, ncp = 0;
  double* Lc = nullptr;          // I x r column-major (read, or written when from_partials)
  double* GL = nullptr;          // r x r
  double* GLinv = nullptr;       // r x r
  double* Mt = nullptr;          // [I][ncp]
  double* gpart = nullptr;       // [grid][r*r]
  double* gs = nullptr;          // r x r scratch (reduced Gram)
  AlsCtrl* ctrl = nullptr;
};

// Sweeps run as the body of a CUDA-graph WHILE node (Engine::run_als): the
// finish step sets the node's condition to "continue" (cudaGraphSetConditional)
// and to 0 on every path that stops; 0 = not in a graph.
using GraphCond = unsigned long long;

struct FinishArgs {
  const double* R = nullptr;     // row-major [F][ld]
  uint64_t F = 0, ld = 0;
  uint32_t r = 0;
  const double* GL = nullptr;
  double* GRinv = nullptr;
  double* gpart = nullptr;       // [grid][ncp*ncp]
  double* gs = nullptr;          // r x r scratch (reduced Gram)
  AlsCtrl* ctrl = nullptr;
  double* history = nullptr;
  int gram_nparts = 0;           // > 0: gpart already holds this many Gram partials
                                 // (fused into the FC epilogue), no R pass
  GraphCond cond = 0;            // WHILE-node condition handle (graph mode)
  int mode = 0;                  // 0 full step; 1 only the R^T R partials of the R pass
                                 // (gpart[grid], see finish_step_grid); 2 only the CTA-0
                                 // part from the reduced Gram in gs (sharded runs)
  int gram_tail = 0;             // set by the launcher: r mod 8 in {1, 2}, the last column
                                 // tile of the R pass runs as a DFMA tail (see fc_tma_kernel)
};

struct CholQrArgs {
  double* Y = nullptr;           // partials [nparts][I][ldp] (summed into slot 0) or
                                 // column-major (ld = ldp, nparts 0, not written)
  int nparts = 0;
  uint64_t ldp = 0;
  uint32_t I = 0, r = 0;
  double* Q = nullptr;           // I x r column-major
  double* rmat = nullptr;        // r x r (nullable)
  double* rt = nullptr;          // R^T padded i-major (nullable)
  uint32_t ldrt = 0;
  int check = 0;
  double* gpart = nullptr;       // [grid][r*r]
  double* gs = nullptr;          // r x r scratch (reduced Gram)
  double* L1 = nullptr;          // r*r scratch
  double* Rinv = nullptr;        // r*r scratch
  double* work = nullptr;        // 2 doubles
  AlsCtrl* ctrl = nullptr;       // degenerate_col
};

// Upper bound on the grid of any launch below (sizes the gpart buffers).
int coop_partials_cap(int num_sms);
int finish_step_grid(uint64_t F, int num_sms);
cudaError_t launch_prep_step(PrepArgs a, int num_sms, cudaStream_t st);
cudaError_t launch_finish_step(FinishArgs a, int num_sms, cudaStream_t st);
cudaError_t launch_cholqr_step(CholQrArgs a, int num_sms, cudaStream_t st);

}  // namespace tkg
