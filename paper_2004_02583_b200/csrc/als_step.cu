// Device-side control of the ALS sweep (als.cpp:121-160).
//
// The stop rule runs on the GPU: finish_step (coop.cu) evaluates the
// closed-form residual, records it in the history, applies
// |prev - res| / ||A|| <= eta and the max_iters cap, and raises `stop`; every
// kernel of the following (speculatively enqueued) sweeps checks `stop` on
// entry and returns, so the host enqueues several sweeps at once and
// synchronises once per batch instead of once per sweep. Errors (singular
// Gram matrices) also raise `stop` with an error code that the host turns
// into the reference's RankTooLargeError (als.cpp:128-135).
#include <cmath>

#include "als_step.cuh"

namespace tkg {

namespace {

__global__ void ctrl_init_kernel(AlsCtrl* ctrl, const double* sumsq, double eta, int max_iters,
                                 int history_cap, int check_degenerate) {
  const double norm = sqrt(*sumsq);  // frobenius_norm (tensor_ops.cpp:391-393)
  const int degenerate = check_degenerate ? ctrl->degenerate_col : 0;
  ctrl->norm = norm;
  ctrl->norm_sq = norm * norm;       // als.cpp:106
  ctrl->prev = norm;                 // als.cpp:123
  ctrl->eta = eta;
  ctrl->max_iters = max_iters < 1 ? 1 : max_iters;
  ctrl->history_cap = history_cap;
  ctrl->iter = 0;
  ctrl->trips = 0;
  ctrl->status = 1;
  ctrl->error = 0;
  ctrl->stop = 0;
  ctrl->residual = 0.0;
  ctrl->achieved = 0.0;
  // als.cpp:102-105 (zero norm) precedes the initializer's collapse test (:74-86)
  if (norm == 0.0) {
    ctrl->error = kAlsErrZeroNorm;
    ctrl->stop = 1;
  } else if (degenerate) {
    ctrl->error = kAlsErrDegenerate;
    ctrl->stop = 1;
  }
}

}  // namespace

cudaError_t launch_ctrl_init(AlsCtrl* ctrl, const double* sumsq, double eta, int max_iters,
                             int history_cap, int check_degenerate, cudaStream_t st) {
  ctrl_init_kernel<<<1, 1, 0, st>>>(ctrl, sumsq, eta, max_iters, history_cap, check_degenerate);
  return cudaGetLastError();
}

}  // namespace tkg
