// Small dense steps of the ALS sweep for ranks above 64 (engine_wide.cpp).
//
// The cooperative steps of coop.cu keep an r x r matrix in registers of one
// CTA (r <= 64). Above that the r x r Gram matrices live in global memory
// (r = 256: 512 KB, L2-resident) and the steps are restated the reference's
// way (kernels.cpp:369-417): a Cholesky factor C of the Gram with spd_solve's
// pivot floor, then forward / back substitution applied row by row to the
// I_n x r factor (one warp per row, the row in shared memory), so
//   L' = L G_L^{-1}   (C C^T z = l per row of L; the FC operand, als.cpp:41)
//   L  = Y G_R^{-1}   (the left solve, als.cpp:49)
//   Q  = Y R^{-1}     (CholQR2 with R = C^T: forward substitution only).
// Reductions inside a row run in a fixed order (deterministic).
#include <cmath>

#include "als_step.cuh"
#include "wide.cuh"

namespace tkg {

namespace {

constexpr int kCholThreads = 1024;
constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;

// Right-looking Cholesky of G (column-major n x n) into C (lower, column-major)
// and CT (C^T, column-major, i.e. C row-major). Pivot test as spd_solve
// (kernels.cpp:378-393): pivot <= floor_rel * max diag or not > 0 fails
// (floor_rel 0: positivity only, the CholQR factorizations). *fail_out =
// failing column (1-based) or 0; with ctrl (solve steps) a failure also
// raises err_code and stop, as the cooperative steps do.
__global__ void __launch_bounds__(kCholThreads) wide_chol_kernel(const double* __restrict__ G, uint32_t n,
                                                                 double floor_rel, double* __restrict__ C,
                                                                 double* __restrict__ CT, int32_t* fail_out,
                                                                 AlsCtrl* ctrl, int err_code) {
  if (ctrl && err_code && ctrl->stop) return;
  __shared__ double red[32];
  __shared__ double md_s;
  const uint32_t nn = n * n;
  double md = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) md = fmax(md, G[i + uint64_t(i) * n]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = md;
  for (uint32_t e = threadIdx.x; e < nn; e += blockDim.x) {
    const uint32_t i = e % n, j = e / n;
    C[e] = i >= j ? G[e] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    md_s = m;
  }
  __syncthreads();
  const double floor_v = floor_rel * md_s;
  for (uint32_t k = 0; k < n; ++k) {
    const double p = C[k + uint64_t(k) * n];
    if (!(p > floor_v) || !(p > 0.0)) {
      if (threadIdx.x == 0) {
        *fail_out = int32_t(k) + 1;
        if (ctrl && err_code) {
          ctrl->error = err_code;
          ctrl->pivot = p;
          ctrl->pad = int32_t(k) + 1;
          ctrl->stop = 1;
        }
      }
      return;
    }
    const double d = sqrt(p);
    __syncthreads();  // everyone has read the pivot
    for (uint32_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) C[i + uint64_t(k) * n] /= d;
    if (threadIdx.x == 0) C[k + uint64_t(k) * n] = d;
    __syncthreads();
    const uint32_t m = n - k - 1;
    for (uint32_t e = threadIdx.x; e < m * m; e += blockDim.x) {
      const uint32_t i = k + 1 + e % m, j = k + 1 + e / m;
      if (i >= j) C[i + uint64_t(j) * n] -= C[i + uint64_t(k) * n] * C[j + uint64_t(k) * n];
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < nn; e += blockDim.x) {
    const uint32_t i = e % n, j = e / n;
    CT[j + uint64_t(i) * n] = C[e];
  }
  if (threadIdx.x == 0) *fail_out = 0;
}

// One warp per row x (x(row, c) = X[row*xr + c*xc]): forward substitution
// C y = x, then (back) C^T z = y; out(row, c) = O[row*or_ + c*oc]. C(i, p)
// for fixed i is CT[p + i*n] (contiguous), C(p, i) for fixed i is C[p + i*n].
// Skipped when ctrl->stop is raised (ctrl nullable).
__global__ void __launch_bounds__(kSolveThreads) wide_rowsolve_kernel(
    const double* X, uint64_t m, uint32_t n, uint64_t xr, uint64_t xc, const double* __restrict__ C,
    const double* __restrict__ CT, int back, double* O, uint64_t or_, uint64_t oc, const AlsCtrl* ctrl) {
  if (ctrl && ctrl->stop) return;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* y = sm + size_t(warp) * n;
  for (uint64_t row = uint64_t(blockIdx.x) * kSolveWarps + warp; row < m; row += uint64_t(gridDim.x) * kSolveWarps) {
    for (uint32_t c = lane; c < n; c += 32) y[c] = X[row * xr + c * xc];
    __syncwarp();
    for (uint32_t i = 0; i < n; ++i) {
      const double* ci = CT + uint64_t(i) * n;
      double s = 0.0;
      for (uint32_t p = lane; p < i; p += 32) s = fma(ci[p], y[p], s);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) y[i] = (y[i] - s) / ci[i];
      __syncwarp();
    }
    if (back) {
      for (uint32_t i = n; i-- > 0;) {
        const double* ci = C + uint64_t(i) * n;
        double s = 0.0;
        for (uint32_t p = i + 1 + lane; p < n; p += 32) s = fma(ci[p], y[p], s);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) y[i] = (y[i] - s) / ci[i];
        __syncwarp();
      }
    }
    for (uint32_t c = lane; c < n; c += 32) O[row * or_ + c * oc] = y[c];
    __syncwarp();
  }
}

// Closed-form residual sqrt(max(0, ||A||^2 - trace(G_L G_R))) with a
// compensated trace, the history entry and the stop rule (als.cpp:52-55,
// 136-150) -- the CTA-0 phase of finish_step for r > 64.
__global__ void __launch_bounds__(256) wide_trace_stop_kernel(const double* __restrict__ GL,
                                                              const double* __restrict__ GR, uint32_t n,
                                                              AlsCtrl* ctrl, double* history) {
  if (ctrl->stop) return;
  __shared__ double hi_s[256], lo_s[256];
  double s = 0.0, c = 0.0;
  for (uint64_t e = threadIdx.x; e < uint64_t(n) * n; e += blockDim.x) {
    const double p = GL[e] * GR[e];
    const double pe = fma(GL[e], GR[e], -p);
    double t, err;
    two_sum(s, p, t, err);
    s = t;
    c += err + pe;
  }
  hi_s[threadIdx.x] = s;
  lo_s[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x != 0) return;
  s = 0.0;
  c = 0.0;
  for (int k = 0; k < int(blockDim.x); ++k) {
    double t, err;
    two_sum(s, hi_s[k], t, err);
    s = t;
    c += err + lo_s[k];
  }
  const double residual = sqrt(fmax(0.0, ctrl->norm_sq - (s + c)));
  const int it = ctrl->iter + 1;
  ctrl->iter = it;
  if (it <= ctrl->history_cap) history[it - 1] = residual;
  ctrl->residual = residual;
  const double achieved = fabs(ctrl->prev - residual) / ctrl->norm;
  ctrl->achieved = achieved;
  bool stop = false;
  if (achieved <= ctrl->eta) {
    ctrl->status = 0;
    stop = true;
  } else if (it >= ctrl->max_iters) {
    ctrl->status = 1;
    stop = true;
  }
  ctrl->prev = residual;
  if (stop) ctrl->stop = 1;
}

// R = R2 R1 = C2^T C1^T (upper, column-major) of CholQR2, and the outcome:
// the first failed factorization's column, else (check) the reference's
// collapse test on diag(R) (als.cpp:74-86), into ctrl->degenerate_col.
__global__ void wide_rprod_kernel(const double* __restrict__ C2, const double* __restrict__ C1, uint32_t n,
                                  double* R, const int32_t* fails, int check, AlsCtrl* ctrl) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool ok = fails[0] == 0 && fails[1] == 0;
  if (R && ok && e < uint64_t(n) * n) {
    const uint32_t i = uint32_t(e % n), j = uint32_t(e / n);
    double acc = 0.0;
    if (i <= j)
      for (uint32_t k = i; k <= j; ++k) acc += C2[k + uint64_t(i) * n] * C1[j + uint64_t(k) * n];
    R[e] = acc;
  }
  if (e != 0 || !ctrl) return;
  int bad = fails[0] ? fails[0] : fails[1];
  if (!bad && check) {
    double md = 0.0;
    for (uint32_t i = 0; i < n; ++i) md = fmax(md, fabs(C2[i + uint64_t(i) * n] * C1[i + uint64_t(i) * n]));
    for (uint32_t i = 0; i < n; ++i)
      if (fabs(C2[i + uint64_t(i) * n] * C1[i + uint64_t(i) * n]) <= 1e-13 * md || md == 0.0) {
        bad = int(i) + 1;
        break;
      }
  }
  ctrl->degenerate_col = bad;
}

}  // namespace

size_t wide_rowsolve_smem(uint32_t n) { return size_t(kSolveWarps) * n * sizeof(double); }

cudaError_t launch_wide_chol(const double* G, uint32_t n, double floor_rel, double* C, double* CT,
                             int32_t* fail_out, AlsCtrl* ctrl, int err_code, cudaStream_t st) {
  wide_chol_kernel<<<1, kCholThreads, 0, st>>>(G, n, floor_rel, C, CT, fail_out, ctrl, err_code);
  return cudaGetLastError();
}

cudaError_t launch_wide_rowsolve(const double* X, uint64_t m, uint32_t n, uint64_t xr, uint64_t xc, const double* C,
                                 const double* CT, int back, double* O, uint64_t or_, uint64_t oc,
                                 const AlsCtrl* ctrl, int num_sms, cudaStream_t st) {
  const size_t smem = wide_rowsolve_smem(n);
  cudaError_t e = raise_smem_limit(wide_rowsolve_kernel, smem);
  if (e != cudaSuccess) return e;
  const uint64_t blocks = (m + kSolveWarps - 1) / kSolveWarps;
  const unsigned grid = unsigned(std::min<uint64_t>(blocks, uint64_t(num_sms) * 8));
  wide_rowsolve_kernel<<<std::max(1u, grid), kSolveThreads, smem, st>>>(X, m, n, xr, xc, C, CT, back, O, or_, oc,
                                                                        ctrl);
  return cudaGetLastError();
}

cudaError_t launch_wide_trace_stop(const double* GL, const double* GR, uint32_t n, AlsCtrl* ctrl, double* history,
                                   cudaStream_t st) {
  wide_trace_stop_kernel<<<1, 256, 0, st>>>(GL, GR, n, ctrl, history);
  return cudaGetLastError();
}

cudaError_t launch_wide_rprod(const double* C2, const double* C1, uint32_t n, double* R, const int32_t* fails,
                              int check, AlsCtrl* ctrl, cudaStream_t st) {
  const uint64_t nn = uint64_t(n) * n;
  wide_rprod_kernel<<<unsigned((nn + 255) / 256), 256, 0, st>>>(C2, C1, n, R, fails, check, ctrl);
  return cudaGetLastError();
}

}  // namespace tkg
