// Device-side control of the ALS sweep (als.cpp:121-160) and the fused small
// dense steps around the two contractions.
//
// The stop rule runs on the GPU: finish_right_kernel evaluates the
// closed-form residual, records it in the history, applies
// |prev - res| / ||A|| <= eta and the max_iters cap, and raises `stop`; every
// kernel of the following (speculatively enqueued) iterations checks `stop`
// on entry and returns, so the host enqueues several sweeps at once and
// synchronises once per batch instead of once per sweep. Errors
// (singular Gram matrices) also raise `stop` with an error code that the
// host turns into the reference's RankTooLargeError (als.cpp:128-135).
#include <algorithm>
#include <cmath>

#include "als_step.cuh"

namespace tkg {

namespace {

__device__ double block_sum_t(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = (blockDim.x + 31) / 32;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

// G(a,b) (column-major r x r, symmetric) = X^T X for column-major X (n x r),
// rows streamed through shared memory in 64-row chunks; each entry is a
// sequential sum in row order (deterministic).
__device__ void block_gram(const double* X, uint32_t n, uint32_t r, double* G, double* tile) {
  const uint32_t ne = r * (r + 1) / 2;
  double acc[4] = {0, 0, 0, 0};
  for (uint32_t r0 = 0; r0 < n; r0 += 64) {
    const uint32_t nr = min(64u, n - r0);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < nr * r; e += blockDim.x) {
      const uint32_t row = e % nr, c = e / nr;
      tile[row * r + c] = X[(r0 + row) + uint64_t(c) * n];
    }
    __syncthreads();
    for (uint32_t k = 0; k < 4; ++k) {
      const uint32_t e = threadIdx.x + k * blockDim.x;
      if (e >= ne) break;
      // e -> (a, b) with a <= b, row-major upper triangle
      uint32_t a = 0, rem = e;
      while (rem >= r - a) { rem -= r - a; ++a; }
      const uint32_t b = a + rem;
      double s = acc[k];
      for (uint32_t row = 0; row < nr; ++row) s += tile[row * r + a] * tile[row * r + b];
      acc[k] = s;
    }
  }
  __syncthreads();
  for (uint32_t k = 0; k < 4; ++k) {
    const uint32_t e = threadIdx.x + k * blockDim.x;
    if (e >= ne) break;
    uint32_t a = 0, rem = e;
    while (rem >= r - a) { rem -= r - a; ++a; }
    const uint32_t b = a + rem;
    G[a + b * r] = acc[k];
    G[b + a * r] = acc[k];
  }
  __syncthreads();
}

// Lower Cholesky factor with spd_solve's pivot floor (kernels.cpp:378-393);
// floor_rel = 0 keeps only the "pivot > 0" test (CholQR). Returns the failing
// column + 1, or 0.
__device__ int block_chol2(const double* G, double* L, uint32_t r, double floor_rel, double* pivot_out) {
  __shared__ double floor_s, piv_s;
  __shared__ int fail_s;
  if (threadIdx.x == 0) {
    double md = 0.0;
    for (uint32_t i = 0; i < r; ++i) md = fmax(md, G[i + i * r]);
    floor_s = floor_rel * md;
    fail_s = 0;
  }
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) L[e] = 0.0;
  __syncthreads();
  for (uint32_t k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      double pivot = G[k + k * r];
      for (uint32_t p = 0; p < k; ++p) pivot -= L[k + p * r] * L[k + p * r];
      if (pivot <= floor_s || !(pivot > 0.0)) {
        fail_s = int(k) + 1;
        piv_s = pivot;
      } else {
        L[k + k * r] = sqrt(pivot);
      }
    }
    __syncthreads();
    if (fail_s) break;
    const double dkk = L[k + k * r];
    for (uint32_t i = k + 1 + threadIdx.x; i < r; i += blockDim.x) {
      double acc = G[i + k * r];
      for (uint32_t p = 0; p < k; ++p) acc -= L[i + p * r] * L[k + p * r];
      L[i + k * r] = acc / dkk;
    }
    __syncthreads();
  }
  if (pivot_out && fail_s && threadIdx.x == 0) *pivot_out = piv_s;
  return fail_s;
}

// x <- L^{-1} x (forward) and, unless forward_only, x <- L^{-T} x, in the
// order of spd_solve (kernels.cpp:401-415). x is strided in shared memory.
__device__ __forceinline__ void row_subst(const double* L, uint32_t r, double* x, uint32_t xs,
                                          bool forward_only) {
  for (uint32_t a = 0; a < r; ++a) {
    double acc = x[a * xs];
    for (uint32_t p = 0; p < a; ++p) acc -= L[a + p * r] * x[p * xs];
    x[a * xs] = acc / L[a + a * r];
  }
  if (forward_only) return;
  for (uint32_t a = r; a-- > 0;) {
    double acc = x[a * xs];
    for (uint32_t p = a + 1; p < r; ++p) acc -= L[p + a * r] * x[p * xs];
    x[a * xs] = acc / L[a + a * r];
  }
}

constexpr int kBig = 1024;  // threads of the one-CTA kernels

// ---- right-update preparation: G_L, chol, L' = L G_L^{-1} (i-major) ----------
__global__ void __launch_bounds__(kBig) prep_right_kernel(const double* __restrict__ L, uint32_t I,
                                                          uint32_t r, uint32_t ncp, double* GL,
                                                          double* cholL, double* Mt, AlsCtrl* ctrl,
                                                          uint32_t rb) {
  if (ctrl->stop) return;
  extern __shared__ double sm[];
  double* Gs = sm;               // r*r
  double* Ls = Gs + r * r;       // r*r
  double* tile = Ls + r * r;     // 64*r (gram) / reused as row buffers [r][kBig]
  block_gram(L, I, r, Gs, tile);
  double piv = 0.0;
  const int fail = block_chol2(Gs, Ls, r, 1e-13, &piv);
  if (fail) {
    if (threadIdx.x == 0) {
      ctrl->error = kAlsErrRightSingular;
      ctrl->pivot = piv;
      ctrl->stop = 1;
    }
    return;
  }
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    GL[e] = Gs[e];
    cholL[e] = Ls[e];
  }
  // rows: rb threads at a time, each solving one row (x in smem, stride rb)
  double* xs = tile;
  for (uint32_t i0 = 0; i0 < I; i0 += rb) {
    const uint32_t i = i0 + threadIdx.x;
    if (threadIdx.x < rb && i < I) {
      double* x = xs + threadIdx.x;
      for (uint32_t c = 0; c < r; ++c) x[c * rb] = L[i + uint64_t(c) * I];
      row_subst(Ls, r, x, rb, false);
      for (uint32_t c = 0; c < ncp; ++c) Mt[uint64_t(i) * ncp + c] = c < r ? x[c * rb] : 0.0;
    }
  }
}

// ---- closed-form residual and the stop rule (als.cpp:52-55, 136-160) ---------
__global__ void __launch_bounds__(kBig) finish_right_kernel2(const double* __restrict__ part, int nparts,
                                                             int rowstride, uint32_t r,
                                                             const double* GL, double* GR,
                                                             double* cholR, AlsCtrl* ctrl,
                                                             double* history) {
  if (ctrl->stop) return;
  extern __shared__ double sm[];
  double* Gs = sm;
  double* Ls = Gs + r * r;
  const uint64_t pld = uint64_t(rowstride) * rowstride;
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;
    const uint32_t a = min(i, j), b = max(i, j);
    const double* p = part + size_t(a) * rowstride + b;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < nparts; ++k) s += p[size_t(k) * pld];
    Gs[e] = s;
  }
  __syncthreads();
  __shared__ double hi_s[32], lo_s[32];
  if (threadIdx.x < 32) {
    double s = 0.0, c = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += 32) {
      const double p = GL[e] * Gs[e];
      const double pe = fma(GL[e], Gs[e], -p);
      double t, err;
      two_sum(s, p, t, err);
      s = t;
      c += err + pe;
    }
    hi_s[threadIdx.x] = s;
    lo_s[threadIdx.x] = c;
  }
  __syncthreads();
  __shared__ int cont_s;
  if (threadIdx.x == 0) {
    double s = 0.0, c = 0.0;
    for (int k = 0; k < 32; ++k) {
      double t, err;
      two_sum(s, hi_s[k], t, err);
      s = t;
      c += err + lo_s[k];
    }
    const double tr = s + c;
    const double residual = sqrt(fmax(0.0, ctrl->norm_sq - tr));
    const int it = ctrl->iter + 1;
    ctrl->iter = it;
    if (it <= ctrl->history_cap) history[it - 1] = residual;
    ctrl->residual = residual;
    const double achieved = fabs(ctrl->prev - residual) / ctrl->norm;
    ctrl->achieved = achieved;
    int cont = 1;
    if (achieved <= ctrl->eta) {
      ctrl->status = 0;  // kConverged
      cont = 0;
    } else if (it >= ctrl->max_iters) {
      ctrl->status = 1;  // kMaxItersReached
      cont = 0;
    }
    ctrl->prev = residual;
    cont_s = cont;
    if (!cont) ctrl->stop = 1;
  }
  __syncthreads();
  if (!cont_s) return;
  double piv = 0.0;
  const int fail = block_chol2(Gs, Ls, r, 1e-13, &piv);
  if (fail) {
    if (threadIdx.x == 0) {
      ctrl->error = kAlsErrLeftSingular;
      ctrl->pivot = piv;
      ctrl->stop = 1;
    }
    return;
  }
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    GR[e] = Gs[e];
    cholR[e] = Ls[e];
  }
}

// ---- left update: L = (sum of FR partials) G_R^{-1}, row blocks ------------------
constexpr int kLeftRows = 32;

__global__ void __launch_bounds__(256) left_solve_kernel(const double* __restrict__ part, int nparts,
                                                         uint32_t ldp, uint32_t I, uint32_t r,
                                                         const double* __restrict__ cholR, double* L,
                                                         const AlsCtrl* ctrl) {
  if (ctrl->stop) return;
  extern __shared__ double sm[];
  double* Ls = sm;                 // r*r
  double* ys = Ls + r * r;         // [r][kLeftRows]
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) Ls[e] = cholR[e];
  const uint32_t i0 = blockIdx.x * kLeftRows;
  const uint32_t nrow = min(uint32_t(kLeftRows), I - i0);
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    const double* p = part + (size_t(i0 + row)) * ldp + c;
    double s = 0.0;
#pragma unroll 4
    for (int k = 0; k < nparts; ++k) s += p[size_t(k) * I * ldp];
    ys[c * kLeftRows + row] = s;
  }
  __syncthreads();
  if (threadIdx.x < nrow) {
    double* x = ys + threadIdx.x;
    row_subst(Ls, r, x, kLeftRows, false);
    for (uint32_t c = 0; c < r; ++c) L[(i0 + threadIdx.x) + uint64_t(c) * I] = x[c * kLeftRows];
  }
}

// ---- one-CTA CholQR2 (Y = Q R, R_ii > 0) with the reference's degeneracy test -----
__global__ void __launch_bounds__(kBig) cholqr_kernel(const double* __restrict__ Yin, int nparts,
                                                      uint64_t ldp, uint32_t I, uint32_t r, double* Yw,
                                                      double* Q, double* rmat, double* rt, uint32_t ldrt,
                                                      int check, AlsCtrl* ctrl, uint32_t rb) {
  extern __shared__ double sm[];
  double* Gs = sm;
  double* L1 = Gs + r * r;
  double* L2 = L1 + r * r;
  double* tile = L2 + r * r;  // 64*r for the Gram, then [r][kBig] row buffers
  // Y (column-major I x r) from partials [k][I][ldp] or a column-major matrix (ld = ldp)
  for (uint64_t e = threadIdx.x; e < uint64_t(I) * r; e += blockDim.x) {
    const uint32_t i = uint32_t(e % I), c = uint32_t(e / I);
    double v;
    if (nparts > 0) {
      v = 0.0;
      for (int k = 0; k < nparts; ++k) v += Yin[(size_t(k) * I + i) * ldp + c];
    } else {
      v = Yin[i + c * ldp];
    }
    Yw[e] = v;
  }
  __syncthreads();
  int fail = 0;
  double* src = Yw;
  double* Ls[2] = {L1, L2};
  for (int pass = 0; pass < 2 && !fail; ++pass) {
    block_gram(src, I, r, Gs, tile);
    fail = block_chol2(Gs, Ls[pass], r, 0.0, nullptr);
    if (fail) break;
    double* dst = pass == 0 ? Yw : Q;  // in place for the first pass
    __syncthreads();
    for (uint32_t i0 = 0; i0 < I; i0 += rb) {
      const uint32_t i = i0 + threadIdx.x;
      if (threadIdx.x < rb && i < I) {
        double* x = tile + threadIdx.x;
        for (uint32_t c = 0; c < r; ++c) x[c * rb] = src[i + uint64_t(c) * I];
        row_subst(Ls[pass], r, x, rb, true);
        for (uint32_t c = 0; c < r; ++c) dst[i + uint64_t(c) * I] = x[c * rb];
      }
    }
    __syncthreads();
    src = dst;
  }
  // R = R2 R1, R_k = L_k^T (upper)
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;
    double acc = 0.0;
    if (!fail && i <= j)
      for (uint32_t k = i; k <= j; ++k) acc += L2[k + i * r] * L1[j + k * r];
    Gs[e] = acc;
    if (rmat) rmat[e] = acc;
  }
  __syncthreads();
  if (rt)
    for (uint32_t e = threadIdx.x; e < r * ldrt; e += blockDim.x) {
      const uint32_t row = e / ldrt, c = e % ldrt;
      rt[e] = c < r ? Gs[c + row * r] : 0.0;
    }
  if (threadIdx.x == 0) {
    int bad = 0;
    if (fail) {
      bad = fail;
    } else if (check) {
      double md = 0.0;  // als.cpp:74-86
      for (uint32_t i = 0; i < r; ++i) md = fmax(md, fabs(Gs[i + i * r]));
      for (uint32_t i = 0; i < r; ++i)
        if (fabs(Gs[i + i * r]) <= 1e-13 * md || md == 0.0) {
          bad = int(i) + 1;
          break;
        }
    }
    ctrl->degenerate_col = bad;
  }
}

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

template <class K>
cudaError_t smem_attr(K k, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

}  // namespace

// One-CTA kernels: kBig threads for the Gram phase; the row solves use rb
// threads at a time so that r*rb row buffers fit in shared memory.
static uint32_t rows_per_round(uint32_t r, int mats) {
  const size_t budget = 200 * 1024 / sizeof(double) - size_t(mats) * r * r;
  size_t t = std::min<size_t>(kBig, budget / std::max<uint32_t>(r, 1));
  return uint32_t(std::max<size_t>(32, t));
}

cudaError_t launch_prep_right(const double* L, uint32_t I, uint32_t r, uint32_t ncp, double* GL,
                              double* cholL, double* Mt, AlsCtrl* ctrl, cudaStream_t st) {
  const uint32_t rb = rows_per_round(r, 2);
  const size_t smem = sizeof(double) * (2 * size_t(r) * r + std::max<size_t>(64 * r, size_t(r) * rb));
  cudaError_t e = smem_attr(prep_right_kernel, smem);
  if (e != cudaSuccess) return e;
  prep_right_kernel<<<1, kBig, smem, st>>>(L, I, r, ncp, GL, cholL, Mt, ctrl, rb);
  return cudaGetLastError();
}

cudaError_t launch_finish_right2(const double* part, int nparts, int rowstride, uint32_t r,
                                 const double* GL, double* GR, double* cholR, AlsCtrl* ctrl,
                                 double* history, cudaStream_t st) {
  finish_right_kernel2<<<1, kBig, sizeof(double) * 2 * r * r, st>>>(part, nparts, rowstride, r, GL, GR,
                                                                     cholR, ctrl, history);
  return cudaGetLastError();
}

cudaError_t launch_left_solve(const double* part, int nparts, uint32_t ldp, uint32_t I, uint32_t r,
                              const double* cholR, double* L, const AlsCtrl* ctrl, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t(r) * r + size_t(r) * kLeftRows);
  left_solve_kernel<<<(I + kLeftRows - 1) / kLeftRows, 256, smem, st>>>(part, nparts, ldp, I, r, cholR,
                                                                          L, ctrl);
  return cudaGetLastError();
}

cudaError_t launch_cholqr(const double* Y, int nparts, uint64_t ldp, uint32_t I, uint32_t r, double* Yw,
                          double* Q, double* rmat, double* rt, uint32_t ldrt, int check, AlsCtrl* ctrl,
                          cudaStream_t st) {
  const uint32_t rb = rows_per_round(r, 3);
  const size_t smem = sizeof(double) * (3 * size_t(r) * r + std::max<size_t>(64 * r, size_t(r) * rb));
  cudaError_t e = smem_attr(cholqr_kernel, smem);
  if (e != cudaSuccess) return e;
  cholqr_kernel<<<1, kBig, smem, st>>>(Y, nparts, ldp, I, r, Yw, Q, rmat, rt, ldrt, check, ctrl, rb);
  return cudaGetLastError();
}

cudaError_t launch_ctrl_init(AlsCtrl* ctrl, const double* sumsq, double eta, int max_iters,
                             int history_cap, int check_degenerate, cudaStream_t st) {
  ctrl_init_kernel<<<1, 1, 0, st>>>(ctrl, sumsq, eta, max_iters, history_cap, check_degenerate);
  return cudaGetLastError();
}

}  // namespace tkg
