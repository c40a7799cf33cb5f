// Cooperative (grid-synchronised) small dense steps of the ALS sweep.
//
// Each step is one launch whose phases are separated by grid.sync(): row
// blocks of the I x r factor are processed by many CTAs (32 rows each), the
// r x r factorizations by CTA 0. The normal-equation solves use the explicit
// inverse of the r x r Gram matrix (from its Cholesky factor, with the
// spd_solve pivot floor, kernels.cpp:378-393), so applying it to a row is an
// r-wide dot product per output instead of a dependent substitution chain.
//
//   prep_step   : [L = (sum FR partials) G_R^{-1}]  G_L = L^T L  chol  G_L^{-1}
//                 Mt = L G_L^{-1} (i-major, the FC operand)     (als.cpp:36-50)
//   finish_step : G_R = R^T R (DMMA), closed-form residual, the stop rule,
//                 chol(G_R) and G_R^{-1} for the next left update (als.cpp:52-55,136-160)
//   cholqr_step : CholQR2 thin QR with R_ii > 0 and the reference's
//                 degeneracy test (kernels.cpp:303-367, als.cpp:74-86)
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "als_step.cuh"
#include "coop.cuh"

namespace cg = cooperative_groups;

namespace tkg {

namespace {

constexpr int kRowsB = 32;     // factor rows per CTA
constexpr int kThreads = 256;

// Lower Cholesky of G (column-major r x r) into L; floor_rel as spd_solve.
// Returns failing column + 1 or 0. One CTA.
__device__ int chol_cta(const double* G, double* L, uint32_t r, double floor_rel, double* piv_out) {
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
  if (piv_out && fail_s && threadIdx.x == 0) *piv_out = piv_s;
  const int f = fail_s;
  __syncthreads();
  return f;
}

// Linv = L^{-1} (lower), column c by forward substitution on e_c. One CTA.
__device__ void tri_inv_cta(const double* L, double* Linv, uint32_t r) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) Linv[e] = 0.0;
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < r; c += blockDim.x) {
    for (uint32_t a = c; a < r; ++a) {
      double acc = a == c ? 1.0 : 0.0;
      for (uint32_t p = c; p < a; ++p) acc -= L[a + p * r] * Linv[p + c * r];
      Linv[a + c * r] = acc / L[a + a * r];
    }
  }
  __syncthreads();
}

// Ginv = L^{-T} L^{-1} (symmetric, column-major). One CTA.
__device__ void spd_inv_cta(const double* Linv, double* Ginv, uint32_t r) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t a = e % r, c = e / r;
    const uint32_t k0 = max(a, c);
    double s = 0.0;
    for (uint32_t k = k0; k < r; ++k) s += Linv[k + a * r] * Linv[k + c * r];
    Ginv[e] = s;
  }
  __syncthreads();
}

// Upper-triangle Gram partial of the CTA's rows (rows x r, row-major in smem,
// pitch ld): part[(a, b)] at a*r + b for a <= b.
__device__ void rows_gram(const double* X, uint32_t nrow, uint32_t r, uint32_t ld, double* part) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t a = e / r, b = e % r;
    double s = 0.0;
    if (a <= b)
      for (uint32_t row = 0; row < nrow; ++row) s += X[row * ld + a] * X[row * ld + b];
    part[e] = s;
  }
}

// G (column-major, symmetric) = sum_k part[k] (upper entries, fixed order).
__device__ void reduce_gram(const double* part, int nparts, uint64_t pld, uint32_t rowstride, uint32_t r,
                            double* G) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;
    const uint32_t a = min(i, j), b = max(i, j);
    const double* p = part + size_t(a) * rowstride + b;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < nparts; ++k) s += p[size_t(k) * pld];
    G[e] = s;
  }
  __syncthreads();
}

// out[row][c] = sum_k X[row][k] M[k + c*r]  (rows in smem, pitch ld)
__device__ void rows_mul(const double* X, uint32_t nrow, uint32_t r, uint32_t ld, const double* M,
                         double* out, uint32_t ldo) {
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    double s = 0.0;
    for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], M[k + c * r], s);
    out[row * ldo + c] = s;
  }
}

// ---- prep_step -------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) prep_step_kernel(PrepArgs a) {
  cg::grid_group grid = cg::this_grid();
  AlsCtrl* ctrl = a.ctrl;
  if (ctrl->stop) return;  // uniform: nobody writes stop before the first grid.sync
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1;
  double* X = sm;                        // [kRowsB][ld]
  double* M = X + kRowsB * ld;           // r*r
  double* W = M + r * r;                 // r*r (CTA 0 scratch)
  double* W2 = W + r * r;                // r*r
  const uint32_t i0 = blockIdx.x * kRowsB;
  const uint32_t nrow = i0 < a.I ? min(uint32_t(kRowsB), a.I - i0) : 0;

  // Phase 1: the CTA's rows of L, and their Gram partial
  if (a.from_partials) {
    for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) M[e] = a.GRinv[e];
    double* Y = W;  // reuse as [kRowsB][ld] only if it fits: use X for Y, compute into W2? keep simple:
    (void)Y;
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e / r, c = e % r;
      const double* p = a.part + size_t(i0 + row) * a.ldp + c;
      double s = 0.0;
#pragma unroll 4
      for (int k = 0; k < a.nparts; ++k) s += p[size_t(k) * a.I * a.ldp];
      X[row * ld + c] = s;
    }
    __syncthreads();
    // L rows = Y rows G_R^{-1}; written back over X through a register pass
    double vals[8];
    uint32_t cnt = 0;
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e / r, c = e % r;
      double s = 0.0;
      for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], M[k + c * r], s);
      vals[cnt++] = s;
    }
    __syncthreads();
    cnt = 0;
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e / r, c = e % r;
      X[row * ld + c] = vals[cnt];
      a.Lc[(i0 + row) + uint64_t(c) * a.I] = vals[cnt];
      ++cnt;
    }
  } else {
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e % nrow, c = e / nrow;
      X[row * ld + c] = a.Lc[(i0 + row) + uint64_t(c) * a.I];
    }
  }
  __syncthreads();
  rows_gram(X, nrow, r, ld, a.gpart + size_t(blockIdx.x) * r * r);
  grid.sync();

  // Phase 2 (CTA 0): G_L, Cholesky with the spd_solve floor, G_L^{-1}
  if (blockIdx.x == 0) {
    reduce_gram(a.gpart, gridDim.x, uint64_t(r) * r, r, r, M);
    double piv = 0.0;
    const int fail = chol_cta(M, W, r, 1e-13, &piv);
    if (fail) {
      if (threadIdx.x == 0) {
        ctrl->error = kAlsErrRightSingular;
        ctrl->pivot = piv;
        ctrl->stop = 1;
      }
    } else {
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.GL[e] = M[e];
      tri_inv_cta(W, W2, r);
      spd_inv_cta(W2, M, r);
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.GLinv[e] = M[e];
    }
  }
  grid.sync();
  if (ctrl->stop) return;

  // Phase 3: Mt rows = L rows G_L^{-1}, padded to ncp
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) M[e] = a.GLinv[e];
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < nrow * a.ncp; e += blockDim.x) {
    const uint32_t row = e / a.ncp, c = e % a.ncp;
    double s = 0.0;
    if (c < r)
      for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], M[k + c * r], s);
    a.Mt[uint64_t(i0 + row) * a.ncp + c] = s;
  }
}

// ---- finish_step -----------------------------------------------------------------
template <int NC>
__global__ void __launch_bounds__(kThreads) finish_step_kernel(FinishArgs a) {
  cg::grid_group grid = cg::this_grid();
  AlsCtrl* ctrl = a.ctrl;
  if (ctrl->stop) return;
  constexpr int kRows = 64, kLd = NC + 4, kNT = NC / 8, kTri = kNT * (kNT + 1) / 2;
  constexpr int kPer = (kTri + 7) / 8;
  extern __shared__ __align__(16) double sm[];
  double* tile = sm;  // [kRows][kLd]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  const uint32_t r = a.r;

  // Phase 1: Gram partial of the CTA's contiguous row range of R (row-major [F][ld])
  {
    double acc[kPer][2];
    int tm[kPer], tn[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      acc[k][0] = acc[k][1] = 0.0;
      int tt = warp + 8 * k, mt = 0;
      if (tt < kTri) {
        int rem = tt;
        while (rem >= kNT - mt) { rem -= kNT - mt; ++mt; }
        tm[k] = mt;
        tn[k] = mt + rem;
      } else {
        tm[k] = tn[k] = -1;
      }
    }
    const uint64_t nblk = (a.F + kRows - 1) / kRows;
    const uint64_t per = (nblk + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    for (uint64_t b = b0; b < b1; ++b) {
      __syncthreads();
      for (int e = threadIdx.x; e < kRows * (NC / 2); e += blockDim.x) {
        const int row = e / (NC / 2), c = (e % (NC / 2)) * 2;
        const uint64_t gr = b * kRows + row;
        double2 v = make_double2(0.0, 0.0);
        if (gr < a.F) v = *reinterpret_cast<const double2*>(a.R + gr * a.ld + c);
        tile[row * kLd + c] = v.x;
        tile[row * kLd + c + 1] = v.y;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        if (tm[k] < 0) continue;
#pragma unroll 8
        for (int k0 = 0; k0 < kRows; k0 += 4) {
          const double* rp = tile + (k0 + q) * kLd;
          dmma(acc[k][0], acc[k][1], rp[tm[k] * 8 + r8], rp[tn[k] * 8 + r8]);
        }
      }
    }
    double* out = a.gpart + size_t(blockIdx.x) * NC * NC;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (tm[k] < 0) continue;
      const int c1 = tm[k] * 8 + r8, c2 = tn[k] * 8 + 2 * q;
      out[c1 * NC + c2] = acc[k][0];
      out[c1 * NC + c2 + 1] = acc[k][1];
    }
  }
  grid.sync();
  if (blockIdx.x != 0) return;

  // Phase 2 (CTA 0): residual, stop rule, G_R^{-1}
  double* G = sm;
  double* L = G + r * r;
  double* Li = L + r * r;
  __syncthreads();
  reduce_gram(a.gpart, gridDim.x, uint64_t(NC) * NC, NC, r, G);
  __shared__ double hi_s[32], lo_s[32];
  if (threadIdx.x < 32) {
    double s = 0.0, c = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += 32) {
      const double p = a.GL[e] * G[e];
      const double pe = fma(a.GL[e], G[e], -p);
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
    if (it <= ctrl->history_cap) a.history[it - 1] = residual;
    ctrl->residual = residual;
    const double achieved = fabs(ctrl->prev - residual) / ctrl->norm;
    ctrl->achieved = achieved;
    int cont = 1;
    if (achieved <= ctrl->eta) {
      ctrl->status = 0;
      cont = 0;
    } else if (it >= ctrl->max_iters) {
      ctrl->status = 1;
      cont = 0;
    }
    ctrl->prev = residual;
    cont_s = cont;
    if (!cont) ctrl->stop = 1;
  }
  __syncthreads();
  if (!cont_s) return;
  double piv = 0.0;
  const int fail = chol_cta(G, L, r, 1e-13, &piv);
  if (fail) {
    if (threadIdx.x == 0) {
      ctrl->error = kAlsErrLeftSingular;
      ctrl->pivot = piv;
      ctrl->stop = 1;
    }
    return;
  }
  tri_inv_cta(L, Li, r);
  spd_inv_cta(Li, G, r);
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.GRinv[e] = G[e];
}

// ---- cholqr_step -------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) cholqr_step_kernel(CholQrArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1;
  double* X = sm;                 // [kRowsB][ld] rows of Y, then Q1
  double* M = X + kRowsB * ld;    // r*r
  double* W = M + r * r;          // r*r
  double* W2 = W + r * r;         // r*r
  double* X2 = W2 + r * r;        // [kRowsB][ld]
  __shared__ int fail_s;
  const uint32_t i0 = blockIdx.x * kRowsB;
  const uint32_t nrow = i0 < a.I ? min(uint32_t(kRowsB), a.I - i0) : 0;

  // Phase 1: rows of Y, Gram partial
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    double v;
    if (a.nparts > 0) {
      const double* p = a.Y + size_t(i0 + row) * a.ldp + c;
      v = 0.0;
#pragma unroll 4
      for (int k = 0; k < a.nparts; ++k) v += p[size_t(k) * a.I * a.ldp];
    } else {
      v = a.Y[(i0 + row) + uint64_t(c) * a.ldp];
    }
    X[row * ld + c] = v;
  }
  __syncthreads();
  rows_gram(X, nrow, r, ld, a.gpart + size_t(blockIdx.x) * r * r);
  grid.sync();
  // Phase 2 (CTA 0): chol (no floor), R1^{-1} = (L1^{-1})^T
  if (blockIdx.x == 0) {
    reduce_gram(a.gpart, gridDim.x, uint64_t(r) * r, r, r, M);
    const int fail = chol_cta(M, W, r, 0.0, nullptr);
    if (threadIdx.x == 0) a.work[0] = fail;  // shared with the other CTAs
    if (!fail) {
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.L1[e] = W[e];
      tri_inv_cta(W, W2, r);  // L1^{-1} (lower)
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.Rinv[e] = W2[e];
    }
  }
  grid.sync();
  if (threadIdx.x == 0) fail_s = int(a.work[0]);
  __syncthreads();
  if (!fail_s) {
    // Phase 3: Q1 rows = Y rows R1^{-1}: Q1[c] = sum_k Y[k] Linv[c + k*r] (R1^{-1} = Linv^T)
    for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
      const uint32_t i = e % r, j = e / r;
      M[i + j * r] = a.Rinv[j + i * r];  // M = Linv^T
    }
    __syncthreads();
    rows_mul(X, nrow, r, ld, M, X2, ld);
    __syncthreads();
    rows_gram(X2, nrow, r, ld, a.gpart + size_t(blockIdx.x) * r * r);
  }
  grid.sync();
  // Phase 4 (CTA 0): second factorization, R = R2 R1, degeneracy
  if (blockIdx.x == 0) {
    int fail = fail_s;
    if (!fail) {
      reduce_gram(a.gpart, gridDim.x, uint64_t(r) * r, r, r, M);
      fail = chol_cta(M, W, r, 0.0, nullptr);
    }
    if (!fail) {
      tri_inv_cta(W, W2, r);  // L2^{-1}
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.Rinv[e] = W2[e];
      // R = R2 R1 = L2^T L1^T
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
        const uint32_t i = e % r, j = e / r;
        double acc = 0.0;
        if (i <= j)
          for (uint32_t k = i; k <= j; ++k) acc += W[k + i * r] * a.L1[j + k * r];
        M[e] = acc;
        if (a.rmat) a.rmat[e] = acc;
      }
      __syncthreads();
      if (a.rt)
        for (uint32_t e = threadIdx.x; e < r * a.ldrt; e += blockDim.x) {
          const uint32_t row = e / a.ldrt, c = e % a.ldrt;
          a.rt[e] = c < r ? M[c + row * r] : 0.0;
        }
    }
    if (threadIdx.x == 0) {
      int bad = fail;
      if (!fail && a.check) {
        double md = 0.0;
        for (uint32_t i = 0; i < r; ++i) md = fmax(md, fabs(M[i + i * r]));
        for (uint32_t i = 0; i < r; ++i)
          if (fabs(M[i + i * r]) <= 1e-13 * md || md == 0.0) {
            bad = int(i) + 1;
            break;
          }
      }
      a.ctrl->degenerate_col = bad;
      a.work[1] = fail;
    }
  }
  grid.sync();
  if (a.work[1] != 0.0 || fail_s) return;
  // Phase 5: Q rows = Q1 rows R2^{-1}
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;
    M[i + j * r] = a.Rinv[j + i * r];
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    double s = 0.0;
    for (uint32_t k = 0; k < r; ++k) s = fma(X2[row * ld + k], M[k + c * r], s);
    a.Q[(i0 + row) + uint64_t(c) * a.I] = s;
  }
}

template <class K>
cudaError_t coop_launch(K kernel, int grid, size_t smem, void* args, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  void* params[] = {args};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kernel), dim3(grid), dim3(kThreads), params,
                                  smem, st);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

}  // namespace

int prep_step_grid(uint32_t I) { return int((I + kRowsB - 1) / kRowsB); }
int finish_step_grid(uint64_t F, int num_sms) {
  return int(std::max<uint64_t>(1, std::min<uint64_t>((F + 63) / 64, uint64_t(num_sms))));
}

cudaError_t launch_prep_step(PrepArgs a, cudaStream_t st) {
  const uint32_t r = a.r, ld = r + 1;
  const size_t smem = sizeof(double) * (kRowsB * ld + 3 * size_t(r) * r);
  return coop_launch(prep_step_kernel, prep_step_grid(a.I), smem, &a, st);
}

cudaError_t launch_finish_step(FinishArgs a, int num_sms, cudaStream_t st) {
  const int grid = finish_step_grid(a.F, num_sms);
  const uint32_t ncp = a.r <= 8 ? 8 : (a.r + 7) / 8 * 8;
  const size_t smem = sizeof(double) * std::max<size_t>(64 * (ncp + 4), 3 * size_t(a.r) * a.r);
  switch (ncp) {
#define TKG_F(N) \
  case N: return coop_launch(finish_step_kernel<N>, grid, smem, &a, st);
    TKG_F(8) TKG_F(16) TKG_F(24) TKG_F(32) TKG_F(40) TKG_F(48) TKG_F(56) TKG_F(64)
#undef TKG_F
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_cholqr_step(CholQrArgs a, cudaStream_t st) {
  const uint32_t r = a.r, ld = r + 1;
  const size_t smem = sizeof(double) * (2 * kRowsB * ld + 3 * size_t(r) * r);
  return coop_launch(cholqr_step_kernel, prep_step_grid(a.I), smem, &a, st);
}

}  // namespace tkg
