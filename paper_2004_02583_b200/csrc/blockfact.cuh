// Blocked r x r factorizations on one CTA (256 threads) for the small steps
// of coop.cu, r up to 64: right-looking Cholesky in 8-column blocks (one warp
// factors the diagonal block, every thread solves panel rows, the trailing
// update runs on DMMA), the inverse of the triangular factor (one warp per
// block column: diagonal-block inverse, then a block forward substitution on
// DMMA), and G^{-1} = L^{-T} L^{-1} on DMMA. The register-resident
// right-looking kernels of coop.cu spend one CTA barrier and a dependent
// fp64 reciprocal per column (0.6 us per step at r = 50); here the
// per-column chains are 8 long and the rest is tensor-core work.
//
// Matrices live in shared memory, column-major with leading dimension
// blk_ld(r) = rp + 4 (rp = r rounded up to 8; 4 mod 16 doubles: conflict-free
// DMMA fragment loads), the padding rows / columns holding the identity.
// Pivot test of spd_solve (kernels.cpp:378-393): pivot (the Schur complement
// diagonal before the square root) <= floor_abs or not > 0 fails.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tkg {

__host__ __device__ constexpr int blk_rp(int r) { return (r + 7) / 8 * 8; }
__host__ __device__ constexpr int blk_ld(int r) { return blk_rp(r) + 4; }
// doubles of scratch a blocked inverse needs: W, X and 8 8x8 staging tiles
__host__ __device__ constexpr int blk_scratch(int r) { return 2 * blk_rp(r) * blk_ld(r) + 8 * 64 + blk_rp(r); }

#ifdef __CUDACC__

// W (rp x ld) <- G (r x r, column-major, leading dimension r) padded with I.
__device__ inline void blk_load(const double* G, uint32_t r, double* W) {
  const int rp = blk_rp(int(r)), ld = blk_ld(int(r));
  for (int e = threadIdx.x; e < rp * rp; e += blockDim.x) {
    const int i = e % rp, j = e / rp;
    W[i + j * ld] = (i < int(r) && j < int(r)) ? G[i + j * int(r)] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
}

// In place: W's lower triangle <- L with G = L L^T; dinv[j] = 1 / L_jj
// (rp doubles, shared). Returns the failing column (1-based, < r) or 0;
// *piv_out = the failing pivot. The diagonal block is factored in registers
// of warp 0 (lane i < 8 holds row i; pivots broadcast by shuffles, 1/sqrt by
// rsqrt: no division on the dependent chain), panel rows use dinv.
__device__ inline int blk_chol(double* W, uint32_t r, double floor_abs, double* piv_out, double* dinv) {
  __shared__ int fail_s;
  __shared__ double piv_s;
  const int rp = blk_rp(int(r)), ld = blk_ld(int(r)), nb = rp / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  if (threadIdx.x == 0) fail_s = 0;
  __syncthreads();
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = 8 * kb;
    if (warp == 0) {
      const int i = lane & 7;  // lanes 8..31 mirror lanes 0..7 (shuffles stay full-warp)
      double a[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = c <= i ? W[(k0 + i) + (k0 + c) * ld] : 0.0;
      int fail = 0;
      double fpiv = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double d = __shfl_sync(0xffffffffu, a[j], j);  // pivot (Schur complement diagonal)
        if (!fail && k0 + j < int(r) && (!(d > floor_abs) || !(d > 0.0))) {
          fail = k0 + j + 1;
          fpiv = d;
        }
        const double inv = fail ? 0.0 : rsqrt(d);
        if (lane == j) dinv[k0 + j] = inv;
        if (i == j) a[j] = d * inv;       // L_jj = sqrt(d)
        else if (i > j) a[j] *= inv;      // L_ij
        const double lij = a[j];
#pragma unroll
        for (int c = j + 1; c < 8; ++c) {
          const double lcj = __shfl_sync(0xffffffffu, a[j], c);  // L_cj
          if (i >= c) a[c] = fma(-lij, lcj, a[c]);
        }
      }
      if (lane < 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c <= i) W[(k0 + i) + (k0 + c) * ld] = a[c];
      }
      if (lane == 0 && fail) {
        fail_s = fail;
        piv_s = fpiv;
      }
    }
    __syncthreads();
    if (fail_s) break;
    // panel rows below the block: x L11^T = a (forward substitution)
    for (int i = k0 + 8 + int(threadIdx.x); i < rp; i += blockDim.x) {
      double x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double s = W[i + (k0 + j) * ld];
#pragma unroll
        for (int m = 0; m < j; ++m) s = fma(-x[m], W[(k0 + j) + (k0 + m) * ld], s);
        x[j] = s * dinv[k0 + j];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) W[i + (k0 + j) * ld] = x[j];
    }
    __syncthreads();
    // trailing update of the lower tiles (bi >= bj > kb): A22 -= L21 L21^T
    const int nt = nb - kb - 1, ntiles = nt * (nt + 1) / 2;
    for (int t = warp; t < ntiles; t += int(blockDim.x >> 5)) {
      int bi = 0, rem = t;
      while (rem > bi) {
        rem -= bi + 1;
        ++bi;
      }
      const int bj = rem;  // 0 <= bj <= bi < nt
      const int ri = k0 + 8 + 8 * bi, rj = k0 + 8 + 8 * bj;
      double* d = W + (ri + r8) + (rj + 2 * q) * ld;
      double d0 = d[0], d1 = d[ld];
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const double a = -W[(ri + r8) + (k0 + kk + q) * ld];
        const double b = W[(rj + r8) + (k0 + kk + q) * ld];
        dmma(d0, d1, a, b);
      }
      d[0] = d0;
      d[ld] = d1;
    }
    __syncthreads();
  }
  const int f = fail_s;
  if (f && piv_out && threadIdx.x == 0) *piv_out = piv_s;
  __syncthreads();
  return f;
}

// X (rp x ld) <- L^{-1} (lower) from the factor in W's lower triangle.
// T: 8 x 64 doubles of staging (one 8x8 tile per warp).
__device__ inline void blk_trinv(const double* W, uint32_t r, double* X, double* T, const double* dinv) {
  const int rp = blk_rp(int(r)), ld = blk_ld(int(r)), nb = rp / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  for (int e = threadIdx.x; e < rp * rp; e += blockDim.x) {
    const int i = e % rp, j = e / rp;
    X[i + j * ld] = 0.0;
  }
  __syncthreads();
  // diagonal blocks: lane c < 8 of warp w solves column c of L_ww^{-1}
  if (warp < nb && lane < 8) {
    const int k0 = 8 * warp, c = lane;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = i == c ? 1.0 : 0.0;
#pragma unroll
      for (int m = 0; m < i; ++m) s = fma(-W[(k0 + i) + (k0 + m) * ld], x[m], s);
      x[i] = i < c ? 0.0 : s * dinv[k0 + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) X[(k0 + i) + (k0 + c) * ld] = x[i];
  }
  __syncthreads();
  // block column jb = warp: X_ib,jb = -D_ib (sum_{kb=jb}^{ib-1} L_ib,kb X_kb,jb), ib ascending
  if (warp < nb) {
    const int jb = warp, cj = 8 * jb;
    double* tw = T + warp * 64;
    for (int ib = jb + 1; ib < nb; ++ib) {
      const int ri = 8 * ib;
      double s0 = 0.0, s1 = 0.0;
      for (int kb = jb; kb < ib; ++kb)
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          const double a = W[(ri + r8) + (8 * kb + kk + q) * ld];   // L[ri + m][8kb + k]
          const double b = X[(8 * kb + kk + q) + (cj + r8) * ld];   // X[8kb + k][cj + n]
          dmma(s0, s1, a, b);
        }
      // stage the sum (row r8, columns 2q, 2q+1), then multiply by -D_ib
      tw[r8 * 8 + 2 * q] = s0;
      tw[r8 * 8 + 2 * q + 1] = s1;
      __syncwarp();
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const double a = -X[(ri + r8) + (ri + kk + q) * ld];  // -D_ib[m][k]
        const double b = tw[(kk + q) * 8 + r8];                 // S[k][n]
        dmma(o0, o1, a, b);
      }
      X[(ri + r8) + (cj + 2 * q) * ld] = o0;
      X[(ri + r8) + (cj + 2 * q + 1) * ld] = o1;
      __syncwarp();
    }
  }
  __syncthreads();
}

// out (r x r, column-major, leading dimension r) <- X^T X (symmetric), X
// lower triangular (rp x ld).
__device__ inline void blk_xtx(const double* X, uint32_t r, double* out) {
  const int rp = blk_rp(int(r)), ld = blk_ld(int(r)), nb = rp / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  const int ntiles = nb * (nb + 1) / 2;
  for (int t = warp; t < ntiles; t += int(blockDim.x >> 5)) {
    int bi = 0, rem = t;
    while (rem > bi) {
      rem -= bi + 1;
      ++bi;
    }
    const int bj = rem;  // bi >= bj
    double d0 = 0.0, d1 = 0.0;
    for (int kb = bi; kb < nb; ++kb)  // X[k][i] vanishes for k < i
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const double a = X[(8 * kb + kk + q) + (8 * bi + r8) * ld];  // (X^T)[i][k]
        const double b = X[(8 * kb + kk + q) + (8 * bj + r8) * ld];  // X[k][j]
        dmma(d0, d1, a, b);
      }
    const int i = 8 * bi + r8, j0 = 8 * bj + 2 * q;
    const double v[2] = {d0, d1};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = j0 + u;
      if (i < int(r) && j < int(r)) {
        out[i + j * int(r)] = v[u];
        out[j + i * int(r)] = v[u];
      }
    }
  }
  __syncthreads();
}

// G^{-1} (out, r x r column-major) of the SPD matrix G (r x r column-major)
// through L L^T with spd_solve's pivot floor (floor_rel * max diag G).
// Returns the failing column (1-based) or 0. scratch: blk_scratch(r) doubles.
__device__ inline int blk_spd_inverse(const double* G, double* out, uint32_t r, double floor_rel, double* piv_out,
                                      double* scratch) {
  double md = 0.0;
  for (uint32_t i = 0; i < r; ++i) md = fmax(md, G[i + i * r]);
  double* W = scratch;
  double* X = W + blk_rp(int(r)) * blk_ld(int(r));
  double* T = X + blk_rp(int(r)) * blk_ld(int(r));
  double* dinv = T + 8 * 64;
  blk_load(G, r, W);
  const int fail = blk_chol(W, r, floor_rel * md, piv_out, dinv);
  if (fail) return fail;
  blk_trinv(W, r, X, T, dinv);
  blk_xtx(X, r, out);
  return 0;
}

#endif  // __CUDACC__

}  // namespace tkg
