// Small dense kernels outside the ALS sweep (the sweep's own small steps are
// in coop.cu): Gram partials + Cholesky with the reference's pivot floor
// (gram / spd_solve primitives), Householder QR with the reference's sign
// convention (reduced_qr primitive), fixed-order sums, sums of squares, the
// st-HOSVD shrink, and operand packing.
#include <algorithm>
#include <cmath>

#include "kernels.cuh"

namespace tkg {

namespace {

constexpr int kGramRows = 128;

// ---- Gram partials ---------------------------------------------------------
__global__ void gram_partials_kernel(const double* __restrict__ X, uint64_t ld, uint32_t rows,
                                     uint32_t r, double* __restrict__ part) {
  extern __shared__ double tile[];  // [kGramRows][r]
  const uint32_t r0 = blockIdx.x * kGramRows;
  const uint32_t nr = min(uint32_t(kGramRows), rows - r0);
  for (uint32_t e = threadIdx.x; e < nr * r; e += blockDim.x) {
    const uint32_t row = e % nr, c = e / nr;
    tile[row * r + c] = X[(r0 + row) + uint64_t(c) * ld];
  }
  __syncthreads();
  double* out = part + size_t(blockIdx.x) * r * r;
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t c1 = e % r, c2 = e / r;
    double s = 0.0;
    if (c1 <= c2)
      for (uint32_t row = 0; row < nr; ++row) s += tile[row * r + c1] * tile[row * r + c2];
    out[c1 * r + c2] = s;  // row-major upper triangle: entry (c1, c2), c1 <= c2
  }
}

// ---- Cholesky (spd_solve's factorisation, kernels.cpp:369-393) -------------
// Single CTA. G(i,j) for i <= j = sum_k part[k][i*rowstride + j].
__device__ void block_chol(double* G, double* L, uint32_t r, int32_t* flag, DevStatus* status,
                           double floor_rel = 1e-13) {
  __shared__ double piv_s;
  __shared__ int fail_s;
  // max diagonal (kernels.cpp:378-379) and floor
  __shared__ double floor_s;
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
        fail_s = 1;
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
  if (threadIdx.x == 0) {
    *flag = fail_s ? 1 : 0;
    if (fail_s && status) status->pivot = piv_s;
  }
}

__device__ void reduce_upper(const double* part, int nparts, uint64_t part_ld, int rowstride,
                             uint32_t r, double* G) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;  // column-major entry (i, j)
    const uint32_t a = min(i, j), b = max(i, j);
    double s = 0.0;
    const double* p = part + size_t(a) * rowstride + b;
#pragma unroll 8
    for (int k = 0; k < nparts; ++k) s += p[size_t(k) * part_ld];
    G[e] = s;
  }
}

__global__ void chol_kernel(const double* __restrict__ part, int nparts, uint64_t part_ld,
                            int rowstride, uint32_t r, double* G, double* chol, int32_t* flag,
                            DevStatus* status, double floor_rel) {
  extern __shared__ double sm[];
  double* Gs = sm;
  double* Ls = sm + r * r;
  reduce_upper(part, nparts, part_ld, rowstride, r, Gs);
  __syncthreads();
  block_chol(Gs, Ls, r, flag, status, floor_rel);
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    if (G) G[e] = Gs[e];
    chol[e] = Ls[e];
  }
}

// ---- Householder QR (kernels.cpp:303-367) ----------------------------------
__device__ double block_sum(double v, double* red) {
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

__global__ void __launch_bounds__(1024) qr_kernel(const double* __restrict__ Y, int nparts,
                                                  uint64_t ldy, uint32_t m, uint32_t n, double* q,
                                                  double* rmat, double* rt, uint32_t ldrt,
                                                  double* work, int check_degenerate,
                                                  DevStatus* status, const int32_t* only_if,
                                                  int32_t* degen_out) {
  if (only_if && *only_if == 0) return;  // fallback mode: the fast path found nothing to redo
  __shared__ double red[32];
  __shared__ double dots[64];
  __shared__ double betas[64];
  double* w = work;            // m x n
  double* V = work + size_t(m) * n;  // m x n (column k holds v_k in rows k..m-1)
  const int tid = threadIdx.x, T = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = T / 32;
  for (size_t e = tid; e < size_t(m) * n; e += T) {
    const uint32_t i = e % m, c = e / m;
    double b;
    if (nparts > 0) {
      b = 0.0;
      for (int k = 0; k < nparts; ++k) b += Y[(size_t(k) * m + i) * ldy + c];
    } else {
      b = Y[i + uint64_t(c) * ldy];
    }
    w[e] = b;
    V[e] = 0.0;
  }
  __syncthreads();
  for (uint32_t k = 0; k < n; ++k) {
    double part = 0.0;
    for (uint32_t i = k + tid; i < m; i += T) part += w[i + size_t(k) * m] * w[i + size_t(k) * m];
    const double xnorm = sqrt(block_sum(part, red));
    if (xnorm == 0.0) {
      if (tid == 0) betas[k] = 0.0;
      __syncthreads();
      continue;
    }
    const double v0 = w[k + size_t(k) * m];
    const double alpha = v0 >= 0.0 ? -xnorm : xnorm;
    for (uint32_t i = k + tid; i < m; i += T)
      V[i + size_t(k) * m] = (i == k) ? v0 - alpha : w[i + size_t(k) * m];
    __syncthreads();
    part = 0.0;
    for (uint32_t i = k + tid; i < m; i += T) part += V[i + size_t(k) * m] * V[i + size_t(k) * m];
    const double beta = 2.0 / block_sum(part, red);
    // dots for columns j = k..n-1 (one warp per column)
    for (uint32_t j = k + warp; j < n; j += nwarps) {
      double d = 0.0;
      for (uint32_t i = k + lane; i < m; i += 32) d += V[i + size_t(k) * m] * w[i + size_t(j) * m];
      for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      if (lane == 0) dots[j] = d;
    }
    __syncthreads();
    for (size_t e = tid; e < size_t(m - k) * (n - k); e += T) {
      const uint32_t i = k + e % (m - k), j = k + e / (m - k);
      w[i + size_t(j) * m] -= beta * dots[j] * V[i + size_t(k) * m];
    }
    __syncthreads();
    if (tid == 0) {
      w[k + size_t(k) * m] = alpha;
      betas[k] = beta;
    }
    __syncthreads();
  }
  // R (upper of w) and the sign convention R_kk >= 0 (kernels.cpp:361-365).
  __shared__ double sgn[64];
  if (tid < int(n)) sgn[tid] = w[tid + size_t(tid) * m] >= 0.0 ? 1.0 : -1.0;
  __syncthreads();
  for (uint32_t e = tid; e < n * n; e += T) {
    const uint32_t i = e % n, j = e / n;
    const double v = (i <= j) ? sgn[i] * w[i + size_t(j) * m] : 0.0;
    if (rmat) rmat[e] = v;
    if (rt) rt[size_t(j) * ldrt + i] = v;  // rt[c'][c] = R[c][c'] -> row c' = j
  }
  if (rt)
    for (uint32_t e = tid; e < n * (ldrt - n); e += T) {
      const uint32_t row = e / (ldrt - n), c = n + e % (ldrt - n);
      rt[size_t(row) * ldrt + c] = 0.0;
    }
  // Thin Q: reflections applied in reverse to the leading identity columns.
  for (size_t e = tid; e < size_t(m) * n; e += T) {
    const uint32_t i = e % m, c = e / m;
    q[e] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (uint32_t k = n; k-- > 0;) {
    if (betas[k] == 0.0) continue;
    for (uint32_t j = k + warp; j < n; j += nwarps) {
      double d = 0.0;
      for (uint32_t i = k + lane; i < m; i += 32) d += V[i + size_t(k) * m] * q[i + size_t(j) * m];
      for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      if (lane == 0) dots[j] = d;
    }
    __syncthreads();
    for (size_t e = tid; e < size_t(m - k) * (n - k); e += T) {
      const uint32_t i = k + e % (m - k), j = k + e / (m - k);
      q[i + size_t(j) * m] -= betas[k] * dots[j] * V[i + size_t(k) * m];
    }
    __syncthreads();
  }
  for (size_t e = tid; e < size_t(m) * n; e += T) {
    const uint32_t c = e / m;
    q[e] *= sgn[c];
  }
  if (check_degenerate && tid == 0) {
    // als.cpp:74-86
    double md = 0.0;
    for (uint32_t i = 0; i < n; ++i) md = fmax(md, fabs(w[i + size_t(i) * m]));
    int bad = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (fabs(w[i + size_t(i) * m]) <= 1e-13 * md || md == 0.0) {
        bad = int(i) + 1;
        break;
      }
    }
    if (status) status->degenerate_col = bad;
    if (degen_out) *degen_out = bad;
  }
}

__global__ void sum_kernel(const double* __restrict__ p, int n, double* dst) {
  __shared__ double red[32];
  // fixed-shape tree: thread t sums p[t], p[t+T], ... then a fixed warp tree
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += p[k];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *dst = s;
}

__global__ void pack_kernel(const double* __restrict__ src, uint64_t rs, uint64_t cs, uint32_t rows,
                            uint32_t cols, double* dst, uint32_t ldd) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e >= uint64_t(rows) * ldd) return;
  const uint32_t row = e / ldd, col = e % ldd;
  dst[e] = col < cols ? src[row * rs + col * cs] : 0.0;
}

constexpr int kSqBlock = 256;
constexpr uint64_t kSqPerBlock = 1u << 20;

__global__ void sumsq_kernel(const double* __restrict__ x, uint64_t n, double* part) {
  __shared__ double red[32];
  const uint64_t lo = blockIdx.x * kSqPerBlock;
  const uint64_t hi = min(n, lo + kSqPerBlock);
  double s = 0.0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s = fma(x[i], x[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void reduce_partials_kernel(const double* __restrict__ part, int nparts, uint32_t rows,
                                       uint32_t ldp, uint32_t r, double* y) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e >= uint64_t(rows) * r) return;
  const uint32_t i = e % rows, c = e / rows;
  double s = 0.0;
  for (int k = 0; k < nparts; ++k) s += part[(size_t(k) * rows + i) * ldp + c];
  y[e] = s;
}

__global__ void sumsq_diff_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  uint64_t n, double* part) {
  __shared__ double red[32];
  const uint64_t lo = blockIdx.x * kSqPerBlock;
  const uint64_t hi = min(n, lo + kSqPerBlock);
  double s = 0.0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double d = b[i] - a[i];
    s = fma(d, d, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---- st-HOSVD shrink ---------------------------------------------------------
// working <- tensorize(R_hat R^T) (hosvd.cpp:176-178): out(jl, c, p) =
// sum_k R[j][k] R_hat(c, k) for every fiber j = jl + p*s, i.e. a tall-skinny
// F x r x r product. A persistent CTA walks 128-fiber tiles of R (row-major
// [F][ld], one contiguous block): the next tile streams into the second
// buffer with cp.async while the current one runs DMMA against R_hat^T held
// in shared memory; the r x 128 result is staged in the current buffer and
// each output column (or, for s = 1, the tile's contiguous fiber-major
// block) written as coalesced runs; ||out||^2 per CTA.
constexpr int kShrinkThreads = 256;
constexpr int kShrinkTile = 64;              // two CTAs per SM overlap each other's phases
constexpr int kShrinkMT = kShrinkTile / 64;  // 8-fiber row tiles per warp

// UPPER: R_hat is upper triangular (the QR factor of the st-HOSVD drivers), so
// k-step t (rows 4t .. 4t+3 of R_hat^T) reaches only the column tiles n with
// 8n <= 4t + 3: 56 of the 98 DMMAs per row tile at 56 columns.
template <int NC, bool UPPER>
__global__ void __launch_bounds__(kShrinkThreads, 2) shrink_kernel(
    const double* __restrict__ R, uint64_t ld, uint64_t s, uint64_t P, uint32_t r,
    const double* __restrict__ rhat, double* __restrict__ out, double* sumsq_part) {
  constexpr int kLd = NC + 4;            // fragment rows 4 (mod 16) apart
  constexpr int kLdO = kShrinkTile + 4;
  constexpr int kBuf = kShrinkTile * kLd;
  constexpr int kChunks = NC / 2;        // 16-byte chunks per row
  extern __shared__ __align__(16) double sm[];
  double* Bs = sm;                       // [NC][kLd]: Bs[k][c] = R_hat(c, k)
  double* Rb = sm + NC * kLd;            // 2 x [128][kLd]; the current one becomes Os
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  for (int e = threadIdx.x; e < NC * NC; e += blockDim.x) {
    const int k = e / NC, c = e % NC;
    Bs[k * kLd + c] = (k < int(r) && c < int(r)) ? rhat[c + k * r] : 0.0;
  }
  const uint64_t F = s * P;
  const uint64_t ntiles = (F + kShrinkTile - 1) / kShrinkTile;
  auto issue = [&](uint64_t tile, double* buf) {
    const uint64_t j0 = tile * kShrinkTile;
    const int nf = int(F - j0 < uint64_t(kShrinkTile) ? F - j0 : uint64_t(kShrinkTile));
    for (int e = threadIdx.x; e < nf * kChunks; e += blockDim.x) {
      const int row = e / kChunks, c = (e % kChunks) * 2;
      cp_async16(buf + row * kLd + c, R + (j0 + row) * ld + c);
    }
  };
  double sq = 0.0;
  uint64_t tile = blockIdx.x;
  if (tile < ntiles) issue(tile, Rb);
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double* cur = Rb + (it & 1) * kBuf;
    const uint64_t nxt = tile + gridDim.x;
    __syncthreads();  // the previous tile's readers of the other buffer (its Os) are done
    if (nxt < ntiles) issue(nxt, Rb + ((it + 1) & 1) * kBuf);
    cp_async_commit();
    cp_async_wait<1>();
    const uint64_t j0 = tile * kShrinkTile;
    const int nf = int(F - j0 < uint64_t(kShrinkTile) ? F - j0 : uint64_t(kShrinkTile));
    __syncthreads();  // the current tile landed for every thread
    // R's padding columns (never written by the contraction kernels) and the
    // rows past F are zero for the product
    const int npad = NC - int(r);
    for (int e = threadIdx.x; e < kShrinkTile * npad; e += blockDim.x) {
      const int row = e / npad, c = int(r) + e % npad;
      cur[row * kLd + c] = 0.0;
    }
    if (nf < kShrinkTile) {
      for (int e = threadIdx.x; e < (kShrinkTile - nf) * int(r); e += blockDim.x) {
        const int row = nf + e / int(r), c = e % int(r);
        cur[row * kLd + c] = 0.0;
      }
    }
    __syncthreads();
    double acc[kShrinkMT][NC / 8][2];
#pragma unroll
    for (int m = 0; m < kShrinkMT; ++m)
#pragma unroll
      for (int n = 0; n < NC / 8; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll
    for (int t = 0; t < NC / 4; ++t) {
      const int kk = 4 * t + q;
      double af[kShrinkMT], bf[NC / 8];
#pragma unroll
      for (int m = 0; m < kShrinkMT; ++m) af[m] = cur[(warp * 8 * kShrinkMT + m * 8 + r8) * kLd + kk];
#pragma unroll
      for (int n = 0; n < NC / 8; ++n)
        if (!UPPER || 8 * n <= 4 * t + 3) bf[n] = Bs[kk * kLd + n * 8 + r8];
#pragma unroll
      for (int n = 0; n < NC / 8; ++n)
        if (!UPPER || 8 * n <= 4 * t + 3) {
#pragma unroll
          for (int m = 0; m < kShrinkMT; ++m) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
        }
    }
    __syncthreads();  // the current buffer becomes the staging buffer Os
    double* Os = cur;
#pragma unroll
    for (int m = 0; m < kShrinkMT; ++m)
#pragma unroll
      for (int n = 0; n < NC / 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int f = warp * 8 * kShrinkMT + m * 8 + r8, c = n * 8 + 2 * q + e;
          Os[s == 1 ? f * (NC + 1) + c : c * kLdO + f] = acc[m][n][e];
        }
    __syncthreads();
    if (s == 1) {  // mode-1 output: the tile's fibers are one contiguous block of nf * r values
      double* o = out + j0 * r;
      for (int e = threadIdx.x; e < int(r) * nf; e += blockDim.x) {
        const int f = e / int(r), c = e - f * int(r);
        const double v = Os[f * (NC + 1) + c];  // fiber-major staging: conflict-free reads
        o[e] = v;
        sq = fma(v, v, sq);
      }
    } else {
      for (int e = threadIdx.x; e < int(r) * kShrinkTile; e += blockDim.x) {
        const int c = e / kShrinkTile, f = e % kShrinkTile;
        if (f >= nf) continue;
        const uint64_t j = j0 + f, p = j / s, jl = j - p * s;
        const double v = Os[c * kLdO + f];
        out[jl + uint64_t(c) * s + p * s * r] = v;
        sq = fma(v, v, sq);
      }
    }
  }
  cp_async_wait<0>();
  sq = block_sum(sq, red);
  if (threadIdx.x == 0) sumsq_part[blockIdx.x] = sq;
}

// R = R2 R1 with R_k = L_k^T (CholQR2), the reference's degeneracy test on
// diag(R) (als.cpp:74-86), and optional outputs R (col-major) / R^T padded.

// ---- recover_singular_vectors (hosvd.cpp:65-72) ----------------------------------
// The left singular vectors of q^T A_(n) are the eigenvectors of its Gram
// matrix G = (A_(n)^T q)^T (A_(n)^T q) (r x r). One CTA runs the cyclic
// parallel Jacobi method on G in shared memory: each round rotates the r/2
// disjoint pairs of a round-robin tournament (player 0 fixed, the others
// rotating), rows first, then columns and the accumulated V; a sweep is
// r-1 rounds (r padded to even), repeated until a sweep finds every
// off-diagonal entry negligible. The columns are then ordered by descending
// eigenvalue (svd_tall's stable sort of the singular values,
// kernels.cpp:273-301) and signed so that each column's largest-magnitude
// entry (the first on ties) is positive (fix_column_signs, kernels.cpp:25-43,
// applied to the left vectors of q^T A_(n) by dense_svd, kernels.cpp:419-427).
constexpr int kEigMax = 64;
constexpr int kEigLd = kEigMax + 1;
constexpr int kEigThreads = 256;

__device__ __forceinline__ void eig_pair(int round, int k, int m, int& p, int& q) {
  if (k == 0) {
    p = 0;
    q = 1 + round;
  } else {
    p = 1 + (round + k) % (m - 1);
    q = 1 + (round - k + (m - 1)) % (m - 1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

__global__ void __launch_bounds__(kEigThreads) sym_eig_kernel(const double* __restrict__ G, uint32_t r,
                                                              double* __restrict__ vt,
                                                              double* __restrict__ evals) {
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                       // [m][kEigLd]
  double* V = sm + kEigMax * kEigLd;    // [m][kEigLd], V(i, c) at V[i*kEigLd + c]
  __shared__ double cs[kEigMax / 2], sn[kEigMax / 2];
  __shared__ int perm[kEigMax];
  __shared__ double sgn[kEigMax];
  __shared__ int rotated;
  const int n = int(r), m = (n + 1) & ~1, half = m / 2, tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    A[i * kEigLd + j] = (i < n && j < n) ? G[i + size_t(j) * r] : 0.0;
    V[i * kEigLd + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round) {
      if (tid < half) {
        int p, q;
        eig_pair(round, tid, m, p, q);
        double c = 1.0, s = 0.0;
        const double apq = A[p * kEigLd + q];
        if (q < n) {
          const double app = A[p * kEigLd + p], aqq = A[q * kEigLd + q];
          // negligible against the diagonal: the classical Jacobi threshold
          if (fabs(apq) > 1e-300 && fabs(apq) > 0x1.0p-60 * sqrt(fabs(app) * fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            rotated = 1;
          }
        }
        cs[tid] = c;
        sn[tid] = s;
      }
      __syncthreads();
      // rows: A <- J^T A (rows p, q of each pair)
      for (int e = tid; e < half * m; e += blockDim.x) {
        const int k = e / m, j = e % m;
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        int p, q;
        eig_pair(round, k, m, p, q);
        const double x = A[p * kEigLd + j], y = A[q * kEigLd + j];
        A[p * kEigLd + j] = c * x - s * y;
        A[q * kEigLd + j] = s * x + c * y;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int e = tid; e < half * m; e += blockDim.x) {
        const int k = e / m, i = e % m;
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        int p, q;
        eig_pair(round, k, m, p, q);
        const double x = A[i * kEigLd + p], y = A[i * kEigLd + q];
        A[i * kEigLd + p] = c * x - s * y;
        A[i * kEigLd + q] = s * x + c * y;
        const double vx = V[i * kEigLd + p], vy = V[i * kEigLd + q];
        V[i * kEigLd + p] = c * vx - s * vy;
        V[i * kEigLd + q] = s * vx + c * vy;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (tid == 0) {  // stable descending order of the eigenvalues
    for (int c = 0; c < n; ++c) perm[c] = c;
    for (int c = 1; c < n; ++c) {
      const int x = perm[c];
      const double vx = A[x * kEigLd + x];
      int k = c;
      while (k > 0 && A[perm[k - 1] * kEigLd + perm[k - 1]] < vx) {
        perm[k] = perm[k - 1];
        --k;
      }
      perm[k] = x;
    }
  }
  __syncthreads();
  if (tid < n) {
    const int col = perm[tid];
    int arg = 0;
    double best = 0.0;
    for (int i = 0; i < n; ++i) {
      const double mag = fabs(V[i * kEigLd + col]);
      if (mag > best) {
        best = mag;
        arg = i;
      }
    }
    sgn[tid] = V[arg * kEigLd + col] >= 0.0 ? 1.0 : -1.0;
    if (evals) evals[tid] = A[col * kEigLd + col];
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int c = e % n, i = e / n;  // vt(c, i) = V(i, perm[c]) * sign
    vt[c + size_t(i) * r] = sgn[c] * V[i * kEigLd + perm[c]];
  }
}


// ---- sharded-decomposition helpers -------------------------------------------------
__global__ void add_kernel(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

// part[0][i][c] = sum_k part[k][i][c] (c < r), in place; 8 lanes per entry,
// each over k = sub, sub + 8, ... in order, then a fixed xor tree.
__global__ void reduce_slot0_kernel(double* __restrict__ part, int nparts, uint32_t I, uint32_t ldp, uint32_t r) {
  const uint64_t n = uint64_t(I) * r;
  const uint64_t e = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 8;
  const int sub = threadIdx.x & 7;
  const bool act = e < n;
  double s = 0.0;
  double* p = nullptr;
  if (act) {
    p = part + (e / r) * ldp + (e % r);
    const uint64_t stride = uint64_t(I) * ldp;
    for (int k = sub; k < nparts; k += 8) s += p[size_t(k) * stride];
  }
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (act && sub == 0) p[0] = s;
}

// G (column-major r x r, symmetric) = sum_k part[k*pld + a*rs + b], a <= b;
// one warp per entry (lanes over k, fixed xor tree).
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nparts, uint64_t pld, uint32_t rs,
                                   uint32_t r, double* __restrict__ G) {
  const uint32_t t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (t >= r * (r + 1) / 2) return;
  uint32_t a = 0, rem = t;
  while (rem >= r - a) {
    rem -= r - a;
    ++a;
  }
  const uint32_t b = a + rem;
  const double* p = part + size_t(a) * rs + b;
  double s = 0.0;
  for (int k = int(lane); k < nparts; k += 32) s += p[size_t(k) * pld];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) {
    G[a + b * r] = s;
    G[b + a * r] = s;
  }
}

// N-d box copy between column-major tensors (strides in elements).
__global__ void copy_box_kernel(const double* __restrict__ src, double* __restrict__ dst, BoxCopy b,
                                uint64_t total) {
  for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t rem = idx, so = b.src_base, dof = b.dst_base;
    for (int k = 0; k < b.N; ++k) {
      const uint64_t c = rem % b.box[k];
      rem /= b.box[k];
      so += c * b.src_stride[k];
      dof += c * b.dst_stride[k];
    }
    dst[dof] = src[so];
  }
}

}  // namespace

int shrink_count(uint64_t F) {
  const uint64_t tiles = (F + kShrinkTile - 1) / kShrinkTile;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, 2 * 148)));
}

cudaError_t launch_shrink(const double* R, uint64_t ld, uint64_t s, uint64_t P, uint32_t r,
                          const double* rhat, double* out, double* sumsq_part, cudaStream_t st,
                          bool rhat_upper) {
  const int grid = shrink_count(s * P);
  const uint32_t nc = r <= 8 ? 8 : (r + 7) / 8 * 8;
#define TKG_S(N)                                                                                    \
  if (nc == N) {                                                                                    \
    const size_t smem = sizeof(double) * (2 * size_t(kShrinkTile) * (N + 4) + size_t(N) * (N + 4)); \
    auto k = rhat_upper ? shrink_kernel<N, true> : shrink_kernel<N, false>;                         \
    cudaError_t e = raise_smem_limit(k, smem);                                                      \
    if (e != cudaSuccess) return e;                                                                 \
    k<<<grid, kShrinkThreads, smem, st>>>(R, ld, s, P, r, rhat, out, sumsq_part);                   \
    return cudaGetLastError();                                                                      \
  }
  TKG_S(8) TKG_S(16) TKG_S(24) TKG_S(32) TKG_S(40) TKG_S(48) TKG_S(56) TKG_S(64)
#undef TKG_S
  return cudaErrorInvalidValue;
}

cudaError_t launch_sumsq_diff(const double* a, const double* b, uint64_t n, double* part,
                              cudaStream_t st) {
  const int nb = sumsq_partials_count(n);
  if (nb == 0) return cudaSuccess;
  sumsq_diff_kernel<<<nb, kSqBlock, 0, st>>>(a, b, n, part);
  return cudaGetLastError();
}

int gram_partials_count(uint32_t rows) { return int((rows + kGramRows - 1) / kGramRows); }

cudaError_t launch_gram_partials(const double* X, uint64_t ld, uint32_t rows, uint32_t r,
                                 double* part, cudaStream_t st) {
  const int nb = gram_partials_count(rows);
  gram_partials_kernel<<<nb, 256, sizeof(double) * kGramRows * r, st>>>(X, ld, rows, r, part);
  return cudaGetLastError();
}

cudaError_t launch_chol(const double* part, int nparts, uint64_t part_ld, int rowstride,
                        uint32_t r, double* G, double* chol, int32_t* flag, DevStatus* status,
                        cudaStream_t st, double floor_rel) {
  chol_kernel<<<1, 256, sizeof(double) * 2 * r * r, st>>>(part, nparts, part_ld, rowstride, r, G,
                                                          chol, flag, status, floor_rel);
  return cudaGetLastError();
}

cudaError_t launch_qr(const double* Y, int nparts, uint64_t ldy, uint32_t rows, uint32_t r,
                      double* q, double* rmat, double* rt, uint32_t ldrt, double* work,
                      int check_degenerate, DevStatus* status, cudaStream_t st, const int32_t* only_if,
                      int32_t* degen_out) {
  qr_kernel<<<1, 1024, 0, st>>>(Y, nparts, ldy, rows, r, q, rmat, rt, ldrt, work,
                                check_degenerate, status, only_if, degen_out);
  return cudaGetLastError();
}

cudaError_t launch_sum(const double* partials, int n, double* dst, cudaStream_t st) {
  sum_kernel<<<1, 256, 0, st>>>(partials, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_pack(const double* src, uint64_t rs, uint64_t cs, uint32_t rows, uint32_t cols,
                        double* dst, uint32_t ldd, cudaStream_t st) {
  const uint64_t n = uint64_t(rows) * ldd;
  pack_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(src, rs, cs, rows, cols, dst, ldd);
  return cudaGetLastError();
}

int sumsq_partials_count(uint64_t n) { return int((n + kSqPerBlock - 1) / kSqPerBlock); }

cudaError_t launch_sumsq(const double* x, uint64_t n, double* part, cudaStream_t st) {
  const int nb = sumsq_partials_count(n);
  if (nb == 0) return cudaSuccess;
  sumsq_kernel<<<nb, kSqBlock, 0, st>>>(x, n, part);
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const double* part, int nparts, uint32_t rows, uint32_t ldp,
                                   uint32_t r, double* y, cudaStream_t st) {
  const uint64_t n = uint64_t(rows) * r;
  reduce_partials_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(part, nparts, rows, ldp, r, y);
  return cudaGetLastError();
}

cudaError_t launch_add(double* dst, const double* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int grid = int(std::min<size_t>((n + 255) / 256, 4096));
  add_kernel<<<grid, 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

cudaError_t launch_reduce_slot0(double* part, int nparts, uint32_t I, uint32_t ldp, uint32_t r, cudaStream_t st) {
  if (nparts <= 1) return cudaSuccess;
  const uint64_t threads = uint64_t(I) * r * 8;
  reduce_slot0_kernel<<<int((threads + 255) / 256), 256, 0, st>>>(part, nparts, I, ldp, r);
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const double* part, int nparts, uint64_t pld, uint32_t rs, uint32_t r, double* G,
                               cudaStream_t st) {
  const uint32_t ntri = r * (r + 1) / 2;
  gram_reduce_kernel<<<(ntri + 7) / 8, 256, 0, st>>>(part, nparts, pld, rs, r, G);
  return cudaGetLastError();
}

cudaError_t launch_copy_box(const double* src, double* dst, const BoxCopy& b, cudaStream_t st) {
  uint64_t total = 1;
  for (int k = 0; k < b.N; ++k) total *= b.box[k];
  if (total == 0) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((total + 255) / 256, 148 * 16));
  copy_box_kernel<<<grid, 256, 0, st>>>(src, dst, b, total);
  return cudaGetLastError();
}

cudaError_t launch_sym_eig(const double* G, uint32_t r, double* vt, double* evals, cudaStream_t st) {
  if (r < 1 || r > uint32_t(kEigMax)) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * 2 * kEigMax * kEigLd;
  cudaError_t e = raise_smem_limit(sym_eig_kernel, smem);
  if (e != cudaSuccess) return e;
  sym_eig_kernel<<<1, kEigThreads, smem, st>>>(G, r, vt, evals);
  return cudaGetLastError();
}




namespace {
__global__ void __launch_bounds__(256) normalize_columns_kernel(double* X, uint32_t rows) {
  __shared__ double red[8];
  double* x = X + size_t(blockIdx.x) * rows;
  double mx = 0.0;
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) mx = fmax(mx, fabs(x[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < 8; ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  if (mx == 0.0) return;
  const double inv = 1.0 / mx;  // scaled first: no overflow in the sum of squares
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) s += (x[i] * inv) * (x[i] * inv);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  s = 0.0;
  for (int w = 0; w < 8; ++w) s += red[w];
  const double f = inv / sqrt(s);
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) x[i] *= f;
}
}  // namespace

cudaError_t launch_normalize_columns(double* X, uint32_t rows, uint32_t cols, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  normalize_columns_kernel<<<cols, 256, 0, st>>>(X, rows);
  return cudaGetLastError();
}

}  // namespace tkg
