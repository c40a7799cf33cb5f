// Small dense kernels of the ALS step (r <= 64, I_n <= a few thousand):
// Gram partials, Cholesky with the reference's pivot floor, row-wise SPD
// solves, Householder QR with the reference's sign convention, and the
// closed-form residual. They run on-device so a sweep never round-trips
// through the host except for the one status read that decides the stop.
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

// ---- row-wise SPD solve ------------------------------------------------------
__global__ void row_solve_kernel(const double* __restrict__ B, int nparts, uint64_t ldb,
                                 uint32_t rows, uint32_t r, const double* __restrict__ chol,
                                 double* x_cm, double* xt, uint32_t ldxt, const int32_t* skip,
                                 int forward_only) {
  if (skip && *skip) return;
  extern __shared__ double sm[];
  double* Ls = sm;                 // r*r
  double* xs = sm + r * r;         // [r][blockDim]
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) Ls[e] = chol[e];
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const uint32_t T = blockDim.x, t = threadIdx.x;
  for (uint32_t c = 0; c < r; ++c) {
    double b;
    if (nparts > 0) {
      b = 0.0;
      for (int k = 0; k < nparts; ++k) b += B[(size_t(k) * rows + i) * ldb + c];
    } else {
      b = B[i + uint64_t(c) * ldb];
    }
    xs[c * T + t] = b;
  }
  // Forward substitution L y = b, then L^T x = y (kernels.cpp:401-415).
  for (uint32_t a = 0; a < r; ++a) {
    double acc = xs[a * T + t];
    for (uint32_t p = 0; p < a; ++p) acc -= Ls[a + p * r] * xs[p * T + t];
    xs[a * T + t] = acc / Ls[a + a * r];
  }
  if (!forward_only) {
    for (uint32_t a = r; a-- > 0;) {
      double acc = xs[a * T + t];
      for (uint32_t p = a + 1; p < r; ++p) acc -= Ls[p + a * r] * xs[p * T + t];
      xs[a * T + t] = acc / Ls[a + a * r];
    }
  }
  for (uint32_t c = 0; c < r; ++c) {
    const double v = xs[c * T + t];
    if (x_cm) x_cm[i + uint64_t(c) * rows] = v;
    if (xt) xt[uint64_t(i) * ldxt + c] = v;
  }
  if (xt)
    for (uint32_t c = r; c < ldxt; ++c) xt[uint64_t(i) * ldxt + c] = 0.0;
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
                                                  DevStatus* status) {
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
    status->degenerate_col = bad;
  }
}

// ---- closed-form residual (als.cpp:18-25,52-55) -----------------------------
__global__ void finish_right_kernel(const double* __restrict__ fc_gram, int nparts, int nc,
                                    uint32_t r, const double* __restrict__ GL, double* GR,
                                    double* cholR, DevStatus* status) {
  extern __shared__ double sm[];
  double* Gs = sm;
  double* Ls = sm + r * r;
  reduce_upper(fc_gram, nparts, uint64_t(nc) * nc, nc, r, Gs);
  __syncthreads();
  // trace(G_L G_R) = sum_ij GL(i,j) GR(i,j), compensated (TwoSum) per lane
  // then combined in a fixed tree.
  __shared__ double hi_s[32], lo_s[32];
  if (threadIdx.x < 32) {
    double s = 0.0, c = 0.0;
    for (uint32_t e = threadIdx.x; e < r * r; e += 32) {
      double p = GL[e] * Gs[e];
      double pe = fma(GL[e], Gs[e], -p);
      double t, err;
      two_sum(s, p, t, err);
      s = t;
      c += err + pe;
    }
    hi_s[threadIdx.x] = s;
    lo_s[threadIdx.x] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, c = 0.0;
    for (int k = 0; k < 32; ++k) {
      double t, err;
      two_sum(s, hi_s[k], t, err);
      s = t;
      c += err + lo_s[k];
    }
    const double tr = s + c;
    const double norm = sqrt(status->sumsq);  // frobenius_norm (tensor_ops.cpp:391-393)
    const double norm_sq = norm * norm;       // als.cpp:106
    status->trace = tr;
    status->residual = sqrt(fmax(0.0, norm_sq - tr));
  }
  __syncthreads();
  block_chol(Gs, Ls, r, &status->left_singular, status);
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    GR[e] = Gs[e];
    cholR[e] = Ls[e];
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

// ---- Gram of a row-major matrix on the tensor pipe ----------------------------
// Each CTA owns a contiguous row range, streams 128-row blocks through a
// double-buffered cp.async ring (row pitch NC+4 = 4 mod 16 doubles) and
// accumulates its upper-triangle 8x8 tiles with DMMA in registers.
template <int NC>
__global__ void __launch_bounds__(256) gram_rm_kernel(const double* __restrict__ X, uint64_t rows,
                                                      uint32_t r, uint64_t ld, double* part,
                                                      const int32_t* skip) {
  if (skip && *skip) return;
  constexpr int kRows = 128, kLd = NC + 4, kNT = NC / 8, kTri = kNT * (kNT + 1) / 2;
  constexpr int kPer = (kTri + 7) / 8;
  extern __shared__ __align__(16) double tile[];  // [2][kRows][kLd]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
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
  const uint64_t nblk = (rows + kRows - 1) / kRows;
  const uint64_t per = (nblk + gridDim.x - 1) / gridDim.x;
  const uint64_t b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
  const bool vec = (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && (NC % 2 == 0);
  auto load = [&](uint64_t b, int buf) {
    double* t = tile + buf * kRows * kLd;
    const uint64_t r0 = b * kRows;
    if (vec) {
      for (int e = threadIdx.x; e < kRows * (NC / 2); e += blockDim.x) {
        const int row = e / (NC / 2), c = (e % (NC / 2)) * 2;
        const uint64_t gr = r0 + row;
        if (gr < rows) cp_async16(t + row * kLd + c, X + gr * ld + c);
        else { t[row * kLd + c] = 0.0; t[row * kLd + c + 1] = 0.0; }
      }
    } else {
      for (int e = threadIdx.x; e < kRows * NC; e += blockDim.x) {
        const int row = e / NC, c = e % NC;
        const uint64_t gr = r0 + row;
        t[row * kLd + c] = gr < rows ? X[gr * ld + c] : 0.0;
      }
    }
    cp_async_commit();
  };
  if (b0 < b1) load(b0, 0);
  for (uint64_t b = b0; b < b1; ++b) {
    const int buf = int((b - b0) & 1);
    if (b + 1 < b1) {
      load(b + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* t = tile + buf * kRows * kLd;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (tm[k] < 0) continue;
#pragma unroll 8
      for (int k0 = 0; k0 < kRows; k0 += 4) {
        const double* rp = t + (k0 + q) * kLd;
        dmma(acc[k][0], acc[k][1], rp[tm[k] * 8 + r8], rp[tn[k] * 8 + r8]);
      }
    }
    __syncthreads();
  }
  // columns >= r hold whatever the padding held; the consumer reads c < r only
  double* out = part + size_t(blockIdx.x) * NC * NC;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (tm[k] < 0) continue;
    const int c1 = tm[k] * 8 + r8, c2 = tn[k] * 8 + 2 * q;
    out[c1 * NC + c2] = acc[k][0];
    out[c1 * NC + c2 + 1] = acc[k][1];
  }
}

// ---- st-HOSVD shrink ---------------------------------------------------------
constexpr int kShrinkThreads = 256;
constexpr int kShrinkFibers = 4096;  // fibers per CTA

__global__ void __launch_bounds__(kShrinkThreads) shrink_kernel(
    const double* __restrict__ R, uint64_t ld, uint64_t s, uint64_t P, uint32_t r,
    const double* __restrict__ rhat, double* __restrict__ out, double* sumsq_part) {
  extern __shared__ double rh[];  // r x r column-major
  __shared__ double red[32];
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) rh[e] = rhat[e];
  __syncthreads();
  const uint64_t F = s * P;
  const uint64_t f0 = uint64_t(blockIdx.x) * kShrinkFibers;
  const uint64_t f1 = min(F, f0 + kShrinkFibers);
  double sq = 0.0;
  for (uint64_t j = f0 + threadIdx.x; j < f1; j += blockDim.x) {
    const uint64_t p = j / s, jl = j - p * s;
    const double* row = R + j * ld;
    double* o = out + jl + p * s * r;
    for (uint32_t c = 0; c < r; ++c) {
      double acc = 0.0;
      for (uint32_t k = 0; k < r; ++k) acc = fma(rh[c + k * r], row[k], acc);
      o[uint64_t(c) * s] = acc;
      sq = fma(acc, acc, sq);
    }
  }
  sq = block_sum(sq, red);
  if (threadIdx.x == 0) sumsq_part[blockIdx.x] = sq;
}

// R = R2 R1 with R_k = L_k^T (CholQR2), the reference's degeneracy test on
// diag(R) (als.cpp:74-86), and optional outputs R (col-major) / R^T padded.
__global__ void cholqr_finish_kernel(const double* __restrict__ L1, const double* __restrict__ L2,
                                     uint32_t r, const int32_t* fail1, const int32_t* fail2,
                                     double* rmat, double* rt, uint32_t ldrt, int check,
                                     DevStatus* status) {
  extern __shared__ double Rs[];
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t i = e % r, j = e / r;
    double acc = 0.0;
    if (i <= j)
      for (uint32_t k = i; k <= j; ++k) acc += L2[k + i * r] * L1[j + k * r];  // R2[i][k] R1[k][j]
    Rs[e] = acc;
    if (rmat) rmat[e] = acc;
  }
  __syncthreads();
  if (rt)
    for (uint32_t e = threadIdx.x; e < r * ldrt; e += blockDim.x) {
      const uint32_t row = e / ldrt, c = e % ldrt;  // rt[c'][c] = R[c][c']
      rt[e] = c < r ? Rs[c + row * r] : 0.0;
    }
  if (check && threadIdx.x == 0) {
    int bad = 0;
    if (*fail1 || *fail2) {
      bad = 1;
    } else {
      double md = 0.0;
      for (uint32_t i = 0; i < r; ++i) md = fmax(md, fabs(Rs[i + i * r]));
      for (uint32_t i = 0; i < r; ++i)
        if (fabs(Rs[i + i * r]) <= 1e-13 * md || md == 0.0) {
          bad = int(i) + 1;
          break;
        }
    }
    status->degenerate_col = bad;
  }
}

}  // namespace

cudaError_t launch_cholqr_finish(const double* L1, const double* L2, uint32_t r, const int32_t* fail1,
                                 const int32_t* fail2, double* rmat, double* rt, uint32_t ldrt,
                                 int check, DevStatus* status, cudaStream_t st) {
  cholqr_finish_kernel<<<1, 256, sizeof(double) * r * r, st>>>(L1, L2, r, fail1, fail2, rmat, rt, ldrt,
                                                               check, status);
  return cudaGetLastError();
}

int gram_rm_count(uint64_t rows, int num_sms) {
  const uint64_t nblk = (rows + 127) / 128;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(nblk, uint64_t(num_sms))));
}

cudaError_t launch_gram_rm(const double* X, uint64_t rows, uint32_t r, uint64_t ld, double* part,
                           int num_sms, cudaStream_t st, const int32_t* skip) {
  const int grid = gram_rm_count(rows, num_sms);
  const uint32_t ncp = r <= 8 ? 8 : (r + 7) / 8 * 8;
  switch (ncp) {
#define TKG_G(N)                                                                          \
  case N: {                                                                               \
    const size_t sm = sizeof(double) * 2 * 128 * (N + 4);                                 \
    cudaFuncSetAttribute(gram_rm_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)); \
    gram_rm_kernel<N><<<grid, 256, sm, st>>>(X, rows, r, ld, part, skip);                  \
    break;                                                                                \
  }
    TKG_G(8) TKG_G(16) TKG_G(24) TKG_G(32) TKG_G(40) TKG_G(48) TKG_G(56) TKG_G(64)
#undef TKG_G
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int shrink_count(uint64_t F) { return int((F + kShrinkFibers - 1) / kShrinkFibers); }

cudaError_t launch_shrink(const double* R, uint64_t ld, uint64_t s, uint64_t P, uint32_t r,
                          const double* rhat, double* out, double* sumsq_part, cudaStream_t st) {
  const int grid = shrink_count(s * P);
  shrink_kernel<<<grid, kShrinkThreads, sizeof(double) * r * r, st>>>(R, ld, s, P, r, rhat, out,
                                                                       sumsq_part);
  return cudaGetLastError();
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

cudaError_t launch_row_solve(const double* B, int nparts, uint64_t ldb, uint32_t rows, uint32_t r,
                             const double* chol, double* x_cm, double* xt, uint32_t ldxt,
                             const int32_t* skip, cudaStream_t st, int forward_only) {
  const int T = 32;
  const size_t smem = sizeof(double) * (size_t(r) * r + size_t(r) * T);
  row_solve_kernel<<<(rows + T - 1) / T, T, smem, st>>>(B, nparts, ldb, rows, r, chol, x_cm, xt,
                                                         ldxt, skip, forward_only);
  return cudaGetLastError();
}

cudaError_t launch_qr(const double* Y, int nparts, uint64_t ldy, uint32_t rows, uint32_t r,
                      double* q, double* rmat, double* rt, uint32_t ldrt, double* work,
                      int check_degenerate, DevStatus* status, cudaStream_t st) {
  qr_kernel<<<1, 1024, 0, st>>>(Y, nparts, ldy, rows, r, q, rmat, rt, ldrt, work,
                                check_degenerate, status);
  return cudaGetLastError();
}

cudaError_t launch_finish_right(const double* fc_gram, int nparts, int nc_stride, uint32_t r,
                                const double* GL, const double* /*norm_sq*/, double* GR,
                                double* cholR, DevStatus* status, cudaStream_t st) {
  finish_right_kernel<<<1, 1024, sizeof(double) * 2 * r * r, st>>>(fc_gram, nparts, nc_stride, r,
                                                                   GL, GR, cholR, status);
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

}  // namespace tkg
