// Small dense kernels of the ALS step (r <= 64, I_n <= a few thousand):
// Gram partials, Cholesky with the reference's pivot floor, row-wise SPD
// solves, Householder QR with the reference's sign convention, and the
// closed-form residual. They run on-device so a sweep never round-trips
// through the host except for the one status read that decides the stop.
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
__device__ void block_chol(double* G, double* L, uint32_t r, int32_t* flag, DevStatus* status) {
  __shared__ double piv_s;
  __shared__ int fail_s;
  // max diagonal (kernels.cpp:378-379) and floor
  __shared__ double floor_s;
  if (threadIdx.x == 0) {
    double md = 0.0;
    for (uint32_t i = 0; i < r; ++i) md = fmax(md, G[i + i * r]);
    floor_s = 1e-13 * md;
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
    for (int k = 0; k < nparts; ++k) s += part[size_t(k) * part_ld + size_t(a) * rowstride + b];
    G[e] = s;
  }
}

__global__ void chol_kernel(const double* __restrict__ part, int nparts, uint64_t part_ld,
                            int rowstride, uint32_t r, double* G, double* chol, int32_t* flag,
                            DevStatus* status) {
  extern __shared__ double sm[];
  double* Gs = sm;
  double* Ls = sm + r * r;
  reduce_upper(part, nparts, part_ld, rowstride, r, Gs);
  __syncthreads();
  block_chol(Gs, Ls, r, flag, status);
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    if (G) G[e] = Gs[e];
    chol[e] = Ls[e];
  }
}

// ---- row-wise SPD solve ------------------------------------------------------
__global__ void row_solve_kernel(const double* __restrict__ B, int nparts, uint64_t ldb,
                                 uint32_t rows, uint32_t r, const double* __restrict__ chol,
                                 double* x_cm, double* xt, uint32_t ldxt, const int32_t* skip) {
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
  for (uint32_t a = r; a-- > 0;) {
    double acc = xs[a * T + t];
    for (uint32_t p = a + 1; p < r; ++p) acc -= Ls[p + a * r] * xs[p * T + t];
    xs[a * T + t] = acc / Ls[a + a * r];
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

}  // namespace

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
                        cudaStream_t st) {
  chol_kernel<<<1, 256, sizeof(double) * 2 * r * r, st>>>(part, nparts, part_ld, rowstride, r, G,
                                                          chol, flag, status);
  return cudaGetLastError();
}

cudaError_t launch_row_solve(const double* B, int nparts, uint64_t ldb, uint32_t rows, uint32_t r,
                             const double* chol, double* x_cm, double* xt, uint32_t ldxt,
                             const int32_t* skip, cudaStream_t st) {
  const int T = 64;
  const size_t smem = sizeof(double) * (size_t(r) * r + size_t(r) * T);
  row_solve_kernel<<<(rows + T - 1) / T, T, smem, st>>>(B, nparts, ldb, rows, r, chol, x_cm, xt,
                                                         ldxt, skip);
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
  finish_right_kernel<<<1, 256, sizeof(double) * 2 * r * r, st>>>(fc_gram, nparts, nc_stride, r,
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
