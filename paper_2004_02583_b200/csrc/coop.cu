// Cooperative (grid-synchronised) small dense steps of the ALS sweep.
//
// Each step is one persistent launch (one CTA per SM) whose phases are
// separated by grid.sync(): the split-K partial sums and the Gram partials
// are reduced by the whole grid, the I x r factor is processed in 32-row
// blocks by a grid-stride loop, and the r x r factorizations run on CTA 0.
// The normal-equation solves use the explicit inverse of the r x r Gram
// matrix (with the spd_solve pivot floor, kernels.cpp:378-393), so applying
// it to a row is an r-wide dot product per output instead of a dependent
// substitution chain.
//
//   prep_step   : [L = (sum FR partials) G_R^{-1}]  G_L = L^T L  G_L^{-1}
//                 Mt = L G_L^{-1} (i-major, the FC operand)     (als.cpp:36-50)
//   finish_step : G_R = R^T R (fused into the FC epilogue up to r = 32, else
//                 a DMMA row pass here), closed-form residual, the stop rule,
//                 G_R^{-1} for the next left update (als.cpp:52-55,136-160)
//   cholqr_step : CholQR2 thin QR with R_ii > 0 and the reference's
//                 degeneracy test (kernels.cpp:303-367, als.cpp:74-86)
//
// The r x r kernels on CTA 0 (Cholesky, triangular inverse, Gauss-Jordan
// inverse) keep each thread's matrix entries in registers; the one row /
// column every step needs is published to a double-buffered shared vector by
// its owners, so a step costs one barrier and a few independent loads.
// Every reduction runs in a fixed order (deterministic results).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cmath>
#include <type_traits>

#include "als_step.cuh"
#include "blockfact.cuh"
#include "coop.cuh"
#include "contract_tma.cuh"

namespace cg = cooperative_groups;

namespace tkg {

#ifdef TKG_PHASE_TIMING
__device__ unsigned long long g_phase_ns[64];
#define PHASE(k)                                                                            \
  do {                                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                              \
      unsigned long long t_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_phase_ns[k] = t_;                                                                   \
    }                                                                                       \
  } while (0)
#else
#define PHASE(k) \
  do {           \
  } while (0)
#endif

namespace {

constexpr int kRB = 32;        // factor rows per block
constexpr int kThreads = 256;
constexpr int kMaxR = 64;
constexpr int kGE = (kMaxR * kMaxR + kThreads - 1) / kThreads;  // Gram entries per thread

// Scratch (doubles) of the blocked factorizations that a launch adds to its
// shared memory: blk_scratch(r) above r = 16 when base + scratch fits 227 KB.
__host__ __device__ constexpr int scratch_for(int r, size_t base_doubles) {
  return (r > 16 && (base_doubles + size_t(blk_scratch(r))) * 8 <= size_t(227) * 1024) ? blk_scratch(r) : 0;
}
__host__ __device__ constexpr size_t rows_base(int r) { return 2 * size_t(kRB) * (r + 1) + 3 * size_t(r) * r; }
__host__ __device__ constexpr size_t prep_cluster_base(int r) { return 2 * size_t(kRB) * (r + 1) + 4 * size_t(r) * r; }
__host__ __device__ constexpr size_t cholqr_cluster_base(int r) {
  return 2 * size_t(kRB) * (r + 1) + 5 * size_t(r) * r;
}
__host__ __device__ constexpr size_t finish_cluster_base(int r) { return 2 * size_t(r) * r; }

// entries of an r x r matrix per thread: a kB x kB block, kB = ceil(r / 16)
__host__ __device__ constexpr int kb_for(int r) { return (r + 15) / 16; }
__host__ __device__ constexpr int ke_for(int r) { return kb_for(r) * kb_for(r); }

// ---- one-CTA dense kernels (CTA 0), register-resident -------------------------------
// The r x r matrix is tiled 16 x 16 over the threads: thread t owns the
// kB x kB block of rows i0 + a, columns j0 + b (i0 = (t % 16) kB,
// j0 = (t / 16) kB), entry t' = a + b kB. A step needs kB entries of the
// published row / column per thread instead of one per owned entry (the
// steps are shared-memory bound). Entries past r are dummies: they read the
// spare slots of the shared vectors (sized kMaxR + 1 >= 16 kB), never
// publish into a live slot and are never stored.
template <int KE>
struct Owned {
  static constexpr int kB = KE == 1 ? 1 : KE == 4 ? 2 : KE == 9 ? 3 : 4;
  static_assert(kB * kB == KE, "KE must be a square");
  double v[KE];
  int i0, j0;
  __device__ explicit Owned(uint32_t) {
    i0 = int(threadIdx.x % 16) * kB;
    j0 = int(threadIdx.x / 16) * kB;
#pragma unroll
    for (int t = 0; t < KE; ++t) v[t] = 0.0;
  }
  __device__ int i(int t) const { return i0 + t % kB; }
  __device__ int j(int t) const { return j0 + t / kB; }
  __device__ bool valid(int t, uint32_t r) const { return i(t) < int(r) && j(t) < int(r); }
};

// Lower Cholesky factor of G (column-major, smem) into L (smem): right-looking
// updates of the unscaled Schur complement; column k+1 is published once its
// last update (step k) is done. Positivity is the only pivot test (CholQR).
// Returns the failing column + 1 or 0.
template <int KE>
__device__ int chol_reg(const double* G, double* L, uint32_t r) {
  constexpr int B = Owned<KE>::kB;
  __shared__ double cb[2][kMaxR + 1];
  __shared__ double dg[kMaxR + 1];
  Owned<KE> o(r);
#pragma unroll
  for (int t = 0; t < KE; ++t) {
    const int i = o.i(t), j = o.j(t);
    if (o.valid(t, r) && i >= j) o.v[t] = G[i + j * r];
    if (j == 0 && i < int(r)) cb[0][i] = o.v[t];
  }
  __syncthreads();
  int fail = 0;
  for (uint32_t k = 0; k < r; ++k) {
    const double* c = cb[k & 1];
    double* cn = cb[(k + 1) & 1];
    const double p = c[k];  // uniform across the CTA
    if (!(p > 0.0)) {
      fail = int(k) + 1;
      break;
    }
    if (threadIdx.x == 0) dg[k] = p;
    const double inv = __drcp_rn(p);
    double ci[B], cj[B];
#pragma unroll
    for (int a = 0; a < B; ++a) {
      ci[a] = c[o.i0 + a];
      cj[a] = c[o.j0 + a];
    }
#pragma unroll
    for (int t = 0; t < KE; ++t) {
      const int i = o.i(t), j = o.j(t);
      if (j > int(k) && i >= j) o.v[t] = fma(-ci[t % B] * inv, cj[t / B], o.v[t]);
      if (j == int(k) + 1 && i < int(r)) cn[i] = o.v[t];
    }
    __syncthreads();
  }
  if (fail) {
    __syncthreads();
    return fail;
  }
#pragma unroll
  for (int t = 0; t < KE; ++t) {
    if (!o.valid(t, r)) continue;
    const int i = o.i(t), j = o.j(t);
    const double d = sqrt(dg[j]);
    L[i + j * r] = i > j ? o.v[t] / d : (i == j ? d : 0.0);
  }
  __syncthreads();
  return 0;
}

// X = L^{-1} (lower) by right-looking forward substitution on the identity:
// row k, final up to its 1/L_kk scale after step k-1, updates the rows below.
template <int KE>
__device__ void tri_inv_reg(const double* L, double* X, uint32_t r) {
  constexpr int B = Owned<KE>::kB;
  __shared__ double rb[2][kMaxR + 1];
  Owned<KE> o(r);
#pragma unroll
  for (int t = 0; t < KE; ++t) {
    const int i = o.i(t), j = o.j(t);
    o.v[t] = i == j ? 1.0 : 0.0;
    if (i == 0 && j < int(r)) rb[0][j] = o.v[t];
  }
  __syncthreads();
  for (uint32_t k = 0; k + 1 < r; ++k) {
    const double* u = rb[k & 1];
    double* un = rb[(k + 1) & 1];
    const double rk = __drcp_rn(L[k + k * r]);
    double lik[B], ukc[B];
#pragma unroll
    for (int a = 0; a < B; ++a) {
      lik[a] = L[min(o.i0 + a, int(r) - 1) + k * r];
      ukc[a] = u[o.j0 + a];
    }
#pragma unroll
    for (int t = 0; t < KE; ++t) {
      const int i = o.i(t), c = o.j(t);
      if (i > int(k) && c <= int(k) && i < int(r)) o.v[t] = fma(-lik[t % B] * rk, ukc[t / B], o.v[t]);
      if (i == int(k) + 1 && c < int(r)) un[c] = o.v[t];
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < KE; ++t) {
    if (!o.valid(t, r)) continue;
    const int i = o.i(t), c = o.j(t);
    X[i + c * r] = i >= c ? o.v[t] / L[i + i * r] : 0.0;
  }
  __syncthreads();
}

// Inverse of the SPD matrix G (column-major, smem) by Gauss-Jordan elimination
// without pivoting into out (smem). The pivot of step k is the Schur
// complement diagonal, i.e. the Cholesky pivot, tested with spd_solve's floor
// (pivot <= floor_rel * max diag fails, kernels.cpp:378-393). Row k and
// column k of the current matrix are published by their owners. Returns the
// failing column + 1 (pivot in *piv_out) or 0.
template <int KE>
__device__ int gj_inv_reg(const double* G, double* out, uint32_t r, double floor_rel, double* piv_out) {
  constexpr int B = Owned<KE>::kB;
  __shared__ double rowb[2][kMaxR + 1], colb[2][kMaxR + 1];
  Owned<KE> o(r);
  double md = 0.0;
  for (uint32_t i = 0; i < r; ++i) md = fmax(md, G[i + i * r]);
  const double floor_v = floor_rel * md;
#pragma unroll
  for (int t = 0; t < KE; ++t) {
    const int i = o.i(t), j = o.j(t);
    if (o.valid(t, r)) o.v[t] = G[i + j * r];
    if (i == 0 && j < int(r)) rowb[0][j] = o.v[t];
    if (j == 0 && i < int(r)) colb[0][i] = o.v[t];
  }
  __syncthreads();
  for (uint32_t k = 0; k < r; ++k) {
    const double* rw = rowb[k & 1];
    const double* cl = colb[k & 1];
    double* rwn = rowb[(k + 1) & 1];
    double* cln = colb[(k + 1) & 1];
    const double p = rw[k];  // uniform across the CTA
    if (!(p > floor_v) || !(p > 0.0)) {
      if (piv_out && threadIdx.x == 0) *piv_out = p;
      __syncthreads();
      return int(k) + 1;
    }
    const double ip = __drcp_rn(p);
    double aik[B], akj[B];
#pragma unroll
    for (int a = 0; a < B; ++a) {
      aik[a] = cl[o.i0 + a];
      akj[a] = rw[o.j0 + a];
    }
#pragma unroll
    for (int t = 0; t < KE; ++t) {
      const int i = o.i(t), j = o.j(t);
      const double old = o.v[t];
      double v;
      if (i == int(k)) v = j == int(k) ? ip : old * ip;
      else if (j == int(k)) v = -old * ip;
      else v = fma(-aik[t % B] * ip, akj[t / B], old);
      o.v[t] = v;
      if (i == int(k) + 1 && j < int(r)) rwn[j] = v;
      if (j == int(k) + 1 && i < int(r)) cln[i] = v;
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < KE; ++t)
    if (o.valid(t, r)) out[o.i(t) + o.j(t) * r] = o.v[t];
  __syncthreads();
  return 0;
}

// ---- dispatch: blocked (blockfact.cuh) above r = 16 when the caller has the
// scratch, else the register-resident kernels above ---------------------------
__device__ __forceinline__ bool use_blk(uint32_t r, const double* scratch, int avail) {
  return r > 16 && scratch != nullptr && avail >= blk_scratch(int(r));
}

template <int KE>
__device__ int spd_inverse(const double* G, double* out, uint32_t r, double floor_rel, double* piv_out,
                           double* scratch, int avail) {
  if (use_blk(r, scratch, avail)) return blk_spd_inverse(G, out, r, floor_rel, piv_out, scratch);
  return gj_inv_reg<KE>(G, out, r, floor_rel, piv_out);
}

// CholQR's factorization: L (lower, r x r column-major) of G by Cholesky with
// the positivity test only; on success Linv = L^{-1}. Returns the failing
// column (1-based) or 0.
template <int KE>
__device__ int chol_and_inverse(const double* G, double* L, double* Linv, uint32_t r, double* scratch, int avail) {
  if (use_blk(r, scratch, avail)) {
    const int ld = blk_ld(int(r)), rp = blk_rp(int(r));
    double* W = scratch;
    double* X = W + rp * ld;
    double* T = X + rp * ld;
    double* dinv = T + 8 * 64;
    blk_load(G, r, W);
    const int fail = blk_chol(W, r, 0.0, nullptr, dinv);
    if (fail) return fail;
    blk_trinv(W, r, X, T, dinv);
    for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
      const uint32_t i = e % r, j = e / r;
      L[e] = i >= j ? W[i + j * ld] : 0.0;
      Linv[e] = i >= j ? X[i + j * ld] : 0.0;
    }
    __syncthreads();
    return 0;
  }
  const int fail = chol_reg<KE>(G, L, r);
  if (!fail) tri_inv_reg<KE>(L, Linv, r);
  return fail;
}

// ---- grid-wide reductions -----------------------------------------------------------

// Gs (global, column-major r x r, symmetric) = sum over k of
// part[k*pld + a*rs + b] for a <= b: one warp per entry, lanes over k, a
// fixed xor tree (lane 0's sum is the result).
__device__ void reduce_gram_grid(const double* part, int nparts, uint64_t pld, uint32_t rs, uint32_t r,
                                 double* Gs) {
  const uint32_t wpb = blockDim.x >> 5;
  const uint32_t nw = gridDim.x * wpb;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t ntri = r * (r + 1) / 2;
  for (uint32_t t = blockIdx.x * wpb + (threadIdx.x >> 5); t < ntri; t += nw) {
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
      Gs[a + b * r] = s;
      Gs[b + a * r] = s;
    }
  }
}

// part[0][i][c] = sum_k part[k][i][c] (c < r), in place. G = 2^g lanes share
// an entry (as many as the grid affords, <= 32): lane `sub` sums k = sub,
// sub + G, ... in order, then a fixed xor tree over the G lanes.
__device__ void reduce_partials_grid(double* part, int nparts, uint32_t I, uint32_t ldp, uint32_t r) {
  const uint64_t n = uint64_t(I) * r;
  const uint64_t stride = uint64_t(I) * ldp;
  const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
  uint32_t G = 1;
  while (G < 32 && uint64_t(2 * G) * n <= T && int(2 * G) <= nparts) G *= 2;
  const uint64_t gt = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t sub = uint32_t(gt % G);
  for (uint64_t e = gt / G;; e += T / G) {
    const bool act = e < n;
    if (!__any_sync(0xffffffffu, act)) break;
    double s = 0.0;
    double* p = nullptr;
    if (act) {
      const uint64_t i = e / r, c = e % r;
      p = part + i * ldp + c;
      int k = int(sub);
      for (; k + 7 * int(G) < nparts; k += 8 * int(G)) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[size_t(k + u * int(G)) * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; k < nparts; k += int(G)) s += p[size_t(k) * stride];
    }
    for (uint32_t off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (act && sub == 0) p[0] = s;
  }
}

// ---- row-block helpers ---------------------------------------------------------------

// X[row][c] (pitch ld) = rows i0.. of a row-major or column-major I x r
// matrix with leading dimension ld_src.
__device__ void load_rows(const double* src, bool row_major, uint64_t ld_src, uint32_t i0, uint32_t nrow,
                          uint32_t r, double* X, uint32_t ld) {
  if (row_major) {
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e / r, c = e % r;
      X[row * ld + c] = src[uint64_t(i0 + row) * ld_src + c];
    }
  } else {
    for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
      const uint32_t row = e % nrow, c = e / nrow;
      X[row * ld + c] = src[(i0 + row) + uint64_t(c) * ld_src];
    }
  }
}

__device__ void store_rows_cm(const double* X, uint32_t ld, uint32_t i0, uint32_t nrow, uint32_t r,
                              double* dst, uint64_t ld_dst) {
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e % nrow, c = e / nrow;
    dst[(i0 + row) + uint64_t(c) * ld_dst] = X[row * ld + c];
  }
}

// out[row][c] = sum_k X[row][k] Mr[k*r + c]  (rows in smem with pitch ld; Mr
// row-major so that a warp's consecutive c read consecutive banks)
__device__ void rows_mul(const double* X, uint32_t nrow, uint32_t r, uint32_t ld, const double* Mr,
                         double* out, uint32_t ldo) {
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    double s = 0.0;
    for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], Mr[k * r + c], s);
    out[row * ldo + c] = s;
  }
}

// Mr[k*r + c] = M(k, c) for a column-major r x r M in global memory.
__device__ void load_mat_rm(const double* M, double* Mr, uint32_t r) {
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t k = e / r, c = e % r;
    Mr[e] = M[k + c * r];
  }
  __syncthreads();
}

__device__ void load_mat(const double* src, double* dst, uint32_t n) {
  for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
  __syncthreads();
}

// Per-thread Gram accumulators: entry e = tid + t*blockDim (a = e / r,
// b = e % r, a <= b) over the CTA's row blocks.
struct GramAcc {
  double g[kGE];
  __device__ void zero() {
#pragma unroll
    for (int t = 0; t < kGE; ++t) g[t] = 0.0;
  }
  __device__ void add(const double* X, uint32_t nrow, uint32_t r, uint32_t ld) {
#pragma unroll
    for (int t = 0; t < kGE; ++t) {
      const uint32_t e = threadIdx.x + t * blockDim.x;
      if (e < r * r) {
        const uint32_t a = e / r, b = e % r;
        if (a <= b) {
          double s = g[t];
          for (uint32_t row = 0; row < nrow; ++row) s = fma(X[row * ld + a], X[row * ld + b], s);
          g[t] = s;
        }
      }
    }
  }
  __device__ void store(double* part, uint32_t r) const {
#pragma unroll
    for (int t = 0; t < kGE; ++t) {
      const uint32_t e = threadIdx.x + t * blockDim.x;
      if (e < r * r) part[e] = g[t];
    }
  }
};

// ---- prep_step -------------------------------------------------------------------
template <int KE>
__global__ void __launch_bounds__(kThreads) prep_step_kernel(PrepArgs a) {
  cg::grid_group grid = cg::this_grid();
  AlsCtrl* ctrl = a.ctrl;
  if (ctrl->stop) return;  // uniform: nobody writes stop before the first grid.sync
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1, I = a.I;
  double* X = sm;                 // [kRB][ld]
  double* X2 = X + kRB * ld;      // [kRB][ld]
  double* M = X2 + kRB * ld;      // r*r
  double* W = M + r * r;          // r*r (CTA 0 scratch)
  const uint32_t nblk = (I + kRB - 1) / kRB;

  PHASE(20);
  // Phase A: sum of the FR partials into slot 0
  if (a.from_partials && a.nparts > 1) {
    reduce_partials_grid(a.part, a.nparts, I, a.ldp, r);
    grid.sync();
  }
  PHASE(21);
  // Phase B: L rows (from partials: Y G_R^{-1}, kept row-major in slot 0 and
  // written to Lc), and their Gram partial
  if (a.from_partials) load_mat_rm(a.GRinv, M, r);
  GramAcc g;
  g.zero();
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const uint32_t i0 = b * kRB, nrow = min(uint32_t(kRB), I - i0);
    if (a.from_partials) {
      load_rows(a.part, true, a.ldp, i0, nrow, r, X, ld);
      __syncthreads();
      rows_mul(X, nrow, r, ld, M, X2, ld);
      __syncthreads();
      for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
        const uint32_t row = e / r, c = e % r;
        a.part[uint64_t(i0 + row) * a.ldp + c] = X2[row * ld + c];
      }
      store_rows_cm(X2, ld, i0, nrow, r, a.Lc, I);
    } else {
      load_rows(a.Lc, false, I, i0, nrow, r, X2, ld);
      __syncthreads();
    }
    g.add(X2, nrow, r, ld);
    __syncthreads();
  }
  g.store(a.gpart + size_t(blockIdx.x) * r * r, r);
  grid.sync();
  PHASE(22);
  reduce_gram_grid(a.gpart, gridDim.x, uint64_t(r) * r, r, r, a.gs);
  grid.sync();
  PHASE(23);

  // Phase C (CTA 0): G_L, its inverse with the spd_solve pivot floor
  if (blockIdx.x == 0) {
    load_mat(a.gs, M, r * r);
    double piv = 0.0;
    const int fail = spd_inverse<KE>(M, W, r, 1e-13, &piv, sm + rows_base(int(r)), scratch_for(int(r), rows_base(int(r))));
    if (fail) {
      if (threadIdx.x == 0) {
        ctrl->error = kAlsErrRightSingular;
        ctrl->pivot = piv;
        ctrl->pad = fail;  // failing column (1-based)
        ctrl->stop = 1;
      }
    } else {
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
        a.GL[e] = M[e];
        a.GLinv[e] = W[e];
      }
    }
  }
  PHASE(24);
  grid.sync();
  PHASE(25);
  if (ctrl->stop) return;

  // Phase D: Mt rows = L rows G_L^{-1}, padded to ncp
  load_mat_rm(a.GLinv, M, r);
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const uint32_t i0 = b * kRB, nrow = min(uint32_t(kRB), I - i0);
    if (a.from_partials) load_rows(a.part, true, a.ldp, i0, nrow, r, X, ld);
    else load_rows(a.Lc, false, I, i0, nrow, r, X, ld);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < nrow * a.ncp; e += blockDim.x) {
      const uint32_t row = e / a.ncp, c = e % a.ncp;
      double s = 0.0;
      if (c < r)
        for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], M[k * r + c], s);
      a.Mt[uint64_t(i0 + row) * a.ncp + c] = s;
    }
    __syncthreads();
  }
  PHASE(26);
}

// ---- finish_step -----------------------------------------------------------------
constexpr int kFinRows = 64;    // rows of R per block of the row pass
constexpr int kFinStages = 3;   // ring depth of the row pass
constexpr int kFinPerSm = 2;    // resident CTAs per SM (grid of the row pass)

// Residual, stop rule and G_R^{-1} from the reduced Gram G (shared memory,
// column-major r x r), on one CTA; Gi: r*r shared scratch.
template <int NC>
__device__ void finish_tail(const FinishArgs& a, double* G, double* Gi, double* scratch = nullptr, int avail = 0) {
  AlsCtrl* ctrl = a.ctrl;
  const uint32_t r = a.r;
  __shared__ double hi_s[32], lo_s[32];
  if (threadIdx.x < 32) {
    // compensated trace(G_L G_R) (als.cpp:136-141)
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
    // graph mode: a device-side trip guard on top of the max_iters rule
    if (a.cond && ++ctrl->trips > ctrl->max_iters + 1) cont = 0;
    cont_s = cont;
    if (!cont) ctrl->stop = 1;
    if (a.cond) cudaGraphSetConditional(a.cond, cont ? 1u : 0u);
  }
  __syncthreads();
  if (!cont_s) return;
  double piv = 0.0;
  const int fail = spd_inverse<ke_for(NC)>(G, Gi, r, 1e-13, &piv, scratch, avail);
  if (fail) {
    if (threadIdx.x == 0) {
      ctrl->error = kAlsErrLeftSingular;
      ctrl->pivot = piv;
      ctrl->pad = fail;  // failing column (1-based)
      ctrl->stop = 1;
      if (a.cond) cudaGraphSetConditional(a.cond, 0u);
    }
    return;
  }
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.GRinv[e] = Gi[e];
}

template <int NC>
__global__ void __launch_bounds__(kThreads, kFinPerSm) finish_step_kernel(FinishArgs a) {
  cg::grid_group grid = cg::this_grid();
  AlsCtrl* ctrl = a.ctrl;
  if (ctrl->stop) {
    if (a.cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0u);
    return;
  }
  constexpr int kRows = kFinRows, kLd = NC + 4, kNT = NC / 8, kTri = kNT * (kNT + 1) / 2, kStg = kFinStages;
  extern __shared__ __align__(16) double sm[];
  double* tile = sm;  // [kStg][kRows][kLd]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  const uint32_t r = a.r;

  // Phase 1 (R^T R not fused into FC): Gram partial of the CTA's contiguous
  // row range of R (row-major [F][ld]), streamed in kFinRows-row blocks through a
  // kStg-deep cp.async ring into padded rows (kLd = NC + 4: conflict-free
  // fragment loads); each thread copies one 16-byte column chunk of every
  // kRpp-th row. Each warp takes kKs consecutive k-steps (4 rows each) of
  // every block and accumulates ALL upper 8x8 tiles for them,
  // loading each column tile's fragment once per k-step (kNT loads for kTri
  // DMMAs); the 8 warp partials are summed in a fixed order.
  if (a.gram_nparts == 0 && a.mode != 2) {
    // copy map: kRpp rows of kCpr 16-byte chunks per pass of the CTA
    constexpr int kCpr = NC / 2, kRpp = kThreads / kCpr, kPasses = (kRows + kRpp - 1) / kRpp;
    // the upper 8x8 tiles are dealt to kSets warp sets (tile idx mod kSets):
    // warp w accumulates set w % kSets over the k-steps of warp group w / kSets
    constexpr int kSets = kTri >= 2 ? 2 : 1, kTriS = (kTri + kSets - 1) / kSets;
    constexpr int kGroups = kThreads / 32 / kSets, kKs = kRows / 4 / kGroups;
    const int set = warp % kSets, group = warp / kSets;
    double acc[kTriS][2];
#pragma unroll
    for (int k = 0; k < kTriS; ++k) acc[k][0] = acc[k][1] = 0.0;
    const uint64_t nblk = (a.F + kRows - 1) / kRows;
    const uint64_t per = (nblk + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    const int crow = threadIdx.x < kRpp * kCpr ? int(threadIdx.x) / kCpr : kRows;
    const int ccol = (int(threadIdx.x) % kCpr) * 2;
    const uint32_t goff = uint32_t(crow) * uint32_t(a.ld) + ccol, gstep = uint32_t(kRpp) * uint32_t(a.ld);
    const int soff = crow * kLd + ccol;
    auto issue = [&](uint64_t b, int slot) {
      double* t = tile + size_t(slot) * kRows * kLd + soff;
      const double* g = a.R + b * kRows * a.ld + goff;
      const uint64_t left = a.F - b * kRows;
      if (left >= uint64_t(kRows)) {
#pragma unroll
        for (int j = 0; j < kPasses; ++j)
          if (crow + j * kRpp < kRows) cp_async16(t + j * kRpp * kLd, g + j * gstep);
      } else {
#pragma unroll
        for (int j = 0; j < kPasses; ++j) {
          const int row = crow + j * kRpp;
          if (row >= kRows) continue;
          if (uint64_t(row) < left) {
            cp_async16(t + j * kRpp * kLd, g + j * gstep);
          } else {
            t[j * kRpp * kLd] = 0.0;
            t[j * kRpp * kLd + 1] = 0.0;
          }
        }
      }
    };
#pragma unroll
    for (int i = 0; i < kStg - 1; ++i) {
      if (b0 + i < b1) issue(b0 + i, i);
      cp_async_commit();
    }
    for (uint64_t b = b0; b < b1; ++b) {
      cp_async_wait<kStg - 2>();
      __syncthreads();  // block b landed everywhere; slot (b-1) is free
      const int slot = int((b - b0) % kStg);
      if (b + kStg - 1 < b1) issue(b + kStg - 1, int((b - b0 + kStg - 1) % kStg));
      cp_async_commit();
      const double* t = tile + size_t(slot) * kRows * kLd;
      // TAIL: the last column tile holds 1-2 real columns (r mod 8 in {1, 2});
      // its kNT tiles (tm, kNT-1) are each lane's own-row products with those
      // two values (DFMA, summed over the 4 k lanes after the pass) instead of
      // DMMA tiles that are three quarters padding
      auto steps = [&](auto S, auto T) {
        constexpr int sset = decltype(S)::value;
        constexpr bool kTail = decltype(T)::value;
#pragma unroll
        for (int ks = 0; ks < kKs; ++ks) {
          const double* rp = t + ((group * kKs + ks) * 4 + q) * kLd;
          double fr[kNT];
#pragma unroll
          for (int c = 0; c < kNT; ++c) fr[c] = rp[c * 8 + r8];
          double2 tv = make_double2(0.0, 0.0);
          if (kTail) tv = *reinterpret_cast<const double2*>(rp + (kNT - 1) * 8);
          int idx = 0;
#pragma unroll
          for (int tm = 0; tm < kNT; ++tm)
#pragma unroll
            for (int tn = tm; tn < kNT; ++tn, ++idx)
              if (idx % kSets == sset) {
                if (kTail && tn == kNT - 1) {
                  acc[idx / kSets][0] = fma(fr[tm], tv.x, acc[idx / kSets][0]);
                  acc[idx / kSets][1] = fma(fr[tm], tv.y, acc[idx / kSets][1]);
                } else {
                  dmma(acc[idx / kSets][0], acc[idx / kSets][1], fr[tm], fr[tn]);
                }
              }
        }
      };
      using std::integral_constant;
      if (a.gram_tail && kNT > 1) {
        if (kSets == 2 && set == 1) steps(integral_constant<int, 1>{}, integral_constant<bool, true>{});
        else steps(integral_constant<int, 0>{}, integral_constant<bool, true>{});
      } else {
        if (kSets == 2 && set == 1) steps(integral_constant<int, 1>{}, integral_constant<bool, false>{});
        else steps(integral_constant<int, 0>{}, integral_constant<bool, false>{});
      }
    }
    if (a.gram_tail && kNT > 1) {
      // the tail tiles in accumulator-tile layout: lane (r8, q = 0) holds columns 0, 1
      int idx = 0;
#pragma unroll
      for (int tm = 0; tm < kNT; ++tm)
#pragma unroll
        for (int tn = tm; tn < kNT; ++tn, ++idx)
          if (tn == kNT - 1 && idx % kSets == set) {
            double v0 = acc[idx / kSets][0], v1 = acc[idx / kSets][1];
            v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
            v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
            v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
            v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
            acc[idx / kSets][0] = q == 0 ? v0 : 0.0;
            acc[idx / kSets][1] = q == 0 ? v1 : 0.0;
          }
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring is free: the warp partials are summed there, warp 0 first
    double* ws = tile;
    for (int w = 0; w < int(kThreads / 32); ++w) {
      if (warp == w) {
#pragma unroll
        for (int k = 0; k < kTriS; ++k) {
          const int idx = k * kSets + set;
          if (idx >= kTri) continue;
          double* p = ws + idx * 64 + lane * 2;
          p[0] = w < kSets ? acc[k][0] : p[0] + acc[k][0];
          p[1] = w < kSets ? acc[k][1] : p[1] + acc[k][1];
        }
      }
      __syncthreads();
    }
    double* out = a.gpart + size_t(blockIdx.x) * NC * NC;
    for (int e = threadIdx.x; e < kTri * 64; e += blockDim.x) {
      const double sum = ws[e];
      const int tt = e / 64, l = (e % 64) / 2, el = e % 2;
      int tm = 0, rem = tt;
      while (rem >= kNT - tm) {
        rem -= kNT - tm;
        ++tm;
      }
      const int tn = tm + rem;
      out[(tm * 8 + (l >> 2)) * NC + tn * 8 + 2 * (l & 3) + el] = sum;
    }
    if (a.mode == 1) return;
    grid.sync();
  }
  if (a.mode != 2) {
    reduce_gram_grid(a.gpart, a.gram_nparts ? a.gram_nparts : int(gridDim.x), uint64_t(NC) * NC, NC, r,
                     a.gs);
    grid.sync();
  }
  if (blockIdx.x != 0) return;

  // Phase 2 (CTA 0): residual, stop rule, G_R^{-1}
  double* G = sm;
  double* Gi = G + r * r;
  __syncthreads();
  load_mat(a.gs, G, r * r);
  finish_tail<NC>(a, G, Gi);
}

// ---- cholqr_step -------------------------------------------------------------------
template <int KE>
__global__ void __launch_bounds__(kThreads) cholqr_step_kernel(CholQrArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1, I = a.I;
  double* X = sm;                 // [kRB][ld]
  double* X2 = X + kRB * ld;      // [kRB][ld]
  double* M = X2 + kRB * ld;      // r*r
  double* W = M + r * r;          // r*r
  double* W2 = W + r * r;         // r*r
  const uint32_t nblk = (I + kRB - 1) / kRB;
  const bool rm = a.nparts > 0;   // Y as row-major partials (summed into slot 0)
  PHASE(0);

  // Phase 1: Y rows, Gram partial
  if (a.nparts > 1) {
    reduce_partials_grid(a.Y, a.nparts, I, uint32_t(a.ldp), r);
    grid.sync();
  }
  PHASE(1);
  GramAcc g;
  g.zero();
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const uint32_t i0 = b * kRB, nrow = min(uint32_t(kRB), I - i0);
    load_rows(a.Y, rm, a.ldp, i0, nrow, r, X, ld);
    __syncthreads();
    g.add(X, nrow, r, ld);
    __syncthreads();
  }
  g.store(a.gpart + size_t(blockIdx.x) * r * r, r);
  grid.sync();
  PHASE(2);
  reduce_gram_grid(a.gpart, gridDim.x, uint64_t(r) * r, r, r, a.gs);
  grid.sync();
  PHASE(3);
  // Phase 2 (CTA 0): chol (no floor), R1^{-1} = (L1^{-1})^T
  double* SC = sm + rows_base(int(r));
  const int SCn = scratch_for(int(r), rows_base(int(r)));
  if (blockIdx.x == 0) {
    load_mat(a.gs, M, r * r);
    const int fail = chol_and_inverse<KE>(M, W, W2, r, SC, SCn);  // L1, L1^{-1} (lower)
    PHASE(4);
    if (threadIdx.x == 0) a.work[0] = fail;
    if (!fail) {
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.L1[e] = W[e];
      PHASE(5);
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.Rinv[e] = W2[e];
    }
  }
  grid.sync();
  PHASE(6);
  const int fail1 = int(a.work[0]);
  if (!fail1) {
    // Phase 3: Q1 rows = Y rows R1^{-1} (into Q), Gram partial of Q1;
    // R1^{-1}(k, c) = L1^{-1}(c, k), i.e. the row-major operand is Rinv itself
    load_mat(a.Rinv, M, r * r);
    g.zero();
    for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
      const uint32_t i0 = b * kRB, nrow = min(uint32_t(kRB), I - i0);
      load_rows(a.Y, rm, a.ldp, i0, nrow, r, X, ld);
      __syncthreads();
      rows_mul(X, nrow, r, ld, M, X2, ld);
      __syncthreads();
      store_rows_cm(X2, ld, i0, nrow, r, a.Q, I);
      g.add(X2, nrow, r, ld);
      __syncthreads();
    }
    g.store(a.gpart + size_t(blockIdx.x) * r * r, r);
    grid.sync();
    PHASE(7);
    reduce_gram_grid(a.gpart, gridDim.x, uint64_t(r) * r, r, r, a.gs);
  }
  grid.sync();
  PHASE(8);
  // Phase 4 (CTA 0): second factorization, R = R2 R1, degeneracy
  if (blockIdx.x == 0) {
    int fail = fail1;
    if (!fail) {
      load_mat(a.gs, M, r * r);
      fail = chol_and_inverse<KE>(M, W, W2, r, SC, SCn);  // L2, L2^{-1}
      PHASE(9);
    }
    if (!fail) {
      PHASE(10);
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
  PHASE(11);
  if (a.work[1] != 0.0 || fail1) return;
  // Phase 5: Q rows = Q1 rows R2^{-1} (row-major operand = Rinv, as above)
  load_mat(a.Rinv, M, r * r);
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const uint32_t i0 = b * kRB, nrow = min(uint32_t(kRB), I - i0);
    load_rows(a.Q, false, I, i0, nrow, r, X, ld);
    __syncthreads();
    rows_mul(X, nrow, r, ld, M, X2, ld);
    __syncthreads();
    store_rows_cm(X2, ld, i0, nrow, r, a.Q, I);
    __syncthreads();
  }
  PHASE(12);
}

// part[0][i][c] = sum_k part[k][i][c] (c < r) over the whole grid, 8 lanes per
// entry (k = lane, lane + 8, ... ascending, four loads in flight per lane) and
// a fixed xor tree: the split-K reduction that precedes a cluster prep.
// Returns at once when the sweep is past the stop decision.
__global__ void __launch_bounds__(256) slot0_reduce_kernel(double* part, int nparts, uint32_t I, uint32_t ldp,
                                                          uint32_t r, const AlsCtrl* ctrl) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (ctrl && ctrl->stop) return;
  const uint64_t n = uint64_t(I) * r;
  const uint64_t e = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  const bool act = e < n;
  double s = 0.0;
  double* p = nullptr;
  if (act) {
    p = part + (e / r) * ldp + (e % r);
    const uint64_t stride = uint64_t(I) * ldp;
    int k = sub;
    for (; k + 24 < nparts; k += 32) {
      const double v0 = __ldcg(p + size_t(k) * stride), v1 = __ldcg(p + size_t(k + 8) * stride);
      const double v2 = __ldcg(p + size_t(k + 16) * stride), v3 = __ldcg(p + size_t(k + 24) * stride);
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; k < nparts; k += 8) s += __ldcg(p + size_t(k) * stride);
  }
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (act && sub == 0) p[0] = s;
}

// ---- cluster steps ---------------------------------------------------------------------
// The same three steps as ONE thread-block cluster (up to 16 CTAs, one per
// SM) instead of a grid-synchronised launch over every SM. CTA q of the
// cluster owns the contiguous factor rows [q*rb, (q+1)*rb), rb = ceil(I/cs),
// and keeps them through every phase; the per-CTA Gram partials live in
// shared memory and every CTA sums all cs of them over DSMEM in the same
// fixed order, so each CTA holds bit-identical r x r Gram matrices and runs
// the r x r factorization itself: no broadcast phase and no grid-wide
// barrier, a step costs 1-4 cluster barriers. The split-K FR partials are
// summed row-block by row-block straight into shared memory (fixed k
// order). Launched with programmatic stream serialization: griddepcontrol.wait
// orders the first dependent read after the preceding kernel's writes while
// the launch itself overlaps that kernel's tail.

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// X[row][c] (pitch ld) = sum_{k < nparts} part[k*stride + (i0+row)*ldp + c],
// k ascending; up to 16 loads per thread in flight.
__device__ void sum_rows(const double* part, int nparts, uint64_t stride, uint32_t ldp, uint32_t i0,
                         uint32_t nrow, uint32_t r, double* X, uint32_t ld) {
  for (uint32_t e = threadIdx.x; e < nrow * r; e += blockDim.x) {
    const uint32_t row = e / r, c = e % r;
    const double* p = part + uint64_t(i0 + row) * ldp + c;
    double s = 0.0;
    int k = 0;
    for (; k + 16 <= nparts; k += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(p + uint64_t(k + u) * stride);
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    for (; k < nparts; ++k) s += __ldcg(p + uint64_t(k) * stride);
    X[row * ld + c] = s;
  }
}

// G (column-major, symmetric) = sum over the cluster's CTAs q = 0..cs-1 of
// their Gram partials gp (GramAcc layout: entry a*r + b, a <= b), read over
// DSMEM in ascending q.
__device__ void cluster_gram_sum(cg::cluster_group& cl, double* gp, uint32_t r, double* G) {
  const uint32_t cs = cl.num_blocks();
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
    const uint32_t a = e / r, b = e % r;
    if (a > b) continue;
    double s = 0.0;
    for (uint32_t q = 0; q < cs; ++q) s += cl.map_shared_rank(gp, q)[e];
    G[a + b * r] = s;
    G[b + a * r] = s;
  }
}

__device__ __forceinline__ void cta_rows(uint32_t I, uint32_t q, uint32_t cs, uint32_t& lo, uint32_t& hi) {
  const uint32_t rb = (I + cs - 1) / cs;
  lo = min(I, q * rb);
  hi = min(I, lo + rb);
}

template <int KE>
__global__ void __launch_bounds__(kThreads) prep_cluster_kernel(PrepArgs a) {
  pdl_wait();
  PHASE(30);
  cg::cluster_group cl = cg::this_cluster();
  AlsCtrl* ctrl = a.ctrl;
  if (ctrl->stop) return;  // uniform over the cluster (written by earlier kernels only)
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1, I = a.I;
  double* X = sm;               // [kRB][ld]
  double* X2 = X + kRB * ld;    // [kRB][ld]
  double* M = X2 + kRB * ld;    // r*r
  double* G = M + r * r;        // r*r
  double* W = G + r * r;        // r*r
  double* gp = W + r * r;       // r*r (read by the whole cluster)
  uint32_t lo, hi;
  cta_rows(I, cl.block_rank(), cl.num_blocks(), lo, hi);

  // L rows (from partials: Y G_R^{-1}) and their Gram partial
  if (a.from_partials) load_mat_rm(a.GRinv, M, r);
  GramAcc g;
  g.zero();
  for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
    const uint32_t nrow = min(uint32_t(kRB), hi - i0);
    if (a.from_partials) {
      sum_rows(a.part, a.nparts, uint64_t(I) * a.ldp, a.ldp, i0, nrow, r, X, ld);
      __syncthreads();
      rows_mul(X, nrow, r, ld, M, X2, ld);
      __syncthreads();
      store_rows_cm(X2, ld, i0, nrow, r, a.Lc, I);
    } else {
      load_rows(a.Lc, false, I, i0, nrow, r, X2, ld);
      __syncthreads();
    }
    g.add(X2, nrow, r, ld);
    __syncthreads();
  }
  PHASE(31);
  g.store(gp, r);
  cl.sync();
  cluster_gram_sum(cl, gp, r, G);
  cl.sync();  // every remote read of gp is done (CTAs may exit from here on)
  PHASE(32);

  // G_L^{-1} with the spd_solve pivot floor, in every CTA (identical bits)
  double piv = 0.0;
  const int fail = spd_inverse<KE>(G, W, r, 1e-13, &piv, sm + prep_cluster_base(int(r)),
                                   scratch_for(int(r), prep_cluster_base(int(r))));
  PHASE(33);
  if (fail) {
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      ctrl->error = kAlsErrRightSingular;
      ctrl->pivot = piv;
      ctrl->pad = fail;  // failing column (1-based)
      ctrl->stop = 1;
    }
    return;
  }
  if (cl.block_rank() == 0)
    for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
      a.GL[e] = G[e];
      a.GLinv[e] = W[e];
    }
  // Mt rows = L rows G_L^{-1} (row-major operand of the column-major inverse)
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) M[e] = W[(e / r) + (e % r) * r];
  __syncthreads();
  for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
    const uint32_t nrow = min(uint32_t(kRB), hi - i0);
    load_rows(a.Lc, false, I, i0, nrow, r, X, ld);  // this CTA's own rows (written above)
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < nrow * a.ncp; e += blockDim.x) {
      const uint32_t row = e / a.ncp, c = e % a.ncp;
      double s = 0.0;
      if (c < r)
        for (uint32_t k = 0; k < r; ++k) s = fma(X[row * ld + k], M[k * r + c], s);
      a.Mt[uint64_t(i0 + row) * a.ncp + c] = s;
    }
    __syncthreads();
  }
  PHASE(34);
}

// finish: G_R = sum of the Gram partials (RᵀR per FC CTA, or per row-pass
// CTA) split over the cluster's warps, each entry written into CTA 0's
// shared memory; CTA 0 then runs the residual / stop rule / G_R^{-1} of
// finish_step_kernel. mode 2 (sharded): G_R already reduced in gs, one CTA.
template <int NC>
__global__ void __launch_bounds__(kThreads) finish_cluster_kernel(FinishArgs a) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  if (a.ctrl->stop) {
    if (a.cond && cl.block_rank() == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0u);
    return;
  }
  extern __shared__ __align__(16) double sm[];
  const uint32_t r = a.r;
  double* G = sm;
  double* Gi = G + r * r;
  if (a.mode == 2) {
    load_mat(a.gs, G, r * r);
  } else {
    const uint32_t wpb = blockDim.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nw = cl.num_blocks() * wpb;
    const uint32_t ntri = r * (r + 1) / 2;
    double* G0 = cl.map_shared_rank(G, 0);
    for (uint32_t t = cl.block_rank() * wpb + (threadIdx.x >> 5); t < ntri; t += nw) {
      uint32_t aa = 0, rem = t;
      while (rem >= r - aa) {
        rem -= r - aa;
        ++aa;
      }
      const uint32_t b = aa + rem;
      const double* p = a.gpart + size_t(aa) * NC + b;
      double s = 0.0;
      for (int k = int(lane); k < a.gram_nparts; k += 32) s += __ldcg(p + size_t(k) * NC * NC);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) {
        G0[aa + b * r] = s;
        G0[b + aa * r] = s;
      }
    }
    cl.sync();
    if (cl.block_rank() != 0) return;
    if (a.gs)
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) a.gs[e] = G[e];
  }
  finish_tail<NC>(a, G, Gi, sm + finish_cluster_base(int(r)), scratch_for(int(r), finish_cluster_base(int(r))));
}

template <int KE>
__global__ void __launch_bounds__(kThreads) cholqr_cluster_kernel(CholQrArgs a) {
  pdl_wait();
  PHASE(40);
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  const uint32_t r = a.r, ld = r + 1, I = a.I;
  double* X = sm;               // [kRB][ld]
  double* X2 = X + kRB * ld;    // [kRB][ld]
  double* G = X2 + kRB * ld;    // r*r
  double* W = G + r * r;        // r*r  (L1, then L2)
  double* W2 = W + r * r;       // r*r  (L1^{-1}, then L2^{-1})
  double* L1 = W2 + r * r;      // r*r
  double* gp = L1 + r * r;      // r*r (read by the whole cluster)
  const bool rm = a.nparts > 0;  // Y as row-major partials, else column-major
  const bool lead = cl.block_rank() == 0;
  uint32_t lo, hi;
  cta_rows(I, cl.block_rank(), cl.num_blocks(), lo, hi);

  // Y rows (partials summed) -> Q as scratch, Gram partial
  GramAcc g;
  g.zero();
  for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
    const uint32_t nrow = min(uint32_t(kRB), hi - i0);
    if (rm) sum_rows(a.Y, a.nparts, uint64_t(I) * a.ldp, uint32_t(a.ldp), i0, nrow, r, X, ld);
    else load_rows(a.Y, false, a.ldp, i0, nrow, r, X, ld);
    __syncthreads();
    store_rows_cm(X, ld, i0, nrow, r, a.Q, I);
    g.add(X, nrow, r, ld);
    __syncthreads();
  }
  PHASE(41);
  g.store(gp, r);
  cl.sync();
  cluster_gram_sum(cl, gp, r, G);
  PHASE(42);
  cl.sync();  // gp is free again
  double* SC = sm + cholqr_cluster_base(int(r));
  const int SCn = scratch_for(int(r), cholqr_cluster_base(int(r)));
  const int fail1 = chol_and_inverse<KE>(G, W, W2, r, SC, SCn);  // L1, L1^{-1}
  if (fail1) {
    if (lead && threadIdx.x == 0) {
      a.work[0] = fail1;
      a.work[1] = fail1;
      a.ctrl->degenerate_col = fail1;
    }
    return;
  }
  for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) L1[e] = W[e];
  __syncthreads();  // R1^{-1}(k, c) = L1^{-1}(c, k): the row-major operand is W2

  PHASE(43);
  // Q1 rows = Y rows R1^{-1} (in place in Q), Gram partial of Q1
  g.zero();
  for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
    const uint32_t nrow = min(uint32_t(kRB), hi - i0);
    load_rows(a.Q, false, I, i0, nrow, r, X, ld);
    __syncthreads();
    rows_mul(X, nrow, r, ld, W2, X2, ld);
    __syncthreads();
    store_rows_cm(X2, ld, i0, nrow, r, a.Q, I);
    g.add(X2, nrow, r, ld);
    __syncthreads();
  }
  PHASE(44);
  g.store(gp, r);
  cl.sync();
  cluster_gram_sum(cl, gp, r, G);
  PHASE(45);
  cl.sync();
  const int fail = chol_and_inverse<KE>(G, W, W2, r, SC, SCn);  // L2, L2^{-1}
  PHASE(46);
  if (lead) {
    // R = R2 R1 = L2^T L1^T, the degeneracy test on its diagonal (als.cpp:74-86)
    double* Rm = G;  // G is no longer needed
    __syncthreads();
    if (!fail) {
      for (uint32_t e = threadIdx.x; e < r * r; e += blockDim.x) {
        const uint32_t i = e % r, j = e / r;
        double acc = 0.0;
        if (i <= j)
          for (uint32_t k = i; k <= j; ++k) acc += W[k + i * r] * L1[j + k * r];
        Rm[e] = acc;
        if (a.rmat) a.rmat[e] = acc;
      }
      __syncthreads();
      if (a.rt)
        for (uint32_t e = threadIdx.x; e < r * a.ldrt; e += blockDim.x) {
          const uint32_t row = e / a.ldrt, c = e % a.ldrt;
          a.rt[e] = c < r ? Rm[c + row * r] : 0.0;
        }
    }
    if (threadIdx.x == 0) {
      int bad = fail;
      if (!fail && a.check) {
        double md = 0.0;
        for (uint32_t i = 0; i < r; ++i) md = fmax(md, fabs(Rm[i + i * r]));
        for (uint32_t i = 0; i < r; ++i)
          if (fabs(Rm[i + i * r]) <= 1e-13 * md || md == 0.0) {
            bad = int(i) + 1;
            break;
          }
      }
      a.ctrl->degenerate_col = bad;
      a.work[0] = 0;
      a.work[1] = fail;
    }
  }
  PHASE(47);
  if (fail) return;
  // Q rows = Q1 rows R2^{-1}
  for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
    const uint32_t nrow = min(uint32_t(kRB), hi - i0);
    load_rows(a.Q, false, I, i0, nrow, r, X, ld);
    __syncthreads();
    rows_mul(X, nrow, r, ld, W2, X2, ld);
    __syncthreads();
    store_rows_cm(X2, ld, i0, nrow, r, a.Q, I);
    __syncthreads();
  }
  PHASE(48);
}

template <class K>
// exact: the caller sized per-CTA partials for `want` CTAs (fail rather than
// launch fewer).
cudaError_t coop_launch(K kernel, int want, int num_sms, size_t smem, void* args, cudaStream_t st,
                        bool exact = false) {
  cudaError_t e = raise_smem_limit(kernel, smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (e != cudaSuccess || occ < 1 || (exact && occ * num_sms < want)) {
    cudaGetLastError();
    return e != cudaSuccess ? e : cudaErrorCooperativeLaunchTooLarge;
  }
  const int grid = std::max(1, std::min(want, occ * num_sms));
  void* params[] = {args};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kernel), dim3(grid), dim3(kThreads), params,
                                  smem, st);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

size_t rows_smem(uint32_t r) { return sizeof(double) * (rows_base(int(r)) + scratch_for(int(r), rows_base(int(r)))); }

// Cluster steps (TKG_COOP_STEPS=1 selects the grid-synchronised kernels).
bool use_grid_steps() {
  static const bool v = [] {
    const char* e = std::getenv("TKG_COOP_STEPS");
    return e != nullptr && e[0] == '1';
  }();
  return v;
}

constexpr uint32_t kClusterPrepMaxI = 1024;  // c3 (concurrent modes) 43.4 -> 43.0 ms; c4 at 2048 rows: slower
constexpr uint32_t kClusterQrMaxI = 512;
// prep (after the grid partial-sum kernel): the cluster kernel up to this many
// rows (TKG_CLUSTER_PREP_MAXI overrides; measured in DESIGN.md §15)
uint32_t cluster_prep_max_i() {
  static const uint32_t v = [] {
    const char* e = std::getenv("TKG_CLUSTER_PREP_MAXI");
    return e ? uint32_t(std::atoi(e)) : kClusterPrepMaxI;
  }();
  return v;
}

template <class K, class... Args>
cudaError_t pdl_launch(K kernel, int grid, int block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

// Largest cluster (16 non-portable, else 8, 4, 2, 1) that the kernel can
// place with `smem` bytes per CTA; cached per kernel and size.
template <class K>
int cluster_size(K kernel, size_t smem) {
  static std::mutex m;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> g(m);
  auto it = cache.find({reinterpret_cast<const void*>(kernel), smem});
  if (it != cache.end()) return it->second;
  int want = 16;
  if (const char* e = std::getenv("TKG_CLUSTER")) want = std::max(1, std::min(16, std::atoi(e)));
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    want = std::min(want, 8);
  }
  int cs = want;
  for (; cs > 1; cs /= 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) == cudaSuccess && n >= 1) break;
    cudaGetLastError();
  }
  cache[{reinterpret_cast<const void*>(kernel), smem}] = cs;
  return cs;
}

template <class K, class A>
cudaError_t cluster_launch(K kernel, int cs, size_t smem, const A& args, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

template <class K, class A>
cudaError_t cluster_step(K kernel, size_t smem, const A& args, cudaStream_t st, int cs_max = 16) {
  cudaError_t e = raise_smem_limit(kernel, smem);
  if (e != cudaSuccess) return e;
  return cluster_launch(kernel, std::min(cs_max, cluster_size(kernel, smem)), smem, args, st);
}

size_t prep_cluster_smem(uint32_t r) {
  return sizeof(double) * (prep_cluster_base(int(r)) + scratch_for(int(r), prep_cluster_base(int(r))));
}
size_t cholqr_cluster_smem(uint32_t r) {
  return sizeof(double) * (cholqr_cluster_base(int(r)) + scratch_for(int(r), cholqr_cluster_base(int(r))));
}

}  // namespace

int coop_partials_cap(int num_sms) { return num_sms * (2048 / kThreads); }

int finish_step_grid(uint64_t F, int num_sms) {
  return int(std::max<uint64_t>(1, std::min<uint64_t>((F + kFinRows - 1) / kFinRows, uint64_t(kFinPerSm) * num_sms)));
}

#define TKG_KE_SWITCH(r, CALL) \
  if ((r) <= 16) return CALL(1); \
  if ((r) <= 32) return CALL(4); \
  if ((r) <= 48) return CALL(9); \
  return CALL(16);

cudaError_t launch_prep_step(PrepArgs a, int num_sms, cudaStream_t st) {
  // Factors of up to 512 rows: the split-K partials are summed by a full-grid
  // kernel (summing them on 16 SMs is latency-bound), then one cluster runs
  // the rest of the step; taller factors keep the grid-synchronised kernel
  // (tools/small_bench.cu).
  if (!use_grid_steps() && a.I <= cluster_prep_max_i()) {
    if (a.from_partials && a.nparts > 1) {
      const uint64_t threads = uint64_t(a.I) * a.r * 8;
      cudaError_t e = pdl_launch(slot0_reduce_kernel, int((threads + 255) / 256), 256, st, a.part, a.nparts, a.I,
                                 a.ldp, a.r, static_cast<const AlsCtrl*>(a.ctrl));
      if (e != cudaSuccess) return e;
      a.nparts = 1;
    }
#define TKG_PC(KE) cluster_step(prep_cluster_kernel<KE>, prep_cluster_smem(a.r), a, st)
    TKG_KE_SWITCH(a.r, TKG_PC)
#undef TKG_PC
  }
#define TKG_P(KE) coop_launch(prep_step_kernel<KE>, num_sms, num_sms, rows_smem(a.r), &a, st)
  TKG_KE_SWITCH(a.r, TKG_P)
#undef TKG_P
}

cudaError_t launch_finish_step(FinishArgs a, int num_sms, cudaStream_t st) {
  a.gram_tail = dfma_tail(a.r) ? 1 : 0;
  const uint32_t ntri = a.r * (a.r + 1) / 2;
  const int want = a.mode == 2 ? 1
                   : a.gram_nparts ? int(std::min<uint32_t>(uint32_t(num_sms), (ntri + 7) / 8))
                                   : finish_step_grid(a.F, num_sms);
  const uint32_t ncp = a.r <= 8 ? 8 : (a.r + 7) / 8 * 8;
  const size_t smem = sizeof(double) * std::max<size_t>(size_t(kFinStages) * kFinRows * (ncp + 4), 2 * size_t(a.r) * a.r);
  if (!use_grid_steps() && a.mode != 1) {
    // the R^T R row pass (r > 32) stays a full-grid launch writing per-CTA
    // partials; the reduction and the CTA-0 tail run as one cluster
    FinishArgs c = a;
    if (a.mode == 0 && a.gram_nparts == 0) {
      c.mode = 1;
      const cudaError_t e = launch_finish_step(c, num_sms, st);
      if (e != cudaSuccess) return e;
      c.mode = 0;
      c.gram_nparts = want;
    }
    const size_t csm =
        sizeof(double) * (finish_cluster_base(int(a.r)) + scratch_for(int(a.r), finish_cluster_base(int(a.r))));
    switch (ncp) {
#define TKG_FC(N) \
  case N: return cluster_step(finish_cluster_kernel<N>, csm, c, st, c.mode == 2 ? 1 : 16);
      TKG_FC(8) TKG_FC(16) TKG_FC(24) TKG_FC(32) TKG_FC(40) TKG_FC(48) TKG_FC(56) TKG_FC(64)
#undef TKG_FC
      default: return cudaErrorInvalidValue;
    }
  }
  switch (ncp) {
#define TKG_F(N) \
  case N: return coop_launch(finish_step_kernel<N>, want, num_sms, smem, &a, st, a.mode == 1);
    TKG_F(8) TKG_F(16) TKG_F(24) TKG_F(32) TKG_F(40) TKG_F(48) TKG_F(56) TKG_F(64)
#undef TKG_F
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_cholqr_step(CholQrArgs a, int num_sms, cudaStream_t st) {
  // cluster CholQR2 while a CTA's rows fit one 32-row block (I <= 512), after
  // a full-grid sum of the split-K partials; taller factors stream more rows
  // per SM than 16 SMs sustain
  if (!use_grid_steps() && a.I <= kClusterQrMaxI) {
    if (a.nparts > 1) {  // no stop check: the initializer runs before ctrl_init
      const uint64_t threads = uint64_t(a.I) * a.r * 8;
      cudaError_t e = pdl_launch(slot0_reduce_kernel, int((threads + 255) / 256), 256, st, a.Y, a.nparts, a.I,
                                 uint32_t(a.ldp), a.r, static_cast<const AlsCtrl*>(nullptr));
      if (e != cudaSuccess) return e;
      a.nparts = 1;
    }
#define TKG_QC(KE) cluster_step(cholqr_cluster_kernel<KE>, cholqr_cluster_smem(a.r), a, st)
    TKG_KE_SWITCH(a.r, TKG_QC)
#undef TKG_QC
  }
#define TKG_Q(KE) coop_launch(cholqr_step_kernel<KE>, num_sms, num_sms, rows_smem(a.r), &a, st)
  TKG_KE_SWITCH(a.r, TKG_Q)
#undef TKG_Q
}

#ifdef TKG_PHASE_TIMING
void phase_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_phase_ns, sizeof(g_phase_ns)); }
#endif

}  // namespace tkg
