// Dense symmetric eigensolver on the device for the EIG / SVD factor engines
// and HOOI (reference sym_eig, kernels.cpp:448-604: Householder
// tridiagonalization, implicit-shift QL, descending order, fix_column_signs).
// Only the k leading pairs are needed, so after the tridiagonalization the
// k largest eigenvalues come from Sturm-count multisection and their vectors
// from inverse iteration on the tridiagonal matrix (LAPACK dsyevx's route),
// then the Householder reflectors are applied to those k vectors in blocks.
//
//   tridiag_kernel   cooperative (one CTA per SM): for j = 0..n-3 the
//                    reflector of column j (every CTA forms it redundantly
//                    from the column it holds in shared memory), p = tau A v
//                    on the columns each CTA owns (c % grid == cta), ONE grid
//                    barrier, w = p - (tau/2)(p^T v) v, the rank-2 update of
//                    the owned columns, and (redundantly, in every CTA) the
//                    updated next column. The owner never writes column j+1
//                    in step j, so the one barrier per step suffices.
//   bisect_kernel    one warp per eigenvalue: 32-point multisection of the
//                    Gershgorin interval with Sturm counts.
//   inviter_kernel   one warp per cluster of close eigenvalues (gap <= 1e-3
//                    ||T||_1, dstein's ORTOL): LU with partial pivoting of
//                    T - lambda I, four solves, modified Gram-Schmidt
//                    against the cluster's earlier vectors.
//   backtransform    cooperative: 32 reflectors at a time as I - V T V^T
//                    (dlarft forward / columnwise), Z -= V (T (V^T Z)), two
//                    grid barriers per block.
//   sign_kernel      the largest-magnitude entry of every column positive
//                    (fix_column_signs, kernels.cpp:25-43).
// Every reduction runs in a fixed order (deterministic results).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "eig.hpp"

namespace cg = cooperative_groups;

namespace tkg {
namespace {

constexpr int kT = 256;      // threads per CTA
constexpr int kNB = 32;      // reflectors per back-transform block
constexpr int kCG = 16;      // owned columns a tridiagonalization pass sweeps at once

// Deterministic CTA-wide sum (identical bits in every CTA for identical
// inputs): per-thread partials in index order, xor tree per warp, warp
// results in order.
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
  __syncthreads();
  return s;
}

// Reflector of step j from col[j..n-1] (column j of the current matrix, in
// shared memory): v (v[j+1] = 1), returns tau; CTA 0 records V, tau, d, e.
__device__ double make_reflector(int j, int n, const double* col, double* v, double* red, double* V,
                                 double* tau, double* d, double* e) {
  const double alpha = col[j + 1];
  double part = 0.0;
  for (int i = j + 2 + threadIdx.x; i < n; i += blockDim.x) part += col[i] * col[i];
  const double sigma = block_sum(part, red);
  double t = 0.0, beta = alpha;
  if (sigma != 0.0) {
    const double mu = sqrt(alpha * alpha + sigma);
    beta = alpha <= 0.0 ? mu : -mu;
    t = (beta - alpha) / beta;
    const double sc = 1.0 / (alpha - beta);
    for (int i = j + 2 + threadIdx.x; i < n; i += blockDim.x) v[i] = col[i] * sc;
  } else {
    for (int i = j + 2 + threadIdx.x; i < n; i += blockDim.x) v[i] = 0.0;
  }
  if (threadIdx.x == 0) v[j + 1] = 1.0;
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) V[i + size_t(j) * n] = v[i];
    if (threadIdx.x == 0) {
      tau[j] = t;
      d[j] = col[j];
      e[j] = beta;
    }
  }
  return t;
}

// A (n x n, column-major, symmetric, both triangles) is destroyed. V column j
// holds v_j (rows j+1..n-1, v_j[j+1] = 1); d, e the tridiagonal matrix.
// Step j: after the grid barrier every CTA forms w_j from p_j, the updated
// column j+1 and the next reflector v_{j+1} (all redundantly, identical
// bits); then ONE pass over its owned columns c >= j+2 applies the rank-2
// update of step j and accumulates p_{j+1} = tau_{j+1} A22' v_{j+1} from the
// updated values (one read and one write of the trailing matrix per step).
// Column j+1 is never written in step j, so its global copy (last written in
// step j-1) is what every CTA reads after the barrier.
__global__ void __launch_bounds__(kT) tridiag_kernel(double* A, int n, double* V, double* tau, double* d,
                                                     double* e, double* pbuf) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* col = sm;        // [n]: current column (absolute rows)
  double* v = col + n;     // [n]: v_j
  double* w = v + n;       // [n]: w_j
  double* vn = w + n;      // [n]: v_{j+1}
  __shared__ double red[32];
  __shared__ double red2[(kT / 32) * kCG];
  const int G = gridDim.x, b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (n <= 2) {
    if (b == 0 && threadIdx.x == 0) {
      d[0] = A[0];
      if (n == 2) {
        d[1] = A[n + 1];
        e[0] = A[1];
      }
      e[n - 1] = 0.0;
    }
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) col[i] = A[i];
  __syncthreads();
  double t = make_reflector(0, n, col, v, red, V, tau, d, e);
  // p_0 = tau_0 A22 v_0 on the owned columns (c >= 1, rows >= 1)
  // (kCG owned columns swept at once, every load independent; fixed-order
  // reductions)
  auto reduce_store = [&](double* acc, int c0, double scale, double* p) {
#pragma unroll
    for (int q = 0; q < kCG; ++q) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    }
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < kCG; ++q) red2[warp * kCG + q] = acc[q];
    __syncthreads();
    if (threadIdx.x < kCG) {
      const int c = c0 + int(threadIdx.x) * G;
      double sum = 0.0;
      for (int i = 0; i < nw; ++i) sum += red2[i * kCG + threadIdx.x];
      if (c < n) p[c] = scale * sum;
    }
  };
  {
    const int first = 1 + ((b - 1) % G + G) % G;
    for (int c0 = first; c0 < n; c0 += kCG * G) {
      double acc[kCG];
#pragma unroll
      for (int q = 0; q < kCG; ++q) acc[q] = 0.0;
      for (int k = 1 + threadIdx.x; k < n; k += blockDim.x) {
        const double vk = v[k];
#pragma unroll
        for (int q = 0; q < kCG; ++q) {
          const int c = c0 + q * G;
          if (c < n) acc[q] = fma(A[size_t(c) * n + k], vk, acc[q]);
        }
      }
      reduce_store(acc, c0, t, pbuf);
    }
  }
  for (int j = 0; j + 2 < n; ++j) {
    grid.sync();
    const double* p = pbuf + size_t(j & 1) * n;
    // w_j = p_j - (tau_j/2)(p_j^T v_j) v_j
    double part = 0.0;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) part += __ldcg(p + i) * v[i];
    const double K = -0.5 * t * block_sum(part, red);
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) w[i] = __ldcg(p + i) + K * v[i];
    __syncthreads();
    // column j+1 after step j (rows j+1..n-1)
    {
      const double vj = v[j + 1], wj = w[j + 1];
      const double* aj = A + size_t(j + 1) * n;
      for (int k = j + 1 + threadIdx.x; k < n; k += blockDim.x) col[k] = __ldcg(aj + k) - (v[k] * wj + w[k] * vj);
    }
    __syncthreads();
    const bool more = j + 3 < n;  // a reflector for column j+1
    const double tn = more ? make_reflector(j + 1, n, col, vn, red, V, tau, d, e) : 0.0;
    // fused pass: update of step j on the owned columns c >= j+2, and p_{j+1}
    double* pn = pbuf + size_t((j + 1) & 1) * n;
    const int first = j + 2 + ((b - (j + 2)) % G + G) % G;
    for (int c0 = first; c0 < n; c0 += kCG * G) {
      double acc[kCG];
#pragma unroll
      for (int q = 0; q < kCG; ++q) acc[q] = 0.0;
      for (int k = j + 1 + threadIdx.x; k < n; k += blockDim.x) {
        const double vk = v[k], wk = w[k], vnk = (more && k >= j + 2) ? vn[k] : 0.0;
#pragma unroll
        for (int q = 0; q < kCG; ++q) {
          const int c = c0 + q * G;
          if (c < n) {
            double* a = A + size_t(c) * n + k;
            const double x = *a - (vk * w[c] + wk * v[c]);
            *a = x;
            acc[q] = fma(x, vnk, acc[q]);
            if (c == n - 1 && k == n - 1) d[n - 1] = x;  // its owner: final diagonal entry
          }
        }
      }
      if (more) reduce_store(acc, c0, tn, pn);
    }
    // v <- v_{j+1}
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) v[i] = more ? vn[i] : 0.0;
    t = tn;
    __syncthreads();
  }
  if (b == 0 && threadIdx.x == 0) {
    d[n - 2] = col[n - 2];
    e[n - 2] = col[n - 1];
    e[n - 1] = 0.0;
  }
}

// Number of eigenvalues of the tridiagonal (d, e2 = e^2) below x.
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// lambda[i] = (i+1)-th largest eigenvalue, i < k: one warp each.
__global__ void __launch_bounds__(kT) bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg,
                                                    int n, int k, double* lambda) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e2 = d + n;
  __shared__ double gl_s, gu_s, pm_s, at_s;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] = dg[i];
    e2[i] = i + 1 < n ? eg[i] * eg[i] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double r = (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < n ? fabs(eg[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pad = 2.0 * DBL_EPSILON * tnorm * n + DBL_MIN;
    gl_s = lo - pad;
    gu_s = hi + pad;
    pm_s = DBL_MIN * fmax(1.0, emax);
    at_s = DBL_EPSILON * tnorm;  // absolute accuracy of QL (eps ||T||)
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= k) return;
  const int target = n - 1 - i;  // 0-based ascending index
  double lo = gl_s, hi = gu_s;   // count(lo) <= target < count(hi)
  const double pivmin = pm_s;
  for (int it = 0; it < 64; ++it) {
    const double width = hi - lo;
    if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + fmin(at_s, 1e-3 * fmax(fabs(lo), fabs(hi))) + pivmin)
      break;
    const double x = lo + width * double(lane + 1) / 33.0;
    const int c = sturm_count(d, e2, n, x, pivmin);
    const unsigned le = __ballot_sync(0xffffffffu, c <= target);  // monotone in lane
    const int nle = __popc(le);
    const double nlo = nle == 0 ? lo : __shfl_sync(0xffffffffu, x, nle - 1);
    const double nhi = nle == 32 ? hi : __shfl_sync(0xffffffffu, x, nle);
    if (nlo == lo && nhi == hi) break;  // no representable progress
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) lambda[i] = 0.5 * (lo + hi);
}

// Eigenvectors of the tridiagonal for lambda[0..k) (descending): one warp
// per cluster, lane 0 runs the O(n) recurrences, the warp the vector ops.
// Z: n x k column-major; scratch: 5n doubles per warp.
__global__ void __launch_bounds__(kT) inviter_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                     int n, int k, const double* __restrict__ lambda, double* Z,
                                                     double* scratch) {
  const int lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c0 >= k) return;
  double tnorm = 0.0;  // ||T||_1
  for (int i = lane; i < n; i += 32)
    tnorm = fmax(tnorm, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tnorm = fmax(tnorm, __shfl_xor_sync(0xffffffffu, tnorm, off));
  const double ortol = 1e-3 * tnorm;
  if (c0 > 0 && lambda[c0 - 1] - lambda[c0] <= ortol) return;  // not the first of its cluster
  int c1 = c0 + 1;
  while (c1 < k && lambda[c1 - 1] - lambda[c1] <= ortol) ++c1;
  double* u = scratch + size_t(c0) * 5 * n;  // U diag, U super1, U super2, L multipliers, pivot flags
  double* u1 = u + n;
  double* u2 = u1 + n;
  double* lm = u2 + n;
  double* pv = lm + n;
  const double tiny = DBL_EPSILON * fmax(tnorm, DBL_MIN);
  double prev = 0.0;
  for (int c = c0; c < c1; ++c) {
    double lam = lambda[c];
    // separate coincident eigenvalues of a cluster (dstein's PERTOL)
    if (c > c0 && prev - lam < 10.0 * DBL_EPSILON * fabs(lam) + tiny) lam = prev - 10.0 * DBL_EPSILON * fabs(prev) - tiny;
    prev = lam;
    // LU with partial pivoting of T - lam I (dgttrf): rows i, i+1
    if (lane == 0) {
      double a = d[0] - lam, bsup = n > 1 ? e[0] : 0.0;
      for (int i = 0; i + 1 < n; ++i) {
        const double sub = e[i], dn = d[i + 1] - lam, sn = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(a) >= fabs(sub)) {  // no interchange
          const double a0 = fabs(a) < tiny ? (a < 0 ? -tiny : tiny) : a;
          const double l = sub / a0;
          u[i] = a0;
          u1[i] = bsup;
          u2[i] = 0.0;
          lm[i] = l;
          pv[i] = 0.0;
          a = dn - l * bsup;
          bsup = sn;
        } else {  // swap rows i and i+1
          const double l = a / sub;
          u[i] = sub;
          u1[i] = dn;
          u2[i] = sn;
          lm[i] = l;
          pv[i] = 1.0;
          a = bsup - l * dn;
          bsup = -l * sn;
        }
      }
      u[n - 1] = fabs(a) < tiny ? (a < 0 ? -tiny : tiny) : a;
    }
    __syncwarp();
    double* x = Z + size_t(c) * n;
    for (int i = lane; i < n; i += 32) {  // deterministic start vector in (-1, 1)
      uint64_t h = (uint64_t(i) + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t(c) + 7) * 0xC2B2AE3D27D4EB4Full;
      h ^= h >> 31;
      h *= 0xBF58476D1CE4E5B9ull;
      h ^= h >> 29;
      x[i] = double(int64_t(h >> 11) - (int64_t(1) << 52)) / double(int64_t(1) << 52);
    }
    __syncwarp();
    for (int it = 0; it < 4; ++it) {
      if (lane == 0) {
        // forward: apply the row interchanges and L
        for (int i = 0; i + 1 < n; ++i) {
          if (pv[i] != 0.0) {
            const double t = x[i];
            x[i] = x[i + 1];
            x[i + 1] = t - lm[i] * x[i];
          } else {
            x[i + 1] -= lm[i] * x[i];
          }
        }
        // back substitution with U (diag u, super u1, super2 u2)
        x[n - 1] /= u[n - 1];
        if (n > 1) x[n - 2] = (x[n - 2] - u1[n - 2] * x[n - 1]) / u[n - 2];
        for (int i = n - 3; i >= 0; --i) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / u[i];
      }
      __syncwarp();
      // modified Gram-Schmidt against the cluster's earlier vectors (twice)
      for (int pass = 0; pass < 2; ++pass)
        for (int q = c0; q < c; ++q) {
          const double* y = Z + size_t(q) * n;
          double s = 0.0;
          for (int i = lane; i < n; i += 32) s += y[i] * x[i];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          for (int i = lane; i < n; i += 32) x[i] -= s * y[i];
          __syncwarp();
        }
      // normalise (scale by the largest entry first: no overflow)
      double mx = 0.0;
      for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(x[i]));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
      double s = 0.0;
      for (int i = lane; i < n; i += 32) {
        x[i] *= inv;
        s += x[i] * x[i];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const double nr = 1.0 / sqrt(s);
      for (int i = lane; i < n; i += 32) x[i] *= nr;
      __syncwarp();
    }
  }
}

// Z (n x k) <- H_0 H_1 ... H_{n-3} Z in blocks of kNB reflectors, last block
// first. part: [grid][kNB*kNB + kNB*k]; sums: 2 x [kNB*kNB + kNB*k].
__global__ void __launch_bounds__(kT) backtransform_kernel(const double* __restrict__ V,
                                                           const double* __restrict__ tau, int n, int k,
                                                           double* Z, double* part, double* sums) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* S = sm;               // kNB x kNB (S[a + b*kNB] = v_a . v_b)
  double* T = S + kNB * kNB;    // kNB x kNB upper triangular
  double* W = T + kNB * kNB;    // kNB x k  (V^T Z, then T V^T Z)
  double* W2 = W + kNB * k;     // kNB x k
  const int G = gridDim.x, b = blockIdx.x;
  const int nent = kNB * kNB + kNB * k;
  const int nref = n - 2;
  if (nref <= 0) return;
  const int rows_per = (n + G - 1) / G;
  const int r0 = min(n, b * rows_per), r1 = min(n, r0 + rows_per);
  int blk = 0;
  for (int j0 = (nref - 1) / kNB * kNB; j0 >= 0; j0 -= kNB, ++blk) {
    const int nb = min(kNB, nref - j0);
    // per-CTA partials of V^T V and V^T Z over the owned rows
    double* pp = part + size_t(b) * nent;
    for (int ent = threadIdx.x; ent < nent; ent += blockDim.x) {
      double s = 0.0;
      if (ent < kNB * kNB) {
        const int a = ent % kNB, bb = ent / kNB;
        if (a < nb && bb < nb && a <= bb)
          for (int r = max(r0, j0 + bb + 1); r < r1; ++r)  // v_a, v_bb vanish above rows j+1
            s += V[r + size_t(j0 + a) * n] * V[r + size_t(j0 + bb) * n];
      } else {
        const int q = ent - kNB * kNB, a = q % kNB, c = q / kNB;
        if (a < nb)
          for (int r = max(r0, j0 + a + 1); r < r1; ++r) s += V[r + size_t(j0 + a) * n] * Z[r + size_t(c) * n];
      }
      pp[ent] = s;
    }
    grid.sync();
    double* sb = sums + size_t(blk & 1) * nent;
    for (int ent = b * blockDim.x + threadIdx.x; ent < nent; ent += G * blockDim.x) {
      double s = 0.0;
      for (int g = 0; g < G; ++g) s += __ldcg(part + size_t(g) * nent + ent);
      sb[ent] = s;
    }
    grid.sync();
    for (int ent = threadIdx.x; ent < nent; ent += blockDim.x) {
      const double x = __ldcg(sb + ent);
      if (ent < kNB * kNB) S[ent] = x;
      else W[ent - kNB * kNB] = x;
    }
    __syncthreads();
    // T (dlarft forward, columnwise): T[i][i] = tau_i, T[0:i, i] = -tau_i T[0:i,0:i] S[0:i, i]
    if (threadIdx.x < 32) {
      for (int e2 = threadIdx.x; e2 < kNB * kNB; e2 += 32) T[e2] = 0.0;
      __syncwarp();
      for (int i = 0; i < nb; ++i) {
        const double ti = tau[j0 + i];
        // column i: entries a < i, T[a][i] = -ti * sum_{c=a}^{i-1} T[a][c] S[c][i]
        double val = 0.0;
        const int a = threadIdx.x;
        if (a < i)
          for (int c = a; c < i; ++c) val += T[a + c * kNB] * S[c + i * kNB];
        __syncwarp();
        if (a < i) T[a + i * kNB] = -ti * val;
        if (a == 0) T[i + i * kNB] = ti;
        __syncwarp();
      }
    }
    __syncthreads();
    // W2 = T W
    for (int ent = threadIdx.x; ent < kNB * k; ent += blockDim.x) {
      const int a = ent % kNB, c = ent / kNB;
      double s = 0.0;
      for (int q = a; q < nb; ++q) s += T[a + q * kNB] * W[q + c * kNB];
      W2[ent] = s;
    }
    __syncthreads();
    // Z rows -= V rows W2
    for (int ent = threadIdx.x; ent < (r1 - r0) * k; ent += blockDim.x) {
      const int r = r0 + ent % (r1 - r0), c = ent / (r1 - r0);
      double s = 0.0;
      for (int a = 0; a < nb; ++a)
        if (r > j0 + a) s += V[r + size_t(j0 + a) * n] * W2[a + c * kNB];
      Z[r + size_t(c) * n] -= s;
    }
    __syncthreads();
  }
}

// U column c = sign * Z column c with its largest-magnitude entry (first on
// ties) made positive (fix_column_signs, kernels.cpp:25-43).
__global__ void __launch_bounds__(256) sign_kernel(const double* __restrict__ Z, int n, double* __restrict__ U) {
  __shared__ double bmag[256];
  __shared__ int bidx[256];
  const int c = blockIdx.x;
  const double* z = Z + size_t(c) * n;
  double best = -1.0;
  int arg = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double m = fabs(z[i]);
    if (m > best) {
      best = m;
      arg = i;
    }
  }
  bmag[threadIdx.x] = best;
  bidx[threadIdx.x] = arg;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (int(threadIdx.x) < off) {
      const double m2 = bmag[threadIdx.x + off];
      const int i2 = bidx[threadIdx.x + off];
      if (m2 > bmag[threadIdx.x] || (m2 == bmag[threadIdx.x] && i2 < bidx[threadIdx.x])) {
        bmag[threadIdx.x] = m2;
        bidx[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  const double sg = z[bidx[0]] >= 0.0 ? 1.0 : -1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) U[i + size_t(c) * n] = sg * z[i];
}

template <class K>
cudaError_t coop(K kernel, int want, size_t smem, void** args, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kT, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorCooperativeLaunchTooLarge;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(want, occ * sms));
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kernel), dim3(grid), dim3(kT), args, smem, st);
}

}  // namespace

SymEig::~SymEig() {
  if (work_) cudaFree(work_);
}

std::string SymEig::leading(double* G, int n, int k, double* U, double* vals, cudaStream_t st) {
  if (n <= 0 || k <= 0) return std::string();
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(sms, std::max(1, n));
  const size_t nn = size_t(n) * n;
  const size_t nent = size_t(kNB) * kNB + size_t(kNB) * k;
  const size_t need = nn + 6 * size_t(n) + 5 * size_t(n) * k + size_t(n) * k + size_t(grid) * nent + 2 * nent;
  if (need > work_n_) {
    if (work_) cudaFree(work_);
    work_ = nullptr;
    work_n_ = 0;
    if (cudaMalloc(&work_, need * sizeof(double)) != cudaSuccess) return "cudaMalloc (sym_eig work) failed";
    work_n_ = need;
  }
  double* w = static_cast<double*>(work_);
  double* V = w;
  double* tau = V + nn;
  double* d = tau + n;
  double* e = d + n;
  double* pbuf = e + n;          // 2n
  double* scratch = pbuf + 2 * size_t(n);
  double* Z = scratch + 5 * size_t(n) * k;
  double* part = Z + size_t(n) * k;
  double* sums = part + size_t(grid) * nent;
  cudaError_t err;
  {
    int nn_ = n;
    void* args[] = {&G, &nn_, &V, &tau, &d, &e, &pbuf};
    err = coop(tridiag_kernel, grid, 4 * size_t(n) * sizeof(double), args, st);
    if (err != cudaSuccess) return std::string("sym_eig: tridiagonalization launch failed: ") + cudaGetErrorString(err);
  }
  double* lam = vals;
  {
    const int wpb = kT / 32;
    const size_t smem = 2 * size_t(n) * sizeof(double);
    cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bisect_kernel<<<(k + wpb - 1) / wpb, kT, smem, st>>>(d, e, n, k, lam);
    inviter_kernel<<<(k + wpb - 1) / wpb, kT, 0, st>>>(d, e, n, k, lam, Z, scratch);
  }
  {
    int nn_ = n, kk = k;
    void* args[] = {&V, &tau, &nn_, &kk, &Z, &part, &sums};
    const size_t smem = (2 * size_t(kNB) * kNB + 2 * size_t(kNB) * k) * sizeof(double);
    err = coop(backtransform_kernel, grid, smem, args, st);
    if (err != cudaSuccess) return std::string("sym_eig: back-transform launch failed: ") + cudaGetErrorString(err);
  }
  sign_kernel<<<k, 256, 0, st>>>(Z, n, U);
  err = cudaGetLastError();
  if (err != cudaSuccess) return std::string("sym_eig: ") + cudaGetErrorString(err);
  return std::string();
}

}  // namespace tkg
