// mode_gram on the FP64 tensor pipe (reference tensor_ops.cpp:332-389):
//   G = A_(n) A_(n)^T = sum over fibers j of x_j x_j^T,   x_j = fiber j (K = I_n values)
// read straight from the tensor's natural layout (FiberView, no unfolding).
//
// The I_n x I_n result is tiled into 64 x 64 blocks; a CTA owns one block of
// the upper triangle (bi <= bc) and a contiguous fiber range (split-K), and
// streams 32-fiber chunks of the two 64-index column panels of the tensor
// through a 3-stage cp.async ring in shared memory. Each element loaded is
// used 64 times (2 x 64 flop per 8 bytes), so the kernel sits on the DMMA
// roof, not HBM. Per-(split, block) partials are summed in a fixed order by
// gram_tensor_reduce_kernel (deterministic, like the reference's
// chunk-ordered combine at :375-383) and mirrored into the lower triangle.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace tkg {

namespace {

constexpr int kGB = 64;          // output block edge
constexpr int kGC = 32;          // fibers per chunk (K of the block product)
constexpr int kGLd = kGB + 8;    // row stride: fragment rows 8 (mod 16) apart, conflict free
constexpr int kGStages = 3;
constexpr int kGThreads = 256;
constexpr int kGStageDoubles = 2 * kGC * kGLd;

__device__ __forceinline__ void block_of_pair(int pair, int nb, int& bi, int& bc) {
  int b = 0, rem = pair;
  while (rem >= nb - b) {
    rem -= nb - b;
    ++b;
  }
  bi = b;
  bc = b + rem;
}

// T[jj][ii] = X(fiber j0 + jj, index i0 + ii), zero outside the fiber range / extent.
__device__ __forceinline__ void gram_issue(const FiberView& v, uint64_t j0, uint64_t j1, uint32_t i0,
                                           double* T) {
  const uint32_t K = v.K;
  if (v.s == 1) {  // fibers contiguous: 64 consecutive indices per fiber
    const bool vec = (K % 2 == 0) && ((reinterpret_cast<uintptr_t>(v.base) & 15) == 0);
    if (vec) {
      for (int e = threadIdx.x; e < kGC * (kGB / 2); e += kGThreads) {
        const int jj = e / (kGB / 2), ii = (e % (kGB / 2)) * 2;
        const uint64_t j = j0 + jj;
        double* d = T + jj * kGLd + ii;
        if (j < j1 && i0 + ii + 1 < K) {
          cp_async16(d, v.base + j * v.is_p + (i0 + ii));
        } else {
          d[0] = (j < j1 && i0 + ii < K) ? v.base[j * v.is_p + i0 + ii] : 0.0;
          d[1] = 0.0;
        }
      }
      return;
    }
  }
  // generic: consecutive threads take consecutive fibers (contiguous inside a panel)
  for (int e = threadIdx.x; e < kGC * kGB; e += kGThreads) {
    const int ii = e / kGC, jj = e % kGC;
    const uint64_t j = j0 + jj;
    double* d = T + jj * kGLd + ii;
    if (j < j1 && i0 + ii < K) {
      const uint64_t p = j / v.s, jl = j - p * v.s;
      cp_async8(d, v.base + jl + uint64_t(i0 + ii) * v.is_i + p * v.is_p);
    } else {
      *d = 0.0;
    }
  }
}

__global__ void __launch_bounds__(kGThreads, 1) gram_tensor_kernel(FiberView v, int nb, int npairs,
                                                                     uint64_t per_split, double* part) {
  extern __shared__ __align__(16) double sm[];
  const int pair = int(blockIdx.x % unsigned(npairs));
  const uint64_t split = blockIdx.x / unsigned(npairs);
  int bi, bc;
  block_of_pair(pair, nb, bi, bc);
  const bool diag = bi == bc;
  const uint64_t F = v.s * v.P;
  const uint64_t f0 = split * per_split, f1 = min(F, f0 + per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  const int wi = warp & 3, wc = warp >> 2;  // warp tile: 16 rows (i) x 32 columns (c)
  double acc[2][4][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

  const uint64_t nchunks = f1 > f0 ? (f1 - f0 + kGC - 1) / kGC : 0;
  auto issue = [&](uint64_t c, int slot) {
    double* Ti = sm + size_t(slot) * kGStageDoubles;
    const uint64_t j0 = f0 + c * kGC;
    gram_issue(v, j0, f1, uint32_t(bi * kGB), Ti);
    if (!diag) gram_issue(v, j0, f1, uint32_t(bc * kGB), Ti + kGC * kGLd);
  };
#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (uint64_t(s) < nchunks) issue(s, s);
    cp_async_commit();
  }
  for (uint64_t c = 0; c < nchunks; ++c) {
    cp_async_wait<kGStages - 2>();
    __syncthreads();
    if (c + kGStages - 1 < nchunks) issue(c + kGStages - 1, int((c + kGStages - 1) % kGStages));
    cp_async_commit();
    const double* Ti = sm + size_t(c % kGStages) * kGStageDoubles;
    const double* Tc = diag ? Ti : Ti + kGC * kGLd;
#pragma unroll
    for (int k0 = 0; k0 < kGC; k0 += 4) {
      const double* ri = Ti + (k0 + q) * kGLd;
      const double* rc = Tc + (k0 + q) * kGLd;
      double af[2], bf[4];
#pragma unroll
      for (int m = 0; m < 2; ++m) af[m] = ri[wi * 16 + m * 8 + r8];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = rc[wc * 32 + n * 8 + r8];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
  cp_async_wait<0>();
  double* out = part + (split * uint64_t(npairs) + uint64_t(pair)) * uint64_t(kGB * kGB);
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const int row = wi * 16 + m * 8 + r8, col = wc * 32 + n * 8 + 2 * q;
      out[row * kGB + col] = acc[m][n][0];
      out[row * kGB + col + 1] = acc[m][n][1];
    }
}

// G(i, c) (column-major K x K) = sum over splits, in order, of the block partial.
__global__ void gram_tensor_reduce_kernel(const double* __restrict__ part, int nsplit, int nb, int npairs,
                                          uint32_t K, double* __restrict__ G) {
  const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= uint64_t(K) * K) return;
  const uint32_t i = uint32_t(idx % K), c = uint32_t(idx / K);
  if (i > c) return;
  const int bi = int(i / kGB), bc = int(c / kGB);
  const int pair = bi * nb - bi * (bi - 1) / 2 + (bc - bi);
  const size_t off = size_t(i % kGB) * kGB + (c % kGB);
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += part[(size_t(k) * npairs + pair) * (kGB * kGB) + off];
  G[i + size_t(c) * K] = s;
  G[c + size_t(i) * K] = s;
}

}  // namespace

GramPlan gram_tensor_plan(const FiberView& v, int num_sms) {
  GramPlan p;
  p.nb = int((v.K + kGB - 1) / kGB);
  p.npairs = p.nb * (p.nb + 1) / 2;
  const uint64_t F = v.s * v.P;
  const uint64_t target = uint64_t(std::max(1, 2 * num_sms / std::max(1, p.npairs)));
  const uint64_t max_split = std::max<uint64_t>(1, (F + 4 * kGC - 1) / (4 * kGC));  // >= 4 chunks each
  p.nsplit = int(std::min<uint64_t>(std::max<uint64_t>(1, target), max_split));
  const uint64_t per = (F + uint64_t(p.nsplit) - 1) / uint64_t(p.nsplit);
  p.per_split = (per + kGC - 1) / kGC * kGC;
  p.nsplit = int((F + p.per_split - 1) / p.per_split);
  if (p.nsplit < 1) p.nsplit = 1;
  p.part_doubles = size_t(p.nsplit) * size_t(p.npairs) * kGB * kGB;
  return p;
}

cudaError_t launch_gram_tensor(const FiberView& v, const GramPlan& p, double* part, double* G, cudaStream_t st) {
  const size_t smem = sizeof(double) * size_t(kGStages) * kGStageDoubles;
  cudaError_t e = raise_smem_limit(gram_tensor_kernel, smem);
  if (e != cudaSuccess) return e;
  gram_tensor_kernel<<<unsigned(p.nsplit) * unsigned(p.npairs), kGThreads, smem, st>>>(v, p.nb, p.npairs,
                                                                                      p.per_split, part);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const uint64_t n = uint64_t(v.K) * v.K;
  gram_tensor_reduce_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(part, p.nsplit, p.nb, p.npairs, v.K, G);
  return cudaGetLastError();
}

}  // namespace tkg
