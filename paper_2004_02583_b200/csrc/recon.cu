// Mode-n expansion X x_n U (U: Iout x K, K = R_n <= 64) with either a store
// epilogue or a fused difference norm against a reference tensor. Used to
// evaluate relative_error(t, reconstruct(tk)) (tensor_ops.cpp:395-440,
// hosvd.cpp:123,189) without materialising the reconstruction: the last
// expansion's outputs are compared with A in registers and only per-CTA
// partial sums of squares leave the SM.
//
// A CTA keeps one 128-fiber tile of the (small-K) input in shared memory and
// sweeps all Iout output columns in blocks of 32, so the input is read once;
// each warp owns 16 fibers x 32 columns of DMMA accumulators, and the next
// block's factor rows and reference values are prefetched with cp.async
// while the current block's MMAs run.
#include <algorithm>

#include "kernels.cuh"

namespace tkg {

namespace {

constexpr int kTile = 128;
constexpr int kLdT = kTile + 4;   // [K][kLdT]: fragment rows 4 (mod 16) apart
constexpr int kCB = 32;           // output columns per block
constexpr int kLdU = kCB + 4;
constexpr int kLdR = kTile + 4;   // reference block [kCB][kLdR]

// Shared memory: Ts [KC][kLdT] | Us[2][KC][kLdU] | Rb[2][kCB][kLdR] (diff only)
template <int KC>
__global__ void __launch_bounds__(256, 2) expand_kernel(ExpandArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* Ts = sm;
  double* Us = Ts + KC * kLdT;
  double* Rb = Us + 2 * KC * kLdU;
  __shared__ double red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r8 = lane >> 2;
  const uint64_t F = a.s * a.P;
  const uint64_t ntiles = (F + kTile - 1) / kTile;
  const int nblocks = int((a.Iout + kCB - 1) / kCB);
  const bool diff = a.ref != nullptr;
  double sq = 0.0;

  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t j0 = tile * kTile;
    // the tile is one panel run when s is a multiple of the tile
    const bool run = (a.s % kTile) == 0;
    const uint64_t p0 = j0 / a.s, jl0 = j0 - p0 * a.s;
    const bool vec = run && (a.s % 2 == 0) && (jl0 % 2 == 0);
    auto issue = [&](int blk, int buf) {
      const uint32_t i0 = blk * kCB;
      double* u = Us + buf * KC * kLdU;
      for (int e = threadIdx.x; e < KC * kCB; e += blockDim.x) {
        const int c = e / kCB, ii = e % kCB;
        const uint32_t i = i0 + ii;
        if (i < a.Iout && c < int(a.K)) cp_async8(u + c * kLdU + ii, a.U + i + uint64_t(c) * a.Iout);
        else u[c * kLdU + ii] = 0.0;
      }
      if (diff) {
        double* rb = Rb + buf * kCB * kLdR;
        if (vec) {
          for (int e = threadIdx.x; e < kCB * (kTile / 2); e += blockDim.x) {
            const int ii = e / (kTile / 2), jt = (e % (kTile / 2)) * 2;
            const uint32_t i = i0 + ii;
            const uint64_t j = j0 + jt;
            if (i < a.Iout && j + 1 < F + 1 && j < F) {
              cp_async16(rb + ii * kLdR + jt, a.ref + jl0 + jt + uint64_t(i) * a.s + p0 * a.s * a.Iout);
            } else {
              rb[ii * kLdR + jt] = 0.0;
              rb[ii * kLdR + jt + 1] = 0.0;
            }
          }
        } else {
          for (int e = threadIdx.x; e < kCB * kTile; e += blockDim.x) {
            const int ii = e / kTile, jt = e % kTile;
            const uint32_t i = i0 + ii;
            const uint64_t j = j0 + jt;
            if (i < a.Iout && j < F) {
              const uint64_t p = j / a.s, jl = j - p * a.s;
              cp_async8(rb + ii * kLdR + jt, a.ref + jl + uint64_t(i) * a.s + p * a.s * a.Iout);
            } else {
              rb[ii * kLdR + jt] = 0.0;
            }
          }
        }
      }
      cp_async_commit();
    };

    __syncthreads();  // previous tile's readers are done with Ts / Us / Rb
    for (int e = threadIdx.x; e < KC * kTile; e += blockDim.x) {
      const int c = e / kTile, jt = e % kTile;
      const uint64_t j = j0 + jt;
      double v = 0.0;
      if (j < F && c < int(a.K)) {
        const uint64_t p = j / a.s, jl = j - p * a.s;
        v = a.in[jl + uint64_t(c) * a.s + p * a.s * a.K];
      }
      Ts[c * kLdT + jt] = v;
    }
    int64_t ob[2];
    bool ok[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const uint64_t j = j0 + warp * 16 + m * 8 + r8;
      ok[m] = j < F;
      const uint64_t jj = ok[m] ? j : 0;
      const uint64_t p = jj / a.s, jl = jj - p * a.s;
      ob[m] = int64_t(jl + p * a.s * a.Iout);
    }
    issue(0, 0);
    for (int blk = 0; blk < nblocks; ++blk) {
      const int buf = blk & 1;
      if (blk + 1 < nblocks) {
        issue(blk + 1, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* u = Us + buf * KC * kLdU;
      double acc[2][kCB / 8][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < kCB / 8; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll
      for (int t = 0; t < KC / 4; ++t) {
        const int kk = 4 * t + q;
        double af[2], bf[kCB / 8];
#pragma unroll
        for (int m = 0; m < 2; ++m) af[m] = Ts[kk * kLdT + warp * 16 + m * 8 + r8];
#pragma unroll
        for (int n = 0; n < kCB / 8; ++n) bf[n] = u[kk * kLdU + n * 8 + r8];
#pragma unroll
        for (int n = 0; n < kCB / 8; ++n)
#pragma unroll
          for (int m = 0; m < 2; ++m) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
      }
      const uint32_t i0 = blk * kCB;
      const double* rb = Rb + buf * kCB * kLdR;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        if (!ok[m]) continue;
        const int jt = warp * 16 + m * 8 + r8;
#pragma unroll
        for (int n = 0; n < kCB / 8; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ii = n * 8 + 2 * q + e;
            const uint32_t i = i0 + ii;
            if (i >= a.Iout) continue;
            if (diff) {
              const double d = rb[ii * kLdR + jt] - acc[m][n][e];  // b - a as relative_error
              sq = fma(d, d, sq);
            } else {
              a.out[ob[m] + int64_t(i) * int64_t(a.s)] = acc[m][n][e];
            }
          }
      }
      __syncthreads();  // buffer `buf` is refilled by the next issue()
    }
  }
  if (a.sumsq_part) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    __syncthreads();
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      a.sumsq_part[blockIdx.x] = s;
    }
  }
}

}  // namespace

int expand_grid(uint64_t F, int num_sms) {
  const uint64_t tiles = (F + kTile - 1) / kTile;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(2 * num_sms))));
}

cudaError_t launch_expand(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used) {
  const int grid = expand_grid(a.s * a.P, num_sms);
  if (grid_used) *grid_used = grid;
  const uint32_t kc = (a.K + 3) / 4 * 4;
#define TKG_E(N)                                                                                \
  if (kc <= N) {                                                                                \
    const size_t smem = sizeof(double) * (size_t(N) * kLdT + 2 * size_t(N) * kLdU +           \
                                          (a.ref ? 2 * size_t(kCB) * kLdR : 0));             \
    cudaError_t e = raise_smem_limit(expand_kernel<N>, smem);                                 \
    if (e != cudaSuccess) return e;                                                             \
    expand_kernel<N><<<grid, 256, smem, st>>>(a);                                               \
    return cudaGetLastError();                                                                  \
  }
  TKG_E(8) TKG_E(16) TKG_E(24) TKG_E(32) TKG_E(40) TKG_E(48) TKG_E(56) TKG_E(64)
#undef TKG_E
  return cudaErrorInvalidValue;
}

}  // namespace tkg
