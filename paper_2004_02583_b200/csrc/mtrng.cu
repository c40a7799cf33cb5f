// Device side of the MT19937-64 jump-ahead (see mt_jump.hpp): chunk states
// by GF(2) XOR-sums over the raw sequence, then one CTA per chunk generates
// its J draws with the standard twist (in-place semantics of
// std::mersenne_twister_engine) and writes uniform01 values
// ((y >> 11) * 2^-53, rng.hpp:19-21) straight into S (storage order, or
// transposed into the row-major FR operand layout).
#include <cstdint>

#include "kernels.cuh"
#include "mt_jump.hpp"

namespace tkg {

namespace {

constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x000000007FFFFFFFull;
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ull;

__device__ __forceinline__ uint64_t twist(uint64_t cur, uint64_t nxt, uint64_t far) {
  const uint64_t y = (cur & kUpper) | (nxt & kLower);
  return far ^ (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
}

__device__ __forceinline__ double to_uniform01(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= (z >> 43);
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

// One warp per (chunk, bit range of the jump polynomial). Lane L owns state
// words t = 10L .. 10L+9 and walks the bits i in groups of 10: the 19 words
// y[i0 + 10L .. i0 + 10L + 18] loaded once serve all 10 bits x 10 outputs
// (the XOR-sum is a Hankel product), so shared-memory traffic is ~5x lower
// than one load per (bit, word). Partial sums are combined with atomicXor.
constexpr int kJumpSplit = 8;
constexpr int kJW = 10;  // words per lane

__global__ void __launch_bounds__(32) mt_jump_kernel(const uint64_t* __restrict__ y,
                                                     const uint64_t* __restrict__ polys,
                                                     uint64_t* __restrict__ states) {
  extern __shared__ uint64_t ys[];
  const int c = blockIdx.x;
  const int part = blockIdx.y;
  const int lane = threadIdx.x;
  const int wpp = (kPolyWords + kJumpSplit - 1) / kJumpSplit;
  const int w0 = part * wpp;
  const int w1 = min(kPolyWords, w0 + wpp);
  if (w0 >= w1) return;
  const int nbits = (w1 - w0) * 64;
  const int nload = nbits + 32 * kJW + kJW;
  for (int k = lane; k < nload; k += 32) {
    const size_t g = size_t(w0) * 64 + k;
    ys[k] = g < size_t(kPolyWords) * 64 + kMtN ? y[g] : 0ull;
  }
  __syncwarp();
  uint64_t acc[kJW];
#pragma unroll
  for (int k = 0; k < kJW; ++k) acc[k] = 0;
  const uint64_t* pw = polys + size_t(c) * kPolyWords + w0;
  const uint64_t* base = ys + kJW * lane;
  for (int i0 = 0; i0 < nbits; i0 += kJW) {
    // bits i0 .. i0+9 of this range (may straddle a polynomial word)
    uint64_t m[kJW];
#pragma unroll
    for (int d = 0; d < kJW; ++d) {
      const int i = i0 + d;
      const uint64_t word = i < nbits ? __ldg(pw + (i >> 6)) : 0ull;
      m[d] = 0ull - ((word >> (i & 63)) & 1ull);
    }
    uint64_t win[2 * kJW - 1];
#pragma unroll
    for (int k = 0; k < 2 * kJW - 1; ++k) win[k] = base[i0 + k];
#pragma unroll
    for (int d = 0; d < kJW; ++d)
#pragma unroll
      for (int k = 0; k < kJW; ++k) acc[k] ^= win[d + k] & m[d];
  }
#pragma unroll
  for (int k = 0; k < kJW; ++k) {
    const int t = kJW * lane + k;
    if (t < kMtN)
      atomicXor(reinterpret_cast<unsigned long long*>(states + size_t(c) * kMtN + t),
                static_cast<unsigned long long>(acc[k]));
  }
}

// One warp per chunk (4 chunks per CTA): the 312-word state lives in shared
// memory; each twist is two independent 156-wide phases (read, __syncwarp,
// write) plus the wrap word, with in-place std::mersenne_twister_engine
// semantics; outputs are written coalesced in storage order.
constexpr int kGenWarps = 4;

__global__ void __launch_bounds__(32 * kGenWarps) mt_gen_kernel(const uint64_t* __restrict__ states,
                                                               int C, uint64_t J, uint64_t total,
                                                               double* __restrict__ out, uint64_t F,
                                                               uint64_t ld) {
  __shared__ uint64_t mts[kGenWarps][kMtN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kGenWarps + warp;
  if (c >= C) return;
  uint64_t* mt = mts[warp];
  const uint64_t start = uint64_t(c) * J;
  const uint64_t end = min(start + J, total);
  for (int k = lane; k < kMtN; k += 32) mt[k] = states[size_t(c) * kMtN + k];
  __syncwarp();
  uint64_t pos = start;
  while (true) {
    if (ld == 0) {
      for (int k = lane; k < kMtN; k += 32)
        if (pos + k < end) out[pos + k] = to_uniform01(mt[k]);
    } else {
      const uint64_t c0 = pos / F;
      const uint64_t j0 = pos - c0 * F;
      for (int k = lane; k < kMtN; k += 32) {
        if (pos + k >= end) continue;
        uint64_t j = j0 + k, col = c0;
        if (j >= F) {
          col += j / F;
          j %= F;
        }
        out[j * ld + col] = to_uniform01(mt[k]);
      }
    }
    pos += kMtN;
    if (pos >= end) break;
    uint64_t nv[5];
    // i = 0..155: reads old i, i+1, i+156
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int i = lane + 32 * r;
      nv[r] = i < 156 ? twist(mt[i], mt[i + 1], mt[i + 156]) : 0ull;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int i = lane + 32 * r;
      if (i < 156) mt[i] = nv[r];
    }
    __syncwarp();
    // i = 156..310: reads old i, i+1 and new i-156
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int i = 156 + lane + 32 * r;
      nv[r] = i < 311 ? twist(mt[i], mt[i + 1], mt[i - 156]) : 0ull;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int i = 156 + lane + 32 * r;
      if (i < 311) mt[i] = nv[r];
    }
    __syncwarp();
    // i = 311: reads old 311, new 0 and new 155
    if (lane == 0) mt[311] = twist(mt[311], mt[0], mt[155]);
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C,
                             uint64_t* d_states, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_states, 0, sizeof(uint64_t) * size_t(C) * kMtN, st);
  if (e != cudaSuccess) return e;
  const int wpp = (kPolyWords + kJumpSplit - 1) / kJumpSplit;
  const size_t smem = sizeof(uint64_t) * (size_t(wpp) * 64 + 32 * kJW + kJW);
  mt_jump_kernel<<<dim3(C, kJumpSplit), 32, smem, st>>>(d_y, d_polys, d_states);
  return cudaGetLastError();
}

cudaError_t launch_mt_generate(const uint64_t* d_states, int C, uint64_t J, uint64_t total,
                               double* d_out, uint64_t F, uint64_t ld, cudaStream_t st) {
  mt_gen_kernel<<<(C + kGenWarps - 1) / kGenWarps, 32 * kGenWarps, 0, st>>>(d_states, C, J, total,
                                                                           d_out, F, ld);
  return cudaGetLastError();
}

}  // namespace tkg
