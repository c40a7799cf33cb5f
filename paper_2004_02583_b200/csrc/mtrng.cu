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

// grid (C, split), block 320 (word t = threadIdx.x < 312).
__global__ void mt_jump_kernel(const uint64_t* __restrict__ y, const uint64_t* __restrict__ polys,
                               int split, uint64_t* __restrict__ states) {
  extern __shared__ uint64_t ys[];
  const int c = blockIdx.x;
  const int part = blockIdx.y;
  const int wpp = (kPolyWords + split - 1) / split;
  const int w0 = part * wpp;
  const int w1 = min(kPolyWords, w0 + wpp);
  if (w0 >= w1) return;
  const int nbits = (w1 - w0) * 64;
  const int nload = nbits + kMtN;
  __shared__ uint64_t pw[64];
  for (int k = threadIdx.x; k < nload; k += blockDim.x) ys[k] = y[size_t(w0) * 64 + k];
  for (int k = threadIdx.x; k < w1 - w0; k += blockDim.x) pw[k] = polys[size_t(c) * kPolyWords + w0 + k];
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= kMtN) return;
  uint64_t acc = 0;
  for (int w = 0; w < w1 - w0; ++w) {
    uint64_t bits = pw[w];  // same word for the whole CTA: uniform control flow
    const uint64_t* row = ys + w * 64 + t;
    while (bits) {
      const int b = __ffsll(static_cast<long long>(bits)) - 1;
      acc ^= row[b];
      bits &= bits - 1;
    }
  }
  atomicXor(reinterpret_cast<unsigned long long*>(states + size_t(c) * kMtN + t),
            static_cast<unsigned long long>(acc));
}

// One CTA (160 threads) per chunk.
__global__ void __launch_bounds__(160) mt_gen_kernel(const uint64_t* __restrict__ states, uint64_t J,
                                                     uint64_t total, double* __restrict__ out,
                                                     uint64_t F, uint64_t ld) {
  __shared__ uint64_t mt[kMtN];
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  const uint64_t start = uint64_t(c) * J;
  const uint64_t end = min(start + J, total);
  for (int k = tid; k < kMtN; k += blockDim.x) mt[k] = states[size_t(c) * kMtN + k];
  __syncthreads();
  uint64_t pos = start;
  while (true) {
    if (ld == 0) {
      for (int k = tid; k < kMtN; k += blockDim.x)
        if (pos + k < end) out[pos + k] = to_uniform01(mt[k]);
    } else {
      // S(j, c) with idx = j + c*F, stored at j*ld + c
      const uint64_t c0 = pos / F;
      const uint64_t j0 = pos - c0 * F;
      for (int k = tid; k < kMtN; k += blockDim.x) {
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
    // In-place twist, i = 0..155 (reads old i, i+1, i+156).
    uint64_t a = 0, b = 0, f = 0;
    if (tid < 156) {
      a = mt[tid];
      b = mt[tid + 1];
      f = mt[tid + 156];
    }
    __syncthreads();
    if (tid < 156) mt[tid] = twist(a, b, f);
    __syncthreads();
    // i = 156..310 (reads old i, i+1 and new i-156).
    if (tid < 155) {
      a = mt[156 + tid];
      b = mt[157 + tid];
      f = mt[tid];
    }
    __syncthreads();
    if (tid < 155) mt[156 + tid] = twist(a, b, f);
    __syncthreads();
    // i = 311 (reads old 311, new 0 and new 155).
    if (tid == 0) mt[311] = twist(mt[311], mt[0], mt[155]);
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C,
                             uint64_t* d_states, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_states, 0, sizeof(uint64_t) * size_t(C) * kMtN, st);
  if (e != cudaSuccess) return e;
  const int split = 8;
  const int wpp = (kPolyWords + split - 1) / split;
  const size_t smem = sizeof(uint64_t) * (size_t(wpp) * 64 + kMtN);
  mt_jump_kernel<<<dim3(C, split), 320, smem, st>>>(d_y, d_polys, split, d_states);
  return cudaGetLastError();
}

cudaError_t launch_mt_generate(const uint64_t* d_states, int C, uint64_t J, uint64_t total,
                               double* d_out, uint64_t F, uint64_t ld, cudaStream_t st) {
  mt_gen_kernel<<<C, 160, 0, st>>>(d_states, J, total, d_out, F, ld);
  return cudaGetLastError();
}

}  // namespace tkg
