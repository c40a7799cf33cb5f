// Device side of the MT19937-64 jump-ahead (see mt_jump.hpp): chunk states
// by GF(2) XOR-sums over the raw sequence, then one CTA per chunk generates
// its J draws with the standard twist (in-place semantics of
// std::mersenne_twister_engine) and writes uniform01 values
// ((y >> 11) * 2^-53, rng.hpp:19-21) straight into S (storage order, or the
// window of one shard's fibers).
#include <algorithm>
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
constexpr int kJW = 10;  // words per lane

__global__ void __launch_bounds__(32) mt_jump_kernel(const uint64_t* __restrict__ y,
                                                     const uint64_t* __restrict__ polys,
                                                     uint64_t* __restrict__ states, int wpp,
                                                     const int* __restrict__ chunk_ids) {
  extern __shared__ uint64_t ys[];
  const int slot = blockIdx.x;
  const int c = chunk_ids ? chunk_ids[slot] : slot;
  const int part = blockIdx.y;
  const int lane = threadIdx.x;
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
      atomicXor(reinterpret_cast<unsigned long long*>(states + size_t(slot) * kMtN + t),
                static_cast<unsigned long long>(acc[k]));
  }
}

// n / d for n < 2^51 from a double reciprocal plus one correction step.
__device__ __forceinline__ uint64_t fast_div(uint64_t n, uint64_t d, double inv) {
  uint64_t q = static_cast<uint64_t>(static_cast<double>(n) * inv);
  const int64_t r = static_cast<int64_t>(n - q * d);
  if (r < 0) --q;
  else if (static_cast<uint64_t>(r) >= d) ++q;
  return q;
}

// One CTA per chunk, one state word per thread (312 of 320 threads): the
// twist's three dependency phases (j < 156 reads old words only; 156 <= j <
// 311 reads new[j-156]; j = 311 reads new[0] and new[155]) are separated by
// CTA barriers on a shared-memory state, so a 312-draw block costs a few
// barriers instead of the warp version's chain of dependent shuffles; each
// thread tempers and stores its own draw (consecutive positions, coalesced).
constexpr int kGenThreads = 320;

__device__ __forceinline__ void store_draw(double* __restrict__ out, const MtWindow& win, uint64_t p, double v) {
  if (win.nloc == 0) {
    out[p] = v;
    return;
  }
  // S window (see MtWindow): position c*Fg + j -> column c, fiber j
  const uint64_t col = fast_div(p, win.Fg, win.inv_fg);
  const uint64_t j = p - col * win.Fg;
  const uint64_t Fl = win.Fg / win.Gsm * win.nloc;
  uint64_t loc = j;
  if (win.Gsm > 1) {  // a shard: keep its own fibers, in its local order
    const uint64_t t = fast_div(j, win.Plo, win.inv_plo);
    const uint64_t jhi = fast_div(t, win.Gsm, win.inv_gsm);
    const uint64_t ism = t - jhi * win.Gsm;
    if (ism < win.o0 || ism >= win.o0 + win.nloc) return;
    loc = (j - t * win.Plo) + win.Plo * ((ism - win.o0) + win.nloc * jhi);
  }
  out[win.ld ? loc * win.ld + col : loc + col * Fl] = v;
}

__global__ void __launch_bounds__(kGenThreads) mt_gen_cta_kernel(const uint64_t* __restrict__ states, uint64_t J,
                                                                 uint64_t total, double* __restrict__ out,
                                                                 MtWindow win, const int* __restrict__ chunk_ids) {
  __shared__ uint64_t mt[kMtN];
  const int slot = blockIdx.x;
  const int c = chunk_ids ? chunk_ids[slot] : slot;
  const int j = threadIdx.x;
  const bool own = j < kMtN;
  const uint64_t start = uint64_t(c) * J;
  const uint64_t end = min(start + J, total);
  if (own) mt[j] = states[size_t(slot) * kMtN + j];
  __syncthreads();
  for (uint64_t pos = start;;) {
    uint64_t cur = 0, nxt = 0, far = 0;
    if (own) {
      cur = mt[j];
      if (pos + j < end) store_draw(out, win, pos + j, to_uniform01(cur));
      nxt = mt[j + 1 < kMtN ? j + 1 : 0];
      far = mt[j < 156 ? j + 156 : j - 156];
    }
    pos += kMtN;
    if (pos >= end) break;
    __syncthreads();                    // every old word is in registers
    if (j < 156) mt[j] = twist(cur, nxt, far);
    __syncthreads();                    // new[0 .. 155]
    if (own && j >= 156) {
      // j < 311: twist(old[j], old[j+1], new[j-156]); j = 311: twist(old[311], new[0], new[155])
      mt[j] = j < kMtN - 1 ? twist(cur, nxt, mt[j - 156]) : twist(cur, mt[0], mt[155]);
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C, const int* d_chunk_ids,
                             uint64_t* d_states, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_states, 0, sizeof(uint64_t) * size_t(C) * kMtN, st);
  if (e != cudaSuccess) return e;
  // enough one-warp blocks to fill the machine (~48 per SM: small shared
  // windows, so the XOR chains have other warps to hide behind)
  const int parts = std::max(4, std::min(64, (7104 + C - 1) / C));
  const int wpp = (kPolyWords + parts - 1) / parts;
  const int nparts = (kPolyWords + wpp - 1) / wpp;
  const size_t smem = sizeof(uint64_t) * (size_t(wpp) * 64 + 32 * kJW + kJW);
  mt_jump_kernel<<<dim3(C, nparts), 32, smem, st>>>(d_y, d_polys, d_states, wpp, d_chunk_ids);
  return cudaGetLastError();
}

cudaError_t launch_mt_generate(const uint64_t* d_states, int C, const int* d_chunk_ids, uint64_t J,
                               uint64_t total, double* d_out, MtWindow win, cudaStream_t st) {
  if (C <= 0) return cudaSuccess;
  mt_gen_cta_kernel<<<C, kGenThreads, 0, st>>>(d_states, J, total, d_out, win, d_chunk_ids);
  return cudaGetLastError();
}

}  // namespace tkg
