// Device side of the MT19937-64 jump-ahead (see mt_jump.hpp): chunk states
// by GF(2) XOR-sums over the raw sequence, then one warp per chunk generates
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

// One warp per chunk with the 312-word state in registers: word j = 32*s + L
// lives in slot s of lane L (slot 9 only for L < 24). A twist (in-place
// std::mersenne_twister_engine semantics) is
//   new[j] = twist(old[j], old[j+1], old[j+156])   j < 156
//   new[j] = twist(old[j], old[j+1], new[j-156])   156 <= j < 311
//   new[311] = twist(old[311], new[0], new[155])
// with the neighbours fetched by warp shuffles: j+1 is lane L+1 (lane 0's
// next slot for L = 31), j+156 = 32(s+4) + L+28 and j-156 = 32(s-5) + L+4, so
// each source lane sends the slot its reader needs. No shared memory, no
// barriers; the ten words of a slot are written as one coalesced row.
constexpr int kGenWarps = 4;

// n / d for n < 2^51 from a double reciprocal plus one correction step.
__device__ __forceinline__ uint64_t fast_div(uint64_t n, uint64_t d, double inv) {
  uint64_t q = static_cast<uint64_t>(static_cast<double>(n) * inv);
  const int64_t r = static_cast<int64_t>(n - q * d);
  if (r < 0) --q;
  else if (static_cast<uint64_t>(r) >= d) ++q;
  return q;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  return static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<unsigned long long>(v), src));
}

__global__ void __launch_bounds__(32 * kGenWarps) mt_gen_kernel(const uint64_t* __restrict__ states,
                                                               int C, uint64_t J, uint64_t total,
                                                               double* __restrict__ out, MtWindow win,
                                                               const int* __restrict__ chunk_ids) {
  const int warp = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int slot = blockIdx.x * kGenWarps + warp;
  if (slot >= C) return;
  const int c = chunk_ids ? chunk_ids[slot] : slot;
  const uint64_t start = uint64_t(c) * J;
  const uint64_t end = min(start + J, total);
  uint64_t w[10];
#pragma unroll
  for (int s = 0; s < 10; ++s) {
    const int j = 32 * s + L;
    w[s] = j < kMtN ? states[size_t(slot) * kMtN + j] : 0ull;
  }
  const int nxt = (L + 1) & 31, far = (L + 28) & 31, back = (L + 4) & 31;
  uint64_t pos = start;
  while (true) {
    if (win.nloc == 0) {
      if (pos + kMtN <= end) {
#pragma unroll
        for (int s = 0; s < 10; ++s)
          if (s < 9 || L < 24) out[pos + 32 * s + L] = to_uniform01(w[s]);
      } else {
#pragma unroll
        for (int s = 0; s < 10; ++s) {
          const uint64_t j = 32 * s + L;
          if ((s < 9 || L < 24) && pos + j < end) out[pos + j] = to_uniform01(w[s]);
        }
      }
    } else {
      // S window (see MtWindow): position c*Fg + j -> column c, fiber j
      const uint64_t c0 = fast_div(pos, win.Fg, win.inv_fg);
      const uint64_t j0 = pos - c0 * win.Fg;
      const uint64_t Fl = win.Fg / win.Gsm * win.nloc;
#pragma unroll
      for (int s = 0; s < 10; ++s) {
        const uint64_t k = 32 * s + L;
        if (!(s < 9 || L < 24) || pos + k >= end) continue;
        uint64_t j = j0 + k, col = c0;
        while (j >= win.Fg) {
          j -= win.Fg;
          ++col;
        }
        uint64_t loc = j;
        if (win.Gsm > 1) {  // a shard: keep its own fibers, in its local order
          const uint64_t t = fast_div(j, win.Plo, win.inv_plo);
          const uint64_t jhi = fast_div(t, win.Gsm, win.inv_gsm);
          const uint64_t ism = t - jhi * win.Gsm;
          if (ism < win.o0 || ism >= win.o0 + win.nloc) continue;
          loc = (j - t * win.Plo) + win.Plo * ((ism - win.o0) + win.nloc * jhi);
        }
        out[win.ld ? loc * win.ld + col : loc + col * Fl] = to_uniform01(w[s]);
      }
    }
    pos += kMtN;
    if (pos >= end) break;
    // phase A: j = 32s + L < 156 (s <= 4; s = 4 for L < 28)
    uint64_t na[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const uint64_t v1 = shfl64(L == 0 ? w[s + 1] : w[s], nxt);
      const uint64_t v2 = shfl64(L >= 28 ? w[s + 4] : w[s + 5], far);
      na[s] = twist(w[s], v1, v2);
    }
    // phase B: 156 <= j < 311 (s = 4 for L >= 28, s = 5..9)
    uint64_t nb[10];
#pragma unroll
    for (int s = 4; s < 10; ++s) {
      const uint64_t v1 = shfl64(L == 0 ? w[s < 9 ? s + 1 : 9] : w[s], nxt);
      const int ia = s - 4 < 4 ? s - 4 : 4, ib = s - 5 > 0 ? s - 5 : 0;
      const uint64_t v3 = shfl64(s == 4 ? na[0] : (L < 4 ? na[ia] : na[ib]), back);
      nb[s] = twist(w[s], v1, v3);
    }
    // j = 311 (lane 23, slot 9)
    const uint64_t n0 = shfl64(na[0], 0), n155 = shfl64(na[4], 27);
    const uint64_t n311 = twist(w[9], n0, n155);
#pragma unroll
    for (int s = 0; s < 4; ++s) w[s] = na[s];
    w[4] = L < 28 ? na[4] : nb[4];
#pragma unroll
    for (int s = 5; s < 9; ++s) w[s] = nb[s];
    w[9] = L < 23 ? nb[9] : (L == 23 ? n311 : 0ull);
  }
}

}  // namespace

cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C, const int* d_chunk_ids,
                             uint64_t* d_states, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_states, 0, sizeof(uint64_t) * size_t(C) * kMtN, st);
  if (e != cudaSuccess) return e;
  // enough warps to fill the machine (~16 per SM), at least 5 words per warp
  const int parts = std::max(4, std::min(64, (2368 + C - 1) / C));
  const int wpp = (kPolyWords + parts - 1) / parts;
  const int nparts = (kPolyWords + wpp - 1) / wpp;
  const size_t smem = sizeof(uint64_t) * (size_t(wpp) * 64 + 32 * kJW + kJW);
  mt_jump_kernel<<<dim3(C, nparts), 32, smem, st>>>(d_y, d_polys, d_states, wpp, d_chunk_ids);
  return cudaGetLastError();
}

cudaError_t launch_mt_generate(const uint64_t* d_states, int C, const int* d_chunk_ids, uint64_t J,
                               uint64_t total, double* d_out, MtWindow win, cudaStream_t st) {
  mt_gen_kernel<<<(C + kGenWarps - 1) / kGenWarps, 32 * kGenWarps, 0, st>>>(d_states, C, J, total, d_out,
                                                                           win, d_chunk_ids);
  return cudaGetLastError();
}

}  // namespace tkg
