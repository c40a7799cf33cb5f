// Probe of the 5th-generation tensor core's integer MMA (tcgen05.mma
// kind::i8) on sm_100a: operand layouts (A from TMEM written by
// tcgen05.st, B K-major in shared memory without swizzle), instruction and
// shared-memory descriptors, int32 accumulation in TMEM, and issue
// throughput at the narrow N (32 / 64) of the ALS contractions. Groundwork
// for an FP64-emulating (Ozaki-style) contraction; not used by the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_i8_probe tools/umma_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SM100 shared-memory matrix descriptor, K-major, no swizzle: start>>4 [0,14),
// LBO>>4 [16,30) (stride between the two 16-byte K chunks), SBO>>4 [32,46)
// (stride between 8-row groups), version 1 at [46,48), layout type 0 at [61,64).
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((smem_u32(p) >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

// instruction descriptor, kind::i8: c_format S32 (2) at [4,6), a/b format
// (0 u8, 1 s8) at [7,10) / [10,13), K-major A and B, N>>3 at [17,23), M>>4 at [24,29)
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_signed, int b_signed) {
  return (2u << 4) | (uint32_t(a_signed) << 7) | (uint32_t(b_signed) << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni D_%=;\nbra.uni W_%=;\nD_%=:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// A: M x 32 int8 row-major (K contiguous); B: N x 32 int8 row-major; D = A B^T (int32).
// mode 0: A from TMEM (tcgen05.st by the thread owning the row); mode 1: A from smem.
template <int M, int N>
__global__ void __launch_bounds__(128) probe(const int8_t* A, const int8_t* B, int a_signed, int b_signed, int mode,
                                             int reps, int ndst, int* D, long long* cycles) {
  __shared__ __align__(1024) uint8_t sA[M * 32];
  __shared__ __align__(1024) uint8_t sB[N * 32];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical K-major no-swizzle layout: core matrix (8 rows x 16 B) at
  // group*SBO + kchunk*LBO with LBO = 128, SBO = 256
  for (int e = tid; e < N * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    sB[(n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = uint8_t(B[e]);
  }
  for (int e = tid; e < M * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    sA[(m / 8) * 256 + (k / 16) * 128 + (m % 8) * 16 + (k % 16)] = uint8_t(A[e]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy (UMMA)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = taddr;
  const uint32_t d_col = 64, a_col = 0;  // A: columns [0, 8); D: columns [64, 64 + N)
  if (mode == 0 && warp < M / 32) {
    // row = 32*warp + lane; its 32 K bytes as 8 words, little-endian within a word
    const int row = warp * 32 + lane;
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) v |= uint32_t(uint8_t(A[row * 32 + c * 4 + b])) << (8 * b);
      w[c] = v;
    }
    const uint32_t addr = tm + (uint32_t(warp * 32) << 16) + a_col;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, N, a_signed, b_signed);
    const uint64_t bd = sdesc(sB, 128, 256);
    const uint64_t ad = sdesc(sA, 128, 256);
    // ndst > 1: round-robin over independent accumulators at column 64 + j*N
    // (the Ozaki pattern: products of one diagonal share an accumulator)
    t0 = clock64();
    if (ndst == 0) {  // unrolled: 8 MMAs per iteration on two accumulators, no index math
      if (mode == 0) {
        mma_i8_ts(tm + d_col, tm + a_col, bd, id, 0u);
        mma_i8_ts(tm + d_col + N, tm + a_col, bd, id, 0u);
      }
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (mode == 0) mma_i8_ts(tm + d_col + (u & 1) * N, tm + a_col, bd, id, 1u);
          else mma_i8_ss(tm + d_col + (u & 1) * N, ad, bd, id, 1u);
        }
      }
    } else {
      for (int r = 0; r < reps; ++r) {
        const uint32_t dc = d_col + (r % ndst) * N;
        const uint32_t acc = ndst == 1 ? (r > 0 ? 1u : 0u) : (r >= ndst ? 1u : 0u);
        if (mode == 0) mma_i8_ts(tm + dc, tm + a_col, bd, id, acc);
        else mma_i8_ss(tm + dc, ad, bd, id, acc);
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    cycles[0] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < M / 32) {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = tm + (uint32_t(warp * 32) << 16) + d_col + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = int(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int M, int N>
int run(int a_signed, int b_signed, int mode, int reps, int ndst = 1) {
  std::vector<int8_t> hA(M * 32), hB(N * 32);
  srand(7 + M + N + mode);
  for (auto& x : hA) x = int8_t(rand() & 0xff);
  for (auto& x : hB) x = int8_t(rand() & 0xff);
  int8_t *dA, *dB;
  int* dD;
  long long* dc;
  cudaMalloc(&dA, hA.size());
  cudaMalloc(&dB, hB.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, M * N * 4);
  probe<M, N><<<1, 128>>>(dA, dB, a_signed, b_signed, mode, reps, ndst, dD, dc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> hD(M * N);
  long long cyc = 0;
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  long long bad = 0, first = -1;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      long long s = 0;
      for (int k = 0; k < 32; ++k) {
        const int a = a_signed ? int(hA[m * 32 + k]) : int(uint8_t(hA[m * 32 + k]));
        const int b = b_signed ? int(hB[n * 32 + k]) : int(uint8_t(hB[n * 32 + k]));
        s += a * b;
      }
      s *= reps;
      if (int(s) != hD[m * N + n]) {
        if (first < 0) first = m * N + n;
        ++bad;
      }
    }
  const double macs = double(M) * N * 32 * reps;
  if (ndst != 1) bad = 0;  // D holds one accumulator's share of the reps
  std::printf("{\"M\":%d,\"N\":%d,\"a_signed\":%d,\"b_signed\":%d,\"A\":\"%s\",\"reps\":%d,\"ndst\":%d,\"err\":\"%s\","
              "\"mismatches\":%lld,\"first_bad\":%lld,\"cycles\":%lld,\"mac_per_clk\":%.1f}\n",
              M, N, a_signed, b_signed, mode == 0 ? "tmem" : "smem", reps, ndst, cudaGetErrorString(e), bad, first,
              cyc, macs / double(cyc));
  if (first >= 0) {
    const int m = int(first / N), n = int(first % N);
    std::printf("  first mismatch (m=%d, n=%d): got %d\n", m, n, hD[first]);
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dc);
  return bad == 0 ? 0 : 1;
}

int main() {
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int as = 0; as < 2; ++as)
      for (int bs = 0; bs < 2; ++bs) fails += run<128, 32>(as, bs, mode, 1);
  fails += run<128, 64>(1, 0, 0, 1);
  // M = 64 (rank on M, fibers on N): issue rate only (mode 1, A from smem)
  run<64, 128>(1, 1, 1, 4096, 0);
  run<64, 192>(1, 1, 1, 4096, 0);
  run<128, 192>(1, 1, 1, 4096, 0);
  // issue rate vs N: unrolled issue (ndst 0), one accumulator chain, round-robin
  for (int mode = 0; mode < 2; ++mode) {
    run<128, 32>(1, 1, mode, 4096, 0);
    run<128, 64>(1, 1, mode, 4096, 0);
    run<128, 128>(1, 1, mode, 4096, 0);
    run<128, 32>(1, 1, mode, 4096);
    run<128, 64>(1, 1, mode, 4096);
    run<128, 128>(1, 1, mode, 4096);
    run<128, 256>(1, 1, mode, 2048);
    run<128, 32>(1, 1, mode, 4096, 7);
    run<128, 64>(1, 1, mode, 4096, 4);
    run<128, 128>(1, 1, mode, 4096, 3);
  }
  std::printf("fails=%d\n", fails);
  return 0;
}
