// TMA-fed, warp-specialised versions of the FC / FR fiber contractions.
//
// One producer warp streams tiles of the tensor and of the small operand
// into a multi-stage shared-memory ring with cp.async.bulk.tensor (TMA,
// SASS UTMALDG), synchronised by mbarrier full/empty pairs; eight consumer
// warps run mma.sync.m8n8k4.f64 (SASS DMMA) on fragments read from the ring.
// No __syncthreads in the main loop: each consumer warp waits only for the
// stage it needs, and the producer runs up to kStages stages ahead.
//
// Bank-conflict-free fragment reads without swizzle: every box is loaded
// with its inner extent padded by 4 elements (36 / 132 / NC+4 doubles), so a
// row pitch is 4 (mod 16) doubles and the 4 rows x 4 columns a half-warp
// touches land in 16 distinct 8-byte bank slots. The padding elements are
// either the next stage's data (an L2 re-read) or TMA out-of-bounds zeros,
// and are never used.
//
// Geometries (see common.cuh for the FiberView vocabulary):
//   FC kFibI : s == 1, contraction index contiguous  (mode 1)     A box 36 x 128
//   FC kFibJ : s % 128 == 0, fibers contiguous         (modes > 1)  A box 132 x 16
//   FR kFibI : s == 1                                               A box 132 x 32
//   FR kFibJ : s % 32 == 0                                           A box 36 x 128
// Other layouts use the register-streaming kernels in contract.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "contract.cuh"
#include "contract_tma.cuh"

namespace tkg {

namespace {

constexpr int kCons = 8;                 // consumer warps
constexpr int kThreadsTma = (kCons + 1) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE_%=;\n"
      "bra.uni WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                       int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------------------
// FC
// ---------------------------------------------------------------------------
template <int NC, int MODE>
struct FcT {
  static constexpr int kTF = 128;                       // fibers per tile (8 warps x 16)
  static constexpr int kKB = MODE == kFibI ? 32 : 16;   // contraction indices per stage
  static constexpr int kStages = MODE == kFibI ? 4 : 6;
  static constexpr int kLdA = MODE == kFibI ? 36 : 132; // padded inner extent of the A box
  static constexpr int kRowsA = MODE == kFibI ? kTF : kKB;
  static constexpr int kLdM = NC + 4;
  static constexpr int kBytesA = kRowsA * kLdA * 8;
  static constexpr int kBytesM = kKB * kLdM * 8;
  static constexpr int kStageBytes = ((kBytesA + kBytesM) + 127) / 128 * 128;
  static constexpr int kNT = NC / 8;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes;
};

template <int NC, int MODE>
__global__ void __launch_bounds__(kThreadsTma, 1)
    fc_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                  FcTmaArgs a) {
  using C = FcT<NC, MODE>;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + C::kStages;
  unsigned char* ring = smem_raw + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t F = a.s * a.P;
  const uint64_t ntiles = (F + C::kTF - 1) / C::kTF;
  const int nkb = int((a.K + C::kKB - 1) / C::kKB);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons) {
    // ---------------- producer ----------------
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmM);
      uint32_t it = 0;
      for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t j0 = tile * C::kTF;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int slot = it % C::kStages;
          const uint32_t ph = (it / C::kStages) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          unsigned char* st = ring + size_t(slot) * C::kStageBytes;
          mbar_arrive_expect_tx(&full[slot], C::kBytesA + C::kBytesM);
          if (MODE == kFibI) {
            tma_2d(st, &tmA, &full[slot], kb * C::kKB, int(j0));
          } else {
            const uint64_t p = j0 / a.s;
            const uint64_t jl = j0 - p * a.s;
            tma_3d(st, &tmA, &full[slot], int(jl), kb * C::kKB, int(p));
          }
          tma_2d(st + C::kBytesA, &tmM, &full[slot], 0, kb * C::kKB);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int q = lane & 3;
  const int r8 = lane >> 2;
  double sq_acc = 0.0;
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t j0 = tile * C::kTF;
    double acc[2][C::kNT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < C::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

    for (int kb = 0; kb < nkb; ++kb, ++it) {
      const int slot = it % C::kStages;
      const uint32_t ph = (it / C::kStages) & 1;
      mbar_wait(&full[slot], ph);
      const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes);
      const double* Ms = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes + C::kBytesA);
#pragma unroll
      for (int t = 0; t < C::kKB / 4; ++t) {
        const int kk = 4 * t + q;
        double af[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int row = warp * 16 + m * 8 + r8;
          af[m] = MODE == kFibI ? As[row * C::kLdA + kk] : As[kk * C::kLdA + row];
        }
        double bf[C::kNT];
#pragma unroll
        for (int n = 0; n < C::kNT; ++n) bf[n] = Ms[kk * C::kLdM + n * 8 + r8];
#pragma unroll
        for (int n = 0; n < C::kNT; ++n)
#pragma unroll
          for (int m = 0; m < 2; ++m) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    // epilogue straight from registers
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const uint64_t j = j0 + warp * 16 + m * 8 + r8;
      if (j >= F) continue;
      const uint64_t p = j / a.s;
      const uint64_t jl = j - p * a.s;
      const int64_t base = int64_t(jl * a.os_j + p * a.os_p);
#pragma unroll
      for (int n = 0; n < C::kNT; ++n) {
        const uint32_t c = n * 8 + 2 * q;
        const double v0 = acc[m][n][0], v1 = acc[m][n][1];
        if (a.diff_ref) {
          if (c < a.nc) {
            const double d = a.diff_ref[base + int64_t(c) * int64_t(a.os_c)] - v0;
            sq_acc += d * d;
          }
          if (c + 1 < a.nc) {
            const double d = a.diff_ref[base + int64_t(c + 1) * int64_t(a.os_c)] - v1;
            sq_acc += d * d;
          }
          continue;
        }
        if (a.os_c == 1 && c + 1 < a.nc && ((base + c) & 1) == 0) {
          *reinterpret_cast<double2*>(a.out + base + c) = make_double2(v0, v1);
        } else {
          if (c < a.nc) a.out[base + int64_t(c) * int64_t(a.os_c)] = v0;
          if (c + 1 < a.nc) a.out[base + int64_t(c + 1) * int64_t(a.os_c)] = v1;
        }
        if (a.sumsq_part) {
          if (c < a.nc) sq_acc += v0 * v0;
          if (c + 1 < a.nc) sq_acc += v1 * v1;
        }
      }
    }
  }
  if (a.sumsq_part) {
    __shared__ double red[kCons];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, off);
    if (lane == 0) red[warp] = sq_acc;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kCons; ++w) s += red[w];
      a.sumsq_part[blockIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// FR
// ---------------------------------------------------------------------------
template <int NC, int MODE, bool MCOL>
struct FrT {
  static constexpr int kIC = 128;   // contraction rows per CTA (8 warps x 16)
  static constexpr int kKB = 32;    // fibers per stage
  static constexpr int kStages = 4;
  static constexpr int kLdA = MODE == kFibI ? 132 : 36;
  static constexpr int kRowsA = MODE == kFibI ? kKB : kIC;
  // M row-major [F][ld]: box (NC+4, 32) -> [32][NC+4];
  // M column-major (F x r):  box (36, NC)  -> [NC][36]
  static constexpr int kLdM = MCOL ? 36 : NC + 4;
  static constexpr int kRowsM = MCOL ? NC : kKB;
  static constexpr int kBytesA = kRowsA * kLdA * 8;
  static constexpr int kBytesM = kRowsM * kLdM * 8;
  static constexpr int kStageBytes = ((kBytesA + kBytesM) + 127) / 128 * 128;
  static constexpr int kNT = NC / 8;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes;
};

template <int NC, int MODE, bool MCOL>
__global__ void __launch_bounds__(kThreadsTma, 1)
    fr_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                  FrTmaArgs a) {
  using C = FrT<NC, MODE, MCOL>;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + C::kStages;
  unsigned char* ring = smem_raw + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t F = a.s * a.P;
  const uint32_t range = blockIdx.x / a.igroups;
  const uint32_t ig = blockIdx.x % a.igroups;
  const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
  const uint64_t f1 = min(F, f0 + a.fibers_per_range);
  const int nkb = f1 > f0 ? int((f1 - f0 + C::kKB - 1) / C::kKB) : 0;
  const int i0 = int(ig) * C::kIC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons) {
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmM);
      for (int kb = 0; kb < nkb; ++kb) {
        const int slot = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        mbar_wait(&empty[slot], ph ^ 1);
        unsigned char* st = ring + size_t(slot) * C::kStageBytes;
        const uint64_t j = f0 + uint64_t(kb) * C::kKB;
        mbar_arrive_expect_tx(&full[slot], C::kBytesA + C::kBytesM);
        if (MODE == kFibI) {
          tma_2d(st, &tmA, &full[slot], i0, int(j));
        } else {
          const uint64_t p = j / a.s;
          const uint64_t jl = j - p * a.s;
          tma_3d(st, &tmA, &full[slot], int(jl), i0, int(p));
        }
        if (MCOL) tma_2d(st + C::kBytesA, &tmM, &full[slot], int(j), 0);
        else tma_2d(st + C::kBytesA, &tmM, &full[slot], 0, int(j));
      }
    }
    return;
  }

  const int q = lane & 3;
  const int r8 = lane >> 2;
  double acc[2][C::kNT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < C::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  double sq_acc = 0.0;
  const bool want_sq = a.sumsq_part != nullptr;

  for (int kb = 0; kb < nkb; ++kb) {
    const int slot = kb % C::kStages;
    const uint32_t ph = (kb / C::kStages) & 1;
    mbar_wait(&full[slot], ph);
    const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes);
    const double* Ms = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes + C::kBytesA);
    // Fibers past f1 in the last stage belong to the next range: drop them.
    const uint64_t left = f1 - (f0 + uint64_t(kb) * C::kKB);
    const int kvalid = left < uint64_t(C::kKB) ? int(left) : C::kKB;
#pragma unroll
    for (int t = 0; t < C::kKB / 4; ++t) {
      const int kk = 4 * t + q;
      const bool kok = kk < kvalid;
      double af[2];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = warp * 16 + m * 8 + r8;
        const double v = MODE == kFibI ? As[kk * C::kLdA + row] : As[row * C::kLdA + kk];
        af[m] = kok ? v : 0.0;
        if (want_sq) sq_acc = fma(af[m], af[m], sq_acc);
      }
      double bf[C::kNT];
#pragma unroll
      for (int n = 0; n < C::kNT; ++n)
        bf[n] = MCOL ? Ms[(n * 8 + r8) * C::kLdM + kk] : Ms[kk * C::kLdM + n * 8 + r8];
#pragma unroll
      for (int n = 0; n < C::kNT; ++n)
#pragma unroll
        for (int m = 0; m < 2; ++m) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  // partial rows of this CTA
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int i = i0 + warp * 16 + m * 8 + r8;
    if (i >= int(a.K)) continue;
    double* dst = a.partial + (size_t(range) * a.K + i) * a.ncp;
#pragma unroll
    for (int n = 0; n < C::kNT; ++n) {
      const int c = n * 8 + 2 * q;
      *reinterpret_cast<double2*>(dst + c) = make_double2(acc[m][n][0], acc[m][n][1]);
    }
  }
  if (want_sq) {
    __shared__ double red[kCons];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, off);
    if (lane == 0) red[warp] = sq_acc;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kCons; ++w) s += red[w];
      a.sumsq_part[blockIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

bool encode(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
            const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int k = 0; k < rank; ++k) {
    gd[k] = dims[k];
    bx[k] = box[k];
    es[k] = 1;
    if (k + 1 < rank) gs[k] = strides[k];
  }
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), gd, gs, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <class K>
cudaError_t set_smem(K k, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

template <int NC, int MODE>
cudaError_t fc_tma_launch(const CUtensorMap& A, const CUtensorMap& M, const FcTmaArgs& a, int grid,
                          cudaStream_t st) {
  using C = FcT<NC, MODE>;
  auto k = fc_tma_kernel<NC, MODE>;
  static bool done = false;
  if (!done) {
    cudaError_t e = set_smem(k, C::kSmem);
    if (e != cudaSuccess) return e;
    done = true;
  }
  k<<<grid, kThreadsTma, C::kSmem, st>>>(A, M, a);
  return cudaGetLastError();
}

template <int NC, int MODE, bool MCOL>
cudaError_t fr_tma_launch(const CUtensorMap& A, const CUtensorMap& M, const FrTmaArgs& a, int grid,
                          cudaStream_t st) {
  using C = FrT<NC, MODE, MCOL>;
  auto k = fr_tma_kernel<NC, MODE, MCOL>;
  static bool done = false;
  if (!done) {
    cudaError_t e = set_smem(k, C::kSmem);
    if (e != cudaSuccess) return e;
    done = true;
  }
  k<<<grid, kThreadsTma, C::kSmem, st>>>(A, M, a);
  return cudaGetLastError();
}

#define TKG_NC_SWITCH(ncp, CALL)            \
  switch (ncp) {                            \
    case 8: return CALL(8);                 \
    case 16: return CALL(16);               \
    case 24: return CALL(24);               \
    case 32: return CALL(32);               \
    case 40: return CALL(40);               \
    case 48: return CALL(48);               \
    case 56: return CALL(56);               \
    case 64: return CALL(64);               \
    default: return cudaErrorInvalidValue;  \
  }

}  // namespace

int fc_tma_mode(const FiberView& v, const double* mt, uint32_t ldmt) {
  if (!encode_fn() || !aligned16(v.base) || !aligned16(mt) || (ldmt % 2) != 0) return -1;
  if (v.s * v.P >= (1ull << 31) || v.K >= (1u << 31)) return -1;
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0) return kFibI;
  if (v.s % 128 == 0 && v.is_i % 2 == 0 && v.is_p % 2 == 0 && v.P < (1ull << 31)) return kFibJ;
  return -1;
}

int fr_tma_mode(const FiberView& v, const double* m, uint64_t mj, uint64_t mc) {
  // M(j, c) = m[j*mj + c*mc]: row-major (mc == 1) or column-major (mj == 1)
  const uint64_t ld = mc == 1 ? mj : (mj == 1 ? mc : 1);
  if (!encode_fn() || !aligned16(v.base) || !aligned16(m) || (ld % 2) != 0) return -1;
  if (v.s * v.P >= (1ull << 31)) return -1;
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0) return kFibI;
  if (v.s % 32 == 0 && v.is_i % 2 == 0 && v.is_p % 2 == 0 && v.P < (1ull << 31)) return kFibJ;
  return -1;
}

int fc_tma_grid(const FiberView& v, int num_sms) {
  const uint64_t tiles = (v.s * v.P + 127) / 128;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms))));
}

cudaError_t launch_fc_tma(const FiberView& v, const double* mt, uint32_t ldmt, FcTmaArgs a, int mode,
                          int num_sms, cudaStream_t st, int* grid_used) {
  const uint32_t ncp = pad_nc(a.nc);
  CUtensorMap A, M;
  const int KB = mode == kFibI ? 32 : 16;
  if (mode == kFibI) {
    const uint64_t dims[2] = {v.K, v.s * v.P};
    const uint64_t strides[1] = {v.is_p * 8};
    const uint32_t box[2] = {36, 128};
    if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {132, 16, 1};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {ncp, v.K};
    const uint64_t strides[1] = {uint64_t(ldmt) * 8};
    const uint32_t box[2] = {ncp + 4, uint32_t(KB)};
    if (!encode(&M, mt, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  a.s = v.s;
  a.P = v.P;
  a.K = v.K;
  const int grid = fc_tma_grid(v, num_sms);
  if (grid_used) *grid_used = grid;
#define TKG_FC_CALL(N) (mode == kFibI ? fc_tma_launch<N, kFibI>(A, M, a, grid, st) \
                                      : fc_tma_launch<N, kFibJ>(A, M, a, grid, st))
  TKG_NC_SWITCH(ncp, TKG_FC_CALL)
#undef TKG_FC_CALL
}

cudaError_t launch_fr_tma(const FiberView& v, const double* m, uint64_t mj, uint64_t mc, FrTmaArgs a,
                          int mode, int num_sms, cudaStream_t st, uint32_t* ranges_used,
                          uint32_t* grid_used) {
  const bool mcol = mc != 1;
  const uint32_t ncp = pad_nc(a.nc);
  CUtensorMap A, M;
  const uint64_t F = v.s * v.P;
  if (mode == kFibI) {
    const uint64_t dims[2] = {v.K, F};
    const uint64_t strides[1] = {v.is_p * 8};
    const uint32_t box[2] = {132, 32};
    if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {36, 128, 1};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  if (!mcol) {
    const uint64_t dims[2] = {ncp, F};
    const uint64_t strides[1] = {mj * 8};
    const uint32_t box[2] = {ncp + 4, 32};
    if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const uint64_t dims[2] = {F, a.nc};
    const uint64_t strides[1] = {mc * 8};
    const uint32_t box[2] = {36, ncp};
    if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  a.s = v.s;
  a.P = v.P;
  a.K = v.K;
  a.ncp = ncp;
  a.igroups = (v.K + 127) / 128;
  const uint64_t steps = (F + 31) / 32;
  uint64_t ranges = std::max<uint64_t>(1, uint64_t(num_sms) / a.igroups);
  ranges = std::min<uint64_t>(ranges, std::max<uint64_t>(1, steps / 4));
  a.fibers_per_range = (steps + ranges - 1) / ranges * 32;
  a.ranges = uint32_t((F + a.fibers_per_range - 1) / a.fibers_per_range);
  if (ranges_used) *ranges_used = a.ranges;
  const int grid = int(a.ranges * a.igroups);
  if (grid_used) *grid_used = grid;
#define TKG_FR_CALL(N)                                                                      \
  (mode == kFibI ? (mcol ? fr_tma_launch<N, kFibI, true>(A, M, a, grid, st)                   \
                         : fr_tma_launch<N, kFibI, false>(A, M, a, grid, st))                 \
                 : (mcol ? fr_tma_launch<N, kFibJ, true>(A, M, a, grid, st)                   \
                         : fr_tma_launch<N, kFibJ, false>(A, M, a, grid, st)))
  TKG_NC_SWITCH(ncp, TKG_FR_CALL)
#undef TKG_FR_CALL
}

uint32_t fr_tma_ranges(const FiberView& v, int num_sms) {
  const uint64_t F = v.s * v.P;
  const uint32_t igroups = (v.K + 127) / 128;
  const uint64_t steps = (F + 31) / 32;
  uint64_t ranges = std::max<uint64_t>(1, uint64_t(num_sms) / igroups);
  ranges = std::min<uint64_t>(ranges, std::max<uint64_t>(1, steps / 4));
  const uint64_t fpr = (steps + ranges - 1) / ranges * 32;
  return uint32_t((F + fpr - 1) / fpr);
}

}  // namespace tkg
