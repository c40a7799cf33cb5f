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
//   FC kFibJ : s even, s % 128 == 0 or s >= 1024      (modes > 1)  A box 132 x 32
//   FR kFibI : s == 1                                               A box 132 x 32
//   FR kFibJ : s even, s % 32 == 0 or s >= 128                      A box 68 x 128
// kFibJ tiles / chunks stay inside one panel p (TMA zero-fills past s).
// Other layouts use the register-streaming kernels in contract.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "contract.cuh"
#include "contract_tma.cuh"
#include "tma_util.cuh"

namespace tkg {

namespace {


// ---------------------------------------------------------------------------
// FC
// ---------------------------------------------------------------------------
template <int NC, int MODE>
struct FcT {
  static constexpr int kTF = 128;                       // fibers per tile (8 warps x 16)
  static constexpr int kKB = 32;                         // contraction indices per stage
  static constexpr int kStages = MODE == kFibS ? 3 : 4;
  static constexpr int kLdA = MODE == kFibI ? 36 : 132; // padded inner extent of the A box
  static constexpr int kRowsA = MODE == kFibI ? kTF : kKB;
  static constexpr int kLdM = NC + 4;
  // kFibS: the A box is {sb, 32, pc} with pc*sb <= 208 (runtime size)
  static constexpr int kBytesA = MODE == kFibS ? kKB * 208 * 8 : kRowsA * kLdA * 8;
  static constexpr int kBytesM = kKB * kLdM * 8;
  static constexpr int kStageBytes = ((kBytesA + kBytesM) + 127) / 128 * 128;
  static constexpr int kNT = NC / 8;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes;
};

// TAIL = 2: the last column tile holds only 1-2 real columns (r mod 8 in
// {1, 2}); they are accumulated with DFMAs on each lane's own k index (two per
// row tile and k-step, summed over the 4 k lanes once per tile) instead of a
// whole DMMA tile: DMMA and DFMA issue to the same FP64 pipe, a DMMA costing
// 8 DFMAs, so r = 10 spends 8+2 columns' worth of the pipe instead of 16 and
// r = 50 48+2 instead of 56 (tools/mix_fp64_probe.cu).
template <int TAIL>
__device__ __forceinline__ void tail_to_tile(double (&t)[2], double& a0, double& a1, int q) {
  double v0 = t[0], v1 = t[1];
  v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
  v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
  // accumulator-tile layout: lane (r8, q) holds columns 2q, 2q+1 of row r8
  a0 = q == 0 ? v0 : 0.0;
  a1 = q == 0 ? v1 : 0.0;
}

template <int NC, int MODE, int TAIL>
__global__ void __launch_bounds__(kThreadsTma, 1)
    fc_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                  FcTmaArgs a) {
  using C = FcT<NC, MODE>;
  constexpr int kND = TAIL ? C::kNT - 1 : C::kNT;  // column tiles on DMMA
  // launched with programmatic stream serialization: this grid's launch
  // overlaps the tail of the previous kernel; wait for its results here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + C::kStages;
  unsigned char* ring = smem_raw + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t F = a.s * a.P;
  // kFibJ tiles never cross a panel: tile t covers fibers jl0 .. jl0+127 of
  // panel p (rows past s are TMA zero-fill and are not stored)
  const uint64_t tpp = MODE == kFibJ ? (a.s + C::kTF - 1) / C::kTF : 1;
  // kFibS tiles are a.pc whole panels (a.pc * s <= 128 fibers)
  const bool strad = MODE == kFibS && a.straddle != 0;
  const uint64_t ntiles = MODE == kFibJ   ? tpp * a.P
                          : MODE == kFibS ? (strad ? (F + C::kTF - 1) / C::kTF : (a.P + a.pc - 1) / a.pc)
                                          : (F + C::kTF - 1) / C::kTF;
  const int nkb = int((a.K + C::kKB - 1) / C::kKB);
  const int stage_bytes = MODE == kFibS ? int(a.stage_bytes) : C::kStageBytes;
  const int bytes_a = MODE == kFibS ? int(a.bytes_a) : C::kBytesA;

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
        const uint64_t tp = tile / tpp, jl0 = (tile - tp * tpp) * C::kTF;
        const uint64_t j0 = tile * C::kTF;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int slot = it % C::kStages;
          const uint32_t ph = (it / C::kStages) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          unsigned char* st = ring + size_t(slot) * stage_bytes;
          mbar_arrive_expect_tx(&full[slot], bytes_a + C::kBytesM);
          if (MODE == kFibI) {
            tma_2d(st, &tmA, &full[slot], kb * C::kKB, int(j0));
          } else if (MODE == kFibJ) {
            tma_3d(st, &tmA, &full[slot], int(jl0), kb * C::kKB, int(tp));
          } else {
            tma_3d(st, &tmA, &full[slot], 0, kb * C::kKB, strad ? int(j0 / a.s) : int(tile * a.pc));
          }
          tma_2d(st + bytes_a, &tmM, &full[slot], 0, kb * C::kKB);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int q = lane & 3;
  const int r8 = lane >> 2;
  // kFibS: tile row m is fiber jl = m % s of panel m / s of the tile; its A
  // column kk sits at (panel*kKB + kk)*sb + jl
  int offS[2] = {0, 0};
  bool okS[2] = {true, true};
  uint32_t pS[2] = {0, 0}, jlS[2] = {0, 0};  // straddling tiles: panel and in-panel index of the rows
  if (MODE == kFibS && !strad) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int row = warp * 16 + m * 8 + r8;
      const int pcm = row / int(a.s), jl = row - pcm * int(a.s);
      okS[m] = pcm < int(a.pc);
      offS[m] = okS[m] ? (pcm * C::kKB) * int(a.sb) + jl : 0;
    }
  }
  double sq_acc = 0.0;
  // Gram of the output rows (fused epilogue): upper 8x8 tiles (tm <= tn)
  constexpr bool kGram = NC <= int(kFcGramMaxNc);
  constexpr int kTri = kGram ? C::kNT * (C::kNT + 1) / 2 : 1;
  double gacc[kTri][2];
#pragma unroll
  for (int t = 0; t < kTri; ++t) gacc[t][0] = gacc[t][1] = 0.0;
  const bool want_gram = kGram && a.gram_part != nullptr;
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t tp = tile / tpp, jl0 = (tile - tp * tpp) * C::kTF;
    const uint64_t j0 = tile * C::kTF;
    double acc[2][C::kNT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < C::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    double tl[2][2] = {{0.0, 0.0}, {0.0, 0.0}};

    if (strad) {
      // row m of the tile is fiber j0 + m: panel j / s (the box starts at the
      // panel of j0), in-panel index j % s
      const uint32_t p0 = uint32_t(j0 / a.s);
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const uint64_t j = j0 + uint64_t(warp * 16 + m * 8 + r8);
        okS[m] = j < F;
        pS[m] = uint32_t(j) / uint32_t(a.s);
        jlS[m] = uint32_t(j) - pS[m] * uint32_t(a.s);
        offS[m] = okS[m] ? int((pS[m] - p0) * C::kKB) * int(a.sb) + int(jlS[m]) : 0;
      }
    }
    // warps whose 16 rows are all past the tile's fibers have nothing to add
    const bool wact = MODE == kFibS   ? (strad ? j0 + uint64_t(warp * 16) < F : uint64_t(warp * 16) < a.pc * a.s)
                      : MODE == kFibJ ? jl0 + uint64_t(warp * 16) < a.s
                                      : j0 + uint64_t(warp * 16) < F;
    for (int kb = 0; kb < nkb; ++kb, ++it) {
      const int slot = it % C::kStages;
      const uint32_t ph = (it / C::kStages) & 1;
      mbar_wait(&full[slot], ph);
      const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * stage_bytes);
      const double* Ms = reinterpret_cast<const double*>(ring + size_t(slot) * stage_bytes + bytes_a);
      // the last block of a contraction extent that is not a multiple of kKB:
      // k-steps past K only add TMA zero-fill
      const int kleft = wact ? int(a.K) - kb * C::kKB : 0;
      auto kstep = [&](int t) {
        const int kk = 4 * t + q;
        double af[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int row = warp * 16 + m * 8 + r8;
          if (MODE == kFibS) af[m] = okS[m] ? As[offS[m] + kk * int(a.sb)] : 0.0;
          else af[m] = MODE == kFibI ? As[row * C::kLdA + kk] : As[kk * C::kLdA + row];
        }
        double bf[kND > 0 ? kND : 1];
#pragma unroll
        for (int n = 0; n < kND; ++n) bf[n] = Ms[kk * C::kLdM + n * 8 + r8];
#pragma unroll
        for (int n = 0; n < kND; ++n)
#pragma unroll
          for (int m = 0; m < 2; ++m) dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
        if constexpr (TAIL != 0) {
          const double2 bt = *reinterpret_cast<const double2*>(Ms + kk * C::kLdM + kND * 8);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            tl[m][0] = fma(af[m], bt.x, tl[m][0]);
            tl[m][1] = fma(af[m], bt.y, tl[m][1]);
          }
        }
      };
      if (kleft >= C::kKB) {  // full block: the straight unrolled path
#pragma unroll
        for (int t = 0; t < C::kKB / 4; ++t) kstep(t);
      } else {
#pragma unroll
        for (int t = 0; t < C::kKB / 4; ++t)
          if (4 * t < kleft) kstep(t);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    if constexpr (TAIL != 0) {
#pragma unroll
      for (int m = 0; m < 2; ++m) tail_to_tile<TAIL>(tl[m], acc[m][kND][0], acc[m][kND][1], q);
    }

    // Gram epilogue: G[c1][c2] += sum_rows R[row][c1] R[row][c2] as DMMAs on
    // fragments rebuilt from the accumulators by shuffles. Fragment t for
    // rows m*8+k0..+3: lane (r8, q) needs R[m*8+k0+q][t*8+r8], held by lane
    // 4*(k0+q) + r8/2 as element r8&1 of acc[m][t]. Rows past F are TMA
    // zero-fill, so they add nothing.
    if constexpr (kGram) {
      if (want_gram) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
#pragma unroll
          for (int k0 = 0; k0 < 8; k0 += 4) {
            const int src = 4 * (k0 + q) + (r8 >> 1);
            double fr[C::kNT];
#pragma unroll
            for (int t = 0; t < C::kNT; ++t) {
              const double v0 = __shfl_sync(0xffffffffu, acc[m][t][0], src);
              const double v1 = __shfl_sync(0xffffffffu, acc[m][t][1], src);
              fr[t] = (r8 & 1) ? v1 : v0;
            }
            int idx = 0;
#pragma unroll
            for (int tm = 0; tm < C::kNT; ++tm)
#pragma unroll
              for (int tn = tm; tn < C::kNT; ++tn, ++idx) dmma(gacc[idx][0], gacc[idx][1], fr[tm], fr[tn]);
          }
        }
      }
    }

    // epilogue straight from registers
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      uint64_t p, jl;
      if (MODE == kFibJ) {
        p = tp;
        jl = jl0 + warp * 16 + m * 8 + r8;
        if (jl >= a.s) continue;
      } else if (MODE == kFibS) {
        if (!okS[m]) continue;
        if (strad) {
          p = pS[m];
          jl = jlS[m];
        } else {
          const int row = warp * 16 + m * 8 + r8;
          const uint64_t pcm = uint64_t(row) / a.s;
          p = tile * a.pc + pcm;
          jl = uint64_t(row) - pcm * a.s;
        }
        if (p >= a.P) continue;
      } else {
        const uint64_t j = j0 + warp * 16 + m * 8 + r8;
        if (j >= F) continue;
        p = j / a.s;
        jl = j - p * a.s;
      }
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
  if constexpr (kGram) {
    if (want_gram) {
      // every stage has been consumed, so the ring is free: per-warp partials
      // there, then a fixed-order sum over the 8 warps (deterministic)
      asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
      double* gs = reinterpret_cast<double*>(ring);
#pragma unroll
      for (int t = 0; t < kTri; ++t) {
        gs[(warp * kTri + t) * 64 + lane * 2] = gacc[t][0];
        gs[(warp * kTri + t) * 64 + lane * 2 + 1] = gacc[t][1];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
      double* out = a.gram_part + size_t(blockIdx.x) * NC * NC;
      for (int e = threadIdx.x; e < kTri * 64; e += kCons * 32) {
        double s = 0.0;
        for (int w = 0; w < kCons; ++w) s += gs[w * kTri * 64 + e];
        const int t = e / 64, l = (e % 64) / 2, el = e % 2;
        int tm = 0, rem = t;
        while (rem >= C::kNT - tm) {
          rem -= C::kNT - tm;
          ++tm;
        }
        const int tn = tm + rem;
        out[(tm * 8 + (l >> 2)) * NC + tn * 8 + 2 * (l & 3) + el] = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// FR
// ---------------------------------------------------------------------------
template <int NC, int MODE, bool MCOL>
struct FrT {
  static constexpr int kIC = 128;   // contraction rows per CTA (8 warps x 16)
  // fibers per stage: kFibJ boxes read kKB+4 contiguous fibers of 128 rows,
  // so longer runs per row (64) and a double-buffered ring
  // kFibS (short panels): a chunk is pc whole panels, kf = pc*s <= 64 fibers
  static constexpr int kKB = MODE == kFibI ? 32 : 64;
  // kFibI with NC <= 32: two CTAs per SM with two stages each (a grid of
  // exactly 2 x #SMs = ranges x row groups fills every SM; one CTA per SM
  // left SMs idle when #SMs is not a multiple of the row-group count)
  static constexpr int kStages = MODE == kFibI ? (NC <= 32 ? 2 : 4) : 2;
  static constexpr int kLdA = MODE == kFibI ? 132 : kKB + 4;
  static constexpr int kRowsA = MODE == kFibI ? kKB : kIC;
  // M row-major [F][ld]: box (NC+4, kKB) -> [kKB][NC+4];
  // M column-major (F x r):  box (kKB+4, NC)  -> [NC][kKB+4]
  static constexpr int kLdM = MCOL ? kKB + 4 : NC + 4;
  static constexpr int kRowsM = MCOL ? NC : kKB;
  static constexpr int kBytesA = MODE == kFibS ? kIC * 64 * 8 : kRowsA * kLdA * 8;  // kFibS: max
  static constexpr int kBytesM = kRowsM * kLdM * 8;
  static constexpr int kStageBytes = ((kBytesA + kBytesM) + 127) / 128 * 128;
  static constexpr int kNT = NC / 8;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes;
};

template <int NC, int MODE, bool MCOL, int TAIL>
__global__ void __launch_bounds__(kThreadsTma, (MODE == kFibI && NC <= 32) ? 2 : 1)
    fr_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                  FrTmaArgs a) {
  using C = FrT<NC, MODE, MCOL>;
  constexpr int kND = TAIL ? C::kNT - 1 : C::kNT;  // column tiles on DMMA (see fc_tma_kernel)
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see fc_tma_kernel
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + C::kStages;
  unsigned char* ring = smem_raw + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t F = a.s * a.P;
  // persistent CTAs: work item = (fiber range, row group); the ring runs on
  // across items
  const uint32_t items = a.ranges * a.igroups;
  // fiber chunks of up to kKB that never cross a panel (kFibJ): the chunk
  // starting at j holds min(kKB, end of j's panel or of the range - j) fibers
  // kFibS: ranges are whole panels and chunks a.kf = a.pc * s fibers, so a
  // chunk is a.pc whole panels (the last one of a range may be shorter)
  const int kmax = MODE == kFibS ? int(a.kf) : C::kKB;
  auto chunk_len = [&](uint64_t j, uint64_t f1) -> int {
    uint64_t end = f1;
    if (MODE == kFibJ) {
      const uint64_t pe = (j / a.s + 1) * a.s;
      end = pe < end ? pe : end;
    }
    return end - j < uint64_t(kmax) ? int(end - j) : kmax;
  };
  const int stage_bytes = MODE == kFibS ? int(a.stage_bytes) : C::kStageBytes;
  const int bytes_a = MODE == kFibS ? int(a.bytes_a) : C::kBytesA;
  const int bytes_m = MODE == kFibS ? int(a.bytes_m) : C::kBytesM;
  const int ldm = MODE == kFibS && MCOL ? int(a.ldm) : C::kLdM;

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
      int kb = 0;
      for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
        const uint32_t range = item / a.igroups, ig = item % a.igroups;
        const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
        const uint64_t f1 = min(F, f0 + a.fibers_per_range);
        const int i0 = int(ig) * C::kIC;
      for (uint64_t j = f0; j < f1; j += chunk_len(j, f1), ++kb) {
        const int slot = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        mbar_wait(&empty[slot], ph ^ 1);
        unsigned char* st = ring + size_t(slot) * stage_bytes;
        mbar_arrive_expect_tx(&full[slot], bytes_a + bytes_m);
        if (MODE == kFibI) {
          tma_2d(st, &tmA, &full[slot], i0, int(j));
        } else {
          const uint64_t p = j / a.s;
          const uint64_t jl = j - p * a.s;
          tma_3d(st, &tmA, &full[slot], int(jl), i0, int(p));
        }
        if (MCOL) tma_2d(st + bytes_a, &tmM, &full[slot], int(j), 0);
        else tma_2d(st + bytes_a, &tmM, &full[slot], 0, int(j));
      }
      }
    }
    return;
  }

  const int q = lane & 3;
  const int r8 = lane >> 2;
  // ||A||^2 of the init pass in 4 independent chains (a single chain of
  // dependent DFMAs between the DMMAs stalls the warp's in-order issue)
  double sq_acc[4] = {0.0, 0.0, 0.0, 0.0};
  const bool want_sq = a.sumsq_part != nullptr;
  // kFibS: fiber kk of a chunk is jl = kk % s of panel kk / s; its A rows sit
  // at ((kk / s)*128 + row)*s + jl
  int koff[C::kKB / 4];
#pragma unroll
  for (int t = 0; t < C::kKB / 4; ++t) {
    const int kk = 4 * t + q;
    const int pc = MODE == kFibS ? kk / int(a.s) : 0;
    koff[t] = MODE == kFibS ? pc * C::kIC * int(a.s) + (kk - pc * int(a.s)) : 0;
  }

  int kb = 0;
  for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
  const uint32_t range = item / a.igroups, ig = item % a.igroups;
  const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
  const uint64_t f1 = min(F, f0 + a.fibers_per_range);
  const int i0 = int(ig) * C::kIC;
  const bool wact = i0 + warp * 16 < int(a.K), m1act = i0 + warp * 16 + 8 < int(a.K);
  double acc[2][C::kNT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < C::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  double tl[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (uint64_t j = f0; j < f1; ++kb) {
    const int slot = kb % C::kStages;
    const uint32_t ph = (kb / C::kStages) & 1;
    mbar_wait(&full[slot], ph);
    const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * stage_bytes);
    const double* Ms = reinterpret_cast<const double*>(ring + size_t(slot) * stage_bytes + bytes_a);
    // fibers past the chunk (next panel / next range) are dropped; warps whose
    // rows are all past the contraction extent skip the chunk
    const int kvalid = chunk_len(j, f1);
    j += kvalid;
    const int kuse = wact ? kvalid : 0;
    auto kstep = [&](int t, bool m1) {
      const int kk = 4 * t + q;
      const bool kok = kk < kvalid;
      double af[2];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = warp * 16 + m * 8 + r8;
        double v;
        if (MODE == kFibS) v = kok ? As[koff[t] + row * int(a.s)] : 0.0;
        else v = MODE == kFibI ? As[kk * C::kLdA + row] : As[row * C::kLdA + kk];
        af[m] = kok ? v : 0.0;
        if (want_sq) sq_acc[(t & 1) * 2 + m] = fma(af[m], af[m], sq_acc[(t & 1) * 2 + m]);
      }
      double bf[kND > 0 ? kND : 1];
#pragma unroll
      for (int n = 0; n < kND; ++n) {
        if (MODE == kFibS) {  // rows past the chunk are not loaded: keep them finite
          const double v = MCOL ? Ms[(n * 8 + r8) * ldm + kk] : Ms[kk * C::kLdM + n * 8 + r8];
          bf[n] = kok ? v : 0.0;
        } else {
          bf[n] = MCOL ? Ms[(n * 8 + r8) * C::kLdM + kk] : Ms[kk * C::kLdM + n * 8 + r8];
        }
      }
#pragma unroll
      for (int n = 0; n < kND; ++n) {
        dmma(acc[0][n][0], acc[0][n][1], af[0], bf[n]);
        if (m1) dmma(acc[1][n][0], acc[1][n][1], af[1], bf[n]);
      }
      if constexpr (TAIL != 0) {
        double2 bt;
        if (MCOL) {
          const int l = MODE == kFibS ? ldm : C::kLdM;
          bt = make_double2(Ms[(kND * 8) * l + kk], Ms[(kND * 8 + 1) * l + kk]);
        } else {
          bt = *reinterpret_cast<const double2*>(Ms + kk * C::kLdM + kND * 8);
        }
        if (MODE == kFibS && !kok) bt = make_double2(0.0, 0.0);
        tl[0][0] = fma(af[0], bt.x, tl[0][0]);
        tl[0][1] = fma(af[0], bt.y, tl[0][1]);
        if (m1) {
          tl[1][0] = fma(af[1], bt.x, tl[1][0]);
          tl[1][1] = fma(af[1], bt.y, tl[1][1]);
        }
      }
    };
    if (kuse == C::kKB && m1act) {  // full chunk, both row tiles live: the straight path
#pragma unroll
      for (int t = 0; t < C::kKB / 4; ++t) kstep(t, true);
    } else {
#pragma unroll
      for (int t = 0; t < C::kKB / 4; ++t)
        if (4 * t < kuse) kstep(t, m1act);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  if constexpr (TAIL != 0) {
#pragma unroll
    for (int m = 0; m < 2; ++m) tail_to_tile<TAIL>(tl[m], acc[m][kND][0], acc[m][kND][1], q);
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
  }  // item
  if (want_sq) {
    __shared__ double red[kCons];
    double sq = (sq_acc[0] + sq_acc[1]) + (sq_acc[2] + sq_acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[warp] = sq;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kCons; ++w) s += red[w];
      a.sumsq_part[blockIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// FR for 128 < K <= 248 rows (e.g. a 200^4 tensor's modes 1..4): ONE CTA
// covers all K contraction rows, so R (or S) is streamed once per pass
// instead of once per 128-row group, and the 8 consumer warps share the
// MT = ceil(K/8) row tiles evenly: warp w owns the full row tiles w, w+8, ...
// (all NC/8 column tiles, base = MT/8 of them) plus every 8th (row tile,
// column tile) pair of the MT % 8 remainder tiles. For K = 200 that is
// 3 x 7 + 1 DMMA tiles per warp (22 each, 175 in all), where two 128-row
// groups left the second group's SM sub-partitions a third idle.
// A stage (rows past K are TMA zero-fill):
//   kFibI (s = 1)      : 16 fibers, two 132-row boxes [16][132] (rows 0.., 128..)
//   kFibJ (s >= 64)    : up to 32 fibers of one panel, box [K][36]
//   kFibS (32 <= s <= 64): one whole panel of s fibers, box [K][sb]
// ---------------------------------------------------------------------------
template <int NC, int MODE, bool MCOL>
struct FrW {
  static constexpr int kMaxKB = MODE == kFibI ? 16 : MODE == kFibJ ? 32 : 64;  // fibers per stage
  static constexpr int kNT = NC / 8;
  static constexpr int kRemP = 2;  // remainder pairs per warp (register budget)
};

struct FrWideGeom {
  uint32_t lda = 0;        // A row pitch in smem (doubles): 132 (kFibI), 36 (kFibJ), sb (kFibS)
  uint32_t kb = 0;         // fibers per stage (kFibS: s)
  uint32_t bytes_a = 0, bytes_m = 0, stage_bytes = 0, stages = 0, ldm = 0;
};

// REBAL: launched with 12 warps: the 8 consumer warps (warpgroups 0 and 1), the
// producer warp and three idle warps that fill its warpgroup. The producer's
// warpgroup hands its registers back (setmaxnreg.dec) and the consumers take
// them (setmaxnreg.inc: 168 -> 232 per thread), which is what the 3 full row
// tiles + 2 remainder pairs + DFMA tail of a warp need without spills.
// REBAL = false keeps the 9-warp launch at 168 registers (no tail): the
// mode-1 left update (kFibI, row-major R) measured faster that way (c5:
// 5.45 ms against 6.00 ms rebalanced, 5.79 ms rebalanced with the tail),
// every other variant faster rebalanced (c5 mode 2: 1.51 -> 1.40 ms, init
// passes 6.43 -> 5.94 ms and 1.59 -> 1.46 ms).
constexpr int kThreadsWide = 12 * 32;

template <int NC, int MODE, bool MCOL, int TAIL, bool REBAL>
__global__ void __launch_bounds__(REBAL ? kThreadsWide : kThreadsTma, 1)
    fr_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                   FrTmaArgs a, FrWideGeom g) {
  using C = FrW<NC, MODE, MCOL>;
  constexpr int kNT = C::kNT;
  // column tiles on DMMA; with TAIL the last tile's 1-2 real columns run as
  // DFMAs (see fc_tma_kernel). The remainder pairs then cover the kND DMMA
  // tiles of a remainder row tile, and the warp holding its column tile 0
  // also accumulates that row tile's tail.
  constexpr int kND = TAIL ? kNT - 1 : kNT;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see fc_tma_kernel
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 4;
  unsigned char* ring = smem_raw + 1024;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t F = a.s * a.P;
  const int stages = int(g.stages);
  // fibers of the stage starting at j: never past the range end, and (kFibJ)
  // never past the panel end; kFibS stages are whole panels
  auto chunk_len = [&](uint64_t j, uint64_t f1) -> int {
    uint64_t end = f1;
    if (MODE == kFibJ) {
      const uint64_t pe = (j / a.s + 1) * a.s;
      end = pe < end ? pe : end;
    }
    return end - j < uint64_t(g.kb) ? int(end - j) : int(g.kb);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= kCons) {
    if constexpr (REBAL) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    if (warp == kCons && lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmM);
      int kb = 0;
      for (uint32_t range = blockIdx.x; range < a.ranges; range += gridDim.x) {
        const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
        const uint64_t f1 = min(F, f0 + a.fibers_per_range);
        for (uint64_t j = f0; j < f1; j += chunk_len(j, f1), ++kb) {
          const int slot = kb % stages;
          const uint32_t ph = (kb / stages) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          unsigned char* st = ring + size_t(slot) * g.stage_bytes;
          mbar_arrive_expect_tx(&full[slot], g.bytes_a + g.bytes_m);
          if (MODE == kFibI) {
            tma_2d(st, &tmA, &full[slot], 0, int(j));
            tma_2d(st + g.bytes_a / 2, &tmA, &full[slot], 128, int(j));
          } else {
            const uint64_t p = j / a.s;
            tma_3d(st, &tmA, &full[slot], int(j - p * a.s), 0, int(p));
          }
          if (MCOL) tma_2d(st + g.bytes_a, &tmM, &full[slot], int(j), 0);
          else tma_2d(st + g.bytes_a, &tmM, &full[slot], 0, int(j));
        }
      }
    }
    return;
  }
  if constexpr (REBAL) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");

  const int q = lane & 3;
  const int r8 = lane >> 2;
  const int MT = int((a.K + 7) / 8);
  const int base = MT / 8;              // 2 or 3 full row tiles per warp
  const int nrem = (MT % 8) * kND;      // remainder (row tile, column tile) pairs
  const int lda = int(g.lda), ldm = int(g.ldm);
  double sq_acc[4] = {0.0, 0.0, 0.0, 0.0};
  // ||A||^2 is fused only into the init pass (column-major S)
  const bool want_sq = MCOL && a.sumsq_part != nullptr;
  // A(row, kk) of the current stage
  auto aval = [&](const double* As, int row, int kk) -> double {
    if (MODE == kFibI) return row < 128 ? As[kk * 132 + row] : As[16 * 132 + kk * 132 + row - 128];
    return As[row * lda + kk];
  };

  int kb = 0;
  for (uint32_t range = blockIdx.x; range < a.ranges; range += gridDim.x) {
    const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
    const uint64_t f1 = min(F, f0 + a.fibers_per_range);
    double acc[3][kNT][2];
    double accr[C::kRemP][2];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int n = 0; n < kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll
    for (int t = 0; t < C::kRemP; ++t) accr[t][0] = accr[t][1] = 0.0;
    double tl[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    double tlr[C::kRemP][2];
#pragma unroll
    for (int t = 0; t < C::kRemP; ++t) tlr[t][0] = tlr[t][1] = 0.0;
    for (uint64_t j = f0; j < f1; ++kb) {
      const int slot = kb % stages;
      const uint32_t ph = (kb / stages) & 1;
      mbar_wait(&full[slot], ph);
      const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * g.stage_bytes);
      const double* Ms = reinterpret_cast<const double*>(ring + size_t(slot) * g.stage_bytes + g.bytes_a);
      const int kvalid = chunk_len(j, f1);
      j += kvalid;
#pragma unroll
      for (int t = 0; t < C::kMaxKB / 4; ++t) {
        if (4 * t >= kvalid) break;
        const int kk = 4 * t + q;
        const bool kok = kk < kvalid;
        // 9 warps: at most 3 per SM sub-partition, so 168 registers per
        // thread; the column-tile fragments are loaded one at a time
        double af[3];
#pragma unroll
        for (int mi = 0; mi < 3; ++mi) {
          const int row = (warp + 8 * mi) * 8 + r8;
          // kFibI: rows of row tiles 0..15 sit in the first box, 16.. in the second
          const double v = MODE == kFibI ? (mi < 2 ? As[kk * 132 + row] : As[16 * 132 + kk * 132 + row - 128])
                                         : As[row * lda + kk];
          af[mi] = (kok && mi < base) ? v : 0.0;
          if (want_sq) sq_acc[(t & 1) * 2 + (mi & 1)] = fma(af[mi], af[mi], sq_acc[(t & 1) * 2 + (mi & 1)]);
        }
        // fibers past the chunk read real data of the next fibers or TMA
        // zero-fill (finite), and their A fragment is zero; the row-major B
        // loads are predicated all the same (measured: 5.96 -> 5.43 ms for the
        // c5 mode-1 left update), the column-major ones are not (7.15 -> 6.47)
#pragma unroll
        for (int n = 0; n < kND; ++n) {
          const double b = MCOL ? Ms[(n * 8 + r8) * ldm + kk] : (kok ? Ms[kk * ldm + n * 8 + r8] : 0.0);
          dmma(acc[0][n][0], acc[0][n][1], af[0], b);
          dmma(acc[1][n][0], acc[1][n][1], af[1], b);
          if (base > 2) dmma(acc[2][n][0], acc[2][n][1], af[2], b);
        }
        double2 bt = make_double2(0.0, 0.0);
        if constexpr (TAIL != 0) {
          if (MCOL) bt = make_double2(Ms[(kND * 8) * ldm + kk], Ms[(kND * 8 + 1) * ldm + kk]);
          else if (kok) bt = *reinterpret_cast<const double2*>(Ms + kk * ldm + kND * 8);
#pragma unroll
          for (int mi = 0; mi < 3; ++mi) {
            tl[mi][0] = fma(af[mi], bt.x, tl[mi][0]);
            tl[mi][1] = fma(af[mi], bt.y, tl[mi][1]);
          }
        }
#pragma unroll
        for (int u = 0; u < C::kRemP; ++u) {
          const int p = warp + 8 * u;
          if (p < nrem) {
            const int m = 8 * base + p / kND, n = p % kND;
            const double af1 = kok ? aval(As, m * 8 + r8, kk) : 0.0;
            // each A element of a remainder tile is squared once (column tile 0)
            if (want_sq && n == 0) sq_acc[(t & 1) * 2 + 1] = fma(af1, af1, sq_acc[(t & 1) * 2 + 1]);
            const double bb = MCOL ? Ms[(n * 8 + r8) * ldm + kk] : (kok ? Ms[kk * ldm + n * 8 + r8] : 0.0);
            dmma(accr[u][0], accr[u][1], af1, bb);
            if constexpr (TAIL != 0) {
              if (n == 0) {
                tlr[u][0] = fma(af1, bt.x, tlr[u][0]);
                tlr[u][1] = fma(af1, bt.y, tlr[u][1]);
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    // this range's partial rows
    double* dst0 = a.partial + size_t(range) * a.K * a.ncp;
    if constexpr (TAIL != 0) {
#pragma unroll
      for (int mi = 0; mi < 3; ++mi) tail_to_tile<TAIL>(tl[mi], acc[mi][kND][0], acc[mi][kND][1], q);
#pragma unroll
      for (int u = 0; u < C::kRemP; ++u) tail_to_tile<TAIL>(tlr[u], tlr[u][0], tlr[u][1], q);
    }
#pragma unroll
    for (int mi = 0; mi < 3; ++mi) {
      if (mi >= base) continue;
      const int i = (warp + 8 * mi) * 8 + r8;
      if (i >= int(a.K)) continue;
#pragma unroll
      for (int n = 0; n < kNT; ++n)
        *reinterpret_cast<double2*>(dst0 + size_t(i) * a.ncp + n * 8 + 2 * q) =
            make_double2(acc[mi][n][0], acc[mi][n][1]);
    }
#pragma unroll
    for (int u = 0; u < C::kRemP; ++u) {
      const int p = warp + 8 * u;
      if (p >= nrem) continue;
      const int i = (8 * base + p / kND) * 8 + r8, n = p % kND;
      if (i < int(a.K)) {
        *reinterpret_cast<double2*>(dst0 + size_t(i) * a.ncp + n * 8 + 2 * q) =
            make_double2(accr[u][0], accr[u][1]);
        if constexpr (TAIL != 0) {
          if (n == 0)
            *reinterpret_cast<double2*>(dst0 + size_t(i) * a.ncp + kND * 8 + 2 * q) =
                make_double2(tlr[u][0], tlr[u][1]);
        }
      }
    }
  }
  if (want_sq) {
    __shared__ double red[kCons];
    double sq = (sq_acc[0] + sq_acc[1]) + (sq_acc[2] + sq_acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[warp] = sq;
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
// ---------------------------------------------------------------------------
// Mode expansion out(jl, i, p) = sum_c X(jl, c, p) U[i + c*Iout], X read as
// the 3-D view X[jl + c*s + p*s*K] (reconstruct, tensor_ops.cpp:395-440).
// A CTA keeps the A fragments of a 128-fiber tile of X (inside one panel) in
// registers for all Iout columns; the producer warp streams 32-column blocks
// of U through the TMA ring. Two epilogues:
//   DIFF  (last mode, s = F, P = 1): fused with the difference norm,
//         sq += sum (ref[j + i*F] - out(j, i))^2 with 32-column blocks of the
//         reference streamed beside U (relative_error(t, reconstruct(tk))
//         without the reconstruction);
//   STORE (intermediate modes): out[jl + i*s + p*s*Iout] written directly.
// ---------------------------------------------------------------------------
template <int KC>
struct ExT {
  static constexpr int kTF = 128, kCB = 32;
  static constexpr int kLdX = 132, kLdU = 36, kLdR = 132;
  static constexpr int kStages = KC <= 32 ? 4 : 3;
  static constexpr int kBytesX = (KC * kLdX * 8 + 127) / 128 * 128;
  static constexpr int kBytesU = KC * kLdU * 8;
  static constexpr int kBytesR = kCB * kLdR * 8;
  static constexpr int kStageBytes = (kBytesU + kBytesR + 127) / 128 * 128;
  static constexpr size_t kSmem = 1024 + size_t(kBytesX) + size_t(kStages) * kStageBytes;
};

template <int KC, bool DIFF>
__global__ void __launch_bounds__(kThreadsTma, 1)
    expand_tma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmR, uint64_t s, uint64_t P, uint32_t Iout,
                      double* sumsq_part, double* out) {
  using C = ExT<KC>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + C::kStages;
  uint64_t* xfull = empty + C::kStages;
  uint64_t* xempty = xfull + 1;
  double* Xs = reinterpret_cast<double*>(smem_raw + 1024);
  unsigned char* ring = smem_raw + 1024 + C::kBytesX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tpp = (s + C::kTF - 1) / C::kTF;  // tiles per panel
  const uint64_t ntiles = tpp * P;
  const int nblk = int((Iout + C::kCB - 1) / C::kCB);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, kCons);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons) {
    if (lane == 0) {
      prefetch_map(&tmX);
      prefetch_map(&tmU);
      prefetch_map(&tmR);
      uint32_t it = 0, xt = 0;
      for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++xt) {
        const int p = int(tile / tpp), j0 = int((tile % tpp) * C::kTF);
        mbar_wait(xempty, (xt & 1) ^ 1);
        mbar_arrive_expect_tx(xfull, KC * C::kLdX * 8);
        tma_3d(Xs, &tmX, xfull, j0, 0, p);
        for (int b = 0; b < nblk; ++b, ++it) {
          const int slot = it % C::kStages;
          const uint32_t ph = (it / C::kStages) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          unsigned char* st = ring + size_t(slot) * C::kStageBytes;
          mbar_arrive_expect_tx(&full[slot], DIFF ? C::kBytesU + C::kBytesR : C::kBytesU);
          tma_2d(st, &tmU, &full[slot], b * C::kCB, 0);
          if (DIFF) tma_2d(st + C::kBytesU, &tmR, &full[slot], j0, b * C::kCB);
        }
      }
    }
    return;
  }

  const int q = lane & 3, r8 = lane >> 2;
  double sqv[4] = {0.0, 0.0, 0.0, 0.0};  // independent chains (see the FR init pass)
  uint32_t it = 0, xt = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++xt) {
    const uint64_t p = tile / tpp, j0 = (tile % tpp) * C::kTF;
    mbar_wait(xfull, xt & 1);
    double af[KC / 4][2];
#pragma unroll
    for (int t = 0; t < KC / 4; ++t)
#pragma unroll
      for (int m = 0; m < 2; ++m) af[t][m] = Xs[(4 * t + q) * C::kLdX + warp * 16 + m * 8 + r8];
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty);
    for (int b = 0; b < nblk; ++b, ++it) {
      const int slot = it % C::kStages;
      const uint32_t ph = (it / C::kStages) & 1;
      mbar_wait(&full[slot], ph);
      const double* Us = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes);
      const double* Rs = reinterpret_cast<const double*>(ring + size_t(slot) * C::kStageBytes + C::kBytesU);
      double acc[2][4][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll
      for (int t = 0; t < KC / 4; ++t) {
        double bf[4];
#pragma unroll
        for (int n = 0; n < 4; ++n) bf[n] = Us[(4 * t + q) * C::kLdU + n * 8 + r8];
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int m = 0; m < 2; ++m) dmma(acc[m][n][0], acc[m][n][1], af[t][m], bf[n]);
      }
      if (DIFF) {
        // rows past F / columns past Iout: TMA zero-fill on both sides
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double d = Rs[(n * 8 + 2 * q + e) * C::kLdR + warp * 16 + m * 8 + r8] - acc[m][n][e];
              sqv[(n & 1) * 2 + e] = fma(d, d, sqv[(n & 1) * 2 + e]);
            }
      } else {
        const uint32_t i0 = b * C::kCB + 2 * q;  // column of acc[.][0][0]
        double* ob = out + (p * Iout + i0) * s + j0 + warp * 16 + r8;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          if (j0 + warp * 16 + m * 8 + r8 >= s) continue;
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (i0 + n * 8 + e < Iout) ob[m * 8 + (n * 8 + e) * s] = acc[m][n][e];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  if (!DIFF) return;
  __shared__ double red[kCons];
  double sq = (sqv[0] + sqv[1]) + (sqv[2] + sqv[3]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
  if (lane == 0) red[warp] = sq;
  asm volatile("bar.sync 1, %0;\n" ::"n"(kCons * 32));
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int w = 0; w < kCons; ++w) s2 += red[w];
    sumsq_part[blockIdx.x] = s2;
  }
}

template <class K>
cudaError_t set_smem(K k, size_t bytes) {
  return raise_smem_limit(k, bytes);
}

template <int NC, int MODE, int TAIL = 0>
cudaError_t fc_tma_launch(const CUtensorMap& A, const CUtensorMap& M, const FcTmaArgs& a, int grid,
                          cudaStream_t st) {
  using C = FcT<NC, MODE>;
  auto k = fc_tma_kernel<NC, MODE, TAIL>;
  cudaError_t e = set_smem(k, C::kSmem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, C::kSmem, st, A, M, a);
}

template <int NC, int MODE, bool MCOL, int TAIL = 0>
cudaError_t fr_wide_launch(const CUtensorMap& A, const CUtensorMap& M, const FrTmaArgs& a, const FrWideGeom& g,
                           int grid, cudaStream_t st) {
  constexpr bool kRebal = !(MODE == kFibI && !MCOL);
  auto k = fr_wide_kernel<NC, MODE, MCOL, kRebal ? TAIL : 0, kRebal>;
  const size_t smem = 1024 + size_t(g.stages) * g.stage_bytes;
  cudaError_t e = set_smem(k, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl_threads(k, grid, kRebal ? kThreadsWide : kThreadsTma, smem, st, A, M, a, g);
}

template <int NC, int MODE, bool MCOL, int TAIL = 0>
cudaError_t fr_tma_launch(const CUtensorMap& A, const CUtensorMap& M, const FrTmaArgs& a, int grid,
                          cudaStream_t st) {
  using C = FrT<NC, MODE, MCOL>;
  auto k = fr_tma_kernel<NC, MODE, MCOL, TAIL>;
  cudaError_t e = set_smem(k, C::kSmem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, C::kSmem, st, A, M, a);
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

// column counts whose last tile may run as a DFMA tail (16 .. 64)
#define TKG_NC_SWITCH_T(ncp, CALL)          \
  switch (ncp) {                            \
    case 16: return CALL(16);               \
    case 24: return CALL(24);               \
    case 32: return CALL(32);               \
    case 40: return CALL(40);               \
    case 48: return CALL(48);               \
    case 56: return CALL(56);               \
    case 64: return CALL(64);               \
    default: break;                         \
  }

template <int KC>
cudaError_t expand_tma_launch(const CUtensorMap& X, const CUtensorMap& U, const CUtensorMap& R,
                              const ExpandArgs& a, int grid, cudaStream_t st) {
  using C = ExT<KC>;
  auto k = a.ref ? expand_tma_kernel<KC, true> : expand_tma_kernel<KC, false>;
  cudaError_t e = set_smem(k, C::kSmem);
  if (e != cudaSuccess) return e;
  k<<<grid, kThreadsTma, C::kSmem, st>>>(X, U, R, a.s, a.P, a.Iout, a.sumsq_part, a.out);
  return cudaGetLastError();
}

}  // namespace

int& pdl_off_count() {
  static int n = 0;  // engines currently profiling (host-side setting, read at launch)
  return n;
}

// r mod 8 in {1, 2} above 8 columns: the last column tile runs as a DFMA
// tail (TKG_DFMA_TAIL=0 keeps the padded DMMA tile)
bool dfma_tail(uint32_t nc) {
  static const bool on = [] {
    const char* e = std::getenv("TKG_DFMA_TAIL");
    return !(e && e[0] == '0');
  }();
  return on && nc > 8 && (nc % 8 == 1 || nc % 8 == 2);
}

int fc_tma_mode(const FiberView& v, const double* mt, uint32_t ldmt) {
  if (!encode_fn() || !aligned16(v.base) || !aligned16(mt) || (ldmt % 2) != 0) return -1;
  if (v.s * v.P >= (1ull << 31) || v.K >= (1u << 31)) return -1;
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0) return kFibI;
  if (v.s % 2 != 0 || v.is_i % 2 != 0 || v.is_p % 2 != 0 || v.P >= (1ull << 31)) return -1;
  // panel-local 128-fiber tiles for long panels, whole-panel tiles for short ones
  return v.s >= 128 ? kFibJ : kFibS;
}

int fr_tma_mode(const FiberView& v, const double* m, uint64_t mj, uint64_t mc) {
  // M(j, c) = m[j*mj + c*mc]: row-major (mc == 1) or column-major (mj == 1)
  const uint64_t ld = mc == 1 ? mj : (mj == 1 ? mc : 1);
  if (!encode_fn() || !aligned16(v.base) || !aligned16(m) || (ld % 2) != 0) return -1;
  if (v.s * v.P >= (1ull << 31)) return -1;
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0) return kFibI;
  if (v.s % 2 != 0 || v.is_i % 2 != 0 || v.is_p % 2 != 0 || v.P >= (1ull << 31)) return -1;
  // panel-local 64-fiber chunks for long panels, whole-panel chunks for short ones
  return (v.s % 32 == 0 || v.s >= 64) ? kFibJ : kFibS;
}

namespace {

// kFibS FC: panels per tile and the padded inner box extent (4 mod 16
// doubles when that costs at most a quarter more)
void fc_short_geometry(uint64_t s, uint32_t* pc, uint32_t* sb) {
  *pc = uint32_t(128 / s);
  uint32_t b = uint32_t(s) + uint32_t((4 + 16 - s % 16) % 16);
  *sb = (b <= s + s / 4) ? b : uint32_t(s);
}

// kFibS FC with every tile row live: tiles of 128 consecutive fibers across
// panel boundaries; a tile starting anywhere in a panel spans at most
// floor((s + 126) / s) + 1 panels. Taken when whole-panel tiles would leave
// rows idle and the wider box still fits the stage (pc * sb <= 208 doubles
// per contraction index); TKG_FC_STRADDLE=0 keeps whole-panel tiles.
bool fc_straddle_geometry(uint64_t s, uint64_t P, uint32_t sb, uint32_t* pc) {
  static const bool on = [] {
    const char* e = std::getenv("TKG_FC_STRADDLE");
    return !(e && e[0] == '0');
  }();
  if (!on || 128 % s == 0) return false;
  const uint32_t span = uint32_t(std::min<uint64_t>((s + 126) / s + 1, P));
  if (span > 256 || uint64_t(span) * sb > 208) return false;
  *pc = span;
  return true;
}

// kFibS FR: panels per chunk (kf = pc * s <= 64 fibers) and the panel ranges
void fr_short_geometry(const FiberView& v, int num_sms, uint32_t* pc, uint64_t* ppr, uint32_t* ranges) {
  *pc = uint32_t(64 / v.s);
  const uint32_t igroups = (v.K + 127) / 128;
  uint64_t r = std::max<uint64_t>(1, uint64_t(num_sms) * 2 / igroups);
  r = std::min<uint64_t>(r, std::max<uint64_t>(1, v.P / (4 * *pc)));
  *ppr = (v.P + r - 1) / r;
  *ranges = uint32_t((v.P + *ppr - 1) / *ppr);
}

}  // namespace

int fc_tma_grid(const FiberView& v, int num_sms) {
  const uint64_t tiles = (v.s * v.P + 127) / 128;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms))));
}

cudaError_t launch_fc_tma(const FiberView& v, const double* mt, uint32_t ldmt, FcTmaArgs a, int mode,
                          int num_sms, cudaStream_t st, int* grid_used) {
  const uint32_t ncp = pad_nc(a.nc);
  CUtensorMap A, M;
  const int KB = 32;
  if (mode == kFibI) {
    const uint64_t dims[2] = {v.K, v.s * v.P};
    const uint64_t strides[1] = {v.is_p * 8};
    const uint32_t box[2] = {36, 128};
    if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else if (mode == kFibJ) {
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {132, 32, 1};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    fc_short_geometry(v.s, &a.pc, &a.sb);
    a.straddle = fc_straddle_geometry(v.s, v.P, a.sb, &a.pc) ? 1 : 0;
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {a.sb, 32, a.pc};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
    a.bytes_a = 32u * a.pc * a.sb * 8u;
    a.stage_bytes = (a.bytes_a + 32u * (ncp + 4) * 8u + 127u) / 128u * 128u;
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
#define TKG_FC_CALL(N) (mode == kFibI   ? fc_tma_launch<N, kFibI>(A, M, a, grid, st) \
                        : mode == kFibJ ? fc_tma_launch<N, kFibJ>(A, M, a, grid, st) \
                                        : fc_tma_launch<N, kFibS>(A, M, a, grid, st))
#define TKG_FC_CALL_T(N) (mode == kFibI   ? fc_tma_launch<N, kFibI, 2>(A, M, a, grid, st) \
                          : mode == kFibJ ? fc_tma_launch<N, kFibJ, 2>(A, M, a, grid, st) \
                                          : fc_tma_launch<N, kFibS, 2>(A, M, a, grid, st))
  if (dfma_tail(a.nc)) {
    TKG_NC_SWITCH_T(ncp, TKG_FC_CALL_T)
  }
  TKG_NC_SWITCH(ncp, TKG_FC_CALL)
#undef TKG_FC_CALL_T
#undef TKG_FC_CALL
}

cudaError_t launch_fr_tma(const FiberView& v, const double* m, uint64_t mj, uint64_t mc, FrTmaArgs a,
                          int mode, int num_sms, cudaStream_t st, uint32_t* ranges_used,
                          uint32_t* grid_used) {
  const bool mcol = mc != 1;
  const uint32_t ncp = pad_nc(a.nc);
  CUtensorMap A, M;
  const uint64_t F = v.s * v.P;
  if (fr_wide_ok(v, ncp, mode)) {
    // one CTA over all K rows (fr_wide_kernel)
    const uint32_t K8 = (v.K + 7) / 8 * 8;
    FrWideGeom g;
    if (mode == kFibI) {
      g.kb = 16;
      g.lda = 132;
      const uint64_t dims[2] = {v.K, F};
      const uint64_t strides[1] = {v.is_p * 8};
      const uint32_t box[2] = {132, g.kb};
      if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
      g.bytes_a = 2 * g.kb * 132 * 8;
    } else {
      uint32_t pcS = 0, sb = 0;
      if (mode == kFibJ) {
        g.kb = 32;
        g.lda = 36;
      } else {
        fc_short_geometry(v.s, &pcS, &sb);
        g.kb = uint32_t(v.s);  // one whole panel per stage
        // the k-steps read fibers up to round4(s) - 1: the A rows and the M
        // boxes cover them (next-panel data or TMA zero-fill, never used)
        g.lda = std::max<uint32_t>(sb, (g.kb + 3) / 4 * 4);
      }
      const uint64_t dims[3] = {v.s, v.K, v.P};
      const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
      const uint32_t box[3] = {g.lda, K8, 1};
      if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
      g.bytes_a = K8 * g.lda * 8;
    }
    const uint32_t mrows = mode == kFibS ? g.lda : g.kb;  // fibers per M box (kFibS: >= round4(s))
    if (!mcol) {
      g.ldm = ncp + 4;
      const uint64_t dims[2] = {ncp, F};
      const uint64_t strides[1] = {mj * 8};
      const uint32_t box[2] = {ncp + 4, mrows};
      if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
      g.bytes_m = mrows * (ncp + 4) * 8;
    } else {
      g.ldm = mode == kFibS ? mrows : g.kb + 4;
      const uint64_t dims[2] = {F, a.nc};
      const uint64_t strides[1] = {mc * 8};
      const uint32_t box[2] = {g.ldm, ncp};
      if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
      g.bytes_m = ncp * g.ldm * 8;
    }
    g.stage_bytes = (g.bytes_a + g.bytes_m + 127) / 128 * 128;
    g.stages = std::min<uint32_t>(4, (220u * 1024u) / g.stage_bytes);
    if (g.stages < 2) return cudaErrorInvalidValue;
    a.s = v.s;
    a.P = v.P;
    a.K = v.K;
    a.ncp = ncp;
    a.igroups = 1;
    if (mode == kFibS) {  // whole-panel ranges
      const uint64_t ranges = std::min<uint64_t>(uint64_t(num_sms), std::max<uint64_t>(1, v.P / 4));
      const uint64_t ppr = (v.P + ranges - 1) / ranges;
      a.fibers_per_range = ppr * v.s;
    } else {
      const uint64_t steps = (F + g.kb - 1) / g.kb;
      const uint64_t ranges = std::min<uint64_t>(uint64_t(num_sms), std::max<uint64_t>(1, steps / 4));
      a.fibers_per_range = (steps + ranges - 1) / ranges * g.kb;
    }
    a.ranges = uint32_t((F + a.fibers_per_range - 1) / a.fibers_per_range);
    if (ranges_used) *ranges_used = a.ranges;
    const int grid = int(std::min<uint64_t>(a.ranges, uint64_t(num_sms)));
    if (grid_used) *grid_used = grid;
#define TKG_FW(N, MO, T)                                                              \
  (mcol ? fr_wide_launch<N, MO, true, T>(A, M, a, g, grid, st)                        \
        : fr_wide_launch<N, MO, false, T>(A, M, a, g, grid, st))
#define TKG_FWM(N, T)                                                                  \
  case N:                                                                             \
    return mode == kFibI ? TKG_FW(N, kFibI, T) : mode == kFibJ ? TKG_FW(N, kFibJ, T) : TKG_FW(N, kFibS, T);
    if (dfma_tail(a.nc)) {
      switch (ncp) {
        TKG_FWM(40, 2) TKG_FWM(48, 2) TKG_FWM(56, 2) TKG_FWM(64, 2)
        default: return cudaErrorInvalidValue;
      }
    }
    switch (ncp) {
      TKG_FWM(40, 0) TKG_FWM(48, 0) TKG_FWM(56, 0) TKG_FWM(64, 0)
      default: return cudaErrorInvalidValue;
    }
#undef TKG_FWM
#undef TKG_FW
  }
  if (mode == kFibI) {
    const uint64_t dims[2] = {v.K, F};
    const uint64_t strides[1] = {v.is_p * 8};
    const uint32_t box[2] = {132, 32};
    if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else if (mode == kFibJ) {
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {68, 128, 1};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    uint64_t ppr = 0;
    uint32_t nr = 0;
    fr_short_geometry(v, num_sms, &a.pc, &ppr, &nr);
    a.kf = a.pc * uint32_t(v.s);
    a.panels_per_range = ppr;
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {uint32_t(v.s), 128, a.pc};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
    a.bytes_a = a.pc * 128u * uint32_t(v.s) * 8u;
    a.ldm = a.kf + 4;
    a.bytes_m = mcol ? ncp * a.ldm * 8u : a.kf * (ncp + 4) * 8u;
    a.stage_bytes = (a.bytes_a + a.bytes_m + 127u) / 128u * 128u;
  }
  const uint32_t kb = mode == kFibI ? 32 : mode == kFibJ ? 64 : a.kf;
  if (!mcol) {
    const uint64_t dims[2] = {ncp, F};
    const uint64_t strides[1] = {mj * 8};
    const uint32_t box[2] = {ncp + 4, kb};
    if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const uint64_t dims[2] = {F, a.nc};
    const uint64_t strides[1] = {mc * 8};
    const uint32_t box[2] = {kb + 4, ncp};
    if (!encode(&M, m, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  a.s = v.s;
  a.P = v.P;
  a.K = v.K;
  a.ncp = ncp;
  a.igroups = (v.K + 127) / 128;
  if (mode == kFibS) {  // whole-panel ranges
    a.fibers_per_range = a.panels_per_range * v.s;
    a.ranges = uint32_t((v.P + a.panels_per_range - 1) / a.panels_per_range);
  } else {
    const uint64_t steps = (F + 31) / 32;
    // one work item per CTA slot; two per SM when the row-group count does
    // not divide the SM count (persistent CTAs then stay busy)
    const int per_sm = (mode == kFibI && ncp <= 32) ? 2 : 1;
    const uint64_t items_per_sm = (num_sms % a.igroups == 0) ? per_sm : 2;
    uint64_t ranges = std::max<uint64_t>(1, uint64_t(num_sms) * items_per_sm / a.igroups);
    ranges = std::min<uint64_t>(ranges, std::max<uint64_t>(1, steps / 4));
    a.fibers_per_range = (steps + ranges - 1) / ranges * 32;
    a.ranges = uint32_t((F + a.fibers_per_range - 1) / a.fibers_per_range);
  }
  if (ranges_used) *ranges_used = a.ranges;
  const int ctas_per_sm = (mode == kFibI && ncp <= 32) ? 2 : 1;
  const int grid = int(std::min<uint64_t>(uint64_t(a.ranges) * a.igroups, uint64_t(num_sms) * ctas_per_sm));
  if (grid_used) *grid_used = grid;
#define TKG_FR_CALL(N)                                                                      \
  (mode == kFibI   ? (mcol ? fr_tma_launch<N, kFibI, true>(A, M, a, grid, st)                 \
                           : fr_tma_launch<N, kFibI, false>(A, M, a, grid, st))               \
   : mode == kFibJ ? (mcol ? fr_tma_launch<N, kFibJ, true>(A, M, a, grid, st)                 \
                           : fr_tma_launch<N, kFibJ, false>(A, M, a, grid, st))               \
                   : (mcol ? fr_tma_launch<N, kFibS, true>(A, M, a, grid, st)                 \
                           : fr_tma_launch<N, kFibS, false>(A, M, a, grid, st)))
#define TKG_FR_CALL_T(N)                                                                    \
  (mode == kFibI   ? (mcol ? fr_tma_launch<N, kFibI, true, 2>(A, M, a, grid, st)              \
                           : fr_tma_launch<N, kFibI, false, 2>(A, M, a, grid, st))            \
   : mode == kFibJ ? (mcol ? fr_tma_launch<N, kFibJ, true, 2>(A, M, a, grid, st)              \
                           : fr_tma_launch<N, kFibJ, false, 2>(A, M, a, grid, st))            \
                   : (mcol ? fr_tma_launch<N, kFibS, true, 2>(A, M, a, grid, st)              \
                           : fr_tma_launch<N, kFibS, false, 2>(A, M, a, grid, st)))
  if (dfma_tail(a.nc)) {
    TKG_NC_SWITCH_T(ncp, TKG_FR_CALL_T)
  }
  TKG_NC_SWITCH(ncp, TKG_FR_CALL)
#undef TKG_FR_CALL_T
#undef TKG_FR_CALL
}

// one CTA over all K rows (fr_wide_kernel): 128 < K <= 248 at the
// 1-CTA-per-SM column counts, when the remainder row tiles give each warp at
// most FrW::kRemP extra pairs; kFibI, kFibJ, and kFibS panels of 32 < s < 64
// fibers (one panel per stage) (TKG_FR_WIDE=0 disables it)
bool fr_wide_ok(const FiberView& v, uint32_t ncp, int mode) {
  static const bool on = [] {
    const char* e = std::getenv("TKG_FR_WIDE");
    return !(e && e[0] == '0');
  }();
  const uint32_t mt = (v.K + 7) / 8, nrem = (mt % 8) * (ncp / 8);
  const bool layout = mode == kFibI || mode == kFibJ || (mode == kFibS && v.s > 32 && v.s < 64);
  return on && layout && v.K > 128 && v.K <= 248 && ncp >= 40 && ncp <= 64 && nrem <= 8 * 2;
}

uint32_t fr_tma_ranges(const FiberView& v, int num_sms) {
  if (v.s > 1 && v.s < 64 && v.s % 32 != 0) {  // kFibS (when that mode is chosen)
    uint32_t pc = 0, nr = 0;
    uint64_t ppr = 0;
    fr_short_geometry(v, num_sms, &pc, &ppr, &nr);
    return nr;
  }
  const uint64_t F = v.s * v.P;
  const uint32_t igroups = (v.K + 127) / 128;
  const uint64_t steps = (F + 31) / 32;
  uint64_t ranges = std::max<uint64_t>(1, uint64_t(num_sms) * 2 / igroups);  // upper bound (buffer sizing)
  ranges = std::min<uint64_t>(ranges, std::max<uint64_t>(1, steps / 4));
  const uint64_t fpr = (steps + ranges - 1) / ranges * 32;
  return uint32_t((F + fpr - 1) / fpr);
}

bool expand_diff_tma_ok(const ExpandArgs& a) {
  const uint64_t F = a.s * a.P;
  return encode_fn() && a.ref && a.P == 1 && a.K >= 1 && a.K <= 64 && F % 2 == 0 && a.Iout % 2 == 0 &&
         F < (1ull << 31) && aligned16(a.in) && aligned16(a.U) && aligned16(a.ref) && a.sumsq_part;
}

bool expand_tma_ok(const ExpandArgs& a) {
  return encode_fn() && !a.ref && a.out && a.K >= 1 && a.K <= 64 && a.s % 2 == 0 && a.Iout % 2 == 0 &&
         a.s < (1ull << 31) && a.P < (1ull << 31) && aligned16(a.in) && aligned16(a.U);
}

int expand_diff_tma_grid(uint64_t F, int num_sms) { return expand_tma_grid(F, 1, num_sms); }

int expand_tma_grid(uint64_t s, uint64_t P, int num_sms) {
  const uint64_t tiles = (s + 127) / 128 * P;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms))));
}

cudaError_t launch_expand_diff_tma(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used) {
  return launch_expand_tma(a, num_sms, st, grid_used);
}

cudaError_t launch_expand_tma(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used) {
  const uint32_t kc = (a.K + 7) / 8 * 8;  // K padded to the DMMA k granularity used here
  CUtensorMap X, U, R;
  {
    const uint64_t dims[3] = {a.s, a.K, a.P};
    const uint64_t strides[2] = {a.s * 8, a.s * a.K * 8};
    const uint32_t box[3] = {132, kc, 1};
    if (!encode(&X, a.in, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {a.Iout, a.K};
    const uint64_t strides[1] = {uint64_t(a.Iout) * 8};
    const uint32_t box[2] = {36, kc};
    if (!encode(&U, a.U, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  if (a.ref) {
    const uint64_t F = a.s * a.P;
    const uint64_t dims[2] = {F, a.Iout};
    const uint64_t strides[1] = {F * 8};
    const uint32_t box[2] = {132, 32};
    if (!encode(&R, a.ref, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    R = U;  // unused by the STORE epilogue
  }
  const int grid = expand_tma_grid(a.s, a.P, num_sms);
  if (grid_used) *grid_used = grid;
  switch (kc) {
    case 8: return expand_tma_launch<8>(X, U, R, a, grid, st);
    case 16: return expand_tma_launch<16>(X, U, R, a, grid, st);
    case 24: return expand_tma_launch<24>(X, U, R, a, grid, st);
    case 32: return expand_tma_launch<32>(X, U, R, a, grid, st);
    case 40: return expand_tma_launch<40>(X, U, R, a, grid, st);
    case 48: return expand_tma_launch<48>(X, U, R, a, grid, st);
    case 56: return expand_tma_launch<56>(X, U, R, a, grid, st);
    default: return expand_tma_launch<64>(X, U, R, a, grid, st);
  }
}

}  // namespace tkg
