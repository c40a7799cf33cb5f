// FC / FR fiber-contraction kernels (see contract.cuh for the math and the
// reference functions they replace). FP64 on the tensor pipe: every MMA is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); tcgen05 has no f64 kind, and the
// measured DMMA peak (37.2 TFLOP/s, profiles/) is the FP64 roof.
//
// Data movement: the streamed tensor X is read straight from HBM into
// registers (each element is used by exactly one warp, so staging it through
// shared memory would only add traffic); loads are 16-byte vectors whenever
// the layout allows (pairs of adjacent fibers, or 4 consecutive contraction
// indices for contiguous mode-1 fibers), giving full 128-byte lines per
// warp instruction. The small contraction matrix is staged through a
// 4-deep cp.async ring in shared memory, padded so every B-fragment load is
// bank-conflict free.
#include <algorithm>
#include <cstdio>

#include "contract.cuh"

namespace tkg {

namespace {

enum LoadMode { kScalar = 0, kPair = 1, kQuad = 2 };
constexpr int kStages = 4;
constexpr int kSub = 16;  // contraction indices per pipeline step

// ---------------------------------------------------------------------------
// FC
// ---------------------------------------------------------------------------
template <int NC, int WF, int MODE>
struct FcCfg {
  static constexpr int kWarps = 8;
  static constexpr int kThreads = kWarps * kWarp;
  static constexpr int kTF = kWarps * WF;         // fibers per CTA tile
  static constexpr int kMT = WF / 8;              // m-tiles per warp
  static constexpr int kNT = NC / 8;              // n-tiles
  static constexpr int kLd = smem_ld(NC);
  static constexpr int kGroups = MODE == kPair ? WF / 16 : WF / 8;  // load groups per lane
  static constexpr int kStageDoubles = kSub * kLd;
  static constexpr size_t kSmem =
      sizeof(double) * (size_t(kStages) * kStageDoubles + size_t(kTF) * kLd + size_t(NC) * NC);
};

template <int NC, int WF, int MODE>
__global__ void __launch_bounds__(256, 1) fc_kernel(FcArgs a) {
  using Cfg = FcCfg<NC, WF, MODE>;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  double* ms = smem;                                    // [kStages][kSub][kLd]
  double* scratch = ms + kStages * Cfg::kStageDoubles;  // [kTF][kLd] output tile (Gram epilogue)
  double* gacc = scratch + Cfg::kTF * Cfg::kLd;         // [NC][NC] CTA Gram accumulator

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int q = lane & 3;
  const int r8 = lane >> 2;

  const FiberView& v = a.in;
  const uint64_t F = v.s * v.P;
  const uint32_t K = v.K;
  const int nsub = (K + kSub - 1) / kSub;
  const uint64_t ntiles = (F + Cfg::kTF - 1) / Cfg::kTF;
  const bool want_gram = a.gram_part != nullptr;
  const bool want_sq = a.sumsq_part != nullptr;

  if (want_gram) {
    for (int e = tid; e < NC * NC; e += Cfg::kThreads) gacc[e] = 0.0;
  }
  double sq_acc = 0.0;

  // Stage 16 rows of Mt (i-major) into ring slot `slot`; QUAD permutes rows
  // so k-step t reads rows 4t..4t+3.
  auto stage = [&](int u, int slot) {
    double* dst = ms + slot * Cfg::kStageDoubles;
    constexpr int chunks = kSub * NC / 2;  // 16-byte chunks
    for (int c = tid; c < chunks; c += Cfg::kThreads) {
      const int il = c / (NC / 2);
      const int col = (c % (NC / 2)) * 2;
      const int srow = MODE == kQuad ? ((il & 3) * 4 + (il >> 2)) : il;
      const uint32_t i = u * kSub + il;
      double* d = dst + srow * Cfg::kLd + col;
      if (i < K) {
        cp_async16(d, a.mt + size_t(i) * a.ldmt + col);
      } else {
        d[0] = 0.0;
        d[1] = 0.0;
      }
    }
  };

  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t j0 = tile * Cfg::kTF + uint64_t(warp) * WF;
    // Per-lane fibers: input base offset per load group, output base per m-tile.
    int64_t ib[Cfg::kGroups];
    bool gok[Cfg::kGroups];
    int64_t ob[Cfg::kMT];
    bool mok[Cfg::kMT];
#pragma unroll
    for (int m = 0; m < Cfg::kMT; ++m) {
      uint64_t j = MODE == kPair ? j0 + (m >> 1) * 16 + 2 * r8 + (m & 1) : j0 + m * 8 + r8;
      mok[m] = j < F;
      if (!mok[m]) j = 0;
      const uint64_t p = j / v.s;
      const uint64_t jl = j - p * v.s;
      ob[m] = int64_t(jl * a.os_j + p * a.os_p);
      const int g = MODE == kPair ? (m >> 1) : m;
      if (MODE != kPair || (m & 1) == 0) {
        ib[g] = int64_t(jl + p * v.is_p);
        gok[g] = mok[m];
      }
    }

    double acc[Cfg::kMT][Cfg::kNT][2];
#pragma unroll
    for (int m = 0; m < Cfg::kMT; ++m)
#pragma unroll
      for (int n = 0; n < Cfg::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

    // A fragments for one 16-index step: af[m][t] (m-tile, k-step).
    double af0[Cfg::kMT][4], af1[Cfg::kMT][4];
    auto load_a = [&](int u, double (&dst)[Cfg::kMT][4]) {
      const uint32_t ibase = u * kSub;
#pragma unroll
      for (int g = 0; g < Cfg::kGroups; ++g) {
        if (MODE == kQuad) {
          const uint32_t i = ibase + 4 * q;
          if (gok[g] && i < K) {  // K % 4 == 0 in quad mode
            const double* p = v.base + ib[g] + i;
            double2 x = ldg2(p);
            double2 y = ldg2(p + 2);
            dst[g][0] = x.x; dst[g][1] = x.y; dst[g][2] = y.x; dst[g][3] = y.y;
          } else {
            dst[g][0] = dst[g][1] = dst[g][2] = dst[g][3] = 0.0;
          }
        } else if (MODE == kPair) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t i = ibase + 4 * t + q;
            if (gok[g] && i < K) {  // the pair partner may be past F: the view still covers it
              double2 x = ldg2(v.base + ib[g] + int64_t(i) * int64_t(v.is_i));
              dst[2 * g][t] = x.x;
              dst[2 * g + 1][t] = x.y;
            } else {
              dst[2 * g][t] = 0.0;
              dst[2 * g + 1][t] = 0.0;
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t i = ibase + 4 * t + q;
            dst[g][t] = (gok[g] && i < K) ? __ldg(v.base + ib[g] + int64_t(i) * int64_t(v.is_i)) : 0.0;
          }
        }
      }
    };

    // Prologue of the Mt ring and first A fragments.
    __syncthreads();  // previous tile's readers of the ring / scratch are done
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nsub) stage(s, s);
      cp_async_commit();
    }
    load_a(0, af0);

    // One pipeline step: Mt slot u landed, refill the ring, prefetch the next
    // A fragments into the other register set, then 4 k-steps of DMMA.
    auto step = [&](int u, const double (&cur)[Cfg::kMT][4], double (&nxt)[Cfg::kMT][4]) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      if (u + kStages - 1 < nsub) stage(u + kStages - 1, (u + kStages - 1) % kStages);
      cp_async_commit();
      if (u + 1 < nsub) load_a(u + 1, nxt);
      const double* mb = ms + (u % kStages) * Cfg::kStageDoubles;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        double bf[Cfg::kNT];
#pragma unroll
        for (int n = 0; n < Cfg::kNT; ++n) bf[n] = mb[(4 * t + q) * Cfg::kLd + n * 8 + r8];
#pragma unroll
        for (int m = 0; m < Cfg::kMT; ++m)
#pragma unroll
          for (int n = 0; n < Cfg::kNT; ++n) dmma(acc[m][n][0], acc[m][n][1], cur[m][t], bf[n]);
      }
    };
    for (int u = 0; u < nsub; u += 2) {
      step(u, af0, af1);
      if (u + 1 < nsub) step(u + 1, af1, af0);
    }
    cp_async_wait<0>();

    // Epilogue: store / diff-norm / sum of squares, and the output tile in
    // shared memory for the Gram partial.
#pragma unroll
    for (int m = 0; m < Cfg::kMT; ++m) {
      const int row = warp * WF + (MODE == kPair ? ((m >> 1) * 16 + 2 * r8 + (m & 1)) : (m * 8 + r8));
#pragma unroll
      for (int n = 0; n < Cfg::kNT; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t c = n * 8 + 2 * q + e;
          const double val = acc[m][n][e];
          const bool valid = mok[m] && c < a.nc;
          if (valid) {
            const int64_t o = ob[m] + int64_t(c) * int64_t(a.os_c);
            if (a.diff_ref) {
              const double d = a.diff_ref[o] - val;
              sq_acc += d * d;
            } else {
              if (a.out) a.out[o] = val;
              if (want_sq) sq_acc += val * val;
            }
          }
          if (want_gram) scratch[row * Cfg::kLd + c] = valid ? val : 0.0;
        }
      }
    }
    if (want_gram) {
      __syncthreads();
      // Upper-triangle 8x8 tiles of out^T out on the tensor pipe; the
      // consumer mirrors the lower triangle (as gram() does, matrix.cpp:121-125).
      constexpr int ntri = Cfg::kNT * (Cfg::kNT + 1) / 2;
      for (int tt = warp; tt < ntri; tt += Cfg::kWarps) {
        int mt = 0, rem = tt;
        while (rem >= Cfg::kNT - mt) { rem -= Cfg::kNT - mt; ++mt; }
        const int nt = mt + rem;
        double* gp = gacc + (mt * 8 + r8) * NC + nt * 8 + 2 * q;
        double d0 = gp[0], d1 = gp[1];
        for (int k0 = 0; k0 < Cfg::kTF; k0 += 4) {
          const double* rowp = scratch + (k0 + q) * Cfg::kLd;
          dmma(d0, d1, rowp[mt * 8 + r8], rowp[nt * 8 + r8]);
        }
        gp[0] = d0;
        gp[1] = d1;
      }
    }
  }

  // CTA-level reductions in fixed warp order (deterministic).
  if (want_sq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, off);
  }
  __syncthreads();
  double* red = ms;  // reuse the ring
  if (want_sq && lane == 0) red[warp] = sq_acc;
  __syncthreads();
  if (want_sq && tid == 0) {
    double s = 0.0;
    for (int w = 0; w < Cfg::kWarps; ++w) s += red[w];
    a.sumsq_part[blockIdx.x] = s;
  }
  if (want_gram) {
    for (int e = tid; e < NC * NC; e += Cfg::kThreads) a.gram_part[size_t(blockIdx.x) * NC * NC + e] = gacc[e];
  }
}

// ---------------------------------------------------------------------------
// FR
// ---------------------------------------------------------------------------
template <int NC, int WI, int MODE>
struct FrCfg {
  static constexpr int kMT = WI / 8;
  static constexpr int kNT = NC / 8;
  static constexpr int kLd = smem_ld(NC);
  static constexpr int kGroups = MODE == kPair ? WI / 16 : WI / 8;
};

// MODE kPair  : s == 1, contraction index contiguous: a lane loads two
//               adjacent i (two m-tiles) of one fiber per 16-byte load.
// MODE kQuad  : 4 adjacent fibers contiguous (s % 4 == 0): a lane loads
//               4 fibers (4 k-steps) of one i with two 16-byte loads.
// MODE kScalar: generic 8-byte loads.
template <int NC, int WI, int MODE>
__global__ void __launch_bounds__(256) fr_kernel(FrArgs a, int wgi, int wgj) {
  using Cfg = FrCfg<NC, WI, MODE>;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int q = lane & 3;
  const int r8 = lane >> 2;
  const int wi = warp % wgi;
  const int wj = warp / wgi;
  const int nthreads = blockDim.x;

  const FiberView& v = a.in;
  const uint64_t F = v.s * v.P;
  const uint32_t K = v.K;
  const uint32_t range = blockIdx.x / a.igroups;
  const uint32_t ig = blockIdx.x % a.igroups;
  const uint64_t f0 = uint64_t(range) * a.fibers_per_range;
  const uint64_t f1 = min(F, f0 + a.fibers_per_range);
  const uint32_t i0 = (ig * wgi + wi) * WI;
  const int step_fibers = kSub * wgj;
  const int stage_doubles = step_fibers * Cfg::kLd;
  double* ms = smem;  // [kStages][step_fibers][kLd]

  const bool want_sq = a.sumsq_part != nullptr;
  double sq_acc = 0.0;

  // Rows owned by this lane (i index per load group) and validity.
  int64_t ioff[Cfg::kGroups];
  bool iok[Cfg::kGroups];
#pragma unroll
  for (int g = 0; g < Cfg::kGroups; ++g) {
    const uint32_t i = MODE == kPair ? i0 + g * 16 + 2 * r8 : i0 + g * 8 + r8;
    iok[g] = i < K;  // for kPair K is even, so i+1 < K too
    ioff[g] = int64_t(iok[g] ? i : 0) * int64_t(v.is_i);
  }

  const uint64_t nsteps = (f1 > f0) ? (f1 - f0 + step_fibers - 1) / step_fibers : 0;

  auto stage = [&](uint64_t u, int slot) {
    double* dst = ms + slot * stage_doubles;
    const uint64_t jb = f0 + u * step_fibers;
    const int total = step_fibers * NC;
    for (int e = tid; e < total; e += nthreads) {
      const int jl = e % step_fibers;
      const int c = e / step_fibers;
      // row permutation inside each 16-fiber block so k-step t reads rows 4t..4t+3
      const int blk = jl >> 4, w = jl & 15;
      const int srow = blk * 16 + (MODE == kQuad ? ((w & 3) * 4 + (w >> 2)) : w);
      const uint64_t j = jb + jl;
      double* d = dst + srow * Cfg::kLd + c;
      if (j < f1 && c < int(a.nc)) {
        cp_async8(d, a.m + j * a.mj + uint64_t(c) * a.mc);
      } else {
        *d = 0.0;
      }
    }
  };

  double acc[Cfg::kMT][Cfg::kNT][2];
#pragma unroll
  for (int m = 0; m < Cfg::kMT; ++m)
#pragma unroll
    for (int n = 0; n < Cfg::kNT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

  double af0[Cfg::kMT][4], af1[Cfg::kMT][4];
  auto load_a = [&](uint64_t u, double (&dst)[Cfg::kMT][4]) {
    const uint64_t jb = f0 + u * step_fibers + wj * kSub;
    if (MODE == kQuad) {
      const uint64_t j = jb + 4 * q;  // 4 fibers j..j+3, same panel (s % 4 == 0)
      const bool jok = j < f1;        // f1 is a multiple of 4 or F
      const uint64_t p = j / v.s;
      const int64_t fb = int64_t((j - p * v.s) + p * v.is_p);
#pragma unroll
      for (int g = 0; g < Cfg::kGroups; ++g) {
        if (jok && iok[g]) {
          const double* ptr = v.base + fb + ioff[g];
          double2 x = ldg2(ptr);
          double2 y = ldg2(ptr + 2);
          dst[g][0] = x.x; dst[g][1] = x.y; dst[g][2] = y.x; dst[g][3] = y.y;
        } else {
          dst[g][0] = dst[g][1] = dst[g][2] = dst[g][3] = 0.0;
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint64_t j = jb + 4 * t + q;
        const bool jok = j < f1;
        const uint64_t p = jok ? j / v.s : 0;
        const int64_t fb = jok ? int64_t((j - p * v.s) + p * v.is_p) : 0;
#pragma unroll
        for (int g = 0; g < Cfg::kGroups; ++g) {
          if (MODE == kPair) {
            if (jok && iok[g]) {
              double2 x = ldg2(v.base + fb + ioff[g]);
              dst[2 * g][t] = x.x;
              dst[2 * g + 1][t] = x.y;
            } else {
              dst[2 * g][t] = 0.0;
              dst[2 * g + 1][t] = 0.0;
            }
          } else {
            dst[g][t] = (jok && iok[g]) ? __ldg(v.base + fb + ioff[g]) : 0.0;
          }
        }
      }
    }
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (uint64_t(s) < nsteps) stage(s, s);
    cp_async_commit();
  }
  if (nsteps > 0) load_a(0, af0);

  auto step = [&](uint64_t u, const double (&cur)[Cfg::kMT][4], double (&nxt)[Cfg::kMT][4]) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (u + kStages - 1 < nsteps) stage(u + kStages - 1, int((u + kStages - 1) % kStages));
    cp_async_commit();
    if (u + 1 < nsteps) load_a(u + 1, nxt);
    if (want_sq) {
#pragma unroll
      for (int m = 0; m < Cfg::kMT; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t) sq_acc = fma(cur[m][t], cur[m][t], sq_acc);
    }
    const double* mb = ms + int(u % kStages) * stage_doubles + wj * kSub * Cfg::kLd;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double bf[Cfg::kNT];
#pragma unroll
      for (int n = 0; n < Cfg::kNT; ++n) bf[n] = mb[(4 * t + q) * Cfg::kLd + n * 8 + r8];
#pragma unroll
      for (int m = 0; m < Cfg::kMT; ++m)
#pragma unroll
        for (int n = 0; n < Cfg::kNT; ++n) dmma(acc[m][n][0], acc[m][n][1], cur[m][t], bf[n]);
    }
  };
  for (uint64_t u = 0; u < nsteps; u += 2) {
    step(u, af0, af1);
    if (u + 1 < nsteps) step(u + 1, af1, af0);
  }
  cp_async_wait<0>();
  __syncthreads();

  // Combine the wgj fiber-split warps in fixed order through shared memory,
  // then write this CTA's partial rows.
  double* red = smem;  // [wgj][wgi*WI][NC]
  const int rows_cta = wgi * WI;
#pragma unroll
  for (int m = 0; m < Cfg::kMT; ++m) {
    const int g = MODE == kPair ? m >> 1 : m;
    const int row = wi * WI + (MODE == kPair ? g * 16 + 2 * r8 + (m & 1) : m * 8 + r8);
#pragma unroll
    for (int n = 0; n < Cfg::kNT; ++n) {
      const int c = n * 8 + 2 * q;
      red[(size_t(wj) * rows_cta + row) * NC + c] = acc[m][n][0];
      red[(size_t(wj) * rows_cta + row) * NC + c + 1] = acc[m][n][1];
    }
  }
  __syncthreads();
  const uint32_t row0 = ig * rows_cta;
  for (int e = tid; e < rows_cta * int(a.ncp); e += nthreads) {
    const int row = e / a.ncp;
    const int c = e % a.ncp;
    const uint32_t i = row0 + row;
    if (i >= K) continue;
    double s = 0.0;
    if (c < NC) {
      for (int w = 0; w < wgj; ++w) s += red[(size_t(w) * rows_cta + row) * NC + c];
    }
    a.partial[(size_t(range) * K + i) * a.ncp + c] = s;
  }
  if (want_sq) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, off);
    __syncthreads();
    if (lane == 0) red[warp] = sq_acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nthreads / 32; ++w) s += red[w];
      a.sumsq_part[blockIdx.x] = s;
    }
  }
}

template <int NC>
constexpr int fc_wf() {
  return NC <= 32 ? 32 : 16;
}
template <int NC>
constexpr int fr_wi() {
  return NC <= 32 ? 32 : 16;
}

template <int NC, int MODE>
cudaError_t fc_launch_t(const FcArgs& a, int grid, cudaStream_t st) {
  constexpr int WF = fc_wf<NC>();
  using Cfg = FcCfg<NC, WF, MODE>;
  auto k = fc_kernel<NC, WF, MODE>;
  cudaError_t e = raise_smem_limit(k, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  k<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(a);
  return cudaGetLastError();
}

template <int NC>
cudaError_t fc_dispatch_mode(const FcArgs& a, int mode, int grid, cudaStream_t st) {
  switch (mode) {
    case kQuad: return fc_launch_t<NC, kQuad>(a, grid, st);
    case kPair: return fc_launch_t<NC, kPair>(a, grid, st);
    default: return fc_launch_t<NC, kScalar>(a, grid, st);
  }
}

int fc_mode(const FiberView& v) {
  const bool even_base = (v.is_p % 2 == 0);
  if (v.s == 1 && v.is_i == 1 && even_base && v.K % 4 == 0) return kQuad;
  const bool adjacent = (v.s % 2 == 0 && v.is_p % 2 == 0) || (v.s == 1 && v.is_p == 1);
  if (adjacent && v.is_i % 2 == 0) return kPair;
  return kScalar;
}

int fr_mode(const FiberView& v) {
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0 && v.K % 2 == 0) return kPair;
  if (v.s % 4 == 0 && v.is_i % 2 == 0 && v.is_p % 2 == 0) return kQuad;
  return kScalar;
}

template <int NC, int MODE>
cudaError_t fr_launch_t(const FrArgs& a, int wgi, int wgj, cudaStream_t st) {
  constexpr int WI = fr_wi<NC>();
  auto k = fr_kernel<NC, WI, MODE>;
  const int rows_cta = wgi * WI;
  const size_t ring = sizeof(double) * kStages * size_t(kSub * wgj) * FrCfg<NC, WI, MODE>::kLd;
  const size_t red = sizeof(double) * size_t(wgj) * rows_cta * NC;
  const size_t smem = std::max(ring, red);
  cudaError_t e = raise_smem_limit(k, smem);
  if (e != cudaSuccess) return e;
  const int grid = int(a.ranges * a.igroups);
  k<<<grid, 32 * wgi * wgj, smem, st>>>(a, wgi, wgj);
  return cudaGetLastError();
}

template <int NC>
cudaError_t fr_dispatch_mode(const FrArgs& a, int mode, int wgi, int wgj, cudaStream_t st) {
  switch (mode) {
    case kQuad: return fr_launch_t<NC, kQuad>(a, wgi, wgj, st);
    case kPair: return fr_launch_t<NC, kPair>(a, wgi, wgj, st);
    default: return fr_launch_t<NC, kScalar>(a, wgi, wgj, st);
  }
}

// CTA shape for FR: wgi warps tile the contraction rows (WI each), wgj warps
// split each 16-fiber step; igroups CTAs cover all rows when K > 8*WI.
void fr_shape(uint32_t K, uint32_t ncp, int* wi_out, int* wgi, int* wgj) {
  const int wi = ncp <= 32 ? 32 : 16;
  const int tiles = int((K + wi - 1) / wi);
  const int igroups = (tiles + 7) / 8;
  const int g = (tiles + igroups - 1) / igroups;
  // keep the M ring (kStages x 16*wgj rows x ld doubles) within 128 KB
  const size_t per_wgj = sizeof(double) * kStages * kSub * size_t(smem_ld(int(ncp)));
  const int cap = int(std::max<size_t>(1, (128u << 10) / per_wgj));
  *wi_out = wi;
  *wgi = g;
  *wgj = std::max(1, std::min(8 / g, cap));
}

}  // namespace

uint32_t pad_nc(uint32_t nc) {
  uint32_t p = (nc + 7) / 8 * 8;
  return p < 8 ? 8 : p;
}

int fc_grid_for(const FiberView& v, uint32_t nc, int num_sms) {
  const uint32_t ncp = pad_nc(nc);
  const int wf = ncp <= 32 ? 32 : 16;
  const uint64_t tf = 8ull * wf;
  const uint64_t tiles = (v.s * v.P + tf - 1) / tf;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms))));
}

cudaError_t launch_fc(const FcArgs& a, int num_sms, cudaStream_t st, int* grid_used) {
  const uint32_t ncp = pad_nc(a.nc);
  const int grid = fc_grid_for(a.in, a.nc, num_sms);
  if (grid_used) *grid_used = grid;
  const int mode = fc_mode(a.in);
  switch (ncp) {
    case 8: return fc_dispatch_mode<8>(a, mode, grid, st);
    case 16: return fc_dispatch_mode<16>(a, mode, grid, st);
    case 24: return fc_dispatch_mode<24>(a, mode, grid, st);
    case 32: return fc_dispatch_mode<32>(a, mode, grid, st);
    case 40: return fc_dispatch_mode<40>(a, mode, grid, st);
    case 48: return fc_dispatch_mode<48>(a, mode, grid, st);
    case 56: return fc_dispatch_mode<56>(a, mode, grid, st);
    case 64: return fc_dispatch_mode<64>(a, mode, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

uint32_t fr_ranges_for(const FiberView& v, uint32_t nc, int num_sms) {
  const uint32_t ncp = pad_nc(nc);
  int wi, wgi, wgj;
  fr_shape(v.K, ncp, &wi, &wgi, &wgj);
  const uint32_t igroups = (v.K + uint32_t(wgi * wi) - 1) / uint32_t(wgi * wi);
  const uint64_t F = v.s * v.P;
  const uint64_t step = uint64_t(kSub) * wgj;
  const uint64_t steps = (F + step - 1) / step;
  // about one CTA per SM, and at least a few steps per range
  uint64_t ranges = std::max<uint64_t>(1, uint64_t(num_sms) / igroups);
  ranges = std::min<uint64_t>(ranges, std::max<uint64_t>(1, steps / 4));
  return uint32_t(ranges);
}

cudaError_t launch_fr(FrArgs a, int num_sms, cudaStream_t st, uint32_t* ranges_used,
                      uint32_t* grid_used) {
  const uint32_t ncp = pad_nc(a.nc);
  int wi, wgi, wgj;
  fr_shape(a.in.K, ncp, &wi, &wgi, &wgj);
  a.igroups = (a.in.K + uint32_t(wgi * wi) - 1) / uint32_t(wgi * wi);
  a.ranges = fr_ranges_for(a.in, a.nc, num_sms);
  const uint64_t F = a.in.s * a.in.P;
  const uint64_t step = uint64_t(kSub) * wgj;
  const uint64_t steps = (F + step - 1) / step;
  a.fibers_per_range = (steps + a.ranges - 1) / a.ranges * step;
  a.ranges = uint32_t((F + a.fibers_per_range - 1) / a.fibers_per_range);
  a.ncp = ncp;
  if (ranges_used) *ranges_used = a.ranges;
  if (grid_used) *grid_used = a.ranges * a.igroups;
  const int mode = fr_mode(a.in);
  switch (ncp) {
    case 8: return fr_dispatch_mode<8>(a, mode, wgi, wgj, st);
    case 16: return fr_dispatch_mode<16>(a, mode, wgi, wgj, st);
    case 24: return fr_dispatch_mode<24>(a, mode, wgi, wgj, st);
    case 32: return fr_dispatch_mode<32>(a, mode, wgi, wgj, st);
    case 40: return fr_dispatch_mode<40>(a, mode, wgi, wgj, st);
    case 48: return fr_dispatch_mode<48>(a, mode, wgi, wgj, st);
    case 56: return fr_dispatch_mode<56>(a, mode, wgi, wgj, st);
    case 64: return fr_dispatch_mode<64>(a, mode, wgi, wgj, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tkg
