// Fused ALS sweep pass for the HBM-bound ranks (r <= 16): one read of the
// tensor gives R = A_(n)^T L' (als.cpp:36-44), R^T R and the left-update sum
// Y = A_(n) R (als.cpp:46-50).
//
// A CTA streams tiles of TF whole fibers (all K = I_n entries of each) through
// a TMA ring (one producer warp, mbarrier full/empty pairs) and works on each
// tile with two warp groups that never meet at a CTA barrier:
//   group A (warps 0-3), step 1: the tile's TF x r block of R, DMMA with the
//      fibers on M and the contraction index on K. TF = 32: one row tile per
//      warp over the whole K. TF = 16 (K > 128): a row tile per warp PAIR, each
//      half of K, the second warp's partial handed over through shared memory
//      behind a 64-thread named barrier. The block goes to R (row-major) from
//      the accumulators and into a 3-deep shared-memory ring (mbarrier
//      R_full / R_empty) for group B;
//   group B (warps 4-7), step 2: Y += A_tile R_tile for the row tiles
//      b, b+4, ... of Y, which the warp keeps in registers for the whole
//      kernel, and one k-step each of the tile's contribution to R^T R.
// Group A runs up to three tiles ahead of group B; both read the same
// shared-memory copy of the tile (the A fragments of step 1, (fiber, index),
// and of step 2, (index, fiber), are conflict-free with the pitch 4 (mod 16)
// the TMA boxes are padded to), and a stage is released when both are done
// with it. Each SM sub-partition holds one warp of either group, so the FP64
// pipe always has two independent DMMA streams. Per CTA the partial of Y goes
// out in the FR kernels' split-K layout and the Gram partial in the FC
// epilogue's, so the surrounding small steps (finish_step, prep_step) are the
// unfused path's. With r mod 8 in {1, 2} the last column tile runs as a DFMA
// tail (see fc_tma_kernel).
//
// Layouts: kFibI (s == 1: box [TF][K + pad], two 128-row boxes when K > 128)
// and kFibJ (panel-local tiles, box [K][TF + 4]).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "contract_tma.cuh"
#include "sweep_fused.cuh"
#include "tma_util.cuh"

namespace tkg {

namespace {

constexpr int kRBuf = 3;  // R blocks in flight between the groups

struct SweepGeom {
  uint64_t s = 0, P = 0, F = 0, tpp = 1, ntiles = 0;
  uint32_t K = 0, K4 = 0, MT = 0;    // contraction extent, rounded up to 32 (K4: zero-filled by TMA), row tiles of Y
  uint32_t ldA = 0, nch = 1;         // A pitch in smem; 128-row boxes per stage (kFibI)
  uint32_t kper = 0;                 // indices per K half of step 1 (TF = 16), else K4
  uint32_t stage_bytes = 0, stages = 0, bytes_tx = 0, bytes_ms = 0;
  uint32_t off_ms = 0, off_ps = 0, off_rs = 0, off_gs = 0, off_ring = 0;
};

template <int NC, int TAIL>
struct SwC {
  static constexpr int kNT = NC / 8;
  static constexpr int kND = TAIL ? kNT - 1 : kNT;          // column tiles on DMMA
  // pitch of the r-column operands in smem: 4 (mod 8) doubles so that the 4 k
  // lanes x 8 column lanes of a B fragment hit distinct banks
  static constexpr int kLdS = (NC == 8 || TAIL) ? 12 : 20;
  static constexpr int kTri = kNT * (kNT + 1) / 2;
};

__device__ __forceinline__ void quad_sum(double& v0, double& v1) {
  v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
  v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
}

template <int NC, int MODE, int TF, int TAIL>
__global__ void __launch_bounds__(kThreadsTma, 1)
    sweep_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                       SweepFusedArgs a, SweepGeom g) {
  using C = SwC<NC, TAIL>;
  constexpr int kND = C::kND, kNT = C::kNT, kLdS = C::kLdS;
  constexpr bool kPair = TF == 16;             // step 1 by warp pairs (two K halves)
  constexpr int kFin = kPair ? 2 : 4;          // warps that publish rows of the R block
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched with PDL (see fc_tma_kernel)
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 8;
  uint64_t* rfull = empty + 8;
  uint64_t* rempty = rfull + kRBuf;
  uint64_t* mfull = rempty + kRBuf;
  double* Ms = reinterpret_cast<double*>(smem_raw + g.off_ms);
  double* Ps = reinterpret_cast<double*>(smem_raw + g.off_ps);   // [2][2][8][kLdS] pair hand-over
  double* Rs = reinterpret_cast<double*>(smem_raw + g.off_rs);   // [kRBuf][TF][kLdS]
  double* Gs = reinterpret_cast<double*>(smem_raw + g.off_gs);   // [4][kTri][64] Gram reduction
  unsigned char* ring = smem_raw + g.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stages = int(g.stages);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    for (int b = 0; b < kRBuf; ++b) {
      mbar_init(&rfull[b], kFin);
      mbar_init(&rempty[b], 4);
    }
    mbar_init(mfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons) {
    // ---------------- producer ----------------
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmM);
      mbar_arrive_expect_tx(mfull, g.bytes_ms);
      tma_2d(Ms, &tmM, mfull, 0, 0);
      uint32_t it = 0;
      for (uint64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
        const int slot = it % stages;
        const uint32_t ph = (it / stages) & 1;
        mbar_wait(&empty[slot], ph ^ 1);
        unsigned char* st = ring + size_t(slot) * g.stage_bytes;
        mbar_arrive_expect_tx(&full[slot], g.bytes_tx);
        if (MODE == kFibI) {
          tma_2d(st, &tmA, &full[slot], 0, int(tile * TF));
          if (g.nch > 1) tma_2d(st + size_t(TF) * g.ldA * 8, &tmA, &full[slot], 128, int(tile * TF));
        } else {
          const uint64_t p = tile / g.tpp;
          tma_3d(st, &tmA, &full[slot], int((tile - p * g.tpp) * TF), 0, int(p));
        }
      }
    }
    return;
  }

  const int q = lane & 3, r8 = lane >> 2;
  const int lda = int(g.ldA);
  // element (fiber f, index i) of a stage:
  //   kFibI: ((i >> 7) * TF + f) * lda + (i & 127)   (a K half never crosses a 128-row box)
  //   kFibJ: i * lda + f

  if (warp < 4) {
    // ---------------- group A: step 1 ----------------
    const int m1 = kPair ? (warp & 1) : warp;       // row tile of the R block
    const int kh = kPair ? (warp >> 1) : 0;         // K half
    const int kbeg = kh * int(g.kper), kend = min(int(g.K4), kbeg + int(g.kper));
    const int nks = kend > kbeg ? (kend - kbeg) / 4 : 0;
    const int f1 = m1 * 8 + r8;
    const int a1off = MODE == kFibI ? ((kbeg >> 7) * TF + f1) * lda + (kbeg & 127) + q : (kbeg + q) * lda + f1;
    const int a1step = MODE == kFibI ? 4 : 4 * lda;
    const double* b1 = Ms + (kbeg + q) * kLdS;
    constexpr int kCh = 4;  // interleaved accumulator chains
    mbar_wait(mfull, 0);
    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
      const int slot = it % stages;
      mbar_wait(&full[slot], (it / stages) & 1);
      const double* a1 = reinterpret_cast<const double*>(ring + size_t(slot) * g.stage_bytes) + a1off;
      double acc[kCh][kND > 0 ? kND : 1][2], tl[kCh][2];
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
#pragma unroll
        for (int n = 0; n < kND; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
        tl[u][0] = tl[u][1] = 0.0;
      }
      // groups of four k-steps (the index range is padded with zero-fill),
      // two operand sets in turn: the loads of the
      // next group fly under this group's DMMAs, without register copies
      double af[2][kCh], bf[2][kCh][kND > 0 ? kND : 1];
      double2 bt[2][kCh];
      auto load = [&](int set, const double* ap, const double* bp) {
#pragma unroll
        for (int u = 0; u < kCh; ++u) {
          af[set][u] = ap[u * a1step];
#pragma unroll
          for (int n = 0; n < kND; ++n) bf[set][u][n] = bp[u * 4 * kLdS + n * 8 + r8];
          if constexpr (TAIL != 0) bt[set][u] = *reinterpret_cast<const double2*>(bp + u * 4 * kLdS + kND * 8);
        }
      };
      auto mma = [&](int set) {
#pragma unroll
        for (int u = 0; u < kCh; ++u) {
#pragma unroll
          for (int n = 0; n < kND; ++n) dmma(acc[u][n][0], acc[u][n][1], af[set][u], bf[set][u][n]);
          if constexpr (TAIL != 0) {
            tl[u][0] = fma(af[set][u], bt[set][u].x, tl[u][0]);
            tl[u][1] = fma(af[set][u], bt[set][u].y, tl[u][1]);
          }
        }
      };
      // (an even number of groups: the index range is padded to a multiple of
      // 32; the load after the last group reads on inside the ring / the
      // slack behind it and is never used)
      const double* ap = a1;
      const double* bp = b1;
      load(0, ap, bp);
      for (int gi = 0; gi < nks / kCh; gi += 2) {
        load(1, ap + kCh * a1step, bp + kCh * 4 * kLdS);
        mma(0);
        ap += 2 * kCh * a1step;
        bp += 2 * kCh * 4 * kLdS;
        load(0, ap, bp);
        mma(1);
      }
      // this warp is done with the stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      // the block's rows in accumulator-tile layout: lane (r8, q) holds columns
      // n*8 + 2q, +1 of row r8; the tail tile from the k-lane sums
      double rt[kNT][2];
#pragma unroll
      for (int n = 0; n < kND; ++n) {
        rt[n][0] = (acc[0][n][0] + acc[1][n][0]) + (acc[2][n][0] + acc[3][n][0]);
        rt[n][1] = (acc[0][n][1] + acc[1][n][1]) + (acc[2][n][1] + acc[3][n][1]);
      }
      if constexpr (TAIL != 0) {
        double t0 = (tl[0][0] + tl[1][0]) + (tl[2][0] + tl[3][0]);
        double t1 = (tl[0][1] + tl[1][1]) + (tl[2][1] + tl[3][1]);
        quad_sum(t0, t1);
        rt[kND][0] = q == 0 ? t0 : 0.0;
        rt[kND][1] = q == 0 ? t1 : 0.0;
      }
      if constexpr (kPair) {
        // the second K half hands its partial to the pair's first warp
        double* pp = Ps + (((it & 1) * 2 + m1) * 8 + r8) * kLdS;
        if (kh == 1) {
#pragma unroll
          for (int n = 0; n < kNT; ++n)
            if (n * 8 + 2 * q < kLdS) *reinterpret_cast<double2*>(pp + n * 8 + 2 * q) = make_double2(rt[n][0], rt[n][1]);
        }
        asm volatile("bar.sync %0, 64;\n" ::"r"(2 + m1) : "memory");
        if (kh == 1) continue;
#pragma unroll
        for (int n = 0; n < kNT; ++n)
          if (n * 8 + 2 * q < kLdS) {
            const double2 p = *reinterpret_cast<const double2*>(pp + n * 8 + 2 * q);
            rt[n][0] += p.x;
            rt[n][1] += p.y;
          }
      }
      // publish: R (row-major, all NC columns) and the shared ring for group B
      const int buf = it % kRBuf;
      mbar_wait(&rempty[buf], ((it / kRBuf) & 1) ^ 1);
      double* rs = Rs + (buf * TF + f1) * kLdS;
#pragma unroll
      for (int n = 0; n < kNT; ++n)
        if (n * 8 + 2 * q < kLdS) *reinterpret_cast<double2*>(rs + n * 8 + 2 * q) = make_double2(rt[n][0], rt[n][1]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfull[buf]);
      uint64_t row;
      bool ok;
      if (MODE == kFibI) {
        row = tile * TF + f1;
        ok = row < g.F;
      } else {
        const uint64_t p = tile / g.tpp, jl = (tile - p * g.tpp) * TF + f1;
        row = p * g.s + jl;
        ok = jl < g.s;
      }
      if (ok) {
#pragma unroll
        for (int n = 0; n < kNT; ++n)
          *reinterpret_cast<double2*>(a.R + row * NC + n * 8 + 2 * q) = make_double2(rt[n][0], rt[n][1]);
      }
    }
    return;
  }

  // ---------------- group B: step 2 and the Gram ----------------
  const int b = warp - 4;
  const int mw = b < int(g.MT) ? (int(g.MT) - b + 3) / 4 : 0;   // row tiles b, b+4, ... of Y
  const int mwmax = (int(g.MT) + 3) / 4;
  int a2off[8];
#pragma unroll
  for (int rt = 0; rt < 8; ++rt) {
    // row tiles past this warp's count read its last one (their sums are never stored)
    const int t = rt < mw ? rt : (mw > 0 ? mw - 1 : 0);
    const int i = (b + 4 * t) * 8 + r8;
    a2off[rt] = MODE == kFibI ? ((i >> 7) * TF + q) * lda + (i & 127) : i * lda + q;
  }
  const int a2step = MODE == kFibI ? 4 * lda : 4;
  double yacc[8][kND > 0 ? kND : 1][2], ytl[8][2];
#pragma unroll
  for (int mi = 0; mi < 8; ++mi) {
#pragma unroll
    for (int n = 0; n < kND; ++n) yacc[mi][n][0] = yacc[mi][n][1] = 0.0;
    ytl[mi][0] = ytl[mi][1] = 0.0;
  }
  double gacc[C::kTri][2];
#pragma unroll
  for (int t = 0; t < C::kTri; ++t) gacc[t][0] = gacc[t][1] = 0.0;

  // one tile for a compile-time row-tile count: every load and DMMA unrolled
  auto step2 = [&](const double* As, const double* rs, auto mw_c) {
    constexpr int MW = decltype(mw_c)::value;
#pragma unroll
    for (int t = 0; t < TF / 4; ++t) {
      const int kk = 4 * t + q;
      double bf[kND > 0 ? kND : 1];
#pragma unroll
      for (int n = 0; n < kND; ++n) bf[n] = rs[kk * kLdS + n * 8 + r8];
      double2 bt = make_double2(0.0, 0.0);
      if constexpr (TAIL != 0) bt = *reinterpret_cast<const double2*>(rs + kk * kLdS + kND * 8);
      double af[MW];
#pragma unroll
      for (int rt = 0; rt < MW; ++rt) af[rt] = As[a2off[rt] + t * a2step];
#pragma unroll
      for (int rt = 0; rt < MW; ++rt) {
#pragma unroll
        for (int n = 0; n < kND; ++n) dmma(yacc[rt][n][0], yacc[rt][n][1], af[rt], bf[n]);
        if constexpr (TAIL != 0) {
          ytl[rt][0] = fma(af[rt], bt.x, ytl[rt][0]);
          ytl[rt][1] = fma(af[rt], bt.y, ytl[rt][1]);
        }
      }
      if ((t & 3) == b) {  // the tile's R^T R: k-steps dealt to the four warps
        double gf[kNT];
#pragma unroll
        for (int n = 0; n < kND; ++n) gf[n] = bf[n];
        if constexpr (TAIL != 0) gf[kND] = r8 < kLdS - kND * 8 ? rs[kk * kLdS + kND * 8 + r8] : 0.0;
        int idx = 0;
#pragma unroll
        for (int tm = 0; tm < kNT; ++tm)
#pragma unroll
          for (int tn = tm; tn < kNT; ++tn, ++idx) dmma(gacc[idx][0], gacc[idx][1], gf[tm], gf[tn]);
      }
    }
  };

  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
    const int slot = it % stages, buf = it % kRBuf;
    mbar_wait(&full[slot], (it / stages) & 1);
    mbar_wait(&rfull[buf], (it / kRBuf) & 1);
    const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * g.stage_bytes);
    const double* rs = Rs + buf * TF * kLdS;
    using std::integral_constant;
    switch (mwmax) {
      case 1: step2(As, rs, integral_constant<int, 1>{}); break;
      case 2: step2(As, rs, integral_constant<int, 2>{}); break;
      case 3: step2(As, rs, integral_constant<int, 3>{}); break;
      case 4: step2(As, rs, integral_constant<int, 4>{}); break;
      case 5: step2(As, rs, integral_constant<int, 5>{}); break;
      case 6: step2(As, rs, integral_constant<int, 6>{}); break;
      case 7: step2(As, rs, integral_constant<int, 7>{}); break;
      default: step2(As, rs, integral_constant<int, 8>{}); break;
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[slot]);
      mbar_arrive(&rempty[buf]);
    }
  }

  // ---- this CTA's partial of Y (the FR split-K layout) ----
  {
    double* dst0 = a.partial + size_t(blockIdx.x) * g.K * NC;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      double t0 = ytl[mi][0], t1 = ytl[mi][1];
      if constexpr (TAIL != 0) quad_sum(t0, t1);
      const int i = (b + 4 * mi) * 8 + r8;
      if (mi >= mw || i >= int(g.K)) continue;
#pragma unroll
      for (int n = 0; n < kND; ++n)
        *reinterpret_cast<double2*>(dst0 + size_t(i) * NC + n * 8 + 2 * q) = make_double2(yacc[mi][n][0], yacc[mi][n][1]);
      if constexpr (TAIL != 0)
        *reinterpret_cast<double2*>(dst0 + size_t(i) * NC + kND * 8 + 2 * q) =
            make_double2(q == 0 ? t0 : 0.0, q == 0 ? t1 : 0.0);
    }
  }
  // ---- Gram partial: fixed-order sum over the four warps ----
#pragma unroll
  for (int t = 0; t < C::kTri; ++t) {
    Gs[(b * C::kTri + t) * 64 + lane * 2] = gacc[t][0];
    Gs[(b * C::kTri + t) * 64 + lane * 2 + 1] = gacc[t][1];
  }
  asm volatile("bar.sync 4, 128;\n" ::: "memory");
  double* gout = a.gram_part + size_t(blockIdx.x) * NC * NC;
  for (int e = threadIdx.x - 128; e < C::kTri * 64; e += 128) {
    double s = 0.0;
    for (int w = 0; w < 4; ++w) s += Gs[w * C::kTri * 64 + e];
    const int t = e / 64, l = (e % 64) / 2, el = e % 2;
    int tm = 0, rem = t;
    while (rem >= kNT - tm) {
      rem -= kNT - tm;
      ++tm;
    }
    const int tn = tm + rem;
    gout[(tm * 8 + (l >> 2)) * NC + tn * 8 + 2 * (l & 3) + el] = s;
  }
}

// TKG_FUSED_SWEEP=0: never; the per-context default is Engine::fused_sweep_
// (off: see DESIGN.md, the pass is faster than FC + FR back to back in
// isolation but not yet inside the decompositions)
bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TKG_FUSED_SWEEP");
    return !(e && e[0] == '0');
  }();
  return on;
}

// fibers per tile: a tile of TF * K elements stays between 2 K and 4 K doubles
int tile_fibers(uint32_t K) { return K <= 128 ? 32 : 16; }

int layout(const FiberView& v) {
  if (v.s == 1 && v.is_i == 1 && v.is_p % 2 == 0) return kFibI;
  if (v.s % 2 == 0 && v.is_i % 2 == 0 && v.is_p % 2 == 0 && v.s >= 64 && v.P < (1ull << 31)) return kFibJ;
  return -1;
}

bool geometry(const FiberView& v, uint32_t ncp, int tail, int mode, SweepGeom* g) {
  const int TF = tile_fibers(v.K);
  g->s = v.s;
  g->P = v.P;
  g->F = v.s * v.P;
  g->K = v.K;
  // step 1 runs pairs of groups of four k-steps: the index range is padded to
  // a multiple of 32 with TMA zero-fill on both operands (no edge predicates)
  g->K4 = (v.K + 31) / 32 * 32;
  g->MT = (v.K + 7) / 8;
  const uint32_t lds = (ncp == 8 || tail) ? 12 : 20;
  if (mode == kFibI) {
    g->nch = v.K > 128 ? 2 : 1;
    g->ldA = g->nch == 2 ? 132 : g->K4 + 4;
    g->tpp = 1;
    g->ntiles = (g->F + TF - 1) / TF;
    g->bytes_tx = g->nch * TF * g->ldA * 8;
    g->stage_bytes = g->bytes_tx;
  } else {
    g->nch = 1;
    g->ldA = TF + 4;
    g->tpp = (v.s + TF - 1) / TF;
    g->ntiles = g->tpp * v.P;
    g->bytes_tx = g->K4 * g->ldA * 8;
    g->stage_bytes = g->K4 * g->ldA * 8;
  }
  g->stage_bytes = (g->stage_bytes + 127) / 128 * 128;
  // step 1: TF = 32 gives each warp a row tile over the whole K; TF = 16 splits
  // K between the two warps of a pair (at the 128-row box boundary for kFibI)
  g->kper = TF == 32 ? g->K4 : (mode == kFibI ? 128 : ((g->K4 / 32 + 1) / 2) * 32);
  g->bytes_ms = g->K4 * lds * 8;
  uint32_t off = 1024;
  g->off_ms = off;
  off += (g->bytes_ms + 16 * lds * 8 + 127) / 128 * 128;  // + the over-read of step 1's last load
  g->off_ps = off;
  off += (2 * 2 * 8 * lds * 8 + 127) / 128 * 128;
  g->off_rs = off;
  off += (kRBuf * TF * lds * 8 + 127) / 128 * 128;
  g->off_gs = off;
  off += 4 * 3 * 64 * 8;
  g->off_ring = off;
  // slack after the ring: step 1's last load reads one group past the stage
  const uint32_t slack = 16u * std::max<uint32_t>(g->ldA, 8u) * 8u + 128u;
  const uint32_t budget = 226u * 1024u - slack;
  if (off + 2 * g->stage_bytes > budget) return false;
  g->stages = std::min<uint32_t>(8, (budget - off) / g->stage_bytes);
  return g->stages >= 2;
}

template <int NC, int MODE, int TF, int TAIL>
cudaError_t sweep_launch(const CUtensorMap& A, const CUtensorMap& M, const SweepFusedArgs& a, const SweepGeom& g,
                         int grid, cudaStream_t st) {
  auto k = sweep_fused_kernel<NC, MODE, TF, TAIL>;
  const size_t smem = size_t(g.off_ring) + size_t(g.stages) * g.stage_bytes + 16 * std::max<uint32_t>(g.ldA, 8u) * 8 + 128;
  cudaError_t e = raise_smem_limit(k, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, smem, st, A, M, a, g);
}

}  // namespace

bool sweep_fused_ok(const FiberView& v, const double* mt, uint32_t nc, const double* R) {
  if (!enabled() || !encode_fn() || nc < 1 || nc > 16 || v.K < 32 || v.K > 256 || v.K % 2 != 0) return false;
  if (!aligned16(v.base) || !aligned16(mt) || !aligned16(R)) return false;
  if (v.s * v.P >= (1ull << 31)) return false;
  const int mode = layout(v);
  if (mode < 0) return false;
  SweepGeom g;
  return geometry(v, pad_nc(nc), dfma_tail(nc) ? 2 : 0, mode, &g);
}

int sweep_fused_grid(const FiberView& v, uint32_t nc, int num_sms) {
  const int TF = tile_fibers(v.K);
  const int mode = layout(v);
  SweepGeom g;
  if (mode < 0 || !geometry(v, pad_nc(nc), dfma_tail(nc) ? 2 : 0, mode, &g)) return 1;
  const uint64_t tiles = mode == kFibI ? (v.s * v.P + TF - 1) / TF : (v.s + TF - 1) / TF * v.P;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms))));
}

cudaError_t launch_sweep_fused(const FiberView& v, const SweepFusedArgs& a, int num_sms, cudaStream_t st,
                               int* grid_used) {
  const uint32_t ncp = pad_nc(a.nc);
  const int tail = dfma_tail(a.nc) ? 2 : 0;
  const int mode = layout(v);
  SweepGeom g;
  if (mode < 0 || !geometry(v, ncp, tail, mode, &g)) return cudaErrorInvalidValue;
  const int TF = tile_fibers(v.K);
  const uint32_t lds = (ncp == 8 || tail) ? 12 : 20;
  CUtensorMap A, M;
  if (mode == kFibI) {
    const uint64_t dims[2] = {v.K, g.F};
    const uint64_t strides[1] = {v.is_p * 8};
    const uint32_t box[2] = {g.ldA, uint32_t(TF)};
    if (!encode(&A, v.base, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const uint64_t dims[3] = {v.s, v.K, v.P};
    const uint64_t strides[2] = {v.is_i * 8, v.is_p * 8};
    const uint32_t box[3] = {g.ldA, g.K4, 1};
    if (!encode(&A, v.base, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {ncp, v.K};
    const uint64_t strides[1] = {uint64_t(ncp) * 8};
    const uint32_t box[2] = {lds, g.K4};
    if (!encode(&M, a.mt, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(g.ntiles, uint64_t(num_sms))));
  if (grid_used) *grid_used = grid;
#define TKG_SW(N, T)                                                                                      \
  (mode == kFibI ? (TF == 32 ? sweep_launch<N, kFibI, 32, T>(A, M, a, g, grid, st)                        \
                             : sweep_launch<N, kFibI, 16, T>(A, M, a, g, grid, st))                       \
                 : (TF == 32 ? sweep_launch<N, kFibJ, 32, T>(A, M, a, g, grid, st)                        \
                             : sweep_launch<N, kFibJ, 16, T>(A, M, a, g, grid, st)))
  if (ncp == 8) return TKG_SW(8, 0);
  if (tail) return TKG_SW(16, 2);
  return TKG_SW(16, 0);
#undef TKG_SW
}

}  // namespace tkg
