// Fused ALS sweep pass for the HBM-bound ranks (r <= 16): one read of the
// tensor gives R = A_(n)^T L' (als.cpp:36-44), R^T R and the left-update sum
// Y = A_(n) R (als.cpp:46-50).
//
// A CTA streams tiles of TF whole fibers (all K = I_n entries of each) through
// a TMA ring: thread 0 issues the load of tile it + stages right after the
// CTA barrier that ends tile it (whose stage it refills), so there is no
// producer warp and no empty
// barriers: 8 warps per CTA, two CTAs per SM at 128 registers. For a tile, the
// eight warps
//   1. form the tile's TF x r block of R: DMMA with the fibers on M and the
//      contraction index on K, K split over 8 / (TF/8) warps per row tile, the
//      K-partials summed through shared memory in a fixed order and the block
//      written to R (row-major) and kept in shared memory;
//   2. add A_tile R_tile to the CTA's K x r accumulator of Y (each warp owns
//      the row tiles w, w+8, ... of Y in registers for the whole kernel), and
//      one k-step each of the tile's contribution to R^T R;
// from the same shared-memory copy of the tile: the A fragments of step 1
// (fiber, index) and step 2 (index, fiber) are both conflict-free with the
// pitch 4 (mod 16) the TMA boxes are padded to. Per CTA the partial of Y goes
// out in the FR kernels' split-K layout and the Gram partial in the FC
// epilogue's, so the surrounding small steps (finish_step, prep_step) are
// the unfused path's. With r mod 8 in {1, 2} the last column tile runs as a
// DFMA tail (see fc_tma_kernel).
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

struct SweepGeom {
  uint64_t s = 0, P = 0, F = 0, tpp = 1, ntiles = 0;
  uint32_t K = 0, K4 = 0, MT = 0;    // contraction extent, rounded to 4, row tiles of Y
  uint32_t ldA = 0, nch = 1;         // A pitch in smem; 128-row boxes per stage (kFibI)
  uint32_t kper = 0;                 // indices per K split of step 1 (multiple of 4)
  uint32_t stage_bytes = 0, stages = 0, bytes_tx = 0, bytes_ms = 0;
  uint32_t off_ms = 0, off_ps = 0, off_rs = 0, off_ring = 0;
  uint32_t ctas_per_sm = 1;
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

template <int TAIL>
__device__ __forceinline__ void tail_sum(double (&t)[2], double& a0, double& a1, int q) {
  double v0 = t[0], v1 = t[1];
  v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
  v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
  v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
  a0 = q == 0 ? v0 : 0.0;  // accumulator-tile layout: lane (r8, q) holds columns 2q, 2q+1
  a1 = q == 0 ? v1 : 0.0;
}

template <int NC, int MODE, int TF, int TAIL>
__global__ void __launch_bounds__(kCons * 32, 2)
    sweep_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmM,
                       SweepFusedArgs a, SweepGeom g) {
  using C = SwC<NC, TAIL>;
  constexpr int kND = C::kND, kNT = C::kNT, kLdS = C::kLdS;
  constexpr int kMT1 = TF / 8;       // row tiles of the tile's R block
  constexpr int kKS = 8 / kMT1;      // K splits of step 1
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched with PDL (see fc_tma_kernel)
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* mfull = full + 8;
  double* Ms = reinterpret_cast<double*>(smem_raw + g.off_ms);
  double* Ps = reinterpret_cast<double*>(smem_raw + g.off_ps);
  double* Rs = reinterpret_cast<double*>(smem_raw + g.off_rs);
  unsigned char* ring = smem_raw + g.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stages = int(g.stages);

  // the load of the CTA's n-th tile into stage n % stages
  auto issue = [&](uint32_t n) {
    const uint64_t tile = blockIdx.x + uint64_t(n) * gridDim.x;
    if (tile >= g.ntiles) return;
    const int slot = n % stages;
    unsigned char* st = ring + size_t(slot) * g.stage_bytes;
    mbar_arrive_expect_tx(&full[slot], g.bytes_tx);
    if (MODE == kFibI) {
      tma_2d(st, &tmA, &full[slot], 0, int(tile * TF));
      if (g.nch > 1) tma_2d(st + size_t(TF) * g.ldA * 8, &tmA, &full[slot], 128, int(tile * TF));
    } else {
      const uint64_t p = tile / g.tpp;
      tma_3d(st, &tmA, &full[slot], int((tile - p * g.tpp) * TF), 0, int(p));
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    mbar_init(mfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    prefetch_map(&tmA);
    prefetch_map(&tmM);
    mbar_arrive_expect_tx(mfull, g.bytes_ms);
    tma_2d(Ms, &tmM, mfull, 0, 0);
    for (int n = 0; n < stages; ++n) issue(uint32_t(n));
  }
  __syncthreads();

  // ---------------- consumers ----------------
  const int q = lane & 3, r8 = lane >> 2;
  const int lda = int(g.ldA);
  // step 1: row tile m1 of the R block, K split ks: indices kbeg + 4*j + q,
  // j < nks1; element (fiber f, index i) of a stage sits at
  //   kFibI: ((i >> 7) * TF + f) * lda + (i & 127)   (a split never crosses a 128-row box)
  //   kFibJ: i * lda + f
  const int m1 = warp % kMT1, ks = warp / kMT1;
  const int kbeg = ks * int(g.kper), kend = min(int(g.K4), kbeg + int(g.kper));
  const int nks1 = kend > kbeg ? (kend - kbeg) / 4 : 0;
  const int f1 = m1 * 8 + r8;
  const int a1off = MODE == kFibI ? ((kbeg >> 7) * TF + f1) * lda + (kbeg & 127) + q : (kbeg + q) * lda + f1;
  const int a1step = MODE == kFibI ? 4 : 4 * lda;
  const int m1off = (kbeg + q) * kLdS;
  // step 2: row tiles warp, warp + 8, ... of Y; fiber kk = 4*t + q
  const int mw = warp < int(g.MT) ? (int(g.MT) - warp + 7) / 8 : 0;
  const bool split = g.MT <= 16;
  int a2off[4];
#pragma unroll
  for (int rt = 0; rt < 4; ++rt) {
    const int i = (warp + 8 * rt) * 8 + r8;
    a2off[rt] = MODE == kFibI ? ((i >> 7) * TF + q) * lda + (i & 127) : i * lda + q;
  }
  const int a2step = MODE == kFibI ? 4 * lda : 4;
  double yacc[4][kND][2], ytl[4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
    for (int n = 0; n < kND; ++n) yacc[mi][n][0] = yacc[mi][n][1] = 0.0;
    ytl[mi][0] = ytl[mi][1] = 0.0;
  }
  double gacc[C::kTri][2];
#pragma unroll
  for (int t = 0; t < C::kTri; ++t) gacc[t][0] = gacc[t][1] = 0.0;

  // step 2 for a compile-time row-tile count MW (and the two-chain split for
  // MW <= 2): every load and DMMA of the tile unrolled and branch-free
  auto step2 = [&](const double* As, auto mw_c, auto split_c) {
    constexpr int MW = decltype(mw_c)::value;
    constexpr bool SPLIT = decltype(split_c)::value;
#pragma unroll
    for (int t = 0; t < TF / 4; ++t) {
      const int kk = 4 * t + q;
      double bf[kND];
#pragma unroll
      for (int n = 0; n < kND; ++n) bf[n] = Rs[kk * kLdS + n * 8 + r8];
      double2 bt = make_double2(0.0, 0.0);
      if constexpr (TAIL != 0) bt = *reinterpret_cast<const double2*>(Rs + kk * kLdS + kND * 8);
      double af[MW > 0 ? MW : 1];
#pragma unroll
      for (int rt = 0; rt < MW; ++rt) af[rt] = As[a2off[rt] + t * a2step];
#pragma unroll
      for (int rt = 0; rt < MW; ++rt) {
        // SPLIT: slots 2, 3 take the odd k-steps of row tiles 0, 1 (two chains per tile)
        const int mi = SPLIT ? rt + 2 * (t & 1) : rt;
#pragma unroll
        for (int n = 0; n < kND; ++n) dmma(yacc[mi][n][0], yacc[mi][n][1], af[rt], bf[n]);
        if constexpr (TAIL != 0) {
          ytl[mi][0] = fma(af[rt], bt.x, ytl[mi][0]);
          ytl[mi][1] = fma(af[rt], bt.y, ytl[mi][1]);
        }
      }
      if (t == warp) {
        double gf[kNT];
#pragma unroll
        for (int n = 0; n < kND; ++n) gf[n] = bf[n];
        if constexpr (TAIL != 0) gf[kND] = r8 < kLdS - kND * 8 ? Rs[kk * kLdS + kND * 8 + r8] : 0.0;
        int idx = 0;
#pragma unroll
        for (int tm = 0; tm < kNT; ++tm)
#pragma unroll
          for (int tn = tm; tn < kNT; ++tn, ++idx) dmma(gacc[idx][0], gacc[idx][1], gf[tm], gf[tn]);
      }
    }
  };

  mbar_wait(mfull, 0);
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
    const int slot = it % stages;
    const uint32_t ph = (it / stages) & 1;
    mbar_wait(&full[slot], ph);
    const double* As = reinterpret_cast<const double*>(ring + size_t(slot) * g.stage_bytes);

    // ---- step 1: K-partial of rows m1*8 .. +7 of the R block ----
    // (kCh interleaved accumulator chains: one row tile gives a warp a single
    // chain of dependent DMMAs, which runs at their latency, not their rate)
    {
      constexpr int kCh = 4;
      double acc[kCh][kND][2], tl[kCh][2];
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
#pragma unroll
        for (int n = 0; n < kND; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
        tl[u][0] = tl[u][1] = 0.0;
      }
      const double* a1 = As + a1off;
      const double* b1 = Ms + m1off;
      for (int j0 = 0; j0 < nks1; j0 += kCh) {
        // k-steps past the split read its last step again with a zero A fragment
        double af[kCh], bf[kCh][kND > 0 ? kND : 1];
        double2 bt[kCh];
#pragma unroll
        for (int u = 0; u < kCh; ++u) {
          const bool ok = j0 + u < nks1;
          const int j = ok ? j0 + u : nks1 - 1;
          const double v = a1[j * a1step];
          af[u] = ok ? v : 0.0;
#pragma unroll
          for (int n = 0; n < kND; ++n) bf[u][n] = b1[j * 4 * kLdS + n * 8 + r8];
          if constexpr (TAIL != 0) bt[u] = *reinterpret_cast<const double2*>(b1 + j * 4 * kLdS + kND * 8);
        }
#pragma unroll
        for (int u = 0; u < kCh; ++u) {
#pragma unroll
          for (int n = 0; n < kND; ++n) dmma(acc[u][n][0], acc[u][n][1], af[u], bf[u][n]);
          if constexpr (TAIL != 0) {
            tl[u][0] = fma(af[u], bt[u].x, tl[u][0]);
            tl[u][1] = fma(af[u], bt[u].y, tl[u][1]);
          }
        }
      }
#pragma unroll
      for (int n = 0; n < kND; ++n) {
        acc[0][n][0] = (acc[0][n][0] + acc[1][n][0]) + (acc[2][n][0] + acc[3][n][0]);
        acc[0][n][1] = (acc[0][n][1] + acc[1][n][1]) + (acc[2][n][1] + acc[3][n][1]);
      }
      double* prow = Ps + (ks * TF + m1 * 8 + r8) * kLdS;
#pragma unroll
      for (int n = 0; n < kND; ++n)
        *reinterpret_cast<double2*>(prow + n * 8 + 2 * q) = make_double2(acc[0][n][0], acc[0][n][1]);
      if constexpr (TAIL != 0) {
        double tt[2] = {(tl[0][0] + tl[1][0]) + (tl[2][0] + tl[3][0]), (tl[0][1] + tl[1][1]) + (tl[2][1] + tl[3][1])};
        double t0, t1;
        tail_sum<TAIL>(tt, t0, t1, q);
        if (kND * 8 + 2 * q < kLdS) *reinterpret_cast<double2*>(prow + kND * 8 + 2 * q) = make_double2(t0, t1);
      }
    }
    __syncthreads();

    // ---- the R block: fixed-order sum of the K partials, to smem and to R ----
    {
      constexpr int kItems = TF * (NC / 2);
      const int t = threadIdx.x;
      if (t < kItems) {
        const int f = t / (NC / 2), c = 2 * (t % (NC / 2));
        double2 v = make_double2(0.0, 0.0);
        if (c < kLdS) {
#pragma unroll
          for (int k = 0; k < kKS; ++k) {
            const double2 p = *reinterpret_cast<const double2*>(Ps + (k * TF + f) * kLdS + c);
            v.x += p.x;
            v.y += p.y;
          }
          *reinterpret_cast<double2*>(Rs + f * kLdS + c) = v;
        }
        uint64_t row;
        bool ok;
        if (MODE == kFibI) {
          row = tile * TF + f;
          ok = row < g.F;
        } else {
          const uint64_t p = tile / g.tpp, jl = (tile - p * g.tpp) * TF + f;
          row = p * g.s + jl;
          ok = jl < g.s;
        }
        if (ok) *reinterpret_cast<double2*>(a.R + row * NC + c) = v;
      }
    }
    __syncthreads();

    // ---- step 2: Y += A_tile R_tile; one k-step of R_tile^T R_tile per warp ----
    {
      using std::integral_constant;
      if (split) {
        if (mw == 2) step2(As, integral_constant<int, 2>{}, integral_constant<bool, true>{});
        else if (mw == 1) step2(As, integral_constant<int, 1>{}, integral_constant<bool, true>{});
        else step2(As, integral_constant<int, 0>{}, integral_constant<bool, true>{});
      } else {
        if (mw == 4) step2(As, integral_constant<int, 4>{}, integral_constant<bool, false>{});
        else if (mw == 3) step2(As, integral_constant<int, 3>{}, integral_constant<bool, false>{});
        else step2(As, integral_constant<int, 2>{}, integral_constant<bool, false>{});
      }
    }
    // every warp is done with the tile: refill its stage at once
    __syncthreads();
    if (threadIdx.x == 0) issue(it + uint32_t(stages));
  }

  // ---- this CTA's partial of Y (the FR split-K layout) ----
  {
    double* dst0 = a.partial + size_t(blockIdx.x) * g.K * NC;
    if (split) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
#pragma unroll
        for (int n = 0; n < kND; ++n) {
          yacc[mi][n][0] += yacc[mi + 2][n][0];
          yacc[mi][n][1] += yacc[mi + 2][n][1];
        }
        ytl[mi][0] += ytl[mi + 2][0];
        ytl[mi][1] += ytl[mi + 2][1];
      }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      double t0 = 0.0, t1 = 0.0;
      if constexpr (TAIL != 0) tail_sum<TAIL>(ytl[mi], t0, t1, q);
      const int i = (warp + 8 * mi) * 8 + r8;
      if (mi >= mw || i >= int(g.K)) continue;
#pragma unroll
      for (int n = 0; n < kND; ++n)
        *reinterpret_cast<double2*>(dst0 + size_t(i) * NC + n * 8 + 2 * q) = make_double2(yacc[mi][n][0], yacc[mi][n][1]);
      if constexpr (TAIL != 0)
        *reinterpret_cast<double2*>(dst0 + size_t(i) * NC + kND * 8 + 2 * q) = make_double2(t0, t1);
    }
  }
  // ---- Gram partial: fixed-order sum over the warps (the ring is free: every
  //      stage has been consumed) ----
  __syncthreads();
  double* gs = reinterpret_cast<double*>(ring);
#pragma unroll
  for (int t = 0; t < C::kTri; ++t) {
    gs[(warp * C::kTri + t) * 64 + lane * 2] = gacc[t][0];
    gs[(warp * C::kTri + t) * 64 + lane * 2 + 1] = gacc[t][1];
  }
  __syncthreads();
  double* gout = a.gram_part + size_t(blockIdx.x) * NC * NC;
  for (int e = threadIdx.x; e < C::kTri * 64; e += kCons * 32) {
    double s = 0.0;
    for (int w = 0; w < kCons; ++w) s += gs[w * C::kTri * 64 + e];
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
  g->K4 = (v.K + 3) / 4 * 4;
  g->MT = (v.K + 7) / 8;
  const uint32_t K8 = g->MT * 8;
  const uint32_t lds = (ncp == 8 || tail) ? 12 : 20;
  if (mode == kFibI) {
    g->nch = v.K > 128 ? 2 : 1;
    g->ldA = g->nch == 2 ? 132 : v.K + (4 + 16 - v.K % 16) % 16;
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
    g->stage_bytes = K8 * g->ldA * 8;  // step 2 reads row tiles up to K8 (rows past K4 are never used)
  }
  g->stage_bytes = (g->stage_bytes + 127) / 128 * 128;
  const int ks = 8 / (TF / 8);
  g->kper = ((g->K4 / 4 + ks - 1) / ks) * 4;
  if (mode == kFibI && g->nch == 2) g->kper = 64;  // 4 splits, none crossing the 128-row box
  g->bytes_ms = g->K4 * lds * 8;
  uint32_t off = 1024;
  g->off_ms = off;
  off += (g->bytes_ms + 127) / 128 * 128;
  g->off_ps = off;
  off += 64 * lds * 8;
  g->off_rs = off;
  off += (TF * lds * 8 + 127) / 128 * 128;
  g->off_ring = off;
  // two CTAs per SM when two stages each fit (the tile steps are short and
  // separated by CTA barriers: a second CTA fills the first one's bubbles);
  // 128 bytes of slack after the ring (row tiles past K read past a stage)
  const uint32_t per_sm = 233472u, reserved = 1024u;
  uint32_t budget = per_sm / 2 - reserved - 128u;
  g->ctas_per_sm = 2;
  if (off + 2 * g->stage_bytes > budget) {
    budget = 226u * 1024u - 128u;
    g->ctas_per_sm = 1;
    if (off + 2 * g->stage_bytes > budget) return false;
  }
  g->stages = std::min<uint32_t>(6, (budget - off) / g->stage_bytes);
  return g->stages >= 2 && g->stages * g->stage_bytes >= 8u * 3u * 64u * 8u;  // the Gram reduction reuses the ring
}

template <int NC, int MODE, int TF, int TAIL>
cudaError_t sweep_launch(const CUtensorMap& A, const CUtensorMap& M, const SweepFusedArgs& a, const SweepGeom& g,
                         int grid, cudaStream_t st) {
  auto k = sweep_fused_kernel<NC, MODE, TF, TAIL>;
  const size_t smem = size_t(g.off_ring) + size_t(g.stages) * g.stage_bytes + 128;
  cudaError_t e = raise_smem_limit(k, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl_threads(k, grid, kCons * 32, smem, st, A, M, a, g);
}

}  // namespace

bool sweep_fused_ok(const FiberView& v, const double* mt, uint32_t nc, const double* R) {
  if (!enabled() || !encode_fn() || nc < 1 || nc > 16 || v.K < 8 || v.K > 256 || v.K % 2 != 0) return false;
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
  return int(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(num_sms) * g.ctas_per_sm)));
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
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(g.ntiles, uint64_t(num_sms) * g.ctas_per_sm)));
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
