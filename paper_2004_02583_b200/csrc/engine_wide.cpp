// ALS for ranks above 64 (the reference has no rank cap: als.cpp:98-161,
// kernels.cpp:369-417; the paper's runs use R = 142 and R = 500).
//
// The FC / FR contraction kernels hold at most 64 columns and the cooperative
// r x r steps of coop.cu keep the matrix in one CTA's registers, so a wide
// rank is tiled: the right factor R (row-major [F][ncp], ncp = r rounded up
// to 8) is produced 64 columns at a time by FC launches on the matching
// columns of L' = L G_L^{-1}, the left update A_(n) R 64 columns at a time by
// FR launches that read the column block of R in place, and the r x r steps
// are the reference's Cholesky + substitutions (wide.cu) on Gram matrices
// formed by the DMMA mode-Gram kernel (gram.cu). Each A pass of the r <= 64
// path becomes ceil(r / 64) passes. The stop rule is the same device-side
// control block; the host reads it once per sweep (no speculation).
#include <algorithm>
#include <string>

#include "als_step.cuh"
#include "contract.cuh"
#include "engine.hpp"
#include "wide.cuh"

namespace tkg {

namespace {
constexpr uint32_t kBlk = 64;  // columns per contraction launch
}  // namespace

// G = X^T X for the r columns of X viewed as fibers (gram.cu): rows of a
// row-major [rows][ld] matrix (row_major) or of a column-major rows x r one.
void Engine::gram_cols(const double* X, uint64_t rows, uint32_t r, uint64_t ld, bool row_major, double* G) {
  const FiberView v = row_major ? FiberView{X, 1, rows, r, 1, ld} : FiberView{X, rows, 1, r, ld, ld * r};
  const GramPlan gp = gram_tensor_plan(v, sms_);
  double* part = wide_gpart_.d(std::max<size_t>(gp.part_doubles, 1));
  CK(launch_gram_tensor(v, gp, part, G, st_));
  count_launch(2);
}

// CholQR2 of Y (column-major I x r) into Q (may alias Y): R1 = chol(Y^T Y)^T,
// Q1 = Y R1^{-1}, R2 = chol(Q1^T Q1)^T, Q = Q1 R2^{-1}, R = R2 R1 (rmat,
// nullable); ctrl->degenerate_col as cholqr_step (coop.cu).
void Engine::qr_wide(const double* Y, uint32_t I, uint32_t r, double* Q, double* rmat, bool check) {
  const size_t rr = size_t(r) * r;
  double* G = wide_g_.d(rr);
  double* C1 = wide_c1_.d(2 * rr);
  double* C1T = C1 + rr;
  double* C2 = wide_c2_.d(2 * rr);
  double* C2T = C2 + rr;
  int32_t* fails = static_cast<int32_t*>(wide_fail_.ensure(4 * sizeof(int32_t)));
  AlsCtrl* ctrl = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
  gram_cols(Y, I, r, I, false, G);
  CK(launch_wide_chol(G, r, 0.0, C1, C1T, fails, nullptr, 0, st_));
  CK(launch_wide_rowsolve(Y, I, r, 1, I, C1, C1T, 0, Q, 1, I, nullptr, sms_, st_));
  gram_cols(Q, I, r, I, false, G);
  CK(launch_wide_chol(G, r, 0.0, C2, C2T, fails + 1, nullptr, 0, st_));
  CK(launch_wide_rowsolve(Q, I, r, 1, I, C2, C2T, 0, Q, 1, I, nullptr, sms_, st_));
  CK(launch_wide_rprod(C2, C1, r, rmat, fails, check ? 1 : 0, ctrl, st_));
  count_launch(5);
}

// out <- X x_mode U^T (U: I x r device column-major) in tensor layout, in
// blocks of 64 output rows (the t-HOSVD core chain, HOOI, the st-HOSVD TTM).
void Engine::ttm_mode(const double* X, const Shape& sh, int mode, const double* U, uint32_t r, double* out,
                      bool count_pass) {
  ClsScope cls(fc_cls_, kClsTTM);
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  FiberView v{X, s, P, uint32_t(I), s, s * I};
  for (uint32_t c0 = 0; c0 < r; c0 += kBlk) {
    const uint32_t nc = std::min(kBlk, r - c0), ncp = pad_nc(nc);
    double* Mt = mt_.d(I * ncp);
    CK(launch_pack(U + uint64_t(c0) * I, 1, I, uint32_t(I), nc, Mt, ncp, st_));  // Mt[i][c] = U[i + (c0+c)*I]
    count_launch();
    fc(v, Mt, ncp, nc, out + uint64_t(c0) * s, 1, s, s * r, nullptr, nullptr, nullptr, count_pass && c0 == 0);
  }
}

Engine::AlsOut Engine::run_als_wide(const double* A, const Shape& sh, int mode, uint32_t r, const AlsCfg& cfg,
                                    bool sumsq_known, int slot) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  const uint32_t ncpR = pad_nc(r);
  const uint32_t nblk = (r + kBlk - 1) / kBlk;
  const std::string mname = "mode " + std::to_string(mode);
  if (dist_) raise(12, mname + ": ranks above 64 are not supported by the sharded drivers");
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  AlsOut out;
  out.rep.mode = mode;
  const size_t rr = size_t(r) * r;
  double* Lc = l_.d(I * r);
  double* Lp = wide_lp_.d(I * r);   // L' = L G_L^{-1}, column-major
  double* Y = qy_.d(I * r);         // A_(n) R, column-major
  double* R = r_.d(F * ncpR + 8);   // row-major [F][ncpR]
  double* GL = gl_.d(rr);
  double* GR = gr_.d(rr);
  double* C = cholL_.d(rr);
  double* CT = cholR_.d(rr);
  int32_t* fails = static_cast<int32_t*>(wide_fail_.ensure(4 * sizeof(int32_t)));
  const uint32_t nranges = fr_ranges(v, kBlk);
  double* part = fr_part_.d(size_t(nranges) * I * kBlk);
  double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(sh.count()))));
  double* sumsq = sumsq_d_.d(2);
  AlsCtrl* ctrl = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
  const int max_iters = std::max(1, cfg.max_iters);
  double* hist = hist_d_.d(size_t(max_iters));
  const int32_t* stop = &ctrl->stop;

  // Y(:, block) = sum of the FR partials of A_(n) M(:, block), M(j, c) = m[j*mj + c*mc]
  auto left_blocks = [&](const double* m, uint64_t mj, uint64_t mc, double* sumsq_part, uint32_t* grid0) {
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t c0 = b * kBlk, nc = std::min(kBlk, r - c0), ncp = pad_nc(nc);
      const uint32_t ranges = fr(v, m + c0 * mc, mj, mc, nc, part, b == 0 ? sumsq_part : nullptr, true,
                                 b == 0 ? grid0 : nullptr, stop);
      CK(launch_reduce_partials(part, int(ranges), uint32_t(I), ncp, nc, Y + uint64_t(c0) * I, st_));
      count_launch();
    }
  };

  // 1. ||A|| and the initial left factor (als.cpp:99-120)
  if (cfg.init) {
    if (!sumsq_known) {
      CK(launch_sumsq(A, sh.count(), sq, st_));
      CK(launch_sum(sq, sumsq_partials_count(sh.count()), sumsq, st_));
      count_launch(2);
    }
    CK(cudaMemcpyAsync(Lc, cfg.init, I * r * sizeof(double), cudaMemcpyHostToDevice, st_));
  } else {
    const double* S = nullptr;
    auto pit = pre_.find(mode);
    if (pit != pre_.end() && pit->second.F == F && pit->second.r == r) {
      CK(cudaStreamWaitEvent(st_, pit->second.ready, 0));
      S = pit->second.ptr;
      pre_.erase(pit);
    } else {
      double* Sg = s_.d(F * r + 8);  // column-major F x r (als.cpp:69-71)
      gen_uniform(cfg.seed, uint32_t(mode), F * r, Sg);
      S = Sg;
    }
    CK(cudaMemsetAsync(ctrl, 0, sizeof(AlsCtrl), st_));  // stop = 0 for the FR skip test
    uint32_t fr_grid = 0;
    left_blocks(S, 1, F, sumsq_known ? nullptr : sq, &fr_grid);
    if (!sumsq_known) {
      CK(launch_sum(sq, int(fr_grid), sumsq, st_));
      count_launch();
    }
    qr_wide(Y, uint32_t(I), r, Lc, nullptr, true);
  }
  CK(launch_ctrl_init(ctrl, sumsq, cfg.eta, max_iters, max_iters, cfg.init ? 0 : 1, st_));
  count_launch();
  if (!pending_pre_.empty()) {
    std::vector<PreGen> items;
    items.swap(pending_pre_);
    pregenerate(items, pending_seed_);
  }

  // 2. Sweeps (als.cpp:121-160), one host read of the control block per sweep
  AlsCtrl h{};
  for (int k = 1; k <= max_iters; ++k) {
    // right update: G_L, L' = L G_L^{-1}, R = A_(n)^T L', G_R (als.cpp:36-44)
    gram_cols(Lc, I, r, I, false, GL);
    CK(launch_wide_chol(GL, r, 1e-13, C, CT, fails, ctrl, kAlsErrRightSingular, st_));
    CK(launch_wide_rowsolve(Lc, I, r, 1, I, C, CT, 1, Lp, 1, I, ctrl, sms_, st_));
    count_launch(2);
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t c0 = b * kBlk, nc = std::min(kBlk, r - c0), ncp = pad_nc(nc);
      double* Mt = mt_.d(I * ncp);
      CK(launch_pack(Lp + uint64_t(c0) * I, 1, I, uint32_t(I), nc, Mt, ncp, st_));
      count_launch();
      fc(v, Mt, ncp, nc, R + c0, ncpR, 1, s * ncpR, nullptr, nullptr, nullptr, true, stop);
    }
    gram_cols(R, F, r, ncpR, true, GR);
    // closed-form residual and the stop rule (als.cpp:52-55, 136-150)
    CK(launch_wide_trace_stop(GL, GR, r, ctrl, hist, st_));
    count_launch();
    CK(cudaMemcpyAsync(&h, ctrl, sizeof(AlsCtrl), cudaMemcpyDeviceToHost, st_));
    sync();
    if (h.stop) break;
    // left update L = (A_(n) R) G_R^{-1} (als.cpp:46-50)
    CK(launch_wide_chol(GR, r, 1e-13, C, CT, fails, ctrl, kAlsErrLeftSingular, st_));
    left_blocks(R, ncpR, 1, nullptr, nullptr);
    CK(launch_wide_rowsolve(Y, I, r, 1, I, C, CT, 1, Lc, 1, I, ctrl, sms_, st_));
    count_launch(2);
  }
  const std::string singular = mname + ": gram matrix is singular, rank " + std::to_string(r) +
                               " exceeds the numerical rank of the iterate";
  switch (h.error) {
    case kAlsErrZeroNorm: raise(3, "als_low_rank: input tensor has zero norm");
    case kAlsErrDegenerate:
      raise(6, "als_init: randomized range collapsed at column " + std::to_string(h.degenerate_col) +
                   " for mode " + std::to_string(mode));
    case kAlsErrRightSingular:
    case kAlsErrLeftSingular: raise(4, singular);
    default: break;
  }
  ModeRep& rep = out.rep;
  rep.iterations = h.iter;
  rep.status = h.status;
  rep.achieved_eta = h.achieved;
  out.norm = h.norm;
  if (stage_n_ < size_t(slot + 1) * size_t(stage_iters_ + 1) || stage_iters_ < max_iters)
    stage_reserve(slot + 1, max_iters);
  double* hs = stage_h_ + size_t(slot) * size_t(stage_iters_ + 1);
  if (h.iter > 0) CK(cudaMemcpyAsync(hs, hist, sizeof(double) * h.iter, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(hs + stage_iters_, sumsq, sizeof(double), cudaMemcpyDeviceToHost, st_));
  out.hist_host = hs;
  out.sumsq_host = hs + stage_iters_;
  return out;
}

}  // namespace tkg
