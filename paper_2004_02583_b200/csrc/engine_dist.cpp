// Sharded t-HOSVD-ALS / st-HOSVD-ALS: one engine per GPU, the tensor split
// along its last mode (BASELINE north star), results replicated on every
// rank and equal to the single-GPU decomposition of the whole tensor.
//
// For a mode whose fibers are split across ranks (every mode but the sharded
// one) the ALS runs unchanged on the local fibers: the right factor's rows
// stay local, and only ||A||^2, the I_n x R_n left-update sum A_(n) R and the
// R_n x R_n Gram matrix R^T R are summed over ranks (Engine::run_als with
// dist_ set). The initializer S keeps the reference's stream: each rank
// generates exactly the draws of its own fibers (MtWindow). The sharded
// mode itself is first moved to another mode by one all-to-all, after which
// its fibers are local too. The core (a sum over the sharded mode of the TTM
// chain) and the residual are summed over ranks.
//
// Reference call sites: hosvd.cpp:74-125 (t_hosvd), 127-191 (st_hosvd).
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <string>

#include "comm.hpp"
#include "engine.hpp"

namespace tkg {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// Column-major strides of a shape.
void strides_of(const Shape& s, uint64_t* st) {
  uint64_t acc = 1;
  for (int k = 0; k < s.N; ++k) {
    st[k] = acc;
    acc *= s.d[k];
  }
}

// Fiber window of `mode` (1-based) when the tensor G is sharded along `sm`
// (1-based, != mode) with this rank holding [o0, o0 + n).
MtWindow fiber_window(const Shape& G, int mode, int sm, uint64_t o0, uint64_t n) {
  MtWindow w;
  w.Fg = G.count() / G.d[mode - 1];
  w.Plo = 1;
  for (int k = 0; k < sm - 1; ++k)
    if (k != mode - 1) w.Plo *= G.d[k];
  w.Gsm = G.d[sm - 1];
  w.o0 = o0;
  w.nloc = n;
  return w;
}

}  // namespace

ShardRange shard_range(uint64_t extent, int rank, int world) {
  ShardRange r;
  r.begin = extent * uint64_t(rank) / uint64_t(world);
  r.len = extent * uint64_t(rank + 1) / uint64_t(world) - r.begin;
  return r;
}

void Engine::set_comm(std::unique_ptr<Comm> c) {
  comm2_.reset();
  comm2_tried_ = false;
  comm_ = std::move(c);
}

std::mutex& Engine::coop_mutex() {
  static std::mutex m;
  return m;
}

// dst (sharded along `to`) <- src (sharded along `from`) of the global shape
// G: pack one box per destination, one alltoallv, unpack one box per source.
void Engine::reshard(const double* src, const Shape& G, int from, int to, double* dst) {
  reshard_on(src, G, from, to, dst, st_, comm_.get());
}

void Engine::reshard_on(const double* src, const Shape& G, int from, int to, double* dst, cudaStream_t st,
                        Comm* comm) {
  const int world = comm->world(), rank = comm->rank();
  Shape Ls = G, Lt = G;
  Ls.d[from - 1] = shard_range(G.d[from - 1], rank, world).len;
  Lt.d[to - 1] = shard_range(G.d[to - 1], rank, world).len;
  uint64_t ss[64], ts[64];
  strides_of(Ls, ss);
  strides_of(Lt, ts);
  std::vector<size_t> scount(world), soff(world), rcount(world), roff(world);
  size_t so = 0, ro = 0;
  for (int q = 0; q < world; ++q) {
    Shape bs = Ls;
    bs.d[to - 1] = shard_range(G.d[to - 1], q, world).len;
    scount[q] = bs.count();
    soff[q] = so;
    so += scount[q];
    Shape br = Lt;
    br.d[from - 1] = shard_range(G.d[from - 1], q, world).len;
    rcount[q] = br.count();
    roff[q] = ro;
    ro += rcount[q];
  }
  double* sendb = send_.d(std::max<size_t>(so, 1));
  double* recvb = recv_.d(std::max<size_t>(ro, 1));
  for (int q = 0; q < world; ++q) {
    BoxCopy b;
    b.N = G.N;
    Shape bs = Ls;
    const ShardRange tr = shard_range(G.d[to - 1], q, world);
    bs.d[to - 1] = tr.len;
    uint64_t bstr[64];
    strides_of(bs, bstr);
    for (int k = 0; k < G.N; ++k) {
      b.box[k] = bs.d[k];
      b.src_stride[k] = ss[k];
      b.dst_stride[k] = bstr[k];
    }
    b.src_base = tr.begin * ss[to - 1];
    b.dst_base = 0;
    CK(launch_copy_box(src, sendb + soff[q], b, st));
  }
  count_launch(world);
  comm->alltoallv(sendb, scount.data(), soff.data(), recvb, rcount.data(), roff.data(), st);
  for (int q = 0; q < world; ++q) {
    BoxCopy b;
    b.N = G.N;
    Shape br = Lt;
    const ShardRange fr_ = shard_range(G.d[from - 1], q, world);
    br.d[from - 1] = fr_.len;
    uint64_t bstr[64];
    strides_of(br, bstr);
    for (int k = 0; k < G.N; ++k) {
      b.box[k] = br.d[k];
      b.src_stride[k] = bstr[k];
      b.dst_stride[k] = ts[k];
    }
    b.src_base = 0;
    b.dst_base = fr_.begin * ts[from - 1];
    CK(launch_copy_box(recvb + roff[q], dst, b, st));
  }
  count_launch(world);
}

void Engine::check_shard(const Shape& G, uint64_t begin, uint64_t len) {
  if (!comm_) raise(12, "sharded decomposition: no communicator attached to this context");
  if (G.N < 2) raise(12, "sharded decomposition: the tensor order must be at least 2");
  const int world = comm_->world(), rank = comm_->rank();
  const ShardRange r = shard_range(G.d[G.N - 1], rank, world);
  if (r.begin != begin || r.len != len)
    raise(2, "sharded decomposition: rank " + std::to_string(rank) + " holds slab [" + std::to_string(begin) +
                 ", " + std::to_string(begin + len) + ") of mode " + std::to_string(G.N) + ", expected [" +
                 std::to_string(r.begin) + ", " + std::to_string(r.begin + r.len) + ")");
  for (int k = 0; k < G.N; ++k)
    if (G.d[k] < uint64_t(world))
      raise(12, "sharded decomposition: every extent must be at least the number of ranks (" +
                    std::to_string(world) + ")");
}

// core (full, replicated) and residual for a tensor sharded along its last
// mode: the TTM chain over the local slab with U_N's slab rows, summed.
void Engine::dist_core_and_residual(const double* A, const Shape& L, uint64_t k0, const Shape& G,
                                    const std::vector<uint64_t>& ranks, std::vector<double*>& U,
                                    double* core_buf, bool compute_core, std::vector<AlsOut>& outs,
                                    DecompRep* rep, double* core_host, double* factors_host, Clock::time_point t0) {
  const int N = G.N;
  const uint64_t nloc = L.d[N - 1];
  const uint32_t rN = uint32_t(ranks[N - 1]);
  double* uslab = uslab_.d(nloc * rN);
  CK(cudaMemcpy2DAsync(uslab, nloc * sizeof(double), U[N - 1] + k0, G.d[N - 1] * sizeof(double),
                       nloc * sizeof(double), rN, cudaMemcpyDeviceToDevice, st_));
  std::vector<double*> Us = U;
  Us[N - 1] = uslab;
  Shape cs;
  cs.N = N;
  for (int k = 0; k < N; ++k) cs.d[k] = ranks[k];
  if (compute_core) {
    core_chain(A, L, ranks, Us, core_buf);
    comm_->allreduce_sum(core_buf, cs.count(), st_);
  }
  sync();
  rep->seconds = since(t0);
  for (size_t k = 0; k < outs.size(); ++k) {
    rep->per_mode.emplace_back();
    collect(outs[k], rep->per_mode.back());
    rep->per_mode.back().seconds = mode_seconds(int(k));
  }
  rep->launches = launches_;
  rep->passes = passes_;
  rep->bytes = bytes_;
  const auto td = Clock::now();
  std::vector<ResultCopy> res;
  res.push_back({core_host, core_buf, cs.count() * sizeof(double)});
  size_t ofs = 0;
  for (int n = 0; n < N; ++n) {
    res.push_back({factors_host + ofs, U[n], G.d[n] * ranks[n] * sizeof(double)});
    ofs += G.d[n] * ranks[n];
  }
  copy_results(res, st_);
  rep->d2h_seconds = since(td);
  const auto tr = Clock::now();
  double rel_cf = 0.0;  // the core and ||A||^2 are replicated: every rank decides alike
  rep->relative_residual = closed_form_residual(core_buf, cs.count(), outs[0].sumsq_host, &rel_cf)
                               ? rel_cf
                               : relative_residual_dev(A, L, ranks, core_buf, Us, outs[0].sumsq_host);
  rep->residual_seconds = since(tr);
}

void Engine::t_hosvd_sharded(const double* a, bool a_dev, const Shape& G, uint64_t k0, uint64_t nloc,
                             const std::vector<uint64_t>& ranks, const AlsCfg& cfg, double* core, double* factors,
                             DecompRep* rep, bool want_sv) {
  validate_truncation(G, ranks);
  check_shard(G, k0, nloc);
  const int N = G.N, world = comm_->world(), rank = comm_->rank();
  Shape L = G;
  L.d[N - 1] = nloc;
  *rep = DecompRep();
  const double* A = upload(a, L.count(), a_dev, tensor_, &rep->h2d_seconds);
  while (factor_bufs_.size() < size_t(N)) factor_bufs_.push_back(new DBuf());
  std::vector<double*> U(N);
  dist_ = comm_.get();
  struct Reset {
    Comm*& d;
    ~Reset() { d = nullptr; }
  } reset{dist_};
  begin_timed();
  const auto t0 = Clock::now();
  // mode N runs on the tensor moved to shards along mode N-1
  const ShardRange bN = shard_range(G.d[N - 2], rank, world);
  Shape LB = G;
  LB.d[N - 2] = bN.len;
  auto window = [&](int n) {
    return n < N ? fiber_window(G, n, N, k0, nloc) : fiber_window(G, N, N - 1, bN.begin, bN.len);
  };
  {
    std::vector<PreGen> items;
    for (int n = 2; n <= N; ++n) {
      const Shape& Ln = n < N ? L : LB;
      items.push_back({n, Ln.count() / Ln.d[n - 1], uint32_t(ranks[n - 1]), window(n)});
    }
    defer_pregenerate(items, cfg.seed);
  }
  stage_reserve(N, cfg.max_iters);
  // Mode N's input (the tensor moved to shards along mode N-1) depends only
  // on A: the all-to-all runs on a second communicator and stream while
  // modes 1..N-1 sweep (NCCL; host-synchronous groups reshard in line).
  double* B = nullptr;
  bool overlapped = false;
  if (world > 1) {
    B = work_a_.d(LB.count());
    if (!comm2_tried_) {  // TKG_NO_SPLIT=1: reshard in line (no second communicator)
      const char* e = std::getenv("TKG_NO_SPLIT");
      if (!(e && e[0] == '1')) comm2_ = comm_->split();
      comm2_tried_ = true;
    }
    if (comm2_) {
      if (!cm_st_) {
        CK(cudaStreamCreateWithFlags(&cm_st_, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&cm_ev_a_, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&cm_ev_b_, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(cm_ev_a_, st_));
      CK(cudaStreamWaitEvent(cm_st_, cm_ev_a_, 0));
      reshard_on(A, G, N, N - 1, B, cm_st_, comm2_.get());
      CK(cudaEventRecord(cm_ev_b_, cm_st_));
      overlapped = true;
    }
  }
  bool sumsq_known = false;
  std::vector<AlsOut> outs;
  for (int n = 1; n <= N; ++n) {
    mode_begin(n - 1);
    const uint32_t r = uint32_t(ranks[n - 1]);
    const uint64_t I = G.d[n - 1];
    const double* An = A;
    const Shape* Ln = &L;
    if (n == N) {
      if (world > 1) {
        if (overlapped) CK(cudaStreamWaitEvent(st_, cm_ev_b_, 0));
        else reshard(A, G, N, N - 1, B);
        An = B;
      }
      Ln = &LB;
    }
    outs.push_back(run_als(An, *Ln, n, r, cfg, sumsq_known, window(n), n - 1));
    sumsq_known = true;
    U[n - 1] = factor_bufs_[n - 1]->d(I * r);
    qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[n - 1], n == N ? rhat_.d(r * r) : nullptr, nullptr, 0, false);
    // singular vectors: the Gram of this rank's fibers of A_(n)^T q is summed
    // over ranks, so every rank forms the same V (see Engine::t_hosvd)
    if (want_sv) recover_sv(An, *Ln, n, r, U[n - 1], n == N ? rhat_.d(r * r) : sv_vt_.d(r * r));
    mode_end(n - 1);
  }
  Shape cs;
  cs.N = N;
  for (int k = 0; k < N; ++k) cs.d[k] = ranks[k];
  double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
  // core: A x_N U_N^T = tensorize(R_hat R^T) of the final pair (see
  // Engine::t_hosvd), here on this rank's fibers of mode N (the tensor is
  // sharded along mode N-1 at that point), then the TTMs of modes 1..N-1 with
  // U_{N-1}'s rows of this shard, summed over ranks
  {
    const uint32_t rN = uint32_t(ranks[N - 1]), ncpN = pad_nc(rN);
    const uint64_t FN = LB.count() / LB.d[N - 1];
    Shape T = LB;
    T.d[N - 1] = rN;
    double* Tbuf = core_t_.d(T.count());
    const int nsh = shrink_count(FN);
    double* sq = sq_part_.d(size_t(std::max(4096, nsh)));
    CK(launch_shrink(r_.d(FN * ncpN + 8), ncpN, LB.stride(N), 1, rN, rhat_.d(rN * rN), Tbuf, sq, st_));
    count_launch();
    const uint32_t rM = uint32_t(ranks[N - 2]);
    double* uM = uslab2_.d(bN.len * rM);
    CK(cudaMemcpy2DAsync(uM, bN.len * sizeof(double), U[N - 2] + bN.begin, G.d[N - 2] * sizeof(double),
                         bN.len * sizeof(double), rM, cudaMemcpyDeviceToDevice, st_));
    std::vector<double*> Us = U;
    Us[N - 2] = uM;
    core_chain(Tbuf, T, ranks, Us, core_buf, N - 1);
    comm_->allreduce_sum(core_buf, cs.count(), st_);
  }
  dist_core_and_residual(A, L, k0, G, ranks, U, core_buf, false, outs, rep, core, factors, t0);
}

void Engine::st_hosvd_sharded(const double* a, bool a_dev, const Shape& G, uint64_t k0, uint64_t nloc,
                              const std::vector<uint64_t>& ranks, const std::vector<int>* order_in,
                              const AlsCfg& cfg, double* core, double* factors, DecompRep* rep) {
  validate_truncation(G, ranks);
  check_shard(G, k0, nloc);
  const std::vector<int> order = checked_order(G, ranks, order_in);
  const int N = G.N, world = comm_->world(), rank = comm_->rank();
  Shape L = G;
  L.d[N - 1] = nloc;
  *rep = DecompRep();
  const double* A = upload(a, L.count(), a_dev, tensor_, &rep->h2d_seconds);
  while (factor_bufs_.size() < size_t(N)) factor_bufs_.push_back(new DBuf());
  std::vector<double*> U(N);
  dist_ = comm_.get();
  struct Reset {
    Comm*& d;
    ~Reset() { d = nullptr; }
  } reset{dist_};
  begin_timed();
  const auto t0 = Clock::now();

  // Plan the shard layout along the processing order: a mode is processed
  // with its fibers local, so when it is the sharded one the tensor first
  // moves to the slowest other mode whose extent still covers every rank.
  struct Step {
    int mode, sm;       // processed mode; sharded mode while processing it
    bool move;          // reshard before processing (from the previous sm)
    int from;
    Shape Gw;           // global shape while processing
  };
  std::vector<Step> plan;
  {
    Shape Gw = G;
    int sm = N;
    for (int m : order) {
      Step st{m, sm, false, sm, Gw};
      if (m == sm) {
        int nsm = 0;
        for (int k = N; k >= 1 && !nsm; --k)
          if (k != m && Gw.d[k - 1] >= uint64_t(world)) nsm = k;
        if (!nsm) raise(12, "sharded st_hosvd: no mode left to shard the tensor along");
        st.move = true;
        st.sm = nsm;
        sm = nsm;
      }
      plan.push_back(st);
      Gw.d[m - 1] = ranks[m - 1];
    }
  }
  auto window = [&](const Step& st) {
    const ShardRange rr = shard_range(st.Gw.d[st.sm - 1], rank, world);
    return fiber_window(st.Gw, st.mode, st.sm, rr.begin, rr.len);
  };
  auto local_shape = [&](const Shape& Gw, int sm) {
    Shape Lw = Gw;
    Lw.d[sm - 1] = shard_range(Gw.d[sm - 1], rank, world).len;
    return Lw;
  };
  {
    std::vector<PreGen> items;
    for (size_t k = 1; k < plan.size(); ++k) {
      const Shape Lw = local_shape(plan[k].Gw, plan[k].sm);
      items.push_back({plan[k].mode, Lw.count() / Lw.d[plan[k].mode - 1], uint32_t(ranks[plan[k].mode - 1]),
                       window(plan[k])});
    }
    defer_pregenerate(items, cfg.seed);
  }
  const double* work = A;
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  bool sumsq_known = false;
  int sm = N;
  Shape Gw = G;
  stage_reserve(N, cfg.max_iters);
  std::vector<AlsOut> outs;
  for (const Step& st : plan) {
    const int k = int(outs.size());
    mode_begin(k);
    const int mode = st.mode;
    if (st.move) {
      const Shape Lnew = local_shape(Gw, st.sm);
      double* dst = reshard_.d(Lnew.count());
      if (world > 1) {
        reshard(work, Gw, st.from, st.sm, dst);
        work = dst;
      }
      sm = st.sm;
    }
    const Shape Lw = local_shape(Gw, sm);
    const uint32_t r = uint32_t(ranks[mode - 1]);
    const uint64_t I = Gw.d[mode - 1], s = Lw.stride(mode), F = Lw.count() / I, P = F / s;
    outs.push_back(run_als(work, Lw, mode, r, cfg, sumsq_known, window(st), k));
    const uint32_t ncp = pad_nc(r);
    U[mode - 1] = factor_bufs_[mode - 1]->d(I * r);
    double* RhT = rhatT_.d(size_t(r) * ncp);
    qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[mode - 1], rhat_.d(r * r), RhT, ncp, false);
    // local shrink (hosvd.cpp:176-178) of this rank's fibers, ||.||^2 summed
    Shape nxt = Lw;
    nxt.d[mode - 1] = r;
    double* dst = bufs[which]->d(nxt.count());
    const int nsh = shrink_count(F);
    double* sq = sq_part_.d(size_t(std::max(4096, nsh)));
    CK(launch_shrink(r_.d(F * ncp + 8), ncp, s, P, r, rhat_.d(r * r), dst, sq, st_, true));  // R_hat: qr_dev's upper factor
    CK(launch_sum(sq, nsh, sumsq_d_.d(2), st_));
    count_launch(2);
    comm_->allreduce_sum(sumsq_d_.d(2), 1, st_);
    sumsq_known = true;
    mode_end(k);
    work = dst;
    Gw.d[mode - 1] = r;
    which ^= 1;
  }
  // core: scatter this rank's block of the final (fully truncated) tensor
  // into the full core and sum over ranks
  Shape cs = Gw;
  double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
  CK(cudaMemsetAsync(core_buf, 0, cs.count() * sizeof(double), st_));
  {
    const Shape Lw = local_shape(Gw, sm);
    uint64_t ls[64], gs[64];
    strides_of(Lw, ls);
    strides_of(cs, gs);
    BoxCopy b;
    b.N = N;
    for (int k = 0; k < N; ++k) {
      b.box[k] = Lw.d[k];
      b.src_stride[k] = ls[k];
      b.dst_stride[k] = gs[k];
    }
    b.dst_base = shard_range(Gw.d[sm - 1], rank, world).begin * gs[sm - 1];
    CK(launch_copy_box(work, core_buf, b, st_));
    count_launch();
  }
  comm_->allreduce_sum(core_buf, cs.count(), st_);
  dist_core_and_residual(A, L, k0, G, ranks, U, core_buf, false, outs, rep, core, factors, t0);
}

}  // namespace tkg
