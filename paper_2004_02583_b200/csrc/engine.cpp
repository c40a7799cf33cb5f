// Host orchestration of the B200 ALS-HOSVD hot path (see engine.hpp).
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <thread>
#include <cstring>
#include <sstream>

#include "als_step.cuh"
#include "coop.cuh"
#include "contract_tma.cuh"
#include "mt_jump.hpp"
#include "sweep_fused.cuh"

namespace tkg {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// TKG_TRACE=1: host timestamps (us) of the orchestration points on stderr.
const bool g_trace = std::getenv("TKG_TRACE") != nullptr;
Clock::time_point g_trace_t0;
void trace(const char* what, int a = -1) {
  if (!g_trace) return;
  std::fprintf(stderr, "[tkg] %9.1f us  %s %d\n",
               std::chrono::duration<double, std::micro>(Clock::now() - g_trace_t0).count(), what, a);
}

int category_of(int subtype) {
  switch (subtype) {
    case 1: case 2: case 3: case 12: return 1;  // usage
    case 8: case 9: case 11: return 2;          // io / runtime
    default: return 3;                          // numerical
  }
}

constexpr uint32_t kMaxRank = 64;
constexpr int kMtSeqPadded = kPolyWords * 64 + kMtN;  // jump kernel reads this far

}  // namespace

[[noreturn]] void raise(int subtype, const std::string& msg) { throw Error(category_of(subtype), subtype, msg); }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(11, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// ---- Shape (shape.cpp:11-45) -------------------------------------------------
uint64_t Shape::count() const {
  uint64_t c = 1;
  for (int k = 0; k < N; ++k) c *= d[k];
  return c;
}
uint64_t Shape::extent(int mode) const {
  if (mode < 1 || mode > N)
    raise(1, "mode " + std::to_string(mode) + " out of range 1.." + std::to_string(N));
  return d[mode - 1];
}
uint64_t Shape::stride(int mode) const {
  extent(mode);
  uint64_t s = 1;
  for (int m = 0; m + 1 < mode; ++m) s *= d[m];
  return s;
}
std::string Shape::str() const {
  std::ostringstream o;
  for (int k = 0; k < N; ++k) o << (k ? "x" : "") << d[k];
  return o.str();
}

void validate_truncation(const Shape& sh, const std::vector<uint64_t>& ranks) {  // shape.cpp:56-69
  if (ranks.size() != size_t(sh.N))
    raise(2, "truncation lists " + std::to_string(ranks.size()) + " ranks for an order-" +
                 std::to_string(sh.N) + " tensor");
  for (int n = 0; n < sh.N; ++n)
    if (ranks[n] < 1 || ranks[n] > sh.d[n])
      raise(4, "mode " + std::to_string(n + 1) + ": rank " + std::to_string(ranks[n]) +
                   " outside 1.." + std::to_string(sh.d[n]));
}

std::vector<int> select_order(const std::vector<uint64_t>& ranks) {  // hosvd.cpp:54-63
  std::vector<int> order(ranks.size());
  for (size_t k = 0; k < ranks.size(); ++k) order[k] = int(k) + 1;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return ranks[a - 1] < ranks[b - 1]; });
  return order;
}

// ---- DBuf ------------------------------------------------------------------------
DBuf::~DBuf() { release(); }
void DBuf::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  bytes_ = 0;
}
void* DBuf::ensure(size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (bytes > bytes_) {
    release();
    CK(cudaMalloc(&p_, bytes));
    bytes_ = bytes;
  }
  return p_;
}

// ---- Engine ----------------------------------------------------------------------
Engine::Engine(int device) : device_(device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    raise(11, "no CUDA device available: the B200 path has no CPU fallback");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  name_ = prop.name;
  if (prop.major < 10) raise(12, std::string("tenkit_b200 is built for sm_100a; device is ") + prop.name);
  sms_ = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&st2_, cudaStreamNonBlocking, lo));  // lowest priority
    CK(cudaEventCreateWithFlags(&pre_gate_, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&cp_st_, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&out_ready_, cudaEventDisableTiming));
  }
  CK(cudaHostAlloc(reinterpret_cast<void**>(&status_h_), sizeof(DevStatus), cudaHostAllocMapped));
  std::memset(status_h_, 0, sizeof(DevStatus));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&status_d_), status_h_, 0));
}

Engine::~Engine() {
  if (profiling_) pdl_off_count() -= 1;
  cudaSetDevice(device_);
  cudaStreamSynchronize(st_);
  for (auto* b : factor_bufs_) delete b;
  for (auto& kv : jump_cache_) delete kv.second;
  for (auto& kv : yseq_cache_) delete kv.second;
  for (auto& r : recs_) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto e : mode_ev_) cudaEventDestroy(e);
  if (sumsq_ev_) cudaEventDestroy(sumsq_ev_);
  for (Lane* L : lanes_) {
    cudaStreamSynchronize(L->st);
    cudaStreamDestroy(L->st);
    cudaEventDestroy(L->done);
    delete L;
  }
  if (stage_h_) cudaFreeHost(stage_h_);
  if (stage_ctrl_) cudaFreeHost(stage_ctrl_);
  if (out_stage_) cudaFreeHost(out_stage_);
  clear_graphs();
  if (cm_st_) {
    cudaStreamSynchronize(cm_st_);
    cudaStreamDestroy(cm_st_);
    cudaEventDestroy(cm_ev_a_);
    cudaEventDestroy(cm_ev_b_);
  }
  if (norm_h_) cudaFreeHost(norm_h_);
  if (t0_) cudaEventDestroy(t0_);
  if (t1_) cudaEventDestroy(t1_);
  cudaStreamSynchronize(st2_);
  for (auto* b : pre_bufs_) delete b;
  for (auto* b : pre_y_) delete b;
  for (auto* b : pre_st_) delete b;
  for (auto* b : pre_ids_) delete b;
  for (auto ev : pre_ev_) cudaEventDestroy(ev);
  cudaEventDestroy(pre_gate_);
  if (status_h_) cudaFreeHost(status_h_);
  cudaStreamSynchronize(cp_st_);
  cudaEventDestroy(out_ready_);
  cudaStreamDestroy(cp_st_);
  cudaStreamDestroy(st2_);
  cudaStreamDestroy(st_);
}

void Engine::sync() { CK(cudaStreamSynchronize(st_)); }

void Engine::timer_start() {
  if (!t0_) {
    CK(cudaEventCreate(&t0_));
    CK(cudaEventCreate(&t1_));
  }
  CK(cudaEventRecord(t0_, st_));
}

double Engine::timer_stop() {
  CK(cudaEventRecord(t1_, st_));
  CK(cudaEventSynchronize(t1_));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, t0_, t1_));
  return ms;
}

void Engine::flush_l2() {
  const size_t bytes = size_t(512) << 20;  // 4x the 126 MB L2
  CK(cudaMemsetAsync(flush_.ensure(bytes), 0, bytes, st_));
}

std::pair<cudaEvent_t, cudaEvent_t> Engine::ev_pair() {
  cudaEvent_t a, b;
  if (ev_pool_.size() >= 2) {
    a = ev_pool_.back();
    ev_pool_.pop_back();
    b = ev_pool_.back();
    ev_pool_.pop_back();
  } else {
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
  }
  return {a, b};
}

std::pair<cudaEvent_t, cudaEvent_t> Engine::small_begin() {
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (profiling_) {
    ev = ev_pair();
    CK(cudaEventRecord(ev.first, st_));
  }
  return ev;
}

void Engine::small_end(std::pair<cudaEvent_t, cudaEvent_t> ev) {
  if (!profiling_) return;
  CK(cudaEventRecord(ev.second, st_));
  record(kClsSmall, ev.first, ev.second, 0.0, 0.0);
}

void Engine::record(int cls, cudaEvent_t a, cudaEvent_t b, double bytes, double flops) {
  recs_.push_back({cls, a, b, bytes, flops});
}

void Engine::kernel_stats(double ms[kNumCls], uint64_t launches[kNumCls], double bytes[kNumCls],
                          double flops[kNumCls]) {
  sync();
  for (auto& r : recs_) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ev_pool_.push_back(r.a);
    ev_pool_.push_back(r.b);
    if (r.cls < 0) continue;  // speculative launch that returned on entry
    stat_ms_[r.cls] += t;
    stat_launch_[r.cls] += 1;
    stat_bytes_[r.cls] += r.bytes;
    stat_flops_[r.cls] += r.flops;
  }
  recs_.clear();
  for (int k = 0; k < kNumCls; ++k) {
    ms[k] = stat_ms_[k];
    launches[k] = stat_launch_[k];
    bytes[k] = stat_bytes_[k];
    flops[k] = stat_flops_[k];
    stat_ms_[k] = 0;
    stat_launch_[k] = 0;
    stat_bytes_[k] = 0;
    stat_flops_[k] = 0;
  }
}

const double* Engine::upload(const double* a, uint64_t n, bool a_dev, DBuf& buf, double* seconds) {
  if (a_dev) return a;
  const auto t0 = Clock::now();
  double* d = buf.d(n);
  CK(cudaMemcpyAsync(d, a, n * sizeof(double), cudaMemcpyHostToDevice, st_));
  sync();
  if (seconds) *seconds += since(t0);
  return d;
}

void Engine::fc(const FiberView& v, const double* mt, uint32_t ldmt, uint32_t nc, double* out,
                uint64_t os_j, uint64_t os_c, uint64_t os_p, double* sumsq_part,
                const double* diff_ref, int* grid_used, bool count_pass, const int32_t* skip,
                double* gram_part) {
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (profiling_) {
    ev = ev_pair();
    CK(cudaEventRecord(ev.first, st_));
  }
  const int mode = force_v1_ ? -1 : fc_tma_mode(v, mt, ldmt);
  if (mode >= 0) {
    FcTmaArgs a;
    a.nc = nc;
    a.out = out;
    a.os_j = os_j;
    a.os_c = os_c;
    a.os_p = os_p;
    a.sumsq_part = sumsq_part;
    a.diff_ref = diff_ref;
    a.skip = skip;
    a.gram_part = gram_part;
    CK(launch_fc_tma(v, mt, ldmt, a, mode, sms_, st_, grid_used));
  } else {
    FcArgs a;
    a.in = v;
    a.mt = mt;
    a.ldmt = ldmt;
    a.out = out;
    a.os_j = os_j;
    a.os_c = os_c;
    a.os_p = os_p;
    a.nc = nc;
    a.gram_part = gram_part;
    a.sumsq_part = sumsq_part;
    a.diff_ref = diff_ref;
    a.skip = skip;
    CK(launch_fc(a, sms_, st_, grid_used));
  }
  count_launch();
  const double elems = double(v.s) * double(v.P) * double(v.K);
  const double F = double(v.s) * double(v.P);
  const double bytes = 8.0 * (elems + F * nc + double(v.K) * nc);
  if (profiling_) {
    CK(cudaEventRecord(ev.second, st_));
    record(fc_cls_, ev.first, ev.second, bytes, 2.0 * elems * nc);
  }
  if (count_pass) {
    passes_ += 1;
    bytes_ += uint64_t(bytes);
  }
}

bool Engine::sweep_fused_usable(const FiberView& v, const double* mt, uint32_t nc, const double* R) const {
  return fused_sweep_ && !force_v1_ && !dist_ && sweep_fused_ok(v, mt, nc, R);
}

int Engine::sweep_fused(const FiberView& v, const double* mt, uint32_t nc, double* R, double* partial,
                        double* gram_part, bool count_pass, const int32_t* skip) {
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (profiling_) {
    ev = ev_pair();
    CK(cudaEventRecord(ev.first, st_));
  }
  SweepFusedArgs a;
  a.mt = mt;
  a.nc = nc;
  a.R = R;
  a.partial = partial;
  a.gram_part = gram_part;
  a.skip = skip;
  int grid = 0;
  CK(launch_sweep_fused(v, a, sms_, st_, &grid));
  count_launch();
  const double elems = double(v.s) * double(v.P) * double(v.K);
  const double F = double(v.s) * double(v.P);
  // the pass reads A and L' and writes R and the K x r sum: one tensor pass
  const double bytes = 8.0 * (elems + F * nc + 2.0 * double(v.K) * nc);
  if (profiling_) {
    CK(cudaEventRecord(ev.second, st_));
    record(kClsSweep, ev.first, ev.second, bytes, 4.0 * elems * nc);
  }
  if (count_pass) {
    passes_ += 1;
    bytes_ += uint64_t(bytes);
  }
  return grid;
}

int Engine::fc_grid(const FiberView& v, const double* mt, uint32_t ldmt, uint32_t nc) {
  const int mode = force_v1_ ? -1 : fc_tma_mode(v, mt, ldmt);
  return mode >= 0 ? fc_tma_grid(v, sms_) : fc_grid_for(v, nc, sms_);
}

uint32_t Engine::fr_ranges(const FiberView& v, uint32_t nc) {
  return std::max(fr_ranges_for(v, nc, sms_), fr_tma_ranges(v, sms_)) + 4;
}

uint32_t Engine::fr(const FiberView& v, const double* m, uint64_t mj, uint64_t mc, uint32_t nc,
                    double* partial, double* sumsq_part, bool count_pass, uint32_t* grid_used,
                    const int32_t* skip) {
  // M(j, c) = m[j*mj + c*mc]
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (profiling_) {
    ev = ev_pair();
    CK(cudaEventRecord(ev.first, st_));
  }
  uint32_t ranges = 0, grid = 0;
  const int mode = force_v1_ ? -1 : fr_tma_mode(v, m, mj, mc);
  if (mode >= 0) {
    FrTmaArgs a;
    a.nc = nc;
    a.partial = partial;
    a.sumsq_part = sumsq_part;
    a.skip = skip;
    CK(launch_fr_tma(v, m, mj, mc, a, mode, sms_, st_, &ranges, &grid));
  } else {
    FrArgs a;
    a.in = v;
    a.m = m;
    a.mj = mj;
    a.mc = mc;
    a.nc = nc;
    a.partial = partial;
    a.sumsq_part = sumsq_part;
    a.skip = skip;
    CK(launch_fr(a, sms_, st_, &ranges, &grid));
  }
  if (grid_used) *grid_used = grid;
  count_launch();
  const double elems = double(v.s) * double(v.P) * double(v.K);
  const double F = double(v.s) * double(v.P);
  const double bytes = 8.0 * (elems + F * nc + double(v.K) * nc);
  if (profiling_) {
    CK(cudaEventRecord(ev.second, st_));
    record(kClsFR, ev.first, ev.second, bytes, 2.0 * elems * nc);
  }
  if (count_pass) {
    passes_ += 1;
    bytes_ += uint64_t(bytes);
  }
  return ranges;
}

// S = uniform01 draws 0..n-1 of seeded_engine(seed, stream), on device,
// enqueued on `st` with its own sequence/state buffers. With a shard window
// only the draws of the shard's fibers are kept (see MtWindow), and when
// those form one position range per column only the chunks that meet them
// are jumped to and generated.
void Engine::gen_uniform_on(uint64_t seed, uint32_t stream, uint64_t n, double* d_out, const MtWindow& win,
                            cudaStream_t st, DBuf& ybuf, DBuf& sbuf, DBuf& cbuf) {
  if (n == 0) return;
  if (mt_charpoly().empty()) raise(11, "MT19937-64 characteristic polynomial check failed");
  const MtPlan plan = mt_plan(n, st != st_);
  const auto key = std::make_pair(plan.J, plan.C);
  DBuf* polys = nullptr;
  auto it = jump_cache_.find(key);
  if (it == jump_cache_.end()) {
    std::vector<uint64_t> tbl = mt_jump_table(plan.J, plan.C);
    polys = new DBuf();
    uint64_t* d = polys->u(tbl.size());
    CK(cudaMemcpyAsync(d, tbl.data(), tbl.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    jump_cache_[key] = polys;
  } else {
    polys = it->second;
  }
  // the engine's first 20 248 raw words depend only on (seed, stream): kept
  // on the device per key, so a repeated decomposition does no host-side
  // recurrence and no upload (bounded cache)
  (void)ybuf;
  uint64_t* d_y = nullptr;
  {
    const auto ykey = std::make_pair(seed, stream);
    auto yit = yseq_cache_.find(ykey);
    if (yit == yseq_cache_.end()) {
      if (yseq_cache_.size() >= 256) {
        CK(cudaDeviceSynchronize());  // no pending kernel reads an evicted sequence
        for (auto& kv : yseq_cache_) delete kv.second;
        yseq_cache_.clear();
      }
      std::vector<uint64_t> y(kMtSeqPadded, 0);
      mt_raw_sequence(seed, stream, y.data(), kMtSeqWords);
      DBuf* b = new DBuf();
      d_y = b->u(kMtSeqPadded);
      // pageable source: the copy is staged before cudaMemcpyAsync returns
      CK(cudaMemcpyAsync(d_y, y.data(), y.size() * 8, cudaMemcpyHostToDevice, st));
      yseq_cache_[ykey] = b;
    } else {
      d_y = yit->second->u(kMtSeqPadded);
    }
  }
  int nchunks = plan.C;
  const int* d_ids = nullptr;
  if (win.nloc > 0 && win.Gsm > 1 && win.Fg == win.Plo * win.Gsm) {
    const uint64_t a0 = win.o0 * win.Plo, a1 = (win.o0 + win.nloc) * win.Plo;
    const uint64_t ncol = n / win.Fg;
    std::vector<int> ids;
    for (int c = 0; c < plan.C; ++c) {
      const uint64_t p0 = uint64_t(c) * plan.J, p1 = std::min(n, p0 + plan.J);
      bool hit = false;
      for (uint64_t col = p0 / win.Fg; col <= (p1 - 1) / win.Fg && col < ncol && !hit; ++col)
        hit = std::max(p0, col * win.Fg + a0) < std::min(p1, col * win.Fg + a1);
      if (hit) ids.push_back(c);
    }
    nchunks = int(ids.size());
    if (nchunks == 0) return;
    int* d = static_cast<int*>(cbuf.ensure(ids.size() * sizeof(int)));
    CK(cudaMemcpyAsync(d, ids.data(), ids.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    d_ids = d;
  }
  uint64_t* d_states = sbuf.u(size_t(nchunks) * kMtN);
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  const bool prof = profiling_ && st == st_;
  if (prof) {
    ev = ev_pair();
    CK(cudaEventRecord(ev.first, st));
  }
  CK(launch_mt_states(d_y, polys->u(0) /*existing*/, nchunks, d_ids, d_states, st));
  CK(launch_mt_generate(d_states, nchunks, d_ids, plan.J, n, d_out, win, st));
  count_launch(3);  // memset + jump + generate
  if (prof) {
    CK(cudaEventRecord(ev.second, st));
    record(kClsRng, ev.first, ev.second, 8.0 * n, 0.0);
  }
}

// The initializer S of a mode (F local fibers), column-major F x r: the
// whole stream in storage order, or a shard's window of it. (A row-major
// [F][ld] S would need scattered 8-byte writes from the generator; the FR
// kernel reads the column-major operand at the same speed.)
MtWindow Engine::s_window(MtWindow win, uint64_t F, uint64_t ld) {
  (void)F;
  if (win.nloc == 0) return win;
  win.ld = ld;
  return mt_window_finish(win);
}

void Engine::gen_uniform(uint64_t seed, uint32_t stream, uint64_t n, double* d_out, const MtWindow& win) {
  gen_uniform_on(seed, stream, n, d_out, win, st_, y_seq_, states_, chunk_ids_);
}

// The initializer streams depend only on (seed, mode, fibers, rank), not on
// the data: generate those of every mode after the first on a second stream
// while the first modes' sweeps run (the RNG kernels fit beside the
// contraction kernels' shared-memory footprint).
void Engine::defer_pregenerate(const std::vector<PreGen>& items, uint64_t seed) {
  pre_.clear();
  pending_pre_ = items;
  pending_seed_ = seed;
}

void Engine::pregenerate(const std::vector<PreGen>& items, uint64_t seed) {
  pre_.clear();
  while (pre_bufs_.size() < items.size()) {
    pre_bufs_.push_back(new DBuf());
    pre_y_.push_back(new DBuf());
    pre_st_.push_back(new DBuf());
    pre_ids_.push_back(new DBuf());
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    pre_ev_.push_back(ev);
  }
  CK(cudaEventRecord(pre_gate_, st_));  // buffers of a previous call are free
  CK(cudaStreamWaitEvent(st2_, pre_gate_, 0));
  for (size_t k = 0; k < items.size(); ++k) {
    const PreGen& g = items[k];
    double* d = pre_bufs_[k]->d(g.F * g.r + 8);
    const uint64_t total = (g.win.nloc ? g.win.Fg : g.F) * g.r;
    gen_uniform_on(seed, uint32_t(g.mode), total, d, s_window(g.win, g.F, 0), st2_, *pre_y_[k], *pre_st_[k],
                   *pre_ids_[k]);
    CK(cudaEventRecord(pre_ev_[k], st2_));
    pre_[g.mode] = {d, pre_ev_[k], g.F, g.r};
  }
}

// Thin QR with a nonnegative R diagonal (reduced_qr, kernels.cpp:303-367) by
// CholQR2 on the device: Y = Q1 R1, Q1 = Q R2, R = R2 R1 — multi-CTA Gram
// partials, a one-CTA Cholesky and row-parallel triangular solves. The thin
// QR with positive diagonal is unique, so Q matches Householder's to rounding
// for the well-conditioned factors ALS produces.
void Engine::qr_dev(const double* Y, int nparts, uint64_t ld, uint32_t I, uint32_t r, double* Q,
                    double* rmat, double* rt, uint32_t ldrt, bool check) {
  if (r > kMaxRank) {  // column-major Y only (the wide ALS reduces its own partials)
    if (nparts != 0 || rt) raise(12, "qr_dev: wide ranks take a column-major Y");
    qr_wide(Y, I, r, Q, rmat, check);
    return;
  }
  CholQrArgs q;
  q.Y = const_cast<double*>(Y);  // written only when nparts > 1 (partials summed in place)
  q.nparts = nparts;
  q.ldp = ld;
  q.I = I;
  q.r = r;
  q.Q = Q;
  q.rmat = rmat;
  q.rt = rt;
  q.ldrt = ldrt;
  q.check = check ? 1 : 0;
  q.gpart = gram_part_.d(size_t(coop_partials_cap(sms_)) * r * r);
  q.gs = gs_.d(size_t(r) * r);
  q.L1 = qrl1_.d(size_t(r) * r);
  q.Rinv = qrl2_.d(size_t(r) * r);
  q.work = qrq1_.d(2);
  q.ctrl = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
  const auto ev = small_begin();
  coop_launch([&] { CK(launch_cholqr_step(q, sms_, st_)); });
  if (check) {
    // CholQR2 meets a rank-deficient Y as a failed Cholesky at a column set by
    // rounding noise; the reference decides on diag(R) of Householder QR
    // (kernels.cpp:303-367, als.cpp:74-86). When the fast path flags a
    // collapse, Householder QR of the same Y (the summed partials stay in
    // slot 0) recomputes Q, R and the collapse column, as the reference does;
    // otherwise this launch returns at once.
    AlsCtrl* c = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
    double* wk = qr_work_.d(2 * size_t(I) * r + r);
    CK(launch_qr(Y, nparts > 1 ? 1 : nparts, ld, I, r, Q, rmat, rt, ldrt, wk, 1, nullptr, st_,
                 &c->degenerate_col, &c->degenerate_col));
    count_launch();
  }
  small_end(ev);
  count_launch();
}

// Sharded runs: Y = sum of this shard's FR partials (into slot 0), summed
// over the shards; returns the new partial count (1).
uint32_t Engine::reduce_left_partials(double* part, uint32_t nparts, uint32_t I, uint32_t ncp, uint32_t r) {
  CK(launch_reduce_slot0(part, int(nparts), I, ncp, r, st_));
  count_launch();
  dist_->allreduce_sum(part, size_t(I) * ncp, st_);
  return 1;
}

int Engine::qr_degenerate_col() {
  AlsCtrl h;
  CK(cudaMemcpyAsync(&h, ctrl_d_.ensure(sizeof(AlsCtrl)), sizeof(AlsCtrl), cudaMemcpyDeviceToHost, st_));
  sync();
  return h.degenerate_col;
}

void Engine::stage_reserve(int modes, int max_iters) {
  const size_t n = size_t(std::max(1, modes)) * size_t(std::max(1, max_iters) + 1);
  if (n > stage_n_) {
    sync();  // no copy into the old buffer is pending
    if (stage_h_) cudaFreeHost(stage_h_);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&stage_h_), n * sizeof(double), cudaHostAllocDefault));
    stage_n_ = n;
  }
  stage_iters_ = std::max(1, max_iters);
  while (mode_ev_.size() < size_t(2 * std::max(1, modes))) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    mode_ev_.push_back(e);
  }
}

void Engine::collect(AlsOut& o, ModeRep& dst) {
  if (o.ctrl_host) settle(o);
  dst = o.rep;
  dst.history.assign(o.hist_host, o.hist_host + o.rep.iterations);
}

// A mode whose sweeps ran as a device-side loop: its report, error and work
// counters from the staged control block (after the final synchronisation).
void Engine::settle(AlsOut& o) {
  const AlsCtrl h = *o.ctrl_host;
  o.ctrl_host = nullptr;
  const std::string mname = "mode " + std::to_string(o.rep.mode);
  switch (h.error) {
    case kAlsErrZeroNorm: raise(3, "als_low_rank: input tensor has zero norm");
    case kAlsErrDegenerate:
      raise(6, "als_init: randomized range collapsed at column " + std::to_string(h.degenerate_col) +
                   " for mode " + std::to_string(o.rep.mode));
    case kAlsErrRightSingular:
    case kAlsErrLeftSingular:
      raise(4, mname + ": gram matrix is singular, rank " + std::to_string(o.r) +
                   " exceeds the numerical rank of the iterate");
    default: break;
  }
  o.rep.iterations = h.iter;
  o.rep.status = h.status;
  o.rep.achieved_eta = h.achieved;
  o.norm = h.norm;
  // FC of sweeps 1..iter, FR of sweeps 1..iter-1 (or iter when the cap ended it)
  const int fr_run = h.stop ? h.iter - 1 : h.iter;
  const int npass = o.fused ? h.iter : h.iter + fr_run;  // a fused sweep is one tensor pass
  passes_ += uint64_t(npass);
  bytes_ += uint64_t(double(npass) * o.fc_bytes);
  launches_ += uint64_t(std::max(1, h.iter)) * uint64_t(o.body_launches);
}

void Engine::mode_begin(int k) { CK(cudaEventRecord(mode_ev_[2 * k], st_)); }
void Engine::mode_end(int k) { CK(cudaEventRecord(mode_ev_[2 * k + 1], st_)); }
double Engine::mode_seconds(int k) {
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, mode_ev_[2 * k], mode_ev_[2 * k + 1]));
  return ms * 1e-3;
}

// Device-side sweep loops (CUDA graphs with a WHILE node): by default only
// for t-HOSVD, whose independent modes then run concurrently (one stream and
// buffer set each, Engine::t_hosvd); TKG_GRAPH=1 uses them for every driver,
// TKG_GRAPH=0 never. Never while profiling (per-launch events) or sharded
// (host-synchronous communicators). Measured: config 1
// 1.51 -> 1.29 ms per step with concurrent modes; for the st-HOSVD configs the
// device loop alone changes nothing measurable (the host already runs ahead
// of the device), so they keep the speculative host batches.
int graph_env() {
  static const int v = [] {
    const char* e = std::getenv("TKG_GRAPH");
    return e == nullptr ? -1 : (e[0] == '1' ? 1 : 0);
  }();
  return v;
}

bool Engine::use_graph_loop() const {
  if (profiling_ || dist_ || graph_failed_) return false;
  const int e = graph_env();
  return e == 1 || (e == -1 && in_lanes_);
}

// Captures `body(cond)` (the kernels of one sweep, enqueued on st_) as the
// body of a WHILE node whose condition starts at 1; returns the instantiated
// graph, or nullptr (and graph mode off for this engine) when the capture is
// not supported for these kernels.
cudaGraphExec_t Engine::capture_sweep_loop(const std::function<void(GraphCond)>& body, int* body_launches) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool capturing = false;
  const uint64_t l0 = launches_;
  try {
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t bg = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(st_, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    capturing = true;
    body(GraphCond(h));
    cudaGraph_t done = nullptr;
    capturing = false;
    CK(cudaStreamEndCapture(st_, &done));
    size_t n = 0;
    CK(cudaGraphGetNodes(bg, nullptr, &n));
    *body_launches = int(n);
    CK(cudaGraphInstantiate(&exec, g, 0));
  } catch (const std::exception& e) {
    trace("sweep graph capture failed; host loop");
    if (capturing) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(st_, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    exec = nullptr;
    graph_failed_ = true;
  }
  if (g) cudaGraphDestroy(g);
  launches_ = l0;  // the captured kernels are counted per executed sweep (settle)
  return exec;
}

void Engine::swap_lane(Lane& L) {
  std::swap(st_, L.st);
  s_.swap(L.s);
  r_.swap(L.r);
  l_.swap(L.l);
  mt_.swap(L.mt);
  gl_.swap(L.gl);
  gr_.swap(L.gr);
  cholL_.swap(L.cholL);
  cholR_.swap(L.cholR);
  fr_part_.swap(L.fr_part);
  fc_gram_.swap(L.fc_gram);
  gram_part_.swap(L.gram_part);
  gs_.swap(L.gs);
  sq_part_.swap(L.sq_part);
  qr_work_.swap(L.qr_work);
  y_seq_.swap(L.y_seq);
  states_.swap(L.states);
  chunk_ids_.swap(L.chunk_ids);
  qrl1_.swap(L.qrl1);
  qrl2_.swap(L.qrl2);
  qrq1_.swap(L.qrq1);
  sumsq_d_.swap(L.sumsq_d);
  ctrl_d_.swap(L.ctrl_d);
  hist_d_.swap(L.hist_d);
  misc2_.swap(L.misc2);
}

// Concurrent modes need the non-blocking (graph) sweep loop and the r <= 64
// path; singular vectors keep the sequential driver.
bool Engine::concurrent_modes_ok(const std::vector<uint64_t>& ranks, bool want_sv) const {
  if (want_sv || profiling_ || dist_ || graph_failed_ || graph_env() == 0) return false;
  for (uint64_t r : ranks)
    if (r > kMaxRank) return false;
  return true;
}

void Engine::clear_graphs() {
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.first);
  graphs_.clear();
}

Engine::AlsOut Engine::run_als(const double* A, const Shape& sh, int mode, uint32_t r,
                               const AlsCfg& cfg, bool sumsq_known, const MtWindow& win, int slot) {
  const uint64_t I = sh.extent(mode);
  const uint64_t s = sh.stride(mode);
  const uint64_t F = sh.count() / I;
  const uint64_t P = F / s;
  const uint32_t ncp = pad_nc(r);
  const std::string mname = "mode " + std::to_string(mode);
  // als.cpp:101-104 (zero norm) precedes als_init's rank guard (:62-66) and
  // the init shape check (:106-113)
  if ((cfg.init == nullptr && (r < 1 || r > I)) ||
      (cfg.init && (cfg.init_rows != I || cfg.init_cols != r))) {
    if (!sumsq_known) {
      double* sq0 = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(sh.count()))));
      CK(launch_sumsq(A, sh.count(), sq0, st_));
      CK(launch_sum(sq0, sumsq_partials_count(sh.count()), sumsq_d_.d(2), st_));
      count_launch(2);
      if (dist_) dist_->allreduce_sum(sumsq_d_.d(2), 1, st_);
    }
    double ss = 0.0;
    CK(cudaMemcpyAsync(&ss, sumsq_d_.d(2), sizeof(double), cudaMemcpyDeviceToHost, st_));
    sync();
    if (ss == 0.0) raise(3, "als_low_rank: input tensor has zero norm");
    if (cfg.init)
      raise(2, "als_low_rank: init is " + std::to_string(cfg.init_rows) + "x" + std::to_string(cfg.init_cols) +
                   ", mode " + std::to_string(mode) + " needs " + std::to_string(I) + "x" + std::to_string(r));
    raise(4, mname + ": rank " + std::to_string(r) + " outside 1.." + std::to_string(I));
  }
  if (r > kMaxRank) return run_als_wide(A, sh, mode, r, cfg, sumsq_known, slot);
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  AlsOut out;
  out.rep.mode = mode;

  double* Lc = l_.d(I * r);
  double* Mt = mt_.d(I * ncp);
  double* R = r_.d(F * ncp + 8);  // row-major [F][ncp]
  double* GL = gl_.d(kMaxRank * kMaxRank);
  double* GR = gr_.d(kMaxRank * kMaxRank);
  double* cholL = cholL_.d(kMaxRank * kMaxRank);
  double* cholR = cholR_.d(kMaxRank * kMaxRank);
  // r <= 16 (HBM-bound): one fused pass per sweep instead of FC + FR
  const bool fused = sweep_fused_usable(v, Mt, r, R);
  const uint32_t nranges = std::max(fr_ranges(v, r), fused ? uint32_t(sweep_fused_grid(v, r, sms_)) : 0u);
  double* part = fr_part_.d(size_t(nranges) * I * ncp);
  double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(sh.count()))));
  double* sumsq = sumsq_d_.d(2);
  AlsCtrl* ctrl = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
  const int max_iters = std::max(1, cfg.max_iters);
  double* hist = hist_d_.d(size_t(max_iters));
  const int32_t* stop = &ctrl->stop;

  // 1. ||A|| and the initial left factor (als.cpp:99-120).
  if (cfg.init) {
    if (!sumsq_known) {
      CK(launch_sumsq(A, sh.count(), sq, st_));
      CK(launch_sum(sq, sumsq_partials_count(sh.count()), sumsq, st_));
      count_launch(2);
      if (dist_) dist_->allreduce_sum(sumsq, 1, st_);
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
      double* Sg = s_.d(F * r + 8);  // column-major F x r, the reference's storage order
      trace("  gen_uniform", mode);
      gen_uniform(cfg.seed, uint32_t(mode), (win.nloc ? win.Fg : F) * r, Sg, s_window(win, F, 0));
      trace("  gen_uniform enqueued", mode);
      S = Sg;
    }
    uint32_t fr_grid = 0;
    uint32_t ranges = fr(v, S, 1, F, r, part, sumsq_known ? nullptr : sq, true, &fr_grid);
    if (!sumsq_known) {  // ||A||^2 fused into the init pass: one partial per CTA
      CK(launch_sum(sq, int(fr_grid), sumsq, st_));
      if (record_sumsq_) CK(cudaEventRecord(sumsq_ev_, st_));  // concurrent modes read it (t_hosvd)
      count_launch();
      if (dist_) dist_->allreduce_sum(sumsq, 1, st_);
    }
    if (dist_) ranges = reduce_left_partials(part, ranges, uint32_t(I), ncp, r);
    qr_dev(part, int(ranges), ncp, uint32_t(I), r, Lc, nullptr, nullptr, 0, true);
  }
  if (sumsq_from_) {  // a concurrent mode: ||A||^2 from the first mode's init pass
    CK(cudaStreamWaitEvent(st_, sumsq_ev_, 0));
    CK(cudaMemcpyAsync(sumsq, sumsq_from_, sizeof(double), cudaMemcpyDeviceToDevice, st_));
  }
  CK(launch_ctrl_init(ctrl, sumsq, cfg.eta, max_iters, max_iters, cfg.init ? 0 : 1, st_));
  count_launch();
  trace("init enqueued", mode);
  // the initializer streams of the later modes are prepared on the host and
  // queued on the side stream once this mode's first kernels are queued
  if (!pending_pre_.empty()) {
    std::vector<PreGen> items;
    items.swap(pending_pre_);
    pregenerate(items, pending_seed_);
  }

  // 2. Sweeps (als.cpp:121-160), enqueued in batches; kernels of sweeps past
  //    the stop decision return on entry.
  int enqueued = 0;
  int batch = 4;
  AlsCtrl h;
  spec_recs_.clear();
  double* GLinv = cholL;
  double* GRinv = cholR;
  double* gpl = gram_part_.d(size_t(coop_partials_cap(sms_)) * r * r);
  double* gs = gs_.d(size_t(r) * r);
  // Gram of R: fused into the FC epilogue up to ncp 32, else a row pass inside finish_step
  const bool fused_gram = ncp <= kFcGramMaxNc;
  const int nfin = std::max({finish_step_grid(F, sms_), fc_grid(v, Mt, ncp, r), fused ? sweep_fused_grid(v, r, sms_) : 0});
  double* gpr = fc_gram_.d(size_t(nfin) * ncp * ncp);
  uint32_t last_ranges = 0;
  auto prep_args = [&](int from_partials, int nparts) {
    PrepArgs pa;
    pa.part = part;
    pa.nparts = nparts;
    pa.ldp = ncp;
    pa.GRinv = GRinv;
    pa.from_partials = from_partials;
    pa.I = uint32_t(I);
    pa.r = r;
    pa.ncp = ncp;
    pa.Lc = Lc;
    pa.GL = GL;
    pa.GLinv = GLinv;
    pa.Mt = Mt;
    pa.gpart = gpl;
    pa.gs = gs;
    pa.ctrl = ctrl;
    return pa;
  };
  auto finish_args = [&](int gram_nparts, GraphCond cond) {
    FinishArgs fa;
    fa.R = R;
    fa.F = F;
    fa.ld = ncp;
    fa.r = r;
    fa.GL = GL;
    fa.GRinv = GRinv;
    fa.gpart = gpr;
    fa.gs = gs;
    fa.ctrl = ctrl;
    fa.history = hist;
    fa.gram_nparts = gram_nparts;
    fa.cond = cond;
    return fa;
  };
  cudaGraphExec_t loop = nullptr;
  int body_launches = 0;
  if (use_graph_loop()) {
    // 2'. Sweeps as a CUDA-graph WHILE loop on the device (no host round trip
    //     per batch): sweep 1's prep on the stream, then
    //       while (cond) { FC(k); finish(k) -> cond; FR(k); prep(k+1) }
    //     the finish step's stop rule ends the loop (kernels past it return on
    //     entry); the report is read after the driver's final synchronisation.
    //     Executable graphs are cached per operand set (bench / repeated calls).
    const std::vector<uint64_t> key = {uint64_t(v.base), v.s, v.P, v.K, v.is_i, v.is_p, r, ncp,
                                       uint64_t(Mt), uint64_t(R), uint64_t(gpr), uint64_t(part), uint64_t(Lc),
                                       uint64_t(GL), uint64_t(GLinv), uint64_t(GRinv), uint64_t(gs),
                                       uint64_t(gpl), uint64_t(ctrl), uint64_t(hist), uint64_t(sms_),
                                       uint64_t(fused)};
    auto it = graphs_.find(key);
    if (it != graphs_.end()) {
      loop = it->second.first;
      body_launches = it->second.second;
    } else {
      loop = capture_sweep_loop([&](GraphCond cond) {
        if (fused) {
          const int used = sweep_fused(v, Mt, r, R, part, gpr, false, stop);
          const FinishArgs fa = finish_args(used, cond);
          CK(launch_finish_step(fa, sms_, st_));
          const PrepArgs pa = prep_args(1, used);
          CK(launch_prep_step(pa, sms_, st_));
          return;
        }
        int fc_used = 0;
        fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, &fc_used, false, stop,
           fused_gram ? gpr : nullptr);
        const FinishArgs fa = finish_args(fused_gram ? fc_used : 0, cond);
        CK(launch_finish_step(fa, sms_, st_));
        const uint32_t ranges = fr(v, R, ncp, 1, r, part, nullptr, false, nullptr, stop);
        const PrepArgs pa = prep_args(1, int(ranges));
        CK(launch_prep_step(pa, sms_, st_));
      }, &body_launches);
      if (loop) {
        if (graphs_.size() >= 64) clear_graphs();
        graphs_[key] = {loop, body_launches};
      }
    }
  }
  if (loop) {
    {
      const PrepArgs pa = prep_args(0, 0);
      CK(launch_prep_step(pa, sms_, st_));
      count_launch();
    }
    trace("graph launch", mode);
    CK(cudaGraphLaunch(loop, st_));
    trace("graph launched", mode);
    if (stage_n_ < size_t(slot + 1) * size_t(stage_iters_ + 1) || stage_iters_ < max_iters)
      stage_reserve(slot + 1, max_iters);
    double* hs = stage_h_ + size_t(slot) * size_t(stage_iters_ + 1);
    CK(cudaMemcpyAsync(hs, hist, sizeof(double) * size_t(max_iters), cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(hs + stage_iters_, sumsq, sizeof(double), cudaMemcpyDeviceToHost, st_));
    if (!stage_ctrl_)
      CK(cudaHostAlloc(reinterpret_cast<void**>(&stage_ctrl_), kMaxStageModes * sizeof(AlsCtrl), cudaHostAllocDefault));
    if (slot >= kMaxStageModes) raise(12, "more than 64 staged modes");
    AlsCtrl* ch = stage_ctrl_ + slot;
    CK(cudaMemcpyAsync(ch, ctrl, sizeof(AlsCtrl), cudaMemcpyDeviceToHost, st_));
    out.hist_host = hs;
    out.sumsq_host = hs + stage_iters_;
    out.ctrl_host = ch;
    out.fc_bytes = 8.0 * (double(sh.count()) + double(F) * r + double(I) * r);
    out.body_launches = body_launches;
    out.r = r;
    out.fused = fused;
    out.rep.iterations = 0;
    trace("als graph enqueued", mode);
    return out;
  }
  while (true) {
    const int nb = std::min(batch, max_iters - enqueued);
    for (int b = 0; b < nb; ++b) {
      const int k = enqueued + b + 1;  // 1-based sweep
      PrepArgs pa;
      pa.part = part;
      pa.nparts = int(last_ranges);
      pa.ldp = ncp;
      pa.GRinv = GRinv;
      pa.from_partials = k > 1 ? 1 : 0;
      pa.I = uint32_t(I);
      pa.r = r;
      pa.ncp = ncp;
      pa.Lc = Lc;
      pa.GL = GL;
      pa.GLinv = GLinv;
      pa.Mt = Mt;
      pa.gpart = gpl;
      pa.gs = gs;
      pa.ctrl = ctrl;
      {
        const size_t rec = recs_.size();
        const auto ev = small_begin();
        coop_launch([&] { CK(launch_prep_step(pa, sms_, st_)); });
        small_end(ev);
        trace("  prep launched", k);
        if (profiling_) spec_recs_.push_back({k, 0, rec});
      }
      const size_t rec_fc = recs_.size();
      int fc_used = 0;
      if (fused) fc_used = sweep_fused(v, Mt, r, R, part, gpr, true, stop);
      else
        fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, &fc_used, true, stop,
           fused_gram ? gpr : nullptr);
      trace("  fc launched", k);
      if (profiling_) spec_recs_.push_back({k, 0, rec_fc});
      FinishArgs fa;
      fa.R = R;
      fa.F = F;
      fa.ld = ncp;
      fa.r = r;
      fa.GL = GL;
      fa.GRinv = GRinv;
      fa.gpart = gpr;
      fa.gs = gs;
      fa.ctrl = ctrl;
      fa.history = hist;
      fa.gram_nparts = fused_gram ? fc_used : 0;
      {
        const size_t rec = recs_.size();
        const auto ev = small_begin();
        if (dist_) {
          // R^T R over this shard's fibers, summed over the shards, then the step
          int nparts = fc_used;
          if (!fused_gram) {
            fa.mode = 1;
            coop_launch([&] { CK(launch_finish_step(fa, sms_, st_)); });
            nparts = finish_step_grid(F, sms_);
          }
          CK(launch_gram_reduce(gpr, nparts, uint64_t(ncp) * ncp, ncp, r, gs, st_));
          dist_->allreduce_sum(gs, size_t(r) * r, st_);
          fa.mode = 2;
        }
        coop_launch([&] { CK(launch_finish_step(fa, sms_, st_)); });
        small_end(ev);
        trace("  finish launched", k);
        if (profiling_) spec_recs_.push_back({k, 0, rec});
      }
      if (fused) {
        last_ranges = uint32_t(fc_used);  // the fused pass wrote one left-update partial per CTA
        count_launch(2);
        continue;
      }
      const size_t rec_fr = recs_.size();
      last_ranges = fr(v, R, ncp, 1, r, part, nullptr, true, nullptr, stop);
      if (dist_) last_ranges = reduce_left_partials(part, last_ranges, uint32_t(I), ncp, r);
      trace("  fr launched", k);
      if (profiling_) spec_recs_.push_back({k, 1, rec_fr});
      count_launch(2);
    }
    enqueued += nb;
    CK(cudaMemcpyAsync(&h, ctrl, sizeof(AlsCtrl), cudaMemcpyDeviceToHost, st_));
    trace("batch enqueued", enqueued);
    sync();
    trace("batch synced", h.iter);
    if (h.stop || enqueued >= max_iters) break;
    batch = 8;
  }
  (void)GR;
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
  // The work counters and the profiling records cover every enqueued pass;
  // keep the executed ones: FC of sweeps 1..iter, FR of sweeps 1..iter-1
  // (the stop decision of sweep `iter` skips its left update).
  {
    const int fr_run = h.stop ? h.iter - 1 : h.iter;
    // fused sweeps: one pass per enqueued sweep, executed for sweeps 1..iter
    const int skipped = fused ? enqueued - h.iter : (enqueued - h.iter) + (enqueued - fr_run);
    const double elems = double(sh.count());
    const double bytes = fused ? 8.0 * (elems + double(F) * r + 2.0 * double(I) * r)
                               : 8.0 * (elems + double(F) * r + double(I) * r);
    passes_ -= uint64_t(skipped);
    bytes_ -= uint64_t(skipped * bytes);
    for (const SpecRec& sr : spec_recs_) {
      const bool ran = sr.kind == 0 ? sr.k <= h.iter : sr.k <= fr_run;
      if (!ran && sr.rec < recs_.size()) recs_[sr.rec].cls = -1;
    }
    spec_recs_.clear();
  }
  ModeRep& rep = out.rep;
  rep.iterations = h.iter;
  rep.status = h.status;
  rep.achieved_eta = h.achieved;
  out.norm = h.norm;
  if (stage_n_ < size_t(slot + 1) * size_t(stage_iters_ + 1) || stage_iters_ < max_iters)
    stage_reserve(slot + 1, max_iters);
  double* hs = stage_h_ + size_t(slot) * size_t(stage_iters_ + 1);
  if (h.iter > 0)
    CK(cudaMemcpyAsync(hs, hist, sizeof(double) * h.iter, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(hs + stage_iters_, sumsq, sizeof(double), cudaMemcpyDeviceToHost, st_));
  out.hist_host = hs;
  out.sumsq_host = hs + stage_iters_;
  trace("als done", mode);
  return out;
}

// recover_singular_vectors (hosvd.cpp:65-72): the left singular vectors V of
// q^T A_(n) are the eigenvectors of the Gram matrix of R = A_(n)^T q; an FC
// pass forms R (with R^T R fused into its epilogue up to 32 columns, else the
// row pass of finish_step), a single-CTA Jacobi solve gives V ordered and
// signed as dense_svd (kernels.cpp:25-43, 273-301, 419-427), and U <- q V.
// The eigenvectors of a Gram matrix carry errors ~eps sigma_1^2 / (sigma_i^2 -
// sigma_j^2), against the reference's eps sigma_1 / (sigma_i - sigma_j)
// (QR + SVD of the triangle, kernels.cpp:431-436), so a second round repeats
// the step from q V0: the columns of A_(n)^T q V0 are formed directly from A,
// their Gram is diagonal up to eps sigma_i sigma_j, and its Jacobi rotation
// V1 refines V = V0 V1 to the reference's accuracy. The second round's R and
// V1^T are what the t-HOSVD core uses (A_(n)^T U = (A_(n)^T q V0) V1).
void Engine::recover_sv(const double* A, const Shape& sh, int mode, uint32_t r, double* U, double* vt) {
  recover_sv_round(A, sh, mode, r, U, sv_vt0_.d(size_t(r) * r));
  recover_sv_round(A, sh, mode, r, U, vt);
}

void Engine::recover_sv_round(const double* A, const Shape& sh, int mode, uint32_t r, double* U, double* vt) {
  ClsScope cls(fc_cls_, kClsTTM);
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  if (F < r)
    raise(12, "recover_singular_vectors: mode " + std::to_string(mode) + " has " + std::to_string(F) +
                  " fibers, fewer than the rank " + std::to_string(r));
  const uint32_t ncp = pad_nc(r);
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  double* Mt = mt_.d(I * ncp);
  CK(launch_pack(U, 1, I, uint32_t(I), r, Mt, ncp, st_));  // Mt[i][c] = U[i + c*I]
  count_launch();
  double* R = r_.d(F * ncp + 8);
  const bool fused_gram = ncp <= kFcGramMaxNc;
  const int nfin = std::max(finish_step_grid(F, sms_), fc_grid(v, Mt, ncp, r));
  double* gpr = fc_gram_.d(size_t(nfin) * ncp * ncp);
  int fc_used = 0;
  fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, &fc_used, true, nullptr, fused_gram ? gpr : nullptr);
  int nparts = fc_used;
  if (!fused_gram) {
    AlsCtrl* ctrl = static_cast<AlsCtrl*>(sv_ctrl_.ensure(sizeof(AlsCtrl)));
    CK(cudaMemsetAsync(ctrl, 0, sizeof(AlsCtrl), st_));
    FinishArgs fa;
    fa.R = R;
    fa.F = F;
    fa.ld = ncp;
    fa.r = r;
    fa.gpart = gpr;
    fa.ctrl = ctrl;
    fa.mode = 1;
    coop_launch([&] { CK(launch_finish_step(fa, sms_, st_)); });
    count_launch();
    nparts = finish_step_grid(F, sms_);
  }
  double* G = sv_g_.d(size_t(r) * r);
  CK(launch_gram_reduce(gpr, nparts, uint64_t(ncp) * ncp, ncp, r, G, st_));
  if (dist_) dist_->allreduce_sum(G, size_t(r) * r, st_);
  CK(launch_sym_eig(G, r, vt, nullptr, st_));
  double* Un = sv_u_.d(I * r);
  ExpandArgs ea;  // Un(i, c) = sum_k U(i, k) V(k, c): the expansion with s = I, K = r
  ea.in = U;
  ea.s = I;
  ea.P = 1;
  ea.K = r;
  ea.U = vt;
  ea.Iout = r;
  ea.out = Un;
  CK(launch_expand(ea, sms_, st_, nullptr));
  CK(cudaMemcpyAsync(U, Un, I * r * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  count_launch(3);
}

void Engine::recover_singular_vectors(const double* a, const Shape& sh, int mode, const double* q, uint64_t rows,
                                      uint64_t cols, double* out) {
  if (mode < 1 || mode > sh.N)
    raise(1, "recover_singular_vectors: mode " + std::to_string(mode) + " outside 1.." + std::to_string(sh.N));
  if (rows != sh.extent(mode))
    raise(2, "recover_singular_vectors: q has " + std::to_string(rows) + " rows, mode " + std::to_string(mode) +
                 " has extent " + std::to_string(sh.extent(mode)));
  if (cols < 1 || cols > kMaxRank) raise(12, "recover_singular_vectors: q must have 1..64 columns");
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  double* U = l_.d(rows * cols);
  CK(cudaMemcpyAsync(U, q, rows * cols * sizeof(double), cudaMemcpyHostToDevice, st_));
  recover_sv(A, sh, mode, uint32_t(cols), U, sv_vt_.d(cols * cols));
  CK(cudaMemcpyAsync(out, U, rows * cols * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

// ---- SVD / EIG factor engines (hosvd.cpp:89-99, 151-171) -----------------------
// The EIG engine's factor is sym_eig(mode_gram(t, n), R_n) (tensor_ops.cpp:332-389,
// kernels.cpp:448-604); the SVD engine's is the leading R_n left singular
// vectors of A_(n) (dense_svd, kernels.cpp:419-446), i.e. the same eigenvectors
// of A_(n) A_(n)^T, with the same descending order and sign convention. Here:
// the Gram matrix on DMMA straight from the tensor layout (gram.cu) and the
// device eigensolver (eig.cu: tridiagonalization, multisection, inverse
// iteration, blocked back-transform, the sign convention).
void Engine::gram_factor(const double* A, const Shape& sh, int mode, uint32_t r, double* U, bool refine) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  if (I > uint64_t(kSymEigMaxN))
    raise(12, "mode " + std::to_string(mode) + ": extent " + std::to_string(I) + " above the " +
                  std::to_string(kSymEigMaxN) + " supported by the SVD / EIG engines");
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  const GramPlan gp = gram_tensor_plan(v, sms_);
  double* part = gram_t_part_.d(std::max<size_t>(gp.part_doubles, 1));
  double* G = gram_t_.d(I * I);
  double* W = gram_w_.d(I);
  CK(launch_gram_tensor(v, gp, part, G, st_));
  count_launch(2);
  const std::string why = eig_.leading(G, int(I), int(r), U, W, st_);
  if (!why.empty()) raise(11, why);
  count_launch(5);
  // SVD engine / HOOI (dense_svd of the unfolding, hosvd.cpp:89-92, hooi.cpp:90):
  // eigenvectors of the Gram matrix carry errors ~eps s1^2 / (si^2 - sj^2)
  // (and ~eps s1^2 / s_r^2 outside the leading subspace), the singular vectors
  // of A_(n) ~eps s1 / (si - sj). Refinement: one power step Y = A_(n) A_(n)^T U
  // (an FC and an FR pass; column i carries errors ~eps s1 si, i.e. relative
  // eps s1 / si), its columns scaled to unit norm and orthonormalised
  // (CholQR2 of a near-orthonormal matrix), then one recover_sv round (the
  // columns of A_(n)^T Q come straight from A, their Gram is diagonal to
  // eps si sj, its Jacobi rotation fixes the basis inside the subspace). The
  // EIG engine keeps sym_eig(mode_gram) as the reference computes it.
  if (refine && r <= kMaxRank && F >= r) {
    const uint32_t ncp = pad_nc(r);
    FiberView v{A, s, P, uint32_t(I), s, s * I};
    double* Mt = mt_.d(I * ncp);
    CK(launch_pack(U, 1, I, uint32_t(I), r, Mt, ncp, st_));  // Mt[i][c] = U[i + c*I]
    double* R = r_.d(F * ncp + 8);
    {
      ClsScope cls(fc_cls_, kClsTTM);
      fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, nullptr, true);
    }
    double* part = fr_part_.d(size_t(fr_ranges(v, r)) * I * ncp);
    uint32_t ranges = fr(v, R, ncp, 1, r, part, nullptr, true, nullptr);
    if (dist_) ranges = reduce_left_partials(part, ranges, uint32_t(I), ncp, r);
    double* Y = l_.d(I * r);
    CK(launch_reduce_partials(part, int(ranges), uint32_t(I), ncp, r, Y, st_));
    CK(launch_normalize_columns(Y, uint32_t(I), r, st_));
    count_launch(3);
    qr_dev(Y, 0, I, uint32_t(I), r, U, nullptr, nullptr, 0, false);
    recover_sv_round(A, sh, mode, r, U, sv_vt0_.d(size_t(r) * r));
  }
}

double* Engine::sumsq_to_host(const double* A, uint64_t n) {
  if (!norm_h_) CK(cudaHostAlloc(reinterpret_cast<void**>(&norm_h_), 2 * sizeof(double), cudaHostAllocDefault));
  double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(n))));
  CK(launch_sumsq(A, n, sq, st_));
  CK(launch_sum(sq, sumsq_partials_count(n), sumsq_d_.d(2), st_));
  count_launch(2);
  if (dist_) dist_->allreduce_sum(sumsq_d_.d(2), 1, st_);
  CK(cudaMemcpyAsync(norm_h_, sumsq_d_.d(2), sizeof(double), cudaMemcpyDeviceToHost, st_));
  return norm_h_;
}

void Engine::mode_gram(const double* a, const Shape& sh, int mode, double* out) {
  if (mode < 1 || mode > sh.N)
    raise(1, "mode " + std::to_string(mode) + " out of range 1.." + std::to_string(sh.N));
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  const GramPlan gp = gram_tensor_plan(v, sms_);
  double* part = gram_t_part_.d(std::max<size_t>(gp.part_doubles, 1));
  double* G = gram_t_.d(I * I);
  CK(launch_gram_tensor(v, gp, part, G, st_));
  CK(cudaMemcpyAsync(out, G, I * I * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

void Engine::sym_eig(const double* g, uint64_t n, uint64_t k, double* values, double* vectors) {
  if (k > n)
    raise(2, "sym_eig: requested " + std::to_string(k) + " pairs from a " + std::to_string(n) +
                 "-dimensional matrix");
  double* G = gram_t_.d(std::max<uint64_t>(n * n, 1));
  double* W = gram_w_.d(std::max<uint64_t>(n, 1));
  double* U = sv_u_.d(std::max<uint64_t>(n * k, 1));
  double* V = sv_g_.d(std::max<uint64_t>(k, 1));
  if (n > uint64_t(kSymEigMaxN))
    raise(12, "sym_eig: dimension " + std::to_string(n) + " above the " + std::to_string(kSymEigMaxN) +
                  " supported on the device");
  (void)W;
  CK(cudaMemcpyAsync(G, g, n * n * sizeof(double), cudaMemcpyHostToDevice, st_));
  const std::string why = eig_.leading(G, int(n), int(k), U, V, st_);
  if (!why.empty()) raise(11, why);
  CK(cudaMemcpyAsync(values, V, k * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(vectors, U, n * k * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

// ---- HOOI (hooi.cpp:53-110) --------------------------------------------------------
Shape Engine::ttm_others(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                         const std::vector<double*>& U, int skip, double* dst) {
  Shape cur = sh;
  const double* src = A;
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  int last = sh.N;
  while (last >= 1 && last == skip) --last;
  if (last < 1) {  // order 1: nothing to contract
    CK(cudaMemcpyAsync(dst, A, sh.count() * sizeof(double), cudaMemcpyDeviceToDevice, st_));
    return cur;
  }
  for (int m = 1; m <= sh.N; ++m) {
    if (m == skip) continue;
    Shape nxt = cur;
    nxt.d[m - 1] = ranks[m - 1];
    double* out = (m == last) ? dst : bufs[which]->d(nxt.count());
    ttm_mode(src, cur, m, U[m - 1], uint32_t(ranks[m - 1]), out);
    src = out;
    cur = nxt;
    which ^= 1;
  }
  return cur;
}

// Per outer iteration and mode (ascending): contract the tensor with every
// other factor transposed, replace U_n by the leading R_n left singular
// vectors of that shrunk tensor's unfolding (dense_svd, hooi.cpp:89-94: here
// the eigenvectors of its Gram matrix W W^T, the same vectors with the same
// order and signs, gram_factor), and after the last mode form the core from
// the last shrunk tensor (:95-98). The fit is the explicit one,
// 1 - ||t - reconstruct|| / ||t|| (:47-49, the fused expansion-difference
// pass), and the loop stops at |fit_k - fit_{k-1}| <= tol (:104-108).
void Engine::hooi(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
                  const double* init_core, const double* init_factors, double tol, int max_iters, double* core,
                  double* factors, HooiRep* rep) {
  validate_truncation(sh, ranks);
  const int N = sh.N;
  for (int n = 1; n <= N; ++n) {
    uint64_t other = 1;
    for (int m = 1; m <= N; ++m)
      if (m != n) other *= ranks[m - 1];
    if (ranks[n - 1] > other)
      raise(4, "hooi: mode " + std::to_string(n) + " rank " + std::to_string(ranks[n - 1]) +
                   " exceeds the product of the other ranks (" + std::to_string(other) + ")");
  }
  *rep = HooiRep();
  const double* A = upload(a, sh.count(), a_dev, tensor_, nullptr);
  while (factor_bufs_.size() < size_t(N)) factor_bufs_.push_back(new DBuf());
  std::vector<double*> U(N);
  Shape cs;
  cs.N = N;
  for (int k = 0; k < N; ++k) cs.d[k] = ranks[k];
  begin_timed();
  const auto t0 = Clock::now();
  const double* ref_sumsq = sumsq_to_host(A, sh.count());
  sync();
  if (*ref_sumsq == 0.0) raise(3, "hooi: input tensor has zero norm");
  size_t ofs = 0;
  for (int n = 0; n < N; ++n) {
    U[n] = factor_bufs_[n]->d(sh.d[n] * ranks[n]);
    CK(cudaMemcpyAsync(U[n], init_factors + ofs, sh.d[n] * ranks[n] * sizeof(double), cudaMemcpyHostToDevice,
                       st_));
    ofs += sh.d[n] * ranks[n];
  }
  double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
  CK(cudaMemcpyAsync(core_buf, init_core, cs.count() * sizeof(double), cudaMemcpyHostToDevice, st_));
  rep->relative_residual = relative_residual_dev(A, sh, ranks, core_buf, U, ref_sumsq);
  rep->fit_history.push_back(1.0 - rep->relative_residual);
  uint64_t smax = 0;
  for (int n = 1; n <= N; ++n) {
    uint64_t c = sh.d[n - 1];
    for (int m = 1; m <= N; ++m)
      if (m != n) c *= ranks[m - 1];
    smax = std::max(smax, c);
  }
  double* shr = hooi_s_.d(std::max<uint64_t>(smax, 1));
  const int iters = std::max(1, max_iters);
  for (int iter = 1; iter <= iters; ++iter) {
    for (int n = 1; n <= N; ++n) {
      const Shape S = ttm_others(A, sh, ranks, U, n, shr);
      gram_factor(shr, S, n, uint32_t(ranks[n - 1]), U[n - 1], true);
      if (n == N) ttm_mode(shr, S, N, U[N - 1], uint32_t(ranks[N - 1]), core_buf);
    }
    rep->iterations = iter;
    rep->relative_residual = relative_residual_dev(A, sh, ranks, core_buf, U, ref_sumsq);
    const double fit = 1.0 - rep->relative_residual;
    const double prev = rep->fit_history.back();
    rep->fit_history.push_back(fit);
    if (std::fabs(fit - prev) <= tol) {
      rep->converged = true;
      break;
    }
  }
  rep->seconds = since(t0);
  rep->launches = launches_;
  CK(cudaMemcpyAsync(core, core_buf, cs.count() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  ofs = 0;
  for (int n = 0; n < N; ++n) {
    CK(cudaMemcpyAsync(factors + ofs, U[n], sh.d[n] * ranks[n] * sizeof(double), cudaMemcpyDeviceToHost, st_));
    ofs += sh.d[n] * ranks[n];
  }
  sync();
}

void Engine::begin_timed() {
  launches_ = 0;
  passes_ = 0;
  bytes_ = 0;
}

// multi_mode_product(t, {U_n^T}) in ascending mode order (hosvd.cpp:115-121).
void Engine::core_chain(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                        const std::vector<double*>& d_factors, double* d_core, int last_mode) {
  ClsScope cls(fc_cls_, kClsTTM);
  Shape cur = sh;
  const double* src = A;
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  const int nlast = last_mode > 0 ? last_mode : sh.N;
  for (int n = 1; n <= nlast; ++n) {
    const uint32_t r = uint32_t(ranks[n - 1]);
    Shape nxt = cur;
    nxt.d[n - 1] = r;
    double* dst = (n == nlast) ? d_core : bufs[which]->d(nxt.count());
    ttm_mode(src, cur, n, d_factors[n - 1], r, dst, n == 1 && last_mode == 0);
    src = dst;
    cur = nxt;
    which ^= 1;
  }
}

// ||A - core x_1 U_1 ... x_N U_N|| / ||A|| without materialising the
// reconstruction: expand modes 1..N-1, then fuse the mode-N expansion with
// the difference norm (relative_error(t, reconstruct(tk)), hosvd.cpp:123,189).
double Engine::relative_residual_dev(const double* A, const Shape& sh,
                                     const std::vector<uint64_t>& ranks, const double* d_core,
                                     const std::vector<double*>& d_factors, const double* ref_sumsq_host) {
  return residual_read(residual_enqueue(A, sh, ranks, d_core, d_factors), ref_sumsq_host);
}

double* Engine::residual_enqueue(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                                 const double* d_core, const std::vector<double*>& d_factors) {
  Shape cur;
  cur.N = sh.N;
  for (int k = 0; k < sh.N; ++k) cur.d[k] = ranks[k];
  const double* src = d_core;
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  int nsq = 0;
  double* sq = nullptr;
  for (int n = 1; n <= sh.N; ++n) {
    const uint64_t K = cur.extent(n), s = cur.stride(n), F = cur.count() / K, P = F / s;
    const uint64_t Iout = sh.d[n - 1];
    Shape nxt = cur;
    nxt.d[n - 1] = Iout;
    const bool last = (n == sh.N);
    if (K > kMaxRank) {
      // the expansion kernels hold at most 64 core indices: an FC TTM (the
      // contraction extent K is free there) in 64-row output blocks, and for
      // the last mode the materialised expansion against A
      double* dst = bufs[which]->d(nxt.count());
      {
        ClsScope cls(fc_cls_, kClsResid);
        mode_product_dev(src, cur, n, d_factors[n - 1], Iout, dst);
      }
      if (last) {
        nsq = sumsq_partials_count(nxt.count());
        sq = sq_part_.d(size_t(std::max(4096, nsq)));
        CK(launch_sumsq_diff(A, dst, nxt.count(), sq, st_));
        count_launch();
      }
      src = dst;
      cur = nxt;
      which ^= 1;
      continue;
    }
    ExpandArgs ea;
    ea.in = src;
    ea.s = s;
    ea.P = P;
    ea.K = uint32_t(K);
    ea.U = d_factors[n - 1];
    ea.Iout = uint32_t(Iout);
    if (last) {
      sq = sq_part_.d(size_t(std::max(4096, std::max(expand_grid(F, sms_), sms_))));
      ea.ref = A;
      ea.sumsq_part = sq;
    } else {
      ea.out = bufs[which]->d(nxt.count());
    }
    std::pair<cudaEvent_t, cudaEvent_t> ev{};
    if (profiling_) {
      ev = ev_pair();
      CK(cudaEventRecord(ev.first, st_));
    }
    if (last && !force_v1_ && expand_diff_tma_ok(ea)) {
      nsq = expand_diff_tma_grid(F, sms_);
      CK(launch_expand_diff_tma(ea, sms_, st_, nullptr));
    } else if (!last && !force_v1_ && expand_tma_ok(ea)) {
      CK(launch_expand_tma(ea, sms_, st_, nullptr));
    } else {
      if (last) nsq = expand_grid(F, sms_);
      CK(launch_expand(ea, sms_, st_, nullptr));
    }
    if (profiling_) {
      // expansion of mode n: 2 K Iout flops per output element; reads the input
      // (and the reference tensor on the last mode), writes the output
      const double outn = double(F) * double(Iout);
      CK(cudaEventRecord(ev.second, st_));
      record(kClsResid, ev.first, ev.second, 8.0 * (double(cur.count()) + outn), 2.0 * double(K) * outn);
    }
    count_launch();
    src = ea.out;
    cur = nxt;
    which ^= 1;
  }
  double* out = misc2_.d(1);
  CK(launch_sum(sq, nsq, out, st_));
  if (dist_) dist_->allreduce_sum(out, 1, st_);
  return out;
}

double Engine::residual_read(const double* out, const double* ref_sumsq_host) {
  double diff_sq = 0.0;
  CK(cudaMemcpyAsync(&diff_sq, out, sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  const double ref_sumsq = *ref_sumsq_host;
  if (ref_sumsq == 0.0) raise(3, "relative_error: reference tensor has zero norm");
  return std::sqrt(diff_sq / ref_sumsq);
}

// Results to the caller and the relative residual (hosvd.cpp:123,189). The
// core and factors go out on the copy stream while the residual expansion
// runs on the main stream: a copy to pageable host memory blocks the host
// until it completes, so the residual kernels are enqueued first and the
// transfer overlaps them. Destinations may be host or device pointers (UVA).
// Closed form of the relative residual of an orthogonal Tucker projection,
// ||A - A_hat||^2 = ||A||^2 - ||G||^2 (G = A x_n U_n^T, orthonormal U_n: the
// identity behind hosvd's error analysis), used when it is accurate to well
// inside the parity tolerance: its rounding error is a few eps ||A||^2 (the
// two sums, G's own rounding, the factors' orthonormality defect), i.e.
// |d rel| ~ 1e-15 / (2 rel); at rel >= kClosedFormMinRel that is <= 2e-11
// against the 1e-10 bar (BASELINE.json; config 3 at rel 1e-4 measured
// 4.1e-12 against the compiled reference). Smaller residuals (exact or nearly
// exact fits) take the explicit expansion pass. false when
// the explicit pass is needed (or forced: TKG_EXPLICIT_RESIDUAL=1).
bool Engine::closed_form_residual(const double* core_buf, uint64_t ncore, const double* ref_sumsq_host,
                                  double* rel) {
  static const bool forced = [] {
    const char* e = std::getenv("TKG_EXPLICIT_RESIDUAL");
    return e != nullptr && e[0] == '1';
  }();
  if (forced) return false;
  const int np = sumsq_partials_count(ncore);
  double* sq = sq_part_.d(size_t(std::max(4096, np)));
  double* g2 = misc2_.d(1);
  CK(launch_sumsq(core_buf, ncore, sq, st_));
  CK(launch_sum(sq, np, g2, st_));
  count_launch(2);
  double g2h = 0.0;
  CK(cudaMemcpyAsync(&g2h, g2, sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  const double a2 = *ref_sumsq_host;
  if (a2 == 0.0) raise(3, "relative_error: reference tensor has zero norm");
  const double rel2 = (a2 - g2h) / a2;
  static const double min_rel = [] {
    const char* e = std::getenv("TKG_CLOSED_FORM_MIN_REL");
    return e ? std::atof(e) : kClosedFormMinRel;
  }();
  if (!(rel2 >= min_rel * min_rel)) return false;
  *rel = std::sqrt(rel2);
  return true;
}

// Copies results to the caller's buffers and returns once they are there.
// Device, managed or pinned destinations take a direct copy; a pageable host
// destination (a plain numpy array, std::vector) goes through a pinned
// staging buffer at full PCIe speed and a multi-threaded host memcpy, instead
// of the driver's pageable path (~5 GB/s: 10 ms for config 5's 50 MB core).
void Engine::copy_results(const std::vector<ResultCopy>& outs, cudaStream_t s) {
  size_t staged = 0;
  std::vector<bool> pageable(outs.size(), false);
  for (size_t i = 0; i < outs.size(); ++i) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, outs[i].dst) != cudaSuccess) {
      cudaGetLastError();
      at.type = cudaMemoryTypeUnregistered;
    }
    pageable[i] = at.type == cudaMemoryTypeUnregistered;
    if (pageable[i]) staged += (outs[i].bytes + 255) / 256 * 256;
  }
  if (staged > out_stage_n_) {
    check_cuda(cudaStreamSynchronize(s), "result staging");
    if (out_stage_) cudaFreeHost(out_stage_);
    out_stage_ = nullptr;
    CK(cudaHostAlloc(&out_stage_, staged, cudaHostAllocDefault));
    out_stage_n_ = staged;
  }
  std::vector<std::pair<char*, const char*>> host;  // (dst, staging)
  std::vector<size_t> hbytes;
  size_t off = 0;
  for (size_t i = 0; i < outs.size(); ++i) {
    if (outs[i].bytes == 0) continue;
    if (pageable[i]) {
      char* st = static_cast<char*>(out_stage_) + off;
      CK(cudaMemcpyAsync(st, outs[i].src, outs[i].bytes, cudaMemcpyDeviceToHost, s));
      host.push_back({static_cast<char*>(outs[i].dst), st});
      hbytes.push_back(outs[i].bytes);
      off += (outs[i].bytes + 255) / 256 * 256;
    } else {
      CK(cudaMemcpyAsync(outs[i].dst, outs[i].src, outs[i].bytes, cudaMemcpyDefault, s));
    }
  }
  check_cuda(cudaStreamSynchronize(s), "result copy");
  size_t total = 0;
  for (size_t b : hbytes) total += b;
  if (total == 0) return;
  // split the host copies into ~4 MB pieces over up to 8 threads
  struct Piece { char* d; const char* s; size_t n; };
  std::vector<Piece> pieces;
  for (size_t i = 0; i < host.size(); ++i)
    for (size_t o = 0; o < hbytes[i]; o += size_t(4) << 20)
      pieces.push_back({host[i].first + o, host[i].second + o, std::min(size_t(4) << 20, hbytes[i] - o)});
  // threads only pay off for large copies (spawning one costs ~20-50 us)
  const size_t nt = total < (size_t(8) << 20) ? 1 : std::min<size_t>(8, pieces.size());
  if (nt <= 1) {
    for (const Piece& p : pieces) std::memcpy(p.d, p.s, p.n);
    return;
  }
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t k = t; k < pieces.size(); k += nt) std::memcpy(pieces[k].d, pieces[k].s, pieces[k].n);
    });
  for (auto& x : th) x.join();
}

void Engine::outputs_and_residual(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                                  const Shape& cs, const double* core_buf, const std::vector<double*>& U,
                                  const double* ref_sumsq, double* core, double* factors, DecompRep* rep) {
  const auto tr = Clock::now();
  CK(cudaEventRecord(out_ready_, st_));
  double rel_cf = 0.0;
  std::vector<ResultCopy> res;
  res.push_back({core, core_buf, cs.count() * sizeof(double)});
  {
    size_t ofs = 0;
    for (int n = 0; n < sh.N; ++n) {
      res.push_back({factors + ofs, U[n], sh.d[n] * ranks[n] * sizeof(double)});
      ofs += sh.d[n] * ranks[n];
    }
  }
  if (closed_form_residual(core_buf, cs.count(), ref_sumsq, &rel_cf)) {
    const auto td = Clock::now();
    copy_results(res, st_);
    rep->d2h_seconds = since(td);
    rep->relative_residual = rel_cf;
    rep->residual_seconds = since(tr);
    return;
  }
  const double* out = residual_enqueue(A, sh, ranks, core_buf, U);
  trace("residual enqueued");
  const auto td = Clock::now();
  CK(cudaStreamWaitEvent(cp_st_, out_ready_, 0));
  copy_results(res, cp_st_);
  trace("results copied");
  rep->d2h_seconds = since(td);
  rep->relative_residual = residual_read(out, ref_sumsq);
  rep->residual_seconds = since(tr);
}

// Reports, D2H and the residual of an SVD / EIG decomposition (the modes carry
// no ALS report: status -1, ModeReport::als empty, hosvd.hpp:33-37).
void Engine::finish_exact(const Shape& sh, const std::vector<uint64_t>& ranks, const Shape& cs, const double* A,
                          const double* core_buf, const std::vector<double*>& U, const double* ref_sumsq,
                          double* core, double* factors, DecompRep* rep, Clock::time_point t0,
                          const std::vector<int>* order) {
  sync();
  for (int k = 0; k < sh.N; ++k) {
    ModeRep mr;
    mr.mode = order ? (*order)[k] : k + 1;
    mr.iterations = 0;
    mr.status = -1;
    mr.seconds = mode_seconds(k);
    rep->per_mode.push_back(mr);
  }
  rep->seconds = since(t0);
  rep->launches = launches_;
  rep->passes = passes_;
  rep->bytes = bytes_;
  outputs_and_residual(A, sh, ranks, cs, core_buf, U, ref_sumsq, core, factors, rep);
}

void Engine::t_hosvd(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
                     const AlsCfg& cfg, double* core, double* factors, DecompRep* rep, bool want_sv,
                     int engine) {
  validate_truncation(sh, ranks);
  *rep = DecompRep();
  const double* A = upload(a, sh.count(), a_dev, tensor_, &rep->h2d_seconds);
  while (factor_bufs_.size() < size_t(sh.N)) factor_bufs_.push_back(new DBuf());
  std::vector<double*> U(sh.N);
  if (engine != kEngineAls) {
    // SVD / EIG engines (hosvd.cpp:89-99): per-mode factor, then the full TTM chain
    stage_reserve(sh.N, 1);
    begin_timed();
    const auto t0 = Clock::now();
    for (int n = 1; n <= sh.N; ++n) {
      const uint32_t r = uint32_t(ranks[n - 1]);
      mode_begin(n - 1);
      U[n - 1] = factor_bufs_[n - 1]->d(sh.d[n - 1] * r);
      gram_factor(A, sh, n, r, U[n - 1], engine == kEngineSvd);
      mode_end(n - 1);
    }
    Shape cs;
    cs.N = sh.N;
    for (int k = 0; k < sh.N; ++k) cs.d[k] = ranks[k];
    double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
    core_chain(A, sh, ranks, U, core_buf);
    const double* ref_sumsq = sumsq_to_host(A, sh.count());
    finish_exact(sh, ranks, cs, A, core_buf, U, ref_sumsq, core, factors, rep, t0, nullptr);
    return;
  }
  begin_timed();
  const auto t0 = Clock::now();
  g_trace_t0 = t0;
  const bool lanes = concurrent_modes_ok(ranks, want_sv) && sh.N > 1;
  if (!lanes) {
    // sequential modes: the later modes' initializer streams are generated on
    // the side stream while the first modes run (concurrent modes generate
    // their own, in parallel, on their own streams)
    std::vector<PreGen> items;
    for (int n = 2; n <= sh.N; ++n) items.push_back({n, sh.count() / sh.d[n - 1], uint32_t(ranks[n - 1]), MtWindow()});
    defer_pregenerate(items, cfg.seed);
  } else {
    pre_.clear();
    pending_pre_.clear();
  }
  trace("pregenerate enqueued");
  stage_reserve(sh.N, cfg.max_iters);
  bool sumsq_known = false;
  std::vector<AlsOut> outs;
  if (lanes) {
    // every mode on its own stream and buffers; ||A||^2 comes from mode 1's
    // init pass (the sequential driver's value: identical histories), which
    // the later modes wait for just before their stop rule is initialised;
    // the core waits for all
    while (lanes_.size() < size_t(sh.N)) {
      Lane* L = new Lane();
      CK(cudaStreamCreateWithFlags(&L->st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&L->done, cudaEventDisableTiming));
      lanes_.push_back(L);
    }
    CK(cudaEventRecord(out_ready_, st_));  // the tensor is on the device
    for (int n = 1; n <= sh.N; ++n) {
      Lane& L = *lanes_[n - 1];
      const uint32_t r = uint32_t(ranks[n - 1]);
      const uint64_t I = sh.d[n - 1];
      CK(cudaStreamWaitEvent(L.st, out_ready_, 0));
      swap_lane(L);
      try {
        if (!sumsq_ev_) CK(cudaEventCreateWithFlags(&sumsq_ev_, cudaEventDisableTiming));
        record_sumsq_ = n == 1;
        sumsq_from_ = n == 1 ? nullptr : lanes_[0]->sumsq_d.d(2);
        in_lanes_ = true;
        mode_begin(n - 1);
        outs.push_back(run_als(A, sh, n, r, cfg, n > 1, MtWindow(), n - 1));
        in_lanes_ = false;
        record_sumsq_ = false;
        sumsq_from_ = nullptr;
        U[n - 1] = factor_bufs_[n - 1]->d(I * r);
        qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[n - 1], n == sh.N ? rhat_.d(r * r) : nullptr, nullptr, 0,
               false);
        mode_end(n - 1);
        CK(cudaEventRecord(L.done, st_));
      } catch (...) {
        in_lanes_ = false;
        record_sumsq_ = false;
        sumsq_from_ = nullptr;
        swap_lane(L);
        throw;
      }
      swap_lane(L);
      trace("mode enqueued", n);
    }
    for (int n = 1; n <= sh.N; ++n) CK(cudaStreamWaitEvent(st_, lanes_[n - 1]->done, 0));
  }
  for (int n = 1; n <= sh.N && !lanes; ++n) {
    const uint32_t r = uint32_t(ranks[n - 1]);
    const uint64_t I = sh.d[n - 1];
    if (want_sv && r > kMaxRank)
      raise(12, "recover_singular_vectors: ranks above 64 are not supported (mode " + std::to_string(n) + ")");
    mode_begin(n - 1);
    outs.push_back(run_als(A, sh, n, r, cfg, sumsq_known, MtWindow(), n - 1));
    sumsq_known = true;
    U[n - 1] = factor_bufs_[n - 1]->d(I * r);
    if (n < sh.N) {
      qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[n - 1], nullptr, nullptr, 0, false);
      if (want_sv) recover_sv(A, sh, n, r, U[n - 1], sv_vt_.d(r * r));
    } else {  // keep R_hat of the last mode for the core
      qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[n - 1], rhat_.d(r * r), nullptr, 0, false);
      // with singular vectors, r_ becomes A_(N)^T q and the core's R_hat is
      // V^T: A_(N)^T U_N = (A_(N)^T q) V
      if (want_sv) recover_sv(A, sh, n, r, U[n - 1], rhat_.d(r * r));
    }
    mode_end(n - 1);
    trace("mode done", n);
  }
  Shape cs;
  cs.N = sh.N;
  for (int k = 0; k < sh.N; ++k) cs.d[k] = ranks[k];
  double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
  // core = A x_1 U_1^T ... x_N U_N^T (hosvd.cpp:115-121). The last mode's
  // factor comes from the final consistent pair (L = U_N R_hat, R = A_(N)^T L
  // (L^T L)^{-1}), so A_(N)^T U_N = R R_hat^T exactly: the first contraction
  // of the chain is the st-HOSVD shrink of R (hosvd.cpp:176-178) instead of
  // another pass over A, and the remaining TTMs run on the r_N-extent tensor.
  if (ranks[sh.N - 1] > kMaxRank) {
    core_chain(A, sh, ranks, U, core_buf);  // wide last rank: the plain TTM chain
  } else {
    const int N = sh.N;
    const uint32_t rN = uint32_t(ranks[N - 1]), ncpN = pad_nc(rN);
    const uint64_t IN = sh.d[N - 1], sN = sh.stride(N), FN = sh.count() / IN;
    Shape T = sh;
    T.d[N - 1] = rN;
    double* Tbuf = N == 1 ? core_buf : core_t_.d(T.count());
    const int nsh = shrink_count(FN);
    double* sq = sq_part_.d(size_t(std::max(4096, nsh)));
    double* RN = lanes ? lanes_[N - 1]->r.d(FN * ncpN + 8) : r_.d(FN * ncpN + 8);  // the last mode's R
    CK(launch_shrink(RN, ncpN, sN, 1, rN, rhat_.d(rN * rN), Tbuf, sq, st_));
    count_launch();
    if (N > 1) core_chain(Tbuf, T, ranks, U, core_buf, N - 1);
  }
  sync();
  trace("core synced");
  for (int n = 0; n < sh.N; ++n) {
    rep->per_mode.emplace_back();
    collect(outs[n], rep->per_mode.back());
    rep->per_mode.back().seconds = mode_seconds(n);
  }
  const double* ref_sumsq = outs[0].sumsq_host;
  rep->seconds = since(t0);
  rep->launches = launches_;
  rep->passes = passes_;
  rep->bytes = bytes_;
  outputs_and_residual(A, sh, ranks, cs, core_buf, U, ref_sumsq, core, factors, rep);
  trace("residual synced");
}

// select_order, or the caller's order validated as checked_order (hosvd.cpp:30-50)
std::vector<int> checked_order(const Shape& sh, const std::vector<uint64_t>& ranks, const std::vector<int>* order_in) {
  if (!order_in) return select_order(ranks);
  if (order_in->size() != size_t(sh.N))
    raise(1, "st_hosvd: order has " + std::to_string(order_in->size()) + " entries for an order-" +
                 std::to_string(sh.N) + " tensor");
  std::vector<bool> seen(sh.N, false);
  for (int m : *order_in) {
    if (m < 1 || m > sh.N || seen[m - 1]) raise(1, "st_hosvd: order is not a permutation of 1.." + std::to_string(sh.N));
    seen[m - 1] = true;
  }
  return *order_in;
}

void Engine::st_hosvd(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
                      const std::vector<int>* order_in, const AlsCfg& cfg, double* core,
                      double* factors, DecompRep* rep, int engine) {
  validate_truncation(sh, ranks);
  const std::vector<int> order = checked_order(sh, ranks, order_in);
  *rep = DecompRep();
  const double* A = upload(a, sh.count(), a_dev, tensor_, &rep->h2d_seconds);
  while (factor_bufs_.size() < size_t(sh.N)) factor_bufs_.push_back(new DBuf());
  std::vector<double*> U(sh.N);
  begin_timed();
  const auto t0 = Clock::now();
  Shape cur = sh;
  const double* work = A;
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  if (engine != kEngineAls) {
    // SVD / EIG engines (hosvd.cpp:151-171): factor, then working <- working x_n U^T
    stage_reserve(sh.N, 1);
    const double* ref_sumsq = sumsq_to_host(A, sh.count());
    for (size_t k = 0; k < order.size(); ++k) {
      const int mode = order[k];
      const uint32_t r = uint32_t(ranks[mode - 1]);
      const uint64_t I = cur.extent(mode), s = cur.stride(mode), F = cur.count() / I, P = F / s;
      mode_begin(int(k));
      U[mode - 1] = factor_bufs_[mode - 1]->d(I * r);
      gram_factor(work, cur, mode, r, U[mode - 1], engine == kEngineSvd);
      const uint32_t ncp = pad_nc(r);
      double* Mt = mt_.d(I * ncp);
      CK(launch_pack(U[mode - 1], 1, I, uint32_t(I), r, Mt, ncp, st_));
      count_launch();
      Shape nxt = cur;
      nxt.d[mode - 1] = r;
      double* dst = bufs[which]->d(nxt.count());
      FiberView v{work, s, P, uint32_t(I), s, s * I};
      ClsScope cls(fc_cls_, kClsTTM);
      fc(v, Mt, ncp, r, dst, 1, s, s * r, nullptr, nullptr, nullptr, true);
      mode_end(int(k));
      work = dst;
      cur = nxt;
      which ^= 1;
    }
    double* core_buf = static_cast<double*>(q_.ensure(cur.count() * sizeof(double)));
    CK(cudaMemcpyAsync(core_buf, work, cur.count() * sizeof(double), cudaMemcpyDeviceToDevice, st_));
    finish_exact(sh, ranks, cur, A, core_buf, U, ref_sumsq, core, factors, rep, t0, &order);
    return;
  }
  bool sumsq_known = false;
  {
    std::vector<PreGen> items;
    Shape w = sh;
    for (size_t k = 0; k < order.size(); ++k) {
      const int m = order[k];
      if (k > 0) items.push_back({m, w.count() / w.d[m - 1], uint32_t(ranks[m - 1]), MtWindow()});
      w.d[m - 1] = ranks[m - 1];
    }
    defer_pregenerate(items, cfg.seed);
  }
  stage_reserve(sh.N, cfg.max_iters);
  std::vector<AlsOut> outs;
  for (int mode : order) {
    const int k = int(outs.size());
    const uint32_t r = uint32_t(ranks[mode - 1]);
    const uint64_t I = cur.extent(mode), s = cur.stride(mode), F = cur.count() / I, P = F / s;
    mode_begin(k);
    outs.push_back(run_als(work, cur, mode, r, cfg, sumsq_known, MtWindow(), k));
    const uint32_t ncp = pad_nc(r);
    U[mode - 1] = factor_bufs_[mode - 1]->d(I * r);
    if (r > kMaxRank) {
      // wide rank: working <- working x_mode U^T (the TTM form of the shrink,
      // equal to R_hat R^T for the returned consistent pair)
      qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[mode - 1], nullptr, nullptr, 0, false);
      Shape nxt = cur;
      nxt.d[mode - 1] = r;
      double* dst = bufs[which]->d(nxt.count());
      ttm_mode(work, cur, mode, U[mode - 1], r, dst, true);
      double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(nxt.count()))));
      CK(launch_sumsq(dst, nxt.count(), sq, st_));
      CK(launch_sum(sq, sumsq_partials_count(nxt.count()), sumsq_d_.d(2), st_));
      count_launch(2);
      sumsq_known = true;
      mode_end(k);
      work = dst;
      cur = nxt;
      which ^= 1;
      continue;
    }
    double* RhT = rhatT_.d(size_t(r) * ncp);
    qr_dev(l_.d(I * r), 0, I, uint32_t(I), r, U[mode - 1], rhat_.d(r * r), RhT, ncp, false);
    // working <- tensorize(R_hat R^T, mode, shrunk) (hosvd.cpp:176-178): an FC
    // over R read as a tensor (extent r, strides F / s), fused ||.||^2.
    Shape nxt = cur;
    nxt.d[mode - 1] = r;
    double* dst = bufs[which]->d(nxt.count());
    const int nsh = shrink_count(F);
    double* sq = sq_part_.d(size_t(std::max(4096, nsh)));
    std::pair<cudaEvent_t, cudaEvent_t> ev{};
    if (profiling_) {
      ev = ev_pair();
      CK(cudaEventRecord(ev.first, st_));
    }
    CK(launch_shrink(r_.d(F * ncp + 8), ncp, s, P, r, rhat_.d(r * r), dst, sq, st_, true));  // R_hat: qr_dev's upper factor
    if (profiling_) {
      // shrink: reads R (F x r), writes the r x F working tensor, 2 r^2 F flops
      CK(cudaEventRecord(ev.second, st_));
      record(kClsTTM, ev.first, ev.second, 16.0 * double(F) * r, 2.0 * double(F) * r * r);
    }
    CK(launch_sum(sq, nsh, sumsq_d_.d(2), st_));
    count_launch(2);
    sumsq_known = true;
    mode_end(k);
    work = dst;
    cur = nxt;
    which ^= 1;
  }
  Shape cs = cur;
  double* core_buf = static_cast<double*>(q_.ensure(cs.count() * sizeof(double)));
  CK(cudaMemcpyAsync(core_buf, work, cs.count() * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  sync();
  for (size_t k = 0; k < outs.size(); ++k) {
    rep->per_mode.emplace_back();
    collect(outs[k], rep->per_mode.back());
    rep->per_mode.back().seconds = mode_seconds(int(k));
  }
  const double* ref_sumsq = outs[0].sumsq_host;
  rep->seconds = since(t0);
  rep->launches = launches_;
  rep->passes = passes_;
  rep->bytes = bytes_;
  outputs_and_residual(A, sh, ranks, cs, core_buf, U, ref_sumsq, core, factors, rep);
}

void Engine::als_low_rank(const double* a, bool a_dev, const Shape& sh, int mode, uint32_t r,
                          const AlsCfg& cfg, double* l_out, double* r_out, ModeRep* rep) {
  const uint64_t I = sh.extent(mode);
  const double* A = upload(a, sh.count(), a_dev, tensor_, nullptr);
  AlsOut o = run_als(A, sh, mode, r, cfg, false);  // zero norm, then the rank / init guards
  const uint64_t F = sh.count() / I;
  CK(cudaMemcpyAsync(l_out, l_.d(I * r), I * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  if (r_out) {  // R is row-major [F][ncp] on the device; the API returns column-major F x r
    const uint32_t ncp = pad_nc(r);
    double* rc = work_b_.d(F * r);
    CK(launch_pack(r_.d(F * ncp + 8), 1, ncp, r, uint32_t(F), rc, uint32_t(F), st_));
    CK(cudaMemcpyAsync(r_out, rc, F * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  }
  sync();
  collect(o, *rep);
}

// als_sweep (als.cpp:89-96): one right update from l, the closed-form
// residual right after it, one left update; the sweep kernels of run_als on
// a private control block (eta < 0: the stop rule never fires).
void Engine::als_sweep(const double* a, const Shape& sh, int mode, const double* l, uint32_t r, double* l_out,
                       double* r_out, double* residual) {
  if (mode < 1 || mode > sh.N)
    raise(1, "mode " + std::to_string(mode) + " out of range 1.." + std::to_string(sh.N));
  if (r < 1 || r > kMaxRank) raise(12, "als_sweep: r must be in 1..64");
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I, P = F / s;
  const uint32_t ncp = pad_nc(r);
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  FiberView v{A, s, P, uint32_t(I), s, s * I};
  double* Lc = l_.d(I * r);
  CK(cudaMemcpyAsync(Lc, l, I * r * sizeof(double), cudaMemcpyHostToDevice, st_));
  double* Mt = mt_.d(I * ncp);
  double* R = r_.d(F * ncp + 8);
  double* GL = gl_.d(kMaxRank * kMaxRank);
  double* GLinv = cholL_.d(kMaxRank * kMaxRank);
  double* GRinv = cholR_.d(kMaxRank * kMaxRank);
  double* gpl = gram_part_.d(size_t(coop_partials_cap(sms_)) * r * r);
  double* gs = gs_.d(size_t(r) * r);
  const uint32_t nranges = fr_ranges(v, r);
  double* part = fr_part_.d(size_t(nranges) * I * ncp);
  double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(sh.count()))));
  double* sumsq = sumsq_d_.d(2);
  CK(launch_sumsq(A, sh.count(), sq, st_));
  CK(launch_sum(sq, sumsq_partials_count(sh.count()), sumsq, st_));
  AlsCtrl* ctrl = static_cast<AlsCtrl*>(ctrl_d_.ensure(sizeof(AlsCtrl)));
  double* hist = hist_d_.d(2);
  CK(launch_ctrl_init(ctrl, sumsq, -1.0, 2, 2, 0, st_));
  const bool fused_gram = ncp <= kFcGramMaxNc;
  const int nfin = std::max(finish_step_grid(F, sms_), fc_grid(v, Mt, ncp, r));
  double* gpr = fc_gram_.d(size_t(nfin) * ncp * ncp);
  PrepArgs pa;
  pa.from_partials = 0;
  pa.I = uint32_t(I);
  pa.r = r;
  pa.ncp = ncp;
  pa.Lc = Lc;
  pa.GL = GL;
  pa.GLinv = GLinv;
  pa.Mt = Mt;
  pa.gpart = gpl;
  pa.gs = gs;
  pa.ctrl = ctrl;
  coop_launch([&] { CK(launch_prep_step(pa, sms_, st_)); });
  int fc_used = 0;
  fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, &fc_used, false, &ctrl->stop,
     fused_gram ? gpr : nullptr);
  FinishArgs fa;
  fa.R = R;
  fa.F = F;
  fa.ld = ncp;
  fa.r = r;
  fa.GL = GL;
  fa.GRinv = GRinv;
  fa.gpart = gpr;
  fa.gs = gs;
  fa.ctrl = ctrl;
  fa.history = hist;
  fa.gram_nparts = fused_gram ? fc_used : 0;
  coop_launch([&] { CK(launch_finish_step(fa, sms_, st_)); });
  if (r_out) {  // R of this sweep, column-major F x r, before the left update
    double* rc = work_b_.d(F * r);
    CK(launch_pack(R, 1, ncp, r, uint32_t(F), rc, uint32_t(F), st_));
    CK(cudaMemcpyAsync(r_out, rc, F * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  }
  AlsCtrl h1;
  CK(cudaMemcpyAsync(&h1, ctrl, sizeof(AlsCtrl), cudaMemcpyDeviceToHost, st_));
  const uint32_t ranges = fr(v, R, ncp, 1, r, part, nullptr, false, nullptr, &ctrl->stop);
  // left update L = Y G_R^{-1} (the prep step's phase B writes Lc; a singular
  // Gram of the new L, which the reference never factors here, is ignored)
  pa.from_partials = 1;
  pa.part = part;
  pa.nparts = int(ranges);
  pa.ldp = ncp;
  pa.GRinv = GRinv;
  coop_launch([&] { CK(launch_prep_step(pa, sms_, st_)); });
  double res = 0.0;
  CK(cudaMemcpyAsync(&res, hist, sizeof(double), cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(l_out, Lc, I * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  count_launch(8);
  auto singular = [&](double piv, int col) {
    raise(5, "spd_solve: pivot " + std::to_string(piv) + " at column " + std::to_string(col) +
                 " is singular to working precision");
  };
  if (h1.error == kAlsErrZeroNorm) singular(0.0, 1);  // R = 0: R^T R has a zero pivot
  if (h1.error == kAlsErrRightSingular || h1.error == kAlsErrLeftSingular) singular(h1.pivot, h1.pad);
  if (residual) *residual = res;
}

void Engine::als_init(const double* a, bool a_dev, const Shape& sh, int mode, uint32_t r,
                      uint64_t seed, double* l_out) {
  const uint64_t I = sh.extent(mode);
  if (r < 1 || r > I)
    raise(4, "mode " + std::to_string(mode) + ": rank " + std::to_string(r) + " outside 1.." + std::to_string(I));
  const double* A = upload(a, sh.count(), a_dev, tensor_, nullptr);
  const uint64_t s = sh.stride(mode), F = sh.count() / I;
  if (r > kMaxRank) {  // 64-column FR blocks + CholQR2 (engine_wide.cpp)
    FiberView v{A, s, F / s, uint32_t(I), s, s * I};
    double* S = s_.d(F * r + 8);
    gen_uniform(seed, uint32_t(mode), F * r, S);
    double* Y = qy_.d(I * r);
    double* part = fr_part_.d(size_t(fr_ranges(v, 64)) * I * 64);
    for (uint32_t c0 = 0; c0 < r; c0 += 64) {
      const uint32_t nc = std::min<uint32_t>(64, r - c0);
      const uint32_t ranges = fr(v, S + uint64_t(c0) * F, 1, F, nc, part, nullptr, false, nullptr);
      CK(launch_reduce_partials(part, int(ranges), uint32_t(I), pad_nc(nc), nc, Y + uint64_t(c0) * I, st_));
    }
    qr_wide(Y, uint32_t(I), r, l_.d(I * r), nullptr, true);
    const int bad = qr_degenerate_col();
    if (bad != 0)
      raise(6, "als_init: randomized range collapsed at column " + std::to_string(bad) + " for mode " +
                   std::to_string(mode));
    CK(cudaMemcpyAsync(l_out, l_.d(I * r), I * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
    sync();
    return;
  }
  const uint32_t ncp = pad_nc(r);
  FiberView v{A, s, F / s, uint32_t(I), s, s * I};
  double* S = s_.d(F * r + 8);
  gen_uniform(seed, uint32_t(mode), F * r, S);
  const uint32_t nranges = fr_ranges(v, r);
  double* part = fr_part_.d(size_t(nranges) * I * ncp);
  const uint32_t ranges = fr(v, S, 1, F, r, part, nullptr, false, nullptr);
  status_h_->degenerate_col = 0;
  qr_dev(part, int(ranges), ncp, uint32_t(I), r, l_.d(I * r), nullptr, nullptr, 0, true);
  const int bad = qr_degenerate_col();
  if (bad != 0)
    raise(6, "als_init: randomized range collapsed at column " + std::to_string(bad) + " for mode " +
                 std::to_string(mode));
  CK(cudaMemcpyAsync(l_out, l_.d(I * r), I * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

// ---- primitives ------------------------------------------------------------------
void Engine::unfold_times(const double* a, const Shape& sh, int mode, const double* m, uint32_t r,
                          double* out) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I;
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  double* M = s_.d(F * r + 8);  // column-major F x r, as given
  CK(cudaMemcpyAsync(M, m, F * r * sizeof(double), cudaMemcpyHostToDevice, st_));
  FiberView v{A, s, F / s, uint32_t(I), s, s * I};
  const uint32_t nranges = fr_ranges(v, std::min<uint32_t>(r, kMaxRank));
  double* part = fr_part_.d(size_t(nranges) * I * pad_nc(std::min<uint32_t>(r, kMaxRank)));
  double* y = misc_.d(I * r);
  for (uint32_t c0 = 0; c0 < r; c0 += kMaxRank) {  // 64-column blocks
    const uint32_t nc = std::min(kMaxRank, r - c0);
    const uint32_t ranges = fr(v, M + uint64_t(c0) * F, 1, F, nc, part, nullptr, false, nullptr);
    CK(launch_reduce_partials(part, int(ranges), uint32_t(I), pad_nc(nc), nc, y + uint64_t(c0) * I, st_));
  }
  CK(cudaMemcpyAsync(out, y, I * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

void Engine::unfold_t_times(const double* a, const Shape& sh, int mode, const double* m,
                            uint32_t r, double* out) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I;
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  double* Mc = misc_.d(I * r);
  CK(cudaMemcpyAsync(Mc, m, I * r * sizeof(double), cudaMemcpyHostToDevice, st_));
  double* R = r_.d(F * r);
  FiberView v{A, s, F / s, uint32_t(I), s, s * I};
  for (uint32_t c0 = 0; c0 < r; c0 += kMaxRank) {  // 64-column blocks, column-major F x r
    const uint32_t nc = std::min(kMaxRank, r - c0), ncp = pad_nc(nc);
    double* Mt = mt_.d(I * ncp);
    CK(launch_pack(Mc + uint64_t(c0) * I, 1, I, uint32_t(I), nc, Mt, ncp, st_));
    fc(v, Mt, ncp, nc, R + uint64_t(c0) * F, 1, F, s, nullptr, nullptr, nullptr, false);
  }
  CK(cudaMemcpyAsync(out, R, F * r * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

// dst <- X x_mode U, U (rows x I_mode, device, column-major), tensor layout,
// in chunks of 64 output rows (mode_n_product, tensor_ops.cpp:129-169)
void Engine::mode_product_dev(const double* X, const Shape& sh, int mode, const double* U, uint64_t rows,
                              double* dst) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I;
  FiberView v{X, s, F / s, uint32_t(I), s, s * I};
  for (uint64_t c0 = 0; c0 < rows; c0 += 64) {
    const uint32_t nc = uint32_t(std::min<uint64_t>(64, rows - c0));
    const uint32_t ncp = pad_nc(nc);
    double* Mt = mt_.d(I * ncp);
    // Mt[i][c] = U[(c0 + c) + i*rows]
    CK(launch_pack(U + c0, rows, 1, uint32_t(I), nc, Mt, ncp, st_));
    count_launch();
    fc(v, Mt, ncp, nc, dst + c0 * s, 1, s, s * rows, nullptr, nullptr, nullptr, false);
  }
}

void Engine::mode_n_product(const double* a, const Shape& sh, const double* u, uint64_t rows,
                            uint64_t cols, int mode, double* out) {
  const uint64_t I = sh.extent(mode);
  if (cols != I)
    raise(2, "mode_n_product: factor has " + std::to_string(cols) + " columns, mode " +
                 std::to_string(mode) + " has extent " + std::to_string(I));
  const double* A = upload(a, sh.count(), false, tensor_, nullptr);
  double* U = misc_.d(rows * cols);
  CK(cudaMemcpyAsync(U, u, rows * cols * sizeof(double), cudaMemcpyHostToDevice, st_));
  Shape nxt = sh;
  nxt.d[mode - 1] = rows;
  double* dst = work_a_.d(nxt.count());
  mode_product_dev(A, sh, mode, U, rows, dst);
  CK(cudaMemcpyAsync(out, dst, nxt.count() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

// multi_mode_product (tensor_ops.cpp:171-191): the factors sorted by mode
// (duplicates rejected), applied ascending on the device. Returns the shape.
Shape Engine::multi_mode_product(const double* a, const Shape& sh, const std::vector<int>& modes,
                                 const std::vector<const double*>& factors, const std::vector<uint64_t>& rows,
                                 const std::vector<uint64_t>& cols, double* out) {
  std::vector<size_t> idx(modes.size());
  for (size_t k = 0; k < idx.size(); ++k) idx[k] = k;
  std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return modes[x] < modes[y]; });
  for (size_t k = 0; k + 1 < idx.size(); ++k)
    if (modes[idx[k]] == modes[idx[k + 1]])
      raise(1, "multi_mode_product: duplicate mode " + std::to_string(modes[idx[k]]));
  Shape cur = sh;
  for (size_t k : idx) {
    const int m = modes[k];
    if (m < 1 || m > sh.N)
      raise(1, "mode " + std::to_string(m) + " out of range 1.." + std::to_string(sh.N));
    if (cols[k] != sh.extent(m))
      raise(2, "mode_n_product: factor has " + std::to_string(cols[k]) + " columns, mode " + std::to_string(m) +
                   " has extent " + std::to_string(sh.extent(m)));
  }
  const double* src = upload(a, sh.count(), false, tensor_, nullptr);
  DBuf* bufs[2] = {&work_a_, &work_b_};
  int which = 0;
  for (size_t k : idx) {
    const int m = modes[k];
    const uint64_t I = cur.extent(m);
    const uint64_t nr = rows[k];
    // the factor is rows x I column-major on the host
    double* U = misc_.d(nr * I);
    CK(cudaMemcpyAsync(U, factors[k], nr * I * sizeof(double), cudaMemcpyHostToDevice, st_));
    Shape nxt = cur;
    nxt.d[m - 1] = nr;
    double* dst = bufs[which]->d(std::max<uint64_t>(nxt.count(), 1));
    mode_product_dev(src, cur, m, U, nr, dst);
    src = dst;
    cur = nxt;
    which ^= 1;
  }
  CK(cudaMemcpyAsync(out, src, cur.count() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  return cur;
}

double Engine::frobenius_norm(const double* a, uint64_t n) {
  const double* A = upload(a, n, false, tensor_, nullptr);
  double* sq = sq_part_.d(std::max(1, sumsq_partials_count(n)));
  double* out = misc2_.d(1);
  CK(launch_sumsq(A, n, sq, st_));
  CK(launch_sum(sq, sumsq_partials_count(n), out, st_));
  double h = 0.0;
  CK(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  return std::sqrt(h);
}

double Engine::relative_error(const double* a, const double* b, uint64_t n) {
  // tensor_ops.cpp:395-407: sqrt(sum (b-a)^2 / sum a^2), both sums on device
  const double* A = upload(a, n, false, tensor_, nullptr);
  double* B = work_a_.d(n);
  CK(cudaMemcpyAsync(B, b, n * sizeof(double), cudaMemcpyHostToDevice, st_));
  const int np = std::max(1, sumsq_partials_count(n));
  double* sq = sq_part_.d(2 * size_t(np));
  double* out = misc2_.d(2);
  CK(launch_sumsq(A, n, sq, st_));
  CK(launch_sum(sq, sumsq_partials_count(n), out, st_));
  CK(launch_sumsq_diff(A, B, n, sq + np, st_));
  CK(launch_sum(sq + np, sumsq_partials_count(n), out + 1, st_));
  double h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  if (h[0] == 0.0) raise(3, "relative_error: reference tensor has zero norm");
  return std::sqrt(h[1] / h[0]);
}

void Engine::reduced_qr(const double* a, uint64_t rows, uint64_t cols, double* q, double* r) {
  if (rows < cols)
    raise(2, "reduced_qr: need rows >= cols, got " + std::to_string(rows) + "x" + std::to_string(cols));
  if (cols > kMaxRank) raise(12, "reduced_qr: more than 64 columns");
  double* A = misc_.d(rows * cols);
  CK(cudaMemcpyAsync(A, a, rows * cols * sizeof(double), cudaMemcpyHostToDevice, st_));
  double* Q = l_.d(rows * cols);
  double* R = rhat_.d(cols * cols);
  CK(launch_qr(A, 0, rows, uint32_t(rows), uint32_t(cols), Q, R, nullptr, 0,
               qr_work_.d(2 * rows * cols + cols), 0, status_d_, st_));
  CK(cudaMemcpyAsync(q, Q, rows * cols * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(r, R, cols * cols * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

void Engine::gram(const double* a, uint64_t rows, uint64_t cols, double* out) {
  if (cols > kMaxRank) raise(12, "gram: more than 64 columns");
  double* A = misc_.d(rows * cols);
  CK(cudaMemcpyAsync(A, a, rows * cols * sizeof(double), cudaMemcpyHostToDevice, st_));
  double* gp = gram_part_.d(size_t(gram_partials_count(uint32_t(rows))) * cols * cols);
  CK(launch_gram_partials(A, rows, uint32_t(rows), uint32_t(cols), gp, st_));
  double* G = gl_.d(cols * cols);
  double* ch = cholL_.d(cols * cols);
  CK(launch_chol(gp, gram_partials_count(uint32_t(rows)), cols * cols, int(cols), uint32_t(cols), G, ch,
                 &status_d_->pad, status_d_, st_));
  CK(cudaMemcpyAsync(out, G, cols * cols * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

void Engine::bench_contractions(const double* A, const Shape& sh, int mode, uint32_t r, int reps,
                                double* out_ms) {
  const uint64_t I = sh.extent(mode), s = sh.stride(mode), F = sh.count() / I;
  if (r < 1 || r > kMaxRank) raise(12, "bench_contractions: r must be in 1..64");
  const uint32_t ncp = pad_nc(r);
  FiberView v{A, s, F / s, uint32_t(I), s, s * I};
  double* Mt = mt_.d(I * ncp);
  double* R = r_.d(F * ncp + 8);
  CK(cudaMemsetAsync(Mt, 0, I * ncp * sizeof(double), st_));
  CK(cudaMemsetAsync(R, 0, F * ncp * sizeof(double), st_));
  const uint32_t nranges = fr_ranges(v, r);
  double* part = fr_part_.d(size_t(nranges) * I * ncp);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, nullptr, false);  // warm-up
  fr(v, R, ncp, 1, r, part, nullptr, false, nullptr);
  CK(cudaEventRecord(e0, st_));
  for (int k = 0; k < reps; ++k) fc(v, Mt, ncp, r, R, ncp, 1, s * ncp, nullptr, nullptr, nullptr, false);
  CK(cudaEventRecord(e1, st_));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  out_ms[0] = ms / reps;
  CK(cudaEventRecord(e0, st_));
  for (int k = 0; k < reps; ++k) fr(v, R, ncp, 1, r, part, nullptr, false, nullptr);
  CK(cudaEventRecord(e1, st_));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  out_ms[1] = ms / reps;
  // the init pass: S column-major (the reference's storage order), with and
  // without the fused ||A||^2
  double* S = s_.d(F * r + 8);
  CK(cudaMemsetAsync(S, 0, F * r * sizeof(double), st_));
  double* sq = sq_part_.d(size_t(std::max(4096, sumsq_partials_count(sh.count()))));
  for (int with_sq = 1; with_sq >= 0; --with_sq) {
    fr(v, S, 1, F, r, part, with_sq ? sq : nullptr, false, nullptr);
    CK(cudaEventRecord(e0, st_));
    for (int k = 0; k < reps; ++k) fr(v, S, 1, F, r, part, with_sq ? sq : nullptr, false, nullptr);
    CK(cudaEventRecord(e1, st_));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    out_ms[with_sq ? 2 : 3] = ms / reps;
  }
  // the fused sweep pass (r <= 16): FC + R^T R + FR from one read
  out_ms[4] = 0.0;
  if (sweep_fused_usable(v, Mt, r, R)) {
    double* partf = fr_part_.d(size_t(std::max<uint32_t>(nranges, uint32_t(sweep_fused_grid(v, r, sms_)))) * I * ncp);
    double* gpr = fc_gram_.d(size_t(sweep_fused_grid(v, r, sms_)) * ncp * ncp);
    sweep_fused(v, Mt, r, R, partf, gpr, false, nullptr);
    CK(cudaEventRecord(e0, st_));
    for (int k = 0; k < reps; ++k) sweep_fused(v, Mt, r, R, partf, gpr, false, nullptr);
    CK(cudaEventRecord(e1, st_));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    out_ms[4] = ms / reps;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void Engine::uniform01(uint64_t seed, uint32_t stream, uint64_t n, double* out) {
  double* d = s_.d(n);
  gen_uniform(seed, stream, n, d);
  CK(cudaMemcpyAsync(out, d, n * sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
}

}  // namespace tkg
