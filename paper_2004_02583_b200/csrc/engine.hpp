// Host orchestration of the B200 ALS-HOSVD path (C++ side of the C-ABI).
//
// One Engine owns a device, a stream, the mapped status block and grow-only
// device workspaces. The control flow mirrors the reference exactly:
//   als_low_rank  als.cpp:98-161   (stop rule, consistent pair, error mapping)
//   t_hosvd       hosvd.cpp:74-125 (per-mode ALS, QR, ascending TTM core)
//   st_hosvd      hosvd.cpp:127-191 (order, ALS, QR, R_hat R^T shrink)
// while every pass over the tensor and every small solve runs on the GPU.
#pragma once
#include <functional>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "comm.hpp"
#include "coop.cuh"
#include "eig.hpp"
#include "kernels.cuh"

namespace tkg {

struct Error : std::runtime_error {
  int code;     // ErrorCategory + 1
  int subtype;  // tkg_subtype
  Error(int code_, int subtype_, const std::string& m) : std::runtime_error(m), code(code_), subtype(subtype_) {}
};

[[noreturn]] void raise(int subtype, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define CK(x) ::tkg::check_cuda((x), #x)

struct Shape {
  int N = 0;
  uint64_t d[64] = {0};  // TKG_MAX_ORDER
  uint64_t count() const;
  uint64_t extent(int mode) const;  // validates, 1-based
  uint64_t stride(int mode) const;
  std::string str() const;
};

struct AlsCfg {
  double eta = 1e-4;
  int max_iters = 50;
  uint64_t seed = 0;
  const double* init = nullptr;  // host I x r col-major
  uint64_t init_rows = 0, init_cols = 0;  // init's shape (checked against I x r, als.cpp:106-113)
};

// FactorEngine::Kind (hosvd.hpp:19-27)
enum EngineKind { kEngineSvd = 0, kEngineEig = 1, kEngineAls = 2 };

struct ModeRep {
  int mode = 0;
  int iterations = 0;
  int status = 1;  // -1: no ALS report (SVD / EIG engine), ModeReport::als empty
  double achieved_eta = 0.0;
  double seconds = 0.0;
  std::vector<double> history;
};

struct DecompRep {
  std::vector<ModeRep> per_mode;
  double relative_residual = 0.0;
  double seconds = 0.0;
  double h2d_seconds = 0.0;
  double d2h_seconds = 0.0;
  double residual_seconds = 0.0;
  uint64_t launches = 0;
  uint64_t passes = 0;
  uint64_t bytes = 0;
};

// HooiResult (hooi.hpp:23-31) minus the Tucker tensor (returned in buffers)
struct HooiRep {
  int iterations = 0;
  bool converged = false;
  std::vector<double> fit_history;  // [0] = the warm start's fit
  double relative_residual = 0.0;   // of the returned decomposition (1 - fit, unrounded)
  double seconds = 0.0;
  uint64_t launches = 0;
};

class DBuf {
 public:
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf();
  void* ensure(size_t bytes);
  double* d(size_t count) { return static_cast<double*>(ensure(count * sizeof(double))); }
  uint64_t* u(size_t count) { return static_cast<uint64_t*>(ensure(count * sizeof(uint64_t))); }
  void release();
  void swap(DBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
  }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// device-time classes of bench.py's per-class breakdown (profiling only):
// FC right updates, FR left updates + init passes, small LA steps, RNG,
// TTM contractions outside the ALS loop (core chain, st TTM, singular
// vectors), the relative-residual expansion passes
enum KernelClass { kClsFC = 0, kClsFR = 1, kClsSmall = 2, kClsRng = 3, kClsTTM = 4, kClsResid = 5, kClsSweep = 6, kNumCls = 8 };

class Engine {
 public:
  explicit Engine(int device);
  ~Engine();

  // Decomposition drivers; `a` is host (a_dev false) or device memory.
  // want_sv: rotate each factor onto singular vectors (recover_singular_vectors)
  // engine: EngineKind (kEngineAls uses cfg)
  void t_hosvd(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
               const AlsCfg& cfg, double* core, double* factors, DecompRep* rep, bool want_sv = false,
               int engine = kEngineAls);
  void st_hosvd(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
                const std::vector<int>* order, const AlsCfg& cfg, double* core, double* factors,
                DecompRep* rep, int engine = kEngineAls);
  void als_low_rank(const double* a, bool a_dev, const Shape& sh, int mode, uint32_t r,
                    const AlsCfg& cfg, double* l_out, double* r_out, ModeRep* rep);
  void als_init(const double* a, bool a_dev, const Shape& sh, int mode, uint32_t r, uint64_t seed,
                double* l_out);
  // als_sweep (als.cpp:89-96): l (I x r, host) -> updated L, this sweep's R
  // (F x r, nullable) and the closed-form residual after the right update
  void als_sweep(const double* a, const Shape& sh, int mode, const double* l, uint32_t r, double* l_out,
                 double* r_out, double* residual);

  // Sharded drivers (engine_dist.cpp): `a` is this rank's slab [begin,
  // begin + len) of the last mode of the global shape G (shard_range split);
  // core / factors / report come back replicated on every rank.
  void set_comm(std::unique_ptr<Comm> c);
  bool has_comm() const { return comm_ != nullptr; }
  void t_hosvd_sharded(const double* a, bool a_dev, const Shape& G, uint64_t begin, uint64_t len,
                       const std::vector<uint64_t>& ranks, const AlsCfg& cfg, double* core, double* factors,
                       DecompRep* rep, bool want_sv = false);
  void st_hosvd_sharded(const double* a, bool a_dev, const Shape& G, uint64_t begin, uint64_t len,
                        const std::vector<uint64_t>& ranks, const std::vector<int>* order, const AlsCfg& cfg,
                        double* core, double* factors, DecompRep* rep);

  // Primitives (host in/out).
  void unfold_times(const double* a, const Shape& sh, int mode, const double* m, uint32_t r, double* out);
  void unfold_t_times(const double* a, const Shape& sh, int mode, const double* m, uint32_t r, double* out);
  void mode_n_product(const double* a, const Shape& sh, const double* u, uint64_t rows, uint64_t cols,
                      int mode, double* out);
  // multi_mode_product (tensor_ops.cpp:171-191): factor k is rows[k] x I_{modes[k]}
  // (host, column-major); returns the result's shape
  Shape multi_mode_product(const double* a, const Shape& sh, const std::vector<int>& modes,
                           const std::vector<const double*>& factors, const std::vector<uint64_t>& rows,
                           const std::vector<uint64_t>& cols, double* out);
  double frobenius_norm(const double* a, uint64_t n);
  double relative_error(const double* a, const double* b, uint64_t n);
  void reduced_qr(const double* a, uint64_t rows, uint64_t cols, double* q, double* r);
  void gram(const double* a, uint64_t rows, uint64_t cols, double* out);
  // hooi (hooi.cpp:53-110) from a warm start (init_core prod R_n, init_factors
  // concatenated I_n x R_n, host); results into core / factors (host).
  void hooi(const double* a, bool a_dev, const Shape& sh, const std::vector<uint64_t>& ranks,
            const double* init_core, const double* init_factors, double tol, int max_iters, double* core,
            double* factors, HooiRep* rep);
  // mode_gram (tensor_ops.cpp:332-389): out = A_(mode) A_(mode)^T, extent^2 doubles
  void mode_gram(const double* a, const Shape& sh, int mode, double* out);
  // sym_eig (kernels.cpp:448-604): g (n x n) -> k leading pairs (values, n x k vectors)
  void sym_eig(const double* g, uint64_t n, uint64_t k, double* values, double* vectors);
  // recover_singular_vectors (hosvd.cpp:65-72): q (I_mode x cols) -> q V
  void recover_singular_vectors(const double* a, const Shape& sh, int mode, const double* q, uint64_t rows,
                                uint64_t cols, double* out);
  void uniform01(uint64_t seed, uint32_t stream, uint64_t n, double* out);

  void bench_contractions(const double* dA, const Shape& sh, int mode, uint32_t r, int reps,
                          double* out_ms);
  int device() const { return device_; }
  void set_profiling(bool on) {
    if (on != profiling_) pdl_off_count() += on ? 1 : -1;
    profiling_ = on;
  }
  void force_v1(bool on) { force_v1_ = on; }
  // the fused sweep pass for r <= 16 (sweep_fused.cu): off unless switched on
  // here or by TKG_FUSED_SWEEP=1 (measured slower inside the decompositions)
  void set_fused_sweep(bool on) { fused_sweep_ = on; }
  void timer_start();
  double timer_stop();
  void flush_l2();
  void kernel_stats(double ms[kNumCls], uint64_t launches[kNumCls], double bytes[kNumCls], double flops[kNumCls]);
  const std::string& device_name() const { return name_; }
  cudaStream_t stream() const { return st_; }

 private:
  struct AlsOut {
    ModeRep rep;          // history filled by collect() after the next sync
    double norm = 0.0;
    const double* hist_host = nullptr;   // pinned staging, rep.iterations values
    const double* sumsq_host = nullptr;  // pinned staging: ||working tensor||^2
    // graph mode (device-side sweep loop): the staged control block, settled
    // by collect() after the final synchronisation
    const AlsCtrl* ctrl_host = nullptr;
    double fc_bytes = 0.0;
    int body_launches = 0;
    uint32_t r = 0;
    bool fused = false;   // sweeps ran as fused passes (one tensor pass per sweep)
  };
  // Host-visible results of the decomposition drivers are staged in pinned
  // memory with asynchronous copies and read after the driver's single final
  // synchronisation (one slot of max_iters + 1 doubles per mode), and the
  // per-mode times are CUDA events on the stream.
  void stage_reserve(int modes, int max_iters);
  void collect(AlsOut& o, ModeRep& dst);
  void settle(AlsOut& o);
  // device-side sweep loops (CUDA graph WHILE nodes), cached per operand set
  bool use_graph_loop() const;
  cudaGraphExec_t capture_sweep_loop(const std::function<void(GraphCond)>& body, int* body_launches);
  void clear_graphs();
  std::map<std::vector<uint64_t>, std::pair<cudaGraphExec_t, int>> graphs_;
  bool graph_failed_ = false;
  struct ResultCopy {
    void* dst;
    const void* src;
    size_t bytes;
  };
  void copy_results(const std::vector<ResultCopy>& outs, cudaStream_t s);
  void* out_stage_ = nullptr;  // pinned (results bound for pageable memory)
  size_t out_stage_n_ = 0;
  static constexpr int kMaxStageModes = 64;
  // t-HOSVD with device-side sweep loops: the modes are independent, so each
  // runs on its own stream with its own working buffers (a "lane"); the
  // engine's members are swapped with the lane's while that mode is enqueued.
  struct Lane {
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
    DBuf s, r, l, mt, gl, gr, cholL, cholR, fr_part, fc_gram, gram_part, gs, sq_part, qr_work;
    DBuf y_seq, states, chunk_ids, qrl1, qrl2, qrq1, sumsq_d, ctrl_d, hist_d, misc2;
  };
  std::vector<Lane*> lanes_;
  std::map<std::pair<uint64_t, uint32_t>, DBuf*> yseq_cache_;  // MT raw sequences per (seed, stream)
  cudaEvent_t sumsq_ev_ = nullptr;     // mode 1's ||A||^2 is ready (concurrent modes)
  bool record_sumsq_ = false;
  bool in_lanes_ = false;  // enqueuing a concurrent t-HOSVD mode
  const double* sumsq_from_ = nullptr;  // a concurrent mode copies ||A||^2 from here
  void swap_lane(Lane& L);
  bool concurrent_modes_ok(const std::vector<uint64_t>& ranks, bool want_sv) const;
  AlsCtrl* stage_ctrl_ = nullptr;  // pinned
  void mode_begin(int k);
  void mode_end(int k);
  double mode_seconds(int k);
  // Runs als_low_rank on a device-resident tensor; L (col-major I x r) is
  // left in l_, R (F x r) in r_. sumsq_known: status_->sumsq already holds
  // ||A||^2 of this tensor.
  AlsOut run_als(const double* A, const Shape& sh, int mode, uint32_t r, const AlsCfg& cfg,
                 bool sumsq_known, const MtWindow& win = MtWindow(), int slot = 0);
  // ranks above 64 (engine_wide.cpp): 64-column contraction blocks, Cholesky
  // + row substitutions for the r x r solves, one host read per sweep
  AlsOut run_als_wide(const double* A, const Shape& sh, int mode, uint32_t r, const AlsCfg& cfg,
                      bool sumsq_known, int slot);
  // CholQR2 of a column-major I x r matrix for r > 64 (Q may alias Y)
  void qr_wide(const double* Y, uint32_t I, uint32_t r, double* Q, double* rmat, bool check);
  // G (r x r) = X^T X of a row-major [rows][ld] or column-major (ld) matrix
  void gram_cols(const double* X, uint64_t rows, uint32_t r, uint64_t ld, bool row_major, double* G);
  uint32_t reduce_left_partials(double* part, uint32_t nparts, uint32_t I, uint32_t ncp, uint32_t r);
  // draws 0..n-1 in storage order, or a shard's window of them (MtWindow)
  void gen_uniform(uint64_t seed, uint32_t stream, uint64_t n, double* d_out, const MtWindow& win = MtWindow());
  static MtWindow s_window(MtWindow win, uint64_t F, uint64_t ld);
  void gen_uniform_on(uint64_t seed, uint32_t stream, uint64_t n, double* d_out, const MtWindow& win,
                      cudaStream_t st, DBuf& ybuf, DBuf& sbuf, DBuf& cbuf);
  struct PreGen {
    int mode;
    uint64_t F;  // local fibers
    uint32_t r;
    MtWindow win;
  };
  void pregenerate(const std::vector<PreGen>& items, uint64_t seed);
  // run by the first run_als of the decomposition after its init is queued
  void defer_pregenerate(const std::vector<PreGen>& items, uint64_t seed);
  std::vector<PreGen> pending_pre_;
  uint64_t pending_seed_ = 0;
  void fc(const FiberView& v, const double* mt, uint32_t ldmt, uint32_t nc, double* out,
          uint64_t os_j, uint64_t os_c, uint64_t os_p, double* sumsq_part,
          const double* diff_ref, int* grid_used, bool count_pass, const int32_t* skip = nullptr,
          double* gram_part = nullptr);
  // one sweep's R = A_(n)^T L', R^T R partials and left-update partials from
  // one read of the tensor (sweep_fused.cu); returns the CTAs launched
  int sweep_fused(const FiberView& v, const double* mt, uint32_t nc, double* R, double* partial,
                  double* gram_part, bool count_pass, const int32_t* skip);
  bool sweep_fused_usable(const FiberView& v, const double* mt, uint32_t nc, const double* R) const;
  int fc_grid(const FiberView& v, const double* mt, uint32_t ldmt, uint32_t nc);
  uint32_t fr_ranges(const FiberView& v, uint32_t nc);
  uint32_t fr(const FiberView& v, const double* m, uint64_t mj, uint64_t mc, uint32_t nc,
              double* partial, double* sumsq_part, bool count_pass, uint32_t* grid_used,
              const int32_t* skip = nullptr);
  void sync();
  void qr_dev(const double* Y, int nparts, uint64_t ld, uint32_t I, uint32_t r, double* Q,
              double* rmat, double* rt, uint32_t ldrt, bool check);
  int qr_degenerate_col();
  // recover_singular_vectors on a device-resident tensor: U (I x r, device,
  // col-major) <- U V; leaves R = A_(n)^T U_old in r_ (row-major [F][ncp])
  // and V^T (r x r, col-major) in vt. Sums the Gram over ranks when dist_.
  void recover_sv(const double* A, const Shape& sh, int mode, uint32_t r, double* U, double* vt);
  void mode_product_dev(const double* X, const Shape& sh, int mode, const double* U, uint64_t rows, double* dst);
  void recover_sv_round(const double* A, const Shape& sh, int mode, uint32_t r, double* U, double* vt);
  // SVD / EIG engines: U (device, I x r) <- leading eigenvectors of A_(n) A_(n)^T
  void gram_factor(const double* A, const Shape& sh, int mode, uint32_t r, double* U, bool refine);
  static constexpr double kClosedFormMinRel = 5e-5;
  bool closed_form_residual(const double* core_buf, uint64_t ncore, const double* ref_sumsq_host, double* rel);
  // dst <- A x_m U_m^T for every m != skip, ascending (multi_mode_product with
  // the other factors, hooi.cpp:82-88); returns dst's shape
  Shape ttm_others(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                   const std::vector<double*>& U, int skip, double* dst);
  // out <- X x_mode U^T (U: I x r device col-major), tensor layout, any r
  void ttm_mode(const double* X, const Shape& sh, int mode, const double* U, uint32_t r, double* out,
                bool count_pass = false);
  double* sumsq_to_host(const double* A, uint64_t n);  // ||A||^2 staged in pinned memory (after sync)
  void finish_exact(const Shape& sh, const std::vector<uint64_t>& ranks, const Shape& cs, const double* A,
                    const double* core_buf, const std::vector<double*>& U, const double* ref_sumsq, double* core,
                    double* factors, DecompRep* rep, std::chrono::steady_clock::time_point t0,
                    const std::vector<int>* order);
  const double* upload(const double* a, uint64_t n, bool a_dev, DBuf& buf, double* seconds);
  // ref_sumsq_host: pinned ||A||^2, read after the function's own sync
  double relative_residual_dev(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                               const double* d_core, const std::vector<double*>& d_factors,
                               const double* ref_sumsq_host);
  // the same split: expansion kernels + difference norm on st_ (returns the
  // device scalar), then the synchronising read
  double* residual_enqueue(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                           const double* d_core, const std::vector<double*>& d_factors);
  double residual_read(const double* d_diff_sq, const double* ref_sumsq_host);
  void outputs_and_residual(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks, const Shape& cs,
                            const double* core_buf, const std::vector<double*>& U, const double* ref_sumsq,
                            double* core, double* factors, DecompRep* rep);
  // TTMs of modes 1..last_mode (0 = all) with U_n^T, ascending (hosvd.cpp:115-121)
  void core_chain(const double* A, const Shape& sh, const std::vector<uint64_t>& ranks,
                  const std::vector<double*>& d_factors, double* d_core, int last_mode = 0);
  void begin_timed();
  void count_launch(int n = 1) { launches_ += n; }
  void reshard(const double* src, const Shape& G, int from, int to, double* dst);
  void reshard_on(const double* src, const Shape& G, int from, int to, double* dst, cudaStream_t st, Comm* comm);
  // Cooperative (grid.sync) launches. Ranks of an in-process group share one
  // device: two partially resident cooperative grids could wait on each
  // other, so there they run one at a time (process-wide lock, synchronised).
  template <class F>
  void coop_launch(F&& launch) {
    if (comm_ && comm_->shares_device()) {
      std::lock_guard<std::mutex> g(coop_mutex());
      launch();
      check_cuda(cudaStreamSynchronize(st_), "coop sync");
    } else {
      launch();
    }
  }
  static std::mutex& coop_mutex();
  void check_shard(const Shape& G, uint64_t begin, uint64_t len);
  void dist_core_and_residual(const double* A, const Shape& L, uint64_t k0, const Shape& G,
                              const std::vector<uint64_t>& ranks, std::vector<double*>& U, double* core_buf,
                              bool compute_core, std::vector<AlsOut>& outs, DecompRep* rep, double* core_host,
                              double* factors_host, std::chrono::steady_clock::time_point t0);
  std::pair<cudaEvent_t, cudaEvent_t> small_begin();
  void small_end(std::pair<cudaEvent_t, cudaEvent_t> ev);
  void record(int cls, cudaEvent_t a, cudaEvent_t b, double bytes, double flops);
  std::pair<cudaEvent_t, cudaEvent_t> ev_pair();

  int device_;
  int sms_;
  std::string name_;
  cudaStream_t st_;
  cudaStream_t st2_;  // low-priority side stream for the initializer streams
  cudaEvent_t pre_gate_;
  cudaStream_t cp_st_;      // result copies (overlap the residual expansion)
  cudaEvent_t out_ready_;
  struct PreS {
    double* ptr;
    cudaEvent_t ready;
    uint64_t F;
    uint32_t r;
  };
  std::map<int, PreS> pre_;
  std::vector<DBuf*> pre_bufs_, pre_y_, pre_st_, pre_ids_;
  std::vector<cudaEvent_t> pre_ev_;
  DevStatus* status_h_ = nullptr;
  DevStatus* status_d_ = nullptr;

  DBuf tensor_, work_a_, work_b_, s_, r_, l_, mt_, gl_, gr_, cholL_, cholR_;
  DBuf fr_part_, fc_gram_, gram_part_, gs_, sq_part_, qr_work_, q_, rhat_, rhatT_;
  DBuf y_seq_, states_, chunk_ids_, misc_, misc2_, flush_, qy_, qrl1_, qrl2_, qrq1_, sumsq_d_, ctrl_d_, hist_d_;
  double* stage_h_ = nullptr;  // pinned
  size_t stage_n_ = 0;
  int stage_iters_ = 0;
  std::vector<cudaEvent_t> mode_ev_;
  cudaEvent_t t0_ = nullptr, t1_ = nullptr;
  std::vector<DBuf*> factor_bufs_;
  std::map<std::pair<uint64_t, int>, DBuf*> jump_cache_;

  bool profiling_ = false;
  bool force_v1_ = false;
  bool fused_sweep_ = [] {
    const char* e = std::getenv("TKG_FUSED_SWEEP");
    return e != nullptr && e[0] == '1';
  }();
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double bytes, flops;
  };
  std::vector<Rec> recs_;
  struct SpecRec {
    int k;       // sweep (1-based)
    int kind;    // 0 FC (right update), 1 FR (left update)
    size_t rec;  // index into recs_
  };
  std::vector<SpecRec> spec_recs_;
  std::vector<cudaEvent_t> ev_pool_;
  double stat_ms_[kNumCls] = {0};
  uint64_t stat_launch_[kNumCls] = {0};
  double stat_bytes_[kNumCls] = {0};
  double stat_flops_[kNumCls] = {0};
  int fc_cls_ = kClsFC;  // class recorded for fc() launches (kClsTTM outside the ALS loop)
  struct ClsScope {
    int& ref;
    int old;
    ClsScope(int& r, int c) : ref(r), old(r) { ref = c; }
    ~ClsScope() { ref = old; }
  };

  uint64_t launches_ = 0;
  uint64_t passes_ = 0;
  uint64_t bytes_ = 0;

  std::unique_ptr<Comm> comm_;
  std::unique_ptr<Comm> comm2_;  // second communicator (overlapped reshard), from comm_->split()
  bool comm2_tried_ = false;
  cudaStream_t cm_st_ = nullptr;
  cudaEvent_t cm_ev_a_ = nullptr, cm_ev_b_ = nullptr;
  Comm* dist_ = nullptr;  // set while a sharded driver runs: run_als sums over ranks
  DBuf send_, recv_, reshard_, uslab_, uslab2_, core_t_;
  DBuf sv_u_, sv_g_, sv_vt_, sv_vt0_, sv_ctrl_;
  DBuf gram_t_, gram_t_part_, gram_w_, hooi_s_;
  DBuf wide_gpart_, wide_g_, wide_c1_, wide_c2_, wide_fail_, wide_lp_;
  SymEig eig_;
  double* norm_h_ = nullptr;  // pinned
};

struct ShardRange {
  uint64_t begin = 0, len = 0;
};
// balanced split of `extent` over `world` ranks
ShardRange shard_range(uint64_t extent, int rank, int world);
std::vector<int> checked_order(const Shape& sh, const std::vector<uint64_t>& ranks, const std::vector<int>* order);

std::vector<int> select_order(const std::vector<uint64_t>& ranks);
void validate_truncation(const Shape& sh, const std::vector<uint64_t>& ranks);

}  // namespace tkg
