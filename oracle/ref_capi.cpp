// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI wrapper around the UNMODIFIED reference library (tenkit, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load this, and only as the checker or the timed CPU
// baseline. Nothing under paper_2004_02583_b200/ links or calls it.
//
// Conventions: tensors are flat column-major doubles (tensor.hpp:10-11),
// matrices column-major (matrix.hpp:8-9), modes 1-based (shape.hpp:10-14).
// Return 0 on success, else ErrorCategory+1 (errors.hpp:10; CLI exit codes
// tenkit_main.cpp:644-664) with *subtype naming the exception class.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "tenkit/als.hpp"
#include "tenkit/errors.hpp"
#include "tenkit/hooi.hpp"
#include "tenkit/io.hpp"
#include "tenkit/hosvd.hpp"
#include "tenkit/kernels.hpp"
#include "tenkit/matrix.hpp"
#include "tenkit/parallel.hpp"
#include "tenkit/reference.hpp"
#include "tenkit/rng.hpp"
#include "tenkit/tensor.hpp"
#include "tenkit/tensor_ops.hpp"

using namespace tenkit;

namespace {

enum Subtype {
  kOk = 0, kInvalidMode = 1, kDimensionMismatch = 2, kZeroReference = 3,
  kRankTooLarge = 4, kSingularGram = 5, kDegenerateInit = 6,
  kNoConvergence = 7, kIo = 8, kFormat = 9, kOther = 10
};

struct ErrSink { int* subtype; char* msg; int len; };

void put(ErrSink e, int st, const char* m) {
  if (e.subtype) *e.subtype = st;
  if (e.msg && e.len > 0) {
    std::strncpy(e.msg, m, static_cast<size_t>(e.len) - 1);
    e.msg[e.len - 1] = '\0';
  }
}

template <class F>
int guarded(ErrSink e, F&& f) {
  try {
    f();
    put(e, kOk, "");
    return 0;
  } catch (const InvalidModeError& x) { put(e, kInvalidMode, x.what()); return 1; }
  catch (const DimensionMismatchError& x) { put(e, kDimensionMismatch, x.what()); return 1; }
  catch (const ZeroReferenceError& x) { put(e, kZeroReference, x.what()); return 1; }
  catch (const RankTooLargeError& x) { put(e, kRankTooLarge, x.what()); return 3; }
  catch (const SingularGramError& x) { put(e, kSingularGram, x.what()); return 3; }
  catch (const DegenerateInitError& x) { put(e, kDegenerateInit, x.what()); return 3; }
  catch (const NoConvergenceError& x) { put(e, kNoConvergence, x.what()); return 3; }
  catch (const Error& x) {
    put(e, kOther, x.what());
    return static_cast<int>(x.category()) + 1;
  } catch (const std::exception& x) { put(e, kOther, x.what()); return 1; }
}

DenseTensor make_tensor(const double* a, int order, const uint64_t* dims) {
  std::vector<std::size_t> d(dims, dims + order);
  Shape s(d);
  return DenseTensor(s, std::vector<double>(a, a + s.element_count()));
}

Matrix make_matrix(const double* m, uint64_t rows, uint64_t cols) {
  return Matrix(rows, cols, std::vector<double>(m, m + rows * cols));
}

void copy_out(const Matrix& m, double* out) {
  if (out) std::copy(m.values().begin(), m.values().end(), out);
}

void copy_out(const DenseTensor& t, double* out) {
  if (out) std::copy(t.values().begin(), t.values().end(), out);
}

// Per-mode report flattened for the C side. Arrays are indexed by
// processing position (hosvd.hpp:33-44: per_mode is in processing order).
struct RefReport {
  int32_t modes[64];
  int32_t iterations[64];
  int32_t status[64];            // 0 converged, 1 max iters (als.hpp:25)
  double achieved_eta[64];
  double mode_seconds[64];
  double residual_history[64][64];  // first min(iterations,64) entries
  double seconds;
  double relative_residual;
};

void fill_report(const DecompositionReport& rep, RefReport* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  for (std::size_t k = 0; k < rep.per_mode.size() && k < 64; ++k) {
    const ModeReport& mr = rep.per_mode[k];
    out->modes[k] = static_cast<int32_t>(mr.mode);
    out->mode_seconds[k] = mr.seconds;
    if (mr.als) {
      out->iterations[k] = mr.als->iterations;
      out->status[k] = mr.als->status == AlsStatus::kConverged ? 0 : 1;
      out->achieved_eta[k] = mr.als->achieved_eta;
      for (std::size_t h = 0; h < mr.als->residual_history.size() && h < 64; ++h) {
        out->residual_history[k][h] = mr.als->residual_history[h];
      }
    }
  }
  out->seconds = rep.seconds;
  out->relative_residual = rep.relative_residual;
}

}  // namespace

extern "C" {

int ref_report_size() { return static_cast<int>(sizeof(RefReport)); }

void ref_set_threads(int n) { set_threads(n); }
int ref_max_threads() { return max_threads(); }

// rng.hpp:19-21,57-61 — n successive uniform01 draws of seeded_engine(seed, stream).
void ref_uniform01(uint64_t seed, uint32_t stream, uint64_t n, double* out) {
  std::mt19937_64 eng = seeded_engine(seed, stream);
  for (uint64_t i = 0; i < n; ++i) out[i] = uniform01(eng);
}

// Raw 64-bit engine outputs (for pinning the MT19937-64 restatements).
void ref_engine_raw(uint64_t seed, uint32_t stream, uint64_t n, uint64_t* out) {
  std::mt19937_64 eng = seeded_engine(seed, stream);
  for (uint64_t i = 0; i < n; ++i) out[i] = eng();
}

// tests/helpers.hpp:34-41 random_tensor: uniform_in(-1,1) in storage order.
void ref_uniform_in(uint64_t seed, uint32_t stream, double lo, double hi,
                    uint64_t n, double* out) {
  std::mt19937_64 eng = seeded_engine(seed, stream);
  for (uint64_t i = 0; i < n; ++i) out[i] = uniform_in(eng, lo, hi);
}

// rng.hpp:30-53 GaussianStream.
void ref_gaussian(uint64_t seed, uint32_t stream, uint64_t n, double* out) {
  std::mt19937_64 eng = seeded_engine(seed, stream);
  GaussianStream g(eng);
  for (uint64_t i = 0; i < n; ++i) out[i] = g.next();
}

int ref_unfold_times(const double* a, int order, const uint64_t* dims,
                     uint32_t mode, const double* m, uint64_t r, double* out,
                     int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    std::size_t fibers = t.size() / t.shape().extent(mode);
    copy_out(unfold_times(t, mode, make_matrix(m, fibers, r)), out);
  });
}

int ref_unfold_t_times(const double* a, int order, const uint64_t* dims,
                       uint32_t mode, const double* m, uint64_t r, double* out,
                       int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    std::size_t extent = t.shape().extent(mode);
    copy_out(unfold_t_times(t, mode, make_matrix(m, extent, r)), out);
  });
}

// mode_n_product with u given as rows x cols (cols == extent of mode).
int ref_mode_n_product(const double* a, int order, const uint64_t* dims,
                       const double* u, uint64_t rows, uint64_t cols,
                       uint32_t mode, double* out, int* subtype, char* msg,
                       int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    copy_out(mode_n_product(t, make_matrix(u, rows, cols), mode), out);
  });
}

int ref_frobenius_norm(const double* a, int order, const uint64_t* dims,
                       double* out, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    *out = frobenius_norm(make_tensor(a, order, dims));
  });
}

int ref_relative_error(const double* a, const double* b, int order,
                       const uint64_t* dims, double* out, int* subtype,
                       char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    *out = relative_error(make_tensor(a, order, dims), make_tensor(b, order, dims));
  });
}

int ref_reduced_qr(const double* a, uint64_t rows, uint64_t cols, double* q,
                   double* r, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    QrFactors f = reduced_qr(make_matrix(a, rows, cols));
    copy_out(f.q, q);
    copy_out(f.r_upper, r);
  });
}

int ref_spd_solve(const double* g, uint64_t n, const double* b, uint64_t k,
                  double* x, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    copy_out(spd_solve(make_matrix(g, n, n), make_matrix(b, n, k)), x);
  });
}

int ref_gram(const double* a, uint64_t rows, uint64_t cols, double* out,
             int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] { copy_out(gram(make_matrix(a, rows, cols)), out); });
}

int ref_dense_svd_values(const double* a, uint64_t rows, uint64_t cols,
                         double* values, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    SpectrumReport sr = dense_svd(make_matrix(a, rows, cols), false);
    std::copy(sr.values.begin(), sr.values.end(), values);
  });
}

int ref_als_init(const double* a, int order, const uint64_t* dims,
                 uint32_t mode, uint64_t r, uint64_t seed, double* l_out,
                 int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    copy_out(als_init(make_tensor(a, order, dims), mode, r, seed), l_out);
  });
}

// als_sweep (als.cpp:89-96): returns the next l, the in-sweep r and residual.
int ref_als_sweep(const double* a, int order, const uint64_t* dims,
                  uint32_t mode, const double* l, uint64_t r, double* l_next,
                  double* r_out, double* residual, int* subtype, char* msg,
                  int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    auto [pair, res] = als_sweep(t, mode, make_matrix(l, t.shape().extent(mode), r));
    copy_out(pair.l, l_next);
    copy_out(pair.r, r_out);
    *residual = res;
  });
}

int ref_als_low_rank(const double* a, int order, const uint64_t* dims,
                     uint32_t mode, uint64_t r, double eta, int max_iters,
                     uint64_t seed, const double* init, double* l_out,
                     double* r_out, int* iterations, int* status,
                     double* achieved_eta, double* history, int history_cap,
                     int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    AlsConfig cfg;
    cfg.eta = eta;
    cfg.max_iters = max_iters;
    cfg.seed = seed;
    if (init) cfg.init = make_matrix(init, t.shape().extent(mode), r);
    auto [pair, rep] = als_low_rank(t, mode, r, cfg);
    copy_out(pair.l, l_out);
    copy_out(pair.r, r_out);
    *iterations = rep.iterations;
    *status = rep.status == AlsStatus::kConverged ? 0 : 1;
    *achieved_eta = rep.achieved_eta;
    for (int h = 0; h < history_cap && h < static_cast<int>(rep.residual_history.size()); ++h) {
      history[h] = rep.residual_history[h];
    }
  });
}

int ref_select_order(int order, const uint64_t* dims, const uint64_t* ranks,
                     uint32_t* out, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    Truncation tr{std::vector<std::size_t>(ranks, ranks + order)};
    ModeOrder o = select_order(tr, Shape(std::vector<std::size_t>(dims, dims + order)));
    for (int k = 0; k < order; ++k) out[k] = static_cast<uint32_t>(o.order[k]);
  });
}

// recover_singular_vectors (hosvd.cpp:65-72), q rows x cols.
int ref_recover_singular_vectors(const double* a, int order, const uint64_t* dims,
                                 uint32_t mode, const double* q, uint64_t rows,
                                 uint64_t cols, double* out, int* subtype, char* msg,
                                 int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    copy_out(recover_singular_vectors(t, mode, make_matrix(q, rows, cols)), out);
  });
}

// t_hosvd / st_hosvd with the ALS engine (hosvd.cpp:74-191). factors_out
// receives the factors concatenated in mode order (I_n x R_n each).
// mode_order: nullable (st only; nullptr = select_order).
// sequential: 0 t_hosvd, 1 st_hosvd, 2 t_hosvd(want_singular_vectors = true).
int ref_hosvd_als(int sequential, const double* a, int order,
                  const uint64_t* dims, const uint64_t* ranks,
                  const uint32_t* mode_order, double eta, int max_iters,
                  uint64_t seed, double* core_out, double* factors_out,
                  void* report, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    Truncation tr{std::vector<std::size_t>(ranks, ranks + order)};
    AlsConfig cfg;
    cfg.eta = eta;
    cfg.max_iters = max_iters;
    cfg.seed = seed;
    FactorEngine eng = FactorEngine::with_als(cfg);
    std::pair<TuckerTensor, DecompositionReport> res =
        sequential == 1
            ? st_hosvd(t, tr,
                       mode_order ? std::optional<ModeOrder>(ModeOrder{
                                        std::vector<std::size_t>(mode_order, mode_order + order)})
                                  : std::nullopt,
                       eng)
            : t_hosvd(t, tr, eng, sequential == 2);
    copy_out(res.first.core, core_out);
    if (factors_out) {
      double* p = factors_out;
      for (const Matrix& u : res.first.factors) {
        std::copy(u.values().begin(), u.values().end(), p);
        p += u.values().size();
      }
    }
    fill_report(res.second, static_cast<RefReport*>(report));
  });
}

// The same decomposition on a tensor read from a TNSR file by the
// reference's own read_tnsr (io.cpp:150-161), so the calling process never
// synthesises or copies the tensor itself (tools/parity_full.py, bench.py's
// reference arm). dims_out receives the file's extents (order <= 64);
// call_seconds the wall time of the t_hosvd / st_hosvd call alone (reading
// excluded; the relative residual, which the API computes, included).
int ref_hosvd_als_tnsr(int sequential, const char* path, const uint64_t* ranks,
                       const uint32_t* mode_order, double eta, int max_iters,
                       uint64_t seed, double* core_out, double* factors_out,
                       void* report, uint64_t* dims_out, double* call_seconds,
                       int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = read_tnsr(std::string(path));
    const std::size_t order = t.shape().order();
    for (std::size_t k = 1; k <= order; ++k) dims_out[k - 1] = t.shape().extent(k);
    Truncation tr{std::vector<std::size_t>(ranks, ranks + order)};
    AlsConfig cfg;
    cfg.eta = eta;
    cfg.max_iters = max_iters;
    cfg.seed = seed;
    FactorEngine eng = FactorEngine::with_als(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    std::pair<TuckerTensor, DecompositionReport> res =
        sequential == 1
            ? st_hosvd(t, tr,
                       mode_order ? std::optional<ModeOrder>(ModeOrder{
                                        std::vector<std::size_t>(mode_order, mode_order + order)})
                                  : std::nullopt,
                       eng)
            : t_hosvd(t, tr, eng, sequential == 2);
    *call_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    copy_out(res.first.core, core_out);
    if (factors_out) {
      double* p = factors_out;
      for (const Matrix& u : res.first.factors) {
        std::copy(u.values().begin(), u.values().end(), p);
        p += u.values().size();
      }
    }
    fill_report(res.second, static_cast<RefReport*>(report));
  });
}

// t_hosvd / st_hosvd with the SVD (kind 0) or EIG (kind 1) engine
// (hosvd.cpp:89-99, 151-171); same buffers as ref_hosvd_als.
int ref_hosvd_exact(int sequential, int kind, const double* a, int order,
                    const uint64_t* dims, const uint64_t* ranks,
                    const uint32_t* mode_order, double* core_out, double* factors_out,
                    void* report, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    Truncation tr{std::vector<std::size_t>(ranks, ranks + order)};
    FactorEngine eng = kind == 0 ? FactorEngine::svd() : FactorEngine::eig();
    std::pair<TuckerTensor, DecompositionReport> res =
        sequential
            ? st_hosvd(t, tr,
                       mode_order ? std::optional<ModeOrder>(ModeOrder{
                                        std::vector<std::size_t>(mode_order, mode_order + order)})
                                  : std::nullopt,
                       eng)
            : t_hosvd(t, tr, eng);
    copy_out(res.first.core, core_out);
    double* p = factors_out;
    for (const Matrix& u : res.first.factors) {
      std::copy(u.values().begin(), u.values().end(), p);
      p += u.values().size();
    }
    fill_report(res.second, static_cast<RefReport*>(report));
  });
}

// hooi (hooi.cpp:53-110) from a warm start (core prod R_n, factors
// concatenated I_n x R_n); fit_history capacity max(1, max_iters) + 1.
int ref_hooi(const double* a, int order, const uint64_t* dims, const uint64_t* ranks,
             const double* init_core, const double* init_factors, double tol, int max_iters,
             double* core_out, double* factors_out, int* iterations, int* converged,
             double* fit_history, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = make_tensor(a, order, dims);
    Truncation tr{std::vector<std::size_t>(ranks, ranks + order)};
    TuckerTensor init{make_tensor(init_core, order, ranks), {}, t.shape()};
    const double* p = init_factors;
    for (int n = 0; n < order; ++n) {
      init.factors.push_back(make_matrix(p, dims[n], ranks[n]));
      p += dims[n] * ranks[n];
    }
    HooiConfig cfg;
    cfg.tol = tol;
    cfg.max_iters = max_iters;
    HooiResult res = hooi(t, tr, init, cfg);
    copy_out(res.tucker.core, core_out);
    double* q = factors_out;
    for (const Matrix& u : res.tucker.factors) {
      std::copy(u.values().begin(), u.values().end(), q);
      q += u.values().size();
    }
    *iterations = res.iterations;
    *converged = res.converged ? 1 : 0;
    std::copy(res.fit_history.begin(), res.fit_history.end(), fit_history);
  });
}

// read_tnsr / write_tnsr / read_tukr (io.cpp:131-224): format pins.
int ref_write_tnsr(const char* path, const double* a, int order, const uint64_t* dims,
                   int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] { write_tnsr(std::string(path), make_tensor(a, order, dims)); });
}

int ref_read_tnsr(const char* path, int* order, uint64_t* dims, double* out, uint64_t cap,
                  int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    DenseTensor t = read_tnsr(std::string(path));
    *order = static_cast<int>(t.shape().order());
    for (std::size_t k = 1; k <= t.shape().order(); ++k) dims[k - 1] = t.shape().extent(k);
    if (out && t.size() <= cap) copy_out(t, out);
  });
}

// core (prod ranks) then factors concatenated; ranks read from the file.
int ref_read_tukr(const char* path, int* order, uint64_t* dims, uint64_t* ranks, double* core,
                  double* factors, uint64_t cap, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    TuckerTensor tk = read_tukr(std::string(path));
    const std::size_t n = tk.origin_shape.order();
    *order = static_cast<int>(n);
    uint64_t need = tk.core.size();
    for (std::size_t k = 1; k <= n; ++k) {
      dims[k - 1] = tk.origin_shape.extent(k);
      ranks[k - 1] = tk.core.shape().extent(k);
      need += dims[k - 1] * ranks[k - 1];
    }
    if (!core || need > cap) return;
    copy_out(tk.core, core);
    double* p = factors;
    for (const Matrix& u : tk.factors) {
      std::copy(u.values().begin(), u.values().end(), p);
      p += u.values().size();
    }
  });
}

// mode_gram (tensor_ops.cpp:332-389), extent x extent.
int ref_mode_gram(const double* a, int order, const uint64_t* dims, uint32_t mode,
                  double* out, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    copy_out(mode_gram(make_tensor(a, order, dims), mode), out);
  });
}

// sym_eig (kernels.cpp:448-604): k leading pairs.
int ref_sym_eig(const double* g, uint64_t n, uint64_t k, double* values,
                double* vectors, int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    SpectrumReport sr = sym_eig(make_matrix(g, n, n), k);
    std::copy(sr.values.begin(), sr.values.end(), values);
    copy_out(*sr.left_vectors, vectors);
  });
}

// reconstruct (tensor_ops.cpp:420-440) from a core and concatenated factors.
int ref_reconstruct(const double* core, int order, const uint64_t* ranks,
                    const uint64_t* dims, const double* factors, double* out,
                    int* subtype, char* msg, int len) {
  return guarded({subtype, msg, len}, [&] {
    TuckerTensor tk{make_tensor(core, order, ranks), {},
                    Shape(std::vector<std::size_t>(dims, dims + order))};
    const double* p = factors;
    for (int n = 0; n < order; ++n) {
      tk.factors.push_back(make_matrix(p, dims[n], ranks[n]));
      p += dims[n] * ranks[n];
    }
    copy_out(reconstruct(tk), out);
  });
}

}  // extern "C"
