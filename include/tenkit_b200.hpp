// Header-only C++ shim over the C-ABI (tenkit_b200.h) that re-exposes the
// reference decomposition API (include/tenkit/hosvd.hpp:55-70,
// include/tenkit/als.hpp:69-71) on the B200 path.
//
// Two modes:
//  * default: self-contained value types (std::vector storage, column-major)
//    and an exception hierarchy mirroring tenkit/errors.hpp;
//  * with TENKIT_B200_USE_TENKIT defined before inclusion and the reference's
//    headers on the include path: the functions take and return the
//    reference's own DenseTensor / Truncation / FactorEngine / TuckerTensor /
//    DecompositionReport and throw the reference's exception classes, so a
//    caller switches engines by changing one namespace
//    (tenkit::t_hosvd -> tenkit_b200::t_hosvd). See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tenkit_b200.h"

#ifdef TENKIT_B200_USE_TENKIT
#include "tenkit/als.hpp"
#include "tenkit/errors.hpp"
#include "tenkit/hooi.hpp"
#include "tenkit/hosvd.hpp"
#include "tenkit/tensor_ops.hpp"
#endif

namespace tenkit_b200 {

#ifdef TENKIT_B200_USE_TENKIT
[[noreturn]] inline void rethrow(const tkg_error& e) {
  const std::string m = e.message;
  switch (e.subtype) {
    case TKG_E_INVALID_MODE: throw tenkit::InvalidModeError(m);
    case TKG_E_DIMENSION_MISMATCH: throw tenkit::DimensionMismatchError(m);
    case TKG_E_ZERO_REFERENCE: throw tenkit::ZeroReferenceError(m);
    case TKG_E_RANK_TOO_LARGE: throw tenkit::RankTooLargeError(m);
    case TKG_E_SINGULAR_GRAM: throw tenkit::SingularGramError(m);
    case TKG_E_DEGENERATE_INIT: throw tenkit::DegenerateInitError(m);
    case TKG_E_NO_CONVERGENCE: throw tenkit::NoConvergenceError(m);
    case TKG_E_IO: throw tenkit::IoError(m);
    case TKG_E_FORMAT: throw tenkit::FormatError(m);
    case TKG_E_CUDA: throw tenkit::IoError(m);
    default: throw tenkit::DimensionMismatchError(m);
  }
}
#else
// Mirrors tenkit/errors.hpp:10-77 (category: 0 usage, 1 io, 2 numerical).
struct Error : std::runtime_error {
  int category;
  Error(int cat, const std::string& m) : std::runtime_error(m), category(cat) {}
};
#define TENKIT_B200_ERR(Name, Cat) \
  struct Name : Error {            \
    explicit Name(const std::string& m) : Error(Cat, m) {} \
  };
TENKIT_B200_ERR(InvalidModeError, 0)
TENKIT_B200_ERR(DimensionMismatchError, 0)
TENKIT_B200_ERR(ZeroReferenceError, 0)
TENKIT_B200_ERR(RankTooLargeError, 2)
TENKIT_B200_ERR(SingularGramError, 2)
TENKIT_B200_ERR(DegenerateInitError, 2)
TENKIT_B200_ERR(NoConvergenceError, 2)
TENKIT_B200_ERR(IoError, 1)
TENKIT_B200_ERR(FormatError, 1)
#undef TENKIT_B200_ERR

[[noreturn]] inline void rethrow(const tkg_error& e) {
  const std::string m = e.message;
  switch (e.subtype) {
    case TKG_E_INVALID_MODE: throw InvalidModeError(m);
    case TKG_E_DIMENSION_MISMATCH: throw DimensionMismatchError(m);
    case TKG_E_ZERO_REFERENCE: throw ZeroReferenceError(m);
    case TKG_E_RANK_TOO_LARGE: throw RankTooLargeError(m);
    case TKG_E_SINGULAR_GRAM: throw SingularGramError(m);
    case TKG_E_DEGENERATE_INIT: throw DegenerateInitError(m);
    case TKG_E_NO_CONVERGENCE: throw NoConvergenceError(m);
    case TKG_E_IO: case TKG_E_CUDA: throw IoError(m);
    case TKG_E_FORMAT: throw FormatError(m);
    default: throw DimensionMismatchError(m);
  }
}
#endif

inline void check(int rc, const tkg_error& e) {
  if (rc != 0) rethrow(e);
}

// One device context (tkg_ctx); not thread-safe, like the reference's
// one-decomposition-per-process contract.
class Context {
 public:
  explicit Context(int device = 0) {
    tkg_error e{};
    check(tkg_create(&ctx_, device, &e), e);
  }
  ~Context() { tkg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tkg_ctx* get() const { return ctx_; }

  static Context& default_context() {
    static Context c(0);
    return c;
  }

 private:
  tkg_ctx* ctx_ = nullptr;
};

// Self-contained result types (column-major storage as the reference).
struct Tucker {
  std::vector<double> core;                  // prod R_n
  std::vector<std::vector<double>> factors;  // I_n x R_n each
  std::vector<uint64_t> dims, ranks;
};

struct Options {
  double eta = 1e-4;  // AlsConfig defaults (als.hpp:17-23)
  int max_iters = 50;
  uint64_t seed = 0;
  int kind = TKG_ENGINE_ALS;  // FactorEngine::Kind (hosvd.hpp:19-27)
};

inline Tucker hosvd_raw(Context& ctx, bool sequential, const double* a, bool a_on_device,
                        const std::vector<uint64_t>& dims, const std::vector<uint64_t>& ranks,
                        const Options& opt, const std::vector<uint32_t>* order, tkg_report* rep,
                        bool want_singular_vectors = false) {
  Tucker t;
  t.dims = dims;
  t.ranks = ranks;
  uint64_t core = 1, fac = 0;
  for (size_t k = 0; k < ranks.size() && k < dims.size(); ++k) {
    core *= ranks[k];
    fac += dims[k] * ranks[k];
  }
  t.core.assign(core, 0.0);
  std::vector<double> flat(fac ? fac : 1, 0.0);
  tkg_factor_engine cfg{opt.kind, {opt.eta, opt.max_iters, opt.seed, nullptr}};
  tkg_error e{};
  int rc;
  if (ranks.size() != dims.size()) {
    e.subtype = TKG_E_DIMENSION_MISMATCH;
    std::snprintf(e.message, sizeof(e.message), "truncation lists %zu ranks for an order-%zu tensor",
                  ranks.size(), dims.size());
    rethrow(e);
  }
  if (sequential)
    rc = tkg_st_hosvd_engine(ctx.get(), a, a_on_device, int32_t(dims.size()), dims.data(), ranks.data(),
                             order ? order->data() : nullptr, &cfg, t.core.data(), flat.data(), rep, &e);
  else
    rc = tkg_t_hosvd_engine(ctx.get(), a, a_on_device, int32_t(dims.size()), dims.data(), ranks.data(), &cfg,
                            want_singular_vectors ? 1 : 0, t.core.data(), flat.data(), rep, &e);
  check(rc, e);
  uint64_t ofs = 0;
  for (size_t k = 0; k < dims.size(); ++k) {
    t.factors.emplace_back(flat.begin() + ofs, flat.begin() + ofs + dims[k] * ranks[k]);
    ofs += dims[k] * ranks[k];
  }
  return t;
}

#ifdef TENKIT_B200_USE_TENKIT
// Drop-in signatures of hosvd.hpp:55-70 for FactorEngine::Kind::kAls.
// One entry per sweep (als.cpp:137-138): the report carries the first
// TKG_MAX_HISTORY inline, the rest comes from tkg_residual_history.
inline std::vector<double> full_history(tkg_ctx* ctx, int position, const tkg_mode_report& m) {
  std::vector<double> h(m.residual_history, m.residual_history + m.history_len);
  if (m.iterations > m.history_len) {
    h.assign(std::size_t(m.iterations), 0.0);
    uint64_t len = 0;
    tkg_error e{};
    check(tkg_residual_history(ctx, position, h.data(), h.size(), &len, &e), e);
    h.resize(std::size_t(len));
  }
  return h;
}

inline tenkit::DecompositionReport to_report(tkg_ctx* ctx, const tkg_report& r) {
  tenkit::DecompositionReport out;
  for (int k = 0; k < r.n_modes; ++k) {
    const tkg_mode_report& m = r.per_mode[k];
    tenkit::ModeReport mr;
    mr.mode = std::size_t(m.mode);
    mr.seconds = m.seconds;
    if (m.status < 0) {  // SVD / EIG engine: no ALS report
      out.per_mode.push_back(mr);
      continue;
    }
    tenkit::AlsReport ar;
    ar.iterations = m.iterations;
    ar.residual_history = full_history(ctx, k, m);
    ar.status = m.status == 0 ? tenkit::AlsStatus::kConverged : tenkit::AlsStatus::kMaxItersReached;
    ar.achieved_eta = m.achieved_eta;
    mr.als = ar;
    out.per_mode.push_back(mr);
  }
  out.relative_residual = r.relative_residual;
  out.seconds = r.seconds;
  return out;
}

inline std::pair<tenkit::TuckerTensor, tenkit::DecompositionReport> run(
    bool sequential, const tenkit::DenseTensor& t, const tenkit::Truncation& trunc,
    const std::optional<tenkit::ModeOrder>& order, const tenkit::FactorEngine& engine,
    bool want_singular_vectors = false) {
  std::vector<uint64_t> dims(t.shape().dims().begin(), t.shape().dims().end());
  std::vector<uint64_t> ranks(trunc.ranks.begin(), trunc.ranks.end());
  std::vector<uint32_t> ord;
  if (order) ord.assign(order->order.begin(), order->order.end());
  Options opt{engine.als.eta, engine.als.max_iters, engine.als.seed, static_cast<int>(engine.kind)};
  tkg_report rep{};
  Tucker r = hosvd_raw(Context::default_context(), sequential, t.data(), false, dims, ranks, opt,
                       order ? &ord : nullptr, &rep, want_singular_vectors);
  std::vector<std::size_t> rk(trunc.ranks.begin(), trunc.ranks.end());
  tenkit::TuckerTensor tk{tenkit::DenseTensor(tenkit::Shape(rk), std::move(r.core)), {}, t.shape()};
  for (size_t k = 0; k < dims.size(); ++k)
    tk.factors.emplace_back(dims[k], ranks[k], std::move(r.factors[k]));
  return {std::move(tk), to_report(Context::default_context().get(), rep)};
}

inline std::pair<tenkit::TuckerTensor, tenkit::DecompositionReport> t_hosvd(
    const tenkit::DenseTensor& t, const tenkit::Truncation& trunc, const tenkit::FactorEngine& engine,
    bool want_singular_vectors = false) {
  return run(false, t, trunc, std::nullopt, engine, want_singular_vectors);
}

// hosvd.hpp:78-82
inline tenkit::Matrix recover_singular_vectors(const tenkit::DenseTensor& t, std::size_t mode,
                                               const tenkit::Matrix& q) {
  std::vector<uint64_t> dims(t.shape().dims().begin(), t.shape().dims().end());
  std::vector<double> out(q.rows() * q.cols(), 0.0);
  tkg_error e{};
  check(tkg_recover_singular_vectors(Context::default_context().get(), t.data(), int32_t(dims.size()),
                                     dims.data(), uint32_t(mode), q.values().data(), q.rows(), q.cols(),
                                     out.data(), &e),
        e);
  return tenkit::Matrix(q.rows(), q.cols(), std::move(out));
}

inline std::pair<tenkit::TuckerTensor, tenkit::DecompositionReport> st_hosvd(
    const tenkit::DenseTensor& t, const tenkit::Truncation& trunc,
    const std::optional<tenkit::ModeOrder>& order, const tenkit::FactorEngine& engine) {
  return run(true, t, trunc, order, engine);
}

// ---- primitives with the reference's signatures --------------------------------
inline std::vector<uint64_t> dims_of(const tenkit::Shape& s) {
  return std::vector<uint64_t>(s.dims().begin(), s.dims().end());
}

// als.hpp:69-71
inline std::pair<tenkit::FactorPair, tenkit::AlsReport> als_low_rank(const tenkit::DenseTensor& t, std::size_t mode,
                                                                     std::size_t r, const tenkit::AlsConfig& cfg) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  const uint64_t I = (mode >= 1 && mode <= dims.size()) ? dims[mode - 1] : 1;
  const uint64_t F = I ? t.size() / I : 0;
  std::vector<double> l(I * r, 0.0), rr(F * r, 0.0);
  tkg_als_config c{cfg.eta, cfg.max_iters, cfg.seed, cfg.init ? cfg.init->data() : nullptr,
                   cfg.init ? cfg.init->rows() : 0, cfg.init ? cfg.init->cols() : 0};
  tkg_mode_report rep{};
  tkg_error e{};
  check(tkg_als_low_rank(Context::default_context().get(), t.data(), 0, int32_t(dims.size()), dims.data(),
                         uint32_t(mode), r, &c, l.data(), rr.data(), &rep, &e),
        e);
  tenkit::AlsReport ar;
  ar.iterations = rep.iterations;
  ar.residual_history = full_history(Context::default_context().get(), 0, rep);
  ar.status = rep.status == 0 ? tenkit::AlsStatus::kConverged : tenkit::AlsStatus::kMaxItersReached;
  ar.achieved_eta = rep.achieved_eta;
  return {tenkit::FactorPair{tenkit::Matrix(I, r, std::move(l)), tenkit::Matrix(F, r, std::move(rr))}, ar};
}

// als.hpp:56-57
inline std::pair<tenkit::FactorPair, double> als_sweep(const tenkit::DenseTensor& t, std::size_t mode,
                                                       const tenkit::Matrix& l) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  const uint64_t I = (mode >= 1 && mode <= dims.size()) ? dims[mode - 1] : 1;
  const uint64_t F = I ? t.size() / I : 0;
  std::vector<double> ln(l.rows() * l.cols(), 0.0), rr(F * l.cols(), 0.0);
  double res = 0.0;
  tkg_error e{};
  check(tkg_als_sweep(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(), uint32_t(mode),
                      l.data(), l.cols(), ln.data(), rr.data(), &res, &e),
        e);
  return {tenkit::FactorPair{tenkit::Matrix(l.rows(), l.cols(), std::move(ln)),
                             tenkit::Matrix(F, l.cols(), std::move(rr))},
          res};
}

// tensor_ops.hpp:39 / :44
inline tenkit::Matrix unfold_times(const tenkit::DenseTensor& t, std::size_t mode, const tenkit::Matrix& m) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  const uint64_t I = (mode >= 1 && mode <= dims.size()) ? dims[mode - 1] : 1;
  std::vector<double> out(I * m.cols(), 0.0);
  tkg_error e{};
  check(tkg_unfold_times(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(),
                         uint32_t(mode), m.data(), m.cols(), out.data(), &e),
        e);
  return tenkit::Matrix(I, m.cols(), std::move(out));
}

inline tenkit::Matrix unfold_t_times(const tenkit::DenseTensor& t, std::size_t mode, const tenkit::Matrix& m) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  const uint64_t I = (mode >= 1 && mode <= dims.size()) ? dims[mode - 1] : 1;
  const uint64_t F = I ? t.size() / I : 0;
  std::vector<double> out(F * m.cols(), 0.0);
  tkg_error e{};
  check(tkg_unfold_t_times(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(),
                           uint32_t(mode), m.data(), m.cols(), out.data(), &e),
        e);
  return tenkit::Matrix(F, m.cols(), std::move(out));
}

// tensor_ops.hpp:22-23
inline tenkit::DenseTensor mode_n_product(const tenkit::DenseTensor& t, const tenkit::Matrix& u, std::size_t mode) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  std::vector<std::size_t> od(t.shape().dims().begin(), t.shape().dims().end());
  if (mode >= 1 && mode <= od.size()) od[mode - 1] = u.rows();
  uint64_t n = 1;
  for (std::size_t d : od) n *= d;
  std::vector<double> out(n, 0.0);
  tkg_error e{};
  check(tkg_mode_n_product(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(), u.data(),
                           u.rows(), u.cols(), uint32_t(mode), out.data(), &e),
        e);
  return tenkit::DenseTensor(tenkit::Shape(od), std::move(out));
}

// tensor_ops.hpp:33-34
inline tenkit::DenseTensor multi_mode_product(const tenkit::DenseTensor& t,
                                              const std::vector<tenkit::ModeFactor>& factors) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  std::vector<std::size_t> od(t.shape().dims().begin(), t.shape().dims().end());
  std::vector<uint32_t> modes;
  std::vector<const double*> ptrs;
  std::vector<uint64_t> rows, cols;
  for (const tenkit::ModeFactor& f : factors) {
    modes.push_back(uint32_t(f.mode));
    ptrs.push_back(f.factor.data());
    rows.push_back(f.factor.rows());
    cols.push_back(f.factor.cols());
    if (f.mode >= 1 && f.mode <= od.size()) od[f.mode - 1] = f.factor.rows();
  }
  uint64_t n = 1;
  for (std::size_t d : od) n *= d;
  std::vector<double> out(n, 0.0);
  tkg_error e{};
  check(tkg_multi_mode_product(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(),
                               int32_t(factors.size()), modes.data(), ptrs.data(), rows.data(), cols.data(),
                               out.data(), &e),
        e);
  return tenkit::DenseTensor(tenkit::Shape(od), std::move(out));
}

// tensor_ops.hpp:52 / :55
inline double frobenius_norm(const tenkit::DenseTensor& t) {
  std::vector<uint64_t> dims = dims_of(t.shape());
  double out = 0.0;
  tkg_error e{};
  check(tkg_frobenius_norm(Context::default_context().get(), t.data(), int32_t(dims.size()), dims.data(), &out, &e),
        e);
  return out;
}

inline double relative_error(const tenkit::DenseTensor& a, const tenkit::DenseTensor& b) {
  if (a.shape() != b.shape())
    throw tenkit::DimensionMismatchError("relative_error: shapes " + a.shape().to_string() + " vs " +
                                         b.shape().to_string());
  std::vector<uint64_t> dims = dims_of(a.shape());
  double out = 0.0;
  tkg_error e{};
  check(tkg_relative_error(Context::default_context().get(), a.data(), b.data(), int32_t(dims.size()), dims.data(),
                           &out, &e),
        e);
  return out;
}

// hooi.hpp:33-37
inline tenkit::HooiResult hooi(const tenkit::DenseTensor& t, const tenkit::Truncation& trunc,
                               const tenkit::TuckerTensor& init, const tenkit::HooiConfig& cfg) {
  if (init.origin_shape != t.shape())
    throw tenkit::DimensionMismatchError("hooi: init origin shape " + init.origin_shape.to_string() +
                                         " does not match tensor " + t.shape().to_string());
  std::vector<uint64_t> dims = dims_of(t.shape());
  std::vector<uint64_t> ranks(trunc.ranks.begin(), trunc.ranks.end());
  const std::size_t n = dims.size();
  if (init.factors.size() != n || init.core.shape().order() != n)
    throw tenkit::DimensionMismatchError("hooi: init is not an order-" + std::to_string(n) + " decomposition");
  std::vector<double> f_in;
  for (std::size_t m = 0; m < n; ++m) {
    const tenkit::Matrix& u = init.factors[m];
    if (ranks.size() != n || u.rows() != dims[m] || u.cols() != ranks[m] || init.core.shape().extent(m + 1) != ranks[m])
      throw tenkit::DimensionMismatchError("hooi: init factor for mode " + std::to_string(m + 1) +
                                           " does not match the truncation");
    f_in.insert(f_in.end(), u.values().begin(), u.values().end());
  }
  uint64_t core_n = 1, fac_n = 0;
  for (std::size_t m = 0; m < n; ++m) {
    core_n *= ranks[m];
    fac_n += dims[m] * ranks[m];
  }
  std::vector<double> core(core_n, 0.0), fac(fac_n, 0.0), fits(std::size_t(cfg.max_iters < 1 ? 1 : cfg.max_iters) + 1);
  int32_t iters = 0, conv = 0;
  tkg_error e{};
  check(tkg_hooi(Context::default_context().get(), t.data(), 0, int32_t(n), dims.data(), ranks.data(),
                 init.core.data(), f_in.data(), cfg.tol, cfg.max_iters, core.data(), fac.data(), &iters, &conv,
                 fits.data(), nullptr, &e),
        e);
  std::vector<std::size_t> rk(trunc.ranks.begin(), trunc.ranks.end());
  tenkit::TuckerTensor tk{tenkit::DenseTensor(tenkit::Shape(rk), std::move(core)), {}, t.shape()};
  uint64_t ofs = 0;
  for (std::size_t m = 0; m < n; ++m) {
    tk.factors.emplace_back(dims[m], ranks[m],
                            std::vector<double>(fac.begin() + ofs, fac.begin() + ofs + dims[m] * ranks[m]));
    ofs += dims[m] * ranks[m];
  }
  tenkit::HooiResult res{std::move(tk)};
  res.iterations = iters;
  res.fit_history.assign(fits.begin(), fits.begin() + iters + 1);
  res.converged = conv != 0;
  return res;
}
#endif

}  // namespace tenkit_b200
