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
#include "tenkit/errors.hpp"
#include "tenkit/hosvd.hpp"
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
inline tenkit::DecompositionReport to_report(const tkg_report& r) {
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
    ar.residual_history.assign(m.residual_history, m.residual_history + m.history_len);
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
  return {std::move(tk), to_report(rep)};
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
#endif

}  // namespace tenkit_b200
