// Minimal C++ caller of the B200 path through include/tenkit_b200.hpp.
// Built two ways by tests/test_abi_cpp.py:
//   - self-contained types;
//   - -DTENKIT_B200_USE_TENKIT with the reference headers, i.e. the exact
//     tenkit::DenseTensor -> t_hosvd/st_hosvd signatures of hosvd.hpp:55-70.
#include <cstdio>
#include <vector>

#include "tenkit_b200.hpp"

int main() {
#ifdef TENKIT_B200_USE_TENKIT
  tenkit::DenseTensor t(tenkit::Shape({6, 5, 4}));
  for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = double((i * 7919) % 101) / 101.0;
  tenkit::AlsConfig cfg;
  cfg.eta = 1e-8;
  try {
    auto [tk, rep] = tenkit_b200::st_hosvd(t, tenkit::Truncation{{2, 2, 2}}, std::nullopt,
                                           tenkit::FactorEngine::with_als(cfg));
    std::printf("rel err %.6e, modes %zu\n", rep.relative_residual, rep.per_mode.size());
    // the primitives with the reference's signatures
    tenkit::Matrix u(3, 5);
    tenkit::DenseTensor p = tenkit_b200::mode_n_product(t, u, 2);
    tenkit::DenseTensor q = tenkit_b200::multi_mode_product(t, {{u, 2}});
    tenkit::HooiResult h = tenkit_b200::hooi(t, tenkit::Truncation{{2, 2, 2}}, tk, tenkit::HooiConfig{});
    auto [pair, ar] = tenkit_b200::als_low_rank(t, 1, 2, cfg);
    std::printf("%zu %zu %d %d %.3e %.3e\n", p.size(), q.size(), h.iterations, ar.iterations,
                tenkit_b200::frobenius_norm(t), tenkit_b200::relative_error(t, p.size() == t.size() ? t : t));
    (void)tenkit_b200::unfold_times(t, 1, pair.r);
    (void)tenkit_b200::unfold_t_times(t, 1, pair.l);
  } catch (const tenkit::Error& e) {
    std::printf("tenkit error (category %d): %s\n", int(e.category()), e.what());
    return 2;
  }
#else
  std::vector<uint64_t> dims{6, 5, 4}, ranks{2, 2, 2};
  std::vector<double> a(120);
  for (std::size_t i = 0; i < a.size(); ++i) a[i] = double((i * 7919) % 101) / 101.0;
  try {
    tkg_report rep{};
    tenkit_b200::Tucker tk = tenkit_b200::hosvd_raw(tenkit_b200::Context::default_context(), false,
                                                    a.data(), false, dims, ranks, {1e-8, 50, 0},
                                                    nullptr, &rep);
    std::printf("rel err %.6e, core %zu\n", rep.relative_residual, tk.core.size());
  } catch (const tenkit_b200::Error& e) {
    std::printf("error (category %d): %s\n", e.category, e.what());
    return 2;
  }
#endif
  return 0;
}
