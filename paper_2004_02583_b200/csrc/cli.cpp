// tenkit_b200: the reference CLI's `compress` subcommand (tenkit_main.cpp:
// 183-266, 565-596) on the B200 path, a client of the C-ABI only
// (include/tenkit_b200.h). The TNSR payload goes straight from disk into HBM
// (tkg_read_tnsr through pinned chunks), the decomposition runs on the
// device, the TUKR file and the CSV record (method, dims, ranks, order, eta,
// seed, threads, rel_residual, seconds, iters_per_mode) are the reference's.
// The `threads` field reports the GPU count (1). Exit codes follow the
// reference: 1 usage, 2 io, 3 numerical (tenkit_main.cpp:644-664).
//
//   tenkit_b200 compress --in A.tnsr --out A.tukr --ranks 32,32,32
//       [--method t-svd|t-eig|t-als|st-svd|st-eig|st-als|hooi] [--init st-svd]
//       [--order auto|2,1,3] [--eta 1e-4] [--max-iters 50] [--seed 0]
//       [--singular-vectors] [--header] [--hooi-tol 1e-12] [--hooi-iters 100]
//       [--threads N (ignored)] [--device D]
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tenkit_b200.h"

namespace {

const char* kCsvHeader = "method,dims,ranks,order,eta,seed,threads,rel_residual,seconds,iters_per_mode";

struct Usage {
  std::string msg;
};

struct Options {
  std::string in, out, method = "st-als", init = "st-svd", order = "auto";
  std::vector<uint64_t> ranks;
  double eta = 1e-4, hooi_tol = 1e-12;
  int max_iters = 50, hooi_iters = 100, device = 0;
  uint64_t seed = 0;
  bool singular_vectors = false, header = false;
};

struct Method {
  bool sequential = false, hooi = false;
  int kind = TKG_ENGINE_SVD;
};

Method parse_method(const std::string& name, const char* flag) {
  Method m;
  if (name == "hooi") {
    m.hooi = true;
    return m;
  }
  std::string engine;
  if (name.rfind("st-", 0) == 0) {
    m.sequential = true;
    engine = name.substr(3);
  } else if (name.rfind("t-", 0) == 0) {
    engine = name.substr(2);
  } else {
    throw Usage{std::string(flag) + ": unknown method '" + name + "'"};
  }
  if (engine == "svd") m.kind = TKG_ENGINE_SVD;
  else if (engine == "eig") m.kind = TKG_ENGINE_EIG;
  else if (engine == "als") m.kind = TKG_ENGINE_ALS;
  else throw Usage{std::string(flag) + ": unknown method '" + name + "'"};
  return m;
}

std::vector<uint64_t> parse_list(const std::string& text, const char* flag) {
  std::vector<uint64_t> out;
  size_t pos = 0;
  while (pos <= text.size()) {
    const size_t comma = text.find(',', pos);
    const std::string item = text.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
    char* end = nullptr;
    const unsigned long long v = std::strtoull(item.c_str(), &end, 10);
    if (item.empty() || *end != '\0') throw Usage{std::string(flag) + ": cannot parse '" + text + "'"};
    out.push_back(v);
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return out;
}

std::string join(const std::vector<uint64_t>& v, char sep) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += sep;
    s += std::to_string(v[i]);
  }
  return s;
}

std::string fmt(const char* f, double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), f, v);
  return buf;
}

// tkg_error -> message + reference exit code
struct Failure {
  int code;
  std::string msg;
};

void check(int rc, const tkg_error& e) {
  if (rc != 0) throw Failure{rc, e.message};
}

struct Run {
  std::vector<double> core, factors;
  tkg_report rep{};
  double rel = 0.0, seconds = 0.0;
  std::vector<uint64_t> order;
  std::string iters;
};

Run decompose(tkg_ctx* ctx, const void* dA, const std::vector<uint64_t>& dims, const Options& o, const Method& m) {
  Run r;
  const int32_t N = int32_t(dims.size());
  uint64_t core_n = 1, fac_n = 0;
  for (size_t k = 0; k < dims.size(); ++k) {
    core_n *= o.ranks[k];
    fac_n += dims[k] * o.ranks[k];
  }
  r.core.assign(core_n, 0.0);
  r.factors.assign(fac_n, 0.0);
  tkg_factor_engine eng{m.kind, {o.eta, o.max_iters, o.seed, nullptr}};
  tkg_error e{};
  std::vector<uint32_t> ord;
  const bool explicit_order = o.order != "auto";
  if (explicit_order) {
    for (uint64_t v : parse_list(o.order, "--order")) ord.push_back(uint32_t(v));
    if (ord.size() != dims.size())
      throw Failure{1, "st_hosvd: order has " + std::to_string(ord.size()) + " entries for an order-" +
                           std::to_string(dims.size()) + " tensor"};
  }
  if (m.sequential)
    check(tkg_st_hosvd_engine(ctx, static_cast<const double*>(dA), 1, N, dims.data(), o.ranks.data(),
                              explicit_order ? ord.data() : nullptr, &eng, r.core.data(), r.factors.data(), &r.rep,
                              &e),
          e);
  else
    check(tkg_t_hosvd_engine(ctx, static_cast<const double*>(dA), 1, N, dims.data(), o.ranks.data(), &eng,
                             o.singular_vectors ? 1 : 0, r.core.data(), r.factors.data(), &r.rep, &e),
          e);
  r.rel = r.rep.relative_residual;
  r.seconds = r.rep.seconds;
  bool any = false;
  for (int k = 0; k < r.rep.n_modes; ++k) {
    r.order.push_back(uint64_t(r.rep.per_mode[k].mode));
    if (r.rep.per_mode[k].status < 0) continue;  // exact engines: no ALS report
    if (any) r.iters += ',';
    r.iters += std::to_string(r.rep.per_mode[k].iterations);
    any = true;
  }
  return r;
}

int compress(const Options& o) {
  const Method m = parse_method(o.method, "--method");
  tkg_error e{};
  int32_t order = 0;
  uint64_t dbuf[TKG_MAX_ORDER] = {0};
  check(tkg_read_tnsr_shape(o.in.c_str(), &order, dbuf, &e), e);
  std::vector<uint64_t> dims(dbuf, dbuf + order);
  if (o.ranks.size() != dims.size())
    throw Failure{1, "truncation lists " + std::to_string(o.ranks.size()) + " ranks for an order-" +
                         std::to_string(dims.size()) + " tensor"};
  tkg_ctx* ctx = nullptr;
  check(tkg_create(&ctx, o.device, &e), e);
  struct Ctx {
    tkg_ctx* c;
    void* buf = nullptr;
    ~Ctx() {
      if (buf) tkg_device_free(c, buf);
      tkg_destroy(c);
    }
  } hold{ctx};
  uint64_t n = 1;
  for (uint64_t d : dims) n *= d;
  check(tkg_device_alloc(ctx, n * sizeof(double), &hold.buf, &e), e);
  check(tkg_read_tnsr(ctx, o.in.c_str(), static_cast<double*>(hold.buf), 1, &e), e);

  Run r;
  if (m.hooi) {
    const Method warm_m = parse_method(o.init, "--init");
    if (warm_m.hooi) throw Failure{1, "--init: hooi cannot warm-start itself"};
    Run warm = decompose(ctx, hold.buf, dims, o, warm_m);
    const int cap = o.hooi_iters < 1 ? 1 : o.hooi_iters;
    std::vector<double> fits(size_t(cap) + 1, 0.0);
    int32_t iters = 0, conv = 0;
    double rel = 0.0;
    r.core.assign(warm.core.size(), 0.0);
    r.factors.assign(warm.factors.size(), 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    check(tkg_hooi(ctx, static_cast<const double*>(hold.buf), 1, order, dims.data(), o.ranks.data(),
                   warm.core.data(), warm.factors.data(), o.hooi_tol, o.hooi_iters, r.core.data(),
                   r.factors.data(), &iters, &conv, fits.data(), &rel, &e),
          e);
    r.rel = rel;
    // warm start + refinement (tenkit_main.cpp:243-246)
    r.seconds = warm.seconds + std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.iters = std::to_string(iters);
  } else {
    r = decompose(ctx, hold.buf, dims, o, m);
  }
  check(tkg_write_tukr(o.out.c_str(), order, dims.data(), o.ranks.data(), r.core.data(), r.factors.data(), &e), e);
  std::string line = o.method + ',' + join(dims, 'x') + ',' + join(o.ranks, 'x') + ',';
  line += '"' + (m.hooi ? std::string() : join(r.order, ',')) + "\",";
  line += fmt("%g", o.eta) + ',' + std::to_string(o.seed) + ",1,";
  line += fmt("%.17g", r.rel) + ',' + fmt("%.6f", r.seconds) + ',';
  line += '"' + r.iters + '"';
  if (o.header) std::printf("%s\n", kCsvHeader);
  std::printf("%s\n", line.c_str());
  return 0;
}

Options parse(int argc, char** argv) {
  Options o;
  bool have_in = false, have_out = false, have_ranks = false;
  auto value = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw Usage{std::string(argv[i]) + ": missing value"};
    return argv[++i];
  };
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--in") o.in = value(i), have_in = true;
    else if (a == "--out") o.out = value(i), have_out = true;
    else if (a == "--ranks") o.ranks = parse_list(value(i), "--ranks"), have_ranks = true;
    else if (a == "--method") o.method = value(i);
    else if (a == "--init") o.init = value(i);
    else if (a == "--order") o.order = value(i);
    else if (a == "--eta") o.eta = std::strtod(value(i).c_str(), nullptr);
    else if (a == "--max-iters") o.max_iters = std::atoi(value(i).c_str());
    else if (a == "--seed") o.seed = std::strtoull(value(i).c_str(), nullptr, 10);
    else if (a == "--threads") (void)value(i);
    else if (a == "--device") o.device = std::atoi(value(i).c_str());
    else if (a == "--singular-vectors") o.singular_vectors = true;
    else if (a == "--header") o.header = true;
    else if (a == "--hooi-tol") o.hooi_tol = std::strtod(value(i).c_str(), nullptr);
    else if (a == "--hooi-iters") o.hooi_iters = std::atoi(value(i).c_str());
    else throw Usage{"unknown option " + a};
  }
  if (!have_in) throw Usage{"--in is required"};
  if (!have_out) throw Usage{"--out is required"};
  if (!have_ranks) throw Usage{"--ranks is required"};
  static const char* methods[] = {"t-svd", "t-eig", "t-als", "st-svd", "st-eig", "st-als", "hooi"};
  bool known = false;
  for (const char* m : methods) known = known || o.method == m;
  if (!known) throw Usage{"--method: " + o.method + " not in {t-svd,t-eig,t-als,st-svd,st-eig,st-als,hooi}"};
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "compress") != 0) {
    std::fprintf(stderr, "usage: %s compress --in A.tnsr --out A.tukr --ranks R1,R2,... [options]\n", argv[0]);
    return 1;
  }
  try {
    return compress(parse(argc, argv));
  } catch (const Usage& u) {
    std::fprintf(stderr, "%s\n", u.msg.c_str());
    return 1;
  } catch (const Failure& f) {
    std::fprintf(stderr, "error: %s\n", f.msg.c_str());
    return f.code >= 1 && f.code <= 3 ? f.code : 1;
  }
}
