// extern "C" entry points declared in include/tenkit_b200.h. Each wraps an
// Engine call, maps tkg::Error onto (return code, subtype, message) exactly
// like the reference's exception taxonomy (errors.hpp:10-77), and never
// lets a C++ exception cross the ABI.
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/tenkit_b200.h"
#include "engine.hpp"
#include "io.hpp"

struct tkg_ctx {
  tkg::Engine* eng;
  // residual histories of the last decomposition / als_low_rank call, per
  // processing position (tkg_residual_history)
  std::vector<std::vector<double>> last_hist;
};

struct tkg_local_group {
  std::shared_ptr<tkg::LocalGroup> g;
};

namespace {

void set_err(tkg_error* err, int code, int subtype, const char* msg) {
  if (!err) return;
  err->code = code;
  err->subtype = subtype;
  std::strncpy(err->message, msg, sizeof(err->message) - 1);
  err->message[sizeof(err->message) - 1] = '\0';
}

template <class F>
int guarded(tkg_error* err, F&& f) {
  try {
    f();
    set_err(err, 0, TKG_OK, "");
    return 0;
  } catch (const tkg::Error& e) {
    set_err(err, e.code, e.subtype, e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err(err, 2, TKG_E_CUDA, "host allocation failed");
    return 2;
  } catch (const std::exception& e) {
    set_err(err, 1, TKG_E_UNSUPPORTED, e.what());
    return 1;
  }
}

tkg::Shape make_shape(int32_t order, const uint64_t* dims) {
  if (order < 1) tkg::raise(TKG_E_DIMENSION_MISMATCH, "Shape: at least one extent required");
  if (order > TKG_MAX_ORDER) tkg::raise(TKG_E_UNSUPPORTED, "order above 64 is not supported");
  tkg::Shape s;
  s.N = order;
  for (int k = 0; k < order; ++k) {
    if (dims[k] == 0) tkg::raise(TKG_E_DIMENSION_MISMATCH, "Shape: extents must be >= 1");
    s.d[k] = dims[k];
  }
  return s;
}

tkg::AlsCfg make_cfg(const tkg_als_config* c) {
  tkg::AlsCfg a;
  if (c) {
    a.eta = c->eta;
    a.max_iters = c->max_iters;
    a.seed = c->seed;
    a.init = c->init;
    a.init_rows = c->init_rows;
    a.init_cols = c->init_cols;
  }
  return a;
}

void fill_mode(const tkg::ModeRep& m, tkg_mode_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->mode = m.mode;
  out->iterations = m.iterations;
  out->status = m.status;
  out->achieved_eta = m.achieved_eta;
  out->seconds = m.seconds;
  const size_t n = std::min<size_t>(m.history.size(), TKG_MAX_HISTORY);
  out->history_len = int32_t(n);
  for (size_t k = 0; k < n; ++k) out->residual_history[k] = m.history[k];
}

void fill_report(tkg_ctx* ctx, const tkg::DecompRep& r, int order, tkg_report* out) {
  ctx->last_hist.clear();
  for (const tkg::ModeRep& m : r.per_mode) ctx->last_hist.push_back(m.history);
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->order = order;
  out->n_modes = int32_t(r.per_mode.size());
  for (size_t k = 0; k < r.per_mode.size() && k < TKG_MAX_ORDER; ++k) fill_mode(r.per_mode[k], &out->per_mode[k]);
  out->relative_residual = r.relative_residual;
  out->seconds = r.seconds;
  out->h2d_seconds = r.h2d_seconds;
  out->d2h_seconds = r.d2h_seconds;
  out->residual_seconds = r.residual_seconds;
  out->kernel_launches = r.launches;
  out->tensor_passes = r.passes;
  out->algorithmic_bytes = r.bytes;
}

tkg::Engine& eng(tkg_ctx* ctx) {
  if (!ctx || !ctx->eng) tkg::raise(TKG_E_UNSUPPORTED, "null tkg context");
  // the calling thread may have another device current (one process driving
  // several contexts): every entry point runs on the context's device
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != ctx->eng->device()) cudaSetDevice(ctx->eng->device());
  return *ctx->eng;
}

}  // namespace

extern "C" {

const char* tkg_version(void) { return "tenkit_b200 0.1 (sm_100a, FP64 DMMA)"; }

int tkg_create(tkg_ctx** ctx, int device, tkg_error* err) {
  return guarded(err, [&] {
    *ctx = nullptr;
    auto* c = new tkg_ctx;
    try {
      c->eng = new tkg::Engine(device);
    } catch (...) {
      delete c;
      throw;
    }
    *ctx = c;
  });
}

int tkg_destroy(tkg_ctx* ctx) {
  if (ctx) {
    delete ctx->eng;
    delete ctx;
  }
  return 0;
}

int tkg_t_hosvd(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                const uint64_t* ranks, const tkg_als_config* cfg, int32_t want_singular_vectors,
                double* core, double* factors, tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    tkg::DecompRep rep;
    eng(ctx).t_hosvd(a, a_on_device != 0, sh, rk, make_cfg(cfg), core, factors, &rep, want_singular_vectors != 0);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_st_hosvd(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                 const uint64_t* ranks, const uint32_t* mode_order, const tkg_als_config* cfg,
                 double* core, double* factors, tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    std::vector<int> mo;
    if (mode_order) mo.assign(mode_order, mode_order + order);
    tkg::DecompRep rep;
    eng(ctx).st_hosvd(a, a_on_device != 0, sh, rk, mode_order ? &mo : nullptr, make_cfg(cfg), core,
                      factors, &rep);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_t_hosvd_engine(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                       const uint64_t* ranks, const tkg_factor_engine* engine, int32_t want_singular_vectors,
                       double* core, double* factors, tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    const int kind = engine ? engine->kind : TKG_ENGINE_ALS;
    if (kind < TKG_ENGINE_SVD || kind > TKG_ENGINE_ALS) tkg::raise(TKG_E_UNSUPPORTED, "unknown factor engine kind");
    tkg::DecompRep rep;
    eng(ctx).t_hosvd(a, a_on_device != 0, sh, rk, make_cfg(engine ? &engine->als : nullptr), core, factors, &rep,
                     kind == TKG_ENGINE_ALS && want_singular_vectors != 0, kind);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_st_hosvd_engine(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                        const uint64_t* ranks, const uint32_t* mode_order, const tkg_factor_engine* engine,
                        double* core, double* factors, tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    std::vector<int> mo;
    if (mode_order) mo.assign(mode_order, mode_order + order);
    const int kind = engine ? engine->kind : TKG_ENGINE_ALS;
    if (kind < TKG_ENGINE_SVD || kind > TKG_ENGINE_ALS) tkg::raise(TKG_E_UNSUPPORTED, "unknown factor engine kind");
    tkg::DecompRep rep;
    eng(ctx).st_hosvd(a, a_on_device != 0, sh, rk, mode_order ? &mo : nullptr,
                      make_cfg(engine ? &engine->als : nullptr), core, factors, &rep, kind);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_hooi(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
             const uint64_t* ranks, const double* init_core, const double* init_factors, double tol,
             int32_t max_iters, double* core, double* factors, int32_t* iterations, int32_t* converged,
             double* fit_history, double* relative_residual, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    if (!init_core || !init_factors) tkg::raise(TKG_E_DIMENSION_MISMATCH, "hooi: init is not an order-" +
                                                                                  std::to_string(order) +
                                                                                  " decomposition");
    tkg::HooiRep rep;
    eng(ctx).hooi(a, a_on_device != 0, sh, rk, init_core, init_factors, tol, max_iters, core, factors, &rep);
    if (iterations) *iterations = rep.iterations;
    if (converged) *converged = rep.converged ? 1 : 0;
    if (fit_history)
      for (size_t k = 0; k < rep.fit_history.size(); ++k) fit_history[k] = rep.fit_history[k];
    if (relative_residual) *relative_residual = rep.relative_residual;
  });
}

int tkg_device_alloc(tkg_ctx* ctx, uint64_t bytes, void** out, tkg_error* err) {
  return guarded(err, [&] {
    eng(ctx);
    *out = nullptr;
    CK(cudaMalloc(out, std::max<uint64_t>(bytes, 1)));
  });
}

int tkg_device_free(tkg_ctx* ctx, void* p) {
  (void)ctx;
  return p && cudaFree(p) != cudaSuccess ? 2 : 0;
}

int tkg_device_copy(tkg_ctx* ctx, void* dst, const void* src, uint64_t bytes, tkg_error* err) {
  return guarded(err, [&] {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, eng(ctx).stream()));
    CK(cudaStreamSynchronize(eng(ctx).stream()));
  });
}

int tkg_read_tnsr_shape(const char* path, int32_t* order, uint64_t* dims, tkg_error* err) {
  return guarded(err, [&] {
    const tkg::Shape sh = tkg::tnsr_shape(path ? path : "");
    *order = sh.N;
    for (int k = 0; k < sh.N; ++k) dims[k] = sh.d[k];
  });
}

int tkg_read_tnsr(tkg_ctx* ctx, const char* path, double* dst, int dst_on_device, tkg_error* err) {
  return guarded(err, [&] {
    tkg::tnsr_load(path ? path : "", dst, dst_on_device != 0, eng(ctx).stream());
  });
}

int tkg_write_tnsr(const char* path, int32_t order, const uint64_t* dims, const double* data, tkg_error* err) {
  return guarded(err, [&] { tkg::tnsr_write(path ? path : "", make_shape(order, dims), data); });
}

int tkg_write_tukr(const char* path, int32_t order, const uint64_t* dims, const uint64_t* ranks, const double* core,
                   const double* factors, tkg_error* err) {
  return guarded(err, [&] {
    tkg::tukr_write(path ? path : "", make_shape(order, dims), std::vector<uint64_t>(ranks, ranks + order), core,
                    factors);
  });
}

int tkg_multi_mode_product(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, int32_t nfactors,
                           const uint32_t* modes, const double* const* factors, const uint64_t* rows,
                           const uint64_t* cols, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<int> m(modes, modes + nfactors);
    std::vector<const double*> f(factors, factors + nfactors);
    std::vector<uint64_t> rw(rows, rows + nfactors), cl(cols, cols + nfactors);
    eng(ctx).multi_mode_product(a, sh, m, f, rw, cl, out);
  });
}

int tkg_reconstruct(tkg_ctx* ctx, const double* core, int32_t order, const uint64_t* ranks, const uint64_t* dims,
                    const double* factors, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape cs = make_shape(order, ranks);
    (void)make_shape(order, dims);
    std::vector<int> m(order);
    std::vector<const double*> f(order);
    std::vector<uint64_t> rw(order), cl(order);
    const double* p = factors;
    for (int n = 0; n < order; ++n) {  // reconstruct (tensor_ops.cpp:420-440): U_n is dims[n] x ranks[n]
      m[n] = n + 1;
      f[n] = p;
      rw[n] = dims[n];
      cl[n] = ranks[n];
      p += dims[n] * ranks[n];
    }
    eng(ctx).multi_mode_product(core, cs, m, f, rw, cl, out);
  });
}

int tkg_mode_gram(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode, double* out,
                  tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).mode_gram(a, sh, int(mode), out);
  });
}

int tkg_sym_eig(tkg_ctx* ctx, const double* g, uint64_t n, uint64_t k, double* values, double* vectors,
                tkg_error* err) {
  return guarded(err, [&] { eng(ctx).sym_eig(g, n, k, values, vectors); });
}

int tkg_nccl_unique_id(void* out128, tkg_error* err) {
  return guarded(err, [&] {
    if (!tkg::nccl_unique_id(out128)) tkg::raise(TKG_E_CUDA, "NCCL (libnccl.so.2) could not be loaded");
  });
}

int tkg_comm_init_nccl(tkg_ctx* ctx, int rank, int world, const void* unique_id128, tkg_error* err) {
  return guarded(err, [&] {
    if (world < 1 || rank < 0 || rank >= world) tkg::raise(TKG_E_DIMENSION_MISMATCH, "comm: bad rank / world");
    eng(ctx).set_comm(tkg::make_nccl_comm(unique_id128, rank, world));
  });
}

int tkg_comm_init_shm(tkg_ctx* ctx, const char* name, int rank, int world, uint64_t slot_bytes, tkg_error* err) {
  return guarded(err, [&] {
    if (world < 1 || rank < 0 || rank >= world || !name || name[0] != '/')
      tkg::raise(TKG_E_DIMENSION_MISMATCH, "comm: bad rank / world / shm name");
    eng(ctx).set_comm(tkg::make_shm_comm(name, rank, world, slot_bytes ? size_t(slot_bytes) : size_t(64) << 20));
  });
}

int tkg_local_group_create(int world, tkg_local_group** out, tkg_error* err) {
  return guarded(err, [&] {
    if (world < 1) tkg::raise(TKG_E_DIMENSION_MISMATCH, "local group: world must be >= 1");
    *out = new tkg_local_group{tkg::make_local_group(world)};
  });
}

void tkg_local_group_destroy(tkg_local_group* g) { delete g; }

int tkg_comm_init_local(tkg_ctx* ctx, tkg_local_group* g, int rank, tkg_error* err) {
  return guarded(err, [&] {
    if (!g || rank < 0 || rank >= tkg::local_group_world(*g->g)) tkg::raise(TKG_E_DIMENSION_MISMATCH, "comm: bad rank / group");
    eng(ctx).set_comm(tkg::make_local_comm(g->g, rank));
  });
}

int tkg_shard_range(uint64_t extent, int rank, int world, uint64_t* begin, uint64_t* len) {
  if (world < 1 || rank < 0 || rank >= world) return 1;
  const tkg::ShardRange r = tkg::shard_range(extent, rank, world);
  *begin = r.begin;
  *len = r.len;
  return 0;
}

int tkg_t_hosvd_sharded(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                        uint64_t slab_begin, uint64_t slab_len, const uint64_t* ranks,
                        const tkg_als_config* cfg, int32_t want_singular_vectors, double* core, double* factors,
                        tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    tkg::DecompRep rep;
    eng(ctx).t_hosvd_sharded(a, a_on_device != 0, sh, slab_begin, slab_len, rk, make_cfg(cfg), core, factors,
                             &rep, want_singular_vectors != 0);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_st_hosvd_sharded(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                         uint64_t slab_begin, uint64_t slab_len, const uint64_t* ranks,
                         const uint32_t* mode_order, const tkg_als_config* cfg, double* core, double* factors,
                         tkg_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    std::vector<int> mo;
    if (mode_order) mo.assign(mode_order, mode_order + order);
    tkg::DecompRep rep;
    eng(ctx).st_hosvd_sharded(a, a_on_device != 0, sh, slab_begin, slab_len, rk, mode_order ? &mo : nullptr,
                              make_cfg(cfg), core, factors, &rep);
    fill_report(ctx, rep, order, report);
  });
}

int tkg_select_order(int32_t order, const uint64_t* dims, const uint64_t* ranks, uint32_t* out,
                     tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    std::vector<uint64_t> rk(ranks, ranks + order);
    tkg::validate_truncation(sh, rk);  // select_order validates first (hosvd.cpp:55)
    std::vector<int> o = tkg::select_order(rk);
    for (int k = 0; k < order; ++k) out[k] = uint32_t(o[k]);
  });
}

int tkg_als_low_rank(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order,
                     const uint64_t* dims, uint32_t mode, uint64_t r, const tkg_als_config* cfg,
                     double* l_out, double* r_out, tkg_mode_report* report, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    sh.extent(int(mode));  // InvalidMode first
    // the zero-norm / rank / init-shape guards run in the engine, in the
    // reference's order (als.cpp:101-113, 62-66)
    if (r > 0xffffffffu) tkg::raise(TKG_E_RANK_TOO_LARGE, "rank too large");
    tkg::ModeRep rep;
    eng(ctx).als_low_rank(a, a_on_device != 0, sh, int(mode), uint32_t(r), make_cfg(cfg), l_out,
                          r_out, &rep);
    ctx->last_hist.assign(1, rep.history);
    if (report) fill_mode(rep, report);
  });
}

int tkg_residual_history(tkg_ctx* ctx, int32_t position, double* out, uint64_t cap, uint64_t* len,
                         tkg_error* err) {
  return guarded(err, [&] {
    eng(ctx);
    if (position < 0 || size_t(position) >= ctx->last_hist.size())
      tkg::raise(TKG_E_INVALID_MODE, "residual_history: no mode at position " + std::to_string(position) +
                                         " in the last decomposition");
    const std::vector<double>& h = ctx->last_hist[size_t(position)];
    if (len) *len = h.size();
    if (out)
      for (size_t k = 0; k < h.size() && k < cap; ++k) out[k] = h[k];
  });
}

int tkg_als_sweep(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode,
                  const double* l, uint64_t r, double* l_out, double* r_out, double* residual, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    if (r > 0xffffffffu) tkg::raise(TKG_E_UNSUPPORTED, "als_sweep: rank too large");
    eng(ctx).als_sweep(a, sh, int(mode), l, uint32_t(r), l_out, r_out, residual);
  });
}

int tkg_als_init(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                 uint32_t mode, uint64_t r, uint64_t seed, double* l_out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).als_init(a, a_on_device != 0, sh, int(mode), uint32_t(r), seed, l_out);
  });
}

int tkg_unfold_times(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode,
                     const double* m, uint64_t r, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).unfold_times(a, sh, int(mode), m, uint32_t(r), out);
  });
}

int tkg_unfold_t_times(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                       uint32_t mode, const double* m, uint64_t r, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).unfold_t_times(a, sh, int(mode), m, uint32_t(r), out);
  });
}

int tkg_mode_n_product(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                       const double* u, uint64_t rows, uint64_t cols, uint32_t mode, double* out,
                       tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).mode_n_product(a, sh, u, rows, cols, int(mode), out);
  });
}

int tkg_frobenius_norm(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, double* out,
                       tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    *out = eng(ctx).frobenius_norm(a, sh.count());
  });
}

int tkg_relative_error(tkg_ctx* ctx, const double* a, const double* b, int32_t order,
                       const uint64_t* dims, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    *out = eng(ctx).relative_error(a, b, sh.count());
  });
}

int tkg_reduced_qr(tkg_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double* q, double* r,
                   tkg_error* err) {
  return guarded(err, [&] { eng(ctx).reduced_qr(a, rows, cols, q, r); });
}

int tkg_gram(tkg_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double* out, tkg_error* err) {
  return guarded(err, [&] { eng(ctx).gram(a, rows, cols, out); });
}

int tkg_recover_singular_vectors(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode,
                                 const double* q, uint64_t rows, uint64_t cols, double* out, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).recover_singular_vectors(a, sh, int(mode), q, rows, cols, out);
  });
}

int tkg_uniform01(tkg_ctx* ctx, uint64_t seed, uint32_t stream, uint64_t n, double* out, tkg_error* err) {
  return guarded(err, [&] { eng(ctx).uniform01(seed, stream, n, out); });
}

int tkg_set_profiling(tkg_ctx* ctx, int on) {
  if (!ctx || !ctx->eng) return 1;
  ctx->eng->set_profiling(on != 0);
  return 0;
}

int tkg_set_fused_sweep(tkg_ctx* ctx, int on) {
  if (!ctx || !ctx->eng) return 1;
  ctx->eng->set_fused_sweep(on != 0);
  return 0;
}

int tkg_get_kernel_stats(tkg_ctx* ctx, tkg_kernel_stats* out) {
  tkg_error err;
  return guarded(&err, [&] {
    std::memset(out, 0, sizeof(*out));
    eng(ctx).kernel_stats(out->ms, out->launches, out->bytes, out->flops);
  });
}

int tkg_bench_contractions(tkg_ctx* ctx, const double* d_a, int32_t order, const uint64_t* dims,
                           uint32_t mode, uint32_t r, int32_t reps, double* out_ms, tkg_error* err) {
  return guarded(err, [&] {
    tkg::Shape sh = make_shape(order, dims);
    eng(ctx).bench_contractions(d_a, sh, int(mode), r, reps < 1 ? 1 : reps, out_ms);
  });
}

int tkg_timer_start(tkg_ctx* ctx) {
  tkg_error err;
  return guarded(&err, [&] { eng(ctx).timer_start(); });
}

int tkg_timer_stop(tkg_ctx* ctx, double* ms) {
  tkg_error err;
  return guarded(&err, [&] { *ms = eng(ctx).timer_stop(); });
}

int tkg_flush_l2(tkg_ctx* ctx) {
  tkg_error err;
  return guarded(&err, [&] { eng(ctx).flush_l2(); });
}

}  // extern "C"
