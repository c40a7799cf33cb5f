/* tenkit_b200 — C-ABI of the B200-native ALS-HOSVD hot path.
 *
 * Drop-in boundary for the reference decomposition API of tenkit
 * (arXiv 2004.02583). Every entry point below replaces one reference
 * function; the citation is /root/reference/proj/<file>:<line>.
 *
 *   tkg_t_hosvd        <- tenkit::t_hosvd        include/tenkit/hosvd.hpp:55-57, src/hosvd.cpp:74-125
 *   tkg_st_hosvd       <- tenkit::st_hosvd       include/tenkit/hosvd.hpp:68-70, src/hosvd.cpp:127-191
 *   tkg_select_order   <- tenkit::select_order   include/tenkit/hosvd.hpp:76,    src/hosvd.cpp:54-63
 *   tkg_als_low_rank   <- tenkit::als_low_rank   include/tenkit/als.hpp:69-71,   src/als.cpp:98-161
 *   tkg_als_init       <- tenkit::als_init       include/tenkit/als.hpp:46-47,   src/als.cpp:59-87
 *   tkg_als_sweep      <- tenkit::als_sweep      include/tenkit/als.hpp:56-57,   src/als.cpp:89-96
 *   tkg_unfold_times   <- tenkit::unfold_times   include/tenkit/tensor_ops.hpp:39, src/tensor_ops.cpp:193-261
 *   tkg_unfold_t_times <- tenkit::unfold_t_times include/tenkit/tensor_ops.hpp:44, src/tensor_ops.cpp:263-330
 *   tkg_mode_n_product <- tenkit::mode_n_product include/tenkit/tensor_ops.hpp:22-23, src/tensor_ops.cpp:129-169
 *   tkg_frobenius_norm <- tenkit::frobenius_norm include/tenkit/tensor_ops.hpp:52, src/tensor_ops.cpp:391-393
 *   tkg_relative_error <- tenkit::relative_error include/tenkit/tensor_ops.hpp:55, src/tensor_ops.cpp:395-407
 *   tkg_reduced_qr     <- tenkit::reduced_qr     include/tenkit/kernels.hpp:23,  src/kernels.cpp:303-367
 *   tkg_gram           <- tenkit::gram           include/tenkit/matrix.hpp:49,   src/matrix.cpp:90-126
 *   tkg_uniform01      <- uniform01(seeded_engine(seed, stream)) include/tenkit/rng.hpp:19-21,57-61
 *   tkg_recover_singular_vectors <- tenkit::recover_singular_vectors include/tenkit/hosvd.hpp:78-82,
 *                                   src/hosvd.cpp:65-72
 *   tkg_t_hosvd_engine / tkg_st_hosvd_engine <- t_hosvd / st_hosvd with any FactorEngine
 *                                   (kSvd, kEig, kAls; hosvd.hpp:19-27, hosvd.cpp:89-110, 150-182)
 *   tkg_hooi           <- tenkit::hooi           include/tenkit/hooi.hpp:33-37, src/hooi.cpp:53-110
 *   tkg_read_tnsr / tkg_write_tnsr / tkg_write_tukr <- read_tnsr / write_tnsr / write_tukr
 *                                   include/tenkit/io.hpp, src/io.cpp:131-193
 *   tkg_multi_mode_product <- tenkit::multi_mode_product include/tenkit/tensor_ops.hpp:33-34,
 *                                   src/tensor_ops.cpp:171-191
 *   tkg_reconstruct    <- tenkit::reconstruct    src/tensor_ops.cpp:420-440
 *   tkg_mode_gram      <- tenkit::mode_gram      include/tenkit/tensor_ops.hpp, src/tensor_ops.cpp:332-389
 *   tkg_sym_eig        <- tenkit::sym_eig        include/tenkit/kernels.hpp:51, src/kernels.cpp:448-604
 *
 * Conventions (identical to the reference):
 *   - tensors: flat doubles, generalized column-major, first index fastest
 *     (tensor.hpp:10-11); matrices column-major (matrix.hpp:8-9);
 *   - modes are 1-based (shape.hpp:10-14);
 *   - buffers are caller-owned; `a` may be a host pointer (a_on_device = 0,
 *     copied to HBM inside the call) or a device pointer (a_on_device = 1);
 *     every other pointer is host memory;
 *   - return value 0 on success, else the reference ErrorCategory + 1
 *     (errors.hpp:10: 1 usage, 2 io, 3 numerical — the CLI exit codes,
 *     tenkit_main.cpp:644-664); err->subtype names the reference exception
 *     class and err->message carries the reference's message text;
 *   - a context is single-threaded (one decomposition at a time).
 */
#ifndef TENKIT_B200_H
#define TENKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKG_MAX_ORDER 64   /* the reference's TNSR limit (io.cpp:24) */
#define TKG_MAX_HISTORY 64 /* inline entries; tkg_residual_history returns all */

/* err->subtype: which tenkit exception the call maps to (errors.hpp:24-77). */
enum tkg_subtype {
  TKG_OK = 0,
  TKG_E_INVALID_MODE = 1,       /* InvalidModeError        (usage)     */
  TKG_E_DIMENSION_MISMATCH = 2, /* DimensionMismatchError  (usage)     */
  TKG_E_ZERO_REFERENCE = 3,     /* ZeroReferenceError      (usage)     */
  TKG_E_RANK_TOO_LARGE = 4,     /* RankTooLargeError       (numerical) */
  TKG_E_SINGULAR_GRAM = 5,      /* SingularGramError       (numerical) */
  TKG_E_DEGENERATE_INIT = 6,    /* DegenerateInitError     (numerical) */
  TKG_E_NO_CONVERGENCE = 7,     /* NoConvergenceError      (numerical) */
  TKG_E_IO = 8,                 /* IoError                 (io)        */
  TKG_E_FORMAT = 9,             /* FormatError             (io)        */
  TKG_E_CUDA = 11,              /* CUDA/NCCL runtime failure (io)      */
  TKG_E_UNSUPPORTED = 12        /* outside this build's limits (usage) */
};

typedef struct tkg_error {
  int32_t code;    /* = return value */
  int32_t subtype; /* enum tkg_subtype */
  char message[512];
} tkg_error;

/* AlsConfig (als.hpp:17-23). init: nullable host column-major warm start
 * of init_rows x init_cols (used by tkg_als_low_rank only, like the
 * reference's drivers which never set it); a shape other than I_mode x r is
 * rejected with DimensionMismatchError as als.cpp:106-113 does. */
typedef struct tkg_als_config {
  double eta;
  int32_t max_iters;
  uint64_t seed;
  const double* init;
  uint64_t init_rows;
  uint64_t init_cols;
} tkg_als_config;

/* FactorEngine (hosvd.hpp:19-27): kind + the ALS configuration (kAls only). */
enum tkg_engine_kind { TKG_ENGINE_SVD = 0, TKG_ENGINE_EIG = 1, TKG_ENGINE_ALS = 2 };
typedef struct tkg_factor_engine {
  int32_t kind; /* enum tkg_engine_kind */
  tkg_als_config als;
} tkg_factor_engine;

/* AlsReport + ModeReport (als.hpp:27-33, hosvd.hpp:33-37). status -1: the
 * mode's factor came from the SVD / EIG engine (ModeReport::als empty). */
typedef struct tkg_mode_report {
  int32_t mode;        /* 1-based */
  int32_t iterations;
  int32_t status;      /* 0 kConverged, 1 kMaxItersReached (als.hpp:25) */
  int32_t history_len; /* min(iterations, TKG_MAX_HISTORY) entries inline below;
                          the full history (one entry per sweep, als.cpp:137-138)
                          via tkg_residual_history */
  double achieved_eta;
  double seconds;      /* factor engine + working-tensor shrink */
  double residual_history[TKG_MAX_HISTORY];
} tkg_mode_report;

/* DecompositionReport (hosvd.hpp:39-44) plus device accounting. */
typedef struct tkg_report {
  int32_t order;
  int32_t n_modes;
  tkg_mode_report per_mode[TKG_MAX_ORDER]; /* processing order */
  double relative_residual; /* outside the timed region, as the reference */
  double seconds;           /* factor + core computation (hosvd.cpp:82,122) */
  double h2d_seconds;       /* host->device copy of a (0 when a_on_device) */
  double d2h_seconds;       /* core + factors device->host (t/st drivers: overlaps
                               the residual evaluation, on a copy stream) */
  double residual_seconds;  /* relative_residual evaluation (incl. the copies) */
  uint64_t kernel_launches; /* our kernels launched for the timed region */
  uint64_t tensor_passes;   /* full passes over the working tensor */
  uint64_t algorithmic_bytes; /* sum of 8*(|A| + F r + I r) per contraction pass */
} tkg_report;

typedef struct tkg_ctx tkg_ctx;

/* One context per device per thread. */
int tkg_create(tkg_ctx** ctx, int device, tkg_error* err);
int tkg_destroy(tkg_ctx* ctx);

/* t_hosvd with the ALS engine (FactorEngine::with_als). core: prod R_n
 * doubles; factors: concatenated I_n x R_n column-major in mode order.
 * want_singular_vectors: rotate every factor onto the leading left singular
 * vectors of its mode (recover_singular_vectors, hosvd.cpp:100-106). */
int tkg_t_hosvd(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order,
                const uint64_t* dims, const uint64_t* ranks, const tkg_als_config* cfg,
                int32_t want_singular_vectors, double* core, double* factors,
                tkg_report* report, tkg_error* err);

/* st_hosvd with the ALS engine. mode_order: nullable permutation of 1..N
 * (nullptr = select_order, i.e. std::nullopt). */
int tkg_st_hosvd(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order,
                 const uint64_t* dims, const uint64_t* ranks, const uint32_t* mode_order,
                 const tkg_als_config* cfg, double* core, double* factors, tkg_report* report,
                 tkg_error* err);

/* t_hosvd / st_hosvd with any factor engine. kSvd / kEig: the factor is the
 * leading R_n eigenvectors of A_(n) A_(n)^T (mode_gram on the device +
 * symmetric eigensolver), descending, signed as the reference
 * (kernels.cpp:25-43, 584-603). want_singular_vectors applies to kAls only. */
int tkg_t_hosvd_engine(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                       const uint64_t* ranks, const tkg_factor_engine* engine, int32_t want_singular_vectors,
                       double* core, double* factors, tkg_report* report, tkg_error* err);
int tkg_st_hosvd_engine(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                        const uint64_t* ranks, const uint32_t* mode_order, const tkg_factor_engine* engine,
                        double* core, double* factors, tkg_report* report, tkg_error* err);

/* hooi (HooiConfig{tol, max_iters}, hooi.hpp:15-18) from a warm start:
 * init_core prod R_n doubles, init_factors concatenated I_n x R_n (host).
 * Results: core, factors, *iterations, *converged, and fit_history[0 ..
 * iterations] (capacity max(1, max_iters) + 1; [0] = the warm start's fit),
 * *relative_residual (nullable) of the returned decomposition. */
int tkg_hooi(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
             const uint64_t* ranks, const double* init_core, const double* init_factors, double tol,
             int32_t max_iters, double* core, double* factors, int32_t* iterations, int32_t* converged,
             double* fit_history, double* relative_residual, tkg_error* err);

/* Device memory on the context's device, for FFI callers without a CUDA
 * runtime of their own (e.g. a TNSR loaded with tkg_read_tnsr and decomposed
 * with a_on_device = 1). tkg_device_copy: any direction (cudaMemcpyDefault),
 * synchronous on the context's stream. */
int tkg_device_alloc(tkg_ctx* ctx, uint64_t bytes, void** out, tkg_error* err);
int tkg_device_free(tkg_ctx* ctx, void* p);
int tkg_device_copy(tkg_ctx* ctx, void* dst, const void* src, uint64_t bytes, tkg_error* err);

/* ---- Sharded decomposition (one context per GPU, tensor split along its
 * last mode; BASELINE north star). The reference is single-process; these
 * entry points keep t_hosvd / st_hosvd's arguments and results (core and
 * factors replicated on every rank, identical to the single-GPU result of
 * the whole tensor) and add the slab this rank holds. */
typedef struct tkg_local_group tkg_local_group;

/* 128-byte NCCL unique id (create on one rank, broadcast to the others).
 * NCCL is loaded at run time (dlopen libnccl.so.2). */
int tkg_nccl_unique_id(void* out128, tkg_error* err);
/* Attach an NCCL communicator (rank of world) to ctx; collectives run on
 * the context's stream. */
int tkg_comm_init_nccl(tkg_ctx* ctx, int rank, int world, const void* unique_id128, tkg_error* err);
/* Host-staged multi-process group: every rank (a separate process with its
 * own context, on one GPU or several) passes the same POSIX shm `name`
 * ("/..."); collectives stage through slot_bytes per rank (0: 64 MiB) in
 * shared memory behind a process-shared barrier. Replaces NCCL where the
 * ranks have no NVLink peers (one-GPU pools, tests). */
int tkg_comm_init_shm(tkg_ctx* ctx, const char* name, int rank, int world, uint64_t slot_bytes, tkg_error* err);
/* In-process group: `world` contexts driven by `world` host threads of one
 * process (host-synchronous collectives; tests on a single device). */
int tkg_local_group_create(int world, tkg_local_group** out, tkg_error* err);
void tkg_local_group_destroy(tkg_local_group* g);
int tkg_comm_init_local(tkg_ctx* ctx, tkg_local_group* g, int rank, tkg_error* err);
/* Balanced split of an extent: rank holds [begin, begin + len). */
int tkg_shard_range(uint64_t extent, int rank, int world, uint64_t* begin, uint64_t* len);
/* a: this rank's slab dims[0..N-2] x [slab_begin, slab_begin + slab_len) of
 * the last mode (column-major, host or device), slab = tkg_shard_range of
 * dims[N-1]; dims: the GLOBAL shape. */
int tkg_t_hosvd_sharded(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                        uint64_t slab_begin, uint64_t slab_len, const uint64_t* ranks,
                        const tkg_als_config* cfg, int32_t want_singular_vectors, double* core,
                        double* factors, tkg_report* report, tkg_error* err);
int tkg_st_hosvd_sharded(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order, const uint64_t* dims,
                         uint64_t slab_begin, uint64_t slab_len, const uint64_t* ranks,
                         const uint32_t* mode_order, const tkg_als_config* cfg, double* core, double* factors,
                         tkg_report* report, tkg_error* err);

/* Full residual history of the mode at processing position `position`
 * (0-based) of the context's last tkg_t_hosvd* / tkg_st_hosvd* /
 * tkg_*_sharded / tkg_als_low_rank call: *len = its entry count (= that
 * mode's iterations, als.cpp:137-138); min(*len, cap) entries go to out
 * (nullable, to query the length). */
int tkg_residual_history(tkg_ctx* ctx, int32_t position, double* out, uint64_t cap, uint64_t* len,
                         tkg_error* err);

/* Stable ascending-rank order (Proposition 1). out: order entries. */
int tkg_select_order(int32_t order, const uint64_t* dims, const uint64_t* ranks, uint32_t* out,
                     tkg_error* err);

/* als_low_rank: l_out I_mode x r, r_out (nullable) fibers x r. */
int tkg_als_low_rank(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order,
                     const uint64_t* dims, uint32_t mode, uint64_t r, const tkg_als_config* cfg,
                     double* l_out, double* r_out, tkg_mode_report* report, tkg_error* err);

/* als_init: the randomized-range initializer, l_out I_mode x r. */
int tkg_als_init(tkg_ctx* ctx, const double* a, int a_on_device, int32_t order,
                 const uint64_t* dims, uint32_t mode, uint64_t r, uint64_t seed, double* l_out,
                 tkg_error* err);

/* als_sweep: one ALS sweep from l (I_mode x r): l_out = the updated left
 * factor, r_out (nullable, fibers x r) = this sweep's right factor,
 * *residual = the closed-form residual after the right update. A singular
 * normal equation raises SingularGramError with spd_solve's message. */
int tkg_als_sweep(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode,
                  const double* l, uint64_t r, double* l_out, double* r_out, double* residual, tkg_error* err);

/* Contraction primitives (host buffers). m is fibers x r (unfold_times) or
 * I_mode x r (unfold_t_times); u is rows x I_mode (mode_n_product). */
int tkg_unfold_times(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                     uint32_t mode, const double* m, uint64_t r, double* out, tkg_error* err);
int tkg_unfold_t_times(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                       uint32_t mode, const double* m, uint64_t r, double* out, tkg_error* err);
int tkg_mode_n_product(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                       const double* u, uint64_t rows, uint64_t cols, uint32_t mode, double* out,
                       tkg_error* err);
int tkg_frobenius_norm(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                       double* out, tkg_error* err);
int tkg_relative_error(tkg_ctx* ctx, const double* a, const double* b, int32_t order,
                       const uint64_t* dims, double* out, tkg_error* err);
int tkg_reduced_qr(tkg_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double* q,
                   double* r, tkg_error* err);
int tkg_gram(tkg_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double* out,
             tkg_error* err);
/* TNSR / TUKR files (io.cpp:131-224; little-endian, version 1). The shape
 * first (dims: TKG_MAX_ORDER entries), then the payload straight into dst:
 * a device buffer is filled through double-buffered pinned chunks whose H2D
 * copies overlap the file reads (dst_on_device = 1), or a host buffer.
 * Errors: IoError / FormatError with the reference's messages (category io). */
int tkg_read_tnsr_shape(const char* path, int32_t* order, uint64_t* dims, tkg_error* err);
int tkg_read_tnsr(tkg_ctx* ctx, const char* path, double* dst, int dst_on_device, tkg_error* err);
int tkg_write_tnsr(const char* path, int32_t order, const uint64_t* dims, const double* data, tkg_error* err);
/* core prod ranks doubles, factors concatenated dims[n] x ranks[n] (host). */
int tkg_write_tukr(const char* path, int32_t order, const uint64_t* dims, const uint64_t* ranks, const double* core,
                   const double* factors, tkg_error* err);

/* multi_mode_product: factor k is rows[k] x cols[k] (cols[k] = extent of
 * modes[k]), column-major host memory; applied in ascending mode order,
 * duplicate modes rejected (InvalidMode). out: the result, dims with
 * dims[modes[k]-1] replaced by rows[k]. */
int tkg_multi_mode_product(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, int32_t nfactors,
                           const uint32_t* modes, const double* const* factors, const uint64_t* rows,
                           const uint64_t* cols, double* out, tkg_error* err);
/* reconstruct: core (ranks) x_n U_n, factors concatenated dims[n] x ranks[n];
 * out has dims. */
int tkg_reconstruct(tkg_ctx* ctx, const double* core, int32_t order, const uint64_t* ranks, const uint64_t* dims,
                    const double* factors, double* out, tkg_error* err);
/* mode_gram: out = A_(mode) A_(mode)^T (extent x extent, column-major). */
int tkg_mode_gram(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims, uint32_t mode, double* out,
                  tkg_error* err);
/* sym_eig: the k leading eigenpairs of the symmetric n x n matrix g,
 * descending; vectors n x k column-major, each column's largest-magnitude
 * entry positive. */
int tkg_sym_eig(tkg_ctx* ctx, const double* g, uint64_t n, uint64_t k, double* values, double* vectors,
                tkg_error* err);
/* recover_singular_vectors: q (rows = I_mode x cols, orthonormal columns)
 * -> out = q V, V the left singular vectors of q^T A_(mode) in descending
 * order, each column's largest-magnitude entry positive (dense_svd's
 * convention, kernels.cpp:25-43). cols <= 64 and at least cols fibers. */
int tkg_recover_singular_vectors(tkg_ctx* ctx, const double* a, int32_t order, const uint64_t* dims,
                                 uint32_t mode, const double* q, uint64_t rows, uint64_t cols, double* out,
                                 tkg_error* err);
/* n draws of uniform01 from seeded_engine(seed, stream), generated on the
 * device by jump-ahead (the ALS initializer's stream). */
int tkg_uniform01(tkg_ctx* ctx, uint64_t seed, uint32_t stream, uint64_t n, double* out,
                  tkg_error* err);

/* Per-kernel-class device time (CUDA events on the launch stream) while
 * profiling is on. classes: 0 FC (ALS right update), 1 FR (left update /
 * init), 2 small LA, 3 RNG, 4 TTM outside the ALS loop (core chain, st TTM,
 * singular vectors), 5 relative-residual expansion, 6 fused sweep pass (right
 * update, R^T R and left-update sum from one read of the tensor, r <= 16),
 * 7 unused. */
#define TKG_KERNEL_CLASSES 8
typedef struct tkg_kernel_stats {
  double ms[TKG_KERNEL_CLASSES];
  uint64_t launches[TKG_KERNEL_CLASSES];
  double bytes[TKG_KERNEL_CLASSES]; /* algorithmic bytes */
  double flops[TKG_KERNEL_CLASSES]; /* algorithmic flops */
} tkg_kernel_stats;
int tkg_set_profiling(tkg_ctx* ctx, int on);
/* The fused sweep pass (ranks up to 16: right update, R^T R and left-update sum
 * from one read of the tensor) on / off for this context; off by default
 * unless the environment sets TKG_FUSED_SWEEP=1 (DESIGN.md has the
 * measurements). Results agree to rounding either way
 * (tests/test_gpu_fused.py). */
int tkg_set_fused_sweep(tkg_ctx* ctx, int on);
int tkg_get_kernel_stats(tkg_ctx* ctx, tkg_kernel_stats* out);

/* Device-side timing on the context's stream (CUDA events): start, then
 * stop returns the elapsed milliseconds (synchronizes). */
int tkg_timer_start(tkg_ctx* ctx);
int tkg_timer_stop(tkg_ctx* ctx, double* ms);
/* Overwrite a buffer larger than L2 on the context's stream (bench hygiene). */
int tkg_flush_l2(tkg_ctx* ctx);

/* Diagnostic: time the contraction kernels of one ALS sweep on a
 * device-resident tensor (d_a) along `mode` with r columns, `reps` times each
 * (CUDA events). out_ms (5 doubles): [0] mean FC (A_(n)^T L) launch, [1] mean
 * FR (A_(n) R) launch, [2] the init pass A_(n) S (S column-major) with the
 * fused ||A||^2, [3] the same without it, [4] the fused sweep pass (0 when
 * the shape does not take it). Used by tools/kernel_bench.py and
 * the ncu captures. */
int tkg_bench_contractions(tkg_ctx* ctx, const double* d_a, int32_t order, const uint64_t* dims,
                           uint32_t mode, uint32_t r, int32_t reps, double* out_ms,
                           tkg_error* err);

/* Library identification (build string, device name). */
const char* tkg_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TENKIT_B200_H */
