/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement ("port") of the reference's ALS-HOSVD hot path
 * (tenkit, arXiv 2004.02583), used only as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. The product path
 * (paper_2004_02583_b200/) never links or calls it.
 *
 * Every function follows the reference loop-for-loop (same summation
 * orders, same chunking), so its results are pinned BITWISE against the
 * compiled reference in oracle/_ref (tests/test_oracle_pins.py) and against
 * the reference's own known-answer tests (tests/golden/).
 *
 * Layout: tensors are flat column-major doubles, first index fastest
 * (tensor.hpp:10-11); matrices column-major (matrix.hpp:8-9); modes 1-based
 * (shape.hpp:10-14). Status codes: 0 ok, else ErrorCategory+1
 * (errors.hpp:10: usage=1, io=2, numerical=3) with *subtype set to one of
 * ORC_E_* and a message.
 */
#ifndef TENKIT_ORACLE_H
#define TENKIT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_E_INVALID_MODE = 1,
  ORC_E_DIMENSION_MISMATCH = 2,
  ORC_E_ZERO_REFERENCE = 3,
  ORC_E_RANK_TOO_LARGE = 4,
  ORC_E_SINGULAR_GRAM = 5,
  ORC_E_DEGENERATE_INIT = 6,
  ORC_E_NO_CONVERGENCE = 7,
  ORC_E_OTHER = 10
};

typedef struct {
  int subtype;
  char msg[256];
} orc_error;

/* ---- rng.hpp ---------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

/* seeded_engine(seed, stream): std::mt19937_64 seeded from
 * std::seed_seq{lo32(seed), hi32(seed), stream} (rng.hpp:57-61). */
void orc_mt64_seeded(orc_mt64* eng, uint64_t seed, uint32_t stream);
uint64_t orc_mt64_next(orc_mt64* eng);
double orc_uniform01(orc_mt64* eng);                          /* rng.hpp:19-21 */
double orc_uniform_in(orc_mt64* eng, double lo, double hi);   /* rng.hpp:24-26 */
/* n draws of GaussianStream (rng.hpp:30-53) from seeded_engine(seed, stream). */
void orc_gaussian_fill(uint64_t seed, uint32_t stream, double* out, size_t n);

/* ---- tensor_ops.cpp ---------------------------------------------------- */
double orc_sum_sq(const double* x, size_t n);                 /* :45-59 */
double orc_frobenius_norm(const double* a, size_t n);         /* :391-393 */
int orc_relative_error(const double* a, const double* b, size_t n,
                       double* out, orc_error* err);          /* :395-407 */
int orc_unfold_times(const double* a, int order, const uint64_t* dims,
                     int mode, const double* m, size_t r, double* out,
                     orc_error* err);                         /* :193-261 */
int orc_unfold_t_times(const double* a, int order, const uint64_t* dims,
                       int mode, const double* m, size_t r, double* out,
                       orc_error* err);                       /* :263-330 */
/* out = t x_mode u, u is rows x cols with cols == I_mode (:129-169). */
int orc_mode_n_product(const double* a, int order, const uint64_t* dims,
                       const double* u, size_t rows, size_t cols, int mode,
                       double* out, orc_error* err);
/* core x_1 U1 ... x_N UN with factors concatenated (I_n x R_n each). */
int orc_reconstruct(const double* core, int order, const uint64_t* ranks,
                    const uint64_t* dims, const double* factors, double* out,
                    orc_error* err);                          /* :420-440 */

/* ---- matrix.cpp -------------------------------------------------------- */
void orc_gram(const double* a, size_t rows, size_t cols, double* out); /* :90-126 */
void orc_matmul(const double* a, size_t m, size_t k, const double* b,
                size_t n, double* out);                        /* :42-69 */
void orc_transpose(const double* a, size_t rows, size_t cols, double* out);

/* ---- kernels.cpp ------------------------------------------------------- */
int orc_reduced_qr(const double* a, size_t m, size_t n, double* q, double* r,
                   orc_error* err);                            /* :303-367 */
int orc_spd_solve(const double* g, size_t n, const double* b, size_t k,
                  double* x, orc_error* err);                  /* :369-417 */

/* ---- als.cpp ------------------------------------------------------------ */
int orc_als_init(const double* a, int order, const uint64_t* dims, int mode,
                 size_t r, uint64_t seed, double* l_out, orc_error* err);
typedef struct {
  int iterations;
  int status; /* 0 converged, 1 max iters (als.hpp:25) */
  double achieved_eta;
  double history[64]; /* first min(iterations, 64) residuals */
} orc_als_report;
/* l_out: I_mode x r; r_out: fibers x r (nullable). init nullable. */
int orc_als_low_rank(const double* a, int order, const uint64_t* dims,
                     int mode, size_t r, double eta, int max_iters,
                     uint64_t seed, const double* init, double* l_out,
                     double* r_out, orc_als_report* rep, orc_error* err);

/* ---- hosvd.cpp ---------------------------------------------------------- */
void orc_select_order(int order, const uint64_t* ranks, int* out_order);
typedef struct {
  int modes[64]; /* processing order */
  orc_als_report als[64];
  double relative_residual;
} orc_hosvd_report;
/* sequential=0: t_hosvd (:74-125); 1: st_hosvd (:127-191).
 * mode_order nullable (= select_order). core_out: prod R_n; factors_out:
 * concatenated I_n x R_n in mode order. */
/* hosvd.cpp:65-72; q is rows x r (rows = extent of mode). */
int orc_recover_singular_vectors(const double* a, int order, const uint64_t* dims, int mode,
                                 const double* q, size_t rows, size_t r, double* out,
                                 orc_error* err);
/* sequential: 0 t_hosvd, 1 st_hosvd, 2 t_hosvd with want_singular_vectors */
int orc_hosvd_als(int sequential, const double* a, int order,
                  const uint64_t* dims, const uint64_t* ranks,
                  const int* mode_order, double eta, int max_iters,
                  uint64_t seed, double* core_out, double* factors_out,
                  orc_hosvd_report* rep, orc_error* err);

#ifdef __cplusplus
}
#endif

#endif
