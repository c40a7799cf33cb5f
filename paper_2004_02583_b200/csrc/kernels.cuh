// Launchers for the small dense kernels around the fiber contractions.
// All of them keep the reference's numerical semantics (pivot floors, sign
// conventions, degeneracy checks) — see each definition for the citation.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "contract.cuh"

namespace tkg {

// Device-written status of one ALS step, read by the host once per sweep
// (lives in mapped pinned memory).
struct DevStatus {
  double sumsq;          // ||working tensor||_F^2
  double residual;       // closed-form residual (als.cpp:52-55)
  double trace;          // trace(G_L G_R)
  double pivot;          // failing Cholesky pivot (for the message)
  int32_t right_singular;  // chol(L^T L) hit the pivot floor
  int32_t left_singular;   // chol(R^T R) hit the pivot floor
  int32_t degenerate_col;  // als_init collapse column (1-based), 0 if none
  int32_t pad;
};

// ---- MT19937-64 (mtrng.cu) -------------------------------------------------
cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C,
                             uint64_t* d_states, cudaStream_t st);
cudaError_t launch_mt_generate(const uint64_t* d_states, int C, uint64_t J, uint64_t total,
                               double* d_out, cudaStream_t st);

// ---- small dense LA (smallla.cu) -------------------------------------------
// part[b] = upper triangle of X_b^T X_b over row blocks of X (rows x r, col-major, ld).
// Returns the number of partials written.
int gram_partials_count(uint32_t rows);
cudaError_t launch_gram_partials(const double* X, uint64_t ld, uint32_t rows, uint32_t r,
                                 double* part, cudaStream_t st);

// G = sum of `nparts` upper-triangle partials (fixed order, lower mirrored),
// chol = lower Cholesky factor with the spd_solve pivot floor
// (kernels.cpp:378-393). On failure sets *flag = 1 and status->pivot.
// part_ld: stride between consecutive partials (>= r*r), part_rowstride:
// row stride inside a partial (r for gram_partials, NC for FC Gram partials).
cudaError_t launch_chol(const double* part, int nparts, uint64_t part_ld, int part_rowstride,
                        uint32_t r, double* G, double* chol, int32_t* flag, DevStatus* status,
                        cudaStream_t st);

// Row-wise SPD solve X(i,:) = B(i,:) G^{-1} via the Cholesky factor, with
// forward/back substitution in the order of spd_solve (kernels.cpp:398-415).
// B is either the sum of `nparts` partials part[k][i][ldp] (FR output) or a
// column-major matrix (nparts == 0: B[i + c*ldb]).
// Output: column-major X (x_cm, ld = rows) and/or i-major padded Xt (xt, ldxt).
cudaError_t launch_row_solve(const double* B, int nparts, uint64_t ldb_or_ldp, uint32_t rows,
                             uint32_t r, const double* chol, double* x_cm, double* xt,
                             uint32_t ldxt, const int32_t* skip_flag, cudaStream_t st);

// Householder thin QR (kernels.cpp:303-367, R_ii >= 0) of Y (rows x r), where
// Y = sum of `nparts` FR partials [k][i][ldp] (or a column-major matrix when
// nparts == 0). Writes Q (col-major), R (r x r col-major), and R^T padded
// i-major into rt (nullable, ld ldrt) for the st-HOSVD shrink. When
// check_degenerate, sets status->degenerate_col per als.cpp:74-86.
// work: rows*r + rows*r + r doubles.
cudaError_t launch_qr(const double* Y, int nparts, uint64_t ldy_or_ldp, uint32_t rows, uint32_t r,
                      double* q, double* rmat, double* rt, uint32_t ldrt, double* work,
                      int check_degenerate, DevStatus* status, cudaStream_t st);

// Closed-form residual step after the right update (als.cpp:36-44,52-55):
// G_R = reduce(FC Gram partials), trace(G_L G_R) (compensated), residual,
// and chol(G_R) for the left update (flag on failure).
cudaError_t launch_finish_right(const double* fc_gram, int nparts, int nc_stride, uint32_t r,
                                const double* GL, const double* norm_sq, double* GR,
                                double* cholR, DevStatus* status, cudaStream_t st);

// out[0] = sum of `n` partials in fixed order (into status->sumsq when dst null).
cudaError_t launch_sum(const double* partials, int n, double* dst, cudaStream_t st);

// dst[row*ldd + col] = src[row*rs + col*cs] for col < cols, 0 for cols <= col < ldd.
// (transpose-and-pad of a factor into the i-major operand layout of FC.)
cudaError_t launch_pack(const double* src, uint64_t rs, uint64_t cs, uint32_t rows, uint32_t cols,
                        double* dst, uint32_t ldd, cudaStream_t st);

// part[b] = sum of x[k]^2 over block b of a flat array; returns #partials.
int sumsq_partials_count(uint64_t n);
cudaError_t launch_sumsq(const double* x, uint64_t n, double* part, cudaStream_t st);
// part[b] = sum of (b[k] - a[k])^2 over block b (same blocking as launch_sumsq).
cudaError_t launch_sumsq_diff(const double* a, const double* b, uint64_t n, double* part,
                              cudaStream_t st);

// Y = sum of FR partials, written column-major (rows x r).
cudaError_t launch_reduce_partials(const double* part, int nparts, uint32_t rows, uint32_t ldp,
                                   uint32_t r, double* y, cudaStream_t st);

}  // namespace tkg
