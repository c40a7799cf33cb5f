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
  int32_t qr_fail1;        // CholQR2 first / second factorisation failed
  int32_t qr_fail2;
};

// ---- MT19937-64 (mtrng.cu) -------------------------------------------------
// Chunk c of J draws starts at position c*J; d_chunk_ids (nullable) lists the
// C chunks to compute (states and outputs are indexed by list slot).
cudaError_t launch_mt_states(const uint64_t* d_y, const uint64_t* d_polys, int C, const int* d_chunk_ids,
                             uint64_t* d_states, cudaStream_t st);
// nloc == 0: out[pos] (storage order). Otherwise the stream is the
// column-major Fg x r matrix S of a mode whose fibers j decompose as
// j = jlo + Plo*(ism + Gsm*jhi), ism the index along the sharded mode; one
// shard keeps ism in [o0, o0 + nloc), stored as its own local fiber order
// jlo + Plo*((ism - o0) + nloc*jhi), column c at c * (Fg / Gsm * nloc).
// ld > 0: the kept draws are written row-major, element (local fiber, c) at
// [fiber*ld + c] (the FR operand layout), instead of column-major.
// Whole tensor: Gsm = 1, o0 = 0, nloc = 1, Plo = Fg (mt_window_all).
struct MtWindow {
  uint64_t Fg = 0, Plo = 1, Gsm = 1, o0 = 0, nloc = 0, ld = 0;
  double inv_fg = 0.0, inv_plo = 0.0, inv_gsm = 0.0;  // set by mt_window_finish
};
inline MtWindow mt_window_finish(MtWindow w) {
  w.inv_fg = w.Fg ? 1.0 / double(w.Fg) : 0.0;
  w.inv_plo = w.Plo ? 1.0 / double(w.Plo) : 0.0;
  w.inv_gsm = w.Gsm ? 1.0 / double(w.Gsm) : 0.0;
  return w;
}
inline MtWindow mt_window_all(uint64_t F, uint64_t ld) {
  MtWindow w;
  w.Fg = F;
  w.Plo = F;
  w.Gsm = 1;
  w.o0 = 0;
  w.nloc = 1;
  w.ld = ld;
  return mt_window_finish(w);
}
cudaError_t launch_mt_generate(const uint64_t* d_states, int C, const int* d_chunk_ids, uint64_t J,
                               uint64_t total, double* d_out, MtWindow win, cudaStream_t st);

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
// floor_rel: pivot floor relative to max diag (1e-13 = spd_solve; 0 = only
// non-positive pivots fail, used by the CholQR2 factorisation).
cudaError_t launch_chol(const double* part, int nparts, uint64_t part_ld, int part_rowstride,
                        uint32_t r, double* G, double* chol, int32_t* flag, DevStatus* status,
                        cudaStream_t st, double floor_rel = 1e-13);



// Householder thin QR (kernels.cpp:303-367, R_ii >= 0) of Y (rows x r), where
// Y = sum of `nparts` FR partials [k][i][ldp] (or a column-major matrix when
// nparts == 0). Writes Q (col-major), R (r x r col-major), and R^T padded
// i-major into rt (nullable, ld ldrt) for the st-HOSVD shrink. When
// check_degenerate, sets status->degenerate_col per als.cpp:74-86.
// work: rows*r + rows*r + r doubles. only_if (nullable): the kernel returns at
// once while *only_if == 0 (the CholQR2 fast path's fallback, see
// Engine::qr_dev); degen_out (nullable) receives the collapse column too.
cudaError_t launch_qr(const double* Y, int nparts, uint64_t ldy_or_ldp, uint32_t rows, uint32_t r,
                      double* q, double* rmat, double* rt, uint32_t ldrt, double* work,
                      int check_degenerate, DevStatus* status, cudaStream_t st,
                      const int32_t* only_if = nullptr, int32_t* degen_out = nullptr);


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


// st-HOSVD shrink B_(n) <- R_hat R^T written in tensor layout (hosvd.cpp:176-178):
// out[jl + c*s + p*s*r] = sum_c' rhat[c + c'*r] * R[(p*s + jl)*ld + c'], plus
// per-CTA partial sums of squares of the output (the next mode's ||B||^2).
int shrink_count(uint64_t F);
// rhat_upper: rhat is upper triangular (a QR factor): the kernel skips the
// products with its zero blocks.
cudaError_t launch_shrink(const double* R, uint64_t ld, uint64_t s, uint64_t P, uint32_t r,
                          const double* rhat, double* out, double* sumsq_part, cudaStream_t st,
                          bool rhat_upper = false);

// Mode expansion out(jl, i, p) = sum_c in(jl, c, p) U[i + c*Iout] (recon.cu);
// with ref set, accumulates sum (ref - out)^2 per CTA instead of storing.
struct ExpandArgs {
  const double* in = nullptr;   // in[jl + c*s + p*s*K]
  uint64_t s = 1, P = 1;
  uint32_t K = 0;
  const double* U = nullptr;    // Iout x K column-major
  uint32_t Iout = 0;
  double* out = nullptr;        // out[jl + i*s + p*s*Iout]
  const double* ref = nullptr;
  double* sumsq_part = nullptr; // [grid]
};
int expand_grid(uint64_t F, int num_sms);
cudaError_t launch_expand(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used);

// Y = sum of FR partials, written column-major (rows x r).
cudaError_t launch_reduce_partials(const double* part, int nparts, uint32_t rows, uint32_t ldp,
                                   uint32_t r, double* y, cudaStream_t st);
// X (rows x cols, column-major) <- X with every column scaled to unit norm
// (zero columns are left as they are); one CTA per column, fixed-order sums.
cudaError_t launch_normalize_columns(double* X, uint32_t rows, uint32_t cols, cudaStream_t st);

// recover_singular_vectors (hosvd.cpp:65-72): eigenvectors of the symmetric
// r x r matrix G (column-major, r <= 64) by parallel cyclic Jacobi, ordered by
// descending eigenvalue and signed per fix_column_signs (kernels.cpp:25-43).
// Writes V^T column-major (vt[c + i*r] = V(i, c)) and, when evals is set, the
// eigenvalues in that order.
cudaError_t launch_sym_eig(const double* G, uint32_t r, double* vt, double* evals, cudaStream_t st);

// ---- mode_gram (gram.cu, tensor_ops.cpp:332-389) ------------------------------
// G = A_(n) A_(n)^T (K x K column-major) from the tensor's natural layout:
// 64 x 64 upper-triangle blocks x fiber splits on DMMA, partials reduced in a
// fixed order.
struct GramPlan {
  int nb = 0, npairs = 0, nsplit = 0;
  uint64_t per_split = 0;
  size_t part_doubles = 0;
};
GramPlan gram_tensor_plan(const FiberView& v, int num_sms);
cudaError_t launch_gram_tensor(const FiberView& v, const GramPlan& p, double* part, double* G, cudaStream_t st);

// ---- sharded decomposition (smallla.cu) -------------------------------------
cudaError_t launch_add(double* dst, const double* src, size_t n, cudaStream_t st);
// part[0][i][c] = sum over the nparts FR partials [k][I][ldp] (c < r), in place.
cudaError_t launch_reduce_slot0(double* part, int nparts, uint32_t I, uint32_t ldp, uint32_t r, cudaStream_t st);
// G (column-major r x r) = sum_k part[k*pld + a*rs + b] (upper entries a <= b).
cudaError_t launch_gram_reduce(const double* part, int nparts, uint64_t pld, uint32_t rs, uint32_t r, double* G,
                               cudaStream_t st);
struct BoxCopy {
  int N = 0;
  uint64_t box[64] = {0};
  uint64_t src_stride[64] = {0}, dst_stride[64] = {0};
  uint64_t src_base = 0, dst_base = 0;
};
cudaError_t launch_copy_box(const double* src, double* dst, const BoxCopy& b, cudaStream_t st);

}  // namespace tkg
