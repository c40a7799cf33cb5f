// Fiber contractions on the FP64 tensor pipe (DMMA m8n8k4), sm_100a.
//
//  FC  ("fiber contraction", reference unfold_t_times tensor_ops.cpp:263-330
//       and mode_n_product :129-169):
//        out(jl, c, p) = sum_i X(jl, i, p) * M[i][c]           c < nc
//      with out written through generic strides (R layout F x r, or the
//      tensor layout of a TTM), plus optional fused epilogues:
//        * per-CTA Gram partial  sum_j out(j,:)^T out(j,:)   (gram(R), matrix.cpp:90-126)
//        * per-CTA sum of squares of the output              (frobenius_norm, :391-393)
//        * diff-norm against a reference tensor instead of a store
//          (relative_error(t, reconstruct(tk)) without materialising it, :395-407)
//  FR  ("fiber reduction", reference unfold_times :193-261):
//        Y(i, c) = sum_{jl,p} X(jl, i, p) * Mr[(p*s + jl) + c*ldm]
//      split over fiber ranges into per-range partials that the consumer
//      sums in a fixed order (deterministic, like the reference's
//      chunk-ordered combine :254-259), optionally fusing sum X^2.
#pragma once

#include "common.cuh"

namespace tkg {

struct FcArgs {
  FiberView in;
  const double* mt;       // [K][ldmt] i-major contraction matrix, zero beyond nc
  uint32_t ldmt;          // >= NC
  double* out;            // output (nullable when only epilogue reductions are wanted)
  uint64_t os_j = 1;      // out(jl, c, p) = out[jl*os_j + c*os_c + p*os_p]
  uint64_t os_c, os_p;
  uint32_t nc;            // true output columns
  double* gram_part;      // [grid][NC*NC] (nullable)
  double* sumsq_part;     // [grid] (nullable)
  const double* diff_ref; // nullable: accumulate (diff_ref[o] - out)^2 instead of storing
  const int32_t* skip = nullptr;  // device flag: return at once when set
};

struct FrArgs {
  FiberView in;           // X(jl, i, p), i < K = I_n
  const double* m;        // Mr(j, c) = m[j*mj + c*mc], j = p*s + jl
  uint64_t mj, mc;
  uint32_t nc;
  uint64_t fibers_per_range;  // multiple of the kernel's chunk
  uint32_t ranges;
  uint32_t igroups;
  double* partial;        // [ranges][K][NCP] partial Y per fiber range
  uint32_t ncp;           // padded nc (row stride of partial)
  double* sumsq_part;     // [ranges*igroups] partial sum X^2 (nullable)
  const int32_t* skip = nullptr;  // device flag: return at once when set
};

// Host launchers (contract.cu). grid_hint = 0 picks the default persistent grid.
cudaError_t launch_fc(const FcArgs& a, int num_sms, cudaStream_t st, int* grid_used);
// Returns the number of fiber ranges (partials) written.
cudaError_t launch_fr(FrArgs a, int num_sms, cudaStream_t st, uint32_t* ranges_used,
                      uint32_t* grid_used);
// Pick the FR range count for a given view (so callers can size partials).
uint32_t fr_ranges_for(const FiberView& v, uint32_t nc, int num_sms);
int fc_grid_for(const FiberView& v, uint32_t nc, int num_sms);
uint32_t pad_nc(uint32_t nc);

}  // namespace tkg
