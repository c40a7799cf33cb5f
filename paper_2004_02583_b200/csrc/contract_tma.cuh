// TMA-fed FC / FR kernels (contract_tma.cu). The FC output / FR operand
// conventions match contract.cuh; FR's small operand M may be row-major
// (R) or column-major (the initializer's S) and is addressed by strides.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace tkg {

enum TmaMode { kFibI = 0, kFibJ = 1, kFibS = 2 };

struct FcTmaArgs {
  uint64_t s = 0, P = 0;
  uint32_t K = 0;
  uint32_t nc = 0;
  double* out = nullptr;                       // out[jl*os_j + c*os_c + p*os_p]
  uint64_t os_j = 1, os_c = 0, os_p = 0;
  double* sumsq_part = nullptr;                // [grid]
  const double* diff_ref = nullptr;            // diff-norm epilogue instead of a store
  const int32_t* skip = nullptr;               // device flag: return at once when set
  double* gram_part = nullptr;                 // [grid][NC*NC] upper tiles of out^T out (NC <= 32)
  // kFibS (short panels): a tile is pc whole panels (pc*s <= 128 fibers), the
  // A box {sb, 32, pc} (sb >= s, TMA zero-fills past s); runtime stage sizes
  uint32_t pc = 1, sb = 0, bytes_a = 0, stage_bytes = 0;
  // kFibS, straddle = 1: a tile is 128 consecutive fibers whatever panels they
  // fall in (every tile row live); its box starts at the first fiber's panel
  // and spans pc panels
  uint32_t straddle = 0;
};

// NC (padded column count) up to which the FC kernel can fuse the Gram of
// its output into the epilogue.
constexpr uint32_t kFcGramMaxNc = 32;

struct FrTmaArgs {
  uint64_t s = 0, P = 0;
  uint32_t K = 0;
  uint32_t nc = 0;
  uint64_t fibers_per_range = 0;
  uint32_t ranges = 0, igroups = 0;
  double* partial = nullptr;                   // [ranges][K][ncp]
  uint32_t ncp = 0;
  double* sumsq_part = nullptr;                // [ranges*igroups]
  const int32_t* skip = nullptr;               // device flag: return at once when set
  // kFibS (short panels): a chunk is pc whole panels (kf = pc*s <= 64 fibers),
  // ranges are panel ranges; A box {s, 128, pc}; runtime sizes
  uint32_t pc = 1, kf = 0, bytes_a = 0, bytes_m = 0, stage_bytes = 0, ldm = 0;
  uint64_t panels_per_range = 0;
};

// -1 when the layout is not covered (the caller uses contract.cu's kernels).
int fc_tma_mode(const FiberView& v, const double* mt, uint32_t ldmt);
int fr_tma_mode(const FiberView& v, const double* m, uint64_t mj, uint64_t mc);
int fc_tma_grid(const FiberView& v, int num_sms);
uint32_t fr_tma_ranges(const FiberView& v, int num_sms);
bool fr_wide_ok(const FiberView& v, uint32_t ncp, int mode);
bool dfma_tail(uint32_t nc);  // the last column tile of nc columns runs as a DFMA tail

cudaError_t launch_fc_tma(const FiberView& v, const double* mt, uint32_t ldmt, FcTmaArgs a, int mode,
                          int num_sms, cudaStream_t st, int* grid_used);
// M(j, c) = m[j*mj + c*mc]; TMA needs mc == 1 (row-major) or mj == 1 (column-major).
cudaError_t launch_fr_tma(const FiberView& v, const double* m, uint64_t mj, uint64_t mc, FrTmaArgs a,
                          int mode, int num_sms, cudaStream_t st, uint32_t* ranges_used,
                          uint32_t* grid_used);

// Last-mode expansion fused with the difference norm against a.ref (P == 1,
// even F and Iout, K <= 64); sumsq_part[grid].
bool expand_diff_tma_ok(const ExpandArgs& a);
int expand_diff_tma_grid(uint64_t F, int num_sms);
cudaError_t launch_expand_diff_tma(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used);
// intermediate-mode expansion (a.ref null, a.out set), s even
bool expand_tma_ok(const ExpandArgs& a);
int expand_tma_grid(uint64_t s, uint64_t P, int num_sms);
cudaError_t launch_expand_tma(const ExpandArgs& a, int num_sms, cudaStream_t st, int* grid_used);

}  // namespace tkg
