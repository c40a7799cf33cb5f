// Shared device helpers for the B200 ALS-HOSVD kernels (sm_100a).
//
// Layout vocabulary (reference tensor_ops.cpp:16-39 "FiberSpace"): for mode n
// of a column-major tensor, s = prod_{m<n} I_m fibers share a panel, the
// contraction index i runs over I_n with stride s, and P = prod_{m>n} I_m
// panels follow each other. Fiber j = p*s + jl starts at jl + p*s*I_n.
// Every kernel here addresses its operand through the generic strided view
//   X(jl, i, p) = base[jl + i*is_i + p*is_p],  jl < s, i < K, p < P,
// which covers the tensor's mode-n fibers (is_i = s, is_p = s*I_n) and the
// F x r factor R read back as a tensor (is_i = F, is_p = s) in the
// st-HOSVD shrink.
#pragma once

#include <map>
#include <mutex>
#include <utility>

#include <cstdint>
#include <cuda_runtime.h>

namespace tkg {

constexpr int kWarp = 32;

struct FiberView {
  const double* base;
  uint64_t s;     // fibers per panel
  uint64_t P;     // panels
  uint32_t K;     // contraction extent
  uint64_t is_i;  // stride of the contraction index
  uint64_t is_p;  // stride between panels
};

#ifdef __CUDACC__
// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor pipe (DMMA).
// Fragment layout (PTX ISA, mma.m8n8k4 .f64): a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = {D[lane/4][2*(lane%4)], D[lane/4][2*(lane%4)+1]}.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Error-free transformation a + b = s + e (Knuth TwoSum); used for
// compensated reductions of the closed-form residual terms.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

#endif  // __CUDACC__

// Shared-memory leading dimension (in doubles) for an [rows][nc] operand
// read as DMMA B fragments: 4 consecutive rows must land 4 doubles apart
// modulo the 16-double bank window, i.e. ld = 4 (mod 16).
__host__ __device__ constexpr int smem_ld(int nc) { return nc + ((4 - nc) % 16 + 16) % 16; }

// Programmatic dependent launch (the kernels' griddepcontrol.wait) for the
// contraction grids and the small steps. Off while an engine records per-launch
// CUDA events (bench.py's per-class pass): a PDL launch starts early and its
// event interval would include the wait for the previous kernel.
int& pdl_off_count();
inline bool pdl_enabled() { return pdl_off_count() == 0; }

// Raise a kernel's dynamic shared-memory limit to at least `bytes` (never
// lowers it): several host threads sharing a device (in-process ranks) may
// launch one kernel with different sizes, and a per-call set could lower the
// limit under another thread's launch.
template <class K>
inline cudaError_t raise_smem_limit(K kernel, size_t bytes) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, size_t> cur;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(m);
  size_t& c = cur[{reinterpret_cast<const void*>(kernel), dev}];
  if (bytes <= c) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  c = bytes;
  return cudaSuccess;
}

}  // namespace tkg
