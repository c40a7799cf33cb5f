// Dense symmetric eigensolver on the device (eig.cu) for the EIG / SVD
// factor engines, HOOI and the sym_eig primitive (reference kernels.cpp:448-604).
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>

namespace tkg {

// Largest n the device eigensolver takes (shared-memory copies of the
// current column, reflectors and tridiagonal: 4n doubles per CTA).
constexpr int kSymEigMaxN = 6144;

class SymEig {
 public:
  SymEig() = default;
  SymEig(const SymEig&) = delete;
  SymEig& operator=(const SymEig&) = delete;
  ~SymEig();
  // The k leading eigenpairs of the symmetric n x n matrix G (column-major,
  // device, destroyed): U (n x k, device) in descending eigenvalue order with
  // each column's largest-magnitude entry positive, vals (k, device). Returns
  // an empty string on success, else why.
  std::string leading(double* G, int n, int k, double* U, double* vals, cudaStream_t st);

 private:
  void* work_ = nullptr;
  size_t work_n_ = 0;
};

}  // namespace tkg
