// Dense symmetric eigensolver (cuSOLVER syevd, loaded at run time) for the
// EIG / SVD factor engines. See eig.cpp.
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>

namespace tkg {

class SymEig {
 public:
  SymEig() = default;
  SymEig(const SymEig&) = delete;
  SymEig& operator=(const SymEig&) = delete;
  ~SymEig();
  // In place: G (n x n, column-major, device) -> eigenvectors, W (device) ->
  // eigenvalues ascending. Returns an empty string on success, else why.
  std::string eig(double* G, int n, double* W, cudaStream_t st);

 private:
  void* handle_ = nullptr;
  void* work_ = nullptr;
  size_t work_n_ = 0;
  void* info_ = nullptr;
};

}  // namespace tkg
