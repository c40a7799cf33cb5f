// Dense symmetric eigensolver for the EIG / SVD factor engines (reference
// sym_eig kernels.cpp:448-604, dense_svd :419-446): cuSOLVER's syevd on the
// device-resident I_n x I_n Gram matrix, loaded at run time (dlopen, like
// NCCL) so the library has no link-time dependency. A library call, as the
// task allows for plain dense linear algebra; the Gram matrix itself and the
// ordering / sign convention are our kernels (gram.cu, smallla.cu).
#include "eig.hpp"

#include <dlfcn.h>

#include <cusolverDn.h>  // types only

#include <mutex>
#include <string>

namespace tkg {

namespace {

struct Api {
  bool ok = false;
  std::string why;
  decltype(&cusolverDnCreate) create = nullptr;
  decltype(&cusolverDnDestroy) destroy = nullptr;
  decltype(&cusolverDnSetStream) set_stream = nullptr;
  decltype(&cusolverDnDsyevd_bufferSize) syevd_buffer = nullptr;
  decltype(&cusolverDnDsyevd) syevd = nullptr;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libcusolver.so.11", "libcusolver.so",
                           "/usr/local/cuda/lib64/libcusolver.so.11"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      a.why = "cuSOLVER (libcusolver.so.11) could not be loaded";
      return;
    }
    a.create = reinterpret_cast<decltype(a.create)>(dlsym(h, "cusolverDnCreate"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "cusolverDnDestroy"));
    a.set_stream = reinterpret_cast<decltype(a.set_stream)>(dlsym(h, "cusolverDnSetStream"));
    a.syevd_buffer = reinterpret_cast<decltype(a.syevd_buffer)>(dlsym(h, "cusolverDnDsyevd_bufferSize"));
    a.syevd = reinterpret_cast<decltype(a.syevd)>(dlsym(h, "cusolverDnDsyevd"));
    a.ok = a.create && a.destroy && a.set_stream && a.syevd_buffer && a.syevd;
    if (!a.ok) a.why = "cuSOLVER: missing cusolverDn symbols";
  });
  return a;
}

}  // namespace

SymEig::~SymEig() {
  if (handle_) api().destroy(static_cast<cusolverDnHandle_t>(handle_));
  if (work_) cudaFree(work_);
  if (info_) cudaFree(info_);
}

std::string SymEig::eig(double* G, int n, double* W, cudaStream_t st) {
  const Api& a = api();
  if (!a.ok) return a.why;
  if (!handle_) {
    cusolverDnHandle_t h = nullptr;
    if (a.create(&h) != CUSOLVER_STATUS_SUCCESS) return "cusolverDnCreate failed";
    handle_ = h;
  }
  auto h = static_cast<cusolverDnHandle_t>(handle_);
  if (a.set_stream(h, st) != CUSOLVER_STATUS_SUCCESS) return "cusolverDnSetStream failed";
  int lwork = 0;
  if (a.syevd_buffer(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, G, n, W, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return "cusolverDnDsyevd_bufferSize failed";
  if (size_t(lwork) > work_n_) {
    if (work_) cudaFree(work_);
    work_ = nullptr;
    if (cudaMalloc(&work_, sizeof(double) * size_t(lwork)) != cudaSuccess) return "cudaMalloc (syevd work) failed";
    work_n_ = size_t(lwork);
  }
  if (!info_ && cudaMalloc(&info_, sizeof(int)) != cudaSuccess) return "cudaMalloc (syevd info) failed";
  if (a.syevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, G, n, W, static_cast<double*>(work_), lwork,
              static_cast<int*>(info_)) != CUSOLVER_STATUS_SUCCESS)
    return "cusolverDnDsyevd failed";
  int info = 0;
  if (cudaMemcpyAsync(&info, info_, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return "syevd: status copy failed";
  if (info != 0) return "sym_eig: no convergence (syevd info " + std::to_string(info) + ")";
  return std::string();
}

}  // namespace tkg
