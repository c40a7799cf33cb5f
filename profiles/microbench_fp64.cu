// Microbenchmarks that set the FP64 roofline denominators on the box:
// DFMA throughput, DMMA (mma.sync m8n8k4 f64) throughput, streaming HBM read,
// and cuBLAS DGEMM for context. Prints one JSON line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { acc[t][0] = 0; acc[t][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += acc[t][0] + acc[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) acc[t][q] = 0;
  double a[8], b[4];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
#pragma unroll
  for (int q = 0; q < 4; ++q) b[q] = 1.0 - threadIdx.x * 1e-4 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) s += acc[t][q];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double2 acc = make_double2(0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(in + i);
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x + acc.y == 12345.678) out[0] = acc.x;
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  const int iters = 4096;
  // DFMA: 16 independent chains per thread, 256 threads/block, 8 blocks/SM.
  int blocks = sms * 8, threads = 256;
  float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); }, 5);
  double dfma_tf = 2.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
  ms = time_ms([&] { dmma_kernel<<<blocks, threads>>>(out, iters); }, 5);
  double dmma_tf = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  ms = time_ms([&] { dmma16_kernel<<<blocks, threads>>>(out, iters / 2); }, 5);
  double dmma16_tf = 2.0 * 2048 * 4 * (iters / 2) * (double)blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  size_t n = (size_t)1 << 30;  // 8 GiB of doubles
  double2* buf; CK(cudaMalloc(&buf, n * sizeof(double)));
  CK(cudaMemset(buf, 0, n * sizeof(double)));
  ms = time_ms([&] { read_kernel<<<sms * 8, 512>>>(buf, n / 2, out); }, 5);
  double read_gbs = n * 8.0 / (ms * 1e-3) / 1e9;
  // cuBLAS DGEMM 8192^3
  cublasHandle_t h; cublasCreate(&h);
  int N = 8192; double *A, *B, *C; CK(cudaMalloc(&A, (size_t)N * N * 8)); CK(cudaMalloc(&B, (size_t)N * N * 8)); CK(cudaMalloc(&C, (size_t)N * N * 8));
  CK(cudaMemset(A, 0, (size_t)N * N * 8)); CK(cudaMemset(B, 0, (size_t)N * N * 8));
  double one = 1, zero = 0;
  ms = time_ms([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N); }, 3);
  double dgemm_tf = 2.0 * N * (double)N * N / (ms * 1e-3) / 1e12;
  // tall-skinny DGEMM like the ALS contraction: (1M x 1024) * (1024 x 32)
  size_t M = 1 << 20; int K = 1024, Nn = 32;
  double* Ab = (double*)buf; double *Lb, *Rb; CK(cudaMalloc(&Lb, K * Nn * 8)); CK(cudaMalloc(&Rb, M * Nn * 8));
  CK(cudaMemset(Lb, 0, K * Nn * 8));
  ms = time_ms([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)M, Nn, K, &one, Ab, (int)M, Lb, K, &zero, Rb, (int)M); }, 5);
  double ts_tf = 2.0 * M * Nn * K / (ms * 1e-3) / 1e12;
  double ts_ms = ms;
  printf("{\"sms\": %d, \"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, \"hbm_read_gbs\": %.1f, \"cublas_dgemm_8192_tflops\": %.2f, \"cublas_dgemm_tallskinny_1Mx1024x32_tflops\": %.2f, \"cublas_ts_ms\": %.3f}\n",
         sms, dfma_tf, dmma_tf, dmma16_tf, read_gbs, dgemm_tf, ts_tf, ts_ms);
  return 0;
}
