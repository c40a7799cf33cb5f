// Do DMMA (mma.sync m8n8k4 f64) and DFMA share one issue pipe on sm_100a?
// Each warp runs D DMMAs and X DFMAs per iteration on independent chains; the
// time per iteration tells whether the DFMAs hide under the DMMAs (separate
// pipes) or add to them (one pipe). Prints one JSON line per mix.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int D, int X>
__global__ void mix_kernel(double* out, int iters, double fa, double fb) {
  double acc[D > 0 ? D : 1][2];
  double x[X > 0 ? X : 1];
#pragma unroll
  for (int t = 0; t < (D > 0 ? D : 1); ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int k = 0; k < (X > 0 ? X : 1); ++k) x[k] = threadIdx.x * 1e-3 + k;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < D; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int k = 0; k < X; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;\n" : "+d"(x[k]) : "d"(fa), "d"(fb));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < (D > 0 ? D : 1); ++t) s += acc[t][0] + acc[t][1];
#pragma unroll
  for (int k = 0; k < (X > 0 ? X : 1); ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

// the same mix with the DFMAs dealt between the DMMAs (X / D after each)
template <int D, int X>
__global__ void alt_kernel(double* out, int iters, double fa, double fb) {
  double acc[D][2];
  double x[X];
#pragma unroll
  for (int t = 0; t < D; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int k = 0; k < X; ++k) x[k] = threadIdx.x * 1e-3 + k;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < D; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int k = 0; k < X / D; ++k)
        asm volatile("fma.rn.f64 %0, %0, %1, %2;\n" : "+d"(x[t * (X / D) + k]) : "d"(fa), "d"(fb));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < D; ++t) s += acc[t][0] + acc[t][1];
#pragma unroll
  for (int k = 0; k < X; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

template <int D, int X>
void run_alt(double* out, int sms, int blocks_per_sm, int threads) {
  const int iters = 2048, blocks = sms * blocks_per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best[2] = {1e30f, 1e30f};
  for (int alt = 0; alt < 2; ++alt)
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0));
      if (alt) alt_kernel<D, X><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      else mix_kernel<D, X><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0 && ms < best[alt]) best[alt] = ms;
    }
  printf("{\"dmma_per_iter\": %d, \"dfma_per_iter\": %d, \"warps_per_sm\": %d, \"ms_blocked\": %.4f, \"ms_alternating\": %.4f}\n",
         D, X, blocks_per_sm * threads / 32, best[0], best[1]);
}

template <int D, int X>
void run(double* out, int sms) {
  const int iters = 2048, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  mix_kernel<D, X><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    mix_kernel<D, X><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double warps = double(blocks) * threads / 32;
  const double dmma_tf = 2.0 * 256 * D * iters * warps / (best * 1e-3) / 1e12;
  const double dfma_tf = 2.0 * 32 * X * iters * warps / (best * 1e-3) / 1e12;
  printf("{\"dmma_per_iter\": %d, \"dfma_per_iter\": %d, \"ms\": %.4f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"sum_tflops\": %.2f}\n",
         D, X, best, dmma_tf, dfma_tf, dmma_tf + dfma_tf);
}

// dependent-issue latency: ONE warp on the device, D independent chains
template <int D>
void latency(double* out) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  mix_kernel<D, 0><<<1, 32>>>(out, iters, 1.0, 0.0);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  mix_kernel<D, 0><<<1, 32>>>(out, iters, 1.0, 0.0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  printf("{\"one_warp_chains\": %d, \"ns_per_round\": %.1f, \"cycles_per_round_at_max_clock\": %.1f}\n", D,
         ms * 1e6 / iters, ms * 1e-3 / iters * khz * 1e3);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  run<8, 0>(out, sms);
  run<0, 16>(out, sms);
  run<8, 4>(out, sms);
  run<8, 8>(out, sms);
  run<8, 16>(out, sms);
  run<8, 32>(out, sms);
  run<6, 4>(out, sms);
  run<7, 0>(out, sms);
  run_alt<8, 16>(out, sms, 8, 256);
  run_alt<8, 16>(out, sms, 1, 256);
  run_alt<4, 8>(out, sms, 1, 256);
  latency<1>(out);
  latency<2>(out);
  latency<4>(out);
  latency<8>(out);
  return 0;
}
