// Microbenchmark: cost of cooperative grid.sync at various grid sizes, and
// of a one-CTA r x r Gauss-Jordan inverse (the CTA-0 phase of coop.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/coop_microbench tools/coop_microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void syncs(int n, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int k = 0; k < n; ++k) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
}

// custom barrier: one atomic per CTA + spin on a generation flag
__device__ unsigned int g_count, g_gen;
__device__ __forceinline__ void bar_grid(unsigned int nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(&g_gen));
    unsigned int arrived = atomicAdd(&g_count, 1) + 1;
    if (arrived == nb) {
      g_count = 0;
      __threadfence();
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_gen), "r"(gen + 1));
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_gen));
      } while (cur == gen);
    }
  }
  __syncthreads();
}
__global__ void syncs2(int n, int* sink) {
  for (int k = 0; k < n; ++k) bar_grid(gridDim.x);
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
}

__global__ void gj(int r, int reps, double* out) {
  extern __shared__ double sm[];
  double* A = sm;
  double* B = sm + r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) A[e] = (e % r == e / r) ? r + 1.0 : 0.5;
  __syncthreads();
  for (int rep = 0; rep < reps; ++rep) {
    double* src = A;
    double* dst = B;
    for (int k = 0; k < r; ++k) {
      const double p = src[k + k * r];
      const double ip = 1.0 / p;
      for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
        const int i = e % r, j = e / r;
        const double aik = src[i + k * r], akj = src[k + j * r];
        double v;
        if (i == k) v = j == k ? ip : akj * ip;
        else if (j == k) v = -aik * ip;
        else v = fma(-aik * ip, akj, src[i + j * r]);
        dst[e] = v;
      }
      __syncthreads();
      double* t = src; src = dst; dst = t;
    }
  }
  if (threadIdx.x == 0) out[0] = A[0];
}

int main() {
  int* sink;
  double* out;
  cudaMalloc(&sink, 4);
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {1, 8, 32, 74, 148, 296}) {
    for (int n : {0, 100}) {
      void* args[] = {&n, &sink};
      cudaLaunchCooperativeKernel((void*)syncs, grid, 256, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)syncs, grid, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"bench\":\"cg_sync\",\"grid\":%d,\"n\":%d,\"us\":%.2f}\n", grid, n, ms * 1000);
      cudaLaunchCooperativeKernel((void*)syncs2, grid, 256, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)syncs2, grid, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"bench\":\"flag_sync\",\"grid\":%d,\"n\":%d,\"us\":%.2f}\n", grid, n, ms * 1000);
    }
  }
  // launch overhead: back-to-back empty kernels, cooperative vs regular launch
  for (int grid : {148}) {
    int n = 0;
    void* args[] = {&n, &sink};
    for (int kind = 0; kind < 2; ++kind) {
      for (int w = 0; w < 3; ++w) {
        if (kind == 0) cudaLaunchCooperativeKernel((void*)syncs, grid, 256, args, 0, 0);
        else syncs<<<grid, 256>>>(n, sink);
      }
      cudaEventRecord(a);
      for (int it = 0; it < 100; ++it) {
        if (kind == 0) cudaLaunchCooperativeKernel((void*)syncs, grid, 256, args, 0, 0);
        else syncs2<<<grid, 256>>>(n, sink);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"bench\":\"%s_launch\",\"grid\":%d,\"us_per_kernel\":%.2f}\n", kind ? "regular" : "cooperative",
             grid, ms * 1000 / 100);
    }
  }
  for (int r : {10, 32, 64}) {
    for (int reps : {1, 11}) {
      gj<<<1, 256, 2 * r * r * 8>>>(r, reps, out);
      cudaEventRecord(a);
      gj<<<1, 256, 2 * r * r * 8>>>(r, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"bench\":\"gj\",\"r\":%d,\"reps\":%d,\"us\":%.2f}\n", r, reps, ms * 1000);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
