// Microbenchmark of the cooperative small-LA steps (coop.cu) in isolation:
// CholQR2 of an I x r matrix (column-major or from split-K partials) and the
// prep step from partials. Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=false \
//     -Ipaper_2004_02583_b200/csrc tools/small_bench.cu \
//     paper_2004_02583_b200/csrc/coop.cu paper_2004_02583_b200/csrc/als_step.cu -o tools/small_bench
#include <cstdio>
#include <vector>
#include <random>
#include <cstdlib>

#include "als_step.cuh"
#include "coop.cuh"

namespace tkg {
void phase_read(unsigned long long* out);
}
using namespace tkg;

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { uint32_t I, r; int nparts; };
  for (Case c : {Case{256, 10, 0}, Case{256, 10, 78}, Case{1024, 32, 0}, Case{1024, 32, 37}, Case{2048, 64, 0},
                 Case{200, 50, 0}, Case{200, 50, 40}, Case{200, 50, 148}, Case{200, 50, 296}}) {
    const uint32_t ncp = (c.r + 7) / 8 * 8;
    const int np = std::max(c.nparts, 1);
    std::vector<double> h(size_t(np) * c.I * ncp);
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> u(-1, 1);
    for (auto& x : h) x = u(g);
    double *Y, *Q, *gpart, *gs, *L1, *Rinv, *work, *Lc, *GL, *GLinv, *GRinv, *Mt;
    AlsCtrl* ctrl;
    cudaMalloc(&Y, h.size() * 8);
    cudaMalloc(&Q, size_t(c.I) * c.r * 8);
    cudaMalloc(&gpart, size_t(sms) * 8 * 64 * 64 * 8);
    cudaMalloc(&gs, 64 * 64 * 8);
    cudaMalloc(&L1, 64 * 64 * 8);
    cudaMalloc(&Rinv, 64 * 64 * 8);
    cudaMalloc(&work, 16);
    cudaMalloc(&Lc, size_t(c.I) * c.r * 8);
    cudaMalloc(&GL, 64 * 64 * 8);
    cudaMalloc(&GLinv, 64 * 64 * 8);
    cudaMalloc(&GRinv, 64 * 64 * 8);
    cudaMalloc(&Mt, size_t(c.I) * ncp * 8);
    cudaMalloc(&ctrl, sizeof(AlsCtrl));
    cudaMemset(ctrl, 0, sizeof(AlsCtrl));
    std::vector<double> eye(c.r * c.r, 0.0);
    for (uint32_t i = 0; i < c.r; ++i) eye[i + i * c.r] = 1.0;
    cudaMemcpy(GRinv, eye.data(), eye.size() * 8, cudaMemcpyHostToDevice);
    auto upload = [&] { cudaMemcpyAsync(Y, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st); };
    for (int kind = 0; kind < 2; ++kind) {
      if (kind == 1 && c.nparts == 0) continue;
      float tot = 0;
      const int reps = 20;
      for (int rep = 0; rep < reps + 2; ++rep) {
        upload();
        cudaEventRecord(a, st);
        cudaError_t e;
        if (kind == 0) {
          CholQrArgs q;
          q.Y = Y; q.nparts = c.nparts; q.ldp = c.nparts ? ncp : c.I; q.I = c.I; q.r = c.r; q.Q = Q;
          q.check = 1; q.gpart = gpart; q.gs = gs; q.L1 = L1; q.Rinv = Rinv; q.work = work; q.ctrl = ctrl;
          e = launch_cholqr_step(q, sms, st);
        } else {
          PrepArgs p;
          p.part = Y; p.nparts = c.nparts; p.ldp = ncp; p.GRinv = GRinv; p.from_partials = 1; p.I = c.I;
          p.r = c.r; p.ncp = ncp; p.Lc = Lc; p.GL = GL; p.GLinv = GLinv; p.Mt = Mt; p.gpart = gpart; p.gs = gs;
          p.ctrl = ctrl;
          e = launch_prep_step(p, sms, st);
        }
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 2) tot += ms;
      }
      printf("{\"kernel\":\"%s\",\"I\":%u,\"r\":%u,\"nparts\":%d,\"us\":%.2f}\n", kind ? "prep" : "cholqr", c.I, c.r,
             c.nparts, tot / reps * 1000);
      {
        unsigned long long ph[64];
        phase_read(ph);
        printf("   phases(us):");
        const bool grid_steps = getenv("TKG_COOP_STEPS") && getenv("TKG_COOP_STEPS")[0] == '1';
        const int k0 = grid_steps ? (kind == 0 ? 1 : 21) : (kind == 0 ? 41 : 31);
        const int k1 = grid_steps ? (kind == 0 ? 12 : 27) : (kind == 0 ? 49 : 35);
        for (int k = k0; k < k1; ++k) printf(" %d:%.1f", k, (ph[k] - ph[k - 1]) * 1e-3);
        printf("\n");
      }
    }
    cudaFree(Y); cudaFree(Q); cudaFree(gpart); cudaFree(gs); cudaFree(L1); cudaFree(Rinv); cudaFree(work);
    cudaFree(Lc); cudaFree(GL); cudaFree(GLinv); cudaFree(GRinv); cudaFree(Mt); cudaFree(ctrl);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
