// tphase_probe.cu — the fused MVM's Toeplitz phase (f2_toeplitz) run alone as
// an ordinary kernel at several grid sizes: per-item cost vs latency.
#include "../paper_1810_12283_b200/csrc/fused2d.cu"

#include <cstdio>
#include <vector>

namespace gk {
namespace {
__global__ void __launch_bounds__(256, 2) k_tprobe(const double* t, int M, int Mp, int P, int Q, const double* X,
                                                   double* Y, int nsplit, unsigned long long* stamps) {
  extern __shared__ __align__(16) double sm[];
  double* ts = sm;
  for (int i = threadIdx.x; i < Mp; i += 256) ts[i] = i < M ? t[i] : 0.0;
  __syncthreads();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  f2_toeplitz(ts, M, Mp, M, P, Q, X, HaloSpec{nullptr, 1, 0, 6}, Y, sm + Mp, nsplit);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    stamps[2 * blockIdx.x] = t0;
    stamps[2 * blockIdx.x + 1] = t1;
  }
}
}  // namespace
}  // namespace gk

int main() {
  using namespace gk;
  const int M = 100, Mp = 104, P = 100, Q = 32;
  std::vector<double> th(M);
  for (int k = 0; k < M; ++k) th[k] = exp(-0.5 * (k * 0.02) * (k * 0.02) / 0.04);
  double *t, *X, *Y;
  cudaMalloc(&t, M * 8);
  cudaMemcpy(t, th.data(), M * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&X, size_t(P) * M * Q * 8);
  cudaMalloc(&Y, size_t(P) * M * Q * 8);
  cudaMemset(X, 0, size_t(P) * M * Q * 8);
  unsigned long long* st;
  cudaMalloc(&st, 4096 * 16);
  const size_t smem = (Mp + (Mp / 8 * 2 + Mp / 4) * 32 + 4 * Mp * 8) * 8 + 64;
  cudaFuncSetAttribute(k_tprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int split : {1, 2}) {
    for (int grid : {1, 8, 74, 148, 296, 400, 800}) {
      for (int rep = 0; rep < 3; ++rep) k_tprobe<<<grid, 256, smem>>>(t, M, Mp, P, Q, X, Y, split, st);
      cudaEventRecord(e0);
      k_tprobe<<<grid, 256, smem>>>(t, M, Mp, P, Q, X, Y, split, st);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> h(2 * grid);
      cudaMemcpy(h.data(), st, 16 * grid, cudaMemcpyDeviceToHost);
      unsigned long long mn = ~0ull, mx = 0, dmax = 0;
      double dsum = 0;
      for (int b = 0; b < grid; ++b) {
        mn = std::min(mn, h[2 * b]);
        mx = std::max(mx, h[2 * b + 1]);
        dmax = std::max(dmax, h[2 * b + 1] - h[2 * b]);
        dsum += h[2 * b + 1] - h[2 * b];
      }
      const int items = (P * Q / 8) * split;
      printf("split %d grid %4d items %4d: event %.2f us, span %.2f us, per-CTA avg %.2f max %.2f us, items/CTA %.1f\n",
             split, grid, items, ms * 1e3, (mx - mn) / 1e3, dsum / grid / 1e3, dmax / 1e3, double(items) / grid);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
