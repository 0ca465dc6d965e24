// dmma_probe.cu — DMMA (mma.sync m8n8k4 f64) issue behaviour on B200:
// cycles per DMMA for C independent accumulator chains per warp, W warps per
// CTA (one CTA per SM), operands from registers or loaded from shared memory
// every step (as in the fused MVM's Toeplitz phase).
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int C, bool LDS>
__global__ void k_probe(double* out, long long* cyc, int iters) {
  __shared__ double sa[2048], sb[2048];
  const int lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    sa[i] = 1.0 + 1e-9 * i;
    sb[i] = 1.0 - 1e-9 * i;
  }
  __syncthreads();
  double acc[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = sa[lane], b = sb[lane];
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if constexpr (LDS) {
        const int o = ((it * C + c) * 32 + lane) & 2047;
        dmma(acc[c][0], acc[c][1], sa[o], sb[o]);
      } else {
        dmma(acc[c][0], acc[c][1], a, b);
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C, bool LDS>
void run(double* out, long long* cyc, int warps) {
  const int iters = 2000;
  k_probe<C, LDS><<<148, 32 * warps>>>(out, cyc, 10);
  k_probe<C, LDS><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp = double(c) / (iters * C);
  printf("chains %d %s warps/SM %2d: %.1f cycles per DMMA per warp, %.2f cycles per DMMA per SM\n", C,
         LDS ? "LDS" : "reg", warps, per_warp, per_warp / warps);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) {
    run<1, false>(out, cyc, w);
    run<2, false>(out, cyc, w);
    run<4, false>(out, cyc, w);
    run<8, false>(out, cyc, w);
    run<2, true>(out, cyc, w);
    run<4, true>(out, cyc, w);
    run<8, true>(out, cyc, w);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
