// fp64_peaks.cu — microbenchmark of the FP64 roofline denominators on this
// B200: DFMA (CUDA cores) and DMMA (mma.sync m8n8k4 f64 tensor cores)
// throughput, plus empty-kernel and small-kernel timing floors.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x % 7), b = 1e-3 * (threadIdx.x % 5);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(acc[k][0], acc[k][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_empty() {}

// dependent-chain latency of DMMA (one warp, accumulator carried)
__global__ void k_dmma_lat(double* out, long long* cycles, int iters) {
  double d0 = 0, d1 = 0;
  const double a = 1e-3 * (threadIdx.x % 7), b = 1e-3 * (threadIdx.x % 5);
  const long long c0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(d0, d1, a, b);
  const long long c1 = clock64();
  out[threadIdx.x] = d0 + d1;
  if (threadIdx.x == 0) *cycles = c1 - c0;
}

// small kernel: few CTAs, a fixed dependent FMA chain; records SM cycles
__global__ void k_small(double* out, long long* cycles, int iters) {
  const long long c0 = clock64();
  double a = threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) a = fma(a, 0.999999, 1e-7);
  const long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = c1 - c0;
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, p.multiProcessorCount);
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  // warm up clocks
  for (int r = 0; r < 20; ++r) k_dfma<<<blocks, threads>>>(out, 2000);
  cudaDeviceSynchronize();
  {
    const int iters = 4000;
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    printf(", \"dfma_tflops\": %.2f", flops / (ms * 1e-3) / 1e12);
  }
  {
    const int iters = 4000;
    for (int r = 0; r < 3; ++r) k_dmma<<<blocks, 128>>>(out, 200);
    cudaEventRecord(e0);
    k_dmma<<<blocks, 128>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // each mma.m8n8k4 = 8*8*4 FMA = 512 flops per warp instruction
    const double flops = 512.0 * 8 * double(iters) * blocks * (128 / 32);
    printf(", \"dmma_tflops\": %.2f", flops / (ms * 1e-3) / 1e12);
  }
  {
    for (int r = 0; r < 10; ++r) k_empty<<<1, 32>>>();
    cudaEventRecord(e0);
    for (int r = 0; r < 1000; ++r) k_empty<<<1, 32>>>();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"empty_kernel_back_to_back_us\": %.3f", ms * 1e3 / 1000);
    float single = 0;
    for (int r = 0; r < 50; ++r) {
      cudaEventRecord(e0);
      k_empty<<<1, 32>>>();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      single += t;
    }
    printf(", \"empty_kernel_events_us\": %.3f", single * 1e3 / 50);
  }
  {
    long long* cyc;
    cudaMalloc(&cyc, 8);
    k_dmma_lat<<<1, 32>>>(out, cyc, 100);
    k_dmma_lat<<<1, 32>>>(out, cyc, 1000);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_dependent_latency_cycles\": %.1f", c / 1000.0);
    k_small<<<1, 32>>>(out, cyc, 1000);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dfma_dependent_latency_cycles\": %.1f", c / 1000.0);
  }
  {
    long long* cyc;
    cudaMalloc(&cyc, 8);
    for (int iters : {100, 1000, 10000}) {
      for (int r = 0; r < 5; ++r) k_small<<<13, 128>>>(out, cyc, iters);
      cudaEventRecord(e0);
      for (int r = 0; r < 200; ++r) k_small<<<13, 128>>>(out, cyc, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf(", \"small_%d_b2b_us\": %.2f, \"small_%d_cycles\": %lld", iters, ms * 1e3 / 200, iters, c);
    }
  }
  {
    const long n = 4L * 1024 * 1024;  // 32 MB: L2-resident copy
    double *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    for (int r = 0; r < 5; ++r) k_copy<<<148 * 8, 256>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 100; ++r) k_copy<<<148 * 8, 256>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"l2_copy_32MB_us\": %.2f, \"l2_copy_gbs\": %.0f", ms * 1e3 / 100, 2.0 * n * 8 * 100 / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
