// slab_probe.cu — phase timing (clock64/globaltimer) of a Toeplitz mode product
// with the same structure as kron.cu's slab kernel, to find where the time goes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_probe(const double* __restrict__ t, int M, long long P, long long Q, const double* __restrict__ X,
                        double* __restrict__ Y, unsigned long long* stamps) {
  constexpr int BN = 8, SB = 8;
  extern __shared__ double sm[];
  const int Mp = (M + 7) / 8 * 8;
  double* ts = sm;
  double* Bs = sm + Mp;
  const long long ncols = P * Q;
  const long long col0 = (long long)blockIdx.x * BN;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  uint64_t t0 = gtimer();
  for (int i = tid; i < Mp; i += 128) ts[i] = i < M ? __ldg(t + i) : 0.0;
  const int total = Mp * BN;
  for (int e = tid; e < total; e += 128) {
    const int cc = e / Mp, c = e % Mp;
    const long long col = col0 + cc;
    double v = 0.0;
    if (c < M && col < ncols) v = __ldg(X + ((col / Q) * M + c) * Q + (col % Q));
    Bs[c * SB + cc] = v;
  }
  __syncthreads();
  uint64_t t1 = gtimer();
  const int mtiles = Mp / 8;
  for (int mt0 = warp * 4; mt0 < mtiles; mt0 += 16) {
    double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    const int ntile = min(4, mtiles - mt0);
    for (int kk = 0; kk < Mp; kk += 4) {
      const int c = kk + t4;
      const double bf = Bs[c * SB + g];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i >= ntile) break;
        const int a = (mt0 + i) * 8 + g;
        const int dist = a > c ? a - c : c - a;
        const double af = (a < M && c < M) ? ts[dist] : 0.0;
        dmma(acc[i][0], acc[i][1], af, bf);
      }
    }
    for (int i = 0; i < ntile; ++i) {
      const int a = (mt0 + i) * 8 + g;
      if (a >= M) continue;
      for (int e = 0; e < 2; ++e) {
        const long long col = col0 + 2 * t4 + e;
        if (col < ncols) Y[((col / Q) * M + a) * Q + (col % Q)] = acc[i][e];
      }
    }
  }
  uint64_t t2 = gtimer();
  __syncthreads();
  if (tid == 0) {
    stamps[blockIdx.x * 3 + 0] = t0;
    stamps[blockIdx.x * 3 + 1] = t1;
    stamps[blockIdx.x * 3 + 2] = t2;
  }
}

__global__ void k_noop(unsigned long long* s) {
  if (threadIdx.x == 0) s[0] = gtimer();
}

int main() {
  const int M = 100;
  for (long long Q : {1LL, 32LL}) {
    const long long P = 100;
    std::vector<double> th(M);
    for (int k = 0; k < M; ++k) th[k] = exp(-0.5 * (k / 9.3) * (k / 9.3));
    double *t, *X, *Y;
    cudaMalloc(&t, M * 8);
    cudaMalloc(&X, P * M * Q * 8);
    cudaMalloc(&Y, P * M * Q * 8);
    cudaMemcpy(t, th.data(), M * 8, cudaMemcpyHostToDevice);
    cudaMemset(X, 0, P * M * Q * 8);
    const int blocks = int((P * Q + 7) / 8);
    unsigned long long* st;
    cudaMalloc(&st, blocks * 3 * 8 + 64);
    const int Mp = 104;
    const size_t shm = 8 * (Mp + Mp * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 10; ++r) k_probe<<<blocks, 128, shm>>>(t, M, P, Q, X, Y, st);
    cudaEventRecord(e0);
    for (int r = 0; r < 100; ++r) k_probe<<<blocks, 128, shm>>>(t, M, P, Q, X, Y, st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long* host_launch;
    cudaMallocHost(&host_launch, 8);
    k_noop<<<1, 32>>>(st + blocks * 3);
    // one more instrumented run
    k_probe<<<blocks, 128, shm>>>(t, M, P, Q, X, Y, st);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(blocks * 3 + 1);
    cudaMemcpy(h.data(), st, (blocks * 3 + 1) * 8, cudaMemcpyDeviceToHost);
    unsigned long long tmin = ~0ULL, tmax = 0;
    double stage = 0, comp = 0;
    for (int b = 0; b < blocks; ++b) {
      tmin = std::min(tmin, h[b * 3]);
      tmax = std::max(tmax, h[b * 3 + 2]);
      stage += h[b * 3 + 1] - h[b * 3];
      comp += h[b * 3 + 2] - h[b * 3 + 1];
    }
    printf("{\"Q\": %lld, \"blocks\": %d, \"b2b_us\": %.2f, \"span_first_start_to_last_end_us\": %.2f, "
           "\"avg_stage_us\": %.2f, \"avg_compute_us\": %.2f}\n",
           Q, blocks, ms * 1e3 / 100, (tmax - tmin) / 1e3, stage / blocks / 1e3, comp / blocks / 1e3);
    cudaFree(t);
    cudaFree(X);
    cudaFree(Y);
    cudaFree(st);
  }
  return 0;
}
