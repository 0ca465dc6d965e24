// lat_probe.cu — round-trip time of one global->shared staging step as used by
// the fused D-SKI MVM: per CTA, ITER dependent iterations of "copy B bytes to
// shared memory, wait, __syncthreads" with (0) 16-byte cp.async per thread,
// (1) one cp.async.bulk + mbarrier, (2) 16-byte ld.global + st.shared.
// Cold (HBM, 1 GB buffer) and hot (L2-resident 8 MB buffer) sources.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_lat(const char* __restrict__ src, size_t span, int bytes, int iters, int mode,
                      unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  double sink = 0.0;
  uint64_t t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
    const size_t off = ((size_t(blockIdx.x) * 7919 + size_t(it) * 104729) * 4096) % (span - bytes);
    const char* s = src + (off & ~size_t(127));
    if (mode == 0) {
      for (int e = tid * 16; e < bytes; e += blockDim.x * 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + e)), "l"(s + e) : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    } else if (mode == 1) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sm)),
                     "l"(s), "r"(bytes), "r"(su32(&mbar))
                     : "memory");
      }
      const unsigned parity = it & 1;
      asm volatile(
          "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&mbar)),
          "r"(parity)
          : "memory");
    } else {
      for (int e = tid * 16; e < bytes; e += blockDim.x * 16) {
        const double2 v = *reinterpret_cast<const double2*>(s + e);
        *reinterpret_cast<double2*>(sm + e) = v;
      }
    }
    __syncthreads();
    sink += reinterpret_cast<const double*>(sm)[tid];
    __syncthreads();
  }
  uint64_t t1 = gtimer();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (sink == 12345.678) out[0] = 0;
}

int main() {
  const size_t big = size_t(1) << 30, hot = size_t(8) << 20;
  char* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 8);
  const int iters = 20;
  cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int grid : {148, 296}) {
    for (size_t span : {big, hot}) {
      for (int bytes : {4096, 20480, 65536}) {
        for (int mode : {0, 1, 2}) {
          for (int rep = 0; rep < 2; ++rep) k_lat<<<grid, 256, bytes>>>(buf, span, bytes, iters, mode, out);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> h(grid);
          cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
          double s = 0, mx = 0;
          for (auto v : h) {
            s += v;
            mx = v > mx ? v : mx;
          }
          printf("grid %3d %s bytes %6d mode %d (%s): per-iteration avg %.3f us, max %.3f us\n", grid,
                 span == big ? "cold" : "hot ", bytes, mode, mode == 0 ? "cp.async16" : mode == 1 ? "bulk" : "ld/st",
                 s / grid / iters / 1e3, mx / iters / 1e3);
        }
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
