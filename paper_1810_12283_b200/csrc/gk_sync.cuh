// gk_sync.cuh — grid-wide barrier for the persistent cooperative kernels
// (fused 2-D MVM, fused PCG vector step).
#pragma once

#include <cuda_runtime.h>

namespace gk {

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
#ifndef GK_BARRIER_SLEEP_NS
#define GK_BARRIER_SLEEP_NS 64
#endif
constexpr unsigned kBarrierSleepNs = GK_BARRIER_SLEEP_NS;
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier on a monotonic 64-bit arrival counter bar[0] (never
// reset: the k-th barrier of a launch completes when the counter reaches a
// multiple of gridDim.x). Arrival is a release atomic, waiting an acquire
// load, so the CTA's prior global writes (ordered by __syncthreads) are
// visible to every CTA after the barrier. Co-residency is guaranteed by the
// cooperative launch; a bounded spin turns a logic error into a trap instead
// of a hang. (A two-level variant — 8-CTA group counters feeding a top
// counter — measured slower on B200: 14.3 vs 11.3 µs for launch + three
// barriers of the 296-CTA one-launch MVM, tools/f2_skip_sweep.py.)
constexpr int kBarSlots = 64;  // counter slots allocated per plan
__device__ __forceinline__ void grid_sync(unsigned long long* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;\n" : "=l"(t) : "l"(bar) : "memory");
    const unsigned long long nb = gridDim.x;
    const unsigned long long target = (t / nb + 1) * nb;
    unsigned spins = 0;
    while (ld_relaxed(bar) < target) {
      if (++spins > (1u << 28)) __trap();
      if (kBarrierSleepNs) __nanosleep(kBarrierSleepNs);
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  __syncthreads();
}

// The same barrier split in two: grid_arrive (every thread calls it; thread
// 0 returns the generation target) and grid_wait(bar, target) (every thread
// calls it with thread 0's target). Work placed between the two overlaps the
// wait for the other CTAs — the one-launch MVM warms its next phase's
// instruction stream there.
__device__ __forceinline__ unsigned long long grid_arrive(unsigned long long* bar) {
  __syncthreads();
  unsigned long long target = 0;
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;\n" : "=l"(t) : "l"(bar) : "memory");
    const unsigned long long nb = gridDim.x;
    target = (t / nb + 1) * nb;
  }
  return target;
}
// grid_arrive that also returns (to every thread) how many CTAs arrived
// before this one in the current generation.
__device__ __forceinline__ unsigned long long grid_arrive_rank(unsigned long long* bar, int& rank) {
  __shared__ int s_rank;
  __syncthreads();
  unsigned long long target = 0;
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;\n" : "=l"(t) : "l"(bar) : "memory");
    const unsigned long long nb = gridDim.x;
    target = (t / nb + 1) * nb;
    s_rank = int(t % nb);
  }
  __syncthreads();
  rank = s_rank;
  return target;
}
__device__ __forceinline__ void grid_wait(unsigned long long* bar, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned spins = 0;
    while (ld_relaxed(bar) < target) {
      if (++spins > (1u << 28)) __trap();
      if (kBarrierSleepNs) __nanosleep(kBarrierSleepNs);
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  __syncthreads();
}

}  // namespace gk

namespace gk {

// Barrier fused with a column reduction: every CTA has written
// partial[cta][0..ncols); the LAST CTA to arrive sums them in fixed CTA order
// (deterministic), publishes out[0..ncols) and releases the others, which then
// read the ncols results. Replaces "barrier + every CTA re-reducing all
// partials". ctr[0] counts arrivals, ctr[1] counts releases; both only grow,
// so one pair serves every launch with the same grid size.
__device__ __forceinline__ void grid_reduce_cols(const double* partial, int ncols, double* out, double* out_sm,
                                                 unsigned long long* ctr) {
  __shared__ int s_last;
  __shared__ unsigned long long s_gen;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;\n" : "=l"(t) : "l"(ctr) : "memory");
    const unsigned long long nb = gridDim.x;
    s_gen = t / nb + 1;
    s_last = (t % nb) == nb - 1;
  }
  __syncthreads();
  if (s_last) {
    // every thread: column c = tid % ncols, CTA group g = tid / ncols sums the
    // CTAs k ≡ g (mod groups), loads in flight 8 at a time; then the group
    // sums are added in group order (fixed order: deterministic)
    __shared__ double gsum[256];
    const int groups = ncols <= (int)blockDim.x ? (int)blockDim.x / ncols : 1;
    for (int c0 = 0; c0 < ncols; c0 += (int)blockDim.x / groups) {
      const int c = c0 + (int)threadIdx.x % ((int)blockDim.x / groups);
      const int g = (int)threadIdx.x / ((int)blockDim.x / groups);
      double s = 0.0;
      if (c < ncols && g < groups) {
        // all of this thread's loads in flight at once, then summed in order
        constexpr int NL = 40;
        double v[NL];
#pragma unroll
        for (int q = 0; q < NL; ++q) {
          const int k = g + q * groups;
          v[q] = k < (int)gridDim.x ? __ldcg(partial + (long long)k * ncols + c) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NL; ++q) s += v[q];
        for (int k = g + NL * groups; k < (int)gridDim.x; k += groups) s += __ldcg(partial + (long long)k * ncols + c);
      }
      gsum[threadIdx.x] = s;
      __syncthreads();
      const int cw = (int)blockDim.x / groups;
      if ((int)threadIdx.x < cw && c0 + (int)threadIdx.x < ncols) {
        double t = 0.0;
        for (int q = 0; q < groups; ++q) t += gsum[q * cw + threadIdx.x];
        out[c0 + threadIdx.x] = t;
        out_sm[c0 + threadIdx.x] = t;
      }
      __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;\n" ::"l"(ctr + 1) : "memory");
    }
  } else {
    if (threadIdx.x == 0) {
      unsigned spins = 0;
      while (ld_relaxed(ctr + 1) < s_gen) {
        if (++spins > (1u << 24)) __trap();
        __nanosleep(kBarrierSleepNs);
      }
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    }
    __syncthreads();
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) out_sm[c] = __ldcg(out + c);
  }
  __syncthreads();
}

}  // namespace gk

namespace gk {

// Barrier, then EVERY CTA sums the CTA partials partial[cta][0..ncols) in
// fixed CTA order into out_sm (all of a thread's loads in flight at once):
// one barrier latency plus one memory latency, no serial hand-off.
__device__ __forceinline__ void grid_allreduce_cols(const double* partial, int ncols, double* out_sm,
                                                    unsigned long long* bar) {
  grid_sync(bar);
  __shared__ double gsum2[256];
  const int groups = ncols <= (int)blockDim.x ? (int)blockDim.x / ncols : 1;
  const int cw = (int)blockDim.x / groups;
  for (int c0 = 0; c0 < ncols; c0 += cw) {
    const int c = c0 + (int)threadIdx.x % cw;
    const int g = (int)threadIdx.x / cw;
    double s = 0.0;
    if (c < ncols && g < groups) {
      constexpr int NL = 40;
      double v[NL];
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int k = g + q * groups;
        v[q] = k < (int)gridDim.x ? __ldcg(partial + (long long)k * ncols + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NL; ++q) s += v[q];
      for (int k = g + NL * groups; k < (int)gridDim.x; k += groups) s += __ldcg(partial + (long long)k * ncols + c);
    }
    gsum2[threadIdx.x] = s;
    __syncthreads();
    if ((int)threadIdx.x < cw && c0 + (int)threadIdx.x < ncols) {
      double t = 0.0;
      for (int q = 0; q < groups; ++q) t += gsum2[q * cw + threadIdx.x];
      out_sm[c0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

}  // namespace gk
