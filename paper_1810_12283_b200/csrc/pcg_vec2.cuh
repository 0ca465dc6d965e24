// pcg_vec2.cuh — the rows-resident fused PCG vector step (device code), shared
// by the standalone cooperative kernel (pcg_fused.cu) and the persistent
// MVM + vector-step kernel (fused2d.cu).
#pragma once

#include "gk_kernels.cuh"
#include "gk_sync.cuh"
#include "pcg_fused.hpp"

namespace gk {
namespace {

constexpr int PV_THREADS = 256;

// Shared-memory row strides ≡ 4 (mod 16) doubles: both DMMA fragment
// patterns (4 rows × 8 words and 8 rows × 4 words) then touch every bank
// exactly twice per warp load — the 2-wavefront minimum, no conflicts.
__host__ __device__ __forceinline__ int pv_pad(int x) { return x + ((4 - x % 16) + 16) % 16; }


// Fixed-order sum of nblocks partials (stride apart) by one warp: each lane
// first loads its ≤ 12 values (all in flight at once), then sums them, then a
// butterfly — deterministic, and one memory latency instead of twelve.
__device__ __forceinline__ double warp_sum_cols(const double* partial, int nblocks, int stride, int idx) {
  const int lane = threadIdx.x & 31;
  double v[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const int k = lane + 32 * q;
    v[q] = k < nblocks ? __ldcg(partial + (i64)k * stride + idx) : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 12; ++q) s += v[q];
  for (int k = lane + 384; k < nblocks; k += 32) s += __ldcg(partial + (i64)k * stride + idx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// per-thread values (slot, b) -> partial[blockIdx][b] (fixed order)
__device__ __forceinline__ void block_cols(double v, int nrhs, double* sm, double* partial) {
  __syncthreads();
  sm[threadIdx.x] = v;
  __syncthreads();
  const int slots = PV_THREADS / nrhs;
  if ((int)threadIdx.x < nrhs) {
    double s = 0.0;
    for (int k = 0; k < slots; ++k) s += sm[k * nrhs + threadIdx.x];
    partial[(i64)blockIdx.x * nrhs + threadIdx.x] = s;
  }
}

// Stage rows [rs, rs+nr) of Q1 (K per row), of r (nrhs per row) and of
// D^{-1/2} in shared memory with cp.async: every copy of the chunk is in
// flight at once (one memory latency per chunk).
__device__ __forceinline__ void pv_cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void pv_cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
// rows [0, nr) of width w (source row stride w) into shared rows of stride
// ws: 16-byte L2-only copies when w is even (16-byte aligned rows), else 8-byte
__device__ __forceinline__ void pv_copy_rows(double* dst, int ws, const double* src, int w, int nr) {
  // warp per row, lanes across the row: no integer division per copy
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if ((w & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    const int cpr = w / 2;
    for (int r = warp; r < nr; r += PV_THREADS / 32)
      for (int c = lane; c < cpr; c += 32) pv_cpa16(dst + r * ws + 2 * c, src + (i64)r * w + 2 * c);
  } else {
    for (int r = warp; r < nr; r += PV_THREADS / 32)
      for (int c = lane; c < w; c += 32) pv_cpa8(dst + r * ws + c, src + (i64)r * w + c);
  }
}
// Stage rows [rs, rs+nr) of Q1 (stride QS), r (stride RS) and D^{-1/2}.
__device__ __forceinline__ void stage_rows(const PcgVecArgs& a, i64 rs, int nr, double* Qs, double* Rs, double* Ds) {
  const int K = a.k, nrhs = a.nrhs, tid = threadIdx.x;
  pv_copy_rows(Qs, pv_pad(K), a.q1 + rs * K, K, nr);
  pv_copy_rows(Rs, pv_pad(nrhs), a.R + rs * nrhs, nrhs, nr);
  for (int e = tid; e < nr; e += PV_THREADS) pv_cpa8(Ds + e, a.dinv + rs + e);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
}

__device__ __forceinline__ void pv_stamp(const PcgVecArgs& a, int k, bool on) {
  if (on && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.prof[blockIdx.x * 16 + k] = t;
  }
}

constexpr int PV_RB = 4;  // rows per thread in flight in the vector passes
constexpr int PV_TT = 4;  // T-partial DMMA tiles per warp (ceil(K/8)·ceil(nrhs/8) ≤ 32)
constexpr int PV_ET = 8;  // E DMMA tiles per warp (ceil(RCH/8)·ceil(nrhs/8) ≤ 64)

__device__ __forceinline__ void pv_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- v2: rows resident
// When a CTA's whole row range fits in shared memory (C2: ~102 rows), the
// step keeps Q1 rows, c = D^{-1/2} r and D^{-1/2} resident for the launch:
//   prologue  cp.async Q1 rows + D^{-1/2} (lands while phase A runs)
//   A  pAp partials                                    | barrier
//   B  alpha / stall / max-iteration logic
//   C  x += a p, r -= a Ap (global), c = D^{-1/2} r into shared memory,
//      ||r||² and ||c||² partials; T partials = Q1ᵀ c (DMMA) | barrier
//   D  convergence; T reduced slice-wise                  | barrier
//   F  r·z = ||c||² − ||T||²  (= Preconditioner::quadratic, linalg.cpp:210-213:
//      rᵀ D^{-1/2}(c − Q1 Q1ᵀ c) = cᵀc − ‖Q1ᵀc‖²), beta = rz_new / rz
//   EG p = D^{-1/2}(c − Q1 T) + beta p straight from the DMMA accumulators
//      (z is never written).
// Three grid barriers instead of five, no z round trip through memory, and no
// re-staging of rows.
__device__ __forceinline__ void block_cols2(double v1, double v2, int nrhs, double* sm, double* partial) {
  __syncthreads();
  sm[threadIdx.x] = v1;
  __syncthreads();
  const int slots = PV_THREADS / nrhs;
  double s1 = 0.0;
  if ((int)threadIdx.x < nrhs)
    for (int k = 0; k < slots; ++k) s1 += sm[k * nrhs + threadIdx.x];
  __syncthreads();
  sm[threadIdx.x] = v2;
  __syncthreads();
  if ((int)threadIdx.x < nrhs) {
    double s2 = 0.0;
    for (int k = 0; k < slots; ++k) s2 += sm[k * nrhs + threadIdx.x];
    partial[(i64)blockIdx.x * 2 * nrhs + threadIdx.x] = s1;
    partial[(i64)blockIdx.x * 2 * nrhs + nrhs + threadIdx.x] = s2;
  }
}

// as block_cols2, stored transposed: tp[c·grid + cta] (v1), tp[(nrhs + c)·grid + cta] (v2)
__device__ __forceinline__ void block_cols2_t(double v1, double v2, int nrhs, double* sm, double* tp) {
  __syncthreads();
  sm[threadIdx.x] = v1;
  __syncthreads();
  const int slots = PV_THREADS / nrhs;
  double s1 = 0.0;
  if ((int)threadIdx.x < nrhs)
    for (int k = 0; k < slots; ++k) s1 += sm[k * nrhs + threadIdx.x];
  __syncthreads();
  sm[threadIdx.x] = v2;
  __syncthreads();
  if ((int)threadIdx.x < nrhs) {
    double s2 = 0.0;
    for (int k = 0; k < slots; ++k) s2 += sm[k * nrhs + threadIdx.x];
    tp[(i64)threadIdx.x * gridDim.x + blockIdx.x] = s1;
    tp[(i64)(nrhs + threadIdx.x) * gridDim.x + blockIdx.x] = s2;
  }
}

// Returns the number of active columns after the step (identical in every CTA).
__device__ __forceinline__ int pcg_vec2_body(const PcgVecArgs& a) {
  extern __shared__ __align__(16) double pv_sm[];
  const int nrhs = a.nrhs, K = a.q1 != nullptr ? a.k : 0, RMAX = a.rch;
  const int K4 = (K + 3) & ~3;
  double* red = pv_sm;                 // [256]
  double* colv = red + PV_THREADS;     // [2*nrhs]
  double* alpha = colv + 2 * nrhs;     // [nrhs]
  double* beta = alpha + nrhs;         // [nrhs]
  double* rz = beta + nrhs;            // [nrhs]
  double* bnorm = rz + nrhs;           // [nrhs]
  const int QS = pv_pad(K4 > 0 ? K4 : 1), RS = pv_pad(nrhs);
  auto al2 = [](double* p) {
    return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  };
  double* Ts = al2(bnorm + nrhs);            // [K4][RS]
  double* Qs = al2(Ts + (size_t)K4 * RS);    // [RMAX][QS] Q1 rows (resident)
  double* Cs = al2(Qs + (size_t)RMAX * QS);  // [RMAX][RS] c = D^{-1/2} r (resident)
  double* Ds = al2(Cs + (size_t)RMAX * RS);  // [RMAX] D^{-1/2}
  int* upd = reinterpret_cast<int*>(Ds + RMAX);
  int* act = upd + nrhs;
  int* its = act + nrhs;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g8 = lane / 4, t4 = lane % 4;
  const int b = tid % nrhs, slot = tid / nrhs, slots = PV_THREADS / nrhs;
  const int ntn = (nrhs + 7) / 8;
  const bool lane_ok = slot < slots;
  const i64 per = (a.N + gridDim.x - 1) / gridDim.x;
  const i64 r0 = min(a.N, (i64)blockIdx.x * per), r1 = min(a.N, r0 + per);
  const int nr = int(r1 - r0), nr8 = (nr + 7) & ~7;
  const PcgState& st = a.st;
  double* part0 = a.part;
  double* part1 = a.part + (size_t)gridDim.x * nrhs;  // [cta][2*nrhs]
  const bool prof_on = a.prof != nullptr && a.st.its[0] == 20;
  pv_stamp(a, 0, prof_on);

  // prologue: resident rows (in flight during phase A); pad rows/columns zeroed
  if (K > 0) {
    pv_copy_rows(Qs, QS, a.q1 + r0 * K, K, nr);
    for (int e = tid; e < nr; e += PV_THREADS) pv_cpa8(Ds + e, a.dinv + r0 + e);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    for (int e = tid; e < nr8 * (K4 - K); e += PV_THREADS) Qs[(e / (K4 - K)) * QS + K + e % (K4 - K)] = 0.0;
    for (int e = tid; e < (nr8 - nr) * K4; e += PV_THREADS) Qs[(nr + e / K4) * QS + e % K4] = 0.0;
    for (int e = tid; e < nr8 - nr; e += PV_THREADS) Ds[nr + e] = 0.0;
    for (int e = tid; e < (K4 - K) * RS; e += PV_THREADS) Ts[K * RS + e] = 0.0;
  }
  for (int e = tid; e < (nr8 - nr) * RS; e += PV_THREADS) Cs[nr * RS + e] = 0.0;
  __shared__ short tileM[8 * PV_ET], tileN[8 * PV_ET];
  for (int t = tid; t < 8 * PV_ET; t += PV_THREADS) {
    tileM[t] = short((t / ntn) * 8);
    tileN[t] = short((t % ntn) * 8);
  }
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    act[c] = st.active[c];
    its[c] = st.its[c];
    rz[c] = st.rz[c];
    bnorm[c] = st.bnorm[c];
  }
  // A: pAp partials
  double acc = 0.0;
  if (lane_ok)
    for (i64 rb = r0 + slot; rb < r1; rb += PV_RB * slots) {
      double pv[PV_RB], qv[PV_RB];
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        const i64 i = r * nrhs + b;
        pv[q] = r < r1 ? a.P[i] : 0.0;
        qv[q] = r < r1 ? a.AP[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) acc += pv[q] * qv[q];
    }
  block_cols(acc, nrhs, red, part0);
  pv_stamp(a, 1, prof_on);
  grid_allreduce_cols(part0, nrhs, colv, a.bar);
  pv_stamp(a, 7, prof_on);

  // B: alpha (linalg.cpp:110-118)
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    int u = 0;
    double al = 0.0;
    int ac = act[c], it = its[c];
    if (ac) {
      if (it >= st.maxit) {
        ac = 0;
      } else if (colv[c] <= 0.0) {
        ac = 0;
      } else {
        al = rz[c] / colv[c];
        u = 1;
        it += 1;
      }
    }
    act[c] = ac;
    its[c] = it;
    upd[c] = u;
    alpha[c] = al;
    if (blockIdx.x == 0) {
      st.active[c] = ac;
      st.its[c] = it;
      st.upd[c] = u;
      st.alpha[c] = al;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // C: x += a p, r -= a Ap; c = D^{-1/2} r resident; ||r||², ||c||² partials
  double arr = 0.0, acc_c = 0.0;
  if (lane_ok) {
    const bool u = upd[b] != 0;
    const double al = alpha[b];
    for (i64 rb = r0 + slot; rb < r1; rb += PV_RB * slots) {
      double xv[PV_RB], pv[PV_RB], rv[PV_RB], qv[PV_RB];
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        const i64 i = r * nrhs + b;
        const bool ok = r < r1;
        rv[q] = ok ? a.R[i] : 0.0;
        xv[q] = ok && u ? a.X[i] : 0.0;
        pv[q] = ok && u ? a.P[i] : 0.0;
        qv[q] = ok && u ? a.AP[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        if (r < r1) {
          const i64 i = r * nrhs + b;
          double rn = rv[q];
          if (u) {
            a.X[i] = xv[q] + al * pv[q];
            rn = rv[q] - al * qv[q];
            a.R[i] = rn;
            arr += rn * rn;
          }
          const int row = int(r - r0);
          const double c = K > 0 ? Ds[row] * rn : rn;
          Cs[row * RS + b] = c;
          acc_c += c * c;
        }
      }
    }
  }
  // ‖r‖², ‖c‖² partials go out transposed behind the T partials and are
  // reduced with them (no all-to-all read of partials by every CTA)
  block_cols2_t(arr, acc_c, nrhs, red, a.tpart + (i64)K * nrhs * gridDim.x);
  pv_stamp(a, 2, prof_on);
  if (K > 0) {  // T partial = Q1ᵀ c over the resident rows (M = j, N = b, K = rows)
    const int ntt = ((K + 7) / 8) * ntn;
    double tacc[PV_TT][2];
    int qa[PV_TT], qb[PV_TT];
#pragma unroll
    for (int q = 0; q < PV_TT; ++q) {
      tacc[q][0] = tacc[q][1] = 0.0;
      const int tile = warp + 8 * q;
      qa[q] = tile < ntt ? tileM[tile] + g8 : 0;
      qb[q] = tile < ntt ? tileN[tile] + g8 : 0;
    }
    for (int k0 = 0; k0 < nr8; k0 += 4) {
      const int r = k0 + t4;
#pragma unroll
      for (int q = 0; q < PV_TT; ++q)
        if (warp + 8 * q < ntt) pv_dmma(tacc[q][0], tacc[q][1], Qs[r * QS + qa[q]], Cs[r * RS + qb[q]]);
    }
#pragma unroll
    for (int q = 0; q < PV_TT; ++q) {
      const int tile = warp + 8 * q;
      if (tile < ntt) {
        const int j = tileM[tile] + g8;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = tileN[tile] + 2 * t4 + e;
          if (j < K && bb < nrhs) a.tpart[(i64)(j * nrhs + bb) * gridDim.x + blockIdx.x] = tacc[q][e];
        }
      }
    }
  }
  pv_stamp(a, 3, prof_on);
  grid_sync(a.bar);  // T, ‖r‖² and ‖c‖² partials visible
  pv_stamp(a, 10, prof_on);
  {  // distributed fixed-order reduction: T (K·nrhs), then ‖r‖² and ‖c‖² (2·nrhs)
    const int nout = (K + 2) * nrhs;
    for (int o = blockIdx.x * (PV_THREADS / 32) + tid / 32; o < nout; o += gridDim.x * (PV_THREADS / 32)) {
      const double v = warp_sum_cols(a.tpart + (i64)o * gridDim.x, gridDim.x, 1, 0);
      if ((tid & 31) == 0) a.T[o] = v;
    }
  }
  pv_stamp(a, 4, prof_on);
  grid_sync(a.bar);
  pv_stamp(a, 9, prof_on);
  for (int c = tid; c < 2 * nrhs; c += PV_THREADS) colv[c] = __ldcg(a.T + (i64)K * nrhs + c);
  for (int j = warp; j < K; j += PV_THREADS / 32)
    for (int cc = lane; cc < nrhs; cc += 32) Ts[j * RS + cc] = __ldcg(a.T + j * nrhs + cc);
  __syncthreads();

  // D: convergence (:119-125)
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    if (upd[c]) {
      const double relres = sqrt(colv[c]) / bnorm[c];
      const bool done = relres <= st.tol;
      if (done) act[c] = 0;
      if (blockIdx.x == 0) {
        st.hist[(i64)its[c] * nrhs + c] = relres;
        if (done) {
          st.conv[c] = 1;
          st.active[c] = 0;
        }
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    int nact = 0;
    for (int c = 0; c < nrhs; ++c) nact += act[c];
    *st.nactive = nact;
  }
  // F: rz_new = ||c||² − ||T||², beta (active columns)
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    if (act[c]) {
      double t2 = 0.0;
      for (int j = 0; j < K; ++j) t2 += Ts[j * RS + c] * Ts[j * RS + c];
      const double rzn = colv[nrhs + c] - t2;
      beta[c] = rzn / rz[c];
      if (blockIdx.x == 0) {
        st.beta[c] = beta[c];
        st.rz[c] = rzn;
      }
    }
  }
  __syncthreads();
  pv_stamp(a, 5, prof_on);

  // EG: p = D^{-1/2}(c − Q1 T) + beta p (active columns), from the DMMA tiles:
  // the warp's tiles in groups of EGQ (not unrolled: keeps the kernel's code
  // small — instruction-fetch stalls dominated with all tiles unrolled); per
  // group the P values are loaded first, the DMMA chains run interleaved,
  // then the epilogue writes.
  if (K > 0) {
    constexpr int EGQ = 4;
    const int nte = (nr8 / 8) * ntn;
    const int nq = nte > warp ? (nte - warp + 7) / 8 : 0;
#pragma unroll 1
    for (int q0 = 0; q0 < nq; q0 += EGQ) {
      double pv[EGQ][2], sacc[EGQ][2];
      const double* qp[EGQ];
      const double* tp[EGQ];
      int rows[EGQ], cols[EGQ];
#pragma unroll
      for (int u = 0; u < EGQ; ++u) {
        const int tile = warp + 8 * min(q0 + u, nq - 1);
        rows[u] = tileM[tile] + g8;
        cols[u] = tileN[tile] + 2 * t4;
        qp[u] = Qs + rows[u] * QS + t4;
        tp[u] = Ts + t4 * RS + tileN[tile] + g8;
        sacc[u][0] = sacc[u][1] = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e)
          pv[u][e] = (q0 + u < nq && rows[u] < nr && cols[u] + e < nrhs) ? a.P[(r0 + rows[u]) * nrhs + cols[u] + e]
                                                                          : 0.0;
      }
      for (int k0 = 0; k0 < K4; k0 += 4)
#pragma unroll
        for (int u = 0; u < EGQ; ++u) pv_dmma(sacc[u][0], sacc[u][1], qp[u][k0], tp[u][k0 * RS]);
#pragma unroll
      for (int u = 0; u < EGQ; ++u) {
        if (q0 + u >= nq || rows[u] >= nr) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = cols[u] + e;
          if (bb < nrhs && act[bb]) {
            const double z = Ds[rows[u]] * (Cs[rows[u] * RS + bb] - sacc[u][e]);
            a.P[(r0 + rows[u]) * nrhs + bb] = z + beta[bb] * pv[u][e];
          }
        }
      }
    }
  } else if (lane_ok && act[b]) {
    const double be = beta[b];
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const i64 i = r * nrhs + b;
      a.P[i] = Cs[int(r - r0) * RS + b] + be * a.P[i];
    }
  }
  pv_stamp(a, 6, prof_on);
  int nact = 0;
  for (int c = 0; c < nrhs; ++c) nact += act[c];
  __syncthreads();  // act[] read by every thread before the shared memory is reused
  return nact;
}


}  // namespace
}  // namespace gk
