#include <chrono>
#include <cstdio>
#include <cstdlib>
// dskip.cu — the D-SKIP operator on B200 (reference dskip.cpp).
//
//   K∇_DSKIP v = (Q_A T_A Q_Aᵀ) ⊙ (Q_B T_B Q_Bᵀ) v + noise
//
// Build (dskip.cpp:162-234): per dimension j a 1-D leaf (OneDimFactor, a 1-D
// D-SKI operator whose group j+1 uses ∂W and every other group W) is
// compressed by Lanczos to rank r; factors are merged pairwise in a balanced
// tree and re-compressed by Lanczos of the Hadamard pair operator until at
// most two remain. All of it runs on the device: leaves reuse the 1-D D-SKI
// kernels, Lanczos is the batched full-reorthogonalisation kernel set of
// solvers.cu, and the Hadamard MVM is the Khatri–Rao contraction below.
//
// Hadamard MVM (dskip.cpp:24-36) for factors A (rank ra), B (rank rb):
//   C[k,l,:] = Σ_i Q_A[i,k] Q_B[i,l] v[i,:]        (rows × (ra·rb) GEMM, split over rows)
//   C'[k,:,:] = T_B C[k,:,:]                       (tridiagonal along l)
//   out[i,:] = Σ_{k,l} (Q_A T_A)[i,k] Q_B[i,l] C'[k,l,:]
// Both contractions run on the fp64 tensor cores (mma.sync m8n8k4 DMMA) with
// the Khatri–Rao operand generated in shared memory.
// Layout: external row order, right-hand sides innermost ([N][nrhs]).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "gk_kernels.cuh"
#include "solvers.hpp"

namespace gk {

std::unique_ptr<Op> make_dski_profile(const gk_kernel& k, const gk_grid& g, const double* X, i64 n, double nv,
                                      double ng, int order, int with_grad, int device, int profile);
void dski_mvm_nonoise(Op& o, const double* in, double* out, int nrhs, cudaStream_t s);

namespace {

// ---------------------------------------------------------------- leaves
// bi[0][s][b] = Σ_{g != dir+1} in[g*n + perm[s]][b]; bi[1][s][b] = in[(dir+1)*n + perm[s]][b]
__global__ void k_leaf_combine(const double* __restrict__ in, const i64* __restrict__ ext, i64 n, int groups,
                               int dir, int nrhs, double* __restrict__ bi) {
  const i64 items = n * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it) % nrhs;
    const i64 s = int(it) / nrhs;
    const i64 i = ext[s];  // group-0 block of the 1-D operator: ext[s] = perm[s]
    double a = 0.0, da = 0.0;
    for (int g = 0; g <= groups; ++g) {
      const double v = in[((i64)g * n + i) * nrhs + b];
      if (g == dir + 1) da = v;
      else a += v;
    }
    bi[s * nrhs + b] = a;
    if (dir >= 0) bi[(n + s) * nrhs + b] = da;
  }
}

// out[g*n + perm[s]][b] = bo[(g == dir+1 ? 1 : 0)*n + s][b]
__global__ void k_leaf_expand(const double* __restrict__ bo, const i64* __restrict__ ext, i64 n, int groups,
                              int dir, int nrhs, double* __restrict__ out) {
  const i64 items = n * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it) % nrhs;
    const i64 s = int(it) / nrhs;
    const i64 i = ext[s];
    const double a = bo[s * nrhs + b];
    const double da = dir >= 0 ? bo[(n + s) * nrhs + b] : 0.0;
    for (int g = 0; g <= groups; ++g) out[((i64)g * n + i) * nrhs + b] = (g == dir + 1) ? da : a;
  }
}

// ---------------------------------------------------------------- factors
// Q (Lanczos output, [r][N] column blocks) -> row-major [N][r]; QT = Q T.
__global__ void k_factor_pack(const double* __restrict__ Qc, i64 N, int r, const double* __restrict__ alpha,
                              const double* __restrict__ beta, double* __restrict__ Q, double* __restrict__ QT) {
  const i64 items = N * r;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int k = int(it) % r;
    const i64 i = it / r;
    const double q = Qc[(i64)k * N + i];
    Q[it] = q;
    double t = alpha[k] * q;  // times_tridiagonal (dskip.cpp:13-22)
    if (k > 0) t += beta[k - 1] * Qc[(i64)(k - 1) * N + i];
    if (k + 1 < r) t += beta[k] * Qc[(i64)(k + 1) * N + i];
    QT[it] = t;
  }
}

// ---------------------------------------------------------------- DMMA helpers
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Stage 1: partial C[m][b] over a chunk of rows, m = k*rb + l.
// CTA tile: 64 m × 32 b, 4 warps (2×2, each 32 m × 16 b = 4×2 DMMA tiles).
// K loop over rows in steps of 16: Zs[row][m] = QA[row][k]·QB[row][l], Vs[row][b].
constexpr int H_BM = 64, H_BN = 32, H_BK = 16;
__global__ void __launch_bounds__(128) k_had_contract(const double* __restrict__ QA, int ra,
                                                      const double* __restrict__ QB, int rb,
                                                      const double* __restrict__ V, i64 N, int nrhs,
                                                      i64 rows_per_chunk, double* __restrict__ partial) {
  __shared__ double Zs[H_BK][H_BM + 1];
  __shared__ double Vs[H_BK][H_BN + 1];
  const int M = ra * rb;
  const int m0 = blockIdx.x * H_BM, b0 = blockIdx.y * H_BN;
  const i64 r_begin = (i64)blockIdx.z * rows_per_chunk;
  const i64 r_end = min(N, r_begin + rows_per_chunk);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = (warp / 2) * 32, wn = (warp % 2) * 16;
  const int g = lane / 4, t4 = lane % 4;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (i64 r0 = r_begin; r0 < r_end; r0 += H_BK) {
    __syncthreads();
    for (int e = tid; e < H_BK * H_BM; e += 128) {
      const int rr = e / H_BM, mm = e % H_BM;
      const i64 r = r0 + rr;
      const int m = m0 + mm;
      double z = 0.0;
      if (r < r_end && m < M) z = QA[r * ra + m / rb] * QB[r * rb + m % rb];
      Zs[rr][mm] = z;
    }
    for (int e = tid; e < H_BK * H_BN; e += 128) {
      const int rr = e / H_BN, bb = e % H_BN;
      const i64 r = r0 + rr;
      const int b = b0 + bb;
      Vs[rr][bb] = (r < r_end && b < nrhs) ? V[r * nrhs + b] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < H_BK; kk += 4) {
      double af[4], bf[2];
      // A = Zᵀ (m × rows): element (row m, col k) = Zs[k][m]
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Zs[kk + t4][wm + i * 8 + g];
      // B = V (rows × b): element (k, n) = Vs[k][n]
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Vs[kk + t4][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  // D fragment: row = g, cols = t4*2 + {0,1}
  double* out = partial + (i64)blockIdx.z * M * nrhs;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + i * 8 + g;
        const int b = b0 + wn + j * 8 + t4 * 2 + e;
        if (m < M && b < nrhs) out[(i64)m * nrhs + b] = acc[i][j][e];
      }
}

// C = Σ_chunks partial; then C'[k][l] = α_l C[k][l] + β_{l-1} C[k][l-1] + β_l C[k][l+1]
__global__ void k_had_reduce(const double* __restrict__ partial, int chunks, int M, int nrhs,
                             double* __restrict__ C) {
  const i64 items = (i64)M * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < chunks; ++c) s += __ldcs(partial + (i64)c * items + it);  // read once: evict-first
    C[it] = s;
  }
}
__global__ void k_had_tridiag(const double* __restrict__ C, int ra, int rb, int nrhs, const double* __restrict__ a,
                              const double* __restrict__ bta, double* __restrict__ Cp) {
  const i64 items = (i64)ra * rb * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it) % nrhs;
    const int m = int(it) / nrhs;
    const int k = m / rb, l = m % rb;
    double v = a[l] * C[it];
    if (l > 0) v += bta[l - 1] * C[((i64)k * rb + l - 1) * nrhs + b];
    if (l + 1 < rb) v += bta[l] * C[((i64)k * rb + l + 1) * nrhs + b];
    Cp[it] = v;
  }
}

// Stage 3: out[i][b] (+)= Σ_m QTA[i][k] QB[i][l] C'[m][b] (+ noise·v).
// CTA tile: 64 rows × 32 b, 4 warps (2×2 of 32×16); K loop over m in steps of 16.
__global__ void __launch_bounds__(128) k_had_expand(const double* __restrict__ QTA, int ra,
                                                    const double* __restrict__ QB, int rb,
                                                    const double* __restrict__ Cp, i64 N, int nrhs,
                                                    const double* __restrict__ v, i64 n_value, double nv2,
                                                    double ng2, int accumulate, double* __restrict__ out) {
  __shared__ double Zs[H_BM][H_BK + 1];  // Z'[row][m]
  __shared__ double Cs[H_BK][H_BN + 1];
  const int M = ra * rb;
  const i64 i0 = (i64)blockIdx.x * H_BM;
  const int b0 = blockIdx.y * H_BN;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = (warp / 2) * 32, wn = (warp % 2) * 16;
  const int g = lane / 4, t4 = lane % 4;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int mb = 0; mb < M; mb += H_BK) {
    __syncthreads();
    for (int e = tid; e < H_BM * H_BK; e += 128) {
      const int rr = e / H_BK, mm = e % H_BK;
      const i64 i = i0 + rr;
      const int m = mb + mm;
      double z = 0.0;
      if (i < N && m < M) z = QTA[i * ra + m / rb] * QB[i * rb + m % rb];
      Zs[rr][mm] = z;
    }
    for (int e = tid; e < H_BK * H_BN; e += 128) {
      const int mm = e / H_BN, bb = e % H_BN;
      const int m = mb + mm, b = b0 + bb;
      Cs[mm][bb] = (m < M && b < nrhs) ? Cp[(i64)m * nrhs + b] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < H_BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Zs[wm + i * 8 + g][kk + t4];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Cs[kk + t4][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const i64 row = i0 + wm + i * 8 + g;
        const int b = b0 + wn + j * 8 + t4 * 2 + e;
        if (row < N && b < nrhs) {
          const i64 idx = row * nrhs + b;
          double val = acc[i][j][e];
          if (v) val += (row < n_value ? nv2 : ng2) * v[idx];
          out[idx] = accumulate ? out[idx] + val : val;
        }
      }
}

// ---------------------------------------------------------------- Khatri–Rao GEMMs v2
// The two Hadamard contractions as fp64 tensor-core GEMMs whose A operand
// Z[row][m] = QA[row][k]·QB[row][l] (m = k·rb + l) is formed in registers at
// fragment load from staged Q rows — never written out. Q rows and the RHS
// block are staged with 16-byte cp.async, double-buffered; shared strides are
// ≡ 4 (mod 16) doubles (conflict-free DMMA fragment loads); (k, l) per m come
// from a per-CTA table (no divisions in the loops). Each warp owns a 32×32
// output tile: 16 independent DMMA accumulator chains.
__host__ __device__ __forceinline__ int hk_pad(int x) { return x + ((4 - x % 16) + 16) % 16; }
__device__ __forceinline__ void hk_cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void hk_cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
// rows [r0, r0+nr), columns [c0, c0+wc) of a [*][ld] row-major matrix into
// smem rows of stride ws; rows [nr, nz) of the tile are zeroed
__device__ __forceinline__ void hk_stage(double* dst, int ws, const double* src, int ld, int c0, int wc, i64 r0,
                                         int nr, int nz) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const double* base = src + r0 * ld + c0;
  if ((wc & 1) == 0 && (ld & 1) == 0 && (((uintptr_t)base) & 15) == 0) {
    const int cpr = wc / 2;
    for (int r = warp; r < nr; r += nw)
      for (int c = lane; c < cpr; c += 32) hk_cpa16(dst + r * ws + 2 * c, base + (i64)r * ld + 2 * c);
  } else {
    for (int r = warp; r < nr; r += nw)
      for (int c = lane; c < wc; c += 32) hk_cpa8(dst + r * ws + c, base + (i64)r * ld + c);
  }
  for (int e = threadIdx.x; e < (nz - nr) * ws; e += blockDim.x) dst[nr * ws + e] = 0.0;
}

constexpr int HK_BK = 32;  // rows per stage (contract)
constexpr int HK_MC = 32;  // m per stage (expand)

// partial[chunk][m][b] = Σ_{rows in chunk} Z[row][m] V[row][b]
// CTA: 64 m × 64 b (4 warps, 2×2 of 32×32); K = rows in stages of HK_BK.
__global__ void __launch_bounds__(128) k_had_contract2(const double* __restrict__ QA, int ra,
                                                       const double* __restrict__ QB, int rb,
                                                       const double* __restrict__ V, i64 N, int nrhs,
                                                       i64 rows_per_chunk, double* __restrict__ partial) {
  extern __shared__ __align__(16) double hk_sm[];
  const int bw = min(64, nrhs - (int)blockIdx.y * 64);
  const int SA = hk_pad(ra), SBq = hk_pad(rb), SV = hk_pad(min(64, nrhs));
  double* QAs = hk_sm;                           // [2][HK_BK][SA]
  double* QBs = QAs + 2 * HK_BK * SA;            // [2][HK_BK][SBq]
  double* Vs = QBs + 2 * HK_BK * SBq;            // [2][HK_BK][SV]
  const int M = ra * rb;
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  const i64 r_begin = (i64)blockIdx.z * rows_per_chunk;
  const i64 r_end = min(N, r_begin + rows_per_chunk);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  const int wm = (warp & 1) * 32, wb = (warp >> 1) * 32;
  int ka[4], la[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + wm + 8 * i + g;
    ka[i] = m < M ? m / rb : -1;
    la[i] = m < M ? m % rb : 0;
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto issue = [&](i64 rs, int buf) {
    const int nr = int(min((i64)HK_BK, r_end - rs));
    hk_stage(QAs + buf * HK_BK * SA, SA, QA, ra, 0, ra, rs, nr, HK_BK);
    hk_stage(QBs + buf * HK_BK * SBq, SBq, QB, rb, 0, rb, rs, nr, HK_BK);
    hk_stage(Vs + buf * HK_BK * SV, SV, V, nrhs, b0, bw, rs, nr, HK_BK);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int buf = 0;
  if (r_begin < r_end) issue(r_begin, 0);
  for (i64 rs = r_begin; rs < r_end; rs += HK_BK) {
    const i64 nx = rs + HK_BK;
    if (nx < r_end) {
      issue(nx, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* A1 = QAs + buf * HK_BK * SA;
    const double* B1 = QBs + buf * HK_BK * SBq;
    const double* V1 = Vs + buf * HK_BK * SV;
    const int nr = int(min((i64)HK_BK, r_end - rs));
    for (int kk = 0; kk < nr; kk += 4) {
      const int row = kk + t4;
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ka[i] >= 0 ? A1[row * SA + ka[i]] * B1[row * SBq + la[i]] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int bl = wb + 8 * j + g;
        bf[j] = bl < bw ? V1[row * SV + bl] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  double* out = partial + (i64)blockIdx.z * M * nrhs;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + g;
        const int b = b0 + wb + 8 * j + 2 * t4 + e;
        if (m < M && b < nrhs) out[(i64)m * nrhs + b] = acc[i][j][e];
      }
}

// out[i][b] (+)= Σ_m QTA[i][k] QB[i][l] C'[m][b] (+ noise·v)
// CTA: 64 rows × 64 b (4 warps, 2×2 of 32×32); the CTA's Q rows staged once,
// C' in double-buffered chunks of HK_MC m.
__global__ void __launch_bounds__(128) k_had_expand2(const double* __restrict__ QTA, int ra,
                                                     const double* __restrict__ QB, int rb,
                                                     const double* __restrict__ Cp, i64 N, int nrhs,
                                                     const double* __restrict__ v, i64 n_value, double nv2,
                                                     double ng2, int accumulate, double* __restrict__ out) {
  extern __shared__ __align__(16) double hk_sm[];
  const int bw = min(64, nrhs - (int)blockIdx.y * 64);
  const int SA = hk_pad(ra), SBq = hk_pad(rb), SV = hk_pad(min(64, nrhs));
  const int M = ra * rb;
  double* QAs = hk_sm;                  // [64][SA]
  double* QBs = QAs + 64 * SA;          // [64][SBq]
  double* Cs = QBs + 64 * SBq;          // [2][HK_MC][SV]
  int2* kl = reinterpret_cast<int2*>(Cs + 2 * HK_MC * SV);  // [M] (k, l)
  const i64 i0 = (i64)blockIdx.x * 64;
  const int b0 = blockIdx.y * 64;
  const int nr = int(min((i64)64, N - i0));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  const int wi = (warp & 1) * 32, wb = (warp >> 1) * 32;
  for (int m = tid; m < M; m += 128) kl[m] = make_int2(m / rb, m % rb);
  hk_stage(QAs, SA, QTA, ra, 0, ra, i0, nr, 64);
  hk_stage(QBs, SBq, QB, rb, 0, rb, i0, nr, 64);
  auto issue = [&](int mc, int buf) {
    const int nm = min(HK_MC, M - mc);
    hk_stage(Cs + buf * HK_MC * SV, SV, Cp, nrhs, b0, bw, mc, nm, HK_MC);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  issue(0, 0);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int buf = 0;
  for (int mc = 0; mc < M; mc += HK_MC) {
    if (mc + HK_MC < M) {
      issue(mc + HK_MC, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* C1 = Cs + buf * HK_MC * SV;
    const int nm = min(HK_MC, M - mc);
    for (int kk = 0; kk < nm; kk += 4) {
      const int m = mc + kk + t4;
      const int2 q = m < M ? kl[m] : make_int2(0, 0);
      const bool mok = m < M;
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = wi + 8 * i + g;
        af[i] = mok ? QAs[row * SA + q.x] * QBs[row * SBq + q.y] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = wb + 8 * j + g < bw ? C1[(kk + t4) * SV + wb + 8 * j + g] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const i64 row = i0 + wi + 8 * i + g;
        const int b = b0 + wb + 8 * j + 2 * t4 + e;
        if (row < N && b < nrhs) {
          const i64 idx = row * nrhs + b;
          double val = acc[i][j][e];
          if (v) val += (row < n_value ? nv2 : ng2) * v[idx];
          out[idx] = accumulate ? out[idx] + val : val;
        }
      }
}

static int device_sm_count() {
  int dev = 0, sms = 0;
  GK_CUDA(cudaGetDevice(&dev));
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}


// ---------------------------------------------------------------- Khatri–Rao GEMMs v3
// Same GEMMs as v2, with the operand rows moved by per-row TMA bulk copies
// (cp.async.bulk, one issuing thread per row, completion on an mbarrier ring)
// instead of per-16-byte cp.async loops, constant-trip fully unrolled stages
// (tails are zero rows, never predicated), and CTA shapes sized for 3-4
// resident CTAs per SM. Needs even ranks and an even RHS count (16-byte rows).
// The B factor's tridiagonal is folded into the expansion through its stored
// QT = Q T (no separate T_B pass over C).
// NJ = 8-column tiles per warp: the CTA covers 16·NJ right-hand sides.
__device__ __forceinline__ unsigned hk_su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void hk_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(hk_su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void hk_mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(hk_su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void hk_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(hk_su32(b)) : "memory");
}
__device__ __forceinline__ void hk_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nHKW_%=:\nmbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n@!P1 bra HKW_%=;\n}\n" ::"r"(
          hk_su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void hk_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   hk_su32(dst)),
               "l"(src), "r"(bytes), "r"(hk_su32(b))
               : "memory");
}
__device__ __forceinline__ void hk_zero_row(double* dst, int w) {
  for (int c = 0; c < w; ++c) dst[c] = 0.0;
}

constexpr int H3_BK = 16, H3_NS = 3;   // contract: rows per stage, ring depth
constexpr int H3_MC = 16, H3_NSE = 4;  // expand: m per stage, ring depth

template <int NJ>
__global__ void __launch_bounds__(128, 4) k_had_contract3(const double* __restrict__ QA, int ra,
                                                          const double* __restrict__ QB, int rb,
                                                          const double* __restrict__ V, i64 N, int nrhs,
                                                          i64 rows_per_chunk, double* __restrict__ partial) {
  extern __shared__ __align__(16) double hk_sm[];
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
  const int SA = hk_pad(ra), SBq = hk_pad(rb);
  const int stage_d = H3_BK * (SA + SBq + SV);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(hk_sm + H3_NS * stage_d);
  unsigned long long* empty = full + H3_NS;
  const int M = ra * rb;
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * BWC;
  const int bw = min(BWC, nrhs - b0);
  const i64 r_begin = (i64)blockIdx.z * rows_per_chunk;
  const i64 r_end = min(N, r_begin + rows_per_chunk);
  const int nst = r_end > r_begin ? int((r_end - r_begin + H3_BK - 1) / H3_BK) : 0;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  // warp w: m rows [16w, 16w+16) × all 16·NJ columns (2 m-tiles × 2·NJ b-tiles)
  constexpr int JT = 2 * NJ;
  const int wm = warp * 16;
  if (tid == 0) {
    for (int s = 0; s < H3_NS; ++s) hk_mbar_init(full + s, 32), hk_mbar_init(empty + s, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // warp 0 fills a stage: lane L moves QA row L (L < 16) or QB row L-16, and
  // lanes 0..15 also V row L; each lane arrives once with the bytes it issued
  const bool lo = lane < H3_BK;
  const int qrow = lo ? lane : lane - H3_BK;
  const int q_soff = lo ? qrow * SA : H3_BK * SA + qrow * SBq;
  const unsigned q_bytes = (lo ? ra : rb) * 8u;
  const double* q_src = lo ? QA + (r_begin + qrow) * ra : QB + (r_begin + qrow) * rb;
  const i64 q_step = (i64)H3_BK * (lo ? ra : rb);
  const int v_soff = H3_BK * (SA + SBq) + qrow * SV;
  const double* v_src = V + (r_begin + qrow) * nrhs + b0;
  auto issue = [&](int st) {
    const i64 rs = r_begin + (i64)st * H3_BK;
    const int nr = int(min((i64)H3_BK, r_end - rs));
    double* base = hk_sm + (st % H3_NS) * stage_d;
    unsigned long long* b = full + st % H3_NS;
    if (nr == H3_BK) {
      hk_mbar_arrive_tx(b, q_bytes + (lo ? bw * 8u : 0u));
      hk_bulk(base + q_soff, q_src + st * q_step, q_bytes, b);
      if (lo) hk_bulk(base + v_soff, v_src + (i64)st * H3_BK * nrhs, bw * 8u, b);
    } else {  // tail stage: rows past the chunk are zero rows
      const bool live = qrow < nr;
      if (live) {
        hk_mbar_arrive_tx(b, q_bytes + (lo ? bw * 8u : 0u));
        hk_bulk(base + q_soff, q_src + st * q_step, q_bytes, b);
        if (lo) hk_bulk(base + v_soff, v_src + (i64)st * H3_BK * nrhs, bw * 8u, b);
      } else {
        hk_zero_row(base + q_soff, lo ? SA : SBq);
        if (lo) hk_zero_row(base + v_soff, SV);
        hk_mbar_arrive(b);
      }
    }
  };
  int ka[2], la[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = min(m0 + wm + 8 * i + g, M - 1);  // rows past M: finite, discarded
    ka[i] = m / rb;
    la[i] = m - ka[i] * rb;
  }
  double acc[2][JT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (warp == 0)
    for (int s = 0; s < min(H3_NS, nst); ++s) issue(s);
  for (int it = 0; it < nst; ++it) {
    const int sb = it % H3_NS;
    const unsigned ph = (it / H3_NS) & 1;
    hk_mbar_wait(full + sb, ph);
    const double* A1 = hk_sm + sb * stage_d;
    const double* B1 = A1 + H3_BK * SA;
    const double* V1 = B1 + H3_BK * SBq;
#pragma unroll
    for (int kk = 0; kk < H3_BK; kk += 4) {
      const int row = kk + t4;
      double af[2], bf[JT];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = A1[row * SA + ka[i]] * B1[row * SBq + la[i]];
#pragma unroll
      for (int j = 0; j < JT; ++j) bf[j] = V1[row * SV + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < JT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) hk_mbar_arrive(empty + sb);  // this warp is done with the stage
    if (warp == 0 && it + H3_NS < nst) {
      hk_mbar_wait(empty + sb, ph);  // all four warps done: refill
      issue(it + H3_NS);
    }
  }
  double* out = partial + (i64)blockIdx.z * M * nrhs;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) {
      const int m = m0 + wm + 8 * i + g;
      const int bl = 8 * j + 2 * t4;
      if (m < M && bl < bw)
        *reinterpret_cast<double2*>(out + (i64)m * nrhs + b0 + bl) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

template <int NJ, int MC, int NSE>
__global__ void __launch_bounds__(128, 3) k_had_expand3(const double* __restrict__ QTA, int ra,
                                                        const double* __restrict__ QB, int rb,
                                                        const double* __restrict__ Cp, i64 N, int nrhs,
                                                        const double* __restrict__ v, i64 n_value, double nv2,
                                                        double ng2, int accumulate, double* __restrict__ out) {
  static_assert(MC <= 32 && MC % 4 == 0, "one warp-0 lane per C' row");
  extern __shared__ __align__(16) double hk_sm[];
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
  const int SA = hk_pad(ra), SBq = hk_pad(rb);
  const int M = ra * rb;
  double* QAs = hk_sm;              // [64][SA]
  double* QBs = QAs + 64 * SA;      // [64][SBq]
  double* Cs = QBs + 64 * SBq;      // [NSE][MC][SV]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(Cs + NSE * MC * SV);
  unsigned long long* empty = full + NSE;
  unsigned long long* qbar = empty + NSE;
  const i64 i0 = (i64)blockIdx.x * 64;
  const int b0 = blockIdx.y * BWC;
  const int bw = min(BWC, nrhs - b0);
  const int nr = int(min((i64)64, N - i0));
  const int nch = (M + MC - 1) / MC;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  // warp w: rows [16w, 16w+16) × all 16·NJ columns
  constexpr int JT = 2 * NJ;
  const int wi = warp * 16;
  if (tid == 0) {
    for (int s = 0; s < NSE; ++s) hk_mbar_init(full + s, 32), hk_mbar_init(empty + s, 4);
    hk_mbar_init(qbar, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  {  // this CTA's factor rows, once: threads 0..63 QTA rows, 64..127 QB rows
    const int row = tid & 63;
    if (row < nr) {
      const bool a = tid < 64;
      hk_mbar_arrive_tx(qbar, (a ? ra : rb) * 8);
      hk_bulk(a ? QAs + row * SA : QBs + row * SBq, a ? QTA + (i0 + row) * ra : QB + (i0 + row) * rb,
              (a ? ra : rb) * 8, qbar);
    } else {
      hk_mbar_arrive(qbar);  // rows past N only feed discarded outputs
    }
  }
  auto issue = [&](int c) {  // warp 0; lane L < MC moves C' row c·MC + L
    const int m = c * MC + lane;
    unsigned long long* b = full + c % NSE;
    if (lane < MC && m < M) {
      hk_mbar_arrive_tx(b, bw * 8);
      hk_bulk(Cs + (c % NSE) * MC * SV + lane * SV, Cp + (i64)m * nrhs + b0, bw * 8, b);
    } else {
      if (lane < MC) hk_zero_row(Cs + (c % NSE) * MC * SV + lane * SV, SV);
      hk_mbar_arrive(b);
    }
  };
  if (warp == 0)
    for (int c = 0; c < min(NSE, nch); ++c) issue(c);
  double acc[2][JT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int k = t4 / rb, l = t4 % rb;  // (k, l) of m = c·MC + kk + t4, advanced by 4 per step
  const double* qa_row[2];
  const double* qb_row[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    qa_row[i] = QAs + (wi + 8 * i + g) * SA;
    qb_row[i] = QBs + (wi + 8 * i + g) * SBq;
  }
  hk_mbar_wait(qbar, 0);
  for (int c = 0; c < nch; ++c) {
    const int sb = c % NSE;
    const unsigned ph = (c / NSE) & 1;
    hk_mbar_wait(full + sb, ph);
    const double* C1 = Cs + sb * MC * SV;
#pragma unroll
    for (int kk = 0; kk < MC; kk += 4) {
      const int kc = k < ra ? k : 0;  // m past M meets a zero C' row
      double af[2], bf[JT];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = qa_row[i][kc] * qb_row[i][l];
#pragma unroll
      for (int j = 0; j < JT; ++j) bf[j] = C1[(kk + t4) * SV + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < JT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      l += 4;
      while (l >= rb) l -= rb, ++k;
    }
    __syncwarp();
    if (lane == 0) hk_mbar_arrive(empty + sb);
    if (warp == 0 && c + NSE < nch) {
      hk_mbar_wait(empty + sb, ph);
      issue(c + NSE);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) {
      const i64 row = i0 + wi + 8 * i + g;
      const int bl = 8 * j + 2 * t4;
      if (row < N && bl < bw) {
        const i64 idx = row * nrhs + b0 + bl;
        double2 val = make_double2(acc[i][j][0], acc[i][j][1]);
        if (v) {
          const double nz = row < n_value ? nv2 : ng2;
          const double2 vv = *reinterpret_cast<const double2*>(v + idx);
          val.x += nz * vv.x, val.y += nz * vv.y;
        }
        if (accumulate) {
          const double2 o = *reinterpret_cast<const double2*>(out + idx);
          val.x += o.x, val.y += o.y;
        }
        *reinterpret_cast<double2*>(out + idx) = val;
      }
    }
}

// ---------------------------------------------------------------- small batches (nrhs ≤ 2)
// One or two right-hand sides (the merge-tree Lanczos of the build, single
// vector MVMs): the Khatri–Rao GEMMs degenerate to GEMVs and the 16-column
// DMMA tiles would waste ≥ 8×. Contraction: CTA = row range, thread t owns
// m = t, t+256, … (register accumulators), rows staged 32 at a time; fixed-
// order reduction of the CTA partials (k_had_reduce). Expansion: thread per
// row, C in shared memory, T_B folded into B's QT as in v3.
constexpr int HS_MMAX = 16;  // m per thread (ra·rb ≤ 256·HS_MMAX)
template <int NR>
__global__ void __launch_bounds__(256) k_had_contract_small(const double* __restrict__ QA, int ra,
                                                            const double* __restrict__ QB, int rb,
                                                            const double* __restrict__ V, i64 N, int nrhs,
                                                            double* __restrict__ partial) {
  __shared__ double qa[32][33], qb[32][33], vs[32][NR];
  const int M = ra * rb, tid = threadIdx.x;
  const i64 per = (N + gridDim.x - 1) / gridDim.x;
  const i64 r0 = min(N, (i64)blockIdx.x * per), r1 = min(N, r0 + per);
  int kk[HS_MMAX], ll[HS_MMAX];
  double acc[HS_MMAX][NR];
#pragma unroll
  for (int q = 0; q < HS_MMAX; ++q) {
    const int m = tid + 256 * q;
    kk[q] = m < M ? m / rb : 0;
    ll[q] = m < M ? m - kk[q] * rb : 0;
#pragma unroll
    for (int b = 0; b < NR; ++b) acc[q][b] = 0.0;
  }
  for (i64 rs = r0; rs < r1; rs += 32) {
    const int nr = int(min((i64)32, r1 - rs));
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int r = e / 32, c = e % 32;
      qa[r][c] = r < nr && c < ra ? QA[(rs + r) * ra + c] : 0.0;
      qb[r][c] = r < nr && c < rb ? QB[(rs + r) * rb + c] : 0.0;
    }
    for (int e = tid; e < 32 * NR; e += 256) {
      const int r = e / NR, b = e % NR;
      vs[r][b] = r < nr && b < nrhs ? V[(rs + r) * nrhs + b] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int q = 0; q < HS_MMAX; ++q) {
        if (tid + 256 * q >= M) break;
        const double z = qa[r][kk[q]] * qb[r][ll[q]];
#pragma unroll
        for (int b = 0; b < NR; ++b) acc[q][b] += z * vs[r][b];
      }
    }
  }
  double* out = partial + (i64)blockIdx.x * M * nrhs;
#pragma unroll
  for (int q = 0; q < HS_MMAX; ++q) {
    const int m = tid + 256 * q;
    if (m < M)
#pragma unroll
      for (int b = 0; b < NR; ++b)
        if (b < nrhs) out[(i64)m * nrhs + b] = acc[q][b];
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_had_expand_small(const double* __restrict__ QTA, int ra,
                                                          const double* __restrict__ QBT, int rb,
                                                          const double* __restrict__ C, i64 N, int nrhs,
                                                          const double* __restrict__ v, i64 n_value, double nv2,
                                                          double ng2, int accumulate, double* __restrict__ out) {
  extern __shared__ double cs[];  // [ra·rb][NR]
  const int M = ra * rb, tid = threadIdx.x;
  for (int e = tid; e < M * NR; e += 256) cs[e] = (e % NR) < nrhs ? C[(e / NR) * nrhs + e % NR] : 0.0;
  __syncthreads();
  const i64 row = (i64)blockIdx.x * 256 + tid;
  if (row >= N) return;
  const double* a = QTA + row * ra;
  const double* bq = QBT + row * rb;
  double res[NR];
#pragma unroll
  for (int b = 0; b < NR; ++b) res[b] = 0.0;
  for (int k = 0; k < ra; ++k) {
    double sk[NR];
#pragma unroll
    for (int b = 0; b < NR; ++b) sk[b] = 0.0;
    const double* ck = cs + (k * rb) * NR;
    for (int l = 0; l < rb; ++l) {
      const double w = __ldg(bq + l);
#pragma unroll
      for (int b = 0; b < NR; ++b) sk[b] += w * ck[l * NR + b];
    }
    const double ak = __ldg(a + k);
#pragma unroll
    for (int b = 0; b < NR; ++b) res[b] += ak * sk[b];
  }
#pragma unroll
  for (int b = 0; b < NR; ++b) {
    if (b >= nrhs) break;
    const i64 idx = row * nrhs + b;
    double val = res[b];
    if (v) val += (row < n_value ? nv2 : ng2) * v[idx];
    out[idx] = accumulate ? out[idx] + val : val;
  }
}

// fp64 tensor-core peak probe: 8 independent DMMA chains per warp, no memory
// traffic — the denominator of the D-SKIP roofline, measured on the running box.
__global__ void __launch_bounds__(128) k_dmma_peak(int iters, double* sink) {
  double acc[8][2];
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma_8x8x4(acc[c][0], acc[c][1], a, b);
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) t += acc[c][0] + acc[c][1];
  if (t == 12345.678) sink[0] = t;  // keep the chains alive
}

// diag = Π_f Σ_k QT_f[i][k] Q_f[i][k] (+ noise)   (dskip.cpp:141-149)
__global__ void k_had_diag(const double* const* __restrict__ Qs, const double* const* __restrict__ QTs,
                           const int* __restrict__ ranks, int nf, i64 N, i64 n_value, double nv2, double ng2,
                           double* __restrict__ d) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < N; i += (i64)gridDim.x * blockDim.x) {
    double prod = 1.0;
    for (int f = 0; f < nf; ++f) {
      const int r = ranks[f];
      double s = 0.0;
      for (int k = 0; k < r; ++k) s += QTs[f][i * r + k] * Qs[f][i * r + k];
      prod *= s;
    }
    d[i] = prod + (i < n_value ? nv2 : ng2);
  }
}

// row_i = Π_f Q_f t_f with t_f = T_f Q_f[i,:]ᵀ  (dskip.cpp:151-160); tvec packs all t_f
__global__ void k_had_row(const double* const* __restrict__ Qs, const int* __restrict__ ranks,
                          const int* __restrict__ toff, int nf, const double* __restrict__ tvec, i64 N,
                          i64 row, double noise, double* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < N; i += (i64)gridDim.x * blockDim.x) {
    double prod = 1.0;
    for (int f = 0; f < nf; ++f) {
      const int r = ranks[f];
      double s = 0.0;
      for (int k = 0; k < r; ++k) s += Qs[f][i * r + k] * tvec[toff[f] + k];
      prod *= s;
    }
    out[i] = prod + (i == row ? noise : 0.0);
  }
}

}  // namespace

double dmma_peak_tflops(int device) {
  DeviceGuard dg(device);
  const int sms = device_sm_count();
  double* sink = nullptr;
  GK_CUDA(cudaMalloc(&sink, sizeof(double)));
  cudaEvent_t e0, e1;
  GK_CUDA(cudaEventCreate(&e0));
  GK_CUDA(cudaEventCreate(&e1));
  const int iters = 4096, ctas = sms * 8;
  k_dmma_peak<<<ctas, 128>>>(64, sink);  // warm up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    GK_CUDA(cudaEventRecord(e0));
    k_dmma_peak<<<ctas, 128>>>(iters, sink);
    launched("dmma peak probe");
    GK_CUDA(cudaEventRecord(e1));
    GK_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    GK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  GK_CUDA(cudaEventDestroy(e0));
  GK_CUDA(cudaEventDestroy(e1));
  GK_CUDA(cudaFree(sink));
  const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (ctas * 4.0);  // per DMMA 512 flop, 8 chains, 4 warps/CTA
  return flops / (best * 1e-3) / 1e12;
}


// ================================================================ factor / ops
struct Factor {
  i64 N = 0;
  int r = 0;
  DevBuf<double> Q, QT;  // [N][r]
  std::vector<double> alpha, beta;
  DevBuf<double> ab;  // alpha (r) then beta (r-1)
  bool breakdown = false;
};

static std::unique_ptr<Factor> factor_from_lanczos(const double* Qc_dev, i64 N, const LanczosBatch& lb,
                                                   cudaStream_t s) {
  auto f = std::make_unique<Factor>();
  f->N = N;
  f->r = lb.len[0];
  f->alpha = lb.alpha[0];
  f->beta = lb.beta[0];
  f->breakdown = lb.breakdown[0] != 0;
  const int r = f->r;
  std::vector<double> ab(static_cast<size_t>(2 * std::max(r, 1)), 0.0);
  std::copy(f->alpha.begin(), f->alpha.end(), ab.begin());
  std::copy(f->beta.begin(), f->beta.end(), ab.begin() + r);
  f->ab.upload(ab.data(), ab.size(), s);
  f->Q.alloc(static_cast<size_t>(N) * std::max(r, 1));
  f->QT.alloc(static_cast<size_t>(N) * std::max(r, 1));
  if (r > 0) {
    k_factor_pack<<<blocks_for(N * r), 256, 0, s>>>(Qc_dev, N, r, f->ab.p, f->ab.p + r, f->Q.p, f->QT.p);
    launched("dskip factor pack");
  }
  GK_CUDA(cudaStreamSynchronize(s));
  return f;
}

// Factor from host data (Q N×r column-major, alpha, beta).
static std::unique_ptr<Factor> factor_from_host(const double* Q, i64 N, int r, const double* a, const double* b,
                                                cudaStream_t s) {
  LanczosBatch lb;
  lb.P = 1;
  lb.len = {r};
  lb.alpha = {std::vector<double>(a, a + r)};
  lb.beta = {std::vector<double>(b, b + std::max(r - 1, 0))};
  lb.breakdown = {0};
  DevBuf<double> Qc(static_cast<size_t>(N) * std::max(r, 1));
  Qc.upload(Q, static_cast<size_t>(N) * r, s);
  return factor_from_lanczos(Qc.p, N, lb, s);
}

// Hadamard pair MVM into `out` (RHS-minor [N][nrhs]); accumulate adds onto out.
struct HadScratch {
  DevBuf<double> partial, C, Cp;
};

static size_t had2_contract_smem(int ra, int rb, int nrhs) {
  return sizeof(double) * size_t(2 * HK_BK) * (hk_pad(ra) + hk_pad(rb) + hk_pad(nrhs));
}
static size_t had2_expand_smem(int ra, int rb, int nrhs) {
  return sizeof(double) * (size_t(64) * (hk_pad(ra) + hk_pad(rb)) + size_t(2 * HK_MC) * hk_pad(nrhs)) +
         sizeof(int2) * size_t(ra) * rb + 16;
}

template <int NJ>
static size_t had3_contract_smem(int ra, int rb) {
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
  return sizeof(double) * size_t(H3_NS) * H3_BK * (hk_pad(ra) + hk_pad(rb) + SV) + 16 * H3_NS;
}
template <int NJ, int MC, int NSE>
static size_t had3_expand_smem(int ra, int rb) {
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
  return sizeof(double) * (size_t(64) * (hk_pad(ra) + hk_pad(rb)) + size_t(NSE) * MC * SV) + 16 * NSE + 8;
}

template <int NJ, int MC, int NSE>
static void had3_expand_launch(const Factor& A, const Factor& B, const double* Cp, int nrhs, double* out,
                               bool accumulate, const double* noise_v, i64 n_value, double nv2, double ng2,
                               cudaStream_t s) {
  const size_t se = had3_expand_smem<NJ, MC, NSE>(A.r, B.r);
  raise_smem_limit((const void*)k_had_expand3<NJ, MC, NSE>, se);
  dim3 g3(static_cast<unsigned>((A.N + 63) / 64), static_cast<unsigned>((nrhs + 16 * NJ - 1) / (16 * NJ)));
  k_had_expand3<NJ, MC, NSE><<<g3, 128, se, s>>>(A.QT.p, A.r, B.QT.p, B.r, Cp, A.N, nrhs, noise_v, n_value, nv2,
                                                 ng2, accumulate ? 1 : 0, out);
  launched("hadamard expand (DMMA v3)");
}

template <int NJ>
static void hadamard_pair3_launch(const Factor& A, const Factor& B, const double* v, int nrhs, double* out,
                                  bool accumulate, const double* noise_v, i64 n_value, double nv2, double ng2,
                                  HadScratch& ws, cudaStream_t s) {
  const i64 N = A.N;
  const int M = A.r * B.r;
  const size_t sc = had3_contract_smem<NJ>(A.r, B.r);
  raise_smem_limit((const void*)k_had_contract3<NJ>, sc);
  const int mt = (M + 63) / 64, bt = (nrhs + 16 * NJ - 1) / (16 * NJ);
  // row-split so that all CTAs of the contraction are co-resident
  int per_sm = 0;
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_had_contract3<NJ>, 128, sc));
  const int slots = std::max(1, per_sm) * device_sm_count();
  int chunks = int(std::max<i64>(1, std::min<i64>(slots / (mt * bt), (N + 4 * H3_BK - 1) / (4 * H3_BK))));
  const i64 rows_per_chunk = ((N + chunks - 1) / chunks + H3_BK - 1) / H3_BK * H3_BK;
  chunks = int((N + rows_per_chunk - 1) / rows_per_chunk);
  ws.partial.reserve(static_cast<size_t>(chunks) * M * nrhs);
  ws.C.reserve(static_cast<size_t>(M) * nrhs);
  ws.Cp.reserve(static_cast<size_t>(M) * nrhs);
  dim3 g1(static_cast<unsigned>(mt), static_cast<unsigned>(bt), static_cast<unsigned>(chunks));
  k_had_contract3<NJ><<<g1, 128, sc, s>>>(A.Q.p, A.r, B.Q.p, B.r, v, N, nrhs, rows_per_chunk, ws.partial.p);
  launched("hadamard contract (DMMA v3)");
  k_had_reduce<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.partial.p, chunks, M, nrhs, ws.C.p);
  launched("hadamard reduce");
  // T_B is folded into the expansion: Σ_l QB[i][l] (T_B C)[k][l] = Σ_l (QB T_B)[i][l] C[k][l],
  // and QB T_B is the factor's stored QT — no tridiagonal pass
  switch (g_tuning.dskip_e.load()) {
    case 1: had3_expand_launch<NJ, 16, 2>(A, B, ws.C.p, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, s); break;
    case 2: had3_expand_launch<NJ, 16, 4>(A, B, ws.C.p, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, s); break;
    case 3: had3_expand_launch<NJ, 32, 2>(A, B, ws.C.p, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, s); break;
    default: had3_expand_launch<NJ, 8, 4>(A, B, ws.C.p, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, s);
  }
}

template <int NR>
static void hadamard_small_launch(const Factor& A, const Factor& B, const double* v, int nrhs, double* out,
                                  bool accumulate, const double* noise_v, i64 n_value, double nv2, double ng2,
                                  HadScratch& ws, cudaStream_t s) {
  const i64 N = A.N;
  const int M = A.r * B.r;
  const int chunks = int(std::max<i64>(1, std::min<i64>(296, (N + 63) / 64)));
  ws.partial.reserve(static_cast<size_t>(chunks) * M * nrhs);
  ws.C.reserve(static_cast<size_t>(M) * nrhs);
  k_had_contract_small<NR><<<chunks, 256, 0, s>>>(A.Q.p, A.r, B.Q.p, B.r, v, N, nrhs, ws.partial.p);
  launched("hadamard contract (small batch)");
  k_had_reduce<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.partial.p, chunks, M, nrhs, ws.C.p);
  launched("hadamard reduce");
  const size_t se = sizeof(double) * size_t(M) * NR;
  raise_smem_limit((const void*)k_had_expand_small<NR>, se);
  k_had_expand_small<NR><<<static_cast<unsigned>((N + 255) / 256), 256, se, s>>>(
      A.QT.p, A.r, B.QT.p, B.r, ws.C.p, N, nrhs, noise_v, n_value, nv2, ng2, accumulate ? 1 : 0, out);
  launched("hadamard expand (small batch)");
}

static bool hadamard_pair3(const Factor& A, const Factor& B, const double* v, int nrhs, double* out, bool accumulate,
                           const double* noise_v, i64 n_value, double nv2, double ng2, HadScratch& ws,
                           cudaStream_t s) {
  if (nrhs <= 2 && g_tuning.dskip.load() == 0 && A.r <= 32 && B.r <= 32 && A.r * B.r <= 256 * HS_MMAX) {
    if (nrhs == 1) hadamard_small_launch<1>(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s);
    else hadamard_small_launch<2>(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s);
    return true;
  }
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (g_tuning.dskip.load() != 0 || (A.r & 1) || (B.r & 1) || (nrhs & 1) || !al16(v) || !al16(out) ||
      (noise_v && !al16(noise_v)) || !al16(A.Q.p) || !al16(A.QT.p) || !al16(B.Q.p) || !al16(B.QT.p))
    return false;
  if (had3_expand_smem<4, 32, 2>(A.r, B.r) > 200 * 1024) return false;
  if (nrhs > 32)
    hadamard_pair3_launch<4>(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s);
  else if (nrhs > 16)
    hadamard_pair3_launch<2>(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s);
  else
    hadamard_pair3_launch<1>(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s);
  return true;
}

static bool hadamard_pair2(const Factor& A, const Factor& B, const double* v, int nrhs, double* out, bool accumulate,
                           const double* noise_v, i64 n_value, double nv2, double ng2, HadScratch& ws,
                           cudaStream_t s) {
  const i64 N = A.N;
  const int M = A.r * B.r;
  const size_t sc = had2_contract_smem(A.r, B.r, std::min(nrhs, 64));
  const size_t se = had2_expand_smem(A.r, B.r, std::min(nrhs, 64));
  if (g_tuning.dskip.load() == 1 || sc > 200 * 1024 || se > 200 * 1024) return false;
  raise_smem_limit((const void*)k_had_contract2, sc);
  raise_smem_limit((const void*)k_had_expand2, se);
  const int mt = (M + 63) / 64, bt = (nrhs + 63) / 64;
  // split rows so the contraction fills ~2 CTAs per SM
  int chunks = int(std::max<i64>(1, std::min<i64>((296 + mt * bt - 1) / (mt * bt), (N + 255) / 256)));
  const i64 rows_per_chunk = ((N + chunks - 1) / chunks + HK_BK - 1) / HK_BK * HK_BK;
  chunks = int((N + rows_per_chunk - 1) / rows_per_chunk);
  ws.partial.reserve(static_cast<size_t>(chunks) * M * nrhs);
  ws.C.reserve(static_cast<size_t>(M) * nrhs);
  ws.Cp.reserve(static_cast<size_t>(M) * nrhs);
  dim3 g1(static_cast<unsigned>(mt), static_cast<unsigned>(bt), static_cast<unsigned>(chunks));
  k_had_contract2<<<g1, 128, sc, s>>>(A.Q.p, A.r, B.Q.p, B.r, v, N, nrhs, rows_per_chunk, ws.partial.p);
  launched("hadamard contract (DMMA v2)");
  k_had_reduce<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.partial.p, chunks, M, nrhs, ws.C.p);
  launched("hadamard reduce");
  k_had_tridiag<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.C.p, A.r, B.r, nrhs, B.ab.p, B.ab.p + B.r, ws.Cp.p);
  launched("hadamard tridiag");
  dim3 g3(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>(bt));
  k_had_expand2<<<g3, 128, se, s>>>(A.QT.p, A.r, B.Q.p, B.r, ws.Cp.p, N, nrhs, noise_v, n_value, nv2, ng2,
                                    accumulate ? 1 : 0, out);
  launched("hadamard expand (DMMA v2)");
  return true;
}

static void hadamard_pair(const Factor& A, const Factor& B, const double* v, int nrhs, double* out, bool accumulate,
                          const double* noise_v, i64 n_value, double nv2, double ng2, HadScratch& ws,
                          cudaStream_t s) {
  if (hadamard_pair3(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s)) return;
  if (hadamard_pair2(A, B, v, nrhs, out, accumulate, noise_v, n_value, nv2, ng2, ws, s)) return;
  const i64 N = A.N;
  const int M = A.r * B.r;
  const int mt = (M + H_BM - 1) / H_BM, bt = (nrhs + H_BN - 1) / H_BN;
  // split rows so the contraction fills ~2 waves of 148 SMs
  int chunks = int(std::max<i64>(1, std::min<i64>((296 + mt * bt - 1) / (mt * bt), (N + 255) / 256)));
  const i64 rows_per_chunk = ((N + chunks - 1) / chunks + H_BK - 1) / H_BK * H_BK;
  chunks = int((N + rows_per_chunk - 1) / rows_per_chunk);
  ws.partial.reserve(static_cast<size_t>(chunks) * M * nrhs);
  ws.C.reserve(static_cast<size_t>(M) * nrhs);
  ws.Cp.reserve(static_cast<size_t>(M) * nrhs);
  dim3 g1(static_cast<unsigned>(mt), static_cast<unsigned>(bt), static_cast<unsigned>(chunks));
  k_had_contract<<<g1, 128, 0, s>>>(A.Q.p, A.r, B.Q.p, B.r, v, N, nrhs, rows_per_chunk, ws.partial.p);
  launched("hadamard contract");
  k_had_reduce<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.partial.p, chunks, M, nrhs, ws.C.p);
  launched("hadamard reduce");
  k_had_tridiag<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(ws.C.p, A.r, B.r, nrhs, B.ab.p, B.ab.p + B.r, ws.Cp.p);
  launched("hadamard tridiag");
  dim3 g3(static_cast<unsigned>((N + H_BM - 1) / H_BM), static_cast<unsigned>(bt));
  k_had_expand<<<g3, 128, 0, s>>>(A.QT.p, A.r, B.Q.p, B.r, ws.Cp.p, N, nrhs, noise_v, n_value, nv2, ng2,
                                  accumulate ? 1 : 0, out);
  launched("hadamard expand");
}

// The all-ones rank-1 factor: Hadamard identity element (Q = 1, T = [1]), so a
// single factor's Q T Qᵀ v runs through the same contraction exactly.
static std::unique_ptr<Factor> ones_factor(i64 N, cudaStream_t s) {
  auto f = std::make_unique<Factor>();
  f->N = N;
  f->r = 1;
  f->alpha = {1.0};
  std::vector<double> ab = {1.0, 0.0};
  f->ab.upload(ab.data(), 2, s);
  std::vector<double> ones(static_cast<size_t>(N), 1.0);
  f->Q.upload(ones.data(), ones.size(), s);
  f->QT.upload(ones.data(), ones.size(), s);
  GK_CUDA(cudaStreamSynchronize(s));
  return f;
}

// Leaf: OneDimFactor (dskip.cpp:40-113) over a 1-D D-SKI core.
struct LeafOp final : Op {
  std::unique_ptr<Op> core;
  i64 n = 0;
  int groups = 0, dir = -1;
  DevBuf<double> bi, bo;
  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {
    const int cg = dir >= 0 ? 2 : 1;
    bi.reserve(static_cast<size_t>(n) * cg * nrhs);
    bo.reserve(static_cast<size_t>(n) * cg * nrhs);
    const i64* ext = core->d_ext_of_int();
    k_leaf_combine<<<blocks_for(n * nrhs), 256, 0, s>>>(in, ext, n, groups, dir, nrhs, bi.p);
    launched("dskip leaf combine");
    dski_mvm_nonoise(*core, bi.p, bo.p, nrhs, s);
    k_leaf_expand<<<blocks_for(n * nrhs), 256, 0, s>>>(bo.p, ext, n, groups, dir, nrhs, out);
    launched("dskip leaf expand");
  }
  void diagonal(double*, cudaStream_t) override { fail(GK_ERR_LOGIC, "leaf diagonal not exposed"); }
  void row(i64, double*, cudaStream_t) override { fail(GK_ERR_LOGIC, "leaf rows not exposed"); }
};

// Lanczos-compressible operator: sum of Hadamard pairs (value merge: one pair;
// product-rule dlog merge: (dA, B) + (A, dB)).
struct PairOp final : Op {
  std::vector<std::pair<const Factor*, const Factor*>> pairs;
  HadScratch ws;
  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {
    for (size_t p = 0; p < pairs.size(); ++p)
      hadamard_pair(*pairs[p].first, *pairs[p].second, in, nrhs, out, p > 0, nullptr, 0, 0.0, 0.0, ws, s);
  }
  void diagonal(double*, cudaStream_t) override { fail(GK_ERR_LOGIC, "pair diagonal not exposed"); }
  void row(i64, double*, cudaStream_t) override { fail(GK_ERR_LOGIC, "pair rows not exposed"); }
};

static std::unique_ptr<Factor> lanczos_factor(Op& op, i64 rank, std::uint64_t seed, cudaStream_t s) {
  // lanczos_lowrank (linalg.cpp:306-314): normalised gaussian_vector(N, seed) start
  const bool prof = std::getenv("GK_BUILD_PROF") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  struct Done {
    bool on;
    std::chrono::steady_clock::time_point t0;
    cudaStream_t s;
    ~Done() {
      if (!on) return;
      cudaStreamSynchronize(s);
      std::fprintf(stderr, "dskip build: lanczos factor %.2f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  } done{prof, t0, s};
  const i64 N = op.N;
  std::vector<double> q(static_cast<size_t>(N));
  gaussian(N, seed, 0, q.data());
  double nn = 0.0;
  for (double v : q) nn += v * v;
  nn = std::sqrt(nn);
  for (double& v : q) v /= nn;
  DevBuf<double> start(static_cast<size_t>(N)), Qc(static_cast<size_t>(N) * rank);
  start.upload(q.data(), q.size(), s);
  if (prof) {
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "dskip build: start vector %.2f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  LanczosBatch lb = lanczos_batch(op, start.p, 1, int(rank), {mix_seed(seed, 1)}, Qc.p, s);
  if (prof) {
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "dskip build: lanczos done %.2f ms (len %d)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), lb.len[0]);
  }
  return factor_from_lanczos(Qc.p, N, lb, s);
}

struct DskipOp final : Op {
  i64 n = 0;
  int d = 0, groups = 0;
  std::vector<std::unique_ptr<Factor>> factors, dlog;
  std::unique_ptr<Factor> ones;
  bool track = false;
  HadScratch ws;

  const Factor& second() const { return factors.size() > 1 ? *factors[1] : *ones; }

  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {  // dskip.cpp:243-250
    const size_t before = ws.partial.n + ws.C.n + ws.Cp.n;
    hadamard_pair(*factors[0], second(), in, nrhs, out, false, in, n_value, nv2, ng2, ws, s);
    if (ws.partial.n + ws.C.n + ws.Cp.n != before) ++epoch;  // scratch moved: drop captured graphs
  }
  void dlogell(const double* in, double* out, int nrhs, cudaStream_t s) {  // dskip.cpp:266-274
    if (!track) fail(GK_ERR_LOGIC, "D-SKIP operator was built without derivative tracking");
    if (factors.size() == 1) {
      hadamard_pair(*dlog[0], *ones, in, nrhs, out, false, nullptr, 0, 0, 0, ws, s);
      return;
    }
    hadamard_pair(*dlog[0], *factors[1], in, nrhs, out, false, nullptr, 0, 0, 0, ws, s);
    hadamard_pair(*factors[0], *dlog[1], in, nrhs, out, true, nullptr, 0, 0, 0, ws, s);
  }
  void diagonal(double* dd, cudaStream_t s) override {
    std::vector<const double*> qs, qts;
    std::vector<int> rk;
    for (auto& f : factors) {
      qs.push_back(f->Q.p);
      qts.push_back(f->QT.p);
      rk.push_back(f->r);
    }
    DevBuf<const double*> dq, dqt;
    DevBuf<int> dr;
    dq.upload(qs.data(), qs.size(), s);
    dqt.upload(qts.data(), qts.size(), s);
    dr.upload(rk.data(), rk.size(), s);
    k_had_diag<<<blocks_for(N), 256, 0, s>>>(dq.p, dqt.p, dr.p, int(factors.size()), N, n_value, nv2, ng2, dd);
    launched("dskip diagonal");
    GK_CUDA(cudaStreamSynchronize(s));
  }
  void row(i64 r, double* out, cudaStream_t s) override {
    if (r < 0 || r >= N) fail(GK_ERR_RANGE, "D-SKIP row index out of range");
    std::vector<const double*> qs;
    std::vector<int> rk, toff;
    std::vector<double> tv;
    for (auto& f : factors) {
      const int rr = f->r;
      std::vector<double> qi(static_cast<size_t>(rr));
      GK_CUDA(cudaMemcpy(qi.data(), f->Q.p + r * rr, sizeof(double) * rr, cudaMemcpyDeviceToHost));
      toff.push_back(int(tv.size()));
      for (int k = 0; k < rr; ++k) {  // t = T q_i
        double t = f->alpha[static_cast<size_t>(k)] * qi[static_cast<size_t>(k)];
        if (k > 0) t += f->beta[static_cast<size_t>(k - 1)] * qi[static_cast<size_t>(k - 1)];
        if (k + 1 < rr) t += f->beta[static_cast<size_t>(k)] * qi[static_cast<size_t>(k + 1)];
        tv.push_back(t);
      }
      qs.push_back(f->Q.p);
      rk.push_back(rr);
    }
    DevBuf<const double*> dq;
    DevBuf<int> dr, dt;
    DevBuf<double> dtv;
    dq.upload(qs.data(), qs.size(), s);
    dr.upload(rk.data(), rk.size(), s);
    dt.upload(toff.data(), toff.size(), s);
    dtv.upload(tv.data(), tv.size(), s);
    const double noise = r < n_value ? nv2 : ng2;
    k_had_row<<<blocks_for(N), 256, 0, s>>>(dq.p, dr.p, dt.p, int(factors.size()), dtv.p, N, r, noise, out);
    launched("dskip row");
    GK_CUDA(cudaStreamSynchronize(s));
  }
};

std::unique_ptr<Op> make_dskip(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                               const gk_dskip_config& cfg, int device) {
  if (k.family != 0)
    fail(GK_ERR_ARG, "kernel family 'spline' is not separable; the Hadamard factorization needs a product kernel");
  if (!(k.lengthscale > 0.0)) fail(GK_ERR_ARG, "lengthscale must be > 0");
  if (!(k.outputscale > 0.0)) fail(GK_ERR_ARG, "outputscale must be > 0");
  if (d < 1 || n < 1) fail(GK_ERR_ARG, "D-SKIP needs points");
  DeviceGuard dg(device);
  auto op = std::make_unique<DskipOp>();
  op->kind = KIND_DSKIP;
  op->device = device;
  op->n = n;
  op->d = d;
  op->groups = cfg.with_gradients ? d : 0;
  op->N = n * (op->groups + 1);
  op->n_value = n;
  op->nv2 = nv * nv;
  op->ng2 = ng * ng;
  op->track = cfg.track_dlogell != 0;
  op->init_stream();
  cudaStream_t s = op->stream;
  const i64 N = op->N;
  const i64 rank = std::min<i64>(cfg.rank, N);
  if (rank < 1) fail(GK_ERR_ARG, "D-SKIP rank must be positive");
  // leaves (dskip.cpp:180-193): s_1d = s^(1/d), 1-D grid per dimension
  gk_kernel k1 = k;
  k1.outputscale = std::pow(k.outputscale, 1.0 / d);
  std::vector<double> col(static_cast<size_t>(n));
  for (int j = 0; j < d; ++j) {
    std::copy(X + j * n, X + (j + 1) * n, col.begin());
    gk_grid g1{};
    {
      // Grid::cover(X.col(j), ell*grid_ratio, 3, max_grid_nodes)
      const double target = k.lengthscale * cfg.grid_ratio;
      if (!(target > 0.0)) fail(GK_ERR_ARG, "grid spacing must be positive");
      double lo = col[0], hi = col[0];
      for (double v : col) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
      }
      const double span = std::max(hi - lo, 1e-12);
      double h = target;
      int m = int(std::ceil(span / h)) + 1 + 6;
      if (m > cfg.max_grid_nodes) {
        m = cfg.max_grid_nodes;
        h = span / double(m - 1 - 6);
      }
      if (m < 12) m = 12;
      g1.d = 1;
      g1.dims[0] = m;
      g1.spacing[0] = h;
      g1.origin[0] = lo - 3 * h;
    }
    const int dir = cfg.with_gradients ? j : -1;
    for (int pass = 0; pass < (op->track ? 2 : 1); ++pass) {
      LeafOp leaf;
      leaf.kind = KIND_DSKIP;
      leaf.device = device;
      leaf.n = n;
      leaf.groups = op->groups;
      leaf.dir = dir;
      leaf.N = N;
      leaf.n_value = n;
      const auto tl0 = std::chrono::steady_clock::now();
      leaf.core = make_dski_profile(k1, g1, col.data(), n, 0.0, 0.0, 0, dir >= 0 ? 1 : 0, device, pass);
      if (std::getenv("GK_BUILD_PROF")) {
        cudaDeviceSynchronize();
        std::fprintf(stderr, "dskip build: leaf core %.2f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count());
      }
      const std::uint64_t seed = mix_seed(cfg.seed, pass == 0 ? std::uint64_t(j) : std::uint64_t(100 + j));
      auto f = lanczos_factor(leaf, rank, seed, s);
      (pass == 0 ? op->factors : op->dlog).push_back(std::move(f));
    }
  }
  // balanced pairwise merges (dskip.cpp:197-233)
  std::uint64_t merge_id = 1000;
  while (op->factors.size() > 2) {
    std::vector<std::unique_ptr<Factor>> next, dnext;
    for (size_t a = 0; a + 1 < op->factors.size(); a += 2) {
      const Factor& A = *op->factors[a];
      const Factor& B = *op->factors[a + 1];
      const i64 product_rank = std::min<i64>(i64(A.r) * B.r, N);
      if (cfg.rank_policy_error && product_rank > rank)
        fail(GK_ERR_RUNTIME, "intermediate Hadamard rank " + std::to_string(product_rank) + " exceeds the cap " +
                                 std::to_string(rank));
      PairOp pop;
      pop.device = device;
      pop.N = N;
      pop.n_value = N;
      pop.pairs = {{&A, &B}};
      next.push_back(lanczos_factor(pop, rank, mix_seed(cfg.seed, ++merge_id), s));
      if (op->track) {
        PairOp dpop;
        dpop.device = device;
        dpop.N = N;
        dpop.n_value = N;
        dpop.pairs = {{op->dlog[a].get(), &B}, {&A, op->dlog[a + 1].get()}};
        dnext.push_back(lanczos_factor(dpop, rank, mix_seed(cfg.seed, ++merge_id), s));
      }
    }
    if (op->factors.size() % 2 == 1) {
      next.push_back(std::move(op->factors.back()));
      if (op->track) dnext.push_back(std::move(op->dlog.back()));
    }
    op->factors = std::move(next);
    op->dlog = std::move(dnext);
  }
  op->ones = ones_factor(N, s);
  return op;
}

// D-SKIP operator from explicit factors (e.g. uploaded from the oracle), so the
// Hadamard MVM itself can be checked at 1e-12 independently of Lanczos.
std::unique_ptr<Op> make_dskip_from_factors(i64 n, int groups, double nv, double ng, int nf, const i64* ranks,
                                            const double* const* Q, const double* const* alpha,
                                            const double* const* beta, int device) {
  if (nf < 1 || nf > 2) fail(GK_ERR_ARG, "D-SKIP needs one or two factors");
  DeviceGuard dg(device);
  auto op = std::make_unique<DskipOp>();
  op->kind = KIND_DSKIP;
  op->device = device;
  op->n = n;
  op->groups = groups;
  op->N = n * (groups + 1);
  op->n_value = n;
  op->nv2 = nv * nv;
  op->ng2 = ng * ng;
  op->init_stream();
  for (int f = 0; f < nf; ++f)
    op->factors.push_back(factor_from_host(Q[f], op->N, int(ranks[f]), alpha[f], beta[f], op->stream));
  op->ones = ones_factor(op->N, op->stream);
  return op;
}

static const DskipOp& as_dskip(const Op& o) {
  if (o.kind != KIND_DSKIP) fail(GK_ERR_ARG, "operator is not a D-SKIP operator");
  return static_cast<const DskipOp&>(o);
}

int dskip_factor_count(const Op& o) { return int(as_dskip(o).factors.size()); }
i64 dskip_factor_rank(const Op& o, int f) {
  const auto& op = as_dskip(o);
  if (f < 0 || f >= int(op.factors.size())) fail(GK_ERR_RANGE, "factor index out of range");
  return op.factors[static_cast<size_t>(f)]->r;
}
void dskip_factor_get(const Op& o, int f, double* Q, double* a, double* b) {
  const auto& op = as_dskip(o);
  if (f < 0 || f >= int(op.factors.size())) fail(GK_ERR_RANGE, "factor index out of range");
  const Factor& F = *op.factors[static_cast<size_t>(f)];
  if (Q) {
    std::vector<double> rm(static_cast<size_t>(F.N) * F.r);
    GK_CUDA(cudaMemcpy(rm.data(), F.Q.p, sizeof(double) * rm.size(), cudaMemcpyDeviceToHost));
    for (i64 i = 0; i < F.N; ++i)
      for (int k = 0; k < F.r; ++k) Q[static_cast<size_t>(k) * F.N + i] = rm[static_cast<size_t>(i) * F.r + k];
  }
  if (a) std::copy(F.alpha.begin(), F.alpha.end(), a);
  if (b) std::copy(F.beta.begin(), F.beta.end(), b);
}
void dskip_dlogell(Op& o, const double* in, double* out, int nrhs, cudaStream_t s) {
  if (o.kind != KIND_DSKIP) fail(GK_ERR_ARG, "operator is not a D-SKIP operator");
  static_cast<DskipOp&>(o).dlogell(in, out, nrhs, s);
}

}  // namespace gk
