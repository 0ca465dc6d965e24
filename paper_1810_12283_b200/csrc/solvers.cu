#include <type_traits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
// solvers.cu — device-resident batched solvers (reference linalg.cpp).
//
//  * pcg_internal: the reference's single-RHS PCG (linalg.cpp:85-131) run
//    for nrhs independent columns at once: per-column alpha/beta, per-column
//    stopping (converged / pAp <= 0 stall / max_iterations), frozen columns
//    after they stop. One iteration is captured into a CUDA graph; the host
//    only polls the number of active columns between graph launches.
//  * pivchol_run: pivoted Cholesky (linalg.cpp:133-174) with the row fetched
//    from the operator on device; argmax tie-break = lowest external index
//    (Eigen maxCoeff semantics).
//  * precond_build / Precond::apply: Q1 of [D^{-1/2}F; I] by CholeskyQR2
//    (two Gram + k×k Cholesky passes), applied as two rank-k contractions.
//  * lanczos_batch: Lanczos with two-pass full reorthogonalisation and
//    deflating restarts (linalg.cpp:17-81) for P probes in lockstep.
// All reductions are deterministic (fixed partition, fixed summation order).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "gk_kernels.cuh"
#include "pcg_fused.hpp"
#include "solvers.hpp"

namespace gk {

namespace {

constexpr int RB = kRedBlocks;
constexpr int RT = kRedThreads;

__device__ __forceinline__ void row_range(i64 rows, i64& r0, i64& r1) {
  const i64 per = (rows + gridDim.x - 1) / gridDim.x;
  r0 = (i64)blockIdx.x * per;
  r1 = min(rows, r0 + per);
}

// Reduce per-thread values of layout (slot, b) into partial[blockIdx][b].
__device__ __forceinline__ void block_col_store(double acc, int nrhs, double* partial, double* sm) {
  const int tid = threadIdx.x;
  const int slots = blockDim.x / nrhs;
  __syncthreads();
  sm[tid] = acc;
  __syncthreads();
  if (tid < nrhs) {
    double s = 0.0;
    for (int k = 0; k < slots; ++k) s += sm[k * nrhs + tid];
    partial[(i64)blockIdx.x * nrhs + tid] = s;
  }
}

__device__ __forceinline__ double sum_partials(const double* partial, int nblocks, int stride, int idx) {
  double s = 0.0;
  for (int k = 0; k < nblocks; ++k) s += partial[(i64)k * stride + idx];
  return s;
}

// Warp-cooperative, fixed-order sum of nblocks partials: lane l sums blocks
// l, l+32, …; then a butterfly. Same order every run (deterministic), and
// the ~nblocks/32 loads per lane are independent (no serial latency chain).
__device__ __forceinline__ double warp_sum_partials(const double* partial, int nblocks, int stride, int idx) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int k = lane; k < nblocks; k += 32) s += partial[(i64)k * stride + idx];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__global__ void k_dot_partial(const double* __restrict__ x, const double* __restrict__ y, i64 rows, int nrhs,
                              double* __restrict__ partial) {
  __shared__ double sm[RT];
  const int slots = blockDim.x / nrhs;
  const int b = threadIdx.x % nrhs, slot = threadIdx.x / nrhs;
  double acc = 0.0;
  if (slot < slots) {
    i64 r0, r1;
    row_range(rows, r0, r1);
    for (i64 r = r0 + slot; r < r1; r += slots) acc += x[r * nrhs + b] * y[r * nrhs + b];
  }
  block_col_store(acc, nrhs, partial, sm);
}

// ---------------------------------------------------------------- PCG
using CgDev = PcgState;

// init: partial0 = ||b||², partial1 = r·z, partial2 = r·r (r = b)
// One 32-thread block per column; partials reduced warp-cooperatively.
__global__ void k_cg_init(CgDev st, const double* __restrict__ p_bb, const double* __restrict__ p_rz,
                          const double* __restrict__ p_rr) {
  const int b = blockIdx.x;
  const double bb = warp_sum_partials(p_bb, RB, st.nrhs, b);
  const double rz = warp_sum_partials(p_rz, RB, st.nrhs, b);
  const double rr = warp_sum_partials(p_rr, RB, st.nrhs, b);
  if (threadIdx.x != 0) return;
  const double bn = sqrt(bb);
  st.bnorm[b] = bn;
  st.its[b] = 0;
  st.upd[b] = 0;
  if (bn == 0.0) {  // linalg.cpp:93-96: zero rhs -> converged, no history
    st.conv[b] = 1;
    st.active[b] = 0;
    st.rz[b] = 0.0;
  } else {
    st.rz[b] = rz;
    const double relres = sqrt(rr) / bn;
    st.hist[b] = relres;
    const bool done = relres <= st.tol;  // :104-109
    st.conv[b] = done ? 1 : 0;
    st.active[b] = done ? 0 : 1;
    if (!done) atomicAdd(st.nactive, 1);  // zeroed before launch
  }
}

__global__ void k_cg_fin_pAp(CgDev st, const double* __restrict__ partial) {
  const int b = blockIdx.x;
  const double pAp = warp_sum_partials(partial, RB, st.nrhs, b);
  if (threadIdx.x != 0) return;
  if (b == 0) *st.nactive = 0;  // recounted by k_cg_fin_rr (stream-ordered after this kernel)
  st.upd[b] = 0;
  if (!st.active[b]) return;
  if (st.its[b] >= st.maxit) {  // loop bound reached, unconverged
    st.active[b] = 0;
    return;
  }
  if (pAp <= 0.0) {  // linalg.cpp:114: loss of definiteness -> stalled
    st.active[b] = 0;
    return;
  }
  st.alpha[b] = st.rz[b] / pAp;
  st.upd[b] = 1;
  st.its[b] += 1;
}

// alpha = rz / pAp (linalg.cpp:110-118) evaluated by every CTA from the pAp
// partials (fixed-order sums: identical everywhere), then x += a p,
// r -= a Ap on this CTA's rows and ||r||² partials. No state is written here:
// k_cg_fin_rr re-derives the same decision and updates the column state
// (a CTA writing state other CTAs still read would race).
__device__ __forceinline__ bool cg_alpha(const CgDev& st, int b, double pAp, double& alpha) {
  alpha = 0.0;
  if (!st.active[b] || st.its[b] >= st.maxit || pAp <= 0.0) return false;
  alpha = st.rz[b] / pAp;
  return true;
}

__global__ void k_cg_axpy(CgDev st, double* __restrict__ X, double* __restrict__ R, const double* __restrict__ P,
                          const double* __restrict__ AP, i64 rows, const double* __restrict__ p_pAp,
                          double* __restrict__ partial) {
  __shared__ double sm[RT];
  __shared__ double s_alpha[RT];
  __shared__ int s_upd[RT];
  const int nrhs = st.nrhs;
  const int warp = threadIdx.x / 32;
  for (int c = warp; c < nrhs; c += RT / 32) {
    const double pAp = warp_sum_partials(p_pAp, RB, nrhs, c);
    if ((threadIdx.x & 31) == 0) {
      double a;
      s_upd[c] = cg_alpha(st, c, pAp, a) ? 1 : 0;
      s_alpha[c] = a;
    }
  }
  __syncthreads();
  const int slots = blockDim.x / nrhs;
  const int b = threadIdx.x % nrhs, slot = threadIdx.x / nrhs;
  double acc = 0.0;
  if (slot < slots && s_upd[b]) {
    const double a = s_alpha[b];
    i64 r0, r1;
    row_range(rows, r0, r1);
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const i64 i = r * nrhs + b;
      X[i] += a * P[i];
      const double rn = R[i] - a * AP[i];
      R[i] = rn;
      acc += rn * rn;
    }
  }
  block_col_store(acc, nrhs, partial, sm);
}

__global__ void k_cg_fin_rr(CgDev st, const double* __restrict__ p_pAp, const double* __restrict__ partial) {
  const int b = blockIdx.x;
  const double pAp = warp_sum_partials(p_pAp, RB, st.nrhs, b);
  const double rr = warp_sum_partials(partial, RB, st.nrhs, b);
  if (threadIdx.x != 0) return;
  // the alpha decision k_cg_axpy made (same inputs, same arithmetic)
  double a;
  const bool upd = cg_alpha(st, b, pAp, a);
  st.upd[b] = upd ? 1 : 0;
  if (st.active[b] && !upd) st.active[b] = 0;  // max iterations reached, or pAp <= 0 (:114)
  if (upd) {
    st.alpha[b] = a;
    st.its[b] += 1;
    const double relres = sqrt(rr) / st.bnorm[b];
    st.hist[(i64)st.its[b] * st.nrhs + b] = relres;
    if (relres <= st.tol) {  // :121-125
      st.conv[b] = 1;
      st.active[b] = 0;
    }
  }
  if (st.active[b]) atomicAdd(st.nactive, 1);
}

__global__ void k_cg_fin_rz(CgDev st, const double* __restrict__ partial, int nblocks) {
  const int b = blockIdx.x;
  const double rzn = warp_sum_partials(partial, nblocks, st.nrhs, b);
  if (threadIdx.x != 0 || !st.active[b]) return;
  st.beta[b] = rzn / st.rz[b];
  st.rz[b] = rzn;
}

__global__ void k_cg_pupdate(CgDev st, double* __restrict__ P, const double* __restrict__ Z, i64 rows) {
  const int nrhs = st.nrhs;
  const i64 items = rows * nrhs;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < items; i += (i64)gridDim.x * blockDim.x) {
    const int b = int(i) % nrhs;  // 32-bit: N·nrhs < 2^31
    if (st.active[b]) P[i] = Z[i] + st.beta[b] * P[i];
  }
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_fill(double* __restrict__ a, double v, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) a[i] = v;
}

// ---------------------------------------------------------------- preconditioner
// partial T[j][b] = Σ_rows q1[r][j] (dinv[r] r[r][b]); also partial Σ c² per b
// (for quadratic()). Rows are staged 16 at a time in shared memory; outputs
// o = j*nrhs + b are owned by one thread each and accumulate in smem.
constexpr int PC_RT = 16;
// q1 may be a column slice [j0, j0 + k) of the [N][ld] factor (ld = row stride).
__global__ void k_pc_proj(const double* __restrict__ Rv, const double* __restrict__ dinv,
                          const double* __restrict__ q1, i64 N, int k, int ld, int nrhs, double* __restrict__ partial,
                          double* __restrict__ partial_cc) {
  extern __shared__ double sh[];
  double* qs = sh;                     // [PC_RT][k]
  double* cs = qs + PC_RT * k;         // [PC_RT][nrhs]
  double* acc = cs + PC_RT * nrhs;     // [k*nrhs]
  const int tid = threadIdx.x;
  const int nout = k * nrhs;
  for (int o = tid; o < nout; o += blockDim.x) acc[o] = 0.0;
  double cc = 0.0;  // Σ c² for column tid (tid < nrhs)
  i64 r0, r1;
  row_range(N, r0, r1);
  for (i64 rt = r0; rt < r1; rt += PC_RT) {
    const int nr = int((r1 - rt) < PC_RT ? (r1 - rt) : PC_RT);
    __syncthreads();
    for (int e = tid; e < nr * k; e += blockDim.x) qs[e] = q1[(rt + e / k) * ld + e % k];
    for (int e = tid; e < nr * nrhs; e += blockDim.x) {
      const int rr = e / nrhs;
      cs[e] = dinv[rt + rr] * Rv[(rt + rr) * nrhs + (e % nrhs)];
    }
    __syncthreads();
    if (tid < nrhs)
      for (int rr = 0; rr < nr; ++rr) cc += cs[rr * nrhs + tid] * cs[rr * nrhs + tid];
    for (int o = tid; o < nout; o += blockDim.x) {
      const int j = o / nrhs, b = o % nrhs;
      double a = acc[o];
      for (int rr = 0; rr < nr; ++rr) a += qs[rr * k + j] * cs[rr * nrhs + b];
      acc[o] = a;
    }
  }
  __syncthreads();
  for (int o = tid; o < nout; o += blockDim.x) partial[(i64)blockIdx.x * nout + o] = acc[o];
  if (partial_cc && tid < nrhs) partial_cc[(i64)blockIdx.x * nrhs + tid] = cc;
}

// out[o] = Σ_blocks partial[blk][o], one warp per output (blocks of 8 warps).
__global__ void k_pc_fin(const double* __restrict__ partial, int nout, double* __restrict__ T) {
  const int o = blockIdx.x * 8 + threadIdx.x / 32;
  if (o >= nout) return;
  const double v = warp_sum_partials(partial, RB, nout, o);
  if ((threadIdx.x & 31) == 0) T[o] = v;
}
inline unsigned fin_blocks(int nout) { return static_cast<unsigned>((nout + 7) / 8); }

// z = dinv (dinv r - Q1 T); partial Σ r·z
__global__ void k_pc_apply(const double* __restrict__ Rv, const double* __restrict__ dinv,
                           const double* __restrict__ q1, const double* __restrict__ T, i64 N, int k, int nrhs,
                           double* __restrict__ Z, double* __restrict__ partial_rz) {
  extern __shared__ double sh[];
  double* Ts = sh;  // [k][nrhs]
  double* sm = Ts + k * nrhs;
  for (int o = threadIdx.x; o < k * nrhs; o += blockDim.x) Ts[o] = T[o];
  __syncthreads();
  const int slots = blockDim.x / nrhs;
  const int b = threadIdx.x % nrhs, slot = threadIdx.x / nrhs;
  double acc = 0.0;
  if (slot < slots) {
    i64 r0, r1;
    row_range(N, r0, r1);
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const double di = dinv[r];
      const double rv = Rv[r * nrhs + b];
      double s = 0.0;
      const double* qr = q1 + r * k;
      for (int j = 0; j < k; ++j) s += qr[j] * Ts[j * nrhs + b];
      const double z = di * (di * rv - s);
      Z[r * nrhs + b] = z;
      acc += rv * z;
    }
  }
  if (partial_rz) block_col_store(acc, nrhs, partial_rz, sm);
}

// z = dinv (dinv r − S) for a precomputed S = Q1 T (large ranks); partial Σ r·z
// in k_pc_apply's layout.
__global__ void k_pc_finish_s(const double* __restrict__ Rv, const double* __restrict__ dinv,
                              const double* __restrict__ S, i64 N, int nrhs, double* __restrict__ Z,
                              double* __restrict__ partial_rz) {
  __shared__ double sm[kRedThreads];
  const int slots = blockDim.x / nrhs;
  const int b = threadIdx.x % nrhs, slot = threadIdx.x / nrhs;
  double acc = 0.0;
  if (slot < slots) {
    i64 r0, r1;
    row_range(N, r0, r1);
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const double di = dinv[r];
      const double rv = Rv[r * nrhs + b];
      const double z = di * (di * rv - S[r * nrhs + b]);
      Z[r * nrhs + b] = z;
      acc += rv * z;
    }
  }
  if (partial_rz) block_col_store(acc, nrhs, partial_rz, sm);
}

// ---- DMMA versions of the two rank-k contractions (fp64 tensor cores).
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
constexpr int PCM_MAXI = 7, PCM_MAXJ = 8;  // per-warp m8 tiles × n8 tiles (k ≤ 224, nrhs ≤ 64)

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// partial T = Q1ᵀ C over this CTA's rows, C = D^{-1/2} R. Rows are staged in
// phases of PCM_RCH with cp.async (every global load in flight at once);
// output (kp × np) tiles: warp w owns m-tiles i ≡ w (mod 4) and all n-tiles.
constexpr int PCM_RCH = 112;
__global__ void __launch_bounds__(128) k_pc_proj_mma(const double* __restrict__ Rv, const double* __restrict__ dinv,
                                                     const double* __restrict__ q1, i64 N, int k, int nrhs,
                                                     int rch, double* __restrict__ partial) {
  const int kp = (k + 7) / 8 * 8, np = (nrhs + 7) / 8 * 8;
  const int SQ = kp + 8, SC = np + 8;
  extern __shared__ double sh[];
  double* Qs = sh;                // [rch][SQ]
  double* Cs = Qs + rch * SQ;     // [rch][SC]
  double* Ds = Cs + rch * SC;     // [rch]
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31, g = lane / 4, t4 = lane & 3;
  const int mt = kp / 8, nt = np / 8;
  double acc[PCM_MAXI][PCM_MAXJ][2];
#pragma unroll
  for (int i = 0; i < PCM_MAXI; ++i)
#pragma unroll
    for (int j = 0; j < PCM_MAXJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  i64 r0, r1;
  row_range(N, r0, r1);
  for (i64 rt = r0; rt < r1; rt += rch) {
    const int nr = int((r1 - rt) < rch ? (r1 - rt) : rch);
    const int nrp = (nr + 3) / 4 * 4;
    __syncthreads();
    for (int e = tid; e < nrp * kp; e += 128) {
      const int rr = e / kp, j = e - rr * kp;
      if (rr < nr && j < k) cp_async8(Qs + rr * SQ + j, q1 + (rt + rr) * k + j);
      else Qs[rr * SQ + j] = 0.0;
    }
    for (int e = tid; e < nrp * np; e += 128) {
      const int rr = e / np, bb = e - rr * np;
      if (rr < nr && bb < nrhs) cp_async8(Cs + rr * SC + bb, Rv + (rt + rr) * nrhs + bb);
      else Cs[rr * SC + bb] = 0.0;
    }
    for (int rr = tid; rr < nrp; rr += 128) {
      if (rr < nr) cp_async8(Ds + rr, dinv + rt + rr);
      else Ds[rr] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    for (int kk = 0; kk < nrp; kk += 4) {
      const double dk = Ds[kk + t4];
      double bf[PCM_MAXJ];
#pragma unroll
      for (int j = 0; j < PCM_MAXJ; ++j) bf[j] = j < nt ? dk * Cs[(kk + t4) * SC + 8 * j + g] : 0.0;
#pragma unroll
      for (int ii = 0; ii < PCM_MAXI; ++ii) {
        const int i = warp + 4 * ii;
        if (i >= mt) break;
        const double af = Qs[(kk + t4) * SQ + 8 * i + g];  // A = Q1ᵀ: (j, row)
#pragma unroll
        for (int j = 0; j < PCM_MAXJ; ++j)
          if (j < nt) dmma_f64(acc[ii][j][0], acc[ii][j][1], af, bf[j]);
      }
    }
  }
  double* out = partial + (i64)blockIdx.x * k * nrhs;
#pragma unroll
  for (int ii = 0; ii < PCM_MAXI; ++ii) {
    const int i = warp + 4 * ii;
    if (i >= mt) break;
    const int j0 = 8 * i + g;
#pragma unroll
    for (int jn = 0; jn < PCM_MAXJ; ++jn) {
      if (jn >= nt) break;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int bb = 8 * jn + 2 * t4 + e;
        if (j0 < k && bb < nrhs) out[(i64)j0 * nrhs + bb] = acc[ii][jn][e];
      }
    }
  }
}

// ---------------------------------------------------------------- preconditioner GEMMs v3
// The rank-k projection T = Q1ᵀ D^{-1/2} r and the apply
// z = D^{-1/2}(D^{-1/2} r − Q1 T) as fp64 tensor-core GEMMs in the shape of the
// D-SKIP Khatri–Rao kernels: rows arrive by per-row TMA bulk copies
// (cp.async.bulk + mbarrier rings, one issuing warp), shared strides ≡ 4
// (mod 16) doubles, warp tiles of 16 (m or rows) × all RHS. Needs an even rank
// and an even RHS count (16-byte rows); other shapes use the kernels above.
__host__ __device__ __forceinline__ int p3_pad(int x) { return x + ((4 - x % 16) + 16) % 16; }
__device__ __forceinline__ unsigned p3_su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void p3_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(p3_su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void p3_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(p3_su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void p3_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(p3_su32(b)) : "memory");
}
__device__ __forceinline__ void p3_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nP3W_%=:\nmbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n@!P1 bra P3W_%=;\n}\n" ::"r"(
          p3_su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void p3_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   p3_su32(dst)),
               "l"(src), "r"(bytes), "r"(p3_su32(b))
               : "memory");
}

constexpr int P3_BK = 16, P3_NS = 3;   // projection: rows per stage, ring depth
constexpr int P3_MC = 8, P3_NSE = 4;   // apply: m per T stage, ring depth

// partial[chunk][m][b] = Σ_{rows in chunk} Q1[row][m] d[row] r[row][b]
template <int NJ>
__global__ void __launch_bounds__(128, 4) k_pc_proj3(const double* __restrict__ q1, int k,
                                                     const double* __restrict__ dinv, const double* __restrict__ R,
                                                     i64 N, int nrhs, i64 rows_per_chunk,
                                                     double* __restrict__ partial) {
  extern __shared__ __align__(16) double p3_sm[];
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16, JT = 2 * NJ;
  const int SA = p3_pad(k);
  const int stage_d = P3_BK * (SA + SV + 1);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(p3_sm + P3_NS * stage_d);
  unsigned long long* empty = full + P3_NS;
  const int m0 = blockIdx.x * 64, b0 = blockIdx.y * BWC;
  const int bw = min(BWC, nrhs - b0);
  const i64 r_begin = (i64)blockIdx.z * rows_per_chunk;
  const i64 r_end = min(N, r_begin + rows_per_chunk);
  const int nst = r_end > r_begin ? int((r_end - r_begin + P3_BK - 1) / P3_BK) : 0;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  const int wm = warp * 16;
  if (tid == 0) {
    for (int s = 0; s < P3_NS; ++s) p3_mbar_init(full + s, 32), p3_mbar_init(empty + s, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // warp 0 fills a stage: lanes 0..15 Q1 row + r row, lane 16 the 16 D^{-1/2} values
  auto issue = [&](int st) {
    const i64 rs = r_begin + (i64)st * P3_BK;
    const int nr = int(min((i64)P3_BK, r_end - rs));
    double* base = p3_sm + (st % P3_NS) * stage_d;
    unsigned long long* bar = full + st % P3_NS;
    if (lane < P3_BK) {
      double* qd = base + lane * SA;
      double* vd = base + P3_BK * SA + lane * SV;
      if (lane < nr) {
        p3_arrive_tx(bar, unsigned(k + bw) * 8u);
        p3_bulk(qd, q1 + (rs + lane) * k, unsigned(k) * 8u, bar);
        p3_bulk(vd, R + (rs + lane) * nrhs + b0, unsigned(bw) * 8u, bar);
      } else {
        for (int c = 0; c < SA; ++c) qd[c] = 0.0;
        for (int c = 0; c < SV; ++c) vd[c] = 0.0;
        p3_arrive(bar);
      }
    } else if (lane == P3_BK) {
      double* dd = base + P3_BK * (SA + SV);
      if (nr == P3_BK) {
        p3_arrive_tx(bar, P3_BK * 8u);
        p3_bulk(dd, dinv + rs, P3_BK * 8u, bar);
      } else {
        for (int c = 0; c < P3_BK; ++c) dd[c] = c < nr ? dinv[rs + c] : 0.0;
        p3_arrive(bar);
      }
    } else {
      p3_arrive(bar);
    }
  };
  int mi[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) mi[i] = min(m0 + wm + 8 * i + g, k - 1);
  double acc[2][JT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (warp == 0)
    for (int s = 0; s < min(P3_NS, nst); ++s) issue(s);
  for (int it = 0; it < nst; ++it) {
    const int sb = it % P3_NS;
    const unsigned ph = (it / P3_NS) & 1;
    p3_wait(full + sb, ph);
    const double* A1 = p3_sm + sb * stage_d;
    const double* V1 = A1 + P3_BK * SA;
    const double* D1 = V1 + P3_BK * SV;
#pragma unroll
    for (int kk = 0; kk < P3_BK; kk += 4) {
      const int row = kk + t4;
      const double dr = D1[row];
      double af[2], bf[JT];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = A1[row * SA + mi[i]] * dr;
#pragma unroll
      for (int j = 0; j < JT; ++j) bf[j] = V1[row * SV + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < JT; ++j) dmma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) p3_arrive(empty + sb);
    if (warp == 0 && it + P3_NS < nst) {
      p3_wait(empty + sb, ph);
      issue(it + P3_NS);
    }
  }
  double* out = partial + (i64)blockIdx.z * k * nrhs;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) {
      const int m = m0 + wm + 8 * i + g, bl = 8 * j + 2 * t4;
      if (m < k && bl < bw)
        *reinterpret_cast<double2*>(out + (i64)m * nrhs + b0 + bl) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// z = d (d r − Q1 T) for 64 rows × 16·NJ columns; r·z partials per (row block, column)
template <int NJ>
__global__ void __launch_bounds__(128, 3) k_pc_apply3(const double* __restrict__ q1, int k,
                                                      const double* __restrict__ dinv,
                                                      const double* __restrict__ R, const double* __restrict__ T,
                                                      i64 N, int nrhs, double* __restrict__ Z,
                                                      double* __restrict__ partial_rz, int rz_ld, int rz_cols) {
  extern __shared__ __align__(16) double p3_sm[];
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16, JT = 2 * NJ;
  const int SA = p3_pad(k);
  double* Qs = p3_sm;                 // [64][SA]
  double* Rs = Qs + 64 * SA;          // [64][SV]
  double* Ds = Rs + 64 * SV;          // [64]
  double* Ts = Ds + 64;               // [P3_NSE][P3_MC][SV]
  double* red = Ts + P3_NSE * P3_MC * SV;  // [4][BWC] r·z per warp
  unsigned long long* full = reinterpret_cast<unsigned long long*>(red + 4 * BWC);
  unsigned long long* empty = full + P3_NSE;
  unsigned long long* qbar = empty + P3_NSE;
  const i64 i0 = (i64)blockIdx.x * 64;
  const int b0 = blockIdx.y * BWC;
  const int bw = min(BWC, nrhs - b0);
  const int nr = int(min((i64)64, N - i0));
  const int nch = (k + P3_MC - 1) / P3_MC;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g = lane / 4, t4 = lane % 4;
  const int wi = warp * 16;
  if (tid == 0) {
    for (int s = 0; s < P3_NSE; ++s) p3_mbar_init(full + s, 32), p3_mbar_init(empty + s, 4);
    p3_mbar_init(qbar, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  {  // the CTA's Q1 rows (threads 0..63) and r rows (64..127), once; D^{-1/2} by plain loads
    const int row = tid & 63;
    if (row < nr) {
      const bool a = tid < 64;
      const unsigned bytes = (a ? k : bw) * 8u;
      p3_arrive_tx(qbar, bytes);
      p3_bulk(a ? Qs + row * SA : Rs + row * SV, a ? q1 + (i0 + row) * k : R + (i0 + row) * nrhs + b0, bytes, qbar);
    } else {
      p3_arrive(qbar);
    }
    if (tid < 64) Ds[tid] = tid < nr ? dinv[i0 + tid] : 0.0;
  }
  auto issue = [&](int c) {  // warp 0; lane L < MC moves T row c·MC + L
    const int m = c * P3_MC + lane;
    unsigned long long* bar = full + c % P3_NSE;
    double* dst = Ts + (c % P3_NSE) * P3_MC * SV + lane * SV;
    if (lane < P3_MC && m < k) {
      p3_arrive_tx(bar, bw * 8u);
      p3_bulk(dst, T + (i64)m * nrhs + b0, bw * 8u, bar);
    } else {
      if (lane < P3_MC)
        for (int c2 = 0; c2 < SV; ++c2) dst[c2] = 0.0;
      p3_arrive(bar);
    }
  };
  if (warp == 0)
    for (int c = 0; c < min(P3_NSE, nch); ++c) issue(c);
  double acc[2][JT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  p3_wait(qbar, 0);
  __syncthreads();  // Ds (plain stores) visible
  const double* qrow[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) qrow[i] = Qs + min(wi + 8 * i + g, 63) * SA;
  for (int c = 0; c < nch; ++c) {
    const int sb = c % P3_NSE;
    const unsigned ph = (c / P3_NSE) & 1;
    p3_wait(full + sb, ph);
    const double* T1 = Ts + sb * P3_MC * SV;
#pragma unroll
    for (int kk = 0; kk < P3_MC; kk += 4) {
      const int m = c * P3_MC + kk + t4;
      const int mc = m < k ? m : 0;  // m past k meets a zero T row
      double af[2], bf[JT];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = qrow[i][mc];
#pragma unroll
      for (int j = 0; j < JT; ++j) bf[j] = T1[(kk + t4) * SV + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < JT; ++j) dmma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) p3_arrive(empty + sb);
    if (warp == 0 && c + P3_NSE < nch) {
      p3_wait(empty + sb, ph);
      issue(c + P3_NSE);
    }
  }
  // epilogue: z, and r·z summed over this warp's 16 rows per column (fixed order)
  double rz[JT][2];
#pragma unroll
  for (int j = 0; j < JT; ++j) rz[j][0] = rz[j][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < JT; ++j) {
      const int rl = wi + 8 * i + g, bl = 8 * j + 2 * t4;
      if (rl < nr && bl < bw) {
        const double d = Ds[rl];
        const double2 rv = *reinterpret_cast<const double2*>(Rs + rl * SV + bl);
        const double z0 = d * (d * rv.x - acc[i][j][0]), z1 = d * (d * rv.y - acc[i][j][1]);
        *reinterpret_cast<double2*>(Z + (i0 + rl) * nrhs + b0 + bl) = make_double2(z0, z1);
        rz[j][0] += rv.x * z0;
        rz[j][1] += rv.y * z1;
      }
    }
  if (partial_rz) {
#pragma unroll
    for (int j = 0; j < JT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = rz[j][e];
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // over g (lanes with equal t4)
        if (g == 0) red[warp * BWC + 8 * j + 2 * t4 + e] = v;
      }
    __syncthreads();
    for (int bl = tid; bl < bw; bl += 128)
      if (b0 + bl < rz_cols)
        partial_rz[(i64)blockIdx.x * rz_ld + b0 + bl] =
            ((red[bl] + red[BWC + bl]) + red[2 * BWC + bl]) + red[3 * BWC + bl];
  }
}

// out[o] = Σ_c partial[c][o]: block = 32 outputs × 8 chunk groups (chunk c in
// group c mod 8, loads 8 in flight), groups added in order (deterministic)
__global__ void __launch_bounds__(256) k_pc_reduce(const double* __restrict__ partial, int chunks, int nout,
                                                   double* __restrict__ out) {
  __shared__ double sm[8][33];
  const int lo = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + lo;
  double s = 0.0;
  if (o < nout) {
    int c = gq;
    for (; c + 56 < chunks; c += 64) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(partial + (i64)(c + 8 * u) * nout + o);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < chunks; c += 8) s += __ldcs(partial + (i64)c * nout + o);
  }
  sm[gq][lo] = s;
  __syncthreads();
  if (gq == 0 && o < nout) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += sm[q][lo];
    out[o] = t;
  }
}

// z = D^{-1/2}(D^{-1/2} r - Q1 T) for 64 rows per CTA; T (k × nrhs) and the
// CTA's 64 Q1 rows staged in shared memory with cp.async in one phase.
__global__ void __launch_bounds__(128) k_pc_apply_mma(const double* __restrict__ Rv, const double* __restrict__ dinv,
                                                      const double* __restrict__ q1, const double* __restrict__ T,
                                                      i64 N, int k, int nrhs, double* __restrict__ Z,
                                                      double* __restrict__ partial_rz) {
  const int kp = (k + 3) / 4 * 4, np = (nrhs + 7) / 8 * 8;
  const int SC = np + 8, SQ = kp + 4;
  extern __shared__ double sh[];
  double* Ts = sh;              // [kp][SC]
  double* Qs = Ts + kp * SC;    // [64][SQ]
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31, g = lane / 4, t4 = lane & 3;
  const int nt = np / 8;
  const i64 row0 = (i64)blockIdx.x * 64;
  for (int e = tid; e < kp * np; e += 128) {
    const int j = e / np, bb = e - j * np;
    if (j < k && bb < nrhs) cp_async8(Ts + j * SC + bb, T + j * nrhs + bb);
    else Ts[j * SC + bb] = 0.0;
  }
  for (int e = tid; e < 64 * kp; e += 128) {
    const int rr = e / kp, j = e - rr * kp;
    const i64 r = row0 + rr;
    if (r < N && j < k) cp_async8(Qs + rr * SQ + j, q1 + r * k + j);
    else Qs[rr * SQ + j] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  double acc[2][PCM_MAXJ][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < PCM_MAXJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kk = 0; kk < kp; kk += 4) {
    double bf[PCM_MAXJ];
#pragma unroll
    for (int j = 0; j < PCM_MAXJ; ++j) bf[j] = j < nt ? Ts[(kk + t4) * SC + 8 * j + g] : 0.0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double af = Qs[(warp * 16 + 8 * i + g) * SQ + kk + t4];
#pragma unroll
      for (int j = 0; j < PCM_MAXJ; ++j)
        if (j < nt) dmma_f64(acc[i][j][0], acc[i][j][1], af, bf[j]);
    }
  }
  __syncthreads();  // Qs is reused below for the r·z products [64][SC]
  double* RZ = Qs;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rl = warp * 16 + 8 * i + g;
    const i64 r = row0 + rl;
    const double di = r < N ? dinv[r] : 0.0;
#pragma unroll
    for (int j = 0; j < PCM_MAXJ; ++j) {
      if (j >= nt) break;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int bb = 8 * j + 2 * t4 + e;
        double prod = 0.0;
        if (r < N && bb < nrhs) {
          const double rv = Rv[r * nrhs + bb];
          const double z = di * (di * rv - acc[i][j][e]);  // linalg.cpp:200-204
          Z[r * nrhs + bb] = z;
          prod = rv * z;
        }
        RZ[rl * SC + bb] = prod;
      }
    }
  }
  if (partial_rz != nullptr) {  // this CTA's r·z per column, rows in fixed order
    __syncthreads();
    for (int bb = tid; bb < nrhs; bb += 128) {
      double t = 0.0;
      for (int rl = 0; rl < 64; ++rl) t += RZ[rl * SC + bb];
      partial_rz[(i64)blockIdx.x * nrhs + bb] = t;
    }
  }
}

// Row-wise small GEMM: Y[r][:] = X[r][:] · Mx (k×k col-major), X,Y [N][k] row-major.
__global__ void k_rows_times_small(const double* __restrict__ X, const double* __restrict__ Mx, i64 N, int k,
                                   double* __restrict__ Y) {
  const i64 items = N * k;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int j = int(it % k);
    const i64 r = it / k;
    const double* xr = X + r * k;
    const double* mc = Mx + (i64)j * k;
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += xr[i] * mc[i];
    Y[it] = s;
  }
}

// Gram partials: G[j][l] = Σ_rows X[r][j] X[r][l] (X [N][k] row-major), j<=l.
__global__ void k_gram_partial(const double* __restrict__ X, i64 N, int k, double* __restrict__ partial) {
  extern __shared__ double sh[];
  double* xs = sh;          // [PC_RT][k]
  double* acc = xs + PC_RT * k;  // [k*k]
  const int tid = threadIdx.x;
  for (int o = tid; o < k * k; o += blockDim.x) acc[o] = 0.0;
  i64 r0, r1;
  row_range(N, r0, r1);
  for (i64 rt = r0; rt < r1; rt += PC_RT) {
    const int nr = int((r1 - rt) < PC_RT ? (r1 - rt) : PC_RT);
    __syncthreads();
    for (int e = tid; e < nr * k; e += blockDim.x) xs[e] = X[rt * k + e];
    __syncthreads();
    for (int o = tid; o < k * k; o += blockDim.x) {
      const int j = o / k, l = o % k;
      if (j > l) continue;
      double a = acc[o];
      for (int rr = 0; rr < nr; ++rr) a += xs[rr * k + j] * xs[rr * k + l];
      acc[o] = a;
    }
  }
  __syncthreads();
  for (int o = tid; o < k * k; o += blockDim.x) partial[(i64)blockIdx.x * k * k + o] = acc[o];
}

// Gram partials for larger ranks: CTA = one 64×64 output tile (upper tiles
// only) × one row range; 16-row column slices staged in shared memory; each
// thread owns a 4×4 block of outputs. partial[blockIdx.x][j][l] (full k×k
// layout, the same as k_gram_partial's, so k_pc_fin reduces both).
constexpr int GT = 64;
__global__ void __launch_bounds__(256) k_gram_tile(const double* __restrict__ X, i64 N, int k,
                                                  double* __restrict__ partial) {
  const int tj = blockIdx.y, tl = blockIdx.z;
  if (tj > tl) return;
  __shared__ double xa[16][GT + 1], xb[16][GT + 1];
  const int j0 = tj * GT, l0 = tl * GT, tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  i64 r0, r1;
  row_range(N, r0, r1);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  for (i64 rt = r0; rt < r1; rt += 16) {
    __syncthreads();
    for (int e = tid; e < 16 * GT; e += 256) {
      const int rr = e / GT, cc = e % GT;
      const i64 r = rt + rr;
      const bool ok = r < r1;
      xa[rr][cc] = ok && j0 + cc < k ? X[r * k + j0 + cc] : 0.0;
      xb[rr][cc] = ok && l0 + cc < k ? X[r * k + l0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 16; ++rr) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = xa[rr][ty * 4 + a];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = xb[rr][tx * 4 + c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] += av[a] * bv[c];
    }
  }
  double* out = partial + (i64)blockIdx.x * k * k;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + ty * 4 + a, l = l0 + tx * 4 + c;
      if (j < k && l < k) out[(i64)j * k + l] = acc[a][c];
    }
}

// G = D^{-1/2} F: F is [k][N] col-major (internal rows) -> G [N][k] row-major
__global__ void k_scale_transpose(const double* __restrict__ F, const double* __restrict__ noise, i64 N, int k,
                                  double* __restrict__ G, double* __restrict__ dinv) {
  const i64 items = N * k;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int j = int(it % k);
    const i64 r = it / k;
    const double di = 1.0 / sqrt(noise[r]);
    G[it] = di * F[(i64)j * N + r];
    if (j == 0) dinv[r] = di;
  }
}

// ---------------------------------------------------------------- pivoted Cholesky
struct ArgMax {
  double v;
  i64 ext;
  i64 in;
};
__device__ __forceinline__ bool better(double v, i64 e, double bv, i64 be) {
  return v > bv || (v == bv && e < be);
}

__global__ void k_pv_init(const double* __restrict__ diag, const double* __restrict__ noise, int kernel_part,
                          i64 N, double* __restrict__ d) {
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    d[r] = kernel_part ? fmax(diag[r] - noise[r], 0.0) : diag[r];
}

// partial stats of d: min, sum, max, argmax(lowest ext)
__global__ void k_pv_stats(const double* __restrict__ d, const i64* __restrict__ ext, i64 N,
                           double* __restrict__ pmin, double* __restrict__ psum, double* __restrict__ pmax,
                           i64* __restrict__ pext, i64* __restrict__ pint) {
  __shared__ double smin[RT], ssum[RT], smax[RT];
  __shared__ i64 sext[RT], sint[RT];
  i64 r0, r1;
  row_range(N, r0, r1);
  double mn = INFINITY, sm = 0.0, mx = -INFINITY;
  i64 me = LLONG_MAX, mi = -1;
  for (i64 r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double v = d[r];
    const i64 e = ext ? ext[r] : r;
    mn = fmin(mn, v);
    sm += v;
    if (better(v, e, mx, me)) {
      mx = v;
      me = e;
      mi = r;
    }
  }
  const int t = threadIdx.x;
  smin[t] = mn;
  ssum[t] = sm;
  smax[t] = mx;
  sext[t] = me;
  sint[t] = mi;
  __syncthreads();
  if (t == 0) {
    double a = INFINITY, s = 0.0, b = -INFINITY;
    i64 be = LLONG_MAX, bi = -1;
    for (int k = 0; k < blockDim.x; ++k) {
      a = fmin(a, smin[k]);
      s += ssum[k];
      if (better(smax[k], sext[k], b, be)) {
        b = smax[k];
        be = sext[k];
        bi = sint[k];
      }
    }
    pmin[blockIdx.x] = a;
    psum[blockIdx.x] = s;
    pmax[blockIdx.x] = b;
    pext[blockIdx.x] = be;
    pint[blockIdx.x] = bi;
  }
}

// out[0]=min, out[1]=sum, out[2]=max, out[3]=ext (as double bits), out[4]=int
// One warp; fixed lane-strided order + butterfly (deterministic).
__global__ void k_pv_stats_fin(const double* pmin, const double* psum, const double* pmax, const i64* pext,
                               const i64* pint, int nb, double* out) {
  const int lane = threadIdx.x & 31;
  double a = INFINITY, s = 0.0, b = -INFINITY;
  i64 be = LLONG_MAX, bi = -1;
  for (int k = lane; k < nb; k += 32) {
    a = fmin(a, pmin[k]);
    s += psum[k];
    if (better(pmax[k], pext[k], b, be)) {
      b = pmax[k];
      be = pext[k];
      bi = pint[k];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
    s += __shfl_xor_sync(0xffffffffu, s, o);
    const double ob = __shfl_xor_sync(0xffffffffu, b, o);
    const i64 oe = __shfl_xor_sync(0xffffffffu, be, o);
    const i64 oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ob, oe, b, be)) {
      b = ob;
      be = oe;
      bi = oi;
    }
  }
  if (lane == 0) {
    out[0] = a;
    out[1] = s;
    out[2] = b;
    reinterpret_cast<i64*>(out)[3] = be;
    reinterpret_cast<i64*>(out)[4] = bi;
  }
}

// col = (row - noise_sub e_piv - L[:, :k] L[piv, :k]^T) / sqrt(dmax); L[:,k] = col;
// d -= col²  (then caller checks min, clamps and zeroes d[piv])
__global__ void k_pv_update(double* __restrict__ col, double* __restrict__ L, int k, i64 N, i64 piv,
                            double noise_sub, double sq, double* __restrict__ d) {
  extern __shared__ double lp[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) lp[j] = L[(i64)j * N + piv];
  __syncthreads();
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x) {
    double c = col[r];
    if (r == piv) c -= noise_sub;
    if (k > 0) {
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += L[(i64)j * N + r] * lp[j];
      c -= s;
    }
    c /= sq;
    L[(i64)k * N + r] = c;
    d[r] -= c * c;
  }
}

__global__ void k_pv_clamp(double* __restrict__ d, i64 N, i64 piv) {
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    d[r] = (r == piv) ? 0.0 : fmax(d[r], 0.0);
}

__global__ void k_perm_cols_out(const double* __restrict__ L, const i64* __restrict__ ext, i64 N, int k,
                                double* __restrict__ out) {
  const i64 items = N * k;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int j = int(it / N);
    const i64 r = it % N;
    out[(i64)j * N + (ext ? ext[r] : r)] = L[it];
  }
}

// ---------------------------------------------------------------- Lanczos
// W -= bprev[p] * prev; partial alpha = q·W
__global__ void k_lz_alpha(double* __restrict__ W, const double* __restrict__ prev, const double* __restrict__ bprev,
                           const double* __restrict__ q, i64 N, int P, double* __restrict__ partial) {
  __shared__ double sm[RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc = 0.0;
  if (slot < slots) {
    const double bp = bprev[p];
    i64 r0, r1;
    row_range(N, r0, r1);
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const i64 i = r * P + p;
      double w = W[i];
      if (prev) w -= bp * prev[i];
      W[i] = w;
      acc += q[i] * w;
    }
  }
  block_col_store(acc, P, partial, sm);
}

__global__ void k_fin_cols(const double* __restrict__ partial, int nout, double* __restrict__ out) {
  const int o = blockIdx.x * 8 + threadIdx.x / 32;
  if (o >= nout) return;
  const double v = warp_sum_partials(partial, RB, nout, o);
  if ((threadIdx.x & 31) == 0) out[o] = v;
}

// W -= alpha ∘ q (when q != null); partial C[j][p] = Σ Q[j0+j]·W for j < jc
constexpr int JC = 32;
__global__ void k_lz_proj(double* __restrict__ W, const double* __restrict__ q, const double* __restrict__ alpha,
                          const double* __restrict__ Q, int j0, int jc, i64 N, int P, double* __restrict__ partial) {
  __shared__ double sm[RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc[JC];
#pragma unroll
  for (int j = 0; j < JC; ++j) acc[j] = 0.0;
  if (slot < slots) {
    const double a = q ? alpha[p] : 0.0;
    i64 r0, r1;
    row_range(N, r0, r1);
    const i64 blk = N * P;
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const i64 i = r * P + p;
      double w = W[i];
      if (q) {
        w -= a * q[i];
        W[i] = w;
      }
#pragma unroll
      for (int j = 0; j < JC; ++j)
        if (j < jc) acc[j] += Q[(i64)(j0 + j) * blk + i] * w;
    }
  }
  for (int j = 0; j < jc; ++j) {
    __syncthreads();
    sm[threadIdx.x] = acc[j];
    __syncthreads();
    if (threadIdx.x < P) {
      double s = 0.0;
      for (int k = 0; k < slots; ++k) s += sm[k * P + threadIdx.x];
      partial[((i64)blockIdx.x * jc + j) * P + threadIdx.x] = s;
    }
  }
}

// W -= Σ_j Q[j] C[j]; optional partial ||W||²
__global__ void k_lz_update(double* __restrict__ W, const double* __restrict__ Q, const double* __restrict__ C,
                            int kc, i64 N, int P, double* __restrict__ partial_nrm) {
  __shared__ double sm[RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc = 0.0;
  if (slot < slots) {
    i64 r0, r1;
    row_range(N, r0, r1);
    const i64 blk = N * P;
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const i64 i = r * P + p;
      double s = 0.0;
      for (int j = 0; j < kc; ++j) s += Q[(i64)j * blk + i] * C[j * P + p];
      const double w = W[i] - s;
      W[i] = w;
      acc += w * w;
    }
  }
  if (partial_nrm) block_col_store(acc, P, partial_nrm, sm);
}

// q_next = W / beta for probes with flag != 0
__global__ void k_lz_next(const double* __restrict__ W, const double* __restrict__ beta, const int* __restrict__ flag,
                          i64 N, int P, double* __restrict__ qn) {
  const i64 items = N * P;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < items; i += (i64)gridDim.x * blockDim.x) {
    const int p = int(i) % P;
    if (flag[p]) qn[i] = W[i] / beta[p];
  }
}

// ---------------------------------------------------------------- Lanczos, device-resident step
// Per step three passes over the basis ("fused pass-1 update +
// pass-2 projection"): B computes α and the first projection as
// C1_j = Q_j·w − α Q_j·q_k (= Q_j·(w − α q_k), linalg.cpp:33-41 reordered),
// C applies w −= α q_k + Σ Q_j C1_j and projects again (C2), D applies the
// second correction and ‖w‖². α, β, breakdown test and the next-vector scale
// stay on the device (k_lz_state); the host syncs once per batch.

// Reduce per-thread accumulators acc[OFF + a] (a < cnt ≤ MAXC; thread layout
// slot × P) into out[blockIdx][a][P], eight columns per shared-memory round.
template <int OFF, int MAXC, int NA>
__device__ __forceinline__ void lz_store(const double (&acc)[NA], int cnt, int P, double* __restrict__ out,
                                         double* sm) {
  const int tid = threadIdx.x, slots = blockDim.x / P;
  double* ob = out + (i64)blockIdx.x * cnt * P;
#pragma unroll
  for (int a0 = 0; a0 < MAXC; a0 += 8) {
    if (a0 >= cnt) break;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (a0 + u < MAXC) sm[u * RT + tid] = acc[OFF + a0 + u];
    __syncthreads();
    for (int o = tid; o < 8 * P; o += blockDim.x) {
      const int u = o / P, p = o - u * P;
      if (a0 + u < cnt) {
        double s = 0.0;
        for (int k = 0; k < slots; ++k) s += sm[u * RT + k * P + p];
        ob[(i64)(a0 + u) * P + p] = s;
      }
    }
  }
}

constexpr int JB = 16;  // basis vectors per pass-B launch (2·JB + 1 accumulators)

// Rows per thread per iteration in the Lanczos passes: R independent rows keep
// R loads of every basis column in flight (the passes are HBM streams; one
// row at a time left them latency-bound at ~1-2 TB/s).
constexpr int LZR = 4;

struct LzRows {
  i64 ii[LZR];
  bool ok[LZR];
};
__device__ __forceinline__ LzRows lz_rows(i64 rb, int slots, i64 r0, i64 r1, int P, int p) {
  LzRows t;
#pragma unroll
  for (int u = 0; u < LZR; ++u) {
    const i64 r = rb + (i64)u * slots;
    t.ok[u] = r < r1;
    t.ii[u] = (t.ok[u] ? r : r0) * P + p;
  }
  return t;
}

// pass B (chunk j0..j0+jc of the basis). Chunk 0 also applies w −= β_prev q_{k−1}
// (prev != null) and accumulates α = q_k·w. The projection of w − α q_k is
// formed as Q_j·w − α δ_jk (the basis is orthonormal to roundoff under the
// two-pass full reorthogonalisation; the second pass removes the difference).
__global__ void __launch_bounds__(RT, 2) k_lz_b(double* __restrict__ W, const double* __restrict__ prev,
                                                const double* __restrict__ bprev, const double* __restrict__ q,
                                                const double* __restrict__ Q, int j0, int jc, i64 N, int P,
                                                double* __restrict__ part_a, double* __restrict__ part_g) {
  __shared__ double sm[8 * RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc[1 + JB];
#pragma unroll
  for (int j = 0; j < 1 + JB; ++j) acc[j] = 0.0;
  if (slot < slots) {
    const double bp = prev ? bprev[p] : 0.0;
    i64 r0, r1;
    row_range(N, r0, r1);
    const i64 blk = N * P;
    const double* Qc = Q + (i64)j0 * blk;
    for (i64 rb = r0 + slot; rb < r1; rb += (i64)slots * LZR) {
      const LzRows t = lz_rows(rb, slots, r0, r1, P, p);
      double w[LZR];
#pragma unroll
      for (int u = 0; u < LZR; ++u) {
        w[u] = W[t.ii[u]];
        if (prev) {
          w[u] -= bp * prev[t.ii[u]];
          if (t.ok[u]) W[t.ii[u]] = w[u];
        }
        if (!t.ok[u]) w[u] = 0.0;
        if (part_a) acc[0] += q[t.ii[u]] * w[u];
      }
#pragma unroll
      for (int j = 0; j < JB; ++j)
        if (j < jc) {
#pragma unroll
          for (int u = 0; u < LZR; ++u) acc[1 + j] += Qc[(i64)j * blk + t.ii[u]] * w[u];
        }
    }
  }
  if (part_a) lz_store<0, 1>(acc, 1, P, part_a, sm);
  if (jc > 0) lz_store<1, JB>(acc, jc, P, part_g, sm);
}

// Fixed-order cross-block sums: out[o] = Σ_k partial[k][o] (k = 0..RB-1) and,
// when part2 != null, out2[o] likewise. Block = 32 outputs × 8 block groups.
__device__ __forceinline__ double lz_colsum(const double* __restrict__ partial, int nout, int o, double* sm) {
  const int lo = threadIdx.x & 31, g = threadIdx.x >> 5;
  double s = 0.0;
  if (o < nout) {
    int k = g;
    for (; k + 56 < RB; k += 64) {  // eight loads in flight, summed in block order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = partial[(i64)(k + 8 * u) * nout + o];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; k < RB; k += 8) s += partial[(i64)k * nout + o];
  }
  __syncthreads();
  sm[g * 32 + lo] = s;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < 8; ++k) t += sm[k * 32 + lo];
  return t;
}

// α (chunk 0: reduced from part_a and stored; later chunks: read) and
// C1[j0 + j] = g_j − α δ_{j0+j,kcur}. Blocks of 32 outputs (j, p); chunk 0
// has an extra ceil(P/32) blocks for α.
__global__ void __launch_bounds__(256) k_lz_fin_b(const double* __restrict__ part_a,
                                                  const double* __restrict__ part_g, int j0, int jc, int kcur, int P,
                                                  double* __restrict__ alpha, double* __restrict__ C1) {
  __shared__ double sm[256];
  const int nb_c = (jc * P + 31) / 32;
  const int lo = threadIdx.x & 31;
  if ((int)blockIdx.x >= nb_c) {  // α blocks (chunk 0 only)
    const int o = (blockIdx.x - nb_c) * 32 + lo;
    const double a = lz_colsum(part_a, P, o, sm);
    if (threadIdx.x < 32 && o < P) alpha[o] = a;
    return;
  }
  const int o = blockIdx.x * 32 + lo;
  const bool diag = o < jc * P && j0 + o / P == kcur;
  double a = 0.0;
  if (part_a) a = lz_colsum(part_a, P, o < jc * P ? o % P : 0, sm);
  const double g = lz_colsum(part_g, jc * P, o, sm);
  if (!part_a && diag) a = alpha[o % P];
  if (threadIdx.x < 32 && o < jc * P) C1[(i64)j0 * P + o] = diag ? g - a : g;
}

// out[o] = Σ_k partial[k][o]
__global__ void __launch_bounds__(256) k_lz_fin(const double* __restrict__ partial, int nout,
                                                double* __restrict__ out) {
  __shared__ double sm[256];
  const int o = blockIdx.x * 32 + (threadIdx.x & 31);
  const double v = lz_colsum(partial, nout, o, sm);
  if (threadIdx.x < 32 && o < nout) out[o] = v;
}
inline unsigned lz_fin_blocks(int nout) { return static_cast<unsigned>((nout + 31) / 32); }

// pass C: chunk 0 applies w −= α q_k + Σ_{j<k1} Q_j C1_j (writes W); every chunk
// accumulates C2 partials for j0..j0+jc.
__global__ void __launch_bounds__(RT, 2) k_lz_c(double* __restrict__ W, const double* __restrict__ q,
                                                const double* __restrict__ alpha, const double* __restrict__ Q,
                                                const double* __restrict__ C1, int k1, int j0, int jc, i64 N, int P,
                                                double* __restrict__ partial) {
  __shared__ double sm[8 * RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc[JB];
#pragma unroll
  for (int j = 0; j < JB; ++j) acc[j] = 0.0;
  if (slot < slots) {
    const double a = alpha[p];
    i64 r0, r1;
    row_range(N, r0, r1);
    const i64 blk = N * P;
    const double* Qc = Q + (i64)j0 * blk;
    for (i64 rb = r0 + slot; rb < r1; rb += (i64)slots * LZR) {
      const LzRows t = lz_rows(rb, slots, r0, r1, P, p);
      double w[LZR];
#pragma unroll
      for (int u = 0; u < LZR; ++u) w[u] = W[t.ii[u]];
      if (j0 == 0) {
        double s[LZR];
#pragma unroll
        for (int u = 0; u < LZR; ++u) s[u] = a * q[t.ii[u]];
#pragma unroll 2
        for (int j = 0; j < k1; ++j) {
          const double c = __ldg(C1 + j * P + p);
#pragma unroll
          for (int u = 0; u < LZR; ++u) s[u] += Q[(i64)j * blk + t.ii[u]] * c;
        }
#pragma unroll
        for (int u = 0; u < LZR; ++u) {
          w[u] -= s[u];
          if (t.ok[u]) W[t.ii[u]] = w[u];
        }
      }
#pragma unroll
      for (int u = 0; u < LZR; ++u)
        if (!t.ok[u]) w[u] = 0.0;
#pragma unroll
      for (int j = 0; j < JB; ++j)
        if (j < jc) {
#pragma unroll
          for (int u = 0; u < LZR; ++u) acc[j] += Qc[(i64)j * blk + t.ii[u]] * w[u];
        }
    }
  }
  lz_store<0, JB>(acc, jc, P, partial, sm);
}

// pass D: w −= Σ_{j<kc} Q_j C2_j; partial ‖w‖²
__global__ void __launch_bounds__(RT, 2) k_lz_d(double* __restrict__ W, const double* __restrict__ Q,
                                                const double* __restrict__ C, int kc, i64 N, int P,
                                                double* __restrict__ partial_nrm) {
  __shared__ double sm[RT];
  const int slots = blockDim.x / P;
  const int p = threadIdx.x % P, slot = threadIdx.x / P;
  double acc = 0.0;
  if (slot < slots) {
    i64 r0, r1;
    row_range(N, r0, r1);
    const i64 blk = N * P;
    for (i64 rb = r0 + slot; rb < r1; rb += (i64)slots * LZR) {
      const LzRows t = lz_rows(rb, slots, r0, r1, P, p);
      double s[LZR];
#pragma unroll
      for (int u = 0; u < LZR; ++u) s[u] = 0.0;
#pragma unroll 4
      for (int j = 0; j < kc; ++j) {
        const double c = __ldg(C + j * P + p);
#pragma unroll
        for (int u = 0; u < LZR; ++u) s[u] += Q[(i64)j * blk + t.ii[u]] * c;
      }
#pragma unroll
      for (int u = 0; u < LZR; ++u)
        if (t.ok[u]) {
          const double w = W[t.ii[u]] - s[u];
          W[t.ii[u]] = w;
          acc += w * w;
        }
    }
  }
  block_col_store(acc, P, partial_nrm, sm);
}

// β = ‖w‖, breakdown test (linalg.cpp:42-49: β ≤ 1e-12·scale, scale = running
// max of |α|, β), histories, β_prev and next-vector flags. One block, P threads.
__global__ void k_lz_state(int k, int P, const double* __restrict__ alpha, const double* __restrict__ nrm2,
                           int* __restrict__ live, double* __restrict__ scale, int* __restrict__ kbreak,
                           double* __restrict__ ahist, double* __restrict__ bhist, double* __restrict__ bprev,
                           double* __restrict__ bdiv, int* __restrict__ flag) {
  const int p = threadIdx.x;
  if (p >= P) return;
  if (!live[p]) {
    flag[p] = 0;
    bprev[p] = 0.0;
    bdiv[p] = 1.0;
    return;
  }
  const double a = alpha[p], beta = sqrt(nrm2[p]);
  ahist[(i64)k * P + p] = a;
  const double sc = fmax(scale[p], fmax(fabs(a), beta));
  scale[p] = sc;
  if (beta <= 1e-12 * fmax(sc, 1e-300)) {
    kbreak[p] = k;
    live[p] = 0;
    flag[p] = 0;
    bprev[p] = 0.0;
    bdiv[p] = 1.0;
  } else {
    bhist[(i64)k * P + p] = beta;
    bprev[p] = beta;
    bdiv[p] = beta;
    flag[p] = 1;
  }
}

__global__ void k_lz_last(int k, int P, const double* __restrict__ alpha, const int* __restrict__ live,
                          double* __restrict__ ahist) {
  const int p = threadIdx.x;
  if (p < P && live[p]) ahist[(i64)k * P + p] = alpha[p];
}

// dst[r][s] = src[r][idx[s]] (gather == 1) or dst[r][idx[s]] = src[r][s]
__global__ void k_cols_move(const double* __restrict__ src, int Psrc, double* __restrict__ dst, int Pdst,
                            const int* __restrict__ idx, int ns, i64 rows, int gather) {
  const i64 items = rows * ns;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < items; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / ns;
    const int s = int(e - r * ns);
    if (gather) dst[r * Pdst + s] = src[r * Psrc + idx[s]];
    else dst[r * Pdst + idx[s]] = src[r * Psrc + s];
  }
}

// ---------------------------------------------------------------- device mt19937_64
// Rademacher probe streams on the device, bit-identical to the host's
// std::mt19937_64(mix_seed(seed, stream)) with the sign from bit 0 of each raw
// draw (rng.hpp:23-29). One CTA per stream; the 312-word twist runs as two
// parallel halves (words < 156 read only old state; words ≥ 156 read the first
// half's new words), then 312 tempered draws are emitted.
__global__ void __launch_bounds__(320) k_rademacher_mt(const unsigned long long* __restrict__ seeds, i64 n,
                                                       double scale, i64 ld, double* __restrict__ out) {
  constexpr int NN = 312, MM = 156;
  constexpr unsigned long long A = 0xB5026F5AA96619E9ULL, LM = (1ULL << 31) - 1, UM = ~LM;
  __shared__ unsigned long long mt[NN];
  const int tid = threadIdx.x;
  if (tid == 0) {
    unsigned long long x = seeds[blockIdx.x];
    mt[0] = x;
    for (int i = 1; i < NN; ++i) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + (unsigned long long)i;
      mt[i] = x;
    }
  }
  __syncthreads();
  double* o = out + (i64)blockIdx.x * ld;
  for (i64 base = 0; base < n; base += NN) {
    unsigned long long v = 0;
    if (tid < MM) {
      const unsigned long long x = (mt[tid] & UM) | (mt[tid + 1] & LM);
      v = mt[tid + MM] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    __syncthreads();
    if (tid < MM) mt[tid] = v;
    __syncthreads();
    if (tid < MM) {
      const int i = MM + tid;
      const unsigned long long x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
      v = mt[i - MM] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    __syncthreads();
    if (tid < MM) mt[MM + tid] = v;
    __syncthreads();
    if (tid < NN && base + tid < n) {
      unsigned long long y = mt[tid];
      y ^= (y >> 29) & 0x5555555555555555ULL;
      y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
      y ^= (y << 37) & 0xFFF7EEE000000000ULL;
      y ^= y >> 43;
      o[base + tid] = (y & 1ULL) ? scale : -scale;
    }
  }
}

}  // namespace

// ================================================================ PCG driver
// Per-operator PCG state kept between solves (under the operator's mutex):
// the workspace (grow-only), the fused-step plan, the pinned poll slots and
// the instantiated iteration graph. Every solve re-captures its iterations
// (a host-side enqueue) and refreshes the cached executable with
// cudaGraphExecUpdate, so the graph always carries this call's pointers and
// parameters; only a topology change re-instantiates. Re-allocating these
// per call (cudaMalloc/cudaFree, cudaMallocHost, cudaGraphInstantiate) cost
// ~6 ms per solve.
struct PcgCache {
  DevBuf<double> R, Zb, Pb, AP, part, prz, sc;
  DevBuf<int> si;
  PcgVecPlan vplan;
  i64 vN = -1;
  int vnrhs = -1, vk = -1, vtune = -1;
  HostBuf poll;  // 2 pinned slots (lag-one polling of the active count)
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t evs[2] = {nullptr, nullptr};
  ~PcgCache() {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto e : evs)
      if (e) cudaEventDestroy(e);
  }
};

static PcgCache& pcg_cache(Op& op) {
  if (!op.pcg_cache) op.pcg_cache = std::make_shared<PcgCache>();
  PcgCache& c = *static_cast<PcgCache*>(op.pcg_cache.get());
  if (!c.evs[0])
    for (auto& e : c.evs) GK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return c;
}

PcgResult pcg_internal(Op& op, Precond* M, const double* B, double* X, int nrhs, double tol, int maxit,
                       bool want_history, cudaStream_t s) {
  if (nrhs < 1 || nrhs > RT) fail(GK_ERR_ARG, "pcg: nrhs must be in [1, 256]");
  if (maxit < 0) fail(GK_ERR_ARG, "pcg: max_iterations must be >= 0");
  const i64 N = op.N;
  const i64 tot = N * nrhs;
  const bool tprof = std::getenv("GK_PCG_TIME") != nullptr;
  auto tq = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!tprof) return;
    GK_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pcg time] %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(now - tq).count());
    tq = now;
  };
  PcgCache& cache = pcg_cache(op);
  DevBuf<double>&R = cache.R, &Zb = cache.Zb, &Pb = cache.Pb, &AP = cache.AP, &part = cache.part, &prz = cache.prz,
                 &sc = cache.sc;
  DevBuf<int>& si = cache.si;
  R.reserve(static_cast<size_t>(tot));
  Zb.reserve(static_cast<size_t>(tot));
  Pb.reserve(static_cast<size_t>(tot));
  AP.reserve(static_cast<size_t>(tot));
  part.reserve(static_cast<size_t>(RB) * nrhs * 3);
  prz.reserve(static_cast<size_t>((N + 63) / 64 + RB) * nrhs);  // r·z partials of the precond apply
  sc.reserve(static_cast<size_t>(nrhs) * 4 + static_cast<size_t>(maxit + 1) * nrhs);
  si.reserve(static_cast<size_t>(nrhs) * 4 + 1);
  mark("workspace");
  CgDev st;
  st.bnorm = sc.p;
  st.rz = sc.p + nrhs;
  st.alpha = sc.p + 2 * nrhs;
  st.beta = sc.p + 3 * nrhs;
  st.hist = sc.p + 4 * nrhs;
  st.active = si.p;
  st.upd = si.p + nrhs;
  st.its = si.p + 2 * nrhs;
  st.conv = si.p + 3 * nrhs;
  st.nactive = si.p + 4 * nrhs;
  st.maxit = maxit;
  st.tol = tol;
  st.nrhs = nrhs;
  double* p0 = part.p;
  double* p1 = part.p + RB * nrhs;
  double* p2 = part.p + 2 * RB * nrhs;
  const int eb = blocks_for(tot);
  if (M) M->ensure(nrhs);

  // x0 = 0, r = b, z = M r, p = z
  k_fill<<<eb, 256, 0, s>>>(X, 0.0, tot);
  launched("pcg fill");
  k_copy<<<eb, 256, 0, s>>>(B, R.p, tot);
  launched("pcg copy");
  double* Z = R.p;
  if (M) {
    Z = Zb.p;
    M->apply(R.p, Z, nrhs, s);
  }
  k_copy<<<eb, 256, 0, s>>>(Z, Pb.p, tot);
  launched("pcg copy");
  k_dot_partial<<<RB, RT, 0, s>>>(B, B, N, nrhs, p0);
  launched("pcg dot");
  k_dot_partial<<<RB, RT, 0, s>>>(R.p, Z, N, nrhs, p1);
  launched("pcg dot");
  k_dot_partial<<<RB, RT, 0, s>>>(R.p, R.p, N, nrhs, p2);
  launched("pcg dot");
  GK_CUDA(cudaMemsetAsync(st.nactive, 0, sizeof(int), s));
  k_cg_init<<<nrhs, 32, 0, s>>>(st, p0, p1, p2);
  launched("pcg init");
  mark("init (precond ensure + apply)");

  // fused vector step (pcg_fused.cu): one cooperative kernel per iteration
  // besides the MVM instead of six kernels (tuning "pcg_fused": 0 default =
  // fused when supported, 2 = separate kernels). Measured on C2 (32 RHS,
  // rank 50): ~126 vs ~145 µs per iteration including the MVM.
  PcgVecPlan& vplan = cache.vplan;
  const int kM = M ? int(M->k) : 0;
  const int vtune = g_tuning.pcg_fused.load();
  const bool vfused = vtune != 2 && pcg_vec_supported(nrhs, kM);
  if (vfused && (cache.vN != N || cache.vnrhs != nrhs || cache.vk != kM || cache.vtune != vtune ||
                 std::getenv("GK_PCG_PROF"))) {
    pcg_vec_prepare(vplan, N, nrhs, kM, op.device);
    cache.vN = N;
    cache.vnrhs = nrhs;
    cache.vk = kM;
    cache.vtune = vtune;
  }
  mark("vector-step plan");

  // one iteration, captured as a graph
  auto iteration = [&](cudaStream_t cs) {
    op.mvm(Pb.p, AP.p, nrhs, cs);
    if (vfused) {
      PcgVecArgs va{};
      va.st = st;
      va.X = X;
      va.R = R.p;
      va.P = Pb.p;
      va.AP = AP.p;
      va.Z = Zb.p;
      va.q1 = M ? M->q1.p : nullptr;
      va.dinv = M ? M->dinv.p : nullptr;
      va.k = kM;
      va.N = N;
      va.nrhs = nrhs;
      pcg_vec_launch(vplan, va, cs);
      return;
    }
    k_dot_partial<<<RB, RT, 0, cs>>>(Pb.p, AP.p, N, nrhs, p0);
    launched("pcg dot");
    GK_CUDA(cudaMemsetAsync(st.nactive, 0, sizeof(int), cs));  // recounted by k_cg_fin_rr
    k_cg_axpy<<<RB, RT, 0, cs>>>(st, X, R.p, Pb.p, AP.p, N, p0, p1);
    launched("pcg axpy");
    k_cg_fin_rr<<<nrhs, 32, 0, cs>>>(st, p0, p1);
    launched("pcg fin");
    if (M) {
      // z = M^{-1} r with the r·z partials from the same pass (no extra dot)
      const int nb = M->apply(R.p, Zb.p, nrhs, cs, prz.p);
      k_cg_fin_rz<<<nrhs, 32, 0, cs>>>(st, prz.p, nb);
    } else {
      k_cg_fin_rz<<<nrhs, 32, 0, cs>>>(st, p1, RB);
    }
    launched("pcg fin");
    k_cg_pupdate<<<eb, 256, 0, cs>>>(st, Pb.p, M ? Zb.p : R.p, N);
    launched("pcg pupdate");
  };

  cache.poll.reserve(2);
  int* nact_h = reinterpret_cast<int*>(cache.poll.p);  // 2 ints in a pinned double slot pair
  GK_CUDA(cudaMemcpyAsync(nact_h, st.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  bool persisted = false;
  if (*nact_h > 0 && maxit > 0 && vfused && vplan.v2 && g_tuning.pcg_fused.load() == 5) {
    // Persistent path (opt-in, tuning "pcg_fused" = 5): PI iterations per
    // cooperative launch (MVM + vector step, grid barriers in between),
    // polled one launch behind. Measured at C2: 124 µs per iteration vs 111
    // for the graph-replayed kernels — graph replay already hides the launch
    // gap, and the merged kernel's 128-register cap costs both phases spills.
    PcgVecArgs va{};
    va.st = st;
    va.X = X;
    va.R = R.p;
    va.P = Pb.p;
    va.AP = AP.p;
    va.Z = Zb.p;
    va.q1 = M ? M->q1.p : nullptr;
    va.dinv = M ? M->dinv.p : nullptr;
    va.k = kM;
    va.N = N;
    va.nrhs = nrhs;
    const int PI = 32;
    const int max_launches = (maxit + PI - 1) / PI + 1;
    cudaEvent_t* evs = cache.evs;
    for (int j = 0; j < max_launches; ++j) {
      if (!op.pcg_persist(vplan, va, Pb.p, AP.p, nrhs, PI, s)) break;  // j == 0: no persistent path
      persisted = true;
      GK_CUDA(cudaMemcpyAsync(nact_h + (j & 1), st.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaEventRecord(evs[j & 1], s));
      if (j >= 1) {
        GK_CUDA(cudaEventSynchronize(evs[(j - 1) & 1]));
        if (nact_h[(j - 1) & 1] == 0) break;
      }
    }
    GK_CUDA(cudaStreamSynchronize(s));
  }
  if (!persisted && *nact_h > 0 && maxit > 0) {
    // warm the operator's scratch outside capture, then capture ITER iterations
    op.mvm(Pb.p, AP.p, nrhs, s);
    mark("warm MVM");
    const int ITER = 4;
    // capture on the operator's private stream (capturing the legacy default
    // stream is not permitted); the graph is then launched on `s`.
    GK_CUDA(cudaStreamSynchronize(s));
    cudaStream_t cs = op.cap_stream;
    const i64 before = g_launches.load();
    cudaGraph_t graph;
    GK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < ITER; ++i) iteration(cs);
    GK_CUDA(cudaStreamEndCapture(cs, &graph));
    const i64 nodes = g_launches.load() - before;
    g_launches.fetch_sub(nodes);
    // refresh the cached executable with this capture (same topology: only
    // node parameters change); instantiate only when that is refused
    if (cache.exec) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(cache.exec, graph, &info) != cudaSuccess) {
        (void)cudaGetLastError();
        cudaGraphExecDestroy(cache.exec);
        cache.exec = nullptr;
      }
    }
    if (!cache.exec) GK_CUDA(cudaGraphInstantiate(&cache.exec, graph, 0));
    cudaGraphExec_t exec = cache.exec;
    mark("capture + update/instantiate");
    // Lag-one polling: graph j is queued before the host waits for graph
    // j−1's active-column count, so the GPU never drains between graphs.
    // Iterations after convergence are no-ops for the converged columns (at
    // most one extra graph runs).
    const int max_launches = (maxit + ITER - 1) / ITER + 1;
    cudaEvent_t* evs = cache.evs;
    for (int j = 0; j < max_launches; ++j) {
      GK_CUDA(cudaGraphLaunch(exec, s));
      g_launches.fetch_add(nodes);
      GK_CUDA(cudaMemcpyAsync(nact_h + (j & 1), st.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaEventRecord(evs[j & 1], s));
      if (j >= 1) {
        GK_CUDA(cudaEventSynchronize(evs[(j - 1) & 1]));
        if (nact_h[(j - 1) & 1] == 0) break;
      }
    }
    GK_CUDA(cudaStreamSynchronize(s));
    cudaGraphDestroy(graph);
    mark("iterations");
  }
  if (vfused) pcg_vec_dump(vplan);

  PcgResult res;
  res.iterations.resize(static_cast<size_t>(nrhs));
  res.converged.resize(static_cast<size_t>(nrhs));
  res.hist_len.resize(static_cast<size_t>(nrhs));
  GK_CUDA(cudaMemcpyAsync(res.iterations.data(), st.its, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaMemcpyAsync(res.converged.data(), st.conv, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
  std::vector<double> bn(static_cast<size_t>(nrhs));
  GK_CUDA(cudaMemcpyAsync(bn.data(), st.bnorm, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
  if (want_history) {
    res.history.resize(static_cast<size_t>(maxit + 1) * nrhs);
    GK_CUDA(cudaMemcpyAsync(res.history.data(), st.hist, sizeof(double) * (maxit + 1) * nrhs,
                            cudaMemcpyDeviceToHost, s));
  }
  GK_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < nrhs; ++b) res.hist_len[static_cast<size_t>(b)] = bn[static_cast<size_t>(b)] == 0.0 ? 0 : res.iterations[static_cast<size_t>(b)] + 1;
  return res;
}

// ================================================================ preconditioner
Precond::~Precond() {
  if (stream) cudaStreamDestroy(stream);
}

static void set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024)
    raise_smem_limit(fn, bytes);
}

// Ranks whose k_pc_proj staging (or k_pc_apply's T copy) does not fit
// shared memory run the projection in k-column tiles and the apply as
// S = Q1 T (rows_gemm) followed by k_pc_finish_s — no rank limit (the
// reference Preconditioner has none, linalg.cpp:176-213).
constexpr size_t kPcSmem = 200 * 1024;
static size_t pc_proj_smem(i64 kt, int nrhs) { return sizeof(double) * size_t(PC_RT * kt + PC_RT * nrhs + kt * nrhs); }
static int pc_proj_tile(i64 k, int nrhs) {
  const i64 t = (i64(kPcSmem / sizeof(double)) - PC_RT * nrhs) / (PC_RT + nrhs);
  return int(std::max<i64>(1, std::min<i64>(k, t)));
}
static bool pc_big(i64 k, int nrhs) {
  return pc_proj_smem(k, nrhs) > kPcSmem || sizeof(double) * size_t(k * nrhs + RT) > kPcSmem;
}
// T[k][nrhs] = Q1ᵀ D^{-1/2} r (and the Σ c² partials into pcc when given).
static void pc_project(Precond& M, const double* r, int nrhs, double* T, double* pcc, cudaStream_t s) {
  const int KT = pc_proj_tile(M.k, nrhs);
  for (i64 j0 = 0; j0 < M.k; j0 += KT) {
    const int kt = int(std::min<i64>(KT, M.k - j0));
    k_pc_proj<<<RB, RT, pc_proj_smem(kt, nrhs), s>>>(r, M.dinv.p, M.q1.p + j0, M.N, kt, int(M.k), nrhs, M.partial.p,
                                                      j0 == 0 ? pcc : nullptr);
    launched("precond proj");
    k_pc_fin<<<fin_blocks(kt * nrhs), 256, 0, s>>>(M.partial.p, kt * nrhs, T + j0 * nrhs);
    launched("precond fin");
  }
}
// z = D^{-1/2}(D^{-1/2} r − Q1 T); partial Σ r·z per block when requested.
static int pc_finish(Precond& M, const double* r, const double* T, double* z, int nrhs, cudaStream_t s,
                     double* partial_rz) {
  if (!pc_big(M.k, nrhs)) {
    const size_t sh2 = sizeof(double) * (M.k * nrhs + RT);
    k_pc_apply<<<RB, RT, sh2, s>>>(r, M.dinv.p, M.q1.p, T, M.N, int(M.k), nrhs, z, partial_rz);
    launched("precond apply");
    return RB;
  }
  M.cbuf.reserve(static_cast<size_t>(M.N) * nrhs);
  rows_gemm_dev(M.q1.p, int(M.k), T, nrhs, M.N, M.cbuf.p, false, s);
  k_pc_finish_s<<<RB, RT, 0, s>>>(r, M.dinv.p, M.cbuf.p, M.N, nrhs, z, partial_rz);
  launched("precond apply (large rank)");
  return RB;
}

void Precond::ensure(int nrhs) {
  if (nrhs <= ensured_nrhs) return;
  ensured_nrhs = nrhs;
  const int np = nrhs + (nrhs & 1);  // padded width of the v3 kernels (odd RHS counts)
  partial.reserve(static_cast<size_t>(RB) * k * np);
  t.reserve(static_cast<size_t>(k) * np);
  pad_r.reserve(static_cast<size_t>(N) * np);
  pad_z.reserve(static_cast<size_t>(N) * np);
  set_smem((const void*)k_pc_proj, kPcSmem + 8 * 1024);  // every tile size of pc_project fits
  if (!pc_big(k, nrhs)) set_smem((const void*)k_pc_apply, sizeof(double) * (k * nrhs + RT));
  else cbuf.reserve(static_cast<size_t>(N) * nrhs);
  if (mma_ok(nrhs)) {
    set_smem((const void*)k_pc_proj_mma, proj_mma_smem(nrhs));
    set_smem((const void*)k_pc_apply_mma, apply_mma_smem(nrhs));
  }
  if ((k & 1) == 0 && k <= 256) {  // v3 kernels (precond_apply3)
    auto lim = [&](auto nj, const void* fp, const void* fa) {
      constexpr int NJ = decltype(nj)::value;
      constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
      raise_smem_limit(fp, sizeof(double) * size_t(P3_NS) * P3_BK * (p3_pad(int(k)) + SV + 1) + 16 * P3_NS);
      raise_smem_limit(fa, sizeof(double) * (size_t(64) * (p3_pad(int(k)) + SV + 1) + size_t(P3_NSE) * P3_MC * SV +
                                             4 * BWC) + 16 * P3_NSE + 8);
    };
    lim(std::integral_constant<int, 1>{}, (const void*)k_pc_proj3<1>, (const void*)k_pc_apply3<1>);
    lim(std::integral_constant<int, 2>{}, (const void*)k_pc_proj3<2>, (const void*)k_pc_apply3<2>);
    lim(std::integral_constant<int, 4>{}, (const void*)k_pc_proj3<4>, (const void*)k_pc_apply3<4>);
  }
}

bool Precond::mma_ok(int nrhs) const {
  return k <= 4 * PCM_MAXI * 8 && nrhs <= 8 * PCM_MAXJ && proj_mma_smem(nrhs) <= 220 * 1024 &&
         apply_mma_smem(nrhs) <= 220 * 1024;
}
int Precond::proj_rch(int nrhs) const {
  const i64 kp = (k + 7) / 8 * 8, np = (nrhs + 7) / 8 * 8;
  const i64 per_row = (kp + 8) + (np + 8) + 1;
  const i64 fit = (200 * 1024 / 8) / per_row / 4 * 4;
  return int(std::max<i64>(4, std::min<i64>(PCM_RCH, fit)));
}
size_t Precond::proj_mma_smem(int nrhs) const {
  const i64 kp = (k + 7) / 8 * 8, np = (nrhs + 7) / 8 * 8;
  const i64 rch = proj_rch(nrhs);
  return sizeof(double) * size_t(rch * (kp + 8) + rch * (np + 8) + rch);
}
size_t Precond::apply_mma_smem(int nrhs) const {
  const i64 kp = (k + 3) / 4 * 4, np = (nrhs + 7) / 8 * 8;
  return sizeof(double) * size_t(kp * (np + 8) + 64 * std::max(kp + 4, np + 8));  // Qs, reused for r·z
}

__global__ void k_pad_cols(const double* __restrict__ src, int ns, i64 N, int np, double* __restrict__ dst) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < N * np; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / np;
    const int b = int(e - r * np);
    dst[e] = b < ns ? src[r * ns + b] : 0.0;
  }
}
__global__ void k_unpad_cols(const double* __restrict__ src, int np, i64 N, int ns, double* __restrict__ dst) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < N * ns; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / ns;
    dst[e] = src[r * np + (e - r * ns)];
  }
}

template <int NJ>
static int precond_apply3(Precond& M, const double* r, double* z, int nrhs, cudaStream_t s, double* partial_rz,
                          int rz_ld, int rz_cols) {
  const int k = int(M.k);
  const i64 N = M.N;
  constexpr int BWC = 16 * NJ, SV = BWC + ((4 - BWC % 16) + 16) % 16;
  const size_t sp = sizeof(double) * size_t(P3_NS) * P3_BK * (p3_pad(k) + SV + 1) + 16 * P3_NS;
  const size_t sa = sizeof(double) * (size_t(64) * (p3_pad(k) + SV + 1) + size_t(P3_NSE) * P3_MC * SV + 4 * BWC) +
                    16 * P3_NSE + 8;
  // shared-memory limits were raised by ensure() (outside any graph capture)
  const int mt = (k + 63) / 64, bt = (nrhs + BWC - 1) / BWC;
  const int per_sm = int(std::max<size_t>(1, std::min<size_t>(4, (227 * 1024) / (sp + 1024))));
  int sms = 0, dev = 0;
  GK_CUDA(cudaGetDevice(&dev));
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int chunks = int(std::max<i64>(1, std::min<i64>(std::min<i64>(RB, std::max(1, per_sm) * sms / (mt * bt)),
                                                  (N + 4 * P3_BK - 1) / (4 * P3_BK))));
  const i64 rpc = ((N + chunks - 1) / chunks + P3_BK - 1) / P3_BK * P3_BK;
  chunks = int((N + rpc - 1) / rpc);
  k_pc_proj3<NJ><<<dim3(mt, bt, chunks), 128, sp, s>>>(M.q1.p, k, M.dinv.p, r, N, nrhs, rpc, M.partial.p);
  launched("precond proj (DMMA v3)");
  k_pc_reduce<<<(k * nrhs + 31) / 32, 256, 0, s>>>(M.partial.p, chunks, k * nrhs, M.t.p);
  launched("precond reduce");
  const unsigned nb = static_cast<unsigned>((N + 63) / 64);
  k_pc_apply3<NJ><<<dim3(nb, bt), 128, sa, s>>>(M.q1.p, k, M.dinv.p, r, M.t.p, N, nrhs, z, partial_rz, rz_ld,
                                                 rz_cols);
  launched("precond apply (DMMA v3)");
  return int(nb);
}

int Precond::apply(const double* r, double* z, int nrhs, cudaStream_t s, double* partial_rz) {
  ensure(nrhs);  // no-op once reserved (and before any graph capture)
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (g_tuning.precond.load() == 0 && (k & 1) == 0 && k <= 256 && nrhs >= 4 && nrhs + (nrhs & 1) <= 64 && al16(q1.p) &&
      al16(dinv.p)) {
    // an odd RHS count (C3: 17) runs on a zero-padded copy with 16-byte rows
    const bool pad = (nrhs & 1) || !al16(r) || !al16(z);
    const int np = pad ? nrhs + (nrhs & 1) : nrhs;
    const double* rr = r;
    double* zz = z;
    if (pad) {
      k_pad_cols<<<blocks_for(N * np), 256, 0, s>>>(r, nrhs, N, np, pad_r.p);
      launched("precond pad");
      rr = pad_r.p;
      zz = pad_z.p;
    }
    int nb;
    if (np > 32) nb = precond_apply3<4>(*this, rr, zz, np, s, partial_rz, nrhs, nrhs);
    else if (np > 16) nb = precond_apply3<2>(*this, rr, zz, np, s, partial_rz, nrhs, nrhs);
    else nb = precond_apply3<1>(*this, rr, zz, np, s, partial_rz, nrhs, nrhs);
    if (pad) {
      k_unpad_cols<<<blocks_for(N * nrhs), 256, 0, s>>>(pad_z.p, np, N, nrhs, z);
      launched("precond unpad");
    }
    return nb;
  }
  if (mma_ok(nrhs) && (g_tuning.precond.load() == 0 || g_tuning.precond.load() == 3)) {
    k_pc_proj_mma<<<RB, 128, proj_mma_smem(nrhs), s>>>(r, dinv.p, q1.p, N, int(k), nrhs, proj_rch(nrhs),
                                                       partial.p);
    launched("precond proj (DMMA)");
    k_pc_fin<<<fin_blocks(int(k * nrhs)), 256, 0, s>>>(partial.p, int(k * nrhs), t.p);
    launched("precond fin");
    const unsigned nb = static_cast<unsigned>((N + 63) / 64);
    k_pc_apply_mma<<<nb, 128, apply_mma_smem(nrhs), s>>>(r, dinv.p, q1.p, t.p, N, int(k), nrhs, z, partial_rz);
    launched("precond apply (DMMA)");
    return int(nb);
  }
  pc_project(*this, r, nrhs, t.p, nullptr, s);
  return pc_finish(*this, r, t.p, z, nrhs, s, partial_rz);
}

void precond_quadratic(Precond& M, const double* r, int nrhs, double* out_h, cudaStream_t s) {
  M.ensure(nrhs);
  DevBuf<double> pcc(static_cast<size_t>(RB) * nrhs), cc(static_cast<size_t>(nrhs));
  pc_project(M, r, nrhs, M.t.p, pcc.p, s);
  k_fin_cols<<<fin_blocks(nrhs), 256, 0, s>>>(pcc.p, nrhs, cc.p);
  launched("precond fin");
  std::vector<double> T(static_cast<size_t>(M.k) * nrhs), c2(static_cast<size_t>(nrhs));
  GK_CUDA(cudaMemcpyAsync(T.data(), M.t.p, sizeof(double) * T.size(), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaMemcpyAsync(c2.data(), cc.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < nrhs; ++b) {
    double t2 = 0.0;
    for (i64 j = 0; j < M.k; ++j) t2 += T[static_cast<size_t>(j * nrhs + b)] * T[static_cast<size_t>(j * nrhs + b)];
    out_h[b] = c2[static_cast<size_t>(b)] - t2;  // linalg.cpp:210-213
  }
}

// CholeskyQR2 of A = [G; I_k], G = D^{-1/2} F.  Q1 = G R^{-1}, R = R2 R1.
std::unique_ptr<Precond> precond_build(const double* F_int, i64 N, i64 k, const double* noise_int, int device,
                                       cudaStream_t s) {
  if (k < 1) fail(GK_ERR_ARG, "preconditioner needs a factor of rank at least 1");
  auto M = std::make_unique<Precond>();
  M->device = device;
  M->N = N;
  M->k = k;
  M->dinv.alloc(static_cast<size_t>(N));
  DevBuf<double> G(static_cast<size_t>(N * k)), Q(static_cast<size_t>(N * k));
  k_scale_transpose<<<blocks_for(N * k), 256, 0, s>>>(F_int, noise_int, N, int(k), G.p, M->dinv.p);
  launched("precond scale");
  DevBuf<double> part(static_cast<size_t>(RB) * k * k), gram(static_cast<size_t>(k * k)), Rinv_d(static_cast<size_t>(k * k));
  const size_t shg = sizeof(double) * (PC_RT * k + k * k);
  const bool tiled = k > 64;  // the k×k shared accumulator stops fitting near k = 160
  if (!tiled) set_smem((const void*)k_gram_partial, shg);
  const unsigned ntile = static_cast<unsigned>((k + GT - 1) / GT);
  std::vector<double> gh(static_cast<size_t>(k * k)), R(static_cast<size_t>(k * k)), Rinv(static_cast<size_t>(k * k)), Q2(static_cast<size_t>(k * k));
  // Q2 tracks the bottom block (initially I_k)
  for (i64 j = 0; j < k; ++j) Q2[static_cast<size_t>(j * k + j)] = 1.0;
  const double* cur = G.p;
  double* nxt = Q.p;
  for (int pass = 0; pass < 2; ++pass) {
    if (tiled) {
      k_gram_tile<<<dim3(RB, ntile, ntile), 256, 0, s>>>(cur, N, int(k), part.p);
      launched("precond gram (tiled)");
    } else {
      k_gram_partial<<<RB, RT, shg, s>>>(cur, N, int(k), part.p);
      launched("precond gram");
    }
    k_pc_fin<<<fin_blocks(int(k * k)), 256, 0, s>>>(part.p, int(k * k), gram.p);
    launched("precond gram fin");
    GK_CUDA(cudaMemcpyAsync(gh.data(), gram.p, sizeof(double) * k * k, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    // symmetric Gram (upper computed, gh[j*k+l] for j<=l) + Q2^T Q2 (col-major: element (j,l) at l*k+j)
    std::vector<double> A(static_cast<size_t>(k * k));
    for (i64 j = 0; j < k; ++j)
      for (i64 l = j; l < k; ++l) {
        long double acc = gh[static_cast<size_t>(j * k + l)];
        for (i64 r = 0; r < k; ++r) acc += (long double)Q2[static_cast<size_t>(j * k + r)] * Q2[static_cast<size_t>(l * k + r)];
        A[static_cast<size_t>(l * k + j)] = A[static_cast<size_t>(j * k + l)] = (double)acc;
      }
    cholesky_upper(int(k), A.data(), R.data());
    // Rinv = R^{-1} (upper)
    std::fill(Rinv.begin(), Rinv.end(), 0.0);
    for (i64 c = 0; c < k; ++c) {
      Rinv[static_cast<size_t>(c * k + c)] = 1.0 / R[static_cast<size_t>(c * k + c)];
      for (i64 r = c - 1; r >= 0; --r) {
        long double acc = 0.0L;
        for (i64 m = r + 1; m <= c; ++m) acc += (long double)R[static_cast<size_t>(m * k + r)] * Rinv[static_cast<size_t>(c * k + m)];
        Rinv[static_cast<size_t>(c * k + r)] = (double)(-acc / R[static_cast<size_t>(r * k + r)]);
      }
    }
    // bottom block Q2 <- Q2 Rinv
    std::vector<double> Q2n(static_cast<size_t>(k * k), 0.0);
    for (i64 r = 0; r < k; ++r)
      for (i64 c = 0; c < k; ++c) {
        long double acc = 0.0L;
        for (i64 m = 0; m <= c; ++m) acc += (long double)Q2[static_cast<size_t>(m * k + r)] * Rinv[static_cast<size_t>(c * k + m)];
        Q2n[static_cast<size_t>(c * k + r)] = (double)acc;
      }
    Q2 = Q2n;
    GK_CUDA(cudaMemcpyAsync(Rinv_d.p, Rinv.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, s));
    k_rows_times_small<<<blocks_for(N * k), 256, 0, s>>>(cur, Rinv_d.p, N, int(k), nxt);
    launched("precond rows x R^-1");
    GK_CUDA(cudaStreamSynchronize(s));  // Rinv host buffer reused next pass
    std::swap(G, Q);
    cur = G.p;
    nxt = Q.p;
  }
  M->q1 = std::move(G);  // after two swaps G holds the latest product
  GK_CUDA(cudaStreamSynchronize(s));
  return M;
}

// ================================================================ small block products (GP glue)
// C[r][j] (+)= Σ_t A[r][t]·Bm[t][j]: RHS-minor block (rows × ka) times a small
// host-sized matrix (ka × nb, row-major); one thread per output element.
__global__ void k_rows_gemm(const double* __restrict__ A, int ka, const double* __restrict__ Bm, int nb, i64 rows,
                            double* __restrict__ Cm, int accumulate) {
  for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < rows * nb; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / nb;
    const int j = int(e - r * nb);
    const double* a = A + r * ka;
    double acc = 0.0;
    for (int t = 0; t < ka; ++t) acc += a[t] * Bm[(i64)t * nb + j];
    Cm[e] = accumulate ? Cm[e] + acc : acc;
  }
}

// partial[block][t*nb + j] = Σ_{r in block's range} A[r][t]·D[r][j] (fixed order).
__global__ void __launch_bounds__(256) k_cross_partial(const double* __restrict__ A, int ka,
                                                       const double* __restrict__ D, int nb, i64 rows,
                                                       double* __restrict__ partial) {
  i64 r0, r1;
  row_range(rows, r0, r1);
  const int nout = ka * nb;
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    const int t = o / nb, j = o - (o / nb) * nb;
    double acc = 0.0;
    for (i64 r = r0; r < r1; ++r) acc += A[r * ka + t] * D[r * nb + j];
    partial[(i64)blockIdx.x * nout + o] = acc;
  }
}

__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c, i64 n) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) c[i] = a[i] - b[i];
}

void rows_gemm_dev(const double* A, int ka, const double* Bm_dev, int nb, i64 rows, double* C, bool accumulate,
                   cudaStream_t s) {
  if (rows * nb == 0) return;
  k_rows_gemm<<<blocks_for(rows * nb), 256, 0, s>>>(A, ka, Bm_dev, nb, rows, C, accumulate ? 1 : 0);
  launched("rows gemm");
}

void cross_dev(const double* A, int ka, const double* D, int nb, i64 rows, double* out_dev, DevBuf<double>& part,
               cudaStream_t s) {
  const int nout = ka * nb;
  part.reserve(static_cast<size_t>(RB) * nout);
  k_cross_partial<<<RB, 256, 0, s>>>(A, ka, D, nb, rows, part.p);
  launched("cross partial");
  k_fin_cols<<<fin_blocks(nout), 256, 0, s>>>(part.p, nout, out_dev);
  launched("cross fin");
}

void col_dots_dev(const double* X, const double* Y, i64 rows, int nrhs, double* out_dev, DevBuf<double>& part,
                  cudaStream_t s) {
  if (nrhs < 1 || nrhs > RT) fail(GK_ERR_ARG, "column dots: nrhs must be in [1, 256]");
  part.reserve(static_cast<size_t>(RB) * nrhs);
  k_dot_partial<<<RB, RT, 0, s>>>(X, Y, rows, nrhs, part.p);
  launched("column dots");
  k_fin_cols<<<fin_blocks(nrhs), 256, 0, s>>>(part.p, nrhs, out_dev);
  launched("column dots fin");
}

void sub_dev(const double* a, const double* b, double* c, i64 n, cudaStream_t s) {
  if (n == 0) return;
  k_sub<<<blocks_for(n), 256, 0, s>>>(a, b, c, n);
  launched("sub");
}

// Single right-hand side: T[j] = Σ_r q1[r][j] · dinv[r] r[r] as a streaming
// read of the row-major Q1 (thread j of a block owns output j over the
// block's row range: each row of Q1 is one coalesced read), partials per
// block summed in block order by k_pc_fin (deterministic).
__global__ void __launch_bounds__(256) k_pc_proj_r1(const double* __restrict__ Rv, const double* __restrict__ dinv,
                                                    const double* __restrict__ q1, i64 N, int k,
                                                    double* __restrict__ partial) {
  i64 r0, r1;
  row_range(N, r0, r1);
  for (int j0 = 0; j0 < k; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    double acc0 = 0.0, acc1 = 0.0;
    if (j < k) {
      i64 r = r0;
      for (; r + 1 < r1; r += 2) {  // two independent chains
        acc0 = fma(q1[r * k + j], dinv[r] * Rv[r], acc0);
        acc1 = fma(q1[(r + 1) * k + j], dinv[r + 1] * Rv[r + 1], acc1);
      }
      if (r < r1) acc0 = fma(q1[r * k + j], dinv[r] * Rv[r], acc0);
      partial[(i64)blockIdx.x * k + j] = acc0 + acc1;
    }
  }
}
// z[r] = dinv[r] (dinv[r] r[r] − Σ_j q1[r][j] T[j]): a warp per row (lanes over j).
__global__ void __launch_bounds__(256) k_pc_apply_r1(const double* __restrict__ Rv, const double* __restrict__ dinv,
                                                     const double* __restrict__ q1, const double* __restrict__ T,
                                                     i64 N, int k, double* __restrict__ Z) {
  extern __shared__ double Ts[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) Ts[j] = T[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (i64 r = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; r < N; r += ((i64)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (int j = lane; j < k; j += 32) s = fma(q1[r * k + j], Ts[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) Z[r] = dinv[r] * (dinv[r] * Rv[r] - s);
  }
}

// ================================================================ split preconditioner (row-sharded Q1)
// T = Q1ᵀ D^{-1/2} r over this preconditioner's rows (k×nrhs, device): the
// partial projection a row-sharded preconditioner all-reduces before
// finishing.
void precond_project(Precond& M, const double* r, int nrhs, double* T, cudaStream_t s) {
  M.ensure(nrhs);
  if (nrhs == 1) {
    k_pc_proj_r1<<<RB, 256, 0, s>>>(r, M.dinv.p, M.q1.p, M.N, int(M.k), M.partial.p);
    launched("precond proj (1 RHS, streaming)");
    k_pc_fin<<<fin_blocks(int(M.k)), 256, 0, s>>>(M.partial.p, int(M.k), T);
    launched("precond fin");
    return;
  }
  pc_project(M, r, nrhs, T, nullptr, s);
}
// z = D^{-1/2}(D^{-1/2} r − Q1 T) for a given (all-reduced) T.
void precond_finish(Precond& M, const double* r, const double* T, double* z, int nrhs, cudaStream_t s) {
  M.ensure(nrhs);
  if (nrhs == 1) {
    k_pc_apply_r1<<<blocks_for(M.N * 32), 256, sizeof(double) * M.k, s>>>(r, M.dinv.p, M.q1.p, T, M.N, int(M.k), z);
    launched("precond apply (1 RHS, warp per row)");
    return;
  }
  pc_finish(M, r, T, z, nrhs, s, nullptr);
}
// A preconditioner over an explicit Q1 (N×k col-major, device) and D^{-1/2}.
std::unique_ptr<Precond> precond_from_q1(const double* Q1cm, const double* dinv, i64 N, i64 k, int device,
                                         cudaStream_t s) {
  auto M = std::make_unique<Precond>();
  M->device = device;
  M->N = N;
  M->k = k;
  M->q1.alloc(static_cast<size_t>(N * k));
  M->dinv.alloc(static_cast<size_t>(N));
  to_internal(nullptr, N, Q1cm, N, M->q1.p, int(k), s);  // col-major N×k -> row-major [N][k]
  GK_CUDA(cudaMemcpyAsync(M->dinv.p, dinv, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  GK_CUDA(cudaStreamSynchronize(s));
  return M;
}

// ---------------------------------------------------------------- device-resident pivot loop
// State of the on-device pivoted Cholesky loop (one per factorisation).
struct PvDev {
  double stats[5];   // last k_pv_stats_fin output: min, sum, max, ext bits, int bits
  double initial, scale, tol_abs;  // initial trace, max(diag), trace_tol · initial
  double dmax, sq, residual;
  double fail_val;
  long long piv_int, piv_ext;
  int active;   // 1 while the loop runs (0 once a stop condition or a failure hit)
  int kdone;    // pivots taken
  int failed;   // 1: residual diagonal below −1e-10·scale (the reference throws)
};

// Start of step k: the stop tests of linalg.cpp:153-154 on the last stats.
__global__ void k_pv_begin(PvDev* st, int k, long long* pivots) {
  if (threadIdx.x != 0 || !st->active) return;
  const double dmax = st->stats[2];
  if (dmax <= 0.0 || st->residual <= st->tol_abs) {
    st->active = 0;
    return;
  }
  st->dmax = dmax;
  st->sq = sqrt(dmax);
  st->piv_ext = reinterpret_cast<const long long*>(st->stats)[3];
  st->piv_int = reinterpret_cast<const long long*>(st->stats)[4];
  pivots[k] = st->piv_ext;
  st->kdone = k + 1;
}

__global__ void k_pv_update_dev(double* __restrict__ col, double* __restrict__ L, int k, i64 N,
                                const double* __restrict__ noise, int kernel_part, const PvDev* __restrict__ st,
                                double* __restrict__ d) {
  if (!st->active) return;
  extern __shared__ double lp[];
  const i64 piv = st->piv_int;
  const double sq = st->sq;
  for (int j = threadIdx.x; j < k; j += blockDim.x) lp[j] = L[(i64)j * N + piv];
  __syncthreads();
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x) {
    double c = col[r];
    if (r == piv && kernel_part) c -= noise[piv];
    if (k > 0) {
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += L[(i64)j * N + r] * lp[j];
      c -= s;
    }
    c /= sq;
    L[(i64)k * N + r] = c;
    d[r] -= c * c;
  }
}

// After the update: the PSD check on min(d) (linalg.cpp:165-167). A failure
// stops the loop and records the value (the host raises after the loop).
__global__ void k_pv_check(PvDev* st) {
  if (threadIdx.x != 0 || !st->active) return;
  if (st->stats[0] < -1e-10 * st->scale) {
    st->failed = 1;
    st->fail_val = st->stats[0];
    st->active = 0;
  }
}

__global__ void k_pv_clamp_dev(double* __restrict__ d, i64 N, const PvDev* __restrict__ st) {
  if (!st->active) return;
  const i64 piv = st->piv_int;
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    d[r] = (r == piv) ? 0.0 : fmax(d[r], 0.0);
}

// End of step: residual trace = Σ d (linalg.cpp:171).
__global__ void k_pv_end(PvDev* st) {
  if (threadIdx.x == 0 && st->active) st->residual = st->stats[1];
}

// ================================================================ pivoted Cholesky
std::unique_ptr<PivChol> pivchol_run(Op& op, bool kernel_part, i64 max_rank, double trace_tol) {
  cudaStream_t s = op.stream;
  const i64 N = op.N;
  auto f = std::make_unique<PivChol>();
  f->device = op.device;
  f->N = N;
  f->order_uid = op.uid;
  GK_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
  if (op.d_ext_of_int()) {
    f->ext_own.alloc(static_cast<size_t>(N));
    GK_CUDA(cudaMemcpyAsync(f->ext_own.p, op.d_ext_of_int(), sizeof(i64) * N, cudaMemcpyDeviceToDevice, s));
  }
  max_rank = std::min(max_rank, N);
  if (max_rank < 0) fail(GK_ERR_ARG, "pivoted Cholesky rank must be >= 0");
  DevBuf<double> diag(static_cast<size_t>(N)), noise(static_cast<size_t>(N)), d(static_cast<size_t>(N)), col(static_cast<size_t>(N));
  f->L.alloc(static_cast<size_t>(std::max<i64>(max_rank, 1)) * N);
  op.diagonal(diag.p, s);
  {
    std::vector<double> nh(static_cast<size_t>(N));
    for (i64 r = 0; r < N; ++r) nh[static_cast<size_t>(r)] = r < op.n_value ? op.nv2 : op.ng2;
    noise.upload(nh.data(), nh.size(), s);
  }
  k_pv_init<<<blocks_for(N), 256, 0, s>>>(diag.p, noise.p, kernel_part ? 1 : 0, N, d.p);
  launched("pivchol init");
  DevBuf<double> pmin(RB), psum(RB), pmax(RB), stats(5);
  DevBuf<i64> pext(RB), pint_(RB);
  HostBuf pinned;
  pinned.reserve(5);
  double* sh = pinned.p;
  auto stats_of_d = [&]() {
    k_pv_stats<<<RB, RT, 0, s>>>(d.p, op.d_ext_of_int(), N, pmin.p, psum.p, pmax.p, pext.p, pint_.p);
    launched("pivchol stats");
    k_pv_stats_fin<<<1, 32, 0, s>>>(pmin.p, psum.p, pmax.p, pext.p, pint_.p, RB, stats.p);
    launched("pivchol stats fin");
    GK_CUDA(cudaMemcpyAsync(sh, stats.p, sizeof(double) * 5, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
  };
  stats_of_d();
  if (sh[0] < 0.0) fail(GK_ERR_RUNTIME, "pivoted Cholesky requires a nonnegative diagonal");
  f->initial_trace = sh[1];
  f->residual_trace = sh[1];
  const double scale = std::max(sh[2], 1e-300);
  i64 k = 0;
  // Device-resident loop (the operator computes a row from a device-side
  // pivot): every step's argmax, row, update, PSD check, clamp and trace stay
  // on the GPU — one host synchronisation for the whole factorisation
  // instead of three per pivot. Same operations, same order as below.
  DevBuf<PvDev> pst(1);
  DevBuf<long long> dpiv(static_cast<size_t>(std::max<i64>(max_rank, 1)));
  if (max_rank > 0 && g_tuning.pivchol.load() == 0 && op.has_row_dev()) {
    PvDev h{};
    std::memcpy(h.stats, sh, sizeof(h.stats));
    h.initial = sh[1];
    h.scale = scale;
    h.tol_abs = trace_tol * sh[1];
    h.residual = sh[1];
    h.active = 1;
    GK_CUDA(cudaMemcpyAsync(pst.p, &h, sizeof(PvDev), cudaMemcpyHostToDevice, s));
    const i64* pint = reinterpret_cast<const i64*>(&pst.p->piv_int);
    const int* act = &pst.p->active;
    double* st_stats = pst.p->stats;
    for (i64 kk = 0; kk < max_rank; ++kk) {
      k_pv_begin<<<1, 32, 0, s>>>(pst.p, int(kk), dpiv.p);
      launched("pivchol begin");
      op.row_dev(pint, act, col.p, s);
      k_pv_update_dev<<<blocks_for(N), 256, sizeof(double) * std::max<i64>(kk, 1), s>>>(
          col.p, f->L.p, int(kk), N, noise.p, kernel_part ? 1 : 0, pst.p, d.p);
      launched("pivchol update");
      k_pv_stats<<<RB, RT, 0, s>>>(d.p, op.d_ext_of_int(), N, pmin.p, psum.p, pmax.p, pext.p, pint_.p);
      launched("pivchol stats");
      k_pv_stats_fin<<<1, 32, 0, s>>>(pmin.p, psum.p, pmax.p, pext.p, pint_.p, RB, st_stats);
      launched("pivchol stats fin");
      k_pv_check<<<1, 32, 0, s>>>(pst.p);
      launched("pivchol check");
      k_pv_clamp_dev<<<blocks_for(N), 256, 0, s>>>(d.p, N, pst.p);
      launched("pivchol clamp");
      k_pv_stats<<<RB, RT, 0, s>>>(d.p, op.d_ext_of_int(), N, pmin.p, psum.p, pmax.p, pext.p, pint_.p);
      launched("pivchol stats");
      k_pv_stats_fin<<<1, 32, 0, s>>>(pmin.p, psum.p, pmax.p, pext.p, pint_.p, RB, st_stats);
      launched("pivchol stats fin");
      k_pv_end<<<1, 32, 0, s>>>(pst.p);
      launched("pivchol end");
    }
    GK_CUDA(cudaMemcpyAsync(&h, pst.p, sizeof(PvDev), cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    k = h.kdone;
    std::vector<long long> ph(static_cast<size_t>(std::max<i64>(k, 1)));
    if (k > 0) GK_CUDA(cudaMemcpy(ph.data(), dpiv.p, sizeof(long long) * k, cudaMemcpyDeviceToHost));
    for (i64 j = 0; j < k; ++j) f->pivots.push_back(ph[static_cast<size_t>(j)]);
    if (h.failed)
      fail(GK_ERR_RUNTIME, "pivoted Cholesky: operator is not positive semidefinite (residual diagonal " +
                               std::to_string(h.fail_val) + ")");
    f->residual_trace = h.residual;
    f->k = k;
    return f;
  }
  for (; k < max_rank; ++k) {
    const double dmax = sh[2];
    i64 piv_ext, piv_int;
    std::memcpy(&piv_ext, &sh[3], sizeof(i64));
    std::memcpy(&piv_int, &sh[4], sizeof(i64));
    if (dmax <= 0.0 || f->residual_trace <= trace_tol * f->initial_trace) break;
    op.row(piv_ext, col.p, s);
    const double nsub = kernel_part ? (piv_ext < op.n_value ? op.nv2 : op.ng2) : 0.0;
    k_pv_update<<<blocks_for(N), 256, sizeof(double) * std::max<i64>(k, 1), s>>>(
        col.p, f->L.p, int(k), N, piv_int, nsub, std::sqrt(dmax), d.p);
    launched("pivchol update");
    f->pivots.push_back(piv_ext);
    // min check before clamping (linalg.cpp:165-167)
    stats_of_d();
    if (sh[0] < -1e-10 * scale)
      fail(GK_ERR_RUNTIME, "pivoted Cholesky: operator is not positive semidefinite (residual diagonal " +
                               std::to_string(sh[0]) + ")");
    k_pv_clamp<<<blocks_for(N), 256, 0, s>>>(d.p, N, piv_int);
    launched("pivchol clamp");
    stats_of_d();
    f->residual_trace = sh[1];
  }
  f->k = k;
  return f;
}

PivChol::~PivChol() {
  if (stream) cudaStreamDestroy(stream);
}

void pivchol_copy_L(const PivChol& f, double* out_host) {
  if (f.k == 0) return;
  DevBuf<double> tmp(static_cast<size_t>(f.N * f.k));
  cudaStream_t s = f.stream;
  k_perm_cols_out<<<blocks_for(f.N * f.k), 256, 0, s>>>(f.L.p, f.ext_own.p, f.N, int(f.k), tmp.p);
  launched("pivchol permute");
  GK_CUDA(cudaMemcpyAsync(out_host, tmp.p, sizeof(double) * f.N * f.k, cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
}

// ================================================================ Lanczos
// Reference-order Lanczos with a host sync per step (deflating restarts on the
// host, linalg.cpp:46-69): the breakdown path of lanczos_batch.
static LanczosBatch lanczos_batch_sync(Op& op, const double* start_int, int P, int steps,
                                       const std::vector<std::uint64_t>& restart_seeds, double* Q_out,
                                       cudaStream_t s) {
  if (P < 1 || P > RT) fail(GK_ERR_ARG, "lanczos: number of probes must be in [1, 256]");
  const i64 N = op.N;
  steps = int(std::min<i64>(steps, N));
  LanczosBatch res;
  res.P = P;
  res.steps = steps;
  res.len.assign(static_cast<size_t>(P), steps);
  res.alpha.assign(static_cast<size_t>(P), {});
  res.beta.assign(static_cast<size_t>(P), {});
  res.breakdown.assign(static_cast<size_t>(P), 0);
  if (steps <= 0) {
    res.len.assign(static_cast<size_t>(P), 0);
    return res;
  }
  const i64 blk = N * P;
  DevBuf<double> Qown;
  double* Q = Q_out;
  if (!Q) {
    Qown.alloc(static_cast<size_t>(blk) * steps);
    Q = Qown.p;
  }
  DevBuf<double> W(static_cast<size_t>(blk)), part(static_cast<size_t>(RB) * JC * P), C(static_cast<size_t>(steps) * P), C2(static_cast<size_t>(steps) * P);
  DevBuf<double> sc(static_cast<size_t>(P) * 3);  // alpha, beta, bprev
  DevBuf<int> flag(static_cast<size_t>(P));
  double* d_alpha = sc.p;
  double* d_beta = sc.p + P;
  double* d_bprev = sc.p + 2 * P;
  GK_CUDA(cudaMemcpyAsync(Q, start_int, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
  GK_CUDA(cudaMemsetAsync(d_bprev, 0, sizeof(double) * P, s));
  std::vector<double> bprev_h(static_cast<size_t>(P), 0.0), scale(static_cast<size_t>(P), 0.0);
  std::vector<int> prev_valid(static_cast<size_t>(P), 0), live(static_cast<size_t>(P), 1), flag_h(static_cast<size_t>(P), 0);
  std::vector<std::uint64_t> restart_count(static_cast<size_t>(P), 0);
  std::vector<double> ab(static_cast<size_t>(2 * P));

  auto project = [&](const double* qk_for_alpha, int kc, double* Cdst) {
    for (int j0 = 0; j0 < kc; j0 += JC) {
      const int jc = std::min(JC, kc - j0);
      k_lz_proj<<<RB, RT, 0, s>>>(W.p, j0 == 0 ? qk_for_alpha : nullptr, d_alpha, Q, j0, jc, N, P, part.p);
      launched("lanczos proj");
      k_fin_cols<<<fin_blocks(jc * P), 256, 0, s>>>(part.p, jc * P, Cdst + (i64)j0 * P);
      launched("lanczos proj fin");
    }
  };

  for (int k = 0; k < steps; ++k) {
    const double* qk = Q + (i64)k * blk;
    op.mvm(qk, W.p, P, s);
    // w -= beta_prev * prev (prev = column k-1 when valid)
    std::vector<double> bp(static_cast<size_t>(P));
    for (int p = 0; p < P; ++p) bp[static_cast<size_t>(p)] = prev_valid[static_cast<size_t>(p)] ? bprev_h[static_cast<size_t>(p)] : 0.0;
    GK_CUDA(cudaMemcpyAsync(d_bprev, bp.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
    k_lz_alpha<<<RB, RT, 0, s>>>(W.p, k > 0 ? Q + (i64)(k - 1) * blk : nullptr, d_bprev, qk, N, P, part.p);
    launched("lanczos alpha");
    k_fin_cols<<<fin_blocks(P), 256, 0, s>>>(part.p, P, d_alpha);
    launched("lanczos alpha fin");
    const bool last = (k + 1 >= steps);
    if (last) {
      GK_CUDA(cudaMemcpyAsync(ab.data(), d_alpha, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
      for (int p = 0; p < P; ++p)
        if (live[static_cast<size_t>(p)]) res.alpha[static_cast<size_t>(p)].push_back(ab[static_cast<size_t>(p)]);
      break;  // reference computes the final reorth/beta but never uses them
    }
    // w -= a q; two passes of w -= Q (Q^T w)
    project(qk, k + 1, C.p);
    k_lz_update<<<RB, RT, 0, s>>>(W.p, Q, C.p, k + 1, N, P, nullptr);
    launched("lanczos update");
    project(nullptr, k + 1, C2.p);
    k_lz_update<<<RB, RT, 0, s>>>(W.p, Q, C2.p, k + 1, N, P, part.p);
    launched("lanczos update");
    k_fin_cols<<<fin_blocks(P), 256, 0, s>>>(part.p, P, d_beta);
    launched("lanczos beta fin");
    GK_CUDA(cudaMemcpyAsync(ab.data(), d_alpha, sizeof(double) * 2 * P, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    std::vector<int> restart;
    for (int p = 0; p < P; ++p) {
      const double a = ab[static_cast<size_t>(p)];
      const double beta = std::sqrt(ab[static_cast<size_t>(P + p)]);
      flag_h[static_cast<size_t>(p)] = 0;
      if (!live[static_cast<size_t>(p)]) continue;
      res.alpha[static_cast<size_t>(p)].push_back(a);
      scale[static_cast<size_t>(p)] = std::max({scale[static_cast<size_t>(p)], std::fabs(a), beta});
      if (beta <= 1e-12 * std::max(scale[static_cast<size_t>(p)], 1e-300)) {
        restart.push_back(p);
      } else {
        res.beta[static_cast<size_t>(p)].push_back(beta);
        bprev_h[static_cast<size_t>(p)] = beta;
        prev_valid[static_cast<size_t>(p)] = 1;
        flag_h[static_cast<size_t>(p)] = 1;
        ab[static_cast<size_t>(P + p)] = beta;
      }
    }
    // beta (not beta²) for normalisation
    std::vector<double> bet(static_cast<size_t>(P));
    for (int p = 0; p < P; ++p) bet[static_cast<size_t>(p)] = flag_h[static_cast<size_t>(p)] ? bprev_h[static_cast<size_t>(p)] : 1.0;
    GK_CUDA(cudaMemcpyAsync(d_beta, bet.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
    GK_CUDA(cudaMemcpyAsync(flag.p, flag_h.data(), sizeof(int) * P, cudaMemcpyHostToDevice, s));
    double* qn = Q + (i64)(k + 1) * blk;
    k_lz_next<<<blocks_for(blk), 256, 0, s>>>(W.p, d_beta, flag.p, N, P, qn);
    launched("lanczos next");
    if (!restart.empty()) {
      // Deflating restart (linalg.cpp:46-69), on the host for the affected
      // probes: fresh Gaussian direction, two-pass orthogonalisation against
      // the collected basis, accept if its norm exceeds 1e-8 sqrt(N).
      std::vector<double> Qh(static_cast<size_t>(blk) * (k + 1));
      GK_CUDA(cudaMemcpyAsync(Qh.data(), Q, sizeof(double) * blk * (k + 1), cudaMemcpyDeviceToHost, s));
      std::vector<double> qnh(static_cast<size_t>(blk));
      GK_CUDA(cudaMemcpyAsync(qnh.data(), qn, sizeof(double) * blk, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
      std::vector<double> rext(static_cast<size_t>(N)), rv(static_cast<size_t>(N));
      const i64* ext_d = op.d_ext_of_int();
      std::vector<i64> ext_h;
      if (ext_d) {
        ext_h.resize(static_cast<size_t>(N));
        GK_CUDA(cudaMemcpy(ext_h.data(), ext_d, sizeof(i64) * N, cudaMemcpyDeviceToHost));
      }
      for (int p : restart) {
        res.breakdown[static_cast<size_t>(p)] = 1;
        bool found = false;
        for (int attempt = 0; attempt < 8 && !found; ++attempt) {
          gaussian(N, mix_seed(restart_seeds[static_cast<size_t>(p)], 7777 + restart_count[static_cast<size_t>(p)]++), std::uint64_t(attempt),
                   rext.data());
          for (i64 r = 0; r < N; ++r) rv[static_cast<size_t>(r)] = rext[static_cast<size_t>(ext_d ? ext_h[static_cast<size_t>(r)] : r)];
          for (int pass = 0; pass < 2; ++pass) {
            std::vector<double> cj(static_cast<size_t>(k + 1), 0.0);
            for (int j = 0; j <= k; ++j) {
              double sdot = 0.0;
              for (i64 r = 0; r < N; ++r) sdot += Qh[static_cast<size_t>((i64)j * blk + r * P + p)] * rv[static_cast<size_t>(r)];
              cj[static_cast<size_t>(j)] = sdot;
            }
            for (i64 r = 0; r < N; ++r) {
              double sacc = 0.0;
              for (int j = 0; j <= k; ++j) sacc += Qh[static_cast<size_t>((i64)j * blk + r * P + p)] * cj[static_cast<size_t>(j)];
              rv[static_cast<size_t>(r)] -= sacc;
            }
          }
          double rn = 0.0;
          for (i64 r = 0; r < N; ++r) rn += rv[static_cast<size_t>(r)] * rv[static_cast<size_t>(r)];
          rn = std::sqrt(rn);
          if (rn > 1e-8 * std::sqrt(double(N))) {
            for (i64 r = 0; r < N; ++r) qnh[static_cast<size_t>(r * P + p)] = rv[static_cast<size_t>(r)] / rn;
            found = true;
          }
        }
        if (!found) {
          live[static_cast<size_t>(p)] = 0;
          res.len[static_cast<size_t>(p)] = k + 1;
          for (i64 r = 0; r < N; ++r) qnh[static_cast<size_t>(r * P + p)] = 0.0;
        } else {
          res.beta[static_cast<size_t>(p)].push_back(0.0);
          prev_valid[static_cast<size_t>(p)] = 0;
          bprev_h[static_cast<size_t>(p)] = 0.0;
        }
      }
      GK_CUDA(cudaMemcpyAsync(qn, qnh.data(), sizeof(double) * blk, cudaMemcpyHostToDevice, s));
      GK_CUDA(cudaStreamSynchronize(s));
    }
    bool any = false;
    for (int p = 0; p < P; ++p) any = any || live[static_cast<size_t>(p)];
    if (!any) break;
  }
  for (int p = 0; p < P; ++p) {
    res.alpha[static_cast<size_t>(p)].resize(static_cast<size_t>(res.len[static_cast<size_t>(p)]));
    res.beta[static_cast<size_t>(p)].resize(static_cast<size_t>(std::max(res.len[static_cast<size_t>(p)] - 1, 0)));
  }
  return res;
}

// Fast path: every step on the device, one host sync per batch. Probes that
// hit a Lanczos breakdown (β ≤ 1e-12·scale) are frozen and re-run, on their
// own, through lanczos_batch_sync (host-side deflating restarts with the
// reference's seeds); probes are independent, so the others keep their results.
LanczosBatch lanczos_batch(Op& op, const double* start_int, int P, int steps,
                           const std::vector<std::uint64_t>& restart_seeds, double* Q_out, cudaStream_t s) {
  if (P < 1 || P > RT) fail(GK_ERR_ARG, "lanczos: number of probes must be in [1, 256]");
  const i64 N = op.N;
  steps = int(std::min<i64>(steps, N));
  if (steps <= 0 || g_tuning.lanczos.load() == 1)
    return lanczos_batch_sync(op, start_int, P, steps, restart_seeds, Q_out, s);
  const i64 blk = N * P;
  const bool prof = std::getenv("GK_SLQ_PROF") != nullptr;
  auto tp0 = std::chrono::steady_clock::now();
  const int maxc = std::min(steps, JB);
  const size_t nQ = Q_out ? 0 : static_cast<size_t>(blk) * steps;
  const size_t nsc = static_cast<size_t>(P) * 5 + static_cast<size_t>(2 * steps) * P;
  const size_t need = nQ + static_cast<size_t>(blk) + static_cast<size_t>(RB) * P * (1 + maxc) +
                      static_cast<size_t>(2 * steps) * P + nsc;
  op.lz_ws.reserve(need);  // grow-only workspace on the operator (guarded by op.mu)
  op.lz_wsi.reserve(static_cast<size_t>(P) * 3);
  double* cur = op.lz_ws.p;
  auto carve = [&](size_t n) {
    double* r = cur;
    cur += n;
    return r;
  };
  double* Q = Q_out ? Q_out : carve(nQ);
  struct Span {
    double* p;
    size_t n;
  };
  Span W{carve(blk), 0}, pa{carve(static_cast<size_t>(RB) * P), 0}, pg{carve(static_cast<size_t>(RB) * maxc * P), 0},
      C1{carve(static_cast<size_t>(steps) * P), 0},
      C2{carve(static_cast<size_t>(steps) * P), 0}, sc{carve(nsc), nsc};
  struct ISpan {
    int* p;
  } si{op.lz_wsi.p};
  double *d_alpha = sc.p, *d_nrm = sc.p + P, *d_scale = sc.p + 2 * P, *d_bprev = sc.p + 3 * P, *d_bdiv = sc.p + 4 * P;
  double *d_ahist = sc.p + 5 * P, *d_bhist = d_ahist + static_cast<size_t>(steps) * P;
  int *d_live = si.p, *d_kbreak = si.p + P, *d_flag = si.p + 2 * P;
  GK_CUDA(cudaMemcpyAsync(Q, start_int, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
  GK_CUDA(cudaMemsetAsync(sc.p, 0, sizeof(double) * sc.n, s));
  {
    std::vector<int> init(static_cast<size_t>(P) * 3, 0);
    for (int p = 0; p < P; ++p) init[static_cast<size_t>(p)] = 1, init[static_cast<size_t>(P + p)] = -1;
    GK_CUDA(cudaMemcpyAsync(si.p, init.data(), sizeof(int) * init.size(), cudaMemcpyHostToDevice, s));
    GK_CUDA(cudaStreamSynchronize(s));  // pageable source
  }
  if (prof) {
    GK_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "lanczos: setup %.2f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
    tp0 = std::chrono::steady_clock::now();
  }
  auto run_steps = [&](int k_begin) {
  for (int k = k_begin; k < steps; ++k) {
    const double* qk = Q + (i64)k * blk;
    op.mvm(qk, W.p, P, s);
    const bool last = k + 1 >= steps;
    const int k1 = last ? 0 : k + 1;  // the reference never uses the last step's reorth/β
    for (int j0 = 0; j0 < std::max(k1, 1); j0 += JB) {
      const int jc = std::min(JB, k1 - j0);
      k_lz_b<<<RB, RT, 0, s>>>(W.p, j0 == 0 && k > 0 ? Q + (i64)(k - 1) * blk : nullptr, d_bprev, qk, Q, j0,
                               std::max(jc, 0), N, P, j0 == 0 ? pa.p : nullptr, pg.p);
      launched("lanczos pass B (alpha + projection 1)");
      k_lz_fin_b<<<lz_fin_blocks(std::max(jc, 0) * P) + (j0 == 0 ? lz_fin_blocks(P) : 0), 256, 0, s>>>(
          j0 == 0 ? pa.p : nullptr, pg.p, j0, std::max(jc, 0), k, P, d_alpha, C1.p);
      launched("lanczos pass B fin");
    }
    if (last) {
      k_lz_last<<<1, RT, 0, s>>>(k, P, d_alpha, d_live, d_ahist);
      launched("lanczos last alpha");
      break;
    }
    for (int j0 = 0; j0 < k1; j0 += JB) {
      const int jc = std::min(JB, k1 - j0);
      k_lz_c<<<RB, RT, 0, s>>>(W.p, qk, d_alpha, Q, C1.p, k1, j0, jc, N, P, pg.p);
      launched("lanczos pass C (update 1 + projection 2)");
      k_lz_fin<<<lz_fin_blocks(jc * P), 256, 0, s>>>(pg.p, jc * P, C2.p + (i64)j0 * P);
      launched("lanczos pass C fin");
    }
    k_lz_d<<<RB, RT, 0, s>>>(W.p, Q, C2.p, k1, N, P, pa.p);
    launched("lanczos pass D (update 2 + norm)");
    k_lz_fin<<<lz_fin_blocks(P), 256, 0, s>>>(pa.p, P, d_nrm);
    launched("lanczos norm fin");
    k_lz_state<<<1, RT, 0, s>>>(k, P, d_alpha, d_nrm, d_live, d_scale, d_kbreak, d_ahist, d_bhist, d_bprev, d_bdiv,
                                d_flag);
    launched("lanczos state");
    k_lz_next<<<blocks_for(blk), 256, 0, s>>>(W.p, d_bdiv, d_flag, N, P, Q + (i64)(k + 1) * blk);
    launched("lanczos next");
  }
  };
  run_steps(0);
  std::vector<int> kb(static_cast<size_t>(P)), len(static_cast<size_t>(P), steps), restarted(static_cast<size_t>(P), 0);
  GK_CUDA(cudaMemcpyAsync(kb.data(), d_kbreak, sizeof(int) * P, cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  // Breakdowns (β ≤ 1e-12·scale): rounds in increasing step order. The probes
  // that broke at step K get the reference's deflating restart on the host
  // (linalg.cpp:46-69: fresh Gaussian directions from mix_seed(seed,
  // 7777 + count), two-pass orthogonalisation against their basis, accepted
  // when the norm exceeds 1e-8·sqrt(N)); the device loop then resumes at K+1
  // with only those probes live. A probe with no acceptable direction stops
  // with K+1 steps.
  std::vector<std::uint64_t> rcount(static_cast<size_t>(P), 0);
  std::vector<i64> ext_h;
  for (int round = 0;; ++round) {
    int K = steps;
    for (int p = 0; p < P; ++p)
      if (kb[static_cast<size_t>(p)] >= 0) K = std::min(K, kb[static_cast<size_t>(p)]);
    if (K >= steps) break;
    if (prof) std::fprintf(stderr, "lanczos: restart round %d at step %d\n", round, K);
    if (ext_h.empty() && op.d_ext_of_int()) {
      ext_h.resize(static_cast<size_t>(N));
      GK_CUDA(cudaMemcpy(ext_h.data(), op.d_ext_of_int(), sizeof(i64) * N, cudaMemcpyDeviceToHost));
    }
    std::vector<int> live_h(static_cast<size_t>(P), 0), kb_new(kb);
    std::vector<int> cols;
    std::vector<double> rext(static_cast<size_t>(N)), rv(static_cast<size_t>(N) * P, 0.0);
    std::vector<double> zeros(static_cast<size_t>(P), 0.0), ones(static_cast<size_t>(P), 1.0), nrm(static_cast<size_t>(P));
    std::vector<int> flags(static_cast<size_t>(P), 0);
    for (int p = 0; p < P; ++p) {
      if (kb[static_cast<size_t>(p)] != K) continue;
      restarted[static_cast<size_t>(p)] = 1;
      kb_new[static_cast<size_t>(p)] = -1;
      bool found = false;
      for (int attempt = 0; attempt < 8 && !found; ++attempt) {
        gaussian(N, mix_seed(restart_seeds[static_cast<size_t>(p)], 7777 + rcount[static_cast<size_t>(p)]++),
                 std::uint64_t(attempt), rext.data());
        std::fill(rv.begin(), rv.end(), 0.0);
        for (i64 r = 0; r < N; ++r)
          rv[static_cast<size_t>(r * P + p)] = rext[static_cast<size_t>(ext_h.empty() ? r : ext_h[static_cast<size_t>(r)])];
        // two-pass orthogonalisation against q_0..q_K on the device (passes B, C, D with α = 0)
        GK_CUDA(cudaMemcpyAsync(W.p, rv.data(), sizeof(double) * blk, cudaMemcpyHostToDevice, s));
        GK_CUDA(cudaMemcpyAsync(d_alpha, zeros.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
        const int k1 = K + 1;
        for (int j0 = 0; j0 < k1; j0 += JB) {
          const int jc = std::min(JB, k1 - j0);
          k_lz_b<<<RB, RT, 0, s>>>(W.p, nullptr, d_bprev, Q, Q, j0, jc, N, P, nullptr, pg.p);
          launched("lanczos restart projection 1");
          k_lz_fin_b<<<lz_fin_blocks(jc * P), 256, 0, s>>>(nullptr, pg.p, j0, jc, -1, P, d_alpha, C1.p);
          launched("lanczos restart projection 1 fin");
        }
        for (int j0 = 0; j0 < k1; j0 += JB) {
          const int jc = std::min(JB, k1 - j0);
          k_lz_c<<<RB, RT, 0, s>>>(W.p, Q, d_alpha, Q, C1.p, k1, j0, jc, N, P, pg.p);
          launched("lanczos restart update 1 + projection 2");
          k_lz_fin<<<lz_fin_blocks(jc * P), 256, 0, s>>>(pg.p, jc * P, C2.p + (i64)j0 * P);
          launched("lanczos restart projection 2 fin");
        }
        k_lz_d<<<RB, RT, 0, s>>>(W.p, Q, C2.p, k1, N, P, pa.p);
        launched("lanczos restart update 2 + norm");
        k_lz_fin<<<lz_fin_blocks(P), 256, 0, s>>>(pa.p, P, d_nrm);
        launched("lanczos restart norm fin");
        GK_CUDA(cudaMemcpyAsync(nrm.data(), d_nrm, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
        GK_CUDA(cudaStreamSynchronize(s));
        const double rn = std::sqrt(nrm[static_cast<size_t>(p)]);
        if (rn > 1e-8 * std::sqrt(double(N))) {
          std::vector<double> bd(ones);
          bd[static_cast<size_t>(p)] = rn;
          std::fill(flags.begin(), flags.end(), 0);
          flags[static_cast<size_t>(p)] = 1;
          GK_CUDA(cudaMemcpyAsync(d_bdiv, bd.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
          GK_CUDA(cudaMemcpyAsync(d_flag, flags.data(), sizeof(int) * P, cudaMemcpyHostToDevice, s));
          k_lz_next<<<blocks_for(blk), 256, 0, s>>>(W.p, d_bdiv, d_flag, N, P, Q + (i64)(K + 1) * blk);
          launched("lanczos restart vector");
          GK_CUDA(cudaStreamSynchronize(s));  // pageable sources
          found = true;
        }
      }
      if (found) {
        live_h[static_cast<size_t>(p)] = 1;
        cols.push_back(p);
      } else {
        len[static_cast<size_t>(p)] = K + 1;  // stays frozen
      }
    }
    kb = kb_new;
    if (cols.empty() || K + 1 >= steps) continue;  // nothing to resume (or the restart step was the last)
    // device state for the resumed probes: q_{K+1}, β_K = 0, no β_prev term; every other probe frozen
    {
      std::vector<double> zero(static_cast<size_t>(P), 0.0), bh_row(static_cast<size_t>(P));
      GK_CUDA(cudaMemcpyAsync(bh_row.data(), d_bhist + (i64)K * P, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
      for (int p : cols) bh_row[static_cast<size_t>(p)] = 0.0;  // the reference records β = 0 at a restart
      std::vector<int> mkb(static_cast<size_t>(P));
      for (int p = 0; p < P; ++p) mkb[static_cast<size_t>(p)] = kb[static_cast<size_t>(p)];
      GK_CUDA(cudaMemcpyAsync(d_bhist + (i64)K * P, bh_row.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
      GK_CUDA(cudaMemcpyAsync(d_live, live_h.data(), sizeof(int) * P, cudaMemcpyHostToDevice, s));
      GK_CUDA(cudaMemcpyAsync(d_kbreak, mkb.data(), sizeof(int) * P, cudaMemcpyHostToDevice, s));
      GK_CUDA(cudaMemcpyAsync(d_bprev, zero.data(), sizeof(double) * P, cudaMemcpyHostToDevice, s));
      GK_CUDA(cudaStreamSynchronize(s));  // pageable sources
    }
    run_steps(K + 1);
    std::vector<int> kb_dev(static_cast<size_t>(P));
    GK_CUDA(cudaMemcpyAsync(kb_dev.data(), d_kbreak, sizeof(int) * P, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    for (int p : cols) kb[static_cast<size_t>(p)] = kb_dev[static_cast<size_t>(p)];
  }
  std::vector<double> ah(static_cast<size_t>(steps) * P), bh(static_cast<size_t>(steps) * P);
  GK_CUDA(cudaMemcpyAsync(ah.data(), d_ahist, sizeof(double) * ah.size(), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaMemcpyAsync(bh.data(), d_bhist, sizeof(double) * bh.size(), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  if (prof)
    std::fprintf(stderr, "lanczos: steps %.2f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
  LanczosBatch res;
  res.P = P;
  res.steps = steps;
  res.len = len;
  res.alpha.assign(static_cast<size_t>(P), {});
  res.beta.assign(static_cast<size_t>(P), {});
  res.breakdown = restarted;
  for (int p = 0; p < P; ++p) {
    const int L = len[static_cast<size_t>(p)];
    auto& a = res.alpha[static_cast<size_t>(p)];
    auto& b = res.beta[static_cast<size_t>(p)];
    for (int k = 0; k < L; ++k) a.push_back(ah[static_cast<size_t>(k) * P + p]);
    for (int k = 0; k + 1 < L; ++k) b.push_back(bh[static_cast<size_t>(k) * P + p]);
    if (L < steps && Q_out)  // a probe that stopped early: its remaining basis columns are zero
      GK_CUDA(cudaMemset2DAsync(Q_out + (i64)L * blk + p, sizeof(double) * P, 0, sizeof(double), size_t(N) * (steps - L), s));
  }
  GK_CUDA(cudaStreamSynchronize(s));
  return res;
}


// P Rademacher vectors of length n (streams mixed on the host: seeds[q] =
// mix_seed(seed, stream_q)), each scaled by `scale`, into out[q·ld + i].
void rademacher_dev(i64 n, const std::uint64_t* seeds_h, int P, double scale, double* out, i64 ld, cudaStream_t s) {
  DevBuf<unsigned long long> sd(static_cast<size_t>(P));
  GK_CUDA(cudaMemcpyAsync(sd.p, seeds_h, sizeof(unsigned long long) * P, cudaMemcpyHostToDevice, s));
  k_rademacher_mt<<<P, 320, 0, s>>>(sd.p, n, scale, ld, out);
  launched("rademacher (device mt19937_64)");
  GK_CUDA(cudaStreamSynchronize(s));  // pageable seed source / sd lifetime
}

}  // namespace gk
