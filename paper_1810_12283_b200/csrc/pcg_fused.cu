// pcg_fused.cu — everything of one PCG iteration except the operator MVM as
// ONE persistent cooperative kernel (reference cg, linalg.cpp:85-131, with the
// pivoted-Cholesky preconditioner apply of linalg.cpp:200-204), for nrhs
// independent columns:
//
//   A  pAp partials                         | barrier
//   B  alpha / stall / max-iteration logic  (every CTA, identical, no writes
//      but CTA 0's bookkeeping)
//   C  x += a p, r -= a Ap, ||r||² partials,
//      T partials = Q1ᵀ D^{-1/2} r           | barrier
//   D  convergence logic; T reduced, slice per CTA | barrier
//   E  z = D^{-1/2}(D^{-1/2} r - Q1 T), r·z partials | barrier
//   F  beta = rz_new / rz
//   G  p = z + beta p
//
// Rows are partitioned into one contiguous range per CTA. Every reduction is a
// fixed-order sum over the CTA partials (deterministic). Per-column state is
// read once at kernel entry (before the first barrier) and CTA 0 writes the
// updated state, so no CTA reads state another CTA is writing.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <mutex>

#include "gk_kernels.cuh"
#include "gk_sync.cuh"
#include "pcg_fused.hpp"
#include "pcg_vec2.cuh"

namespace gk {

namespace {

__global__ void __launch_bounds__(PV_THREADS, 2) k_pcg_vec(PcgVecArgs a) {
  extern __shared__ __align__(16) double pv_sm[];
  const int nrhs = a.nrhs, K = a.k, RCH = a.rch;
  double* red = pv_sm;                 // [256] block reduction scratch
  double* colv = red + PV_THREADS;     // [nrhs] reduced column values
  double* alpha = colv + nrhs;         // [nrhs]
  double* beta = alpha + nrhs;         // [nrhs]
  double* rz = beta + nrhs;            // [nrhs]
  double* bnorm = rz + nrhs;           // [nrhs]
  const int QS = pv_pad(K), RS = pv_pad(nrhs);  // conflict-free row strides
  auto al2 = [](double* p) {  // 16-byte alignment for the cp.async / bulk targets
    return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  };
  double* Ts = al2(bnorm + nrhs);          // [K][RS]
  double* Qs = al2(Ts + (size_t)K * RS);   // [RCH][QS] staged Q1 rows
  double* Rs = al2(Qs + (size_t)RCH * QS); // [RCH][RS] staged r rows
  double* Ds = al2(Rs + (size_t)RCH * RS); // [RCH] staged D^{-1/2}
  double* Ss = al2(Ds + RCH);              // [RCH][RS] Q1·T rows (phase E)
  int* upd = reinterpret_cast<int*>(Ss + (size_t)RCH * RS);  // [nrhs]
  int* act = upd + nrhs;                                       // [nrhs]
  int* its = act + nrhs;                                       // [nrhs]
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, g8 = lane / 4, t4 = lane % 4;
  const int b = tid % nrhs, slot = tid / nrhs, slots = PV_THREADS / nrhs;
  const int ntn = (nrhs + 7) / 8;  // n8 tiles over the right-hand sides
  const bool lane_ok = slot < slots;
  const i64 per = (a.N + gridDim.x - 1) / gridDim.x;
  const i64 r0 = min(a.N, (i64)blockIdx.x * per), r1 = min(a.N, r0 + per);
  PcgState& st = a.st;
  double* part0 = a.part;
  double* part1 = a.part + (size_t)gridDim.x * nrhs;
  double* part2 = a.part + 2 * (size_t)gridDim.x * nrhs;

  const bool prof_on = a.prof != nullptr && a.st.its[0] == 20;  // debug: one mid-solve launch
  pv_stamp(a, 0, prof_on);
  // tile -> (m0, n0) tables for the DMMA loops (no divisions inside them)
  __shared__ short tileM[8 * PV_ET], tileN[8 * PV_ET];
  for (int t = tid; t < 8 * PV_ET; t += PV_THREADS) {
    tileM[t] = short((t / ntn) * 8);
    tileN[t] = short((t % ntn) * 8);
  }
  // entry: column state (written only by CTA 0, after the first barrier)
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    act[c] = st.active[c];
    its[c] = st.its[c];
    rz[c] = st.rz[c];
    bnorm[c] = st.bnorm[c];
  }
  // A: pAp partials (PV_RB rows per thread per batch: loads in flight together)
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

  // B: alpha (linalg.cpp:110-118), identical in every CTA
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    int u = 0;
    double al = 0.0;
    int ac = act[c], it = its[c];
    if (ac) {
      if (it >= st.maxit) {
        ac = 0;  // loop bound reached, unconverged
      } else if (colv[c] <= 0.0) {
        ac = 0;  // loss of definiteness -> stalled (:114)
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
  __syncthreads();

  // C: x += a p, r -= a Ap on own rows; ||r||² partials
  acc = 0.0;
  if (lane_ok && upd[b]) {
    const double al = alpha[b];
    for (i64 rb = r0 + slot; rb < r1; rb += PV_RB * slots) {
      double xv[PV_RB], pv[PV_RB], rv[PV_RB], qv[PV_RB];
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        const i64 i = r * nrhs + b;
        const bool ok = r < r1;
        xv[q] = ok ? a.X[i] : 0.0;
        pv[q] = ok ? a.P[i] : 0.0;
        rv[q] = ok ? a.R[i] : 0.0;
        qv[q] = ok ? a.AP[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        if (r < r1) {
          const i64 i = r * nrhs + b;
          a.X[i] = xv[q] + al * pv[q];
          const double rn = rv[q] - al * qv[q];
          a.R[i] = rn;
          acc += rn * rn;
        }
      }
    }
  }
  block_cols(acc, nrhs, red, part1);
  pv_stamp(a, 2, prof_on);
  // T partial = Q1ᵀ D^{-1/2} r over own rows on the fp64 tensor cores (DMMA
  // m8n8k4): M = j (rank), N = b (RHS), K = rows; chunks of RCH rows staged
  // in shared memory; warp w owns tiles w, w+8, … (≤ PV_TT, fixed for the
  // whole row range so accumulators persist across chunks)
  if (a.q1 != nullptr) {
    const int ntt = ((K + 7) / 8) * ntn;
    double tacc[PV_TT][2];
#pragma unroll
    for (int q = 0; q < PV_TT; ++q) tacc[q][0] = tacc[q][1] = 0.0;
    for (i64 rs = r0; rs < r1; rs += RCH) {
      const int nr = int(min((i64)RCH, r1 - rs));
      __syncthreads();  // previous chunk consumed (and the r writes above visible)
      stage_rows(a, rs, nr, Qs, Rs, Ds);
      pv_stamp(a, rs == r0 ? 13 : 8, prof_on);
      for (int rr = warp; rr < nr; rr += PV_THREADS / 32)  // c = D^{-1/2} r
        for (int cc = lane; cc < nrhs; cc += 32) Rs[rr * RS + cc] *= Ds[rr];
      __syncthreads();
      // per-tile fragment columns hoisted out of the k loop (no divisions inside)
      int qa[PV_TT], qb[PV_TT];
#pragma unroll
      for (int q = 0; q < PV_TT; ++q) {
        const int tile = warp + 8 * q;
        const int m = tileM[tile] + g8, n = tileN[tile] + g8;
        qa[q] = (tile < ntt && m < K) ? m : -1;
        qb[q] = (tile < ntt && n < nrhs) ? n : -1;
      }
      for (int k0 = 0; k0 < nr; k0 += 4) {
        const int r = k0 + t4;
        const bool rok = r < nr;
#pragma unroll
        for (int q = 0; q < PV_TT; ++q) {
          if (warp + 8 * q < ntt) {
            const double av = (rok && qa[q] >= 0) ? Qs[r * QS + qa[q]] : 0.0;
            const double bv = (rok && qb[q] >= 0) ? Rs[r * RS + qb[q]] : 0.0;
            pv_dmma(tacc[q][0], tacc[q][1], av, bv);
          }
        }
      }
      if (rs == r0) {
        __syncthreads();
        pv_stamp(a, 14, prof_on);
      }
    }
    // partial layout [o][cta] (o = j*nrhs + b): the reduction reads each output's
    // CTA partials contiguously
#pragma unroll
    for (int q = 0; q < PV_TT; ++q) {
      const int tile = warp + 8 * q;
      if (tile < ntt) {
        const int m0 = tileM[tile], n0 = tileN[tile];
        const int j = m0 + g8;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = n0 + 2 * t4 + e;
          if (j < K && bb < nrhs) a.tpart[(i64)(j * nrhs + bb) * gridDim.x + blockIdx.x] = tacc[q][e];
        }
      }
    }
  }
  pv_stamp(a, 3, prof_on);
  grid_allreduce_cols(part1, nrhs, colv, a.bar);  // also a full barrier (tpart visible)
  pv_stamp(a, 10, prof_on);

  // D: convergence (:119-125), identical in every CTA; T reduced slice-wise
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
  if (a.q1 != nullptr) {
    const int nout = K * nrhs;
    for (int o = blockIdx.x * (PV_THREADS / 32) + tid / 32; o < nout; o += gridDim.x * (PV_THREADS / 32)) {
      const double v = warp_sum_cols(a.tpart + (i64)o * gridDim.x, gridDim.x, 1, 0);
      if ((tid & 31) == 0) a.T[o] = v;
    }
    pv_stamp(a, 4, prof_on);
    grid_sync(a.bar);
    pv_stamp(a, 9, prof_on);
    for (int j = warp; j < K; j += PV_THREADS / 32)
      for (int cc = lane; cc < nrhs; cc += 32) Ts[j * RS + cc] = __ldcg(a.T + j * nrhs + cc);
    __syncthreads();
  }

  // E: z = D^{-1/2}(D^{-1/2} r - Q1 T) on own rows (active columns); r·z
  // partials. S = Q1·T per chunk on DMMA (M = rows, N = b, K = j), then the
  // element-wise epilogue by (slot, b) threads in fixed row order.
  acc = 0.0;
  if (a.q1 != nullptr) {
    for (i64 rs = r0; rs < r1; rs += RCH) {
      const int nr = int(min((i64)RCH, r1 - rs));
      __syncthreads();
      stage_rows(a, rs, nr, Qs, Rs, Ds);
      pv_stamp(a, 11, prof_on);
      const int nte = ((nr + 7) / 8) * ntn;
      double sacc[PV_ET][2];
#pragma unroll
      for (int q = 0; q < PV_ET; ++q) sacc[q][0] = sacc[q][1] = 0.0;
      int ea[PV_ET], eb[PV_ET];  // fragment row (A) / column (B) per tile, hoisted
#pragma unroll
      for (int q = 0; q < PV_ET; ++q) {
        const int tile = warp + 8 * q;
        const int m = tileM[tile] + g8, n = tileN[tile] + g8;
        ea[q] = (tile < nte && m < nr) ? m * QS : -1;
        eb[q] = (tile < nte && n < nrhs) ? n : -1;
      }
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int j = k0 + t4;
        const bool jok = j < K;
#pragma unroll
        for (int q = 0; q < PV_ET; ++q) {
          if (warp + 8 * q < nte) {
            const double av = (jok && ea[q] >= 0) ? Qs[ea[q] + j] : 0.0;
            const double bv = (jok && eb[q] >= 0) ? Ts[j * RS + eb[q]] : 0.0;
            pv_dmma(sacc[q][0], sacc[q][1], av, bv);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < PV_ET; ++q) {
        const int tile = warp + 8 * q;
        if (tile < nte) {
          const int m0 = tileM[tile], n0 = tileN[tile];
          const int rr = m0 + g8;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int bb = n0 + 2 * t4 + e;
            if (rr < nr && bb < nrhs) Ss[rr * RS + bb] = sacc[q][e];
          }
        }
      }
      __syncthreads();
      if (lane_ok && act[b])
        for (int rr = slot; rr < nr; rr += slots) {
          const double di = Ds[rr], rv = Rs[rr * RS + b];
          const double z = di * (di * rv - Ss[rr * RS + b]);  // linalg.cpp:200-204
          a.Z[(rs + rr) * nrhs + b] = z;
          acc += rv * z;
        }
    }
  } else if (lane_ok && act[b]) {
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const double rv = a.R[r * nrhs + b];
      acc += rv * rv;
    }
  }
  block_cols(acc, nrhs, red, part2);
  pv_stamp(a, 5, prof_on);
  grid_allreduce_cols(part2, nrhs, colv, a.bar);
  pv_stamp(a, 12, prof_on);

  // F: beta = rz_new / rz (active columns)
  for (int c = tid; c < nrhs; c += PV_THREADS) {
    if (act[c]) {
      beta[c] = colv[c] / rz[c];
      if (blockIdx.x == 0) {
        st.beta[c] = beta[c];
        st.rz[c] = colv[c];
      }
    }
  }
  __syncthreads();

  // G: p = z + beta p
  if (lane_ok && act[b]) {
    const double be = beta[b];
    const double* Zs = a.q1 != nullptr ? a.Z : a.R;
    for (i64 rb = r0 + slot; rb < r1; rb += PV_RB * slots) {
      double zv[PV_RB], pv[PV_RB];
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        const i64 i = r * nrhs + b;
        zv[q] = r < r1 ? Zs[i] : 0.0;
        pv[q] = r < r1 ? a.P[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < PV_RB; ++q) {
        const i64 r = rb + q * slots;
        if (r < r1) a.P[r * nrhs + b] = zv[q] + be * pv[q];
      }
    }
  }
  __syncthreads();
  pv_stamp(a, 6, prof_on);
}

// v2 (rows resident): the body lives in pcg_vec2.cuh (also used by the
// persistent MVM + vector-step kernel in fused2d.cu).
__global__ void __launch_bounds__(PV_THREADS, 2) k_pcg_vec2(PcgVecArgs a) { (void)pcg_vec2_body(a); }

// ---------------------------------------------------------------- single RHS
// nrhs = 1 (C4: N = 450,000, rank 200): the Q1 products are GEMVs, so the
// DMMA tiles of v1/v2 would waste 7 of 8 columns and the row staging exposes
// its latency. Here a warp reads one Q1 row (K ≤ 256 doubles, coalesced) per
// step; T lives in the lanes' registers (lane l holds j = l, l+32, …); the
// apply reduces each row with shuffles. Same phases as v2: r·z = ‖c‖² − ‖T‖²,
// p updated directly, three grid barriers; Q1 is streamed twice (the bound).
constexpr int R1_KQ = 8;  // K ≤ 32·R1_KQ
__global__ void __launch_bounds__(PV_THREADS, 2) k_pcg_vec_r1(PcgVecArgs a) {
  __shared__ double red[PV_THREADS];
  __shared__ double colv[2];
  __shared__ double tred[PV_THREADS / 32][32 * R1_KQ];
  __shared__ int sh_flags[3];  // act, upd, its
  __shared__ double sh_vals[4];  // alpha, beta, rz, bnorm
  const int K = a.q1 != nullptr ? a.k : 0;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const i64 per = (a.N + gridDim.x - 1) / gridDim.x;
  const i64 r0 = min(a.N, (i64)blockIdx.x * per), r1 = min(a.N, r0 + per);
  PcgState& st = a.st;
  double* part0 = a.part;
  double* part1 = a.part + gridDim.x;  // [cta][2]
  if (tid == 0) {
    sh_flags[0] = st.active[0];
    sh_flags[2] = st.its[0];
    sh_vals[2] = st.rz[0];
    sh_vals[3] = st.bnorm[0];
  }
  // A: pAp partials
  double acc = 0.0;
  for (i64 r = r0 + tid; r < r1; r += PV_THREADS) acc += a.P[r] * a.AP[r];
  block_cols(acc, 1, red, part0);
  grid_allreduce_cols(part0, 1, colv, a.bar);
  // B: alpha
  if (tid == 0) {
    int u = 0, ac = sh_flags[0], it = sh_flags[2];
    double al = 0.0;
    if (ac) {
      if (it >= st.maxit || colv[0] <= 0.0) {
        ac = 0;
      } else {
        al = sh_vals[2] / colv[0];
        u = 1;
        it += 1;
      }
    }
    sh_flags[0] = ac;
    sh_flags[1] = u;
    sh_flags[2] = it;
    sh_vals[0] = al;
    if (blockIdx.x == 0) {
      st.active[0] = ac;
      st.its[0] = it;
      st.upd[0] = u;
      st.alpha[0] = al;
    }
  }
  __syncthreads();
  const bool u = sh_flags[1] != 0;
  const double al = sh_vals[0];
  // C: x, r update; ||r||², ||c||² partials (c = D^{-1/2} r)
  double arr = 0.0, acc_c = 0.0;
  for (i64 r = r0 + tid; r < r1; r += PV_THREADS) {
    double rn = a.R[r];
    if (u) {
      a.X[r] += al * a.P[r];
      rn -= al * a.AP[r];
      a.R[r] = rn;
      arr += rn * rn;
    }
    const double c = K > 0 ? a.dinv[r] * rn : rn;
    acc_c += c * c;
  }
  __syncthreads();  // R rows of this CTA written before the T pass reads them
  // T partial = Q1ᵀ c: warp per row, lanes over j
  double tq[R1_KQ];
#pragma unroll
  for (int q = 0; q < R1_KQ; ++q) tq[q] = 0.0;
  if (K > 0) {
    constexpr int RR = 4;  // rows per warp step: their loads are in flight together
    for (i64 rb = r0 + warp; rb < r1; rb += RR * (PV_THREADS / 32)) {
      double qv[RR][R1_KQ], cv[RR];
#pragma unroll
      for (int u = 0; u < RR; ++u) {
        const i64 r = rb + u * (PV_THREADS / 32);
        const bool ok = r < r1;
        cv[u] = ok ? a.dinv[r] * a.R[r] : 0.0;
        const double* qr = a.q1 + (ok ? r : r0) * K;
#pragma unroll
        for (int q = 0; q < R1_KQ; ++q) {
          const int j = lane + 32 * q;
          qv[u][q] = j < K ? __ldcs(qr + j) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < RR; ++u)
#pragma unroll
        for (int q = 0; q < R1_KQ; ++q) tq[q] += qv[u][q] * cv[u];
    }
#pragma unroll
    for (int q = 0; q < R1_KQ; ++q) tred[warp][lane + 32 * q] = tq[q];
  }
  __syncthreads();
  if (K > 0)
    for (int j = tid; j < K; j += PV_THREADS) {
      double s = 0.0;
      for (int w = 0; w < PV_THREADS / 32; ++w) s += tred[w][j];
      a.tpart[(i64)j * gridDim.x + blockIdx.x] = s;
    }
  // rr | cc partials
  __syncthreads();
  red[tid] = arr;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int k = 0; k < PV_THREADS; ++k) s += red[k];
    part1[(i64)blockIdx.x * 2] = s;
  }
  __syncthreads();
  red[tid] = acc_c;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int k = 0; k < PV_THREADS; ++k) s += red[k];
    part1[(i64)blockIdx.x * 2 + 1] = s;
  }
  grid_allreduce_cols(part1, 2, colv, a.bar);  // also a full barrier (tpart visible)
  // D: convergence
  if (tid == 0 && sh_flags[1]) {
    const double relres = sqrt(colv[0]) / sh_vals[3];
    const bool done = relres <= st.tol;
    if (done) sh_flags[0] = 0;
    if (blockIdx.x == 0) {
      st.hist[(i64)sh_flags[2]] = relres;
      if (done) {
        st.conv[0] = 1;
        st.active[0] = 0;
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) *st.nactive = sh_flags[0];
  if (K > 0) {
    for (int o = blockIdx.x * (PV_THREADS / 32) + warp; o < K; o += gridDim.x * (PV_THREADS / 32)) {
      const double v = warp_sum_cols(a.tpart + (i64)o * gridDim.x, gridDim.x, 1, 0);
      if (lane == 0) a.T[o] = v;
    }
    grid_sync(a.bar);
#pragma unroll
    for (int q = 0; q < R1_KQ; ++q) {
      const int j = lane + 32 * q;
      tq[q] = j < K ? __ldcg(a.T + j) : 0.0;
    }
  }
  // F: rz_new = ||c||² − ||T||², beta
  if (tid == 0 && sh_flags[0]) {
    double t2 = 0.0;
    for (int j = 0; j < K; ++j) {
      const double t = __ldcg(a.T + j);
      t2 += t * t;
    }
    const double rzn = colv[1] - t2;
    sh_vals[1] = rzn / sh_vals[2];
    if (blockIdx.x == 0) {
      st.beta[0] = sh_vals[1];
      st.rz[0] = rzn;
    }
  }
  __syncthreads();
  if (!sh_flags[0]) return;
  const double be = sh_vals[1];
  // EG: p = D^{-1/2}(c − Q1 T) + beta p, warp per row
  if (K > 0) {
    constexpr int RR = 4;
    for (i64 rb = r0 + warp; rb < r1; rb += RR * (PV_THREADS / 32)) {
      double sv[RR];
#pragma unroll
      for (int u = 0; u < RR; ++u) {
        const i64 r = rb + u * (PV_THREADS / 32);
        const double* qr = a.q1 + (r < r1 ? r : r0) * K;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < R1_KQ; ++q) {
          const int j = lane + 32 * q;
          if (j < K) s += __ldcs(qr + j) * tq[q];
        }
        sv[u] = s;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < RR; ++u) sv[u] += __shfl_xor_sync(0xffffffffu, sv[u], o);
      if (lane < RR) {
        double s = sv[0];
#pragma unroll
        for (int u = 1; u < RR; ++u)
          if (lane == u) s = sv[u];
        const i64 r = rb + lane * (PV_THREADS / 32);
        if (r < r1) {
          const double di = a.dinv[r];
          const double z = di * (di * a.R[r] - s);
          a.P[r] = z + be * a.P[r];
        }
      }
    }
  } else {
    for (i64 r = r0 + tid; r < r1; r += PV_THREADS) a.P[r] = a.R[r] + be * a.P[r];
  }
}

}  // namespace

bool pcg_vec_supported(int nrhs, int k) {
  const int ntn = (nrhs + 7) / 8;
  return nrhs >= 1 && nrhs <= 64 && (PV_THREADS % nrhs) == 0 && i64(k) * nrhs <= 8192 &&
         ((k + 7) / 8) * ntn <= 8 * PV_TT;
}

static void pcg_vec_prepare_impl(PcgVecPlan& p, i64 N, int nrhs, int k, int device, bool allow_v2);
void pcg_vec_prepare(PcgVecPlan& p, i64 N, int nrhs, int k, int device) {
  pcg_vec_prepare_impl(p, N, nrhs, k, device, true);
}
static void pcg_vec_prepare_impl(PcgVecPlan& p, i64 N, int nrhs, int k, int device, bool allow_v2) {
  int sms = 0;
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const i64 rows_per_cta = (N + 2 * sms - 1) / (2 * sms);
  p.rch = k > 0 ? int(std::max<i64>(8, std::min<i64>(rows_per_cta, 10240 / (pv_pad(k) + 2 * pv_pad(nrhs) + 1)))) : 1;
  // phase E tiles per warp: ceil(rch/8)·ceil(nrhs/8) ≤ 8·PV_ET
  const int ntn = (nrhs + 7) / 8;
  while (p.rch > 8 && ((p.rch + 7) / 8) * ntn > 8 * PV_ET) p.rch -= 8;
  // row chunk staged for the rank-k contractions: ~40 KB of shared memory
  // row chunk staged for the rank-k contractions: the CTA's whole row range
  // when it fits ~80 KB of shared memory (one staging latency per pass)
  (void)0;
  p.smem = sizeof(double) * (PV_THREADS + 5 * nrhs + size_t(k) * pv_pad(nrhs) +
                             size_t(p.rch) * (pv_pad(k) + 2 * pv_pad(nrhs)) + size_t(p.rch) + 8) +
           sizeof(int) * 4 * nrhs + 64;
  // v2 (rows resident) when the CTA's whole row range fits beside a second CTA
  {
    const int K4 = (k + 3) & ~3;
    const int rmax = int(((rows_per_cta + 7) / 8) * 8);
    const size_t smem2 = sizeof(double) * (PV_THREADS + 6 * nrhs + size_t(K4) * pv_pad(nrhs) +
                                           size_t(rmax) * (pv_pad(std::max(K4, 1)) + pv_pad(nrhs) + 1) + 8) +
                         sizeof(int) * 3 * nrhs + 64;
    const bool tiles_ok = (rmax / 8) * ntn <= 8 * PV_ET;
    p.v2 = allow_v2 && g_tuning.pcg_fused.load() != 3 && tiles_ok && smem2 <= 110 * 1024;
    if (p.v2) {
      p.rch = rmax;
      p.smem = smem2;
    }
  }
  // single right-hand side: streamed GEMVs (k_pcg_vec_r1) instead of DMMA tiles
  p.r1 = nrhs == 1 && k <= 32 * R1_KQ && g_tuning.pcg_fused.load() != 3;
  if (p.r1) {
    p.v2 = false;
    p.smem = 0;
  }
  raise_smem_limit(p.r1 ? (const void*)k_pcg_vec_r1 : p.v2 ? (const void*)k_pcg_vec2 : (const void*)k_pcg_vec, p.smem);
  if (p.v2)
    GK_CUDA(cudaFuncSetAttribute((const void*)k_pcg_vec2, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 int(cudaSharedmemCarveoutMaxShared)));
  GK_CUDA(cudaFuncSetAttribute((const void*)k_pcg_vec, cudaFuncAttributePreferredSharedMemoryCarveout,
                               int(cudaSharedmemCarveoutMaxShared)));
  int occ = 0;
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p.r1 ? k_pcg_vec_r1 : p.v2 ? k_pcg_vec2 : k_pcg_vec,
                                                        PV_THREADS, p.smem));
  if (occ < 1) fail(GK_ERR_RUNTIME, "fused PCG step does not fit on an SM");
  if (p.r1 && occ < 2) p.r1 = false;
  if (p.v2 && occ < 2) {  // v2's row ranges were sized for two CTAs per SM
    return pcg_vec_prepare_impl(p, N, nrhs, k, device, false);
  }
  p.grid = std::min(occ, 2) * sms;
  p.part.alloc(size_t(3) * p.grid * nrhs);
  p.tpart.alloc(size_t(p.grid) * (k + 2) * nrhs);  // + ‖r‖², ‖c‖² rows (v2)
  p.T.alloc(size_t(k + 2) * nrhs);
  p.bar.alloc(kBarSlots);
  GK_CUDA(cudaMemset(p.bar.p, 0, sizeof(unsigned long long) * kBarSlots));
  p.red_out.alloc(size_t(3) * nrhs);
  p.rctr.alloc(2);
  GK_CUDA(cudaMemset(p.rctr.p, 0, 2 * sizeof(unsigned long long)));
  if (std::getenv("GK_PCG_PROF")) {
    std::fprintf(stderr, "[pcg_vec] %s grid %d (occ %d) smem %zu rch %d k %d nrhs %d\n", p.r1 ? "r1" : p.v2 ? "v2" : "v1", p.grid,
                 occ, p.smem, p.rch, k, nrhs);
    p.prof.alloc(size_t(p.grid) * 16);
    GK_CUDA(cudaMemset(p.prof.p, 0, sizeof(unsigned long long) * p.prof.n));
  }
}

void pcg_vec_launch(PcgVecPlan& p, PcgVecArgs a, cudaStream_t s) {
  a.rch = p.rch;
  a.prof = p.prof.p;  // allocated by pcg_vec_prepare under GK_PCG_PROF
  a.part = p.part.p;
  a.red_out = p.red_out.p;
  a.rctr = p.rctr.p;
  a.tpart = p.tpart.p;
  a.T = p.T.p;
  a.bar = p.bar.p;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.grid));
  cfg.blockDim = dim3(PV_THREADS);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.r1) GK_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_vec_r1, a));
  else if (p.v2) GK_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_vec2, a));
  else GK_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_vec, a));
  launched("pcg fused vector step");
}

void pcg_vec_dump(PcgVecPlan& p) {
  if (!p.prof.p) return;
  std::vector<unsigned long long> h(size_t(p.grid) * 16);
  GK_CUDA(cudaDeviceSynchronize());
  GK_CUDA(cudaMemcpy(h.data(), p.prof.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  double mx[16] = {0};
  for (int c = 0; c < p.grid; ++c) t0 = std::min(t0, h[size_t(c) * 16]);
  for (int c = 0; c < p.grid; ++c)
    for (int k = 1; k < 16; ++k)
      if (h[size_t(c) * 16 + k] >= t0 && h[size_t(c) * 16 + k] - t0 < 1000000000ull)
        mx[k] = std::max(mx[k], double(h[size_t(c) * 16 + k] - t0) / 1e3);
  std::fprintf(stderr, "[pcg_vec] cumulative max over CTAs (us):");
  for (int k = 1; k < 16; ++k)
    if (mx[k] > 0) std::fprintf(stderr, " s%d=%.2f", k, mx[k]);
  std::fprintf(stderr, "\n");
}

}  // namespace gk
