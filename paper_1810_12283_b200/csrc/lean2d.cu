// lean2d.cu — the D-SKI MVM for 2-D grids with gradients as ONE persistent
// cooperative kernel with lean phases (reference DskiOperator::mvm,
// dski.cpp:228-238: stacked_transpose_apply → grid_operator().apply →
// stacked_apply + noise_diagonal).
//
//   phase S  u  = Bᵀ v        segment-parity scatter (no atomics, no smem)
//   phase T1 y1 = (I ⊗ T_1) u  Toeplitz mode product along axis 1 (DMMA)
//   phase T0 w  = (T_0 ⊗ I) y1 Toeplitz mode product along axis 0 (DMMA)
//   phase G  out = B w + Σ v   gather + noise
//
// Design (B200): every phase is a flat list of independent per-thread or
// per-warp jobs with all operands read straight from L1/L2 — no shared-memory
// staging rings, no per-row block barriers — so the only synchronisation is
// the three grid barriers between phases. The inputs (point records, v) are
// bulk-prefetched into L2 by TMA at kernel start, so the scatter's first
// touches hit L2 instead of HBM.
//
// Scatter: thread (cell-row segment s of L = T-1 rows, node column j, RHS
// group) walks its segment's cell rows in order keeping T register
// accumulators (rolling window). A segment's node rows [sL, sL+L+T-1) go to
// buffer U[s & 1]: with L >= T-1 two segments of the same parity never
// overlap, so every node row is the fixed-order sum of at most two buffer
// entries (its own segment, then the previous one), formed when phase T1
// loads it — deterministic, no atomics.
//
// Toeplitz phases: K_UU = T_0 ⊗ T_1 (the operator the reference applies by
// circulant-embedding FFT, dski.cpp:146-166). Warp job = (8-column n-tile, a
// run of m-tiles); DMMA m8n8k4 (fp64 tensor cores; tcgen05 has no fp64 kind).
// A fragments come from a per-CTA table F[D][lane] (A[a][c] = t[|a-c|]
// depends on D = 2·mtile − kstep only), B fragments straight from L2 into
// registers, 8 k-steps per batch.
//
// Gather: thread (point, RHS group): the 6×6 window, sum-factorised along
// axis 1 first (interpolation.cpp:66-97 weights, staged as (w, dw) pairs).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "lean2d.hpp"
#include "gk_sync.cuh"

namespace gk {

namespace {

constexpr int L2D_THREADS = 256;
constexpr int kLeanProf = 8;

struct LArgs {
  int m0, m1, nb0, nb1, n, nrhs, BRP, L, nseg;
  const int4* base;
  const double2* wd;  // [n][2][T] (w, dw): axis 0 then axis 1
  const int* cs;      // cell_start [nb0*nb1 + 1]
  const double* t0;
  const double* t1;
  double nv2, ng2;
  int noise, prefetch;
  const double* v;
  double* out;
  double* uu;  // scatter output, [M][R][2]: slot = segment parity (both slots summed by T1)
  double* y1;
  double* w;
  unsigned long long* bar;
  unsigned long long* prof;
  // Toeplitz job geometry
  int kp1, mt1, nt1, mc1, ms1, dlo1, nd1;  // mode 1: K = m1, M = m1, N = m0·R
  int kp0, mt0, nt0, mc0, ms0, dlo0, nd0;  // mode 0: K = m0, M = m0, N = m1·R
};



__device__ __forceinline__ void stamp(const LArgs& a, int k) {
  if (a.prof != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.prof[blockIdx.x * kLeanProf + k] = t;
  }
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// This CTA's share of a byte range, prefetched into L2 by TMA (16-byte granules).
__device__ __forceinline__ void prefetch_share(const void* base, size_t bytes) {
  const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
  const size_t lo = per * blockIdx.x;
  if (lo >= bytes) return;
  size_t len = min(per, bytes - lo) & ~size_t(15);
  const char* p = static_cast<const char*>(base) + lo;
  while (len > 0) {
    const unsigned c = unsigned(min(len, size_t(1) << 20));
    prefetch_l2(p, c);
    p += c;
    len -= c;
  }
}

// Warp-granular round robin over CTAs: consecutive 32-task groups go to
// different CTAs (and SMs), so a phase with fewer tasks than threads still
// spreads over the whole chip instead of filling the first CTAs.
__device__ __forceinline__ int first_task() {
  return ((threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31);
}
__device__ __forceinline__ int task_stride() { return gridDim.x * L2D_THREADS; }
__device__ __forceinline__ int first_warp_job() { return (threadIdx.x >> 5) * gridDim.x + blockIdx.x; }

template <int RP>
__device__ __forceinline__ void ldv(const double* p, double (&x)[RP]) {
  if constexpr (RP == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = t.x;
    x[1] = t.y;
  } else {
    x[0] = __ldg(p);
  }
}
template <int RP>
__device__ __forceinline__ void ldcg(const double* p, double (&x)[RP]) {
  if constexpr (RP == 2) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    x[0] = t.x;
    x[1] = t.y;
  } else {
    x[0] = __ldcg(p);
  }
}
template <int RP>
__device__ __forceinline__ void stv(double* p, const double (&x)[RP]) {
  if constexpr (RP == 2) *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
  else *p = x[0];
}

// ---------------------------------------------------------------- phase S
template <int T, int RP>
__device__ __forceinline__ void phase_scatter(const LArgs& a) {
  const int R = a.nrhs, BRP = a.BRP, L = a.L;
  const size_t gstride = size_t(a.n) * R;
  // With 2·BRP ≤ 32, a task's points are split between two lanes of one warp
  // (halves h = 0, 1 take alternate points); completed node rows are combined
  // as half0 + half1 by a shuffle (fixed order: deterministic).
  const bool split = 2 * BRP <= 32;
  const int HB = BRP;                                // lanes per half
  const int gpw = split ? 32 / (2 * HB) : 32 / HB;   // task groups per warp
  const int tpw = gpw * HB;                          // logical tasks per warp
  const int nlog = a.nseg * a.m1 * BRP;
  const int nwarps = (nlog + tpw - 1) / tpw;
  const int lane = threadIdx.x & 31;
  const int grp = split ? lane / (2 * HB) : lane / HB;
  const int inl = split ? lane % (2 * HB) : lane % HB;
  const int half = split ? inl / HB : 0, sub = split ? inl % HB : inl;
  const int pstep = split ? 2 : 1;
  for (int wi = (blockIdx.x * L2D_THREADS + threadIdx.x) >> 5; wi < nwarps; wi += task_stride() >> 5) {
    const int task = wi * tpw + grp * HB + sub;  // logical (seg, col, rp) task
    const bool live = grp < gpw && task < nlog;
    const int rp = live ? task % BRP : 0;
    const int t2 = live ? task / BRP : 0;
    const int col = t2 % a.m1;
    const int seg = t2 / a.m1;
    const int r = rp * RP;
    const int b_lo = live ? seg * L : 0, b_hi = live ? min(b_lo + L, a.nb0) : 0;
    const int clo = max(0, col - (T - 1)), chi = min(a.nb1 - 1, col);
    // row `row` of this segment goes to slot (seg & 1); the other slot gets an
    // explicit 0 where no other segment covers the row (the first segment's
    // head rows, the last segment's rows past the previous one's reach)
    const int par = seg & 1;
    auto store = [&](int row, const double (&o)[RP]) {
      double* e = a.uu + ((size_t(row) * a.m1 + col) * R + r) * 2;
      const bool zero_other = (seg == 0 && row < L) || (seg == a.nseg - 1 && row >= seg * L + (T - 1));
#pragma unroll
      for (int k = 0; k < RP; ++k) {
        e[2 * k + par] = o[k];
        if (zero_other) e[2 * k + 1 - par] = 0.0;
      }
    };
    int row = b_lo;
    double acc[T][RP];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int k = 0; k < RP; ++k) acc[t][k] = 0.0;
    const int nc = chi - clo + 1;  // cells (b0, clo..chi) reach this column; tl = col - cell
#pragma unroll 1
    for (int i = 0; i < L; ++i) {  // uniform trip count (the row combine shuffles)
      const bool rowok = b_lo + i < b_hi;
      // the cell boundaries of this row in registers: a point's axis-1 tap
      // offset follows from comparisons, not from a load of its base cell
      const int* cr = a.cs + size_t(b_lo + i) * a.nb1 + clo;
      int bnd[T + 1];
#pragma unroll
      for (int c = 0; c <= T; ++c) bnd[c] = (rowok && c <= nc) ? __ldg(cr + c) : 0;
      int pend = bnd[0];
#pragma unroll
      for (int c = 1; c <= T; ++c)
        if (c == nc) pend = bnd[c];
#pragma unroll 2
      for (int p = bnd[0] + half; p < pend; p += pstep) {
        int cidx = 0;
#pragma unroll
        for (int c = 1; c < T; ++c) cidx += (c < nc && p >= bnd[c]) ? 1 : 0;
        const int tl = col - clo - cidx;
        const double2* wr = a.wd + size_t(p) * 2 * T;
        const double* vr = a.v + size_t(p) * R + r;
        double v0[RP], v1[RP], v2[RP];
        ldv<RP>(vr, v0);
        ldv<RP>(vr + gstride, v1);
        ldv<RP>(vr + 2 * gstride, v2);
        const double2 w1 = __ldg(wr + T + tl);
        double A[RP], Cc[RP];
#pragma unroll
        for (int k = 0; k < RP; ++k) {
          A[k] = fma(w1.y, v2[k], w1.x * v0[k]);
          Cc[k] = w1.x * v1[k];
        }
#pragma unroll
        for (int t0 = 0; t0 < T; ++t0) {
          const double2 w0 = __ldg(wr + t0);
#pragma unroll
          for (int k = 0; k < RP; ++k) acc[t0][k] = fma(w0.y, Cc[k], fma(w0.x, A[k], acc[t0][k]));
        }
      }
      {
        double o[RP];
#pragma unroll
        for (int k = 0; k < RP; ++k) o[k] = split ? acc[0][k] + __shfl_down_sync(0xffffffffu, acc[0][k], HB) : acc[0][k];
        if (half == 0 && rowok) store(row, o);  // node row b_lo + i is complete for this segment
      }
      if (rowok) {  // advance the window (rows past the segment's last cell row keep it)
        ++row;
#pragma unroll
        for (int t = 0; t < T - 1; ++t)
#pragma unroll
          for (int k = 0; k < RP; ++k) acc[t][k] = acc[t + 1][k];
#pragma unroll
        for (int k = 0; k < RP; ++k) acc[T - 1][k] = 0.0;
      }
    }
    // node rows b_hi .. b_hi + T - 2 (the next segment adds its part in T1)
#pragma unroll
    for (int t = 0; t < T - 1; ++t) {
      double o[RP];
#pragma unroll
      for (int k = 0; k < RP; ++k) o[k] = split ? acc[t][k] + __shfl_down_sync(0xffffffffu, acc[t][k], HB) : acc[t][k];
      if (half == 0 && live) store(row + t, o);
      
    }
  }
}

// ---------------------------------------------------------------- Toeplitz
// F[D - dlo][lane] = t[|4D + lane/4 - lane%4|] (0 beyond the sequence).
// ts: the sequence already staged in shared memory.
__device__ __forceinline__ void build_table(double* F, const double* ts, int len, int dlo, int nd) {
  for (int e = threadIdx.x; e < nd * 32; e += L2D_THREADS) {
    const int D = e / 32 + dlo, ln = e % 32;
    int x = 4 * D + ln / 4 - ln % 4;
    x = x < 0 ? -x : x;
    F[e] = x < len ? ts[x] : 0.0;
  }
}

// One Toeplitz mode product over the whole batch: D[m][n] = Σ_k t[|m-k|] B[k][n]
// for m in [0, M), n in [0, Nn). MODE 1: n = (i, r) (i < m0, r < R), B[k][n] =
// u(i, k, r) read as the sum of the covering segment buffers, D -> y1(i, m, r).
// MODE 0: n = (j, r) contiguous, B[k][n] = y1(k, ·)[n], D -> w(m, ·)[n].
template <int MODE, int MC, int KS>
__device__ __forceinline__ void phase_toeplitz(const LArgs& a, const double* F) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int R = a.nrhs;
  const int K = MODE == 1 ? a.m1 : a.m0;   // contraction length (= output length M)
  const int kp = MODE == 1 ? a.kp1 : a.kp0;
  const int mtiles = MODE == 1 ? a.mt1 : a.mt0;
  const int ntiles = MODE == 1 ? a.nt1 : a.nt0;
  const int ms = MODE == 1 ? a.ms1 : a.ms0;
  const int dlo = MODE == 1 ? a.dlo1 : a.dlo0;
  const int Nn = MODE == 1 ? a.m0 * R : a.m1 * R;
  const int njobs = ntiles * ms;
  const int gw = first_warp_job();
  const int nw = (gridDim.x * L2D_THREADS) >> 5;
  const size_t rowlen = size_t(a.m1) * R;  // one grid row, all RHS
  for (int job = gw; job < njobs; job += nw) {
    const int nt = job % ntiles, mh = job / ntiles;
    const int mt_lo = mh * MC;
    const int nmt = min(MC, mtiles - mt_lo);
    // this lane's B column (k-row t4 of each step, column g of the tile)
    const int nb = nt * 8 + g;
    const bool nok = nb < Nn;
    // MODE 1: column (i, r); its node row i is covered by segment s_hi (and
    // s_hi - 1 when within its T-1 tail rows)
    const double* src0 = nullptr;
    size_t kstride;
    if constexpr (MODE == 1) {  // u(i, k, r) = slot 0 + slot 1 (one 16-byte load)
      const int i = nok ? nb / R : 0, r = nok ? nb - (nb / R) * R : 0;
      src0 = a.uu + (size_t(i) * rowlen + r) * 2;
      kstride = size_t(R) * 2;
    } else {
      src0 = a.y1 + nb;
      kstride = rowlen;
    }
    double acc[MC][2];
#pragma unroll
    for (int q = 0; q < MC; ++q) acc[q][0] = acc[q][1] = 0.0;
    // B column block of this n-tile in chunks of 8 k-steps, the next chunk's
    // loads in flight while the current one feeds the DMMAs
    const int ksteps = kp >> 2;
    auto loadb = [&](int kc, double (&bb)[8]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = 4 * (kc + q) + t4;
        double x = 0.0;
        if (nok && k < K) {
          if constexpr (MODE == 1) {
            const double2 t = __ldcg(reinterpret_cast<const double2*>(src0 + size_t(k) * kstride));
            x = t.x + t.y;
          } else {
            x = __ldcg(src0 + size_t(k) * kstride);
          }
        }
        bb[q] = x;
      }
    };
    double b[8], bn[8];
    loadb(0, b);
    // A fragments for k-step s: f[q] = F[2(mt_lo+q) - s - dlo][lane] (table
    // rows padded, so the loads are unconditional); the next step's fragments
    // are loaded while the current step's DMMAs issue
    const double* Fb = F + (2 * mt_lo - dlo) * 32 + lane;
    double f[MC], fn[MC];
#pragma unroll
    for (int q = 0; q < MC; ++q) f[q] = Fb[2 * q * 32];
#pragma unroll 1
    for (int kc = 0; kc < ksteps; kc += 8) {
      if (kc + 8 < ksteps) loadb(kc + 8, bn);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int ks = kc + s;
#pragma unroll
        for (int q = 0; q < MC; ++q) fn[q] = Fb[(2 * q - ks - 1) * 32];
        if (ks < ksteps) {
#pragma unroll
          for (int q = 0; q < MC; ++q)
            if (q < nmt) dmma(acc[q][0], acc[q][1], f[q], b[s]);
        }
#pragma unroll
        for (int q = 0; q < MC; ++q) f[q] = fn[q];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = bn[q];
    }
    // store: lane holds rows m = 8·mt + g, columns n = 8·nt + 2·t4 + {0,1}
#pragma unroll
    for (int q = 0; q < MC; ++q) {
      if (q < nmt) {
        const int m = 8 * (mt_lo + q) + g;
        if (m < K) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = nt * 8 + 2 * t4 + e;
            if (n < Nn) {
              if constexpr (MODE == 1) {
                const int i = n / R, r = n - (n / R) * R;
                a.y1[size_t(i) * rowlen + size_t(m) * R + r] = acc[q][e];
              } else {
                a.w[size_t(m) * rowlen + n] = acc[q][e];
              }
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- phase G
template <int T, int RP>
__device__ __forceinline__ void phase_gather(const LArgs& a) {
  const int R = a.nrhs, BRP = a.BRP;
  const size_t gstride = size_t(a.n) * R;
  const size_t rowlen = size_t(a.m1) * R;
  const int ntask = a.n * BRP;
  for (int task = blockIdx.x * L2D_THREADS + threadIdx.x; task < ntask; task += task_stride()) {
    const int rp = task % BRP, p = task / BRP;
    const int r = rp * RP;
    const int4 bs = __ldg(a.base + p);
    const double2* wr = a.wd + size_t(p) * 2 * T;
    double2 w1[T];
#pragma unroll
    for (int t = 0; t < T; ++t) w1[t] = __ldg(wr + T + t);
    const double* wrow = a.w + (size_t(bs.x) * a.m1 + bs.y) * R + r;
    double o0[RP], o1[RP], o2[RP];
#pragma unroll
    for (int k = 0; k < RP; ++k) o0[k] = o1[k] = o2[k] = 0.0;
    double2 w0a[T];
#pragma unroll
    for (int t = 0; t < T; ++t) w0a[t] = __ldg(wr + t);
#pragma unroll
    for (int t0 = 0; t0 < T; t0 += 2) {
      double x[2][T][RP];  // two node rows of the window: 2·T independent loads
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) ldcg<RP>(wrow + size_t(h) * rowlen + size_t(t1) * R, x[h][t1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double s[RP], q[RP];
#pragma unroll
        for (int k = 0; k < RP; ++k) {
          s[k] = 0.0;
          q[k] = 0.0;
        }
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1)
#pragma unroll
          for (int k = 0; k < RP; ++k) {
            s[k] = fma(w1[t1].x, x[h][t1][k], s[k]);
            q[k] = fma(w1[t1].y, x[h][t1][k], q[k]);
          }
        const double2 w0 = w0a[t0 + h];
#pragma unroll
        for (int k = 0; k < RP; ++k) {
          o0[k] = fma(w0.x, s[k], o0[k]);
          o1[k] = fma(w0.y, s[k], o1[k]);
          o2[k] = fma(w0.x, q[k], o2[k]);
        }
      }
      wrow += 2 * rowlen;
    }
    const size_t e0 = size_t(p) * R + r;
    if (a.noise) {
      double n0[RP], n1[RP], n2[RP];
      ldv<RP>(a.v + e0, n0);
      ldv<RP>(a.v + e0 + gstride, n1);
      ldv<RP>(a.v + e0 + 2 * gstride, n2);
#pragma unroll
      for (int k = 0; k < RP; ++k) {
        o0[k] = fma(a.nv2, n0[k], o0[k]);
        o1[k] = fma(a.ng2, n1[k], o1[k]);
        o2[k] = fma(a.ng2, n2[k], o2[k]);
      }
    }
    stv<RP>(a.out + e0, o0);
    stv<RP>(a.out + e0 + gstride, o1);
    stv<RP>(a.out + e0 + 2 * gstride, o2);
  }
}

template <int T, int RP, int MC>
__global__ void __launch_bounds__(L2D_THREADS, 2) k_lean2d(LArgs a) {
  extern __shared__ double sm[];
  double* F1 = sm;                 // [nd1][32]
  double* F0 = sm + a.nd1 * 32;    // [nd0][32]
  double* ts = F0 + a.nd0 * 32;    // [m1 + m0] the two Toeplitz sequences
  stamp(a, 0);
  // inputs into L2 (TMA bulk prefetch, no registers held)
  if (a.prefetch && threadIdx.x == 0) {
    prefetch_share(a.v, size_t(3) * a.n * a.nrhs * sizeof(double));
    prefetch_share(a.wd, size_t(a.n) * 2 * T * sizeof(double2));
    prefetch_share(a.base, size_t(a.n) * sizeof(int4));
  }
  for (int e = threadIdx.x; e < a.m1 + a.m0; e += L2D_THREADS)
    ts[e] = e < a.m1 ? __ldg(a.t1 + e) : __ldg(a.t0 + e - a.m1);
  __syncthreads();
  build_table(F1, ts, a.m1, a.dlo1, a.nd1);
  build_table(F0, ts + a.m1, a.m0, a.dlo0, a.nd0);
  phase_scatter<T, RP>(a);
  stamp(a, 1);
  grid_sync(a.bar);  // also publishes the tables (__syncthreads inside)
  stamp(a, 2);
  phase_toeplitz<1, MC, 8>(a, F1);
  stamp(a, 3);
  grid_sync(a.bar);
  stamp(a, 4);
  phase_toeplitz<0, MC, 8>(a, F0);
  stamp(a, 5);
  grid_sync(a.bar);
  stamp(a, 6);
  phase_gather<T, RP>(a);
  stamp(a, 7);
}

constexpr int kMC = 8;  // m-tiles per Toeplitz warp job (register accumulators)

const void* pick(int T, int RP) {
  if (T == 6) return RP == 2 ? (const void*)k_lean2d<6, 2, kMC> : (const void*)k_lean2d<6, 1, kMC>;
  return RP == 2 ? (const void*)k_lean2d<4, 2, kMC> : (const void*)k_lean2d<4, 1, kMC>;
}

}  // namespace

void lean2d_plan(const Fused2dGeom& g, int nrhs, int device, Lean2dPlan& p) {
  p.ok = false;
  p.nrhs = nrhs;
  if (nrhs < 1 || nrhs > 64 || (g.T != 6 && g.T != 4)) return;
  if (g.m0 < g.T || g.m1 < g.T || g.m0 > 128 || g.m1 > 128) return;
  p.RP = nrhs % 2 == 0 ? 2 : 1;
  p.BRP = nrhs / p.RP;
  if (p.BRP > 32) return;
  p.L = g.T - 1;
  p.nseg = (g.nb0 + p.L - 1) / p.L;
  const int kp1 = (g.m1 + 3) / 4 * 4, kp0 = (g.m0 + 3) / 4 * 4;
  p.mt1 = (g.m1 + 7) / 8;
  p.mt0 = (g.m0 + 7) / 8;
  p.kp1 = kp1;
  p.kp0 = kp0;
  p.nt1 = (g.m0 * nrhs + 7) / 8;
  p.nt0 = (g.m1 * nrhs + 7) / 8;
  p.ms1 = (p.mt1 + kMC - 1) / kMC;
  p.ms0 = (p.mt0 + kMC - 1) / kMC;
  // table rows D = 2·mt − kstep over mt < mtiles, kstep < kp/4 (and the
  // 8-step batches read up to 7 steps past kp/4 only when masked off)
  p.dlo1 = -(kp1 / 4 - 1) - 10;
  p.dlo0 = -(kp0 / 4 - 1) - 10;
  // upper rows: up to 2·(mt_lo + MC - 1) for masked m-tiles of the last job
  p.nd1 = 2 * (p.ms1 * kMC - 1) - p.dlo1 + 1;
  p.nd0 = 2 * (p.ms0 * kMC - 1) - p.dlo0 + 1;
  p.smem = sizeof(double) * (32 * size_t(p.nd1 + p.nd0) + g.m0 + g.m1);
  const void* fn = pick(g.T, p.RP);
  raise_smem_limit(fn, p.smem);
  int sms = 0, occ = 0;
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, L2D_THREADS, p.smem));
  if (occ < 1) return;
  p.grid = std::min(occ, 2) * sms;
  p.bar.alloc(kBarSlots);
  GK_CUDA(cudaMemset(p.bar.p, 0, sizeof(unsigned long long) * kBarSlots));
  p.ok = true;
}

void lean2d_mvm(const Fused2dGeom& g, Lean2dPlan& p, const double* v, double* out, double* uu,
                double* y1, double* w, bool noise, cudaStream_t s) {
  LArgs a{};
  a.m0 = g.m0;
  a.m1 = g.m1;
  a.nb0 = g.nb0;
  a.nb1 = g.nb1;
  a.n = g.n;
  a.nrhs = p.nrhs;
  a.BRP = p.BRP;
  a.L = p.L;
  a.nseg = p.nseg;
  a.base = g.base;
  a.wd = g.wd;
  a.cs = g.cell_start;
  a.t0 = g.t0;
  a.t1 = g.t1;
  a.nv2 = g.nv2;
  a.ng2 = g.ng2;
  a.noise = noise ? 1 : 0;
  a.prefetch = g_tuning.f2_nst.load() == 7 ? 0 : 1;  // A/B knob: 7 = no L2 prefetch
  a.v = v;
  a.out = out;
  a.uu = uu;
  a.y1 = y1;
  a.w = w;
  a.bar = p.bar.p;
  a.prof = nullptr;
  if (g_tuning.fused_prof.load() != 0) {
    if (p.prof.n < size_t(p.grid) * kLeanProf) {
      p.prof.alloc(size_t(p.grid) * kLeanProf);
      GK_CUDA(cudaMemset(p.prof.p, 0, sizeof(unsigned long long) * p.prof.n));
    }
    a.prof = p.prof.p;
  }
  a.kp1 = p.kp1;
  a.mt1 = p.mt1;
  a.nt1 = p.nt1;
  a.mc1 = kMC;
  a.ms1 = p.ms1;
  a.dlo1 = p.dlo1;
  a.nd1 = p.nd1;
  a.kp0 = p.kp0;
  a.mt0 = p.mt0;
  a.nt0 = p.nt0;
  a.mc0 = kMC;
  a.ms0 = p.ms0;
  a.dlo0 = p.dlo0;
  a.nd0 = p.nd0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.grid));
  cfg.blockDim = dim3(L2D_THREADS);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  GK_CUDA(cudaLaunchKernelExC(&cfg, pick(g.T, p.RP), args));
  launched("dski lean 2-D MVM");
}

}  // namespace gk
