// kron.cu — K_UU mode products and column reductions.
//
// K_UU for a separable stationary kernel on a regular grid is ⊗_j T_j with
// T_j the symmetric Toeplitz matrix of the 1-D profile (reference builds the
// same operator through a circulant embedding, dski.cpp:80-166). One mode
// product is a batched GEMM  Y[p] = T_j X[p]  with X[p] an (m_j × Q) slab;
// the Toeplitz tile is generated in shared memory from the 1-D sequence so
// T_j is never stored.
#include "gk_kernels.cuh"

namespace gk {

namespace {

template <int TM, int TN>
__global__ void __launch_bounds__(256) k_toeplitz(const double* __restrict__ t, int M, int band, i64 P,
                                                  i64 Q, const double* __restrict__ X,
                                                  double* __restrict__ Y) {
  constexpr int BM = 16 * TM, BN = 16 * TN, BK = 16;
  __shared__ double As[BK][BM];
  __shared__ double Bs[BK][BN + 1];
  const i64 ncols = P * Q;
  const i64 col0 = (i64)blockIdx.x * BN;
  const int a0 = blockIdx.y * BM;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const bool q_major = Q >= 16;

  // Per-thread load slots for Bs: BK*BN elements over 256 threads.
  constexpr int SLOTS = (BK * BN + 255) / 256;
  i64 soff[SLOTS];
  int skk[SLOTS], scc[SLOTS];
  bool sval[SLOTS];
#pragma unroll
  for (int r = 0; r < SLOTS; ++r) {
    const int idx = tid + 256 * r;
    int kk, cc;
    if (q_major) {
      kk = idx / BN;
      cc = idx % BN;
    } else {
      kk = idx % BK;
      cc = idx / BK;
    }
    skk[r] = kk;
    scc[r] = cc;
    const i64 col = col0 + cc;
    sval[r] = idx < BK * BN && col < ncols;
    const i64 p = sval[r] ? col / Q : 0, q = sval[r] ? col % Q : 0;
    soff[r] = p * (i64)M * Q + q;
  }

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

  for (int c0 = 0; c0 < M; c0 += BK) {
    const int dmin = max(0, max(c0 - (a0 + BM - 1), a0 - (c0 + BK - 1)));
    if (dmin >= band) continue;  // block-uniform
    for (int idx = tid; idx < BK * BM; idx += 256) {
      const int kk = idx / BM, mm = idx % BM;
      const int a = a0 + mm, c = c0 + kk;
      As[kk][mm] = (a < M && c < M) ? __ldg(t + (a > c ? a - c : c - a)) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < SLOTS; ++r) {
      if (tid + 256 * r < BK * BN) {
        const int c = c0 + skk[r];
        Bs[skk[r]][scc[r]] = (sval[r] && c < M) ? __ldg(X + soff[r] + (i64)c * Q) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const i64 col = col0 + tx + 16 * j;
    if (col >= ncols) continue;
    const i64 p = col / Q, q = col % Q;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int a = a0 + ty + 16 * i;
      if (a < M) Y[(p * M + a) * Q + q] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------- DMMA path
// Same product on the fp64 tensor cores: mma.sync.m8n8k4 (DMMA). CTA = 2×2
// warps, warp tile (8·WM)×(8·WN); the Toeplitz A tile is generated from the
// 1-D sequence into shared memory, B is staged with the layout-aware slots.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int WM, int WN>
__global__ void __launch_bounds__(128) k_toeplitz_dmma(const double* __restrict__ t, int M, int band, i64 P,
                                                       i64 Q, const double* __restrict__ X,
                                                       double* __restrict__ Y) {
  constexpr int BM = 16 * WM, BN = 16 * WN, BK = 16;
  constexpr int SA = BM + 8, SB = BN + 8;  // row strides ≡ 8 (mod 16) doubles: conflict-free fragments
  __shared__ double As[BK * SA];
  __shared__ double Bs[BK * SB];
  const i64 ncols = P * Q;
  const i64 col0 = (i64)blockIdx.x * BN;
  const int a0 = blockIdx.y * BM;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = (warp / 2) * (8 * WM), wn = (warp % 2) * (8 * WN);
  const int g = lane / 4, t4 = lane % 4;
  const bool q_major = Q >= 16;
  __shared__ long long coff[BN];
  if (tid < BN) {
    const long long col = col0 + tid;
    coff[tid] = col < ncols ? (long long)(int(col) / int(Q)) * M * Q + int(col) % int(Q) : -1;
  }
  __syncthreads();
  constexpr int SLOTS = (BK * BN + 127) / 128;
  i64 soff[SLOTS];
  int skk[SLOTS], scc[SLOTS];
  bool sval[SLOTS];
#pragma unroll
  for (int r = 0; r < SLOTS; ++r) {
    const int idx = tid + 128 * r;
    const int kk = q_major ? idx / BN : idx % BK;
    const int cc = q_major ? idx % BN : idx / BK;
    skk[r] = kk;
    scc[r] = cc;
    sval[r] = idx < BK * BN && coff[cc] >= 0;
    soff[r] = sval[r] ? coff[cc] : 0;
  }
  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // k tiles that meet the band of rows [a0, a0 + BM): one contiguous range.
  // The next tile's A and B values are loaded into registers while the
  // current one computes (one global latency per launch, not per k tile).
  constexpr int ASL = (BK * BM + 127) / 128;
  const int lo = a0 - BK + 2 - band;  // first k-tile start whose last column is within the band
  const int c_begin = lo <= 0 ? 0 : (lo + BK - 1) / BK * BK;
  const int c_end = min(M, a0 + BM - 1 + band);
  double ra[ASL], rb[SLOTS];
  auto load = [&](int c0) {
#pragma unroll
    for (int r = 0; r < ASL; ++r) {
      const int idx = tid + 128 * r;
      const int kk = idx / BM, mm = idx % BM;
      const int a = a0 + mm, c = c0 + kk;
      ra[r] = (idx < BK * BM && a < M && c < M) ? __ldg(t + (a > c ? a - c : c - a)) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < SLOTS; ++r) {
      const int c = c0 + skk[r];
      rb[r] = (sval[r] && c < M) ? __ldg(X + soff[r] + (i64)c * Q) : 0.0;
    }
  };
  if (c_begin < c_end) load(c_begin);
  for (int c0 = c_begin; c0 < c_end; c0 += BK) {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ASL; ++r) {
      const int idx = tid + 128 * r;
      if (idx < BK * BM) As[(idx / BM) * SA + idx % BM] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < SLOTS; ++r)
      if (tid + 128 * r < BK * BN) Bs[skk[r] * SB + scc[r]] = rb[r];
    __syncthreads();
    if (c0 + BK < c_end) load(c0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[WM], bf[WN];
#pragma unroll
      for (int i = 0; i < WM; ++i) af[i] = As[(kk + t4) * SA + wm + 8 * i + g];
#pragma unroll
      for (int j = 0; j < WN; ++j) bf[j] = Bs[(kk + t4) * SB + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < WN; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const long long o = coff[wn + 8 * j + 2 * t4 + e];
      if (o < 0) continue;
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const int a = a0 + wm + 8 * i + g;
        if (a < M) Y[o + (long long)a * Q] = acc[i][j][e];
      }
    }
}

// Slab variant: a CTA owns BN output columns and ALL M rows; the whole K
// extent of its B slab (M × BN) and the 1-D sequence are staged in shared
// memory in one burst, so there is a single global-latency phase. A fragments
// are generated from the staged sequence (A[a][c] = t[|a-c|]); each warp takes
// m8-tiles round-robin in groups of 4, skipping k-steps outside the band.
template <int NT>  // n8-tiles per CTA (BN = 8·NT)
__global__ void __launch_bounds__(128) k_toeplitz_slab(const double* __restrict__ t, int M, int band, i64 P,
                                                       i64 Q, const double* __restrict__ X,
                                                       double* __restrict__ Y) {
  constexpr int BN = 8 * NT;
  constexpr int SB = BN + ((BN % 16 == 0) ? 8 : 0) + ((BN % 16 == 8) ? 0 : 0);
  extern __shared__ double sm[];
  const int Mp = (M + 7) / 8 * 8;
  double* ts = sm;                 // [Mp]
  double* Bs = sm + Mp;            // [Mp][SB]
  const i64 ncols = P * Q;
  const i64 col0 = (i64)blockIdx.x * BN;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t4 = lane % 4;
  for (int i = tid; i < Mp; i += 128) ts[i] = i < M ? __ldg(t + i) : 0.0;
  // Stage the B slab in batches of 8 independent loads per thread (issued
  // together, then stored), int32 index math: one L2 latency per batch
  // instead of one per element.
  // per-CTA column offsets (one 32-bit division per column, not per element)
  __shared__ long long coff[BN];
  const int Qi = int(Q), Mi = M;
  if (tid < BN) {
    const long long col = col0 + tid;
    coff[tid] = col < ncols ? (long long)(int(col) / Qi) * Mi * Qi + int(col) % Qi : -1;
  }
  __syncthreads();
  // Stage the B slab in batches of 8 independent loads per thread (issued
  // together, then stored): one L2 latency per batch.
  const bool q_major = Q >= BN;
  const int total = Mp * BN;
  for (int e0 = tid; e0 < total; e0 += 128 * 8) {
    double vals[8];
    int dst[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128;
      int c, cc;
      if (q_major) {
        c = e / BN;
        cc = e % BN;
      } else {
        cc = e / Mp;
        c = e - cc * Mp;
      }
      dst[u] = (e < total) ? c * SB + cc : -1;
      double v = 0.0;
      if (e < total && c < Mi) {
        const long long o = coff[cc];
        if (o >= 0) v = __ldg(X + o + (long long)c * Qi);
      }
      vals[u] = v;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dst[u] >= 0) Bs[dst[u]] = vals[u];
  }
  __syncthreads();
  const int mtiles = Mp / 8;
  const int ksteps = Mp / 4;
  for (int mt0 = warp * 4; mt0 < mtiles; mt0 += 16) {
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int ntile = min(4, mtiles - mt0);
    const int row_lo = mt0 * 8, row_hi = (mt0 + ntile) * 8 - 1;
    // k range whose |a - c| < band for some row in [row_lo, row_hi]
    const int k_lo = max(0, (row_lo - band + 1) / 4 * 4);
    const int k_hi = min(Mp, (row_hi + band + 4) / 4 * 4);
    for (int kk = k_lo; kk < k_hi; kk += 4) {
      const int c = kk + t4;
      double bf[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = Bs[c * SB + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i >= ntile) break;
        const int a = (mt0 + i) * 8 + g;
        const int dist = a > c ? a - c : c - a;
        const double af = (a < M && c < M) ? ts[dist] : 0.0;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af, bf[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i >= ntile) break;
      const int a = (mt0 + i) * 8 + g;
      if (a >= M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const long long o = coff[8 * j + 2 * t4 + e];
          if (o >= 0) Y[o + (long long)a * Qi] = acc[i][j][e];
        }
    }
  }
}

// Persistent variant for M ≤ 16·WM (one row block holds every row): the A
// operand is the same Toeplitz matrix for every column tile, so each warp
// keeps its A fragments in registers for the whole launch; CTAs (grid sized
// to the resident capacity) walk column tiles with the next tile's B slab
// copied by 8-byte cp.async while the current one computes. Same k order and
// fragment mapping as k_toeplitz_dmma<WM, WN>: bit-identical.
template <int WM, int WN>
__global__ void __launch_bounds__(128) k_toeplitz_pers(const double* __restrict__ t, int M, i64 P, i64 Q,
                                                       const double* __restrict__ X, double* __restrict__ Y) {
  constexpr int BM = 16 * WM, BN = 16 * WN;
  constexpr int SB = BN + 8;
  constexpr int KS = BM / 4;  // k steps covering every row (M ≤ BM, zero-padded)
  extern __shared__ __align__(16) double smp[];
  double* ts = smp;               // [BM]
  double* Bs = smp + BM;          // [2][BM][SB]
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = (warp / 2) * (8 * WM), wn = (warp % 2) * (8 * WN);
  const int g = lane / 4, t4 = lane % 4;
  const i64 ncols = P * Q;
  const i64 ntiles = (ncols + BN - 1) / BN;
  const int Qi = int(Q);
  for (int i = tid; i < BM; i += 128) ts[i] = i < M ? __ldg(t + i) : 0.0;
  __syncthreads();
  double af[KS][WM];
#pragma unroll
  for (int k = 0; k < KS; ++k)
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int a = wm + 8 * i + g, c = 4 * k + t4;
      af[k][i] = (a < M && c < M) ? ts[a > c ? a - c : c - a] : 0.0;
    }
  // staging slot: thread -> column cc = tid % BN, rows c = tid / BN + r·(128 / BN)
  constexpr int RSTEP = 128 / BN;
  const int scc = tid % BN, sc0 = tid / BN;
  auto issue = [&](i64 tile, int buf) {
    const i64 col = tile * BN + scc;
    double* dst = Bs + buf * (BM * SB);
    if (col < ncols) {
      const int p = int(col / Qi), q = int(col - (i64)p * Qi);
      const double* src = X + (i64)p * M * Qi + q;
      for (int c = sc0; c < BM; c += RSTEP) {
        if (c < M) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(
                           __cvta_generic_to_shared(dst + c * SB + scc))),
                       "l"(src + (i64)c * Qi)
                       : "memory");
        } else {
          dst[c * SB + scc] = 0.0;
        }
      }
    } else {
      for (int c = sc0; c < BM; c += RSTEP) dst[c * SB + scc] = 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  i64 tile = blockIdx.x;
  if (tile < ntiles) issue(tile, 0);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int buf = it & 1;
    if (tile + gridDim.x < ntiles) {
      issue(tile + gridDim.x, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* B = Bs + buf * (BM * SB);
    double acc[WM][WN][2];
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      double bf[WN];
#pragma unroll
      for (int j = 0; j < WN; ++j) bf[j] = B[(4 * k + t4) * SB + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[k][i], bf[j]);
    }
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const i64 col = tile * BN + wn + 8 * j + 2 * t4 + e;
        if (col >= ncols) continue;
        const int p = int(col / Qi), q = int(col - (i64)p * Qi);
        double* yo = Y + (i64)p * M * Qi + q;
#pragma unroll
        for (int i = 0; i < WM; ++i) {
          const int a = wm + 8 * i + g;
          if (a < M) yo[(i64)a * Qi] = acc[i][j][e];
        }
      }
    __syncthreads();  // every warp is done with this buffer before it is refilled
  }
}

template <int WM, int WN>
void launch_toeplitz_pers(const double* t, int M, i64 P, i64 Q, const double* X, double* Y, cudaStream_t s) {
  constexpr int BM = 16 * WM, BN = 16 * WN;
  const size_t shm = sizeof(double) * (BM + 2 * size_t(BM) * (BN + 8));
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    if (shm > 48 * 1024) raise_smem_limit((const void*)k_toeplitz_pers<WM, WN>, shm);
    GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_toeplitz_pers<WM, WN>, 128, shm));
    blocks_per_sm = std::max(1, blocks_per_sm);
  }
  const i64 ntiles = (P * Q + BN - 1) / BN;
  const unsigned grid = static_cast<unsigned>(std::min<i64>(ntiles, 148LL * blocks_per_sm));
  k_toeplitz_pers<WM, WN><<<grid, 128, shm, s>>>(t, M, P, Q, X, Y);
  launched("toeplitz mode product (DMMA, persistent)");
}

template <int NT>
void launch_toeplitz_slab(const double* t, int M, int band, i64 P, i64 Q, const double* X, double* Y,
                          cudaStream_t s) {
  constexpr int BN = 8 * NT;
  constexpr int SB = BN + ((BN % 16 == 0) ? 8 : 0);
  const int Mp = (M + 7) / 8 * 8;
  const size_t shm = sizeof(double) * (size_t(Mp) + size_t(Mp) * SB);
  if (shm > 48 * 1024)
    raise_smem_limit((const void*)k_toeplitz_slab<NT>, shm);
  const i64 ncols = P * Q;
  k_toeplitz_slab<NT><<<static_cast<unsigned>((ncols + BN - 1) / BN), 128, shm, s>>>(t, M, band, P, Q, X, Y);
  launched("toeplitz mode product (DMMA slab)");
}

template <int WM, int WN>
void launch_toeplitz_dmma(const double* t, int M, int band, i64 P, i64 Q, const double* X, double* Y,
                          cudaStream_t s) {
  constexpr int BM = 16 * WM, BN = 16 * WN;
  const i64 ncols = P * Q;
  dim3 grid(static_cast<unsigned>((ncols + BN - 1) / BN), static_cast<unsigned>((M + BM - 1) / BM));
  k_toeplitz_dmma<WM, WN><<<grid, 128, 0, s>>>(t, M, band, P, Q, X, Y);
  launched("toeplitz mode product (DMMA)");
}

template <int TM, int TN>
void launch_toeplitz(const double* t, int M, int band, i64 P, i64 Q, const double* X, double* Y,
                     cudaStream_t s) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  const i64 ncols = P * Q;
  dim3 grid(unsigned((ncols + BN - 1) / BN), unsigned((M + BM - 1) / BM));
  k_toeplitz<TM, TN><<<grid, 256, 0, s>>>(t, M, band, P, Q, X, Y);
  launched("toeplitz mode product");
}

// Deterministic per-column dot products over an RHS-minor block: each of
// kRedBlocks CTAs reduces a fixed row range; a second pass sums partials in
// CTA order.
__global__ void k_col_dot_partial(const double* __restrict__ x, const double* __restrict__ y, i64 rows,
                                  int nrhs, double* __restrict__ partial) {
  extern __shared__ double sm[];
  const int slots = blockDim.x / nrhs;  // row slots per pass
  const int tid = threadIdx.x;
  const int b = tid % nrhs, slot = tid / nrhs;
  double acc = 0.0;
  if (slot < slots) {
    const i64 per = (rows + gridDim.x - 1) / gridDim.x;
    const i64 r0 = (i64)blockIdx.x * per, r1 = min(rows, r0 + per);
    for (i64 r = r0 + slot; r < r1; r += slots) {
      const double a = x[r * nrhs + b];
      acc += a * (y ? y[r * nrhs + b] : a);
    }
  }
  sm[tid] = acc;
  __syncthreads();
  if (tid < nrhs) {
    double s = 0.0;
    for (int k = 0; k < slots; ++k) s += sm[k * nrhs + tid];
    partial[(i64)blockIdx.x * nrhs + tid] = s;
  }
}

__global__ void k_col_sum(const double* __restrict__ partial, int nblocks, int nrhs, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nrhs) return;
  double s = 0.0;
  for (int k = 0; k < nblocks; ++k) s += partial[(i64)k * nrhs + b];
  out[b] = s;
}

}  // namespace

void toeplitz_mode(const double* t, int M, int band, i64 P, i64 Q, const double* X, double* Y,
                   cudaStream_t s) {
  const i64 ncols = P * Q;
  auto ctas = [&](int bm, int bn) { return ((ncols + bn - 1) / bn) * ((M + bm - 1) / bm); };
  const int variant = g_tuning.toeplitz.load();
  if (variant == 1) {  // SIMT fp64 FMA, largest tile with >= 2 waves
    if (M > 32 && ctas(64, 64) >= 296) launch_toeplitz<4, 4>(t, M, band, P, Q, X, Y, s);
    else if (ctas(32, 64) >= 296) launch_toeplitz<2, 4>(t, M, band, P, Q, X, Y, s);
    else launch_toeplitz<2, 2>(t, M, band, P, Q, X, Y, s);
    return;
  }
  if ((variant == 0 || variant == 5) && M > 32 && M <= 64) {
    // one row block covering every row (no half-empty second block): C3's
    // 48-node axes 60.4 -> 48.1 µs for K_UU at 17 RHS (bit-identical: the
    // same k order per output)
    const bool wide = ctas(64, 64) >= 192;
    // persistent, A fragments in registers, next tile's B in flight: C3's
    // 48-node modes at 17 RHS 48.1 -> 46.1 µs (the 64-column persistent tile,
    // 152 registers, measured 52.3); bit-identical
    if (variant == 0 && M <= 48 && !(g_tuning.d3.load() & 8)) {
      // 16-column tiles when 32-column ones would leave SMs idle (1 RHS: 72 tiles)
      if (ncols < 148 * 32 && !(g_tuning.d3.load() & 8192)) launch_toeplitz_pers<3, 1>(t, M, P, Q, X, Y, s);
      else launch_toeplitz_pers<3, 2>(t, M, P, Q, X, Y, s);
      return;
    }
    if (M <= 48) { if (wide) launch_toeplitz_dmma<3, 4>(t, M, band, P, Q, X, Y, s); else launch_toeplitz_dmma<3, 2>(t, M, band, P, Q, X, Y, s); }
    else { if (wide) launch_toeplitz_dmma<4, 4>(t, M, band, P, Q, X, Y, s); else launch_toeplitz_dmma<4, 2>(t, M, band, P, Q, X, Y, s); }
    return;
  }
  if (variant == 0 || variant == 3 || variant == 5) {  // DMMA, smallest tile (most CTAs): best measured at C1-C4 sizes
    launch_toeplitz_dmma<2, 2>(t, M, band, P, Q, X, Y, s);
    return;
  }
  if (variant == 4) {  // DMMA slab: one staging phase per CTA
    const int Mp = (M + 7) / 8 * 8;
    // widest slab that keeps >= ~1.5 CTAs per SM and fits shared memory
    if (ncols >= 16 * 222 && size_t(Mp) * 24 * 8 <= 200 * 1024) launch_toeplitz_slab<2>(t, M, band, P, Q, X, Y, s);
    else if (size_t(Mp) * 8 * 8 <= 200 * 1024) launch_toeplitz_slab<1>(t, M, band, P, Q, X, Y, s);
    else launch_toeplitz_dmma<2, 2>(t, M, band, P, Q, X, Y, s);
    return;
  }
  // DMMA tiles; pick the largest that still gives >= ~1.3 waves over 148 SMs.
  if (M > 32 && ctas(64, 64) >= 192) launch_toeplitz_dmma<4, 4>(t, M, band, P, Q, X, Y, s);
  else if (ctas(32, 64) >= 192) launch_toeplitz_dmma<2, 4>(t, M, band, P, Q, X, Y, s);
  else launch_toeplitz_dmma<2, 2>(t, M, band, P, Q, X, Y, s);
}

void col_dot(const double* x, const double* y, i64 rows, int nrhs, double* out, double* partial,
             cudaStream_t s) {
  if (nrhs > kRedThreads) fail(GK_ERR_ARG, "col_dot: too many right-hand sides");
  k_col_dot_partial<<<kRedBlocks, kRedThreads, kRedThreads * sizeof(double), s>>>(x, y, rows, nrhs, partial);
  launched("col_dot partial");
  k_col_sum<<<(nrhs + 127) / 128, 128, 0, s>>>(partial, kRedBlocks, nrhs, out);
  launched("col_dot sum");
}

}  // namespace gk
