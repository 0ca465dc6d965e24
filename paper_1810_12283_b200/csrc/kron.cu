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
  // Pick the largest tile that still gives >= 2 waves of CTAs over 148 SMs.
  const i64 ncols = P * Q;
  auto ctas = [&](int bm, int bn) { return ((ncols + bn - 1) / bn) * ((M + bm - 1) / bm); };
  if (M > 32 && ctas(64, 64) >= 296) launch_toeplitz<4, 4>(t, M, band, P, Q, X, Y, s);
  else if (ctas(32, 64) >= 296) launch_toeplitz<2, 4>(t, M, band, P, Q, X, Y, s);
  else launch_toeplitz<2, 2>(t, M, band, P, Q, X, Y, s);
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
