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
    for (int c = 0; c < chunks; ++c) s += partial[(i64)c * items + it];
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

static void hadamard_pair(const Factor& A, const Factor& B, const double* v, int nrhs, double* out, bool accumulate,
                          const double* noise_v, i64 n_value, double nv2, double ng2, HadScratch& ws,
                          cudaStream_t s) {
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
  const i64 N = op.N;
  std::vector<double> q(static_cast<size_t>(N));
  gaussian(N, seed, 0, q.data());
  double nn = 0.0;
  for (double v : q) nn += v * v;
  nn = std::sqrt(nn);
  for (double& v : q) v /= nn;
  DevBuf<double> start(static_cast<size_t>(N)), Qc(static_cast<size_t>(N) * rank);
  start.upload(q.data(), q.size(), s);
  LanczosBatch lb = lanczos_batch(op, start.p, 1, int(rank), {mix_seed(seed, 1)}, Qc.p, s);
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
      leaf.core = make_dski_profile(k1, g1, col.data(), n, 0.0, 0.0, 0, dir >= 0 ? 1 : 0, device, pass);
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
