// solvers.hpp — device-resident solvers over gk::Op (reference linalg.cpp).
#pragma once

#include <vector>

#include "gk_common.hpp"

namespace gk {

// Preconditioner (linalg.cpp:176-213): Q1 (N×k, internal row order, stored
// row-major so a row's k coefficients are contiguous) and D^{-1/2}.
struct Precond {
  int device = 0;
  i64 N = 0, k = 0;
  DevBuf<double> q1;       // [N][k]
  DevBuf<double> dinv;     // [N] internal order
  DevBuf<double> partial;  // [kRedBlocks][k][nrhs] scratch
  DevBuf<double> t;        // [k][nrhs]
  DevBuf<double> cbuf;     // scratch
  DevBuf<double> pad_r, pad_z;  // zero-padded (even-width) r / z for the v3 kernels
  // Row order of q1/dinv: the internal order of operator `order_uid`
  // (0 = external order). `ext` points at this object's own copy of that
  // operator's internal->external row map, so it outlives the operator.
  std::uint64_t order_uid = 0;
  DevBuf<i64> ext_own;
  const i64* ext = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int ensured_nrhs = 0;
  ~Precond();
  // z = M^{-1} r; optionally rz[b] partials. All internal layout.
  // z = M^{-1} r (internal layout); optionally r·z partials per column into
  // partial_rz[block][nrhs]. Returns the number of partial blocks written.
  int apply(const double* r, double* z, int nrhs, cudaStream_t s, double* partial_rz = nullptr);
  void ensure(int nrhs);
  bool mma_ok(int nrhs) const;
  int proj_rch(int nrhs) const;
  size_t proj_mma_smem(int nrhs) const;
  size_t apply_mma_smem(int nrhs) const;
};

struct PivChol {
  int device = 0;
  i64 N = 0, k = 0;
  DevBuf<double> L;  // [k][N] column-major, internal row order
  std::vector<i64> pivots;  // external indices
  double initial_trace = 0, residual_trace = 0;
  // owned copies so the factor outlives its operator
  std::uint64_t order_uid = 0;
  DevBuf<i64> ext_own;  // internal -> external row map (empty = identity)
  cudaStream_t stream = nullptr;
  ~PivChol();
};

struct PcgResult {
  std::vector<int> iterations, converged, hist_len;
  std::vector<double> history;  // (maxit+1) × nrhs, row = iteration
};

// Batched PCG on internal-layout blocks B (N×nrhs), X output.
PcgResult pcg_internal(Op& op, Precond* M, const double* B, double* X, int nrhs, double tol, int maxit,
                       bool want_history, cudaStream_t s);

std::unique_ptr<PivChol> pivchol_run(Op& op, bool kernel_part, i64 max_rank, double trace_tol);

std::unique_ptr<Precond> precond_build(const double* F_int /*[k][N] dev col-major*/, i64 N, i64 k,
                                       const double* noise_int /*dev [N]*/, int device, cudaStream_t s);

struct LanczosBatch {
  int P = 0;
  int steps = 0;
  std::vector<int> len;                 // achieved rank per probe
  std::vector<std::vector<double>> alpha, beta;
  std::vector<int> breakdown;
};
// Lanczos with two-pass full reorthogonalisation (linalg.cpp:17-81) for P
// start vectors at once (internal layout, N×P). Q_out (optional, device) receives
// [steps][N][P].
LanczosBatch lanczos_batch(Op& op, const double* start_int, int P, int steps,
                           const std::vector<std::uint64_t>& restart_seeds, double* Q_out,
                           cudaStream_t s);

// P Rademacher probe vectors generated on the device, bit-identical to the
// host's std::mt19937_64(seeds[q]) streams (sign = bit 0 of each draw).
void rademacher_dev(i64 n, const std::uint64_t* seeds_h, int P, double scale, double* out, i64 ld, cudaStream_t s);

// Row-sharded preconditioner pieces: T = Q1ᵀ D^{-1/2} r, then
// z = D^{-1/2}(D^{-1/2} r − Q1 T) with an all-reduced T; and a Precond over an
// explicit Q1 (N×k col-major) and D^{-1/2} (device).
void precond_project(Precond& M, const double* r, int nrhs, double* T, cudaStream_t s);
void precond_finish(Precond& M, const double* r, const double* T, double* z, int nrhs, cudaStream_t s);
std::unique_ptr<Precond> precond_from_q1(const double* Q1cm, const double* dinv, i64 N, i64 k, int device,
                                         cudaStream_t s);

// Small block products used by the GP glue (internal RHS-minor layouts; all
// results deterministic, fixed summation order).
//   C = A·Bm (rows×ka times ka×nb, Bm on the device, row-major)
void rows_gemm_dev(const double* A, int ka, const double* Bm_dev, int nb, i64 rows, double* C, bool accumulate,
                   cudaStream_t s);
//   out[t][j] = Σ_r A[r][t]·D[r][j]  (ka×nb, device)
void cross_dev(const double* A, int ka, const double* D, int nb, i64 rows, double* out_dev, DevBuf<double>& part,
               cudaStream_t s);
//   out[b] = Σ_r X[r][b]·Y[r][b]  (device)
void col_dots_dev(const double* X, const double* Y, i64 rows, int nrhs, double* out_dev, DevBuf<double>& part,
                  cudaStream_t s);
void sub_dev(const double* a, const double* b, double* c, i64 n, cudaStream_t s);

}  // namespace gk
