// kuu_fft.hpp — K_UU for a general (non-separable) stationary profile on a
// d-dimensional grid (d ≤ 3): the circulant-embedding route of the reference
// GridKernelOperator (dski.cpp:80-172), with an in-house batched complex FFT.
#pragma once

#include <vector>

#include "gk_common.hpp"

namespace gk {

struct KuuFft {
  int d = 0;
  int m[3] = {1, 1, 1};     // grid nodes per axis
  int E[3] = {1, 1, 1};     // embedding size per axis: the power of two ≥ 2m − 1
  int logE[3] = {0, 0, 0};
  i64 Etot = 1, M = 1;
  DevBuf<double> spec;      // real spectrum of the embedded profile slice, divided by Etot
  DevBuf<double2> tw[3];    // per axis: exp(−2πi k / E), k < E/2
  mutable DevBuf<double2> buf;  // [pair][E0][E1][E2] complex work array
  // Embedding sizes for a grid; `slice` receives the profile at the wrapped
  // offsets of the embedded torus (row-major over E), filled by the caller.
  void init(int d, const int* dims);
  // Offset (in nodes) of embedded index i along axis j: i ≤ E/2 ? i : i − E.
  int wrap(int j, int i) const { return i <= E[j] / 2 ? i : i - E[j]; }
  void build(const std::vector<double>& slice, cudaStream_t s);
  // W = K_UU U for nrhs RHS-minor columns ([M][nrhs], node row-major).
  void apply(const double* U, double* W, int nrhs, cudaStream_t s) const;
};

// Our embedding's slice from the reference's (2(m_j − 1) nodes per axis,
// row-major): offsets |w_j| ≤ m_j − 1 copied, the rest (never reached by a
// corner product) zero.
std::vector<double> slice_from_reference(const KuuFft& f, const std::vector<double>& slice_ref);

// Smallest eigenvalue of the reference's own embedding (size 2(m_j − 1) per
// axis, GridKernelOperator::min_embedding_eigenvalue, dski.hpp:40-43): the
// even slice's real DFT, by separable cosine sums on the host (long double).
double min_embedding_eigenvalue_host(int d, const int* dims, const std::vector<double>& slice_ref);

}  // namespace gk
