// gk_kernels.cuh — device helpers and launchers shared across translation
// units of libgk_b200.
#pragma once

#include <cuda_runtime.h>

#include "gk_common.hpp"

namespace gk {

// ---------------------------------------------------------------- stencils
// Quintic / Keys-cubic convolution weights (reference interpolation.cpp:15-57)
// evaluated on the device for test points.
__device__ __forceinline__ double d_quintic_piece(double s) {
  if (s < 1.0) return (((-25.0 * s + 63.0) * s - 35.0) * s * s * s - 15.0 * s * s + 12.0) / 12.0;
  if (s < 2.0) return (s - 2.0) * (s - 1.0) * ((25.0 * s - 114.0) * s * s + 153.0 * s - 48.0) / 24.0;
  if (s < 3.0) {
    const double t = s - 3.0;
    return -t * t * t * (s - 2.0) * (5.0 * s - 8.0) / 24.0;
  }
  return 0.0;
}
__device__ __forceinline__ double d_quintic_piece_deriv(double s) {
  if (s < 1.0) return ((((-125.0 * s + 252.0) * s - 105.0) * s - 30.0) * s) / 12.0;
  if (s < 2.0) return ((((125.0 * s - 756.0) * s + 1635.0) * s - 1470.0) * s + 450.0) / 24.0;
  if (s < 3.0) return ((((-25.0 * s + 252.0) * s - 939.0) * s + 1530.0) * s - 918.0) / 24.0;
  return 0.0;
}
template <int T>
__device__ __forceinline__ void stencil_weights(double t, double h, double* w, double* dw) {
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const double arg = t - double(k - (T == 6 ? 2 : 1));
    if (T == 6) {
      w[k] = d_quintic_piece(fabs(arg));
      dw[k] = (arg < 0.0 ? -d_quintic_piece_deriv(-arg) : d_quintic_piece_deriv(arg)) / h;
    } else {
      const double a = fabs(arg);
      w[k] = a < 1.0 ? ((1.5 * a - 2.5) * a) * a + 1.0 : (a < 2.0 ? ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0 : 0.0);
      const double v = a < 1.0 ? (4.5 * a - 5.0) * a : (a < 2.0 ? (-1.5 * a + 5.0) * a - 4.0 : 0.0);
      dw[k] = (arg < 0.0 ? -v : v) / h;
    }
  }
}

// ---------------------------------------------------------------- launchers
// Y[p][a][q] = Σ_c t[|a-c|] X[p][c][q]   (p < P, a,c < M, q < Q); entries
// with |a-c| >= band are skipped tile-wise (band = M disables skipping).
void toeplitz_mode(const double* t, int M, int band, i64 P, i64 Q, const double* X, double* Y,
                   cudaStream_t s);

// Column reductions over RHS-minor blocks (rows × nrhs), deterministic:
// out[b] = Σ_r x[r,b]·y[r,b]  (y = null → Σ x²)
void col_dot(const double* x, const double* y, i64 rows, int nrhs, double* out, double* partial,
             cudaStream_t s);

// External column-major block <-> internal RHS-minor block with row map ext
// (internal row -> external row; null = identity).
void to_internal(const i64* ext, i64 N, const double* V, i64 ldv, double* I, int nrhs, cudaStream_t s);
void from_internal(const i64* ext, i64 N, const double* I, double* V, i64 ldv, int nrhs, cudaStream_t s);

inline int blocks_for(i64 items, int threads = 256, int cap = 148 * 16) {
  i64 b = (items + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return int(b);
}

}  // namespace gk
