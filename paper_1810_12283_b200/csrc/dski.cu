#include <chrono>
#include <cstdio>
#include <cstdlib>
// dski.cu — the D-SKI operator on B200 (reference dski.cpp:174-304,
// interpolation.cpp:59-97,212-266).
//
//   K∇_DSKI v = B K_UU B^T v + diag(σ1² I_n, σ2² I_nd) v,  B = [W; ∂W_1; …; ∂W_d]
//
// Design:
//  * Points are sorted once by stencil base cell. Per sorted point we keep the
//    base multi-index and the d 1-D quintic (or cubic) weight/derivative
//    stencils (interpolation.cpp:66-97); W/∂W are never stored as CSR.
//  * B^T (scatter) is an atomic-free gather by grid node: every (node, rhs)
//    item walks the T^(d-1) runs of candidate base cells whose points cover it
//    (contiguous in the sorted order along the last axis) — deterministic
//    order, no atomics.
//  * K_UU is the Kronecker product of per-axis symmetric Toeplitz matrices
//    (SE is separable: profile(o) = s² Π_j exp(-o_j²/2ℓ²)), applied mode by
//    mode as register-tiled fp64 GEMMs with the Toeplitz tile generated from
//    the 1-D sequence. This is the same linear map as the reference's
//    circulant-embedding FFT (dski.cpp:146-166) — the embedding reproduces
//    the Toeplitz product exactly — evaluated without the 2^d-fold
//    embedding.
//  * B (gather) + noise is one kernel, sum-factorised across axes.
// All vectors are in the internal layout: rows = g*n + sorted point,
// right-hand sides innermost.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <sstream>

#include "fused2d.hpp"
#include "kuu_fft.hpp"
#include "lean2d.hpp"

#include <cub/cub.cuh>
#include "gk_common.hpp"
#include "gk_kernels.cuh"

namespace gk {

namespace {

// ---------------------------------------------------------------- host stencil
// interpolation.cpp:15-57: quintic (C², degree-4 reproduction) and Keys cubic.
inline double quintic_piece(double s) {
  if (s < 1.0) return (((-25.0 * s + 63.0) * s - 35.0) * s * s * s - 15.0 * s * s + 12.0) / 12.0;
  if (s < 2.0) return (s - 2.0) * (s - 1.0) * ((25.0 * s - 114.0) * s * s + 153.0 * s - 48.0) / 24.0;
  if (s < 3.0) {
    const double t = s - 3.0;
    return -t * t * t * (s - 2.0) * (5.0 * s - 8.0) / 24.0;
  }
  return 0.0;
}
inline double quintic_piece_deriv(double s) {
  if (s < 1.0) return ((((-125.0 * s + 252.0) * s - 105.0) * s - 30.0) * s) / 12.0;
  if (s < 2.0) return ((((125.0 * s - 756.0) * s + 1635.0) * s - 1470.0) * s + 450.0) / 24.0;
  if (s < 3.0) return ((((-25.0 * s + 252.0) * s - 939.0) * s + 1530.0) * s - 918.0) / 24.0;
  return 0.0;
}
inline double cubic_val(double s) {
  const double a = std::fabs(s);
  if (a < 1.0) return ((1.5 * a - 2.5) * a) * a + 1.0;
  if (a < 2.0) return ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0;
  return 0.0;
}
inline double cubic_der(double s) {
  const double sg = s < 0.0 ? -1.0 : 1.0;
  const double a = std::fabs(s);
  double v = 0.0;
  if (a < 1.0) v = (4.5 * a - 5.0) * a;
  else if (a < 2.0) v = (-1.5 * a + 5.0) * a - 4.0;
  return sg * v;
}

// One axis of one point: base node, value and derivative weights (÷h).
void axis_weights(double x, double origin, double h, int m, int T, i64 point, int axis, int* base,
                  double* w, double* dw) {
  const double s = (x - origin) / h;
  const i64 cell = static_cast<i64>(std::floor(s));
  const double t = s - static_cast<double>(cell);
  const i64 b = cell - (T == 6 ? 2 : 1);
  if (!(t >= 0.0 && t < 1.0) || b < 0 || b + T > m) {
    std::ostringstream msg;
    msg << "point " << point << " (coordinate " << x << " on axis " << axis
        << ") lies outside the interior of the grid";
    fail(GK_ERR_OUT_OF_GRID, msg.str(), point);
  }
  for (int k = 0; k < T; ++k) {
    const double arg = t - static_cast<double>(k - (T == 6 ? 2 : 1));
    if (T == 6) {
      w[k] = quintic_piece(std::fabs(arg));
      dw[k] = (arg < 0.0 ? -quintic_piece_deriv(-arg) : quintic_piece_deriv(arg)) / h;
    } else {
      w[k] = cubic_val(arg);
      dw[k] = cubic_der(arg) / h;
    }
  }
  *base = static_cast<int>(b);
}

}  // namespace

// ================================================================ kernels
struct DskiView {
  int d, T, G;  // dims, taps, groups (0 or d)
  int m[3];     // grid nodes per axis
  int nb[3];    // base cells per axis (m - T + 1)
  i64 n, M;
  const int4* base;      // [n] sorted
  const double* wts;     // [n][d][2][T]
  const double2* wd;     // [n][d][T] (w, dw) pairs: one 16-byte load per tap
  const int* cell_start; // [ncells + 1]
  double nv2, ng2;
};

template <int D, int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter(DskiView op, const double* __restrict__ v,
                                                 double* __restrict__ u, int nrhs) {
  constexpr int STRIDE = D * 2 * T;
  const i64 items = op.M * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items;
       it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it % nrhs);
    i64 node = it / nrhs;
    int k[3];
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      k[j] = int(node % op.m[j]);
      node /= op.m[j];
    }
    double acc = 0.0;
    const int kl = k[D - 1];
    const int bl_lo = max(0, kl - (T - 1));
    const int bl_hi = min(op.nb[D - 1] - 1, kl);
    if (bl_lo <= bl_hi) {
      // leading axes: T^(D-1) combinations of offsets t_0..t_{D-2}
      constexpr int LEAD = (D == 1) ? 1 : (D == 2 ? T : T * T);
      for (int lc = 0; lc < LEAD; ++lc) {
        int t0 = 0, t1 = 0;
        i64 cell_row = 0;
        bool ok = true;
        if constexpr (D >= 2) {
          t0 = (D == 2) ? lc : lc / T;
          const int b0 = k[0] - t0;
          ok = b0 >= 0 && b0 < op.nb[0];
          cell_row = b0;
          if constexpr (D == 3) {
            t1 = lc % T;
            const int b1 = k[1] - t1;
            ok = ok && b1 >= 0 && b1 < op.nb[1];
            cell_row = cell_row * op.nb[1] + b1;
          }
        }
        if (!ok) continue;
        const i64 c0 = cell_row * op.nb[D - 1];
        const int s_lo = __ldg(op.cell_start + c0 + bl_lo);
        const int s_hi = __ldg(op.cell_start + c0 + bl_hi + 1);
        for (int s = s_lo; s < s_hi; ++s) {
          const int4 bs = __ldg(op.base + s);
          const double* p = op.wts + (i64)s * STRIDE;
          const int tl = kl - (D == 1 ? bs.x : (D == 2 ? bs.y : bs.z));
          if constexpr (D == 1) {
            const double w0 = __ldg(p + tl);
            if constexpr (GRAD) {
              const double dw0 = __ldg(p + T + tl);
              acc += w0 * __ldg(v + (i64)s * nrhs + b) + dw0 * __ldg(v + ((i64)op.n + s) * nrhs + b);
            } else {
              acc += w0 * __ldg(v + (i64)s * nrhs + b);
            }
          } else if constexpr (D == 2) {
            const double w0 = __ldg(p + t0), w1 = __ldg(p + 2 * T + tl);
            const double v0 = __ldg(v + (i64)s * nrhs + b);
            if constexpr (GRAD) {
              const double dw0 = __ldg(p + T + t0), dw1 = __ldg(p + 3 * T + tl);
              const double v1 = __ldg(v + ((i64)op.n + s) * nrhs + b);
              const double v2 = __ldg(v + (2 * (i64)op.n + s) * nrhs + b);
              acc += w1 * (v0 * w0 + v1 * dw0) + dw1 * (v2 * w0);
            } else {
              acc += w0 * w1 * v0;
            }
          } else {
            const double w0 = __ldg(p + t0), w1 = __ldg(p + 2 * T + t1), w2 = __ldg(p + 4 * T + tl);
            const double v0 = __ldg(v + (i64)s * nrhs + b);
            if constexpr (GRAD) {
              const double dw0 = __ldg(p + T + t0), dw1 = __ldg(p + 3 * T + t1),
                           dw2 = __ldg(p + 5 * T + tl);
              const double v1 = __ldg(v + ((i64)op.n + s) * nrhs + b);
              const double v2 = __ldg(v + (2 * (i64)op.n + s) * nrhs + b);
              const double v3 = __ldg(v + (3 * (i64)op.n + s) * nrhs + b);
              // w2*(w1*(v0 w0 + v1 dw0) + dw1*(v2 w0)) + dw2*(w1*(v3 w0))
              acc += w2 * (w1 * (v0 * w0 + v1 * dw0) + dw1 * (v2 * w0)) + dw2 * (w1 * (v3 * w0));
            } else {
              acc += w0 * w1 * w2 * v0;
            }
          }
        }
      }
    }
    u[it] = acc;
  }
}

template <int D, int T, bool GRAD>
__global__ void __launch_bounds__(256) k_gather(DskiView op, const double* __restrict__ w,
                                                const double* __restrict__ v,
                                                double* __restrict__ out, int nrhs, int noise) {
  constexpr int STRIDE = D * 2 * T;
  const i64 items = op.n * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items;
       it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it % nrhs);
    const i64 s = it / nrhs;
    const int4 bs = __ldg(op.base + s);
    const double* p = op.wts + s * STRIDE;
    double o[D + 1];
#pragma unroll
    for (int g = 0; g <= D; ++g) o[g] = 0.0;
    if constexpr (D == 1) {
      const double* wr = w + (i64)bs.x * nrhs + b;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double uu = __ldg(wr + (i64)t * nrhs);
        o[0] += __ldg(p + t) * uu;
        if constexpr (GRAD) o[1] += __ldg(p + T + t) * uu;
      }
    } else if constexpr (D == 2) {
      double w1[T], dw1[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        w1[t] = __ldg(p + 2 * T + t);
        if constexpr (GRAD) dw1[t] = __ldg(p + 3 * T + t);
      }
#pragma unroll
      for (int t0 = 0; t0 < T; ++t0) {
        const double* wr = w + ((i64)(bs.x + t0) * op.m[1] + bs.y) * nrhs + b;
        double r = 0.0, q = 0.0;
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) {
          const double uu = __ldg(wr + (i64)t1 * nrhs);
          r += w1[t1] * uu;
          if constexpr (GRAD) q += dw1[t1] * uu;
        }
        const double w0 = __ldg(p + t0);
        o[0] += w0 * r;
        if constexpr (GRAD) {
          o[1] += __ldg(p + T + t0) * r;
          o[2] += w0 * q;
        }
      }
    } else {
      double w2[T], dw2[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        w2[t] = __ldg(p + 4 * T + t);
        if constexpr (GRAD) dw2[t] = __ldg(p + 5 * T + t);
      }
#pragma unroll
      for (int t0 = 0; t0 < T; ++t0) {
        double R0 = 0.0, R1 = 0.0, R2 = 0.0;  // value, ∂1 (axis 1), ∂2 (axis 2) partials
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) {
          const double* wr = w + (((i64)(bs.x + t0) * op.m[1] + bs.y + t1) * op.m[2] + bs.z) * nrhs + b;
          double r = 0.0, q = 0.0;
#pragma unroll
          for (int t2 = 0; t2 < T; ++t2) {
            const double uu = __ldg(wr + (i64)t2 * nrhs);
            r += w2[t2] * uu;
            if constexpr (GRAD) q += dw2[t2] * uu;
          }
          const double w1 = __ldg(p + 2 * T + t1);
          R0 += w1 * r;
          if constexpr (GRAD) {
            R1 += __ldg(p + 3 * T + t1) * r;
            R2 += w1 * q;
          }
        }
        const double w0 = __ldg(p + t0);
        o[0] += w0 * R0;
        if constexpr (GRAD) {
          o[1] += __ldg(p + T + t0) * R0;
          o[2] += w0 * R1;
          o[3] += w0 * R2;
        }
      }
    }
    constexpr int NG = GRAD ? D + 1 : 1;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const i64 idx = ((i64)g * op.n + s) * nrhs + b;
      double val = o[g];
      if (noise) val += (g == 0 ? op.nv2 : op.ng2) * __ldg(v + idx);
      out[idx] = val;
    }
  }
}

// ---------------------------------------------------------------- lean kernels
// 2-D thread blocks: x = right-hand sides (lanes), y = nodes/points. One item
// per thread, 32-bit index math, no per-item divisions by nrhs; for nrhs ≥ 32
// a warp is one node/point × 32 RHS, so all control flow is warp-uniform and
// stencil loads are broadcasts.
template <int D, int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter_lean(DskiView op, const double* __restrict__ v,
                                                      double* __restrict__ u, int nrhs) {
  const int node = blockIdx.x * blockDim.y + threadIdx.y;
  const int b = blockIdx.y * blockDim.x + threadIdx.x;
  if (node >= op.M || b >= nrhs) return;
  constexpr int REC = D * 2 * T;
  int k[3];
  {
    int rem = node;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      k[j] = rem % op.m[j];
      rem /= op.m[j];
    }
  }
  const int kl = k[D - 1];
  const int lo = max(0, kl - (T - 1)), hi = min(op.nb[D - 1] - 1, kl);
  const size_t gstride = (size_t)op.n * nrhs;
  const double* vb = v + b;
  double acc = 0.0;
  if (lo <= hi) {
    constexpr int LEAD = (D == 1) ? 1 : (D == 2 ? T : T * T);
#pragma unroll 1
    for (int lc = 0; lc < LEAD; ++lc) {
      int t0 = 0, t1 = 0, crow = 0;
      if constexpr (D >= 2) {
        t0 = (D == 2) ? lc : lc / T;
        const int b0 = k[0] - t0;
        if (b0 < 0 || b0 >= op.nb[0]) continue;
        crow = b0;
        if constexpr (D == 3) {
          t1 = lc % T;
          const int b1 = k[1] - t1;
          if (b1 < 0 || b1 >= op.nb[1]) continue;
          crow = crow * op.nb[1] + b1;
        }
      }
      const int cb = crow * op.nb[D - 1];
      const int s_lo = __ldg(op.cell_start + cb + lo);
      const int s_hi = __ldg(op.cell_start + cb + hi + 1);
      for (int s = s_lo; s < s_hi; ++s) {
        const double* rec = op.wts + (size_t)s * REC;
        const int4 bs = __ldg(op.base + s);
        const int tl = kl - (D == 1 ? bs.x : (D == 2 ? bs.y : bs.z));
        const double* vs = vb + (size_t)s * nrhs;
        const double v0 = __ldg(vs);
        if constexpr (D == 1) {
          acc += __ldg(rec + tl) * v0;
          if constexpr (GRAD) acc += __ldg(rec + T + tl) * __ldg(vs + gstride);
        } else if constexpr (D == 2) {
          const double w0 = __ldg(rec + t0), w1 = __ldg(rec + 2 * T + tl);
          if constexpr (GRAD) {
            const double dw0 = __ldg(rec + T + t0), dw1 = __ldg(rec + 3 * T + tl);
            const double v1 = __ldg(vs + gstride), v2 = __ldg(vs + 2 * gstride);
            acc += w1 * (v0 * w0 + v1 * dw0) + dw1 * (v2 * w0);
          } else {
            acc += w0 * w1 * v0;
          }
        } else {
          const double w0 = __ldg(rec + t0), w1 = __ldg(rec + 2 * T + t1), w2 = __ldg(rec + 4 * T + tl);
          if constexpr (GRAD) {
            const double dw0 = __ldg(rec + T + t0), dw1 = __ldg(rec + 3 * T + t1), dw2 = __ldg(rec + 5 * T + tl);
            const double v1 = __ldg(vs + gstride), v2 = __ldg(vs + 2 * gstride), v3 = __ldg(vs + 3 * gstride);
            acc += w2 * (w1 * (v0 * w0 + v1 * dw0) + dw1 * (v2 * w0)) + dw2 * (w1 * (v3 * w0));
          } else {
            acc += w0 * w1 * w2 * v0;
          }
        }
      }
    }
  }
  u[(size_t)node * nrhs + b] = acc;
}

// d = 3 scatter Bᵀv as node columns: warp = one (k0, k1) node column × 32 RHS
// lanes, rolling over the cells b2 along the last axis. Points are sorted by
// base cell (row-major), so for each b2 the points of the 36 covering cell
// columns (k0−t0, k1−t1, b2) are contiguous ranges; each point adds to the T
// window nodes k2 = b2 .. b2+T−1 held in registers, and node b2 is final (and
// stored) once cell b2 is done. The last axis is split into segments
// (grid.y); a segment re-reads the T−1 cells below it instead of exchanging
// halos. Each point is read by its 36 covering columns (the pull kernel read
// it once per covered node: 216×). No atomics; fixed order (deterministic).
template <int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter_col3(DskiView op, const double* __restrict__ v,
                                                      double* __restrict__ u, int nrhs, int zseg) {
  const int lane = threadIdx.x;
  const int col = blockIdx.x * blockDim.y + threadIdx.y;
  const int m1 = op.m[1], m2 = op.m[2];
  if (col >= op.m[0] * m1) return;
  const int k0 = col / m1, k1 = col - k0 * m1;
  const int z0 = blockIdx.y * zseg, z1 = min(m2, z0 + zseg);
  const int bb = blockIdx.z * 32 + lane;
  const bool bok = bb < nrhs;
  const int b = bok ? bb : 0;
  const int nb1 = op.nb[1], nb2 = op.nb[2];
  const int t0lo = max(0, k0 - (op.nb[0] - 1)), t0hi = min(T - 1, k0);
  const int t1lo = max(0, k1 - (nb1 - 1)), t1hi = min(T - 1, k1);
  const size_t gs = (size_t)op.n * nrhs;
  double acc[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
  for (int b2 = max(0, z0 - (T - 1)); b2 < z1; ++b2) {
    if (b2 < nb2) {
      for (int t0 = t0lo; t0 <= t0hi; ++t0) {
        const int c0 = (k0 - t0) * nb1;
        for (int t1 = t1lo; t1 <= t1hi; ++t1) {
          const int cell = (c0 + (k1 - t1)) * nb2 + b2;
          const int s_lo = __ldg(op.cell_start + cell), s_hi = __ldg(op.cell_start + cell + 1);
          for (int s = s_lo; s < s_hi; ++s) {
            const double2* wd = op.wd + (size_t)s * 3 * T;
            const double2 a0 = __ldg(wd + t0), a1 = __ldg(wd + T + t1);
            const double* vs = v + (size_t)s * nrhs + b;
            const double v0 = __ldg(vs);
            double A, Bc = 0.0;
            if constexpr (GRAD) {
              const double v1 = __ldg(vs + gs), v2 = __ldg(vs + 2 * gs), v3 = __ldg(vs + 3 * gs);
              A = a1.x * (v0 * a0.x + v1 * a0.y) + a1.y * (v2 * a0.x);
              Bc = a1.x * (v3 * a0.x);
            } else {
              A = a1.x * a0.x * v0;
            }
#pragma unroll
            for (int t2 = 0; t2 < T; ++t2) {
              const double2 a2 = __ldg(wd + 2 * T + t2);
              acc[t2] += GRAD ? a2.x * A + a2.y * Bc : a2.x * A;
            }
          }
        }
      }
    }
    if (b2 >= z0 && bok) u[((size_t)col * m2 + b2) * nrhs + bb] = acc[0];
#pragma unroll
    for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
    acc[T - 1] = 0.0;
  }
}

// d = 3 scatter from the per-column sorted point lists (built once with the
// operator): warp = (node column, z-segment, 32 RHS lanes). Entries are taken
// 32 at a time: first lane-parallel — lane l turns entry l's stencil weights
// into the coefficients α0 = w1·w0, α1 = w1·∂w0, α2 = ∂w1·w0 and the T axis-2
// (w, ∂w) pairs, kept in per-warp shared memory — then the warp walks the
// chunk with RHS lanes, where only the v loads (independent across entries)
// touch memory, and the rolling window emits node b2 when the walk reaches a
// larger base b2. No atomics; fixed order (deterministic).
constexpr int L3_WARPS = 4;
template <int T, bool GRAD>
__global__ void __launch_bounds__(32 * L3_WARPS) k_scatter_list3(DskiView op, const int2* __restrict__ list,
                                                                const int* __restrict__ cstart,
                                                                const int* __restrict__ cseg, int nseg, int zseg,
                                                                const double* __restrict__ v, double* __restrict__ u,
                                                                int nrhs) {
  constexpr int NC = 3 + 2 * T;  // α0, α1, α2, (w2, ∂w2) × T
  __shared__ double coef[L3_WARPS][32][NC + 1];
  __shared__ int cpt[L3_WARPS][32], cmeta[L3_WARPS][32];
  const int lane = threadIdx.x, wy = threadIdx.y;
  const int col = blockIdx.x * blockDim.y + wy;
  const int m2 = op.m[2];
  if (col >= op.m[0] * op.m[1]) return;
  const int seg = blockIdx.y;
  const int z0 = seg * zseg, z1 = min(m2, z0 + zseg);
  const int bb = blockIdx.z * 32 + lane;
  const bool bok = bb < nrhs;
  const int b = bok ? bb : 0;
  const size_t gs = (size_t)op.n * nrhs;
  double acc[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
  int cur = max(0, z0 - (T - 1));  // acc[i] <-> node cur + i
  double* ucol = u + (size_t)col * m2 * nrhs + bb;
  const int e_end = __ldg(cstart + col + 1);
  bool done = false;
  for (int e0 = __ldg(cseg + col * nseg + seg); e0 < e_end && !done; e0 += 32) {
    const int cnt = min(32, e_end - e0);
    // phase 1: lane l prepares entry e0 + l
    if (lane < cnt) {
      const int2 me = __ldg(list + e0 + lane);
      const int t0 = (me.y >> 4) & 15, t1 = me.y & 15;
      const double2* wd = op.wd + (size_t)me.x * 3 * T;
      const double2 a0 = __ldg(wd + t0), a1 = __ldg(wd + T + t1);
      double* c = coef[wy][lane];
      c[0] = a1.x * a0.x;
      c[1] = a1.x * a0.y;
      c[2] = a1.y * a0.x;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double2 a2 = __ldg(wd + 2 * T + t);
        c[3 + 2 * t] = a2.x;
        c[4 + 2 * t] = a2.y;
      }
      cpt[wy][lane] = me.x;
      cmeta[wy][lane] = me.y;
    }
    __syncwarp();
    // phase 2: the walk
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const int meta = cmeta[wy][j];
      const int b2 = meta >> 8;
      if (b2 >= z1) {
        done = true;
        break;
      }
      const double* vs = v + (size_t)cpt[wy][j] * nrhs + b;
      const double* c = coef[wy][j];
      const double v0 = __ldg(vs);
      double A, Bc = 0.0;
      if constexpr (GRAD) {
        const double v1 = __ldg(vs + gs), v2 = __ldg(vs + 2 * gs), v3 = __ldg(vs + 3 * gs);
        A = c[0] * v0 + c[1] * v1 + c[2] * v2;
        Bc = c[0] * v3;
      } else {
        A = c[0] * v0;
      }
      while (cur < b2) {
        if (cur >= z0 && bok) ucol[(size_t)cur * nrhs] = acc[0];
#pragma unroll
        for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
        acc[T - 1] = 0.0;
        ++cur;
      }
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] += GRAD ? c[3 + 2 * t] * A + c[4 + 2 * t] * Bc : c[3 + 2 * t] * A;
    }
    __syncwarp();
  }
  while (cur < z1) {
    if (cur >= z0 && bok) ucol[(size_t)cur * nrhs] = acc[0];
#pragma unroll
    for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
    acc[T - 1] = 0.0;
    ++cur;
  }
}

// d = 3 scatter over balanced work units (warp = one unit × 32 RHS lanes):
// same rolling window as k_scatter_list3, but each unit carries ~64 list
// entries, so surface-concentrated point sets (C3) do not leave a few
// columns with all the work. u must be zeroed first.
template <int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter_units3(DskiView op, const int2* __restrict__ list,
                                                        const int* __restrict__ cstart,
                                                        const int4* __restrict__ units, int nunits,
                                                        const double* __restrict__ v, double* __restrict__ u,
                                                        int nrhs) {
  const int lane = threadIdx.x;
  const int ui = blockIdx.x * blockDim.y + threadIdx.y;
  if (ui >= nunits) return;
  const int4 un = __ldg(units + ui);
  const int col = un.x, za = un.y, zb = un.z;
  const int m2 = op.m[2];
  const int bb = blockIdx.y * 32 + lane;
  const bool bok = bb < nrhs;
  const int b = bok ? bb : 0;
  const size_t gs = (size_t)op.n * nrhs;
  double acc[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
  int cur = max(0, za - (T - 1));
  double* ucol = u + (size_t)col * m2 * nrhs + bb;
  const int e_end = __ldg(cstart + col + 1);
  bool done = false;
  for (int e0 = un.w; e0 < e_end && !done; e0 += 32) {
    const int2 mine = e0 + lane < e_end ? __ldg(list + e0 + lane) : make_int2(0, 0x7fffff00);
    const int cnt = min(32, e_end - e0);
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const int sp = __shfl_sync(0xffffffffu, mine.x, j);
      const int meta = __shfl_sync(0xffffffffu, mine.y, j);
      const int b2 = meta >> 8, t0 = (meta >> 4) & 15, t1 = meta & 15;
      if (b2 >= zb) {
        done = true;
        break;
      }
      const double2* wd = op.wd + (size_t)sp * 3 * T;
      const double2 a0 = __ldg(wd + t0), a1 = __ldg(wd + T + t1);
      double2 a2[T];
#pragma unroll
      for (int t = 0; t < T; ++t) a2[t] = __ldg(wd + 2 * T + t);
      const double* vs = v + (size_t)sp * nrhs + b;
      const double v0 = __ldg(vs);
      double A, Bc = 0.0;
      if constexpr (GRAD) {
        const double v1 = __ldg(vs + gs), v2 = __ldg(vs + 2 * gs), v3 = __ldg(vs + 3 * gs);
        A = a1.x * (v0 * a0.x + v1 * a0.y) + a1.y * (v2 * a0.x);
        Bc = a1.x * (v3 * a0.x);
      } else {
        A = a1.x * a0.x * v0;
      }
      while (cur < b2) {
        if (cur >= za && bok) ucol[(size_t)cur * nrhs] = acc[0];
#pragma unroll
        for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
        acc[T - 1] = 0.0;
        ++cur;
      }
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] += GRAD ? a2[t].x * A + a2[t].y * Bc : a2[t].x * A;
    }
  }
  while (cur < zb) {
    if (cur >= za && bok) ucol[(size_t)cur * nrhs] = acc[0];
#pragma unroll
    for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
    acc[T - 1] = 0.0;
    ++cur;
  }
}

// d = 3 scatter over node-column TILES ("per-grid-tile sorting of points"):
// a CTA owns a TB×TB tile of node columns × a z-range [za, zb) × RC
// right-hand sides, one thread per (column, RHS). The points whose stencils
// reach the tile are listed once per tile in last-axis base-cell order (built
// with the operator); chunks of E of them — base, the three (w, ∂w) stencils
// and the 4 value/derivative rows — are staged in shared memory by cp.async
// (double-buffered), and every thread walks the same chunk: a point that
// covers its column adds its T contributions to the thread's rolling z
// window, which emits node z when the walk passes base cell z. A point's v
// rows are read once per tile instead of once per column (36× for T = 6).
// Fixed order, no atomics: deterministic. u must be fully written by the
// units (they partition [0, m2) for every tile).
constexpr int B3_E = 32;
template <int T, bool GRAD>
__global__ void __launch_bounds__(1024, 1) k_scatter_tile3(DskiView op, const int* __restrict__ list,
                                                          const int4* __restrict__ units, int TB, int RC,
                                                          int tiles1, const double* __restrict__ v,
                                                          double* __restrict__ u, int nrhs) {
  extern __shared__ __align__(16) double b3_sm[];
  constexpr int G = GRAD ? 4 : 1;
  const int4 un = __ldg(units + blockIdx.x);
  const int tile = un.x, za = un.y & 0xffff, zb = un.y >> 16, e_lo = un.z, e_hi = un.w;
  const int K0 = (tile / tiles1) * TB, K1 = (tile % tiles1) * TB;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int r = tid % RC, c = tid / RC;
  const int k0 = K0 + c / TB, k1 = K1 + c % TB;
  const int rc0 = blockIdx.y * RC;
  const bool active = c < TB * TB && k0 < op.m[0] && k1 < op.m[1] && rc0 + r < nrhs;
  const int m2 = op.m[2];
  const size_t gs = (size_t)op.n * nrhs;
  // stage buffers: [2][E] int4 base | [2][E][3T] double2 | [2][G][E][RC] double
  int4* sb = reinterpret_cast<int4*>(b3_sm);
  double2* sw = reinterpret_cast<double2*>(sb + 2 * B3_E);
  double* sv = reinterpret_cast<double*>(sw + 2 * B3_E * 3 * T);
  const int rcn = min(RC, nrhs - rc0);
  auto issue = [&](int e0, int buf) {
    const int cnt = min(B3_E, e_hi - e0);
    int4* db = sb + buf * B3_E;
    double2* dw = sw + buf * B3_E * 3 * T;
    double* dv = sv + (size_t)buf * G * B3_E * RC;
    for (int q = tid; q < cnt * (1 + 3 * T); q += nthr) {
      const int j = q / (1 + 3 * T), k = q - j * (1 + 3 * T);
      const int sp = __ldg(list + e0 + j);
      if (k == 0) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(db + j))),
                     "l"(op.base + sp)
                     : "memory");
      } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(dw + j * 3 * T + k - 1))),
                     "l"(op.wd + (size_t)sp * 3 * T + k - 1)
                     : "memory");
      }
    }
    for (int q = tid; q < cnt * G * rcn; q += nthr) {
      const int j = q / (G * rcn), rest = q - j * (G * rcn), g = rest / rcn, rr = rest - g * rcn;
      const int sp = __ldg(list + e0 + j);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(
                       __cvta_generic_to_shared(dv + ((size_t)g * B3_E + j) * RC + rr))),
                   "l"(v + g * gs + (size_t)sp * nrhs + rc0 + rr)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
  int cur = max(0, za - (T - 1));  // acc[i] <-> node cur + i
  double* ucol = u + ((size_t)k0 * op.m[1] + k1) * m2 * nrhs + rc0 + r;
  auto emit = [&]() {
    if (cur >= za && active) ucol[(size_t)cur * nrhs] = acc[0];
#pragma unroll
    for (int i = 0; i < T - 1; ++i) acc[i] = acc[i + 1];
    acc[T - 1] = 0.0;
    ++cur;
  };
  if (e_lo < e_hi) issue(e_lo, 0);
  int buf = 0;
  for (int e0 = e_lo; e0 < e_hi; e0 += B3_E) {
    if (e0 + B3_E < e_hi) {
      issue(e0 + B3_E, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const int cnt = min(B3_E, e_hi - e0);
    const int4* B = sb + buf * B3_E;
    const double2* W = sw + buf * B3_E * 3 * T;
    const double* V = sv + (size_t)buf * G * B3_E * RC + r;
    for (int j = 0; j < cnt; ++j) {
      const int4 b = B[j];
      while (cur < b.z) emit();
      const int t0 = k0 - b.x, t1 = k1 - b.y;
      if (active && unsigned(t0) < unsigned(T) && unsigned(t1) < unsigned(T)) {
        const double2* w = W + j * 3 * T;
        const double2 a0 = w[t0], a1 = w[T + t1];
        const double v0 = V[j * RC];
        double A, Bc = 0.0;
        if constexpr (GRAD) {
          const double v1 = V[(B3_E + j) * RC], v2 = V[(2 * B3_E + j) * RC], v3 = V[(3 * B3_E + j) * RC];
          A = a1.x * (v0 * a0.x + v1 * a0.y) + a1.y * (v2 * a0.x);
          Bc = a1.x * (v3 * a0.x);
        } else {
          A = a1.x * a0.x * v0;
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const double2 a2 = w[2 * T + t];
          acc[t] += GRAD ? a2.x * A + a2.y * Bc : a2.x * A;
        }
      }
    }
    __syncthreads();  // buffer `buf` free for the chunk after next
    buf ^= 1;
  }
  while (cur < zb) emit();
}

// d = 1 scatter: CTA per (node, RHS). The points covering node k (base cells
// k−T+1 .. k) are ONE contiguous range of the sorted order; 256 threads stride
// over it and reduce in a fixed shared-memory tree (deterministic). The pull
// kernel gave a whole node to one thread — 100 threads for a 100-node leaf
// grid (the D-SKIP leaves).
template <int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter_1d(DskiView op, const double* __restrict__ v,
                                                    double* __restrict__ u, int nrhs) {
  __shared__ double red[256];
  const int k = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int nb = op.nb[0];
  const int clo = max(0, k - (T - 1)), chi = min(nb - 1, k);
  double acc = 0.0;
  if (clo <= chi) {
    const int s_lo = __ldg(op.cell_start + clo), s_hi = __ldg(op.cell_start + chi + 1);
    const size_t gs = (size_t)op.n * nrhs;
    for (int sp = s_lo + tid; sp < s_hi; sp += 256) {
      const int tl = k - __ldg(op.base + sp).x;
      const double2 a = __ldg(op.wd + (size_t)sp * T + tl);
      const double* vs = v + (size_t)sp * nrhs + b;
      acc += a.x * __ldg(vs);
      if constexpr (GRAD) acc += a.y * __ldg(vs + gs);
    }
  }
  red[tid] = acc;
  __syncthreads();
#pragma unroll
  for (int w = 128; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) u[(size_t)k * nrhs + b] = red[0];
}

template <int D, int T, bool GRAD>
__global__ void __launch_bounds__(256) k_gather_lean(DskiView op, const double* __restrict__ w,
                                                     const double* __restrict__ v, double* __restrict__ out,
                                                     int nrhs, int noise) {
  const int s = blockIdx.x * blockDim.y + threadIdx.y;
  const int b = blockIdx.y * blockDim.x + threadIdx.x;
  if (s >= op.n || b >= nrhs) return;
  constexpr int REC = D * 2 * T;
  const double* rec = op.wts + (size_t)s * REC;
  const int4 bs = __ldg(op.base + s);
  double o[D + 1];
#pragma unroll
  for (int g = 0; g <= D; ++g) o[g] = 0.0;
  if constexpr (D == 1) {
    const double* wr = w + (size_t)bs.x * nrhs + b;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const double uu = __ldg(wr + (size_t)t * nrhs);
      o[0] += __ldg(rec + t) * uu;
      if constexpr (GRAD) o[1] += __ldg(rec + T + t) * uu;
    }
  } else if constexpr (D == 2) {
    const size_t rs = (size_t)op.m[1] * nrhs;
    const double* wr = w + ((size_t)bs.x * op.m[1] + bs.y) * nrhs + b;
    double uu[T][T];
#pragma unroll
    for (int t0 = 0; t0 < T; ++t0)
#pragma unroll
      for (int t1 = 0; t1 < T; ++t1) uu[t0][t1] = __ldg(wr + t0 * rs + (size_t)t1 * nrhs);
#pragma unroll
    for (int t0 = 0; t0 < T; ++t0) {
      double r = 0.0, q = 0.0;
#pragma unroll
      for (int t1 = 0; t1 < T; ++t1) {
        r += __ldg(rec + 2 * T + t1) * uu[t0][t1];
        if constexpr (GRAD) q += __ldg(rec + 3 * T + t1) * uu[t0][t1];
      }
      const double w0 = __ldg(rec + t0);
      o[0] += w0 * r;
      if constexpr (GRAD) {
        o[1] += __ldg(rec + T + t0) * r;
        o[2] += w0 * q;
      }
    }
  } else {
    const size_t rs2 = (size_t)op.m[2] * nrhs, rs1 = (size_t)op.m[1] * rs2;
    const double* wbase = w + (((size_t)bs.x * op.m[1] + bs.y) * op.m[2] + bs.z) * nrhs + b;
#pragma unroll 1
    for (int t0 = 0; t0 < T; ++t0) {
      double R0 = 0.0, R1 = 0.0, R2 = 0.0;
#pragma unroll
      for (int t1 = 0; t1 < T; ++t1) {
        const double* wr = wbase + t0 * rs1 + t1 * rs2;
        double uu[T];
#pragma unroll
        for (int t2 = 0; t2 < T; ++t2) uu[t2] = __ldg(wr + (size_t)t2 * nrhs);
        double r = 0.0, q = 0.0;
#pragma unroll
        for (int t2 = 0; t2 < T; ++t2) {
          r += __ldg(rec + 4 * T + t2) * uu[t2];
          if constexpr (GRAD) q += __ldg(rec + 5 * T + t2) * uu[t2];
        }
        const double w1 = __ldg(rec + 2 * T + t1);
        R0 += w1 * r;
        if constexpr (GRAD) {
          R1 += __ldg(rec + 3 * T + t1) * r;
          R2 += w1 * q;
        }
      }
      const double w0 = __ldg(rec + t0);
      o[0] += w0 * R0;
      if constexpr (GRAD) {
        o[1] += __ldg(rec + T + t0) * R0;
        o[2] += w0 * R1;
        o[3] += w0 * R2;
      }
    }
  }
  constexpr int NG = GRAD ? D + 1 : 1;
  const size_t gstride = (size_t)op.n * nrhs;
  const size_t idx0 = (size_t)s * nrhs + b;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const size_t idx = idx0 + g * gstride;
    double val = o[g];
    if (noise) val += (g == 0 ? op.nv2 : op.ng2) * __ldg(v + idx);
    out[idx] = val;
  }
}

// Scatter v2: iterate candidate CELLS (base1 known from the cell index, so no
// dependent per-point base load) and read each tap's (w, dw) pair with one
// 16-byte load.
template <int D, int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter_cells(DskiView op, const double* __restrict__ v,
                                                       double* __restrict__ u, int nrhs) {
  const int node = blockIdx.x * blockDim.y + threadIdx.y;
  const int b = blockIdx.y * blockDim.x + threadIdx.x;
  if (node >= op.M || b >= nrhs) return;
  int k[3];
  {
    int rem = node;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      k[j] = rem % op.m[j];
      rem /= op.m[j];
    }
  }
  const int kl = k[D - 1];
  const int lo = max(0, kl - (T - 1)), hi = min(op.nb[D - 1] - 1, kl);
  const size_t gstride = (size_t)op.n * nrhs;
  const double* vb = v + b;
  double acc = 0.0;
  if (lo <= hi) {
    constexpr int LEAD = (D == 1) ? 1 : (D == 2 ? T : T * T);
#pragma unroll 1
    for (int lc = 0; lc < LEAD; ++lc) {
      int t0 = 0, t1 = 0, crow = 0;
      if constexpr (D >= 2) {
        t0 = (D == 2) ? lc : lc / T;
        const int b0 = k[0] - t0;
        if (b0 < 0 || b0 >= op.nb[0]) continue;
        crow = b0;
        if constexpr (D == 3) {
          t1 = lc % T;
          const int b1 = k[1] - t1;
          if (b1 < 0 || b1 >= op.nb[1]) continue;
          crow = crow * op.nb[1] + b1;
        }
      }
      const int* cs = op.cell_start + crow * op.nb[D - 1];
      int s = __ldg(cs + lo);
#pragma unroll 1
      for (int c = lo; c <= hi; ++c) {
        const int s_end = __ldg(cs + c + 1);
        const int tl = kl - c;
        for (; s < s_end; ++s) {
          const double2* wd = op.wd + (size_t)s * (D * T);
          const double* vs = vb + (size_t)s * nrhs;
          const double v0 = __ldg(vs);
          if constexpr (D == 1) {
            const double2 a = __ldg(wd + tl);
            acc += a.x * v0;
            if constexpr (GRAD) acc += a.y * __ldg(vs + gstride);
          } else if constexpr (D == 2) {
            const double2 a0 = __ldg(wd + t0), a1 = __ldg(wd + T + tl);
            if constexpr (GRAD) {
              const double v1 = __ldg(vs + gstride), v2 = __ldg(vs + 2 * gstride);
              acc += a1.x * (v0 * a0.x + v1 * a0.y) + a1.y * (v2 * a0.x);
            } else {
              acc += a0.x * a1.x * v0;
            }
          } else {
            const double2 a0 = __ldg(wd + t0), a1 = __ldg(wd + T + t1), a2 = __ldg(wd + 2 * T + tl);
            if constexpr (GRAD) {
              const double v1 = __ldg(vs + gstride), v2 = __ldg(vs + 2 * gstride), v3 = __ldg(vs + 3 * gstride);
              acc += a2.x * (a1.x * (v0 * a0.x + v1 * a0.y) + a1.y * (v2 * a0.x)) + a2.y * (a1.x * (v3 * a0.x));
            } else {
              acc += a0.x * a1.x * a2.x * v0;
            }
          }
        }
      }
    }
  }
  u[(size_t)node * nrhs + b] = acc;
}

// ---------------------------------------------------------------- d = 2 band kernels
// Gather B w (+ noise) with the grid rows a band of points needs staged in
// shared memory. CTA = (R base rows of points, chunk of BC right-hand sides).
// Points are sorted by (base0, base1), so the band's points are one
// contiguous range; their stencil records are staged in chunks of PCH.
constexpr int G2_R = 2, G2_PCH = 128;
template <int T, bool GRAD>
__global__ void __launch_bounds__(256) k_gather2d(DskiView op, const double* __restrict__ w,
                                                  const double* __restrict__ v, double* __restrict__ out,
                                                  int nrhs, int BC, int noise) {
  extern __shared__ double sm[];
  constexpr int PW = 4 * T;  // w0, dw0, w1, dw1
  const int m1 = op.m[1];
  const int row_lo = blockIdx.x * G2_R;
  const int row_hi = min(row_lo + G2_R, op.nb[0]);
  const int nrows = row_hi - row_lo + T - 1;
  const int b0 = blockIdx.y * BC;
  const int bc = min(BC, nrhs - b0);
  double* Wt = sm;                                  // [nrows][m1][BC]
  double* Pw = Wt + (size_t)nrows * m1 * BC;        // [PCH][PW]
  int* Pb = reinterpret_cast<int*>(Pw + G2_PCH * PW);  // [PCH][2]
  const int tid = threadIdx.x;
  const int tile = nrows * m1 * bc;
  for (int e = tid; e < tile; e += blockDim.x) {
    const int bb = e % bc;
    const int node = e / bc;  // (row, col) within the tile
    Wt[node * BC + bb] = __ldg(w + ((i64)row_lo * m1 + node) * nrhs + b0 + bb);
  }
  const int S0 = __ldg(op.cell_start + (i64)row_lo * op.nb[1]);
  const int S1 = __ldg(op.cell_start + (i64)row_hi * op.nb[1]);
  for (int c0 = S0; c0 < S1; c0 += G2_PCH) {
    const int cnt = min(G2_PCH, S1 - c0);
    __syncthreads();
    for (int e = tid; e < cnt * PW; e += blockDim.x) {
      const int p = e / PW, k = e % PW;
      // record layout [axis][w|dw][T]: axis0 w, axis0 dw, axis1 w, axis1 dw
      Pw[e] = __ldg(op.wts + (i64)(c0 + p) * (2 * 2 * T) + k);
    }
    for (int p = tid; p < cnt; p += blockDim.x) {
      const int4 b4 = __ldg(op.base + c0 + p);
      Pb[2 * p] = b4.x - row_lo;
      Pb[2 * p + 1] = b4.y;
    }
    __syncthreads();
    for (int it = tid; it < cnt * bc; it += blockDim.x) {
      const int p = it / bc, bb = it % bc;
      const double* pw = Pw + p * PW;
      const double* wr = Wt + ((size_t)Pb[2 * p] * m1 + Pb[2 * p + 1]) * BC + bb;
      double o0 = 0.0, o1 = 0.0, o2 = 0.0;
#pragma unroll
      for (int t0 = 0; t0 < T; ++t0) {
        double r = 0.0, q = 0.0;
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) {
          const double uu = wr[(t0 * m1 + t1) * BC];
          r += pw[2 * T + t1] * uu;
          if constexpr (GRAD) q += pw[3 * T + t1] * uu;
        }
        o0 += pw[t0] * r;
        if constexpr (GRAD) {
          o1 += pw[T + t0] * r;
          o2 += pw[t0] * q;
        }
      }
      const i64 s = c0 + p;
      const int b = b0 + bb;
      i64 idx = s * nrhs + b;
      out[idx] = o0 + (noise ? op.nv2 * __ldg(v + idx) : 0.0);
      if constexpr (GRAD) {
        idx = ((i64)op.n + s) * nrhs + b;
        out[idx] = o1 + (noise ? op.ng2 * __ldg(v + idx) : 0.0);
        idx = (2 * (i64)op.n + s) * nrhs + b;
        out[idx] = o2 + (noise ? op.ng2 * __ldg(v + idx) : 0.0);
      }
    }
  }
}

// Scatter B^T v by grid row: CTA = (node row a, chunk of BC right-hand sides).
// For each of the T base rows b0 that reach row a (t0 = a - b0 fixed), the
// row's points are staged with their combined row factors
//   P = v0 w0[t0] + v1 dw0[t0],  Q = v2 w0[t0]
// and each (node column, rhs) item sums w1[t1] P + dw1[t1] Q over the points
// whose base1 covers it — deterministic order, no atomics.
constexpr int S2_ITEMS = 8;
template <int T, bool GRAD>
__global__ void __launch_bounds__(256) k_scatter2d(DskiView op, const double* __restrict__ v,
                                                   double* __restrict__ u, int nrhs, int BC, int max_row_pts) {
  extern __shared__ double sm[];
  const int m1 = op.m[1];
  const int a = blockIdx.x;
  const int b0 = blockIdx.y * BC;
  const int bc = min(BC, nrhs - b0);
  const int NQ = GRAD ? 2 : 1;
  double* W1 = sm;                                   // [max_row_pts][2T]  (w1, dw1)
  double* PQ = W1 + (size_t)max_row_pts * 2 * T;     // [max_row_pts][NQ][BC]
  int* B1 = reinterpret_cast<int*>(PQ + (size_t)max_row_pts * NQ * BC);  // [max_row_pts]
  const int tid = threadIdx.x;
  const int items = m1 * bc;
  double acc[S2_ITEMS];
#pragma unroll
  for (int k = 0; k < S2_ITEMS; ++k) acc[k] = 0.0;
  const int brow_lo = max(0, a - (T - 1)), brow_hi = min(op.nb[0] - 1, a);
  for (int br = brow_lo; br <= brow_hi; ++br) {
    const int t0 = a - br;
    const i64 cbase = (i64)br * op.nb[1];
    const int S0 = __ldg(op.cell_start + cbase);
    const int S1 = __ldg(op.cell_start + cbase + op.nb[1]);
    const int cnt = S1 - S0;
    __syncthreads();
    for (int e = tid; e < cnt * 2 * T; e += blockDim.x) {
      const int p = e / (2 * T), k = e % (2 * T);
      W1[e] = __ldg(op.wts + (i64)(S0 + p) * (2 * 2 * T) + 2 * T + k);
    }
    for (int e = tid; e < cnt * bc; e += blockDim.x) {
      const int p = e / bc, bb = e % bc;
      const i64 s = S0 + p;
      const double* pw = op.wts + s * (2 * 2 * T);
      const double w0 = __ldg(pw + t0);
      const double v0 = __ldg(v + s * nrhs + b0 + bb);
      if constexpr (GRAD) {
        const double dw0 = __ldg(pw + T + t0);
        const double v1 = __ldg(v + ((i64)op.n + s) * nrhs + b0 + bb);
        const double v2 = __ldg(v + (2 * (i64)op.n + s) * nrhs + b0 + bb);
        PQ[(p * 2) * BC + bb] = v0 * w0 + v1 * dw0;
        PQ[(p * 2 + 1) * BC + bb] = v2 * w0;
      } else {
        PQ[p * BC + bb] = v0 * w0;
      }
    }
    for (int p = tid; p < cnt; p += blockDim.x) B1[p] = __ldg(op.base + S0 + p).y;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < S2_ITEMS; ++k) {
      const int it = tid + k * blockDim.x;
      if (it >= items) break;
      const int c = it / bc, bb = it % bc;
      const int lo = max(0, c - (T - 1)), hi = min(op.nb[1] - 1, c);
      if (lo > hi) continue;
      const int p_lo = __ldg(op.cell_start + cbase + lo) - S0;
      const int p_hi = __ldg(op.cell_start + cbase + hi + 1) - S0;
      double s = 0.0;
      for (int p = p_lo; p < p_hi; ++p) {
        const int t1 = c - B1[p];
        const double* w1 = W1 + p * 2 * T;
        if constexpr (GRAD) s += w1[t1] * PQ[(p * 2) * BC + bb] + w1[T + t1] * PQ[(p * 2 + 1) * BC + bb];
        else s += w1[t1] * PQ[p * BC + bb];
      }
      acc[k] += s;
    }
  }
#pragma unroll
  for (int k = 0; k < S2_ITEMS; ++k) {
    const int it = tid + k * blockDim.x;
    if (it >= items) break;
    const int c = it / bc, bb = it % bc;
    u[((i64)a * m1 + c) * nrhs + b0 + bb] = acc[k];
  }
}

// Diagonal via separability: for SE, Σ_ab w_a w_b k(u_a-u_b) over a
// tensor-product stencil factorises into Π_j Σ_ab c_j[a] c_j[b] t_j[|a-b|]
// (same quantity as dski.cpp:240-290's offset-table double loop).
template <int D, int T>
__global__ void k_diagonal(DskiView op, const double* __restrict__ tvec, const int* __restrict__ toff,
                           double* __restrict__ diag) {
  constexpr int STRIDE = D * 2 * T;
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < op.n; s += (i64)gridDim.x * blockDim.x) {
    const double* p = op.wts + s * STRIDE;
    double S[D][2];  // per axis: plain and derivative quadratic forms
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double* tj = tvec + toff[j];
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int a = 0; a < T; ++a)
#pragma unroll
        for (int c = 0; c < T; ++c) {
          const double kk = __ldg(tj + (a > c ? a - c : c - a));
          a0 += p[j * 2 * T + a] * p[j * 2 * T + c] * kk;
          a1 += p[j * 2 * T + T + a] * p[j * 2 * T + T + c] * kk;
        }
      S[j][0] = a0;
      S[j][1] = a1;
    }
    const int NG = op.G + 1;
    for (int g = 0; g < NG; ++g) {
      double prod = 1.0;
#pragma unroll
      for (int j = 0; j < D; ++j) prod *= S[j][g == j + 1 ? 1 : 0];
      diag[(i64)g * op.n + s] = prod + (g == 0 ? op.nv2 : op.ng2);
    }
  }
}

// Row r of the operator (dski.cpp:292-304) via separability: K_UU applied to
// the tensor-product stencil of row r is ⊗_j α_j with α_j = T_j c_j (each a
// short 1-D Toeplitz–stencil product), so row entries are products of 1-D
// stencil dots. Each CTA rebuilds the α_j in shared memory.
template <int D, int T>
__device__ __forceinline__ void row_body(const DskiView& op, const double* __restrict__ tvec,
                                         const int* __restrict__ toff, int src_s, int src_g, double* __restrict__ out) {
  extern __shared__ double alpha[];  // Σ m_j
  constexpr int STRIDE = D * 2 * T;
  const int4 sb = op.base[src_s];
  const int sbase[3] = {sb.x, sb.y, sb.z};
  const double* sp = op.wts + (i64)src_s * STRIDE;
  int aoff[3];
  int tot = 0;
  for (int j = 0; j < D; ++j) {
    aoff[j] = tot;
    tot += op.m[j];
  }
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int j = 0;
    while (j + 1 < D && idx >= aoff[j + 1]) ++j;
    const int kk = idx - aoff[j];
    const double* c = sp + j * 2 * T + (src_g == j + 1 ? T : 0);
    const double* tj = tvec + toff[j];
    double acc = 0.0;
    for (int t = 0; t < T; ++t) {
      const int off = kk - (sbase[j] + t);
      acc += tj[off < 0 ? -off : off] * c[t];
    }
    alpha[idx] = acc;
  }
  __syncthreads();
  const int NG = op.G + 1;
  const i64 items = op.n * NG;
  const i64 r_self = (i64)src_g * op.n + src_s;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int g = int(it / op.n);
    const i64 s = it % op.n;
    const int4 bs = op.base[s];
    const int bb[3] = {bs.x, bs.y, bs.z};
    const double* p = op.wts + s * STRIDE;
    double prod = 1.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double* c = p + j * 2 * T + (g == j + 1 ? T : 0);
      double dot = 0.0;
#pragma unroll
      for (int t = 0; t < T; ++t) dot += c[t] * alpha[aoff[j] + bb[j] + t];
      prod *= dot;
    }
    if (it == r_self) prod += (g == 0 ? op.nv2 : op.ng2);
    out[it] = prod;
  }
}

template <int D, int T>
__global__ void k_row(DskiView op, const double* __restrict__ tvec, const int* __restrict__ toff,
                      int src_s, int src_g, double* __restrict__ out) {
  row_body<D, T>(op, tvec, toff, src_s, src_g, out);
}

// The same row with the INTERNAL row index read from device memory (a
// device-side pivot), skipped when *active == 0: lets the pivoted Cholesky
// loop run without a host round trip per pivot.
template <int D, int T>
__global__ void k_row_dev(DskiView op, const double* __restrict__ tvec, const int* __restrict__ toff,
                          const long long* __restrict__ r_int, const int* __restrict__ active,
                          double* __restrict__ out) {
  if (!*active) return;
  const long long r = *r_int;
  row_body<D, T>(op, tvec, toff, int(r % op.n), int(r / op.n), out);
}

// Test-point stencils for prediction (gp.cpp:480-495): values/grads from a
// grid vector g (single column).
template <int D, int T>
__global__ void k_predict(DskiView op, const double* __restrict__ X, i64 nT, const double* origin3,
                          const double* h3, const double* __restrict__ g, double mean,
                          double* __restrict__ vals, double* __restrict__ grads, int* __restrict__ bad) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nT; i += (i64)gridDim.x * blockDim.x) {
    int base[3];
    double w[3][T], dw[3][T];
    bool ok = true;
    for (int j = 0; j < D; ++j) {
      const double h = h3[j];
      const double sv = (X[j * nT + i] - origin3[j]) / h;
      const double cell = floor(sv);
      const double t = sv - cell;
      const int b = int(cell) - (T == 6 ? 2 : 1);
      if (!(t >= 0.0 && t < 1.0) || b < 0 || b + T > op.m[j]) ok = false;
      base[j] = b;
      stencil_weights<T>(t, h, w[j], dw[j]);
    }
    if (!ok) {
      atomicMin(bad, int(i));
      continue;
    }
    double acc = 0.0, gr[3] = {0, 0, 0};
    if constexpr (D == 1) {
      for (int a = 0; a < T; ++a) {
        const double gv = g[base[0] + a];
        acc += w[0][a] * gv;
        gr[0] += dw[0][a] * gv;
      }
    } else if constexpr (D == 2) {
      for (int a = 0; a < T; ++a)
        for (int c = 0; c < T; ++c) {
          const double gv = g[(i64)(base[0] + a) * op.m[1] + base[1] + c];
          acc += w[0][a] * w[1][c] * gv;
          gr[0] += dw[0][a] * w[1][c] * gv;
          gr[1] += w[0][a] * dw[1][c] * gv;
        }
    } else {
      for (int a = 0; a < T; ++a)
        for (int c = 0; c < T; ++c)
          for (int e = 0; e < T; ++e) {
            const double gv = g[((i64)(base[0] + a) * op.m[1] + base[1] + c) * op.m[2] + base[2] + e];
            acc += w[0][a] * w[1][c] * w[2][e] * gv;
            gr[0] += dw[0][a] * w[1][c] * w[2][e] * gv;
            gr[1] += w[0][a] * dw[1][c] * w[2][e] * gv;
            gr[2] += w[0][a] * w[1][c] * dw[2][e] * gv;
          }
    }
    vals[i] = mean + acc;
    for (int j = 0; j < D; ++j) grads[j * nT + i] = gr[j];
  }
}

// Scatter the stencils of test points as columns of a grid block (for
// cross_covariance, gp.cpp:412-417): U[node][t] = w(point t, node).
template <int D, int T>
__global__ void k_test_stencils(DskiView op, const double* __restrict__ X, i64 nT,
                                const double* origin3, const double* h3, double* __restrict__ U,
                                int* __restrict__ bad, int dir) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nT; i += (i64)gridDim.x * blockDim.x) {
    int base[3] = {0, 0, 0};
    double w[3][T], dw[3][T];
    bool ok = true;
    for (int j = 0; j < D; ++j) {
      const double sv = (X[j * nT + i] - origin3[j]) / h3[j];
      const double cell = floor(sv);
      const double t = sv - cell;
      const int b = int(cell) - (T == 6 ? 2 : 1);
      if (!(t >= 0.0 && t < 1.0) || b < 0 || b + T > op.m[j]) ok = false;
      base[j] = b;
      stencil_weights<T>(t, h3[j], w[j], dw[j]);
    }
    if (!ok) {
      atomicMin(bad, int(i));
      continue;
    }
    int cnt = 1;
    for (int j = 0; j < D; ++j) cnt *= T;
    for (int c = 0; c < cnt; ++c) {
      int rem = c;
      i64 node = 0;
      double wt = 1.0;
      int tt[3];
      for (int j = D - 1; j >= 0; --j) {
        tt[j] = rem % T;
        rem /= T;
      }
      for (int j = 0; j < D; ++j) {
        node = node * op.m[j] + base[j] + tt[j];
        wt *= (j == dir ? dw[j] : w[j])[tt[j]];  // dir ≥ 0: ∂/∂x_dir stencil (point_stencil derivative)
      }
      U[node * nT + i] = wt;
    }
  }
}

// ================================================================ on-device point tables
// The D-SKI constructor's per-point work (DskiOperator ctor, dski.cpp:174-204;
// build_interpolation, interpolation.cpp:212-266) on the GPU: stencil base
// cells and (w, ∂w) weights per axis, a stable sort by base cell (CUB radix
// sort of (cell, point) pairs), the cell start table and the sorted-order
// copies. The weights are evaluated with explicitly rounded operations in the
// host formula's exact order (no FMA contraction), so the device tables are
// bit-identical to the host build's (tuning "devbuild" = 1 keeps the host path).
namespace {
__device__ __forceinline__ double M_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double A_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double S_(double a, double b) { return __dsub_rn(a, b); }
__device__ double dq_piece(double s) {
  if (s < 1.0) {
    const double B = S_(M_(A_(M_(-25.0, s), 63.0), s), 35.0);
    const double C = M_(M_(M_(B, s), s), s);
    const double D = M_(M_(15.0, s), s);
    return __ddiv_rn(A_(S_(C, D), 12.0), 12.0);
  }
  if (s < 2.0) {
    const double Q = S_(A_(M_(M_(S_(M_(25.0, s), 114.0), s), s), M_(153.0, s)), 48.0);
    return __ddiv_rn(M_(M_(S_(s, 2.0), S_(s, 1.0)), Q), 24.0);
  }
  if (s < 3.0) {
    const double t = S_(s, 3.0);
    return __ddiv_rn(M_(M_(M_(M_(-t, t), t), S_(s, 2.0)), S_(M_(5.0, s), 8.0)), 24.0);
  }
  return 0.0;
}
__device__ double dq_deriv(double s) {
  if (s < 1.0) return __ddiv_rn(M_(S_(M_(A_(M_(A_(M_(-125.0, s), 252.0), s), -105.0), s), 30.0), s), 12.0);
  if (s < 2.0)
    return __ddiv_rn(A_(M_(S_(M_(A_(M_(S_(M_(125.0, s), 756.0), s), 1635.0), s), 1470.0), s), 450.0), 24.0);
  if (s < 3.0)
    return __ddiv_rn(S_(M_(A_(M_(S_(M_(A_(M_(-25.0, s), 252.0), s), 939.0), s), 1530.0), s), 918.0), 24.0);
  return 0.0;
}
__device__ double dc_val(double s) {
  const double a = fabs(s);
  if (a < 1.0) return A_(M_(M_(S_(M_(1.5, a), 2.5), a), a), 1.0);
  if (a < 2.0) return A_(M_(S_(M_(A_(M_(-0.5, a), 2.5), a), 4.0), a), 2.0);
  return 0.0;
}
__device__ double dc_der(double s) {
  const double sg = s < 0.0 ? -1.0 : 1.0;
  const double a = fabs(s);
  double v = 0.0;
  if (a < 1.0) v = M_(S_(M_(4.5, a), 5.0), a);
  else if (a < 2.0) v = S_(M_(A_(M_(-1.5, a), 5.0), a), 4.0);
  return M_(sg, v);
}

struct PtGeom {
  int d, T;
  double origin[3], h[3];
  int m[3], nb[3];
};

__global__ void k_pts_weights(PtGeom g, const double* __restrict__ X, i64 n, int* __restrict__ base_o,
                              double* __restrict__ wts_o, int* __restrict__ key, int* __restrict__ bad) {
  const int STRIDE = g.d * 2 * g.T;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    long long c = 0;
    bool ok = true;
    for (int j = 0; j < g.d; ++j) {
      const double x = X[(i64)j * n + i];
      const double s = __ddiv_rn(S_(x, g.origin[j]), g.h[j]);
      const double cell = floor(s);
      const double t = S_(s, cell);
      const long long b = (long long)cell - (g.T == 6 ? 2 : 1);
      if (!(t >= 0.0 && t < 1.0) || b < 0 || b + g.T > g.m[j]) {
        ok = false;
        break;
      }
      double* w = wts_o + i * STRIDE + j * 2 * g.T;
      for (int k = 0; k < g.T; ++k) {
        const double arg = S_(t, double(k - (g.T == 6 ? 2 : 1)));
        if (g.T == 6) {
          w[k] = dq_piece(fabs(arg));
          w[g.T + k] = __ddiv_rn(arg < 0.0 ? -dq_deriv(-arg) : dq_deriv(arg), g.h[j]);
        } else {
          w[k] = dc_val(arg);
          w[g.T + k] = __ddiv_rn(dc_der(arg), g.h[j]);
        }
      }
      base_o[i * 4 + j] = int(b);
      c = c * g.nb[j] + b;
    }
    if (!ok) {
      atomicMin(bad, int(i));
      key[i] = 0;
      continue;
    }
    key[i] = int(c);
  }
}

// d = 2 scatter records of the one-launch MVM: a point's 2T (w, dw) pairs
// followed by its int4 base (fused2d.cu f2_scatter).
__global__ void k_pack_records(const double2* __restrict__ wd, const int4* __restrict__ base, i64 n, int T,
                               double2* __restrict__ rec) {
  const int RW = 2 * T + 1;
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < n; s += (i64)gridDim.x * blockDim.x) {
    for (int k = 0; k < 2 * T; ++k) rec[s * RW + k] = wd[s * 2 * T + k];
    *reinterpret_cast<int4*>(rec + s * RW + 2 * T) = base[s];
  }
}

// cstart[c] = first sorted position with key ≥ c (keys ascending).
__global__ void k_cell_start(const int* __restrict__ key, i64 n, i64 ncells, int* __restrict__ cstart) {
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < n; s += (i64)gridDim.x * blockDim.x) {
    const i64 k = key[s], prev = s ? key[s - 1] : -1;
    for (i64 c = prev + 1; c <= k; ++c) cstart[c] = int(s);
    if (s == n - 1)
      for (i64 c = k + 1; c <= ncells; ++c) cstart[c] = int(n);
  }
}

__global__ void k_gather_pts(const int* __restrict__ perm, const int* __restrict__ base_o,
                             const double* __restrict__ wts_o, i64 n, int d, int T, int G, int4* __restrict__ base_s,
                             double* __restrict__ wts_s, double2* __restrict__ wd, i64* __restrict__ ext) {
  const int STRIDE = d * 2 * T;
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < n; s += (i64)gridDim.x * blockDim.x) {
    const i64 i = perm[s];
    base_s[s] = make_int4(base_o[i * 4], d > 1 ? base_o[i * 4 + 1] : 0, d > 2 ? base_o[i * 4 + 2] : 0, 0);
    for (int e = 0; e < STRIDE; ++e) wts_s[s * STRIDE + e] = wts_o[i * STRIDE + e];
    for (int j = 0; j < d; ++j)
      for (int t = 0; t < T; ++t)
        wd[(s * d + j) * T + t] = make_double2(wts_o[i * STRIDE + j * 2 * T + t], wts_o[i * STRIDE + j * 2 * T + T + t]);
    for (int gg = 0; gg <= G; ++gg) ext[gg * n + s] = gg * n + i;
  }
}
}  // namespace

// ================================================================ operator
struct DskiOp final : Op {
  int d = 0, T = 6, G = 0;
  int m[3] = {1, 1, 1}, nb[3] = {1, 1, 1};
  i64 n = 0, M = 0;
  gk_grid grid{};
  gk_kernel kernel{};
  DevBuf<int4> base;
  DevBuf<double> wts;
  DevBuf<double2> wd;
  DevBuf<double2> rec;  // d = 2 with gradients: [n][2T+1] scatter records of the one-launch MVM (fused2d)
  DevBuf<int> cell_start;
  // Non-separable profile (spline kernel): K_UU by circulant embedding + FFT
  // (kuu_fft.cu); diagonal from the stencil-offset table, rows through K_UU.
  bool generic = false;
  std::unique_ptr<KuuFft> kfft, kfft_dl;  // value and d/dlog(ell) profiles (the latter built on first use)
  DevBuf<double> gtab;                    // profile at stencil offsets, (2T-1)^d row-major
  std::vector<double> slice_ref_h;        // caller-supplied profile slice (family 2)
  DevBuf<double> tvec;  // concatenated per-axis Toeplitz sequences (axis 0 carries s²)
  DevBuf<int> toff;
  std::vector<int> toff_h;
  std::vector<int> band;  // per-axis numerical band of the Toeplitz sequence
  // ∂/∂log ℓ of the SE profile, s² Π_j t_j(o_j) · Σ_j ρ_j² (ρ_j = o_j/ℓ): a sum of
  // d Kronecker terms, term j with axis j's sequence t_j·ρ_j² (kernels.cpp:172-188)
  DevBuf<double> tvec_dl;
  std::vector<int> band_dl;
  DevBuf<double> grid_a, grid_b;  // dlogell scratch
  // d = 3 scatter: per node column (k0, k1) the covering points sorted by
  // last-axis base cell, entries {sorted point, b2 << 8 | t0 << 4 | t1};
  // col3_start[col] and per (col, z-segment) first entry
  DevBuf<int2> col3_list;
  DevBuf<int> col3_start, col3_seg;
  int col3_zseg = 12, col3_nseg = 0;
  // balanced work units over the column lists: {col, za, zb, first entry};
  // a unit emits nodes [za, zb) of its column (nodes no point touches are 0)
  DevBuf<int4> col3_units;
  int col3_nunits = 0;
  // d = 3 gather units (k_gather_units3): {b0, b1, za, zb} cell-line runs and
  // their sorted-point ranges; zspan = the longest block z extent (zb - za + T - 1)
  DevBuf<int4> g3_units;
  DevBuf<int2> g3_range;
  int g3_nunits = 0, g3_zspan = 0;
  // d = 3 unit-push scatter: scratch node offsets per unit, and per node
  // column the entries {unit, ab} sorted by (za, unit) with per-(column,
  // 8-node z segment) first entries
  DevBuf<long long> s3_uoff;
  DevBuf<int> s3_cstart, s3_cseg;
  DevBuf<int2> s3_cent;
  // per node (column, z): [zoff, zoff+1) in zlist = scratch node offsets of
  // the blocks covering it, in (za, unit) order (k_scatter_merge3f)
  DevBuf<int> s3_zoff, s3_zlist;
  int s3_maxl = 0;
  long long s3_nodes = 0;
  int s3_nzs = 0;
  // tile scatter (k_scatter_tile3): per TB×TB tile of node columns the points
  // reaching it in base-cell order (b2 major); units {tile, za | zb << 16,
  // first entry (window halo included), end entry}
  DevBuf<int> tile3_list;
  DevBuf<int4> tile3_units;
  int tile3_nunits = 0, tile3_tb = 6, tile3_tiles1 = 0;
  int max_row_pts = 0;    // d = 2: most points sharing one base row (band kernels' staging)
  DevBuf<i64> ext;        // internal row -> external row
  std::vector<i64> perm_h, inv_h;
  DevBuf<double> origin_d, h_d;
  DevBuf<double> grid_u, grid_w, grid_t, grid_h, grid_p;  // per-MVM grid scratch (guarded by mu / caller)
  mutable DevBuf<double> s3_scratch;  // unit-push scatter blocks (s3_nodes × nrhs)
  DevBuf<int> oog;                     // out-of-grid flag of the device cross-covariance
  std::vector<int> cell_start_h;          // host copy (fused-plan sizing)
  std::vector<std::unique_ptr<Fused2dPlan>> fplans;  // one-launch d = 2 MVM plans, per nrhs
  std::vector<std::unique_ptr<Lean2dPlan>> lplans;   // lean one-launch d = 2 MVM plans, per nrhs

  Fused2dGeom geom2d() const {
    Fused2dGeom g;
    g.T = T;
    g.m0 = m[0];
    g.m1 = m[1];
    g.nb0 = nb[0];
    g.nb1 = nb[1];
    g.n = int(n);
    g.base = base.p;
    g.wd = wd.p;
    g.rec = rec.p;
    g.cell_start = cell_start.p;
    g.t0 = tvec.p + toff_h[0];
    g.t1 = tvec.p + toff_h[1];
    g.band0 = band[0];
    g.band1 = band[1];
    g.nv2 = nv2;
    g.ng2 = ng2;
    return g;
  }
  // The fused one-launch MVM applies to d = 2 with gradients (C1, C2, C4).
  Fused2dPlan* fused_plan(int nrhs) {
    if (generic || d != 2 || G != 2 || g_tuning.fused.load() != 0 || n >= (i64(1) << 31)) return nullptr;
    const int gen = g_tuning.gen.load();
    for (auto it = fplans.begin(); it != fplans.end(); ++it)
      if ((*it)->nrhs == nrhs) {
        if ((*it)->tuning_gen == gen) return (*it)->ok ? it->get() : nullptr;
        fplans.erase(it);  // knobs changed: rebuild (captured graphs held the old plan)
        ++epoch;
        break;
      }
    auto p = std::make_unique<Fused2dPlan>();
    p->tuning_gen = gen;
    fused2d_plan(geom2d(), cell_start_h, nrhs, device, *p);
    fplans.push_back(std::move(p));
    return fplans.back()->ok ? fplans.back().get() : nullptr;
  }

  // The lean one-launch MVM (lean2d.cu): d = 2 with gradients, grids up to
  // 128² and up to 64 right-hand sides. Chosen where it measured faster than
  // fused2d on B200 (tools/lean_timing.py): odd RHS counts ≥ 3 (C1 9 RHS 31.8
  // vs 33.7 µs, C2 31 RHS 56.3 vs 62.4 µs) and more than 32 RHS (C2 64 RHS
  // 74.9 vs 87.0 µs). Tuning "lean": 0 = this policy, 1 = never, 2 = always.
  Lean2dPlan* lean_plan(int nrhs) {
    const int pol = g_tuning.lean.load();
    if (generic || d != 2 || G != 2 || g_tuning.fused.load() != 0 || pol == 1 || n >= (i64(1) << 31)) return nullptr;
    if (pol == 0 && !((nrhs % 2 == 1 && nrhs >= 3) || nrhs > 32)) return nullptr;
    const int gen = g_tuning.gen.load();
    for (auto it = lplans.begin(); it != lplans.end(); ++it)
      if ((*it)->nrhs == nrhs) {
        if ((*it)->tuning_gen == gen) return (*it)->ok ? it->get() : nullptr;
        lplans.erase(it);
        ++epoch;
        break;
      }
    auto p = std::make_unique<Lean2dPlan>();
    p->tuning_gen = gen;
    lean2d_plan(geom2d(), nrhs, device, *p);
    lplans.push_back(std::move(p));
    return lplans.back()->ok ? lplans.back().get() : nullptr;
  }

  DskiView view() const {
    DskiView v;
    v.d = d;
    v.T = T;
    v.G = G;
    for (int j = 0; j < 3; ++j) {
      v.m[j] = m[j];
      v.nb[j] = nb[j];
    }
    v.n = n;
    v.M = M;
    v.base = base.p;
    v.wts = wts.p;
    v.wd = wd.p;
    v.cell_start = cell_start.p;
    v.nv2 = nv2;
    v.ng2 = ng2;
    return v;
  }

  const i64* d_ext_of_int() const override { return ext.p; }
  i64 int_of_ext(i64 r) const override {
    const i64 g = r / n, i = r % n;
    return g * n + inv_h[static_cast<size_t>(i)];
  }

  void scatter(const double* v, double* u, int nrhs, cudaStream_t s) const;
  bool scatter_band(const double* v, double* u, int nrhs, cudaStream_t s) const;
  bool gather_band(const double* w, const double* v, double* out, int nrhs, bool noise, cudaStream_t s) const;
  void kuu(const double* u, double* w, int nrhs, cudaStream_t s) const;
  void kuu_dlogell(const double* u, double* w, int nrhs, cudaStream_t s);
  void gather(const double* w, const double* v, double* out, int nrhs, bool noise, cudaStream_t s) const;

  void grow(DevBuf<double>& b, size_t count) {
    if (count > b.n) {
      b.alloc(count);
      ++epoch;  // invalidates captured MVM graphs
    }
  }
  void ensure_scratch(int nrhs) {
    if (generic && kfft && kfft->buf.n < static_cast<size_t>(kfft->Etot) * ((nrhs + 1) / 2)) {
      kfft->buf.reserve(static_cast<size_t>(kfft->Etot) * ((nrhs + 1) / 2));
      ++epoch;
    }
    grow(grid_u, static_cast<size_t>(M) * nrhs);
    grow(grid_w, static_cast<size_t>(M) * nrhs + 8);  // + 8: the one-launch gather's aligned window loads
    grow(grid_t, static_cast<size_t>(M) * nrhs);
    if (d == 2 && G == 2) grow(grid_h, static_cast<size_t>(M) * nrhs);
  }

  bool pcg_persist(PcgVecPlan& vp, const PcgVecArgs& va, double* P, double* AP, int nrhs, int iters,
                   cudaStream_t s) override {
    if (d != 2 || G != 2) return false;
    Fused2dPlan* fp = fused_plan(nrhs);
    if (!fp) return false;
    ensure_scratch(nrhs);
    if (fp->s_mode == 1) grow(grid_p, static_cast<size_t>(fp->s_nbuf) * M * nrhs);
    return fused2d_pcg_persist(geom2d(), *fp, vp, va, P, AP, grid_u.p, grid_h.p, grid_t.p, grid_w.p, grid_p.p,
                               iters, s);
  }

  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {
    ensure_scratch(nrhs);
    if (Lean2dPlan* lp = lean_plan(nrhs)) {
      grow(grid_p, static_cast<size_t>(2) * M * nrhs);
      lean2d_mvm(geom2d(), *lp, in, out, grid_p.p, grid_t.p, grid_w.p, true, s);
      return;
    }
    if (Fused2dPlan* fp = fused_plan(nrhs)) {
      if (fp->s_mode == 1) grow(grid_p, static_cast<size_t>(fp->s_nbuf) * M * nrhs);
      fused2d_mvm(geom2d(), *fp, in, out, grid_u.p, grid_h.p, grid_t.p, grid_w.p, grid_p.p, true, s);
      return;
    }
    scatter(in, grid_u.p, nrhs, s);
    kuu(grid_u.p, grid_w.p, nrhs, s);
    gather(grid_w.p, in, out, nrhs, true, s);
  }
  // The one-launch 2-D MVM split at its first grid barrier, for the grid-slab
  // sharded MVM: phase 0 scatters v into [u; h] (u2: 2·M·nrhs), phase 1 runs
  // K_UU and the gather + noise from an (all-reduced) [u; h]. False when the
  // fused plan does not apply (or uses the partial-buffer scatter).
  bool fused_split(int phase, const double* v, double* u2, double* out, int nrhs, cudaStream_t s) {
    Fused2dPlan* fp = fused_plan(nrhs);
    if (!fp || fp->s_mode != 0) return false;
    if (phase == 2) return true;  // availability query
    ensure_scratch(nrhs);
    double* h = u2 + static_cast<size_t>(M) * nrhs;
    if (phase == 0) fused2d_mvm(geom2d(), *fp, v, grid_w.p, u2, h, grid_t.p, grid_w.p, grid_p.p, true, s, 14);
    else fused2d_mvm(geom2d(), *fp, v, out, u2, h, grid_t.p, grid_w.p, grid_p.p, true, s, 1);
    return true;
  }
  void stage(int st, const double* in, double* out, int nrhs, cudaStream_t s) override {
    ensure_scratch(nrhs);
    switch (st) {
      case 0: scatter(in, out, nrhs, s); break;
      case 1: kuu(in, out, nrhs, s); break;
      case 2: gather(in, in, out, nrhs, false, s); break;
      case 3: mvm(in, out, nrhs, s); break;
      case 4: mvm_graph(in, out, nrhs, s); break;
      default: fail(GK_ERR_ARG, "unknown stage");
    }
  }
  void diagonal(double* dd, cudaStream_t s) override;
  void row(i64 r_ext, double* out, cudaStream_t s) override;
  bool row_dev(const i64* d_r_int, const int* d_active, double* out, cudaStream_t s) override;
  bool has_row_dev() const override { return !generic; }
  double min_embedding_eigenvalue() const;
};

#define GK_DISPATCH_DT(D_, T_, ...)                                   \
  do {                                                                \
    if (D_ == 1 && T_ == 6) { constexpr int D = 1, T = 6; __VA_ARGS__; } \
    else if (D_ == 2 && T_ == 6) { constexpr int D = 2, T = 6; __VA_ARGS__; } \
    else if (D_ == 3 && T_ == 6) { constexpr int D = 3, T = 6; __VA_ARGS__; } \
    else if (D_ == 1 && T_ == 4) { constexpr int D = 1, T = 4; __VA_ARGS__; } \
    else if (D_ == 2 && T_ == 4) { constexpr int D = 2, T = 4; __VA_ARGS__; } \
    else if (D_ == 3 && T_ == 4) { constexpr int D = 3, T = 4; __VA_ARGS__; } \
    else fail(GK_ERR_UNSUPPORTED, "D-SKI grid dimension must be 1, 2 or 3");  \
  } while (0)

static int grid_blocks(i64 items, int threads = 256) {
  i64 b = (items + threads - 1) / threads;
  return int(std::max<i64>(1, std::min<i64>(b, 148LL * 16)));
}

static void smem_attr(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) raise_smem_limit(fn, bytes);
}

// d = 3 gather over cell-line units (B w + noise, dski.cpp:221-226): a unit
// is a run of occupied base cells (b0, b1, [za, zb)) of one cell line; its
// points are contiguous in the sorted order and all read the node block
// [b0, b0+T) × [b1, b1+T) × [za, zb+T-1) × RHS. The CTA stages that block in
// shared memory once (36 contiguous z-runs), then every (point, RHS) task
// contracts its 6×6×6 stencil from shared memory — instead of 216 L2 reads
// per (point, RHS), one L2 read of the block per unit (C3's surface points
// pile up to ~180 per cell). Same summation order as k_gather_lean.
__device__ __forceinline__ void g3_cp8(double* s, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void g3_cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void g3_cp4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void g3_cp_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
constexpr int G3U_THREADS = 128;
// RHS columns go in chunks (blockIdx.y; chunk width cw, the last one may be
// narrower): the staged block holds one chunk, so wide RHS counts keep the
// shared footprint — and the occupancy — of a ~16-column block.
template <int T, bool GRAD, int NR = 0, bool ONE = false>  // NR > 0: the chunk width as a compile-time constant
                                                            // (immediate offsets); ONE: a single chunk (ldr == NR)
__global__ void __launch_bounds__(G3U_THREADS) k_gather_units3(DskiView op, const int4* __restrict__ units, int nunits,
                                                               const int2* __restrict__ urange,
                                                               const double* __restrict__ w,
                                                               const double* __restrict__ v,
                                                               double* __restrict__ out, int ldr_rt, int cw_rt, int noise,
                                                               int zmax, int g_tuning_d3) {
  const int ldr = (NR > 0 && ONE) ? NR : ldr_rt;
  // ldr: the RHS count (the stride of w, v, out); columns [r0, r0 + nrhs) here
  const int r0 = ONE ? 0 : blockIdx.y * cw_rt;
  const int nrhs = NR > 0 ? NR : min(cw_rt, ldr - r0);
  extern __shared__ double blk[];  // [T][T][nzb][nrhs]
  const int m1 = op.m[1], m2 = op.m[2];
  constexpr int REC = 3 * 2 * T;
  const size_t gstride = (size_t)op.n * ldr;
  const unsigned inv = (65536u + nrhs - 1) / nrhs;  // q / nrhs = (q * inv) >> 16 for q < 2048
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int4 U = __ldg(units + u);  // b0, b1, za, zb
    const int2 pr = __ldg(urange + u);
    const int za = U.z, nzb = min(U.w - U.z + T - 1, zmax);
    const int run = nzb * nrhs;  // one (k0, k1) z-run (contiguous in w when the chunk is every column)
    __syncthreads();  // the previous unit is done with the block
    // 36 contiguous z-runs (one per node column of the block), a warp per run
    for (int ab = threadIdx.x >> 5; ab < T * T; ab += G3U_THREADS / 32) {
      const int a = ab / T, b = ab - a * T;
      const double* src = w + (((size_t)(U.x + a) * m1 + (U.y + b)) * m2 + za) * ldr + r0;
      double* dst = blk + ab * run;
      // cp.async: every copy of the block in flight at once (a load→store
      // loop paid one L2 round trip per iteration)
      if (nrhs == ldr) {
        for (int q = threadIdx.x & 31; q < run; q += 32) g3_cp8(dst + q, src + q);
      } else {
        for (int q = threadIdx.x & 31; q < run; q += 32) {
          const int z = int((unsigned(q) * inv) >> 16);
          g3_cp8(dst + q, src + (size_t)z * ldr + (q - z * nrhs));
        }
      }
    }
    g3_cp_wait_all();
    __syncthreads();
    // Tasks (point, RHS). With ≥ 16 RHS the first 16·⌊nrhs/16⌋ columns of
    // every point go in blocks of 16 (a half-warp reads 16 consecutive
    // doubles of one point: conflict-free), the remaining columns RHS-major
    // (lanes over the unit's points: same cell = same address, neighbouring
    // cells = neighbouring banks). r-fastest over all nrhs (the old order)
    // put two points' runs in one half-warp: 17 RHS measured 80 µs against
    // 63.5 µs for 16.
    const int np = pr.y - pr.x;
    const int ntask = np * nrhs;
    const int rmain = (nrhs >= 16 && !(g_tuning_d3 & 2)) ? (nrhs & ~15) : 0;
    for (int t = threadIdx.x; t < ntask; t += G3U_THREADS) {
      int pl, r;
      if (t < np * rmain) {
        const int blk16 = t >> 4;  // (point, 16-column block)
        pl = blk16 / (rmain >> 4);
        r = ((blk16 - pl * (rmain >> 4)) << 4) + (t & 15);
      } else if (rmain) {
        const int tt = t - np * rmain;
        const int rr = tt / np;
        pl = tt - rr * np;
        r = rmain + rr;
      } else {
        pl = t / nrhs;
        r = t - pl * nrhs;
      }
      const int sidx = pr.x + pl;
      const double* rec = op.wts + (size_t)sidx * REC;
      const int zo = __ldg(&op.base[sidx].z) - za;
      double wr_[REC];  // the point's (w, ∂w) per axis in registers
#pragma unroll
      for (int q = 0; q < REC; ++q) wr_[q] = __ldg(rec + q);
      double o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int t0 = 0; t0 < T; ++t0) {
        double R0 = 0.0, R1 = 0.0, R2 = 0.0;
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) {
          const double* wr = blk + ((t0 * T + t1) * nzb + zo) * nrhs + r;
          double uu[T];
#pragma unroll
          for (int t2 = 0; t2 < T; ++t2) uu[t2] = wr[t2 * nrhs];
          double rr = 0.0, qq = 0.0;
#pragma unroll
          for (int t2 = 0; t2 < T; ++t2) {
            rr += wr_[4 * T + t2] * uu[t2];
            if constexpr (GRAD) qq += wr_[5 * T + t2] * uu[t2];
          }
          const double w1 = wr_[2 * T + t1];
          R0 += w1 * rr;
          if constexpr (GRAD) {
            R1 += wr_[3 * T + t1] * rr;
            R2 += w1 * qq;
          }
        }
        const double w0 = wr_[t0];
        o[0] += w0 * R0;
        if constexpr (GRAD) {
          o[1] += wr_[T + t0] * R0;
          o[2] += w0 * R1;
          o[3] += w0 * R2;
        }
      }
      constexpr int NG = GRAD ? 4 : 1;
      const size_t idx0 = (size_t)sidx * ldr + r0 + r;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const size_t idx = idx0 + g * gstride;
        double val = o[g];
        if (noise) val += (g == 0 ? op.nv2 : op.ng2) * __ldg(v + idx);
        out[idx] = val;
      }
    }
  }
}

// Few right-hand sides: a warp per unit (4 per CTA). The CTA-per-unit gather
// above runs ~10 tasks per unit at 1 RHS, leaving three of its four warps
// idle in every CTA slot; here each warp stages its unit's block with
// cp.async and runs the unit's (point, RHS) tasks alone. Same per-task
// arithmetic and order as k_gather_units3.
template <int T, bool GRAD>
__global__ void __launch_bounds__(128) k_gather_units3w(DskiView op, const int4* __restrict__ units, int nunits,
                                                         const int2* __restrict__ urange,
                                                         const double* __restrict__ w,
                                                         const double* __restrict__ v,
                                                         double* __restrict__ out, int nrhs, int noise, int zmax) {
  extern __shared__ double blkw[];  // per warp [T][T][zmax][nrhs]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* blk = blkw + (size_t)warp * T * T * zmax * nrhs;
  const int m1 = op.m[1], m2 = op.m[2];
  constexpr int REC = 3 * 2 * T;
  const size_t gstride = (size_t)op.n * nrhs;
  for (int u = blockIdx.x * 4 + warp; u < nunits; u += gridDim.x * 4) {
    const int4 U = __ldg(units + u);
    const int2 pr = __ldg(urange + u);
    const int za = U.z, nzb = min(U.w - U.z + T - 1, zmax);
    const int run = nzb * nrhs;
    __syncwarp();  // the previous unit's tasks are done with the block
    for (int ab = 0; ab < T * T; ++ab) {
      const int a = ab / T, b = ab - a * T;
      const double* src = w + (((size_t)(U.x + a) * m1 + (U.y + b)) * m2 + za) * nrhs;
      for (int q = lane; q < run; q += 32) g3_cp8(blk + ab * run + q, src + q);
    }
    g3_cp_wait_all();
    __syncwarp();
    const int ntask = (pr.y - pr.x) * nrhs;
    for (int t = lane; t < ntask; t += 32) {
      const int pl = t / nrhs, r = t - pl * nrhs;
      const int sidx = pr.x + pl;
      const double* rec = op.wts + (size_t)sidx * REC;
      const int zo = __ldg(&op.base[sidx].z) - za;
      double wr_[REC];
#pragma unroll
      for (int q = 0; q < REC; ++q) wr_[q] = __ldg(rec + q);
      double o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int t0 = 0; t0 < T; ++t0) {
        double R0 = 0.0, R1 = 0.0, R2 = 0.0;
#pragma unroll
        for (int t1 = 0; t1 < T; ++t1) {
          const double* wr = blk + ((t0 * T + t1) * nzb + zo) * nrhs + r;
          double uu[T];
#pragma unroll
          for (int t2 = 0; t2 < T; ++t2) uu[t2] = wr[t2 * nrhs];
          double rr = 0.0, qq = 0.0;
#pragma unroll
          for (int t2 = 0; t2 < T; ++t2) {
            rr += wr_[4 * T + t2] * uu[t2];
            if constexpr (GRAD) qq += wr_[5 * T + t2] * uu[t2];
          }
          const double w1 = wr_[2 * T + t1];
          R0 += w1 * rr;
          if constexpr (GRAD) {
            R1 += wr_[3 * T + t1] * rr;
            R2 += w1 * qq;
          }
        }
        const double w0 = wr_[t0];
        o[0] += w0 * R0;
        if constexpr (GRAD) {
          o[1] += wr_[T + t0] * R0;
          o[2] += w0 * R1;
          o[3] += w0 * R2;
        }
      }
      constexpr int NG = GRAD ? 4 : 1;
      const size_t idx0 = (size_t)sidx * nrhs + r;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const size_t idx = idx0 + g * gstride;
        double val = o[g];
        if (noise) val += (g == 0 ? op.nv2 : op.ng2) * __ldg(v + idx);
        out[idx] = val;
      }
    }
  }
}

// d = 3 scatter Bᵀv (dski.cpp:213-219) as a push per cell-line unit plus a
// deterministic merge. Push: CTA per unit (the gather's units: a run of
// occupied base cells of one cell line); its points are staged in shared
// memory and thread (node column ab of the unit's 6×6 block, RHS) walks them in
// order (sorted by base z) with a rolling register window along z, writing
// the unit's block of Bᵀv contributions once per node into a scratch area.
// Every point's data is read once (not once per covering node column).
// Merge: thread (node column, 8-node z segment, RHS) sums the blocks of the
// units covering it in fixed (z-start, unit) order. No atomics anywhere.
constexpr int S3U_THREADS = 128;
constexpr int S3U_MAXP = 40;  // points staged per pass (a unit with more takes several passes)
template <int T, bool GRAD>
__global__ void __launch_bounds__(S3U_THREADS) k_scatter_upush3(DskiView op, const int4* __restrict__ units,
                                                                int nunits, const int2* __restrict__ urange,
                                                                const long long* __restrict__ uoff,
                                                                const double* __restrict__ v,
                                                                double* __restrict__ scratch, int nrhs, int cw) {
  // RHS columns [r0, r0 + cw) of nrhs (blockIdx.y = column chunk; cw·T ≤ threads)
  const int r0 = blockIdx.y * cw, cwa = cw;  // cwa: the staging width allocated
  cw = min(cw, nrhs - r0);
  constexpr int REC = 3 * 2 * T;
  constexpr int NG = GRAD ? 4 : 1;
  extern __shared__ double sm3[];
  double* sw = sm3;                       // [S3U_MAXP][REC]
  double* sv = sw + S3U_MAXP * REC;       // [S3U_MAXP][NG][cw]
  int* sz = reinterpret_cast<int*>(sv + S3U_MAXP * NG * cwa);  // [S3U_MAXP]
  const size_t gstride = (size_t)op.n * nrhs;
  const int ntask = T * cw;  // thread (a, r) owns the T node columns (a, 0..T-1) of the block
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int4 U = __ldg(units + u);
    const int2 pr = __ldg(urange + u);
    const int za = U.z, nzb = U.w - U.z + T - 1;
    double* out = scratch + (size_t)__ldg(uoff + u) * nrhs;
    // rolling windows acc[b][t] <-> node (a, b, zc + t)
    double acc[T][T];
#pragma unroll
    for (int b = 0; b < T; ++b)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[b][t] = 0.0;
    int zc = 0;
    const int tk = threadIdx.x;
    const bool live = tk < ntask;
    const int a = live ? tk / cw : 0, rl = live ? tk - (tk / cw) * cw : 0, r = r0 + rl;
    auto emit = [&]() {  // node zc of the T columns is final
      if (live)
#pragma unroll
        for (int b = 0; b < T; ++b) out[((size_t)(a * T + b) * nzb + zc) * nrhs + r] = acc[b][0];
#pragma unroll
      for (int b = 0; b < T; ++b) {
#pragma unroll
        for (int k = 0; k < T - 1; ++k) acc[b][k] = acc[b][k + 1];
        acc[b][T - 1] = 0.0;
      }
      ++zc;
    };
    for (int p0 = pr.x; p0 < pr.y; p0 += S3U_MAXP) {
      const int np = min(S3U_MAXP, pr.y - p0);
      __syncthreads();  // previous chunk / unit done with the stage
      // staged by cp.async (all copies in flight at once)
      for (int e = threadIdx.x; e < np * REC / 2; e += S3U_THREADS)
        g3_cp16(sw + 2 * e, op.wts + (size_t)p0 * REC + 2 * e);
      for (int pl = threadIdx.x / 32; pl < np; pl += S3U_THREADS / 32)
        for (int q = threadIdx.x & 31; q < NG * cw; q += 32) {
          const int g = q / cw, rr = q - g * cw;
          g3_cp8(sv + pl * NG * cw + q, v + g * gstride + (size_t)(p0 + pl) * nrhs + r0 + rr);
        }
      for (int e = threadIdx.x; e < np; e += S3U_THREADS) g3_cp4(sz + e, &op.base[p0 + e].z);
      g3_cp_wait_all();
      __syncthreads();
      for (int pl = 0; pl < np; ++pl) {
        const double* w = sw + pl * REC;
        const int zo = sz[pl] - za;
        while (zc < zo) emit();
        const double* vv = sv + pl * NG * cw + rl;
        const double wa = w[a], v0 = vv[0];
        double ca, cb = 0.0, cc = 0.0;  // per-b coefficients: A_b = wb·ca + dwb·cb, B_b = wb·cc
        ca = wa * v0;
        if constexpr (GRAD) {
          ca = fma(w[T + a], vv[cw], ca);
          cb = wa * vv[2 * cw];
          cc = wa * vv[3 * cw];
        }
        double z2[T], dz2[T];
#pragma unroll
        for (int c = 0; c < T; ++c) {
          z2[c] = w[4 * T + c];
          dz2[c] = GRAD ? w[5 * T + c] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < T; ++b) {
          const double wb = w[2 * T + b];
          const double A = GRAD ? fma(w[3 * T + b], cb, wb * ca) : wb * ca;
          const double Bc = wb * cc;
#pragma unroll
          for (int c = 0; c < T; ++c) acc[b][c] = GRAD ? fma(dz2[c], Bc, fma(z2[c], A, acc[b][c])) : fma(z2[c], A, acc[b][c]);
        }
      }
    }
    while (zc < nzb) emit();
  }
}

// The same push for few right-hand sides (T·nrhs ≤ 32): one unit per group
// of T·nrhs threads, many units per CTA, point data read straight from L1/L2
// (the per-unit staging of k_scatter_upush3 serves only T·nrhs threads here:
// at 1 RHS its CTA ran 6 live threads of 128). Same per-node order.
template <int T, bool GRAD>
__global__ void __launch_bounds__(64) k_scatter_upush3d(DskiView op, const int4* __restrict__ units, int nunits,
                                                         const int2* __restrict__ urange,
                                                         const long long* __restrict__ uoff,
                                                         const double* __restrict__ v,
                                                         double* __restrict__ scratch, int nrhs) {
  constexpr int REC = 3 * 2 * T;
  const size_t gstride = (size_t)op.n * nrhs;
  const int per = T * nrhs;
  const long long ntask = (long long)nunits * per;
  for (long long g = blockIdx.x * 64LL + threadIdx.x; g < ntask; g += (long long)gridDim.x * 64) {
    const int u = int(g / per), wi = int(g - (long long)u * per);
    const int a = wi / nrhs, r = wi - a * nrhs;
    const int4 U = __ldg(units + u);
    const int2 pr = __ldg(urange + u);
    const int za = U.z, nzb = U.w - U.z + T - 1;
    double* out = scratch + (size_t)__ldg(uoff + u) * nrhs;
    double acc[T][T];
#pragma unroll
    for (int b = 0; b < T; ++b)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[b][t] = 0.0;
    int zc = 0;
    auto emit = [&]() {
#pragma unroll
      for (int b = 0; b < T; ++b) out[((size_t)(a * T + b) * nzb + zc) * nrhs + r] = acc[b][0];
#pragma unroll
      for (int b = 0; b < T; ++b) {
#pragma unroll
        for (int k = 0; k < T - 1; ++k) acc[b][k] = acc[b][k + 1];
        acc[b][T - 1] = 0.0;
      }
      ++zc;
    };
    for (int p = pr.x; p < pr.y; ++p) {
      const double* w = op.wts + (size_t)p * REC;
      const int zo = __ldg(&op.base[p].z) - za;
      while (zc < zo) emit();
      const double wa = __ldg(w + a), v0 = __ldg(v + (size_t)p * nrhs + r);
      double ca = wa * v0, cb = 0.0, cc = 0.0;
      if constexpr (GRAD) {
        ca = fma(__ldg(w + T + a), __ldg(v + gstride + (size_t)p * nrhs + r), ca);
        cb = wa * __ldg(v + 2 * gstride + (size_t)p * nrhs + r);
        cc = wa * __ldg(v + 3 * gstride + (size_t)p * nrhs + r);
      }
      double z2[T], dz2[T];
#pragma unroll
      for (int c = 0; c < T; ++c) {
        z2[c] = __ldg(w + 4 * T + c);
        dz2[c] = GRAD ? __ldg(w + 5 * T + c) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < T; ++b) {
        const double wb = __ldg(w + 2 * T + b);
        const double A = GRAD ? fma(__ldg(w + 3 * T + b), cb, wb * ca) : wb * ca;
        const double Bc = wb * cc;
#pragma unroll
        for (int c = 0; c < T; ++c) acc[b][c] = GRAD ? fma(dz2[c], Bc, fma(z2[c], A, acc[b][c])) : fma(z2[c], A, acc[b][c]);
      }
    }
    while (zc < nzb) emit();
  }
}

// Few right-hand sides (T·nrhs ≤ 32): a warp per unit. The warp stages a
// chunk of the unit's points (weights, v rows, base z) with cp.async — one
// L2 round trip per 32 points instead of one per point in the direct walk
// (k_scatter_upush3d) — then lanes (a, r) run the rolling window over it.
// Same per-node order as k_scatter_upush3.
constexpr int S3W_CH = 32;
template <int T, bool GRAD>
__global__ void __launch_bounds__(128) k_scatter_upush3w(DskiView op, const int4* __restrict__ units, int nunits,
                                                         const int2* __restrict__ urange,
                                                         const long long* __restrict__ uoff,
                                                         const double* __restrict__ v,
                                                         double* __restrict__ scratch, int nrhs) {
  constexpr int REC = 3 * 2 * T;
  constexpr int NG = GRAD ? 4 : 1;
  extern __shared__ __align__(16) double smw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per_warp = S3W_CH * (REC + NG * nrhs) + S3W_CH / 2;  // doubles (+ the z ints)
  double* sw = smw + (size_t)warp * per_warp;  // [CH][REC]
  double* sv = sw + S3W_CH * REC;              // [CH][NG][nrhs]
  int* sz = reinterpret_cast<int*>(sv + S3W_CH * NG * nrhs);  // [CH]
  const size_t gstride = (size_t)op.n * nrhs;
  const int ntask = T * nrhs;
  const bool live = lane < ntask;
  const int a = live ? lane / nrhs : 0, r = live ? lane - (lane / nrhs) * nrhs : 0;
  for (int u = blockIdx.x * 4 + warp; u < nunits; u += gridDim.x * 4) {
    const int4 U = __ldg(units + u);
    const int2 pr = __ldg(urange + u);
    const int za = U.z, nzb = U.w - U.z + T - 1;
    double* out = scratch + (size_t)__ldg(uoff + u) * nrhs;
    double acc[T][T];
#pragma unroll
    for (int b = 0; b < T; ++b)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[b][t] = 0.0;
    int zc = 0;
    auto emit = [&]() {
      if (live)
#pragma unroll
        for (int b = 0; b < T; ++b) out[((size_t)(a * T + b) * nzb + zc) * nrhs + r] = acc[b][0];
#pragma unroll
      for (int b = 0; b < T; ++b) {
#pragma unroll
        for (int k = 0; k < T - 1; ++k) acc[b][k] = acc[b][k + 1];
        acc[b][T - 1] = 0.0;
      }
      ++zc;
    };
    for (int p0 = pr.x; p0 < pr.y; p0 += S3W_CH) {
      const int np = min(S3W_CH, pr.y - p0);
      __syncwarp();  // the previous chunk is consumed
      for (int e = lane; e < np * REC / 2; e += 32) g3_cp16(sw + 2 * e, op.wts + (size_t)p0 * REC + 2 * e);
      for (int q = lane; q < np * NG * nrhs; q += 32) {
        const int pl = q / (NG * nrhs), rem = q - pl * (NG * nrhs);
        const int g = rem / nrhs, rr = rem - g * nrhs;
        g3_cp8(sv + q, v + g * gstride + (size_t)(p0 + pl) * nrhs + rr);
      }
      for (int e = lane; e < np; e += 32) g3_cp4(sz + e, &op.base[p0 + e].z);
      g3_cp_wait_all();
      __syncwarp();
      for (int pl = 0; pl < np; ++pl) {
        const double* w = sw + pl * REC;
        const int zo = sz[pl] - za;
        while (zc < zo) emit();
        const double* vv = sv + pl * NG * nrhs + r;
        const double wa = w[a], v0 = vv[0];
        double ca = wa * v0, cb = 0.0, cc = 0.0;
        if constexpr (GRAD) {
          ca = fma(w[T + a], vv[nrhs], ca);
          cb = wa * vv[2 * nrhs];
          cc = wa * vv[3 * nrhs];
        }
        double z2[T], dz2[T];
#pragma unroll
        for (int c = 0; c < T; ++c) {
          z2[c] = w[4 * T + c];
          dz2[c] = GRAD ? w[5 * T + c] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < T; ++b) {
          const double wb = w[2 * T + b];
          const double A = GRAD ? fma(w[3 * T + b], cb, wb * ca) : wb * ca;
          const double Bc = wb * cc;
#pragma unroll
          for (int c = 0; c < T; ++c) acc[b][c] = GRAD ? fma(dz2[c], Bc, fma(z2[c], A, acc[b][c])) : fma(z2[c], A, acc[b][c]);
        }
      }
    }
    while (zc < nzb) emit();
  }
}

// Merge: u(col, z, r) = Σ over the entries {unit, ab} of column col whose
// block covers z, in the column's fixed (za, unit) order.
__global__ void __launch_bounds__(256) k_scatter_merge3(int ncol, int m2, int nzs, int T,
                                                       const int* __restrict__ cstart,
                                                       const int2* __restrict__ cent,
                                                       const int* __restrict__ cseg,
                                                       const int4* __restrict__ units,
                                                       const long long* __restrict__ uoff,
                                                       const double* __restrict__ scratch, double* __restrict__ u,
                                                       int nrhs) {
  const i64 ntask = (i64)ncol * nzs * nrhs;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < ntask; t += (i64)gridDim.x * blockDim.x) {
    const int r = int(t % nrhs);
    const i64 cz = t / nrhs;
    const int zs = int(cz % nzs), col = int(cz / nzs);
    const int z0 = zs * 8;
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    const int e1 = __ldg(cstart + col + 1);
    for (int e = __ldg(cseg + cz); e < e1; ++e) {
      const int2 en = __ldg(cent + e);
      const int4 U = __ldg(units + en.x);
      const int za = U.z, nzb = U.w - U.z + T - 1;
      if (za >= z0 + 8) break;  // entries sorted by za
      if (za + nzb <= z0) continue;
      const double* src = scratch + ((size_t)__ldg(uoff + en.x) + (size_t)en.y * nzb) * nrhs + r;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int zl = z0 + k - za;
        if (zl >= 0 && zl < nzb) acc[k] += __ldcg(src + (size_t)zl * nrhs);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (z0 + k < m2) u[((size_t)col * m2 + z0 + k) * nrhs + r] = acc[k];
  }
}

// Merge over flattened per-node lists: for every node (column, z) the
// scratch node offsets of exactly the blocks covering it, in the column's
// (za, unit) order (built with the operator). CTA per node column: its
// per-z starts and list are staged in shared memory by all threads at once,
// then thread (z, RHS) sums its list four entries at a time (the four loads
// issued together). No candidate scanning or coverage predicates (the
// per-segment entry walk of k_scatter_merge3 visits ~33 entries per node of
// which ~6 cover it). Same per-node summation order: bit-identical.
constexpr int M3F_THREADS = 256;
constexpr int M3F_UNROLL = 8;  // a node's list (~6 blocks) in one round of loads
__global__ void __launch_bounds__(M3F_THREADS) k_scatter_merge3f(int ngroups, int gn, int nnodes,
                                                                const int* __restrict__ zoff,
                                                                const int* __restrict__ zlist,
                                                                const double* __restrict__ scratch,
                                                                double* __restrict__ u, int nrhs) {
  // CTA per group of gn consecutive nodes (whole node columns: one column, or
  // several when a column has fewer outputs than threads); nodes (col, z)
  // are consecutive in both zoff and u
  extern __shared__ int sl[];  // [gn + 1] list starts relative to the group, then the group's list
  int* li = sl + gn + 1;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int n0 = grp * gn, nn = min(gn, nnodes - n0);
    const int* zo = zoff + n0;
    const int b0 = __ldg(zo), nl = __ldg(zo + nn) - b0;
    __syncthreads();
    for (int z = threadIdx.x; z <= nn; z += M3F_THREADS) sl[z] = __ldg(zo + z) - b0;
    for (int i = threadIdx.x; i < nl; i += M3F_THREADS) li[i] = __ldg(zlist + b0 + i);
    __syncthreads();
    double* uc = u + (size_t)n0 * nrhs;
    const int nout = nn * nrhs;
    for (int o = threadIdx.x; o < nout; o += M3F_THREADS) {
      const int z = o / nrhs, r = o - z * nrhs;
      const int s1 = sl[z + 1];
      double acc = 0.0;
      for (int i = sl[z]; i < s1; i += M3F_UNROLL) {
        double val[M3F_UNROLL];
#pragma unroll
        for (int j = 0; j < M3F_UNROLL; ++j)
          val[j] = i + j < s1 ? __ldcg(scratch + (size_t)li[i + j] * nrhs + r) : 0.0;
#pragma unroll
        for (int j = 0; j < M3F_UNROLL; ++j)
          if (i + j < s1) acc += val[j];
      }
      uc[o] = acc;
    }
  }
}

// Lean-kernel launch shape: x = RHS lanes (≤ 32), y = items per block, shrunk
// (down to one warp) when there are too few items to give every SM ~4 CTAs.
static dim3 lean_block(int nrhs, i64 items) {
  const int bx = nrhs >= 32 ? 32 : nrhs;
  int by = 256 / bx;
  const i64 lanes_total = items * std::min(nrhs, 32);
  while (by * bx > 32 && (lanes_total + by * bx - 1) / (by * bx) < 4 * 148) by /= 2;
  if (by < 1) by = 1;
  return dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by));
}

bool DskiOp::scatter_band(const double* v, double* u, int nrhs, cudaStream_t s) const {
  const DskiView vw = view();
  const int BC = std::max(1, std::min({nrhs, 256 * S2_ITEMS / m[1], 32}));
  const int NQ = G ? 2 : 1;
  const size_t shm = size_t(max_row_pts) * (2 * T + NQ * BC) * sizeof(double) + size_t(max_row_pts) * 4 + 16;
  if (d != 2 || m[1] > 256 * S2_ITEMS || shm > 200 * 1024) return false;
  dim3 grid(static_cast<unsigned>(m[0]), static_cast<unsigned>((nrhs + BC - 1) / BC));
#define GK_S2(TT, GG)                                                                \
  smem_attr((const void*)k_scatter2d<TT, GG>, shm);                                  \
  k_scatter2d<TT, GG><<<grid, 256, shm, s>>>(vw, v, u, nrhs, BC, max_row_pts);
  if (T == 6) {
    if (G) { GK_S2(6, true) } else { GK_S2(6, false) }
  } else {
    if (G) { GK_S2(4, true) } else { GK_S2(4, false) }
  }
#undef GK_S2
  launched("dski scatter (2-D band)");
  return true;
}

bool DskiOp::gather_band(const double* w, const double* v, double* out, int nrhs, bool noise,
                         cudaStream_t s) const {
  if (d != 2) return false;
  const DskiView vw = view();
  const int rows = G2_R + T - 1;
  const size_t fixed = size_t(G2_PCH) * (4 * T * sizeof(double) + 2 * sizeof(int)) + 16;
  int BC = std::min(nrhs, 8);
  while (BC > 1 && size_t(rows) * m[1] * BC * sizeof(double) + fixed > 100 * 1024) --BC;
  const size_t shm = size_t(rows) * m[1] * BC * sizeof(double) + fixed;
  if (shm > 200 * 1024) return false;
  dim3 grid(static_cast<unsigned>((nb[0] + G2_R - 1) / G2_R), static_cast<unsigned>((nrhs + BC - 1) / BC));
  const int nz = noise ? 1 : 0;
#define GK_G2(TT, GG)                                                    \
  smem_attr((const void*)k_gather2d<TT, GG>, shm);                       \
  k_gather2d<TT, GG><<<grid, 256, shm, s>>>(vw, w, v, out, nrhs, BC, nz);
  if (T == 6) {
    if (G) { GK_G2(6, true) } else { GK_G2(6, false) }
  } else {
    if (G) { GK_G2(4, true) } else { GK_G2(4, false) }
  }
#undef GK_G2
  launched("dski gather (2-D band)");
  return true;
}

void DskiOp::scatter(const double* v, double* u, int nrhs, cudaStream_t s) const {
  const DskiView vw = view();
  const int variant = g_tuning.scatter.load();
  if (variant == 2 && scatter_band(v, u, nrhs, s)) return;
  if (variant == 1) {
    const int blocks = grid_blocks(M * nrhs);
    GK_DISPATCH_DT(d, T, {
      if (G) k_scatter<D, T, true><<<blocks, 256, 0, s>>>(vw, v, u, nrhs);
      else k_scatter<D, T, false><<<blocks, 256, 0, s>>>(vw, v, u, nrhs);
    });
    launched("dski scatter");
    return;
  }
  const dim3 blk = lean_block(nrhs, M);
  const dim3 grid(static_cast<unsigned>((M + blk.y - 1) / blk.y), static_cast<unsigned>((nrhs + blk.x - 1) / blk.x));
  if (variant == 3) {
    GK_DISPATCH_DT(d, T, {
      if (G) k_scatter_cells<D, T, true><<<grid, blk, 0, s>>>(vw, v, u, nrhs);
      else k_scatter_cells<D, T, false><<<grid, blk, 0, s>>>(vw, v, u, nrhs);
    });
    launched("dski scatter (cells)");
    return;
  }
  if (d == 1 && variant == 0) {
    const dim3 g1(static_cast<unsigned>(M), static_cast<unsigned>(nrhs));
    if (T == 6) {
      if (G) k_scatter_1d<6, true><<<g1, 256, 0, s>>>(vw, v, u, nrhs);
      else k_scatter_1d<6, false><<<g1, 256, 0, s>>>(vw, v, u, nrhs);
    } else {
      if (G) k_scatter_1d<4, true><<<g1, 256, 0, s>>>(vw, v, u, nrhs);
      else k_scatter_1d<4, false><<<g1, 256, 0, s>>>(vw, v, u, nrhs);
    }
    launched("dski scatter (d=1 node blocks)");
    return;
  }
  if (d == 3 && variant == 0 && s3_uoff.p && G) {  // unit push + merge
    const int NG = 4;
    // RHS columns in chunks of at most S3U_THREADS / T (blockIdx.y), so the
    // unit path serves any RHS count (beyond 21 columns it used to fall back
    // to the per-column lists: 32 RHS 362 µs)
    const int nch = (T * nrhs + S3U_THREADS - 1) / S3U_THREADS;
    const int cw = (nrhs + nch - 1) / nch;
    const size_t smem = sizeof(double) * size_t(S3U_MAXP) * (3 * 2 * T + NG * cw) + sizeof(int) * S3U_MAXP;
    const void* fn = T == 6 ? (const void*)k_scatter_upush3<6, true> : (const void*)k_scatter_upush3<4, true>;
    if (smem > 48 * 1024) raise_smem_limit(fn, smem);
    s3_scratch.reserve(static_cast<size_t>(s3_nodes) * nrhs);
    if (T * nrhs <= 32 && !(g_tuning.d3.load() & (4 | 2048))) {
      const size_t wsm = sizeof(double) * 4 * (size_t(S3W_CH) * (3 * 2 * T + NG * nrhs) + S3W_CH / 2);
      const void* fw = T == 6 ? (const void*)k_scatter_upush3w<6, true> : (const void*)k_scatter_upush3w<4, true>;
      if (wsm > 48 * 1024) raise_smem_limit(fw, wsm);
      const unsigned gw = static_cast<unsigned>(std::max(1, (g3_nunits + 3) / 4));
      if (T == 6) k_scatter_upush3w<6, true><<<gw, 128, wsm, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs);
      else k_scatter_upush3w<4, true><<<gw, 128, wsm, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs);
      launched("dski scatter (d=3 unit push, warp per unit)");
    } else if (T * nrhs <= 32 && !(g_tuning.d3.load() & 4)) {
      const long long nt = static_cast<long long>(g3_nunits) * T * nrhs;
      const unsigned gd = static_cast<unsigned>(std::max<long long>(1, (nt + 63) / 64));
      if (T == 6) k_scatter_upush3d<6, true><<<gd, 64, 0, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs);
      else k_scatter_upush3d<4, true><<<gd, 64, 0, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs);
      launched("dski scatter (d=3 unit push, direct)");
    } else {
    const dim3 gp(static_cast<unsigned>(std::max(1, std::min(g3_nunits, 148 * 16 / nch))), static_cast<unsigned>(nch));
    if (T == 6) k_scatter_upush3<6, true><<<gp, S3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs, cw);
    else k_scatter_upush3<4, true><<<gp, S3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, s3_uoff.p, v, s3_scratch.p, nrhs, cw);
    launched("dski scatter (d=3 unit push)");
    }
    const int ncol = m[0] * m[1];
    // columns per CTA: one, or several when a column's outputs (m2 · nrhs)
    // leave most of the CTA idle (1 RHS: 48 outputs for 256 threads)
    const int cpb = (g_tuning.d3.load() & 4096) ? 1 : std::max(1, M3F_THREADS / (m[2] * nrhs));
    const size_t msm = sizeof(int) * (size_t(cpb) * m[2] + 1 + size_t(cpb) * s3_maxl);
    if (s3_zoff.p && msm <= 96 * 1024 && !(g_tuning.d3.load() & 1)) {
      raise_smem_limit((const void*)k_scatter_merge3f, msm);
      const int ngroups = (ncol + cpb - 1) / cpb;
      k_scatter_merge3f<<<static_cast<unsigned>(std::min(ngroups, 148 * 32)), M3F_THREADS, msm, s>>>(
          ngroups, cpb * m[2], ncol * m[2], s3_zoff.p, s3_zlist.p, s3_scratch.p, u, nrhs);
      launched("dski scatter (d=3 unit merge, per-node lists)");
      return;
    }
    k_scatter_merge3<<<grid_blocks(i64(ncol) * s3_nzs * nrhs), 256, 0, s>>>(ncol, m[2], s3_nzs, T, s3_cstart.p, s3_cent.p,
                                                                          s3_cseg.p, g3_units.p, s3_uoff.p,
                                                                          s3_scratch.p, u, nrhs);
    launched("dski scatter (d=3 unit merge)");
    return;
  }
  // column tiles: measured faster than the per-column lists for 1-2 RHS at C3
  // (1 RHS: 228 vs 323 us), slower for 17+ RHS (every warp walks every
  // point of the tile; 578 vs 365 us)
  if (d == 3 && (variant == 8 || (variant == 0 && nrhs <= 2)) && tile3_units.p) {
    const int TB = tile3_tb;
    const int nch = int((i64(TB) * TB * nrhs + 1023) / 1024);
    const int RC = (nrhs + nch - 1) / nch;
    const int nthr = (TB * TB * RC + 31) / 32 * 32;
    const int G4 = G ? 4 : 1;
    const size_t shm = 2 * B3_E * (16 + size_t(3) * T * 16 + size_t(G4) * RC * 8);
    const dim3 tgrid(static_cast<unsigned>(tile3_nunits), static_cast<unsigned>(nch));
    auto go = [&](const void* fn, auto kern) {
      if (shm > 48 * 1024) raise_smem_limit(fn, shm);
      kern<<<tgrid, nthr, shm, s>>>(vw, tile3_list.p, tile3_units.p, TB, RC, tile3_tiles1, v, u, nrhs);
    };
    if (T == 6) {
      if (G) go((const void*)k_scatter_tile3<6, true>, k_scatter_tile3<6, true>);
      else go((const void*)k_scatter_tile3<6, false>, k_scatter_tile3<6, false>);
    } else {
      if (G) go((const void*)k_scatter_tile3<4, true>, k_scatter_tile3<4, true>);
      else go((const void*)k_scatter_tile3<4, false>, k_scatter_tile3<4, false>);
    }
    launched("dski scatter (d=3 column tiles)");
    return;
  }
  if (d == 3 && variant == 7 && col3_units.p) {  // balanced units over the per-column sorted lists
    GK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * size_t(M) * nrhs, s));
    const dim3 cblk(32, 8);
    const dim3 cgrid(static_cast<unsigned>((col3_nunits + 7) / 8), static_cast<unsigned>((nrhs + 31) / 32));
    if (T == 6) {
      if (G) k_scatter_units3<6, true><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_units.p, col3_nunits, v, u, nrhs);
      else k_scatter_units3<6, false><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_units.p, col3_nunits, v, u, nrhs);
    } else {
      if (G) k_scatter_units3<4, true><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_units.p, col3_nunits, v, u, nrhs);
      else k_scatter_units3<4, false><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_units.p, col3_nunits, v, u, nrhs);
    }
    launched("dski scatter (d=3 balanced column units)");
    return;
  }
  if (d == 3 && (variant == 0 || variant == 6) && col3_list.p) {  // per-column sorted point lists
    const dim3 cblk(32, L3_WARPS);
    const dim3 cgrid(static_cast<unsigned>((m[0] * m[1] + L3_WARPS - 1) / L3_WARPS), static_cast<unsigned>(col3_nseg),
                     static_cast<unsigned>((nrhs + 31) / 32));
    if (T == 6) {
      if (G) k_scatter_list3<6, true><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_seg.p, col3_nseg, col3_zseg, v, u, nrhs);
      else k_scatter_list3<6, false><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_seg.p, col3_nseg, col3_zseg, v, u, nrhs);
    } else {
      if (G) k_scatter_list3<4, true><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_seg.p, col3_nseg, col3_zseg, v, u, nrhs);
      else k_scatter_list3<4, false><<<cgrid, cblk, 0, s>>>(vw, col3_list.p, col3_start.p, col3_seg.p, col3_nseg, col3_zseg, v, u, nrhs);
    }
    launched("dski scatter (d=3 column lists)");
    return;
  }
  if (d == 3 && (variant == 0 || variant == 5)) {  // node columns with a rolling window along the last axis
    const int zseg = 12;
    const dim3 cblk(32, 8);
    const dim3 cgrid(static_cast<unsigned>((m[0] * m[1] + 7) / 8), static_cast<unsigned>((m[2] + zseg - 1) / zseg),
                     static_cast<unsigned>((nrhs + 31) / 32));
    if (T == 6) {
      if (G) k_scatter_col3<6, true><<<cgrid, cblk, 0, s>>>(vw, v, u, nrhs, zseg);
      else k_scatter_col3<6, false><<<cgrid, cblk, 0, s>>>(vw, v, u, nrhs, zseg);
    } else {
      if (G) k_scatter_col3<4, true><<<cgrid, cblk, 0, s>>>(vw, v, u, nrhs, zseg);
      else k_scatter_col3<4, false><<<cgrid, cblk, 0, s>>>(vw, v, u, nrhs, zseg);
    }
    launched("dski scatter (d=3 node columns)");
    return;
  }
  GK_DISPATCH_DT(d, T, {
    if (G) k_scatter_lean<D, T, true><<<grid, blk, 0, s>>>(vw, v, u, nrhs);
    else k_scatter_lean<D, T, false><<<grid, blk, 0, s>>>(vw, v, u, nrhs);
  });
  launched("dski scatter (lean)");
}

void DskiOp::gather(const double* w, const double* v, double* out, int nrhs, bool noise,
                    cudaStream_t s) const {
  const DskiView vw = view();
  const int variant = g_tuning.gather.load();
  if (variant == 2 && gather_band(w, v, out, nrhs, noise, s)) return;
  if (variant == 1) {
    const int blocks = grid_blocks(n * nrhs);
    GK_DISPATCH_DT(d, T, {
      if (G) k_gather<D, T, true><<<blocks, 256, 0, s>>>(vw, w, v, out, nrhs, noise ? 1 : 0);
      else k_gather<D, T, false><<<blocks, 256, 0, s>>>(vw, w, v, out, nrhs, noise ? 1 : 0);
    });
    launched("dski gather");
    return;
  }
  // (every RHS count since the cp.async staging: 1 RHS 34.8 -> 30.8 µs and
  // 3 RHS 43.0 -> 32.7 µs against the lean gather)
  if (d == 3 && variant == 0 && g3_units.p && nrhs <= 4 && !(g_tuning.d3.load() & (1024 | 16384))) {
    const size_t smem = sizeof(double) * 4 * size_t(T) * T * g3_zspan * nrhs;
    const void* fn = T == 6 ? (G ? (const void*)k_gather_units3w<6, true> : (const void*)k_gather_units3w<6, false>)
                            : (G ? (const void*)k_gather_units3w<4, true> : (const void*)k_gather_units3w<4, false>);
    raise_smem_limit(fn, smem);
    const unsigned grid = static_cast<unsigned>(std::max(1, (g3_nunits + 3) / 4));
    const int nz = noise ? 1 : 0;
    if (T == 6) {
      if (G) k_gather_units3w<6, true><<<grid, 128, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, nz, g3_zspan);
      else k_gather_units3w<6, false><<<grid, 128, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, nz, g3_zspan);
    } else {
      if (G) k_gather_units3w<4, true><<<grid, 128, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, nz, g3_zspan);
      else k_gather_units3w<4, false><<<grid, 128, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, nz, g3_zspan);
    }
    launched("dski gather (d=3 cell-line units, warp per unit)");
    return;
  }
  if (d == 3 && variant == 0 && g3_units.p && !(g_tuning.d3.load() & 1024)) {
    // RHS chunks of ≤ 17 columns (blockIdx.y): 64 RHS staged whole took
    // 166 KB per CTA (one CTA per SM)
    const int nch = (nrhs + 16) / 17;
    const int cw = (nrhs + nch - 1) / nch;
    const size_t smem = sizeof(double) * size_t(T) * T * g3_zspan * cw;
    if (smem <= 200 * 1024) {
      const void* fn = T == 6 ? (G ? (const void*)k_gather_units3<6, true> : (const void*)k_gather_units3<6, false>)
                              : (G ? (const void*)k_gather_units3<4, true> : (const void*)k_gather_units3<4, false>);
      raise_smem_limit(fn, smem);
      GK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared)));
      const dim3 grid(static_cast<unsigned>(std::max(1, std::min(g3_nunits, 148 * 16 / nch))), static_cast<unsigned>(nch));
      const int d3 = g_tuning.d3.load();
      const int nz = noise ? 1 : 0;
      if (T == 6 && G && (cw == 16 || cw == 17) && nrhs % cw == 0 && !(d3 & 512)) {
        const void* fs = nch == 1 ? (cw == 16 ? (const void*)k_gather_units3<6, true, 16, true> : (const void*)k_gather_units3<6, true, 17, true>)
                                  : (cw == 16 ? (const void*)k_gather_units3<6, true, 16> : (const void*)k_gather_units3<6, true, 17>);
        raise_smem_limit(fs, smem);
        GK_CUDA(cudaFuncSetAttribute(fs, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared)));
        auto args = [&](auto kern) {
          kern<<<grid, G3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, cw, nz, g3_zspan, d3);
        };
        if (nch == 1) {
          if (cw == 16) args(k_gather_units3<6, true, 16, true>);
          else args(k_gather_units3<6, true, 17, true>);
        } else {
          if (cw == 16) args(k_gather_units3<6, true, 16>);
          else args(k_gather_units3<6, true, 17>);
        }
      } else if (T == 6) {
        if (G) k_gather_units3<6, true><<<grid, G3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, cw, nz, g3_zspan, d3);
        else k_gather_units3<6, false><<<grid, G3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, cw, nz, g3_zspan, d3);
      } else {
        if (G) k_gather_units3<4, true><<<grid, G3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, cw, nz, g3_zspan, d3);
        else k_gather_units3<4, false><<<grid, G3U_THREADS, smem, s>>>(vw, g3_units.p, g3_nunits, g3_range.p, w, v, out, nrhs, cw, nz, g3_zspan, d3);
      }
      launched("dski gather (d=3 cell-line units)");
      return;
    }
  }
  const dim3 blk = lean_block(nrhs, n);
  const dim3 grid(static_cast<unsigned>((n + blk.y - 1) / blk.y), static_cast<unsigned>((nrhs + blk.x - 1) / blk.x));
  GK_DISPATCH_DT(d, T, {
    if (G) k_gather_lean<D, T, true><<<grid, blk, 0, s>>>(vw, w, v, out, nrhs, noise ? 1 : 0);
    else k_gather_lean<D, T, false><<<grid, blk, 0, s>>>(vw, w, v, out, nrhs, noise ? 1 : 0);
  });
  launched("dski gather (lean)");
}

__global__ void k_axpy_inplace(double* __restrict__ w, const double* __restrict__ x, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) w[i] += x[i];
}

// ---------------------------------------------------------------- general profiles
// Stationary profile κ(offset) = eval(kernel, offset, 0) (kernels.cpp:104-118)
// and its ∂/∂log ℓ (eval_dlogell, kernels.cpp:172-188), on the host.
static double profile_value(const gk_kernel& k, const double* off, int d, bool dlogell) {
  const double s2 = k.outputscale * k.outputscale, ell = k.lengthscale;
  double r2 = 0.0;
  for (int j = 0; j < d; ++j) r2 += off[j] * off[j];
  if (k.family == 0) {
    const double v = s2 * std::exp(-0.5 * r2 / (ell * ell));
    return dlogell ? v * (r2 / (ell * ell)) : v;
  }
  if (!dlogell) {
    const double rho = std::sqrt(r2) / ell;
    const double radial = k.spline_even ? (rho > 0 ? rho * rho * std::log(rho) : 0.0) : rho * rho * rho;
    return s2 * (radial + k.spline_a * rho * rho + k.spline_b);
  }
  if (r2 == 0.0) return 0.0;
  const double rho2 = r2 / (ell * ell);
  const double rho = std::sqrt(rho2);
  if (!k.spline_even) return s2 * (-3.0 * rho * rho2 - 2.0 * k.spline_a * rho2);
  return s2 * (-2.0 * rho2 * std::log(rho) - rho2 - 2.0 * k.spline_a * rho2);
}

// The profile on an embedded torus of E[j] nodes per axis at the wrapped
// offsets (i ≤ E/2 ? i : i − E)·h_j, row-major (dski.cpp:97-114).
static std::vector<double> embedded_slice(const gk_kernel& k, const gk_grid& g, const int* E, bool dlogell) {
  const int d = g.d;
  i64 tot = 1;
  for (int j = 0; j < d; ++j) tot *= E[j];
  std::vector<double> out(static_cast<size_t>(tot));
  int idx[3] = {0, 0, 0};
  double off[3];
  for (i64 t = 0; t < tot; ++t) {
    for (int j = 0; j < d; ++j) off[j] = double(idx[j] <= E[j] / 2 ? idx[j] : idx[j] - E[j]) * g.spacing[j];
    out[static_cast<size_t>(t)] = profile_value(k, off, d, dlogell);
    for (int j = d - 1; j >= 0; --j) {
      if (++idx[j] < E[j]) break;
      idx[j] = 0;
    }
  }
  return out;
}

double DskiOp::min_embedding_eigenvalue() const {
  if (!slice_ref_h.empty()) return min_embedding_eigenvalue_host(d, m, slice_ref_h);
  int E[3] = {1, 1, 1};
  for (int j = 0; j < d; ++j) E[j] = 2 * (m[j] - 1);
  return min_embedding_eigenvalue_host(d, m, embedded_slice(kernel, grid, E, false));
}

// diag = Σ_δ κ(δ) Π_j P_j(δ_j), P_j the autocorrelation of axis j's stencil
// weights (derivative weights on the group's axis): the offset-table double
// loop of dski.cpp:240-290 regrouped by offset.
template <int D, int T>
__global__ void k_diagonal_generic(DskiView op, const double* __restrict__ tab, double* __restrict__ diag) {
  constexpr int W = 2 * T - 1, STRIDE = D * 2 * T;
  int nt = 1;
  for (int j = 0; j < D; ++j) nt *= W;
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < op.n; s += (i64)gridDim.x * blockDim.x) {
    const double* p = op.wts + s * STRIDE;
    for (int g = 0; g <= op.G; ++g) {
      double P[D][W];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double* c = p + j * 2 * T + (g == j + 1 ? T : 0);
#pragma unroll
        for (int dl = 0; dl < W; ++dl) {
          const int del = dl - (T - 1);
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < T; ++a)
            if (a - del >= 0 && a - del < T) acc += c[a] * c[a - del];
          P[j][dl] = acc;
        }
      }
      double sum = 0.0;
      for (int t = 0; t < nt; ++t) {
        int r = t;
        double prod = __ldg(tab + t);
#pragma unroll
        for (int j = D - 1; j >= 0; --j) {
          prod *= P[j][r % W];
          r /= W;
        }
        sum += prod;
      }
      diag[(i64)g * op.n + s] = sum + (g == 0 ? op.nv2 : op.ng2);
    }
  }
}

// grid vector e (zeroed by the caller) = the stencil of point si, group g
template <int D, int T>
__global__ void k_stencil_to_grid(DskiView op, int si, int g, double* __restrict__ e) {
  constexpr int STRIDE = D * 2 * T;
  int nt = 1;
  for (int j = 0; j < D; ++j) nt *= T;
  const int4 b = op.base[si];
  const int bb[3] = {b.x, b.y, b.z};
  const double* p = op.wts + (i64)si * STRIDE;
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    int r = t, tj[3] = {0, 0, 0};
    for (int j = D - 1; j >= 0; --j) {
      tj[j] = r % T;
      r /= T;
    }
    double w = 1.0;
    i64 node = 0;
    for (int j = 0; j < D; ++j) {
      w *= p[j * 2 * T + (g == j + 1 ? T : 0) + tj[j]];
      node = node * op.m[j] + bb[j] + tj[j];
    }
    e[node] = w;
  }
}

__global__ void k_add_scalar(double* __restrict__ x, double v) { *x += v; }

void DskiOp::kuu(const double* u, double* w, int nrhs, cudaStream_t s) const {
  if (generic) {
    kfft->apply(u, w, nrhs, s);
    return;
  }
  // Modes from the last axis to the first: u -> ... -> w, intermediates
  // alternating between w and the scratch grid_t so the last mode lands in w
  // (caller has reserved grid_t for nrhs columns; u must not alias w/grid_t).
  const double* src = u;
  for (int j = d - 1; j >= 0; --j) {
    i64 P = 1, Q = nrhs;
    for (int i = 0; i < j; ++i) P *= m[i];
    for (int i = j + 1; i < d; ++i) Q *= m[i];
    double* dst = (j % 2 == 0) ? w : grid_t.p;
    toeplitz_mode(tvec.p + toff_h[static_cast<size_t>(j)], m[j], band[static_cast<size_t>(j)], P, Q, src, dst, s);
    src = dst;
  }
}

// w = ∂K_UU/∂log ℓ · u = Σ_j (⊗_i S_i^{(j)}) u with S_j^{(j)} = T_j ρ_j², S_i^{(j)} = T_i
// (the reference applies the same operator through a second circulant
// embedding of kernel_dlogell_profile, dski.cpp:36-40, gp.cpp:212-213).
void DskiOp::kuu_dlogell(const double* u, double* w, int nrhs, cudaStream_t s) {
  if (generic) {  // the reference's second embedding of kernel_dlogell_profile (dski.cpp:36-40)
    if (kernel.family == 2)
      fail(GK_ERR_UNSUPPORTED, "d/dlog(ell) needs a kernel family (the operator was built from a profile slice)");
    if (!kfft_dl) {
      auto f = std::make_unique<KuuFft>();
      f->init(d, m);
      f->build(embedded_slice(kernel, grid, f->E, true), s);
      kfft_dl = std::move(f);
    }
    kfft_dl->apply(u, w, nrhs, s);
    return;
  }
  grow(grid_a, static_cast<size_t>(M) * nrhs);
  grow(grid_b, static_cast<size_t>(M) * nrhs);
  for (int term = 0; term < d; ++term) {
    const double* src = u;
    for (int j = d - 1; j >= 0; --j) {
      i64 P = 1, Q = nrhs;
      for (int i = 0; i < j; ++i) P *= m[i];
      for (int i = j + 1; i < d; ++i) Q *= m[i];
      const bool last = j == 0;
      double* dst = last && term == 0 ? w : (src == grid_a.p ? grid_b.p : grid_a.p);
      const bool deriv = j == term;
      const double* t = (deriv ? tvec_dl.p : tvec.p) + toff_h[static_cast<size_t>(j)];
      toeplitz_mode(t, m[j], (deriv ? band_dl : band)[static_cast<size_t>(j)], P, Q, src, dst, s);
      src = dst;
    }
    if (term > 0) {
      k_axpy_inplace<<<blocks_for((i64)M * nrhs), 256, 0, s>>>(w, src, (i64)M * nrhs);
      launched("dski dlogell accumulate");
    }
  }
}

void DskiOp::diagonal(double* dd, cudaStream_t s) {
  const DskiView vw = view();
  if (generic) {
    if (!gtab.p) {
      const int W = 2 * T - 1;
      int E[3] = {W, W, W};
      gk_grid tg = grid;  // offsets (i − (T−1))·h: a W^d table centred on 0
      std::vector<double> tab;
      i64 tot = 1;
      for (int j = 0; j < d; ++j) tot *= W;
      tab.resize(static_cast<size_t>(tot));
      int idx[3] = {0, 0, 0};
      double off[3];
      for (i64 t = 0; t < tot; ++t) {
        for (int j = 0; j < d; ++j) off[j] = double(idx[j] - (T - 1)) * tg.spacing[j];
        tab[static_cast<size_t>(t)] = profile_value(kernel, off, d, false);
        for (int j = d - 1; j >= 0; --j) {
          if (++idx[j] < E[j]) break;
          idx[j] = 0;
        }
      }
      gtab.upload(tab.data(), tab.size(), s);
      GK_CUDA(cudaStreamSynchronize(s));
    }
    GK_DISPATCH_DT(d, T, { k_diagonal_generic<D, T><<<grid_blocks(n), 256, 0, s>>>(vw, gtab.p, dd); });
    launched("dski diagonal (general profile)");
    return;
  }
  GK_DISPATCH_DT(d, T, { k_diagonal<D, T><<<grid_blocks(n), 256, 0, s>>>(vw, tvec.p, toff.p, dd); });
  launched("dski diagonal");
}

bool DskiOp::row_dev(const i64* d_r_int, const int* d_active, double* out, cudaStream_t s) {
  const DskiView vw = view();
  const int shm = int(sizeof(double)) * (m[0] + (d > 1 ? m[1] : 0) + (d > 2 ? m[2] : 0));
  GK_DISPATCH_DT(d, T, {
    k_row_dev<D, T><<<grid_blocks(N), 256, shm, s>>>(vw, tvec.p, toff.p, reinterpret_cast<const long long*>(d_r_int),
                                                    d_active, out);
  });
  launched("dski row (device pivot)");
  return true;
}

void DskiOp::row(i64 r_ext, double* out, cudaStream_t s) {
  if (r_ext < 0 || r_ext >= N) fail(GK_ERR_RANGE, "D-SKI row index out of range");
  const int g = int(r_ext / n);
  const int si = int(inv_h[static_cast<size_t>(r_ext % n)]);
  const DskiView vw = view();
  if (generic) {  // row = B K_UU (stencil of the row) + its noise entry (dski.cpp:292-304)
    ensure_scratch(1);
    GK_CUDA(cudaMemsetAsync(grid_u.p, 0, sizeof(double) * M, s));
    GK_DISPATCH_DT(d, T, { k_stencil_to_grid<D, T><<<1, 256, 0, s>>>(vw, si, g, grid_u.p); });
    launched("dski row stencil");
    kfft->apply(grid_u.p, grid_w.p, 1, s);
    gather(grid_w.p, grid_w.p, out, 1, false, s);
    k_add_scalar<<<1, 1, 0, s>>>(out + (i64)g * n + si, g == 0 ? nv2 : ng2);
    launched("dski row noise");
    return;
  }
  const int shm = int(sizeof(double)) * (m[0] + (d > 1 ? m[1] : 0) + (d > 2 ? m[2] : 0));
  GK_DISPATCH_DT(d, T, { k_row<D, T><<<grid_blocks(N), 256, shm, s>>>(vw, tvec.p, toff.p, si, g, out); });
  launched("dski row");
}

// ---------------------------------------------------------------- creation
// profile 0: SE value; profile 1: d/dlog(ell) of the SE profile
// (kernel_dlogell_profile, dski.cpp:36-40) — separable only for d = 1, which
// is all the D-SKIP leaves need (dskip.cpp:171).
std::unique_ptr<Op> make_dski_profile(const gk_kernel& k, const gk_grid& g, const double* X, i64 n,
                                      double nv, double ng, int order, int with_grad, int device,
                                      int profile, const double* slice_ref, const double* offset_table);
// the entry the D-SKIP leaves use (dskip.cu)
std::unique_ptr<Op> make_dski_profile(const gk_kernel& k, const gk_grid& g, const double* X, i64 n,
                                      double nv, double ng, int order, int with_grad, int device, int profile) {
  return make_dski_profile(k, g, X, n, nv, ng, order, with_grad, device, profile, nullptr, nullptr);
}

// DskiOperator over a caller-evaluated stationary profile (the boundary's
// profile-agnostic form): slice_ref = the profile on the reference embedding
// (2(m_j − 1) nodes per axis, dski.cpp:97-114), offset_table = the profile at
// the (2T − 1)^d stencil offsets (kernel_offset_table_, dski.cpp:181-203).
std::unique_ptr<Op> make_dski_slices(const gk_grid& g, const double* X, i64 n, double nv, double ng, int order,
                                     int with_grad, int device, const double* slice_ref, const double* offset_table) {
  if (!slice_ref || !offset_table) fail(GK_ERR_ARG, "profile slice and offset table are required");
  gk_kernel k{2, 1.0, 1.0, 0.0, 0.0, 0};  // family 2: caller-supplied profile
  return make_dski_profile(k, g, X, n, nv, ng, order, with_grad, device, 0, slice_ref, offset_table);
}

std::unique_ptr<Op> make_dski(const gk_kernel& k, const gk_grid& g, const double* X, i64 n,
                              double nv, double ng, int order, int with_grad, int device) {
  return make_dski_profile(k, g, X, n, nv, ng, order, with_grad, device, 0, nullptr, nullptr);
}

std::unique_ptr<Op> make_dski_profile(const gk_kernel& k, const gk_grid& g, const double* X, i64 n,
                                      double nv, double ng, int order, int with_grad, int device,
                                      int profile, const double* slice_ref, const double* offset_table) {
  if (profile == 1 && g.d != 1)
    fail(GK_ERR_UNSUPPORTED, "the d/dlog(ell) grid profile is implemented for 1-D grids only");
  if (k.family != 0 && k.family != 1 && !(k.family == 2 && slice_ref)) fail(GK_ERR_ARG, "unknown kernel family");
  if (k.family != 0 && profile != 0)
    fail(GK_ERR_UNSUPPORTED, "the d/dlog(ell) 1-D grid profile is the D-SKIP leaf's (separable kernels only)");
  if (!(k.lengthscale > 0.0)) fail(GK_ERR_ARG, "lengthscale must be > 0");
  if (!(k.outputscale > 0.0)) fail(GK_ERR_ARG, "outputscale must be > 0");
  if (g.d < 1 || g.d > 3) fail(GK_ERR_UNSUPPORTED, "D-SKI grid dimension must be 1, 2 or 3");
  if (n < 1) fail(GK_ERR_ARG, "D-SKI needs at least one point");
  if (order != 0 && order != 1) fail(GK_ERR_ARG, "interpolation order must be 0 (quintic) or 1 (cubic)");
  DeviceGuard dg(device);
  const bool bprof = std::getenv("GK_BUILD_PROF") != nullptr;
  auto bt0 = std::chrono::steady_clock::now();
  auto bmark = [&](const char* what) {
    if (!bprof) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "dski build: %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t - bt0).count());
    bt0 = t;
  };
  auto op = std::make_unique<DskiOp>();
  op->kind = KIND_DSKI;
  op->device = device;
  op->d = g.d;
  op->T = order == 0 ? 6 : 4;
  op->G = with_grad ? g.d : 0;
  op->n = n;
  op->N = n * (op->G + 1);
  op->n_value = n;
  op->nv2 = nv * nv;
  op->ng2 = ng * ng;
  op->grid = g;
  op->kernel = k;
  const int d = g.d, T = op->T;
  op->M = 1;
  for (int j = 0; j < d; ++j) {
    if (g.dims[j] < T) fail(GK_ERR_ARG, "grid needs at least as many nodes as stencil taps per dimension");
    op->m[j] = g.dims[j];
    op->nb[j] = g.dims[j] - T + 1;
    op->M *= g.dims[j];
  }
  // Toeplitz sequences t_j[k] = exp(-(k h_j)²/(2ℓ²)), s² folded into axis 0
  // (SE profile, kernels.cpp:22-27 / dski.cpp:30-34).
  std::vector<double> tv;
  op->toff_h.resize(static_cast<size_t>(d));
  op->band.resize(static_cast<size_t>(d));
  const double ell2 = k.lengthscale * k.lengthscale;
  for (int j = 0; j < d; ++j) {
    op->toff_h[static_cast<size_t>(j)] = int(tv.size());
    int band = g.dims[j];
    double peak = 0.0;
    for (int kk = 0; kk < g.dims[j]; ++kk) {
      const double o = kk * g.spacing[j];
      double val = std::exp(-0.5 * o * o / ell2);
      if (j == 0) val *= k.outputscale * k.outputscale;
      if (profile == 1) val *= o * o / ell2;  // SE: dk/dlog(ell) = k ρ² (kernels.cpp:172-181)
      tv.push_back(val);
      peak = std::max(peak, std::fabs(val));
    }
    // numerical band: beyond the peak the profile decays monotonically; entries
    // below 1e-30 of the peak contribute far below fp64 roundoff of the
    // product and are skipped tile-wise.
    for (int kk = g.dims[j] - 1; kk >= 0; --kk)
      if (std::fabs(tv[static_cast<size_t>(op->toff_h[static_cast<size_t>(j)] + kk)]) >= 1e-30 * peak) {
        band = kk + 1;
        break;
      }
    op->band[static_cast<size_t>(j)] = band;
  }
  std::vector<double> tvd(tv.size());
  op->band_dl.resize(static_cast<size_t>(d));
  for (int j = 0; j < d; ++j) {
    const int off = op->toff_h[static_cast<size_t>(j)];
    double peak = 0.0;
    for (int kk = 0; kk < g.dims[j]; ++kk) {
      const double o = kk * g.spacing[j];
      tvd[static_cast<size_t>(off + kk)] = tv[static_cast<size_t>(off + kk)] * (o * o / ell2);
      peak = std::max(peak, std::fabs(tvd[static_cast<size_t>(off + kk)]));
    }
    int band = g.dims[j];
    for (int kk = g.dims[j] - 1; kk >= 0; --kk)
      if (std::fabs(tvd[static_cast<size_t>(off + kk)]) >= 1e-30 * peak) {
        band = kk + 1;
        break;
      }
    op->band_dl[static_cast<size_t>(j)] = band;
  }
  const int STRIDE = d * 2 * T;
  i64 ncells = 1;
  for (int j = 0; j < d; ++j) ncells *= op->nb[j];
  op->init_stream();
  cudaStream_t st = op->stream;
  if (k.family != 0) {  // general profile: circulant embedding + FFT (dski.cpp:80-172)
    op->generic = true;
    op->kfft = std::make_unique<KuuFft>();
    op->kfft->init(d, op->m);
    if (slice_ref) {
      i64 tot = 1, ttot = 1;
      for (int j = 0; j < d; ++j) {
        tot *= 2 * (op->m[j] - 1);
        ttot *= 2 * T - 1;
      }
      op->kfft->build(slice_from_reference(*op->kfft, std::vector<double>(slice_ref, slice_ref + tot)), st);
      op->slice_ref_h.assign(slice_ref, slice_ref + tot);
      op->gtab.upload(offset_table, static_cast<size_t>(ttot), st);
      GK_CUDA(cudaStreamSynchronize(st));
    } else {
      op->kfft->build(embedded_slice(k, g, op->kfft->E, false), st);
    }
  }
  std::vector<int> cstart;
  std::vector<i64> ext;
  const bool host_build = g_tuning.devbuild.load() != 0 || ncells >= (i64(1) << 31) || n >= (i64(1) << 31);
  if (!host_build) {
    // on-device point tables (bit-identical to the host build below)
    PtGeom pg{};
    pg.d = d;
    pg.T = T;
    for (int j = 0; j < d; ++j) {
      pg.origin[j] = g.origin[j];
      pg.h[j] = g.spacing[j];
      pg.m[j] = g.dims[j];
      pg.nb[j] = op->nb[j];
    }
    DevBuf<double> Xd(static_cast<size_t>(n) * d), wts_o(static_cast<size_t>(n) * STRIDE);
    DevBuf<int> base_o(static_cast<size_t>(n) * 4), key(static_cast<size_t>(n)), key_s(static_cast<size_t>(n)),
        idx(static_cast<size_t>(n)), perm(static_cast<size_t>(n)), bad(1);
    Xd.upload(X, static_cast<size_t>(n) * d, st);
    const int big = INT_MAX;
    GK_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_pts_weights<<<grid_blocks(n), 256, 0, st>>>(pg, Xd.p, n, base_o.p, wts_o.p, key.p, bad.p);
    launched("dski build: stencils");
    int badh = INT_MAX;
    GK_CUDA(cudaMemcpyAsync(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    if (badh != INT_MAX) {  // the host formula names the point and axis (OutOfGridError text)
      int bb;
      std::vector<double> w(static_cast<size_t>(T)), dw(static_cast<size_t>(T));
      for (int j = 0; j < d; ++j)
        axis_weights(X[j * n + badh], g.origin[j], g.spacing[j], g.dims[j], T, badh, j, &bb, w.data(), dw.data());
      fail(GK_ERR_OUT_OF_GRID, "point " + std::to_string(badh) + " lies outside the interior of the grid", badh);
    }
    std::vector<int> iota(static_cast<size_t>(n));
    std::iota(iota.begin(), iota.end(), 0);
    idx.upload(iota.data(), iota.size(), st);
    int bits = 1;
    while ((i64(1) << bits) < ncells) ++bits;
    size_t tmp_bytes = 0;
    GK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.p, key_s.p, idx.p, perm.p, int(n), 0, bits, st));
    DevBuf<unsigned char> tmp(tmp_bytes);
    GK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key.p, key_s.p, idx.p, perm.p, int(n), 0, bits, st));
    launched("dski build: radix sort");
    op->cell_start.alloc(static_cast<size_t>(ncells) + 1);
    k_cell_start<<<grid_blocks(n), 256, 0, st>>>(key_s.p, n, ncells, op->cell_start.p);
    launched("dski build: cell starts");
    op->base.alloc(static_cast<size_t>(n));
    op->wts.alloc(static_cast<size_t>(n) * STRIDE);
    op->wd.alloc(static_cast<size_t>(n) * d * T);
    op->ext.alloc(static_cast<size_t>(op->N));
    k_gather_pts<<<grid_blocks(n), 256, 0, st>>>(perm.p, base_o.p, wts_o.p, n, d, T, op->G, op->base.p, op->wts.p,
                                                 op->wd.p, op->ext.p);
    launched("dski build: sorted tables");
    // host copies the operator keeps: cell starts (plans, d = 3 lists), the permutation
    cstart.resize(static_cast<size_t>(ncells) + 1);
    std::vector<int> ph(static_cast<size_t>(n));
    GK_CUDA(cudaMemcpyAsync(cstart.data(), op->cell_start.p, sizeof(int) * cstart.size(), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaMemcpyAsync(ph.data(), perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    op->perm_h.resize(static_cast<size_t>(n));
    op->inv_h.resize(static_cast<size_t>(n));
    for (i64 q = 0; q < n; ++q) {
      op->perm_h[static_cast<size_t>(q)] = ph[static_cast<size_t>(q)];
      op->inv_h[static_cast<size_t>(ph[static_cast<size_t>(q)])] = q;
    }
    if (d == 2)
      for (int br = 0; br < op->nb[0]; ++br)
        op->max_row_pts = std::max(op->max_row_pts, cstart[static_cast<size_t>(br + 1) * op->nb[1]] -
                                                        cstart[static_cast<size_t>(br) * op->nb[1]]);
    op->cell_start_h = cstart;
    bmark("device point tables");
  } else {
  // per-point stencils in original order (interpolation.cpp:66-97)
  std::vector<int> base(static_cast<size_t>(n) * d);
  std::vector<double> wts(static_cast<size_t>(n) * STRIDE);
  for (i64 i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j)
      axis_weights(X[j * n + i], g.origin[j], g.spacing[j], g.dims[j], T, i, j,
                   &base[static_cast<size_t>(i) * d + j], &wts[static_cast<size_t>(i) * STRIDE + j * 2 * T],
                   &wts[static_cast<size_t>(i) * STRIDE + j * 2 * T + T]);
  bmark("stencil weights");
  // sort by base cell (counting sort: stable, deterministic)
  std::vector<i64> cell(static_cast<size_t>(n));
  cstart.assign(static_cast<size_t>(ncells) + 1, 0);
  for (i64 i = 0; i < n; ++i) {
    i64 c = 0;
    for (int j = 0; j < d; ++j) c = c * op->nb[j] + base[static_cast<size_t>(i) * d + j];
    cell[static_cast<size_t>(i)] = c;
    cstart[static_cast<size_t>(c) + 1]++;
  }
  for (i64 c = 0; c < ncells; ++c) cstart[static_cast<size_t>(c) + 1] += cstart[static_cast<size_t>(c)];
  if (d == 2)
    for (int br = 0; br < op->nb[0]; ++br)
      op->max_row_pts = std::max(op->max_row_pts, cstart[static_cast<size_t>(br + 1) * op->nb[1]] -
                                                      cstart[static_cast<size_t>(br) * op->nb[1]]);
  op->perm_h.assign(static_cast<size_t>(n), 0);
  op->inv_h.assign(static_cast<size_t>(n), 0);
  {
    std::vector<int> fill(cstart.begin(), cstart.end() - 1);
    for (i64 i = 0; i < n; ++i) {
      const int pos = fill[static_cast<size_t>(cell[static_cast<size_t>(i)])]++;
      op->perm_h[static_cast<size_t>(pos)] = i;
      op->inv_h[static_cast<size_t>(i)] = pos;
    }
  }
  std::vector<int4> base_s(static_cast<size_t>(n));
  std::vector<double> wts_s(static_cast<size_t>(n) * STRIDE);
  for (i64 s = 0; s < n; ++s) {
    const i64 i = op->perm_h[static_cast<size_t>(s)];
    int4 b4 = make_int4(0, 0, 0, 0);
    b4.x = base[static_cast<size_t>(i) * d + 0];
    if (d > 1) b4.y = base[static_cast<size_t>(i) * d + 1];
    if (d > 2) b4.z = base[static_cast<size_t>(i) * d + 2];
    base_s[static_cast<size_t>(s)] = b4;
    std::memcpy(&wts_s[static_cast<size_t>(s) * STRIDE], &wts[static_cast<size_t>(i) * STRIDE], sizeof(double) * STRIDE);
  }
  ext.resize(static_cast<size_t>(op->N));
  for (int gg = 0; gg <= op->G; ++gg)
    for (i64 s = 0; s < n; ++s) ext[static_cast<size_t>(gg * n + s)] = gg * n + op->perm_h[static_cast<size_t>(s)];
  bmark("sort + host tables");
  op->base.upload(base_s.data(), base_s.size(), st);
  op->wts.upload(wts_s.data(), wts_s.size(), st);
  {
    std::vector<double2> wd(static_cast<size_t>(n) * d * T);
    for (i64 q = 0; q < n; ++q)
      for (int j = 0; j < d; ++j)
        for (int t = 0; t < T; ++t) {
          const double* r = &wts_s[static_cast<size_t>(q) * STRIDE + j * 2 * T];
          wd[(static_cast<size_t>(q) * d + j) * T + t] = make_double2(r[t], r[T + t]);
        }
    op->wd.upload(wd.data(), wd.size(), st);
  }
  op->cell_start.upload(cstart.data(), cstart.size(), st);
  op->cell_start_h = cstart;
  op->ext.upload(ext.data(), ext.size(), st);
  }
  if (d == 2 && op->G == 2) {
    op->rec.alloc(static_cast<size_t>(n) * (2 * T + 1));
    k_pack_records<<<grid_blocks(n), 256, 0, st>>>(op->wd.p, op->base.p, n, T, op->rec.p);
    launched("dski build: scatter records");
  }
  if (d == 3) {  // gather units: runs of ≤ kZU occupied base cells along z per cell line
    constexpr int kZU = 4;
    const int nb1 = op->nb[1], nb2 = op->nb[2];
    std::vector<int4> gu;
    std::vector<int2> gr;
    int zspan = 0;
    for (int b0 = 0; b0 < op->nb[0]; ++b0)
      for (int b1 = 0; b1 < nb1; ++b1) {
        const size_t c0 = (static_cast<size_t>(b0) * nb1 + b1) * nb2;
        int b2 = 0;
        while (b2 < nb2) {
          if (cstart[c0 + b2 + 1] == cstart[c0 + b2]) {
            ++b2;
            continue;
          }
          const int za = b2;
          int zb = b2;
          while (zb < nb2 && zb - za < kZU && (zb == za || cstart[c0 + zb + 1] > cstart[c0 + zb])) ++zb;
          gu.push_back(make_int4(b0, b1, za, zb));
          gr.push_back(make_int2(cstart[c0 + za], cstart[c0 + zb]));
          zspan = std::max(zspan, zb - za + T - 1);
          b2 = zb;
        }
      }
    op->g3_nunits = int(gu.size());
    op->g3_zspan = zspan;
    op->g3_units.upload(gu.data(), gu.size(), op->stream);
    op->g3_range.upload(gr.data(), gr.size(), op->stream);
    // unit-push scatter tables
    const int m1 = g.dims[1], m2 = g.dims[2], ncol = g.dims[0] * m1;
    std::vector<long long> uoff(gu.size());
    long long tot = 0;
    std::vector<std::vector<int2>> per(static_cast<size_t>(ncol));
    for (size_t ui = 0; ui < gu.size(); ++ui) {
      const int nzb = gu[ui].w - gu[ui].z + T - 1;
      uoff[ui] = tot;
      tot += static_cast<long long>(T) * T * nzb;
      for (int a = 0; a < T; ++a)
        for (int b = 0; b < T; ++b)
          per[static_cast<size_t>((gu[ui].x + a) * m1 + gu[ui].y + b)].push_back(make_int2(int(ui), a * T + b));
    }
    const int nzs = (m2 + 7) / 8;
    std::vector<int> cst(static_cast<size_t>(ncol) + 1, 0), cseg(static_cast<size_t>(ncol) * nzs);
    std::vector<int2> cent;
    std::vector<int> zoff(static_cast<size_t>(ncol) * m2 + 1, 0), zlist;
    int maxl = 0;
    for (int c = 0; c < ncol; ++c) {
      auto& L = per[static_cast<size_t>(c)];
      std::stable_sort(L.begin(), L.end(), [&](const int2& x, const int2& y) {
        return gu[static_cast<size_t>(x.x)].z < gu[static_cast<size_t>(y.x)].z;  // (za, unit): units already ascending
      });
      cst[static_cast<size_t>(c)] = int(cent.size());
      for (int zs = 0; zs < nzs; ++zs) {  // first entry whose block can reach segment zs
        size_t e = 0;
        while (e < L.size() && gu[static_cast<size_t>(L[e].x)].z + zspan <= zs * 8) ++e;
        cseg[static_cast<size_t>(c) * nzs + zs] = int(cent.size() + e);
      }
      {  // flattened per-node lists of this column: count per z, prefix sum,
         // fill in entry order (O(blocks · nzb), entry order kept per node)
        const size_t l0 = zlist.size();
        std::vector<int> cnt(static_cast<size_t>(m2) + 1, 0);
        for (const int2& en : L) {
          const int4& U = gu[static_cast<size_t>(en.x)];
          const int nzb = U.w - U.z + T - 1;
          for (int z = U.z; z < std::min(m2, U.z + nzb); ++z) ++cnt[static_cast<size_t>(z) + 1];
        }
        for (int z = 0; z < m2; ++z) cnt[static_cast<size_t>(z) + 1] += cnt[static_cast<size_t>(z)];
        for (int z = 0; z < m2; ++z) zoff[static_cast<size_t>(c) * m2 + z] = int(l0) + cnt[static_cast<size_t>(z)];
        zlist.resize(l0 + static_cast<size_t>(cnt[static_cast<size_t>(m2)]));
        for (const int2& en : L) {
          const int4& U = gu[static_cast<size_t>(en.x)];
          const int nzb = U.w - U.z + T - 1;
          const long long o = uoff[static_cast<size_t>(en.x)] + static_cast<long long>(en.y) * nzb;
          for (int z = U.z; z < std::min(m2, U.z + nzb); ++z)
            zlist[l0 + static_cast<size_t>(cnt[static_cast<size_t>(z)]++)] = int(o + (z - U.z));
        }
        maxl = std::max(maxl, int(zlist.size() - l0));
      }
      cent.insert(cent.end(), L.begin(), L.end());
    }
    cst[static_cast<size_t>(ncol)] = int(cent.size());
    op->s3_nodes = tot;
    op->s3_nzs = nzs;
    op->s3_uoff.upload(uoff.data(), uoff.size(), op->stream);
    op->s3_cstart.upload(cst.data(), cst.size(), op->stream);
    op->s3_cseg.upload(cseg.data(), cseg.size(), op->stream);
    op->s3_cent.upload(cent.data(), std::max<size_t>(cent.size(), 1), op->stream);
    zoff[static_cast<size_t>(ncol) * m2] = int(zlist.size());
    if (tot < (1LL << 31)) {
      if (zlist.empty()) zlist.push_back(0);
      op->s3_zoff.upload(zoff.data(), zoff.size(), op->stream);
      op->s3_zlist.upload(zlist.data(), zlist.size(), op->stream);
      op->s3_maxl = maxl;
    }
  }
  if (d == 3) {  // per node column (k0, k1): covering points ordered by (b2, t0, t1, point)
    const int m0 = g.dims[0], m1 = g.dims[1], m2 = g.dims[2];
    const int nb0 = op->nb[0], nb1 = op->nb[1], nb2 = op->nb[2];
    const int ncol = m0 * m1;
    std::vector<int> start(static_cast<size_t>(ncol) + 1, 0);
    for (int k0 = 0; k0 < m0; ++k0)
      for (int k1 = 0; k1 < m1; ++k1) {
        int cnt = 0;
        for (int t0 = 0; t0 < T; ++t0)
          for (int t1 = 0; t1 < T; ++t1) {
            const int b0 = k0 - t0, b1 = k1 - t1;
            if (b0 < 0 || b0 >= nb0 || b1 < 0 || b1 >= nb1) continue;
            const int c = (b0 * nb1 + b1) * nb2;
            cnt += cstart[static_cast<size_t>(c + nb2)] - cstart[static_cast<size_t>(c)];
          }
        start[static_cast<size_t>(k0 * m1 + k1) + 1] = cnt;
      }
    for (int c = 0; c < ncol; ++c) start[static_cast<size_t>(c) + 1] += start[static_cast<size_t>(c)];
    const int zseg = op->col3_zseg, nseg = (m2 + zseg - 1) / zseg;
    std::vector<int2> list(static_cast<size_t>(start[static_cast<size_t>(ncol)]));
    std::vector<int> segs(static_cast<size_t>(ncol) * nseg);
    for (int k0 = 0; k0 < m0; ++k0)
      for (int k1 = 0; k1 < m1; ++k1) {
        const int col = k0 * m1 + k1;
        int e = start[static_cast<size_t>(col)];
        int sg = 0;
        for (int b2 = 0; b2 < nb2; ++b2) {
          while (sg < nseg && b2 >= std::max(0, sg * zseg - (T - 1))) segs[static_cast<size_t>(col) * nseg + sg++] = e;
          for (int t0 = 0; t0 < T; ++t0)
            for (int t1 = 0; t1 < T; ++t1) {
              const int b0 = k0 - t0, b1 = k1 - t1;
              if (b0 < 0 || b0 >= nb0 || b1 < 0 || b1 >= nb1) continue;
              const int c = (b0 * nb1 + b1) * nb2 + b2;
              for (int q = cstart[static_cast<size_t>(c)]; q < cstart[static_cast<size_t>(c) + 1]; ++q)
                list[static_cast<size_t>(e++)] = make_int2(q, (b2 << 8) | (t0 << 4) | t1);
            }
        }
        while (sg < nseg) segs[static_cast<size_t>(col) * nseg + sg++] = e;
      }
    // balanced units: ~64 entries with b2 in [za, zb) each (+ the T−1 halo cells)
    std::vector<int4> units;
    constexpr int kUnitEntries = 64;
    for (int col = 0; col < ncol; ++col) {
      const int e0 = start[static_cast<size_t>(col)], e1 = start[static_cast<size_t>(col) + 1];
      if (e0 == e1) continue;
      const int zfirst = list[static_cast<size_t>(e0)].y >> 8;
      const int zend = std::min(m2, (list[static_cast<size_t>(e1 - 1)].y >> 8) + T);
      int za = zfirst, ea = e0;  // ea: first entry with b2 >= za
      while (za < zend) {
        int eh = ea;  // first entry with b2 >= za - (T - 1) (the window's halo cells)
        while (eh > e0 && (list[static_cast<size_t>(eh - 1)].y >> 8) >= za - (T - 1)) --eh;
        int zb = za, eb = ea, cnt = 0;
        while (zb < zend) {
          int e = eb;
          while (e < e1 && (list[static_cast<size_t>(e)].y >> 8) == zb) ++e;
          if (cnt > 0 && cnt + (e - eb) > kUnitEntries) break;
          cnt += e - eb;
          eb = e;
          ++zb;
        }
        units.push_back(make_int4(col, za, zb, eh));
        za = zb;
        ea = eb;
      }
    }
    op->col3_nunits = int(units.size());
    op->col3_units.upload(units.data(), units.size(), st);
    if (m2 < 65536) {  // tile lists for k_scatter_tile3 (z packed in 16 bits)
      const int TB = op->tile3_tb;
      const int tiles0 = (m0 + TB - 1) / TB, tiles1 = (m1 + TB - 1) / TB;
      std::vector<int> tl;
      std::vector<int4> tu;
      std::vector<int> zs;  // b2 of each entry of the current tile
      constexpr int kTileEntries = 192;
      for (int K0 = 0; K0 < tiles0; ++K0)
        for (int K1 = 0; K1 < tiles1; ++K1) {
          const int e0 = int(tl.size());
          zs.clear();
          const int blo = std::max(0, K0 * TB - (T - 1)), bhi = std::min(nb0 - 1, K0 * TB + TB - 1);
          const int clo = std::max(0, K1 * TB - (T - 1)), chi = std::min(nb1 - 1, K1 * TB + TB - 1);
          for (int b2 = 0; b2 < nb2; ++b2)
            for (int b0 = blo; b0 <= bhi; ++b0)
              for (int b1 = clo; b1 <= chi; ++b1) {
                const int cc = (b0 * nb1 + b1) * nb2 + b2;
                for (int q = cstart[static_cast<size_t>(cc)]; q < cstart[static_cast<size_t>(cc) + 1]; ++q) {
                  tl.push_back(q);
                  zs.push_back(b2);
                }
              }
          const int e1 = int(tl.size()), ne = e1 - e0;
          // units partition [0, m2): ~kTileEntries entries with b2 in [za, zb)
          int za = 0, ia = 0;  // ia: first local entry with b2 >= za
          const int tile = K0 * tiles1 + K1;
          while (za < m2) {
            int ih = ia;
            while (ih > 0 && zs[static_cast<size_t>(ih - 1)] >= za - (T - 1)) --ih;
            int zb = za, ib = ia, cnt = 0;
            while (zb < m2) {
              int i = ib;
              while (i < ne && zs[static_cast<size_t>(i)] == zb) ++i;
              if (cnt > 0 && cnt + (i - ib) > kTileEntries) break;
              cnt += i - ib;
              ib = i;
              ++zb;
            }
            if (ib >= ne) zb = m2;  // the last unit of the tile runs to the top
            tu.push_back(make_int4(tile, za | (zb << 16), e0 + ih, e0 + ib));
            za = zb;
            ia = ib;
          }
        }
      op->tile3_tiles1 = tiles1;
      op->tile3_nunits = int(tu.size());
      op->tile3_list.upload(tl.data(), std::max<size_t>(1, tl.size()), st);
      op->tile3_units.upload(tu.data(), tu.size(), st);
    }
    op->col3_nseg = nseg;
    op->col3_list.upload(list.data(), list.size(), st);
    op->col3_start.upload(start.data(), start.size(), st);
    op->col3_seg.upload(segs.data(), segs.size(), st);
  }
  op->tvec.upload(tv.data(), tv.size(), st);
  op->tvec_dl.upload(tvd.data(), tvd.size(), st);
  op->toff.upload(op->toff_h.data(), op->toff_h.size(), st);
  double o3[3] = {0, 0, 0}, h3[3] = {1, 1, 1};
  for (int j = 0; j < d; ++j) {
    o3[j] = g.origin[j];
    h3[j] = g.spacing[j];
  }
  op->origin_d.upload(o3, 3, st);
  op->h_d.upload(h3, 3, st);
  GK_CUDA(cudaStreamSynchronize(st));
  bmark("uploads");
  return op;
}

// ---------------------------------------------------------------- D-SKI extras
int64_t dski_grid_size(const Op& o) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  return static_cast<const DskiOp&>(o).M;
}
gk_grid dski_grid(const Op& o) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  return static_cast<const DskiOp&>(o).grid;
}
double dski_min_embedding_eigenvalue(const Op& o) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  return static_cast<const DskiOp&>(o).min_embedding_eigenvalue();
}

// B K_UU B^T without the noise diagonal (internal layout), for D-SKIP leaves.
void dski_mvm_nonoise(Op& o, const double* in, double* out, int nrhs, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(nrhs);
  op.scatter(in, op.grid_u.p, nrhs, s);
  op.kuu(op.grid_u.p, op.grid_w.p, nrhs, s);
  op.gather(op.grid_w.p, in, out, nrhs, false, s);
}

// Scatter with grid output (internal V -> grid U), grid K_UU and gather w/o noise.
void dski_transpose_apply(Op& o, const double* Vi, double* U, int nrhs, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.scatter(Vi, U, nrhs, s);
}
void dski_gather_noise(Op& o, const double* W, const double* V, double* out, int nrhs, cudaStream_t s) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  auto& op = static_cast<DskiOp&>(o);
  op.gather(W, V, out, nrhs, true, s);
}
void dski_apply(Op& o, const double* U, double* Oi, int nrhs, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.gather(U, U, Oi, nrhs, false, s);
}
// ∂K∇/∂log ℓ · v = B (∂K_UU/∂log ℓ) Bᵀ v, no noise (GpModel::dlogell_apply, gp.cpp:212-213)
void dski_dlogell(Op& o, const double* Vi, double* Oi, int nrhs, cudaStream_t s) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(nrhs);
  op.scatter(Vi, op.grid_u.p, nrhs, s);
  op.kuu_dlogell(op.grid_u.p, op.grid_w.p, nrhs, s);
  op.gather(op.grid_w.p, op.grid_w.p, Oi, nrhs, false, s);
}

void dski_grid_mvm(Op& o, const double* U, double* W, int nrhs, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(nrhs);
  op.kuu(U, W, nrhs, s);
}

// predict_mean_grad (gp.cpp:471-496) given alpha (internal layout, 1 column)
void dski_predict(Op& o, const double* alpha_i, double mean, const double* dXt, i64 nT, double* dvals,
                  double* dgrads, int* dbad, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(1);
  DevBuf<double> g(static_cast<size_t>(op.M)), tmp(static_cast<size_t>(op.M));
  op.scatter(alpha_i, tmp.p, 1, s);
  op.kuu(tmp.p, g.p, 1, s);
  const DskiView vw = op.view();
  GK_DISPATCH_DT(op.d, op.T, {
    k_predict<D, T><<<grid_blocks(nT), 256, 0, s>>>(vw, dXt, nT, op.origin_d.p, op.h_d.p, g.p, mean,
                                                     dvals, dgrads, dbad);
  });
  launched("dski predict");
  GK_CUDA(cudaStreamSynchronize(s));
}

// cross_covariance for T test points (gp.cpp:412-417): Q = B K_UU w_t.
void dski_cross_cov(Op& o, const double* dXt, i64 nT, double* Qi, int* dbad, cudaStream_t s, int dir) {
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(int(nT));
  DevBuf<double> U(static_cast<size_t>(op.M) * nT), W(static_cast<size_t>(op.M) * nT);
  GK_CUDA(cudaMemsetAsync(U.p, 0, sizeof(double) * op.M * nT, s));
  const DskiView vw = op.view();
  GK_DISPATCH_DT(op.d, op.T, {
    k_test_stencils<D, T><<<grid_blocks(nT), 256, 0, s>>>(vw, dXt, nT, op.origin_d.p, op.h_d.p, U.p, dbad, dir);
  });
  launched("dski test stencils");
  op.kuu(U.p, W.p, int(nT), s);
  op.gather(W.p, W.p, Qi, int(nT), false, s);
  GK_CUDA(cudaStreamSynchronize(s));
}

// Device-pointer cross-covariance (gp.cpp:412-417 / 431-461 for one stencil
// direction): columns B K_UU w(x_t) for nT test points (dXt nT×d col-major,
// device) written in EXTERNAL row order into dQ (ld ldq); the operator's grid
// scratch is reused (no allocation); one synchronisation for the
// out-of-grid check. dir < 0: value stencil, else ∂/∂x_dir.
void dski_cross_cov_dev(Op& o, const double* dXt, i64 nT, int dir, double* dQ, i64 ldq, cudaStream_t s) {
  auto& op = static_cast<DskiOp&>(o);
  op.ensure_scratch(int(nT));
  op.scratch_a.reserve(static_cast<size_t>(op.N) * nT);
  op.oog.reserve(1);
  const int big = INT_MAX;
  GK_CUDA(cudaMemcpyAsync(op.oog.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  GK_CUDA(cudaMemsetAsync(op.grid_u.p, 0, sizeof(double) * op.M * nT, s));
  const DskiView vw = op.view();
  GK_DISPATCH_DT(op.d, op.T, {
    k_test_stencils<D, T><<<grid_blocks(nT), 256, 0, s>>>(vw, dXt, nT, op.origin_d.p, op.h_d.p, op.grid_u.p, op.oog.p, dir);
  });
  launched("dski test stencils");
  op.kuu(op.grid_u.p, op.grid_w.p, int(nT), s);
  op.gather(op.grid_w.p, op.grid_w.p, op.scratch_a.p, int(nT), false, s);
  op.from_internal(op.scratch_a.p, dQ, ldq, int(nT), s);
  int badh = INT_MAX;
  GK_CUDA(cudaMemcpyAsync(&badh, op.oog.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  if (badh != INT_MAX)
    fail(GK_ERR_OUT_OF_GRID, "test point " + std::to_string(badh) + " lies outside the interior of the grid", badh);
}

}  // namespace gk

namespace gk {
// gk_debug_fused_phases backend
bool dski_fused_split(Op& o, int phase, const double* v, double* u2, double* out, int nrhs, cudaStream_t s) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  return static_cast<DskiOp&>(o).fused_split(phase, v, u2, out, nrhs, s);
}

int dski_fused_phases(Op& o, int nrhs, i64* out, int max_ctas) {
  if (o.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
  auto& op = static_cast<DskiOp&>(o);
  for (auto& p : op.lplans)
    if (p->nrhs == nrhs && p->ok && p->prof.p) {
      const int n = std::min(p->grid, max_ctas);
      std::vector<i64> h(p->prof.n);
      GK_CUDA(cudaDeviceSynchronize());
      GK_CUDA(cudaMemcpy(h.data(), p->prof.p, sizeof(i64) * h.size(), cudaMemcpyDeviceToHost));
      for (int c = 0; c < n; ++c)
        for (int k = 0; k < 8; ++k) out[size_t(c) * 8 + k] = h[size_t(c) * 8 + k];
      return n;
    }
  for (auto& p : op.fplans)
    if (p->nrhs == nrhs && p->ok && p->prof.p) {
      const int n = std::min(p->grid, max_ctas);
      const size_t slots = 8;
      std::vector<i64> h(p->prof.n);
      GK_CUDA(cudaDeviceSynchronize());
      GK_CUDA(cudaMemcpy(h.data(), p->prof.p, sizeof(i64) * h.size(), cudaMemcpyDeviceToHost));
      for (int c = 0; c < n; ++c)
        for (int k = 0; k < 8; ++k) out[size_t(c) * 8 + k] = h[size_t(c) * slots + k];
      if (const char* f = std::getenv("GK_FUSED_PROF_DUMP")) {
        if (FILE* fp = std::fopen(f, "wb")) {
          std::fwrite(h.data(), sizeof(i64), h.size(), fp);
          std::fclose(fp);
        }
      }
      return n;
    }
  return 0;
}
}  // namespace gk
