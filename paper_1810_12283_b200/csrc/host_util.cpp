// host_util.cpp — host-side pieces of libgk_b200 that are inherently
// sequential and tiny: seeded RNG streams (must reproduce the reference's
// libstdc++ std::mt19937_64 / normal_distribution bit for bit), the
// tridiagonal eigensolver for SLQ quadrature, a k×k Cholesky for the
// preconditioner QR, Grid::cover, and the seeded synthetic datasets.
#include <mutex>
#include <utility>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>

#include "gk_common.hpp"

namespace gk {

std::atomic<i64> g_launches{0};
Tuning g_tuning;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(GK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// rng.hpp:12-17 (splitmix64 finaliser over seed + golden-ratio * (stream+1))
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// rng.hpp:23-29: sign from bit 0 of each raw 64-bit draw.
void rademacher(i64 n, std::uint64_t seed, std::uint64_t stream, double* out) {
  std::mt19937_64 rng(mix_seed(seed, stream));
  for (i64 i = 0; i < n; ++i) out[i] = (rng() & 1ULL) ? 1.0 : -1.0;
}

// rng.hpp:31-38: libstdc++ normal_distribution over the same engine.
void gaussian(i64 n, std::uint64_t seed, std::uint64_t stream, double* out) {
  std::mt19937_64 rng(mix_seed(seed, stream));
  std::normal_distribution<double> dist(0.0, 1.0);
  for (i64 i = 0; i < n; ++i) out[i] = dist(rng);
}

// std::uniform_real_distribution<double>(a, b) over seeded_rng(seed, stream)
// (libstdc++: one 64-bit draw per value, generate_canonical · (b − a) + a);
// the restart jitter of GpModel::fit (gp.cpp:328-331).
void uniform(i64 n, std::uint64_t seed, std::uint64_t stream, double a, double b, double* out) {
  std::mt19937_64 rng(mix_seed(seed, stream));
  std::uniform_real_distribution<double> dist(a, b);
  for (i64 i = 0; i < n; ++i) out[i] = dist(rng);
}

// Symmetric tridiagonal QL iteration with implicit shifts; eigenvectors are
// rotated along (Z = I initially) so Z's first row gives the Gauss
// quadrature weights SLQ needs (linalg.cpp:231-245).
void tridiag_eig(int n, const double* alpha, const double* beta, double* evals, double* Zout) {
  std::vector<double> dg(alpha, alpha + n), off(static_cast<size_t>(n), 0.0);
  for (int i = 0; i + 1 < n; ++i) off[static_cast<size_t>(i)] = beta[i];
  std::vector<double> Z(static_cast<size_t>(n) * static_cast<size_t>(n), 0.0);
  for (int i = 0; i < n; ++i) Z[static_cast<size_t>(i) * n + i] = 1.0;
  auto z = [&](int r, int c) -> double& { return Z[static_cast<size_t>(c) * n + r]; };
  const double eps = std::numeric_limits<double>::epsilon();
  for (int l = 0; l < n; ++l) {
    for (int iter = 0;; ++iter) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double s = std::fabs(dg[static_cast<size_t>(m)]) + std::fabs(dg[static_cast<size_t>(m + 1)]);
        if (std::fabs(off[static_cast<size_t>(m)]) <= eps * s) break;
      }
      if (m == l) break;
      if (iter > 300) fail(GK_ERR_RUNTIME, "tridiagonal eigensolver did not converge");
      double g = (dg[static_cast<size_t>(l + 1)] - dg[static_cast<size_t>(l)]) / (2.0 * off[static_cast<size_t>(l)]);
      double r = std::hypot(g, 1.0);
      g = dg[static_cast<size_t>(m)] - dg[static_cast<size_t>(l)] + off[static_cast<size_t>(l)] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      bool underflow = false;
      for (; i >= l; --i) {
        double f = s * off[static_cast<size_t>(i)];
        const double b = c * off[static_cast<size_t>(i)];
        r = std::hypot(f, g);
        off[static_cast<size_t>(i + 1)] = r;
        if (r == 0.0) {
          dg[static_cast<size_t>(i + 1)] -= p;
          off[static_cast<size_t>(m)] = 0.0;
          underflow = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = dg[static_cast<size_t>(i + 1)] - p;
        r = (dg[static_cast<size_t>(i)] - g) * s + 2.0 * c * b;
        p = s * r;
        dg[static_cast<size_t>(i + 1)] = g + p;
        g = c * r - b;
        for (int k = 0; k < n; ++k) {
          f = z(k, i + 1);
          z(k, i + 1) = s * z(k, i) + c * f;
          z(k, i) = c * z(k, i) - s * f;
        }
      }
      if (underflow) continue;
      dg[static_cast<size_t>(l)] -= p;
      off[static_cast<size_t>(l)] = g;
      off[static_cast<size_t>(m)] = 0.0;
    }
  }
  std::vector<int> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return dg[static_cast<size_t>(a)] < dg[static_cast<size_t>(b)]; });
  for (int j = 0; j < n; ++j) {
    evals[j] = dg[static_cast<size_t>(ord[static_cast<size_t>(j)])];
    if (Zout)
      for (int r = 0; r < n; ++r) Zout[static_cast<size_t>(j) * n + r] = z(r, ord[static_cast<size_t>(j)]);
  }
}

void cholesky_upper(int k, const double* A, double* R) {
  // A = R^T R, R upper triangular (col-major); long double accumulation.
  std::fill(R, R + static_cast<size_t>(k) * k, 0.0);
  for (int j = 0; j < k; ++j) {
    for (int i = 0; i <= j; ++i) {
      long double s = A[static_cast<size_t>(j) * k + i];
      for (int p = 0; p < i; ++p) s -= (long double)R[static_cast<size_t>(i) * k + p] * R[static_cast<size_t>(j) * k + p];
      if (i == j) {
        if (!(s > 0.0L)) fail(GK_ERR_RUNTIME, "preconditioner QR: Gram matrix is not positive definite");
        R[static_cast<size_t>(j) * k + j] = (double)sqrtl(s);
      } else {
        R[static_cast<size_t>(j) * k + i] = (double)(s / R[static_cast<size_t>(i) * k + i]);
      }
    }
  }
}

std::uint64_t next_op_uid() {
  static std::atomic<std::uint64_t> counter{1};
  return counter.fetch_add(1);
}

Op::~Op() {
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  for (auto e : io_events) cudaEventDestroy(e);
  if (io_in) cudaStreamDestroy(io_in);
  if (io_out) cudaStreamDestroy(io_out);
  if (io_pin) cudaStreamDestroy(io_pin);
  if (io_pout) cudaStreamDestroy(io_pout);
  if (stream) cudaStreamDestroy(stream);
  if (cap_stream) cudaStreamDestroy(cap_stream);
  if (last_use) cudaEventDestroy(last_use);
}

void Op::init_stream() {
  GK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  GK_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
}

// The dynamic shared memory limit is a per-function attribute shared by every
// plan (and operator) using that instantiation: only ever raise it, so a plan
// built later with less shared memory cannot invalidate an earlier one.
void raise_smem_limit(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> limits;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& l : limits)
    if (l.first == fn) {
      if (bytes > l.second) {
        GK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
        l.second = bytes;
      }
      return;
    }
  GK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max<size_t>(bytes, 48 * 1024))));
  limits.emplace_back(fn, std::max<size_t>(bytes, 48 * 1024));
}


}  // namespace gk

// ==================================================================== datasets
namespace {

using gk::i64;

// Dual number carrying a 3-gradient, for exact normals of the star surface.
struct D3 {
  double v, g[3];
};
D3 mk(double v) { return {v, {0, 0, 0}}; }
D3 operator+(D3 a, D3 b) { return {a.v + b.v, {a.g[0] + b.g[0], a.g[1] + b.g[1], a.g[2] + b.g[2]}}; }
D3 operator-(D3 a, D3 b) { return {a.v - b.v, {a.g[0] - b.g[0], a.g[1] - b.g[1], a.g[2] - b.g[2]}}; }
D3 operator*(D3 a, D3 b) {
  return {a.v * b.v, {a.g[0] * b.v + a.v * b.g[0], a.g[1] * b.v + a.v * b.g[1], a.g[2] * b.v + a.v * b.g[2]}};
}
D3 operator*(double c, D3 a) { return {c * a.v, {c * a.g[0], c * a.g[1], c * a.g[2]}}; }

// 25 orthonormal real spherical harmonics (l <= 4) as polynomials of a unit vector.
void real_sh(const D3& x, const D3& y, const D3& z, D3* Y) {
  const double pi = 3.14159265358979323846;
  const D3 x2 = x * x, y2 = y * y, z2 = z * z, r2 = x2 + y2 + z2;
  int k = 0;
  Y[k++] = mk(0.5 * std::sqrt(1.0 / pi));
  const double c1 = std::sqrt(3.0 / (4.0 * pi));
  Y[k++] = c1 * y;
  Y[k++] = c1 * z;
  Y[k++] = c1 * x;
  const double c2 = 0.5 * std::sqrt(15.0 / pi);
  Y[k++] = c2 * (x * y);
  Y[k++] = c2 * (y * z);
  Y[k++] = (0.25 * std::sqrt(5.0 / pi)) * (3.0 * z2 - r2);
  Y[k++] = c2 * (x * z);
  Y[k++] = (0.25 * std::sqrt(15.0 / pi)) * (x2 - y2);
  Y[k++] = (0.25 * std::sqrt(35.0 / (2 * pi))) * (y * (3.0 * x2 - y2));
  Y[k++] = (0.5 * std::sqrt(105.0 / pi)) * (x * y * z);
  Y[k++] = (0.25 * std::sqrt(21.0 / (2 * pi))) * (y * (5.0 * z2 - r2));
  Y[k++] = (0.25 * std::sqrt(7.0 / pi)) * (z * (5.0 * z2 - 3.0 * r2));
  Y[k++] = (0.25 * std::sqrt(21.0 / (2 * pi))) * (x * (5.0 * z2 - r2));
  Y[k++] = (0.25 * std::sqrt(105.0 / pi)) * (z * (x2 - y2));
  Y[k++] = (0.25 * std::sqrt(35.0 / (2 * pi))) * (x * (x2 - 3.0 * y2));
  Y[k++] = (0.75 * std::sqrt(35.0 / pi)) * (x * y * (x2 - y2));
  Y[k++] = (0.75 * std::sqrt(35.0 / (2 * pi))) * (y * z * (3.0 * x2 - y2));
  Y[k++] = (0.75 * std::sqrt(5.0 / pi)) * (x * y * (7.0 * z2 - r2));
  Y[k++] = (0.75 * std::sqrt(5.0 / (2 * pi))) * (y * z * (7.0 * z2 - 3.0 * r2));
  Y[k++] = ((3.0 / 16.0) * std::sqrt(1.0 / pi)) * (35.0 * (z2 * z2) - 30.0 * (z2 * r2) + 3.0 * (r2 * r2));
  Y[k++] = (0.75 * std::sqrt(5.0 / (2 * pi))) * (x * z * (7.0 * z2 - 3.0 * r2));
  Y[k++] = ((3.0 / 8.0) * std::sqrt(5.0 / pi)) * ((x2 - y2) * (7.0 * z2 - r2));
  Y[k++] = (0.75 * std::sqrt(35.0 / (2 * pi))) * (x * z * (x2 - 3.0 * y2));
  Y[k++] = ((3.0 / 16.0) * std::sqrt(35.0 / pi)) * (x2 * (x2 - 3.0 * y2) - y2 * (3.0 * x2 - y2));
}

}  // namespace

// sample_dataset(fn, n, Uniform, seed, σ₁, σ₂, with_gradients) for the two
// test functions the precond-study tool sweeps (testfns.cpp:67-92 Franke,
// :290-310 Friedman #1, :355-402 sampling): X row by row from
// uniform(0, 1) over seeded_rng(seed), then per point the value and its
// gradient plus σ·N(0, 1) draws from the same engine.
extern "C" gk_status gk_sample_test_function_impl(const char* name, i64 n, std::uint64_t seed, double nv,
                                                  double ng, int with_gradients, int* d_out, double* X,
                                                  double* y, double* dY) {
  const std::string fn(name ? name : "");
  int d = 0;
  if (fn == "franke") d = 2;
  else if (fn == "friedman") d = 5;
  else return GK_ERR_ARG;
  *d_out = d;
  if (!X) return GK_OK;
  std::mt19937_64 rng(gk::mix_seed(seed, 0));
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  for (i64 i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) X[j * n + i] = 0.0 + (1.0 - 0.0) * unif(rng);
  std::normal_distribution<double> gauss(0.0, 1.0);
  const double kPi = 3.14159265358979323846;
  for (i64 i = 0; i < n; ++i) {
    double v, g[5];
    if (d == 2) {
      const double x = X[i], yv = X[n + i];
      const double t1 = 0.75 * std::exp(-(std::pow(9 * x - 2, 2) + std::pow(9 * yv - 2, 2)) / 4.0);
      const double t2 = 0.75 * std::exp(-std::pow(9 * x + 1, 2) / 49.0 - (9 * yv + 1) / 10.0);
      const double t3 = 0.5 * std::exp(-(std::pow(9 * x - 7, 2) + std::pow(9 * yv - 3, 2)) / 4.0);
      const double t4 = -0.2 * std::exp(-std::pow(9 * x - 4, 2) - std::pow(9 * yv - 7, 2));
      v = t1 + t2 + t3 + t4;
      g[0] = t1 * (-9.0 * (9 * x - 2) / 2.0) + t2 * (-18.0 * (9 * x + 1) / 49.0) + t3 * (-9.0 * (9 * x - 7) / 2.0) +
             t4 * (-18.0 * (9 * x - 4));
      g[1] = t1 * (-9.0 * (9 * yv - 2) / 2.0) + t2 * (-9.0 / 10.0) + t3 * (-9.0 * (9 * yv - 3) / 2.0) +
             t4 * (-18.0 * (9 * yv - 7));
    } else {
      double x[5];
      for (int j = 0; j < 5; ++j) x[j] = X[j * n + i];
      v = 10.0 * std::sin(kPi * x[0] * x[1]) + 20.0 * std::pow(x[2] - 0.5, 2) + 10.0 * x[3] + 5.0 * x[4];
      const double c = 10.0 * kPi * std::cos(kPi * x[0] * x[1]);
      g[0] = c * x[1];
      g[1] = c * x[0];
      g[2] = 40.0 * (x[2] - 0.5);
      g[3] = 10.0;
      g[4] = 5.0;
    }
    y[i] = v + nv * gauss(rng);
    if (with_gradients)
      for (int j = 0; j < d; ++j) dY[j * n + i] = g[j] + ng * gauss(rng);
  }
  return GK_OK;
}

extern "C" gk_status gk_make_dataset_impl(int config, std::uint64_t seed, i64* n_out, int* d_out,
                                          double* X, double* y, double* dY) {
  // Streams: 1 = inputs, 2 = target parameters, 3 = noise.
  auto rx = std::mt19937_64(gk::mix_seed(seed, 1));
  auto rp = std::mt19937_64(gk::mix_seed(seed, 2));
  auto rn = std::mt19937_64(gk::mix_seed(seed, 3));
  std::uniform_real_distribution<double> U01(0.0, 1.0);
  std::normal_distribution<double> N01(0.0, 1.0);
  i64 n = 0;
  int d = 0;
  switch (config) {
    case 1: n = 2000; d = 2; break;
    case 2: n = 10000; d = 2; break;
    case 3: n = 25001; d = 3; break;
    case 4: n = 150000; d = 2; break;
    case 5: n = 10000; d = 6; break;
    default: return GK_ERR_ARG;
  }
  if (n_out) *n_out = n;
  if (d_out) *d_out = d;
  if (!X) return GK_OK;
  auto Xa = [&](i64 i, int j) -> double& { return X[j * n + i]; };
  auto G = [&](i64 i, int j) -> double& { return dY[j * n + i]; };
  if (config == 1) {  // sin(6x1)cos(4x2) + 0.5 x1 x2 on U[0,1]^2
    for (i64 i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) Xa(i, j) = U01(rx);
    for (i64 i = 0; i < n; ++i) {
      const double a = Xa(i, 0), b = Xa(i, 1);
      y[i] = std::sin(6 * a) * std::cos(4 * b) + 0.5 * a * b;
      G(i, 0) = 6 * std::cos(6 * a) * std::cos(4 * b) + 0.5 * b;
      G(i, 1) = -4 * std::sin(6 * a) * std::sin(4 * b) + 0.5 * a;
    }
  } else if (config == 2) {  // 20 random sinusoids on U[-1,1]^2, + N(0,1e-4)
    for (i64 i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) Xa(i, j) = -1.0 + 2.0 * U01(rx);
    double w[20][2], amp[20], ph[20];
    for (int k = 0; k < 20; ++k) {
      w[k][0] = 3.0 * N01(rp);
      w[k][1] = 3.0 * N01(rp);
      amp[k] = N01(rp);
      ph[k] = 2.0 * M_PI * U01(rp);
    }
    for (i64 i = 0; i < n; ++i) {
      double v = 0, g0 = 0, g1 = 0;
      for (int k = 0; k < 20; ++k) {
        const double arg = w[k][0] * Xa(i, 0) + w[k][1] * Xa(i, 1) + ph[k];
        v += amp[k] * std::sin(arg);
        g0 += amp[k] * w[k][0] * std::cos(arg);
        g1 += amp[k] * w[k][1] * std::cos(arg);
      }
      y[i] = v + 1e-2 * N01(rn);
      G(i, 0) = g0 + 1e-2 * N01(rn);
      G(i, 1) = g1 + 1e-2 * N01(rn);
    }
  } else if (config == 3) {  // star-shaped surface, unit normals; one interior point
    double c[25];
    for (int k = 0; k < 25; ++k) c[k] = 0.05 * N01(rp);
    const i64 ns = n - 1;
    for (i64 i = 0; i < ns; ++i) {
      const double zc = -1.0 + 2.0 * U01(rx);
      const double ph = 2.0 * M_PI * U01(rx);
      const double rho = std::sqrt(std::max(0.0, 1.0 - zc * zc));
      const double u[3] = {rho * std::cos(ph), rho * std::sin(ph), zc};
      // r(u/|u|) with gradient w.r.t. u (at |u| = 1 the chain rule through
      // the normalisation is carried by the duals)
      D3 U[3];
      for (int a = 0; a < 3; ++a) {
        U[a] = mk(u[a]);
        U[a].g[a] = 1.0;
      }
      const D3 r2 = U[0] * U[0] + U[1] * U[1] + U[2] * U[2];
      const double inv = 1.0 / std::sqrt(r2.v);
      D3 nrm[3];
      for (int a = 0; a < 3; ++a) {
        // d(u_a/|u|)/du_b = (delta_ab - u_a u_b/|u|^2)/|u|
        nrm[a] = mk(u[a] * inv);
        for (int b = 0; b < 3; ++b) nrm[a].g[b] = ((a == b ? 1.0 : 0.0) - u[a] * u[b] * inv * inv) * inv;
      }
      D3 Y[25];
      real_sh(nrm[0], nrm[1], nrm[2], Y);
      D3 r = mk(1.0);
      for (int k = 0; k < 25; ++k) r = r + c[k] * Y[k];
      // surface point x = r(u) u; F(x) = |x| - r(x/|x|); grad F = u - grad_u r / r
      double gF[3], len = 0.0;
      for (int a = 0; a < 3; ++a) {
        Xa(i, a) = r.v * u[a];
        gF[a] = u[a] - r.g[a] / r.v;
        len += gF[a] * gF[a];
      }
      len = std::sqrt(len);
      y[i] = 0.0;
      for (int a = 0; a < 3; ++a) G(i, a) = gF[a] / len;
    }
    for (int a = 0; a < 3; ++a) {  // interior point: value -1, gradient pinned to 0
      Xa(ns, a) = 0.0;
      G(ns, a) = 0.0;
    }
    y[ns] = -1.0;
  } else if (config == 4) {  // rough terrain: 500 Gaussian bumps, + N(0,1e-4)
    for (i64 i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) Xa(i, j) = U01(rx);
    const int J = 500;
    std::vector<double> a(J), cx(J), cy(J), s2(J);
    const double lo = std::log(0.005), hi = std::log(0.1);
    for (int k = 0; k < J; ++k) {
      a[static_cast<size_t>(k)] = N01(rp);
      cx[static_cast<size_t>(k)] = U01(rp);
      cy[static_cast<size_t>(k)] = U01(rp);
      const double s = std::exp(lo + (hi - lo) * U01(rp));
      s2[static_cast<size_t>(k)] = s * s;
    }
    for (i64 i = 0; i < n; ++i) {
      double v = 0, g0 = 0, g1 = 0;
      for (int k = 0; k < J; ++k) {
        const double dx = Xa(i, 0) - cx[static_cast<size_t>(k)], dy = Xa(i, 1) - cy[static_cast<size_t>(k)];
        const double e = a[static_cast<size_t>(k)] * std::exp(-(dx * dx + dy * dy) / (2.0 * s2[static_cast<size_t>(k)]));
        v += e;
        g0 -= e * dx / s2[static_cast<size_t>(k)];
        g1 -= e * dy / s2[static_cast<size_t>(k)];
      }
      y[i] = v + 1e-2 * N01(rn);
      G(i, 0) = g0 + 1e-2 * N01(rn);
      G(i, 1) = g1 + 1e-2 * N01(rn);
    }
  } else {  // config 5: 6-D Hartmann form with seeded constants
    for (i64 i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) Xa(i, j) = U01(rx);
    double al[4], A[4][6], P[4][6];
    for (int k = 0; k < 4; ++k) al[k] = 1.0 + 3.0 * U01(rp);
    for (int k = 0; k < 4; ++k)
      for (int j = 0; j < 6; ++j) A[k][j] = 0.1 + 19.9 * U01(rp);
    for (int k = 0; k < 4; ++k)
      for (int j = 0; j < 6; ++j) P[k][j] = U01(rp);
    for (i64 i = 0; i < n; ++i) {
      double v = 0, g[6] = {0};
      for (int k = 0; k < 4; ++k) {
        double q = 0;
        for (int j = 0; j < 6; ++j) q += A[k][j] * (Xa(i, j) - P[k][j]) * (Xa(i, j) - P[k][j]);
        const double e = al[k] * std::exp(-q);
        v += e;
        for (int j = 0; j < 6; ++j) g[j] += -2.0 * A[k][j] * (Xa(i, j) - P[k][j]) * e;
      }
      y[i] = v;
      for (int j = 0; j < 6; ++j) G(i, j) = g[j];
    }
  }
  return GK_OK;
}
