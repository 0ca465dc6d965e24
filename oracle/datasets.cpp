// datasets.cpp — TEST INFRASTRUCTURE ONLY. The seeded synthetic workloads
// C1..C5 of BASELINE.json (configs[0..4]) generated on the oracle side, so
// bench.py's reference arm and the oracle-side fixtures never load the
// product library. Streams follow SURVEY §8(d): seeded_rng(seed, 1) = inputs,
// 2 = target parameters, 3 = observation noise (reference rng.hpp:19-21,
// libstdc++ uniform_real_distribution / normal_distribution as in
// testfns.cpp:355-402). tests/test_capi_host.py checks that these arrays are
// bit-identical to the product's gk_make_dataset.
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>
#include <algorithm>

#include "gk_oracle.hpp"

// ==================================================================== datasets
namespace {

using i64 = long long;

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

extern "C" int orc_make_dataset(int config, unsigned long long seed, long long* n_out, int* d_out, double* X,
                                double* y, double* dY) {
  // Streams: 1 = inputs, 2 = target parameters, 3 = noise.
  auto rx = std::mt19937_64(gko::mix_seed(seed, 1));
  auto rp = std::mt19937_64(gko::mix_seed(seed, 2));
  auto rn = std::mt19937_64(gko::mix_seed(seed, 3));
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
    default: return 1;
  }
  if (n_out) *n_out = n;
  if (d_out) *d_out = d;
  if (!X) return 0;
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
  return 0;
}

// sample_dataset (testfns.cpp:355-402) for the precond-study functions:
// Franke (testfns.cpp:67-92, d = 2) and Friedman #1 (:290-310, d = 5), uniform
// sampling on [0, 1]^d. Returns 1 for an unknown name.
extern "C" int orc_sample_test_function(const char* name, long long n, unsigned long long seed, double nv,
                                        double ng, int with_gradients, int* d_out, double* X, double* y,
                                        double* dY) {
  const std::string fn(name ? name : "");
  const int d = fn == "franke" ? 2 : fn == "friedman" ? 5 : 0;
  if (d == 0) return 1;
  *d_out = d;
  if (!X) return 0;
  auto rng = std::mt19937_64(gko::mix_seed(seed, 0));
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  for (i64 i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) X[j * n + i] = 0.0 + 1.0 * unif(rng);
  std::normal_distribution<double> gauss(0.0, 1.0);
  const double pi = 3.14159265358979323846;
  std::vector<double> g(static_cast<size_t>(d));
  for (i64 i = 0; i < n; ++i) {
    double v;
    if (d == 2) {
      const double a = X[i], b = X[n + i];
      const double e1 = 0.75 * std::exp(-(std::pow(9 * a - 2, 2) + std::pow(9 * b - 2, 2)) / 4.0);
      const double e2 = 0.75 * std::exp(-std::pow(9 * a + 1, 2) / 49.0 - (9 * b + 1) / 10.0);
      const double e3 = 0.5 * std::exp(-(std::pow(9 * a - 7, 2) + std::pow(9 * b - 3, 2)) / 4.0);
      const double e4 = -0.2 * std::exp(-std::pow(9 * a - 4, 2) - std::pow(9 * b - 7, 2));
      v = e1 + e2 + e3 + e4;
      g[0] = e1 * (-9.0 * (9 * a - 2) / 2.0) + e2 * (-18.0 * (9 * a + 1) / 49.0) + e3 * (-9.0 * (9 * a - 7) / 2.0) +
             e4 * (-18.0 * (9 * a - 4));
      g[1] = e1 * (-9.0 * (9 * b - 2) / 2.0) + e2 * (-9.0 / 10.0) + e3 * (-9.0 * (9 * b - 3) / 2.0) +
             e4 * (-18.0 * (9 * b - 7));
    } else {
      const double x0 = X[i], x1 = X[n + i], x2 = X[2 * n + i], x3 = X[3 * n + i], x4 = X[4 * n + i];
      v = 10.0 * std::sin(pi * x0 * x1) + 20.0 * std::pow(x2 - 0.5, 2) + 10.0 * x3 + 5.0 * x4;
      const double c = 10.0 * pi * std::cos(pi * x0 * x1);
      g[0] = c * x1;
      g[1] = c * x0;
      g[2] = 40.0 * (x2 - 0.5);
      g[3] = 10.0;
      g[4] = 5.0;
    }
    y[i] = v + nv * gauss(rng);
    if (with_gradients)
      for (int j = 0; j < d; ++j) dY[j * n + i] = g[j] + ng * gauss(rng);
  }
  return 0;
}
