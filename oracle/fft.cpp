// fft.cpp — TEST INFRASTRUCTURE ONLY (oracle). See fft.hpp.
#include "fft.hpp"

#include <cmath>
#include <stdexcept>

namespace gko {

Fft::Fft(int n) : n_(n) {
  if (n < 1) throw std::invalid_argument("fft length must be positive");
  int m = n;
  for (int p : {4, 2, 3, 5}) {
    while (m % p == 0) {
      factors_.push_back(p);
      m /= p;
    }
  }
  for (int p = 7; m > 1; p += 2) {
    while (m % p == 0) {
      factors_.push_back(p);
      m /= p;
    }
  }
  cosv_.resize(n);
  sinv_.resize(n);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int j = 0; j < n; ++j) {
    const long double a = two_pi * (long double)j / (long double)n;
    cosv_[j] = (double)cosl(a);
    sinv_[j] = (double)sinl(a);
  }
}

// out[k] = sum_j in[j * istride] * w^(jk), w = exp(∓2πi/n), computed by
// splitting j = q + p*j' over the radix p of this level.
void Fft::rec(const double* ire, const double* iim, std::int64_t istride, double* ore, double* oim,
              int n, int level, bool inverse, double* tmp) const {
  if (n == 1) {
    ore[0] = ire[0];
    oim[0] = iim[0];
    return;
  }
  const int p = factors_[level];
  const int m = n / p;
  for (int q = 0; q < p; ++q)
    rec(ire + q * istride, iim + q * istride, istride * p, ore + q * m, oim + q * m, m, level + 1,
        inverse, tmp);
  const int tw_step = n_ / n;  // twiddle w_n^t = table[t * n_/n]
  const double sgn = inverse ? 1.0 : -1.0;
  double* xr = tmp;
  double* xi = tmp + p;
  for (int k = 0; k < m; ++k) {
    // twiddled inputs x_q = out[q*m + k] * w_n^{qk}
    for (int q = 0; q < p; ++q) {
      const double ar = ore[q * m + k], ai = oim[q * m + k];
      const long long t = (long long)q * k % n;
      const double c = cosv_[t * tw_step], s = sgn * sinv_[t * tw_step];
      xr[q] = ar * c - ai * s;
      xi[q] = ar * s + ai * c;
    }
    if (p == 2) {
      ore[k] = xr[0] + xr[1];
      oim[k] = xi[0] + xi[1];
      ore[k + m] = xr[0] - xr[1];
      oim[k + m] = xi[0] - xi[1];
      continue;
    }
    if (p == 4) {
      const double t0r = xr[0] + xr[2], t0i = xi[0] + xi[2];
      const double t1r = xr[0] - xr[2], t1i = xi[0] - xi[2];
      const double t2r = xr[1] + xr[3], t2i = xi[1] + xi[3];
      // (x1 - x3) * (∓i)
      const double dr = xr[1] - xr[3], di = xi[1] - xi[3];
      const double t3r = inverse ? -di : di, t3i = inverse ? dr : -dr;
      ore[k] = t0r + t2r;
      oim[k] = t0i + t2i;
      ore[k + m] = t1r + t3r;
      oim[k + m] = t1i + t3i;
      ore[k + 2 * m] = t0r - t2r;
      oim[k + 2 * m] = t0i - t2i;
      ore[k + 3 * m] = t1r - t3r;
      oim[k + 3 * m] = t1i - t3i;
      continue;
    }
    const int pstep = n_ / p;  // w_p^t = table[t * n_/p]
    for (int r = 0; r < p; ++r) {
      double sr = 0.0, si = 0.0;
      for (int q = 0; q < p; ++q) {
        const int t = (q * r) % p;
        const double c = cosv_[t * pstep], s = sgn * sinv_[t * pstep];
        sr += xr[q] * c - xi[q] * s;
        si += xr[q] * s + xi[q] * c;
      }
      ore[k + r * m] = sr;
      oim[k + r * m] = si;
    }
  }
}

void Fft::run(double* re, double* im, std::int64_t stride, bool inverse, double* work) const {
  double* ir = work;
  double* ii = work + n_;
  for (int j = 0; j < n_; ++j) {
    ir[j] = re[j * stride];
    ii[j] = im[j * stride];
  }
  double* orr = work + 2 * n_;
  double* oi = work + 3 * n_;
  std::vector<double> tmp(2 * 64 + 2 * (size_t)n_);
  rec(ir, ii, 1, orr, oi, n_, 0, inverse, tmp.data());
  for (int j = 0; j < n_; ++j) {
    re[j * stride] = orr[j];
    im[j * stride] = oi[j];
  }
}

}  // namespace gko
