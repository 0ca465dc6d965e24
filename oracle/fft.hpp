// fft.hpp — TEST INFRASTRUCTURE ONLY (oracle). Mixed-radix complex FFT
// standing in for FFTW's r2c/c2r (reference dski.cpp:119-122,157,162).
// Any exact DFT gives the same circulant-embedding product up to roundoff;
// this one is a recursive decimation-in-time Cooley–Tukey over the prime
// factors of the length with directly evaluated twiddles.
#pragma once

#include <cstdint>
#include <vector>

namespace gko {

class Fft {
 public:
  explicit Fft(int n);
  int size() const { return n_; }
  // In-place transform of split re/im arrays of length n with element
  // stride `stride`. Forward uses exp(-2πi jk/n); inverse is unnormalised.
  void run(double* re, double* im, std::int64_t stride, bool inverse, double* work) const;
  int work_size() const { return 4 * n_; }

 private:
  int n_;
  std::vector<int> factors_;
  std::vector<double> cosv_, sinv_;  // cos/sin(2π j / n)
  void rec(const double* ire, const double* iim, std::int64_t istride, double* ore, double* oim,
           int n, int level, bool inverse, double* tmp) const;
};

}  // namespace gko
