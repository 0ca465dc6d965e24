// gk_oracle.cpp — TEST INFRASTRUCTURE ONLY. CPU restatement of the
// reference hot path (see gk_oracle.hpp). Citations are reference
// file:line under proj/core/src unless stated.
#include "gk_oracle.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <numeric>
#include <sstream>

#include "fft.hpp"

namespace gko {

// ============================================================== rng.hpp:12-38
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

Vec rademacher_vector(Index n, std::uint64_t seed, std::uint64_t stream) {
  auto rng = seeded_rng(seed, stream);
  Vec z(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) z[size_t(i)] = (rng() & 1ULL) ? 1.0 : -1.0;
  return z;
}

Vec gaussian_vector(Index n, std::uint64_t seed, std::uint64_t stream) {
  auto rng = seeded_rng(seed, stream);
  std::normal_distribution<double> dist(0.0, 1.0);
  Vec z(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) z[size_t(i)] = dist(rng);
  return z;
}

// ============================================================== kernels.cpp
namespace {
double sqnorm_diff(const double* x, const double* y, int d) {
  double r = 0.0;
  for (int j = 0; j < d; ++j) r += (x[j] - y[j]) * (x[j] - y[j]);
  return r;
}
}  // namespace

double k_eval(const KernelSpec& k, const double* x, const double* xp, int d) {  // :104-118
  const double s2 = k.s * k.s, ell = k.ell;
  const double r2 = sqnorm_diff(x, xp, d);
  if (k.family == SE) return s2 * std::exp(-0.5 * r2 / (ell * ell));
  const double rho = std::sqrt(r2) / ell;
  const double radial =
      k.spline_even ? (rho > 0 ? rho * rho * std::log(rho) : 0.0) : rho * rho * rho;
  return s2 * (radial + k.spline_a * rho * rho + k.spline_b);
}

void k_eval_grad(const KernelSpec& k, const double* x, const double* xp, int d, double* g) {
  const double s2 = k.s * k.s, ell = k.ell;
  double r2 = 0.0;
  for (int j = 0; j < d; ++j) r2 += (x[j] - xp[j]) * (x[j] - xp[j]);
  const double r = std::sqrt(r2);
  double c;
  if (k.family == SE) {  // kernels.cpp:128-130: grad_coeff(r^2) * u
    c = s2 * std::exp(-0.5 * (r * r) / (ell * ell)) / (ell * ell);
  } else if (r == 0.0) {
    c = 0.0;
  } else if (!k.spline_even) {
    c = -s2 * (3.0 * r / std::pow(ell, 3) + 2.0 * k.spline_a / (ell * ell));
  } else {
    c = -s2 * (2.0 * std::log(r / ell) + 1.0 + 2.0 * k.spline_a) / (ell * ell);
  }
  for (int j = 0; j < d; ++j) g[j] = c * (x[j] - xp[j]);
}

void k_eval_hess(const KernelSpec& k, const double* x, const double* xp, int d, double* H) {
  const double s2 = k.s * k.s, ell = k.ell, ell2 = ell * ell;
  double r2 = 0.0;
  for (int j = 0; j < d; ++j) r2 += (x[j] - xp[j]) * (x[j] - xp[j]);
  const double r = std::sqrt(r2);
  for (int p = 0; p < d; ++p)
    for (int q = 0; q < d; ++q) {
      const double up = x[p] - xp[p], uq = x[q] - xp[q];
      const double I = p == q ? 1.0 : 0.0;
      double h;
      if (k.family == SE) {  // :149-153
        const double kv = s2 * std::exp(-0.5 * (r * r) / ell2);
        h = (kv / (ell2 * ell2)) * (ell2 * I - up * uq);
      } else if (r == 0.0) {
        h = (-2.0 * k.spline_a * s2 / ell2) * I;
      } else if (!k.spline_even) {
        const double c1 = 3.0 * r / (ell2 * ell) + 2.0 * k.spline_a / ell2;
        h = -s2 * (c1 * I + (3.0 / (r * ell2 * ell)) * up * uq);
      } else {
        const double lr = std::log(r / ell);
        h = (-s2 / ell2) * ((2.0 * lr + 1.0 + 2.0 * k.spline_a) * I + (2.0 / (r * r)) * up * uq);
      }
      H[p * d + q] = h;
    }
}

double k_eval_dlogell(const KernelSpec& k, const double* x, const double* xp, int d) {  // :172-188
  const double s2 = k.s * k.s, ell = k.ell;
  const double r2 = sqnorm_diff(x, xp, d);
  const double rho2 = r2 / (ell * ell);
  if (k.family == SE) return s2 * std::exp(-0.5 * r2 / (ell * ell)) * rho2;
  if (r2 == 0.0) return 0.0;
  const double rho = std::sqrt(rho2);
  if (!k.spline_even) return s2 * (-3.0 * rho * rho2 - 2.0 * k.spline_a * rho2);
  return s2 * (-2.0 * rho2 * std::log(rho) - rho2 - 2.0 * k.spline_a * rho2);
}

Mat assemble_dense(const KernelSpec& k, const double* X, Index n, const double* Xp, Index np, int d,
                   bool with_derivatives, Index size_cap) {  // kernels.cpp:242-285
  const Index rows = with_derivatives ? n * (d + 1) : n;
  const Index cols = with_derivatives ? np * (d + 1) : np;
  if (rows * cols > size_cap)
    throw std::length_error("dense assembly of " + std::to_string(rows) + " x " +
                            std::to_string(cols) + " exceeds the configured size cap");
  Mat K(rows, cols);
#pragma omp parallel for schedule(static) if (n * np > 4096)
  for (Index i = 0; i < n; ++i) {
    double xi[16], xj[16], g[16], H[256];
    for (int c = 0; c < d; ++c) xi[c] = X[c * n + i];
    for (Index j = 0; j < np; ++j) {
      for (int c = 0; c < d; ++c) xj[c] = Xp[c * np + j];
      K(i, j) = k_eval(k, xi, xj, d);
      if (!with_derivatives) continue;
      k_eval_grad(k, xi, xj, d, g);
      k_eval_hess(k, xi, xj, d, H);
      for (int p = 0; p < d; ++p) {
        K(i, (p + 1) * np + j) = g[p];
        K((p + 1) * n + i, j) = -g[p];
        for (int q = 0; q < d; ++q) K((p + 1) * n + i, (q + 1) * np + j) = H[p * d + q];
      }
    }
  }
  return K;
}

// ============================================================== interpolation.cpp
namespace {
double quintic_piece(double s) {  // interpolation.cpp:15-23
  if (s < 1.0) return (((-25.0 * s + 63.0) * s - 35.0) * s * s * s - 15.0 * s * s + 12.0) / 12.0;
  if (s < 2.0) return (s - 2.0) * (s - 1.0) * ((25.0 * s - 114.0) * s * s + 153.0 * s - 48.0) / 24.0;
  if (s < 3.0) {
    const double t = s - 3.0;
    return -t * t * t * (s - 2.0) * (5.0 * s - 8.0) / 24.0;
  }
  return 0.0;
}
double quintic_piece_deriv(double s) {  // :27-34
  if (s < 1.0) return ((((-125.0 * s + 252.0) * s - 105.0) * s - 30.0) * s) / 12.0;
  if (s < 2.0) return ((((125.0 * s - 756.0) * s + 1635.0) * s - 1470.0) * s + 450.0) / 24.0;
  if (s < 3.0) return ((((-25.0 * s + 252.0) * s - 939.0) * s + 1530.0) * s - 918.0) / 24.0;
  return 0.0;
}
double quintic_kernel(double s) { return quintic_piece(std::abs(s)); }
double quintic_kernel_deriv(double s) { return s < 0.0 ? -quintic_piece_deriv(-s) : quintic_piece_deriv(s); }
double cubic_kernel(double s) {  // :42-47
  const double a = std::abs(s);
  if (a < 1.0) return ((1.5 * a - 2.5) * a) * a + 1.0;
  if (a < 2.0) return ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0;
  return 0.0;
}
double cubic_kernel_deriv(double s) {  // :48-57
  const double sg = s < 0.0 ? -1.0 : 1.0;
  const double a = std::abs(s);
  double v = 0.0;
  if (a < 1.0) v = (4.5 * a - 5.0) * a;
  else if (a < 2.0) v = (-1.5 * a + 5.0) * a - 4.0;
  return sg * v;
}

struct Axis1D {
  Index base = 0;
  double w[6] = {0}, dw[6] = {0};
  int count = 6;
};

Axis1D axis_stencil(const Grid& g, int axis, double x, int order, Index point) {  // :66-97
  const double h = g.spacing[axis];
  const double s = (x - g.origin[axis]) / h;
  const Index cell = static_cast<Index>(std::floor(s));
  const double t = s - static_cast<double>(cell);
  Axis1D out;
  double w[6], dw[6];
  if (order == 0) {
    quintic_weights(t, w, dw);
    out.count = 6;
    out.base = cell - 2;
  } else {
    cubic_weights(t, w, dw);
    out.count = 4;
    out.base = cell - 1;
  }
  for (int k = 0; k < out.count; ++k) {
    out.w[k] = w[k];
    out.dw[k] = dw[k] / h;
  }
  if (out.base < 0 || out.base + out.count > g.dims[axis]) {
    std::ostringstream msg;
    msg << "point " << point << " (coordinate " << x << " on axis " << axis
        << ") lies outside the interior of the grid";
    throw OutOfGridError(msg.str(), point);
  }
  return out;
}
}  // namespace

Index Grid::size() const {
  Index m = 1;
  for (int v : dims) m *= v;
  return m;
}

Grid grid_cover(const double* X, Index n, int d, double target, int margin, int max_nodes) {
  if (n == 0) throw std::invalid_argument("cannot build a grid over no points");
  if (!(target > 0.0)) throw std::invalid_argument("grid spacing must be positive");
  margin = std::max(margin, 3);
  Grid g;
  g.dims.resize(d);
  g.origin.resize(d);
  g.spacing.resize(d);
  for (int j = 0; j < d; ++j) {
    double lo = X[j * n], hi = X[j * n];
    for (Index i = 0; i < n; ++i) {
      lo = std::min(lo, X[j * n + i]);
      hi = std::max(hi, X[j * n + i]);
    }
    const double span = std::max(hi - lo, 1e-12);
    double h = target;
    int interior = static_cast<int>(std::ceil(span / h)) + 1;
    int m = interior + 2 * margin;
    if (m > max_nodes) {
      m = max_nodes;
      h = span / static_cast<double>(m - 1 - 2 * margin);
    }
    if (m < 6 + 2 * margin) m = 6 + 2 * margin;
    g.dims[j] = m;
    g.spacing[j] = h;
    g.origin[j] = lo - margin * h;
  }
  return g;
}

void quintic_weights(double t, double w[6], double dw[6]) {
  if (t < 0.0 || t >= 1.0) throw std::invalid_argument("fractional offset must lie in [0, 1)");
  for (int k = 0; k < 6; ++k) {
    const double arg = t - static_cast<double>(k - 2);
    w[k] = quintic_kernel(arg);
    dw[k] = quintic_kernel_deriv(arg);
  }
}

void cubic_weights(double t, double w[4], double dw[4]) {
  if (t < 0.0 || t >= 1.0) throw std::invalid_argument("fractional offset must lie in [0, 1)");
  for (int k = 0; k < 4; ++k) {
    const double arg = t - static_cast<double>(k - 1);
    w[k] = cubic_kernel(arg);
    dw[k] = cubic_kernel_deriv(arg);
  }
}

void Csr::mul(const double* x, double* y) const {
#pragma omp parallel for schedule(static) if (val.size() > 20000)
  for (Index i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (Index e = ptr[size_t(i)]; e < ptr[size_t(i + 1)]; ++e) acc += val[size_t(e)] * x[idx[size_t(e)]];
    y[i] = acc;
  }
}

void Csr::tmul_add(const double* x, double* y) const {
  for (Index i = 0; i < rows; ++i) {
    const double xi = x[i];
    for (Index e = ptr[size_t(i)]; e < ptr[size_t(i + 1)]; ++e) y[idx[size_t(e)]] += val[size_t(e)] * xi;
  }
}

SparseInterpolation build_interpolation(const Grid& g, const double* X, Index n, int order) {
  const int d = g.dim();
  const Index m = g.size();
  const int cnt = order == 0 ? 6 : 4;
  Index per_row = 1;
  for (int j = 0; j < d; ++j) per_row *= cnt;
  SparseInterpolation out;
  auto init = [&](Csr& A) {
    A.rows = n;
    A.cols = m;
    A.ptr.resize(static_cast<size_t>(n + 1));
    A.idx.resize(static_cast<size_t>(n * per_row));
    A.val.resize(static_cast<size_t>(n * per_row));
    for (Index i = 0; i <= n; ++i) A.ptr[size_t(i)] = i * per_row;
  };
  init(out.W);
  out.dW.resize(d);
  for (auto& A : out.dW) init(A);
  std::vector<Axis1D> axes(d);
  std::vector<int> id(d);
  for (Index i = 0; i < n; ++i) {
    for (int j = 0; j < d; ++j) axes[j] = axis_stencil(g, j, X[j * n + i], order, i);
    std::fill(id.begin(), id.end(), 0);
    for (Index c = 0; c < per_row; ++c) {
      Index flat = 0;
      double w = 1.0;
      for (int j = 0; j < d; ++j) {
        flat = flat * g.dims[j] + (axes[j].base + id[j]);
        w *= axes[j].w[id[j]];
      }
      const size_t e = static_cast<size_t>(i * per_row + c);
      out.W.idx[e] = flat;
      out.W.val[e] = w;
      for (int p = 0; p < d; ++p) {
        double dw = 1.0;
        for (int j = 0; j < d; ++j) dw *= (j == p) ? axes[j].dw[id[j]] : axes[j].w[id[j]];
        out.dW[p].idx[e] = flat;
        out.dW[p].val[e] = dw;
      }
      for (int j = d - 1; j >= 0; --j) {
        if (++id[j] < axes[j].count) break;
        id[j] = 0;
      }
    }
  }
  return out;
}

PointStencil point_stencil(const Grid& g, const double* x, int order) {  // :172-210
  const int d = g.dim();
  std::vector<Axis1D> axes(d);
  for (int j = 0; j < d; ++j) axes[j] = axis_stencil(g, j, x[j], order, 0);
  Index nnz = 1;
  for (auto& a : axes) nnz *= a.count;
  PointStencil st;
  st.indices.resize(static_cast<size_t>(nnz));
  st.value.resize(static_cast<size_t>(nnz));
  st.derivative = Mat(nnz, d);
  std::vector<int> id(d, 0);
  for (Index c = 0; c < nnz; ++c) {
    Index flat = 0;
    double w = 1.0;
    for (int j = 0; j < d; ++j) {
      flat = flat * g.dims[j] + (axes[j].base + id[j]);
      w *= axes[j].w[id[j]];
    }
    st.indices[size_t(c)] = flat;
    st.value[size_t(c)] = w;
    for (int p = 0; p < d; ++p) {
      double dw = 1.0;
      for (int j = 0; j < d; ++j) dw *= (j == p) ? axes[j].dw[id[j]] : axes[j].w[id[j]];
      st.derivative(c, p) = dw;
    }
    for (int j = d - 1; j >= 0; --j) {
      if (++id[j] < axes[j].count) break;
      id[j] = 0;
    }
  }
  return st;
}

// ============================================================== linear_operator.cpp
Mat LinearOperator::dense() const {  // linear_operator.cpp:15-27
  const Index n = size();
  Mat A(n, n);
  Vec e(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < n; ++j) {
    e[size_t(j)] = 1.0;
    mvm(e.data(), A.col(j));
    e[size_t(j)] = 0.0;
  }
  return A;
}

void DenseOperator::mvm(const double* x, double* y) const {
  const Index n = A_.rows;
  for (Index i = 0; i < n; ++i) y[i] = 0.0;
  for (Index j = 0; j < A_.cols; ++j) {
    const double xj = x[j];
    const double* c = A_.col(j);
    for (Index i = 0; i < n; ++i) y[i] += c[i] * xj;
  }
}
Vec DenseOperator::diagonal() const {
  Vec d(static_cast<size_t>(A_.rows));
  for (Index i = 0; i < A_.rows; ++i) d[size_t(i)] = A_(i, i);
  return d;
}
Vec DenseOperator::row(Index i) const {
  Vec r(static_cast<size_t>(A_.cols));
  for (Index j = 0; j < A_.cols; ++j) r[size_t(j)] = A_(i, j);
  return r;
}

// ============================================================== dski.cpp
Profile kernel_profile(const KernelSpec& k) {  // dski.cpp:30-34
  return [k](const double* off, int d) {
    double z[16] = {0};
    return k_eval(k, off, z, d);
  };
}
Profile kernel_dlogell_profile(const KernelSpec& k) {  // dski.cpp:36-40
  return [k](const double* off, int d) {
    double z[16] = {0};
    return k_eval_dlogell(k, off, z, d);
  };
}

GridKernelOperator::GridKernelOperator(Grid g, const Profile& profile) : grid_(std::move(g)) {
  const int d = grid_.dim();  // dski.cpp:80-133
  edims_.resize(d);
  embed_total_ = 1;
  for (int j = 0; j < d; ++j) {
    if (grid_.dims[j] < 2) throw std::invalid_argument("grid needs at least 2 nodes per dimension");
    edims_[j] = 2 * (grid_.dims[j] - 1);
    embed_total_ *= edims_[j];
  }
  for (int j = 0; j < d; ++j) plans_.emplace_back(std::make_unique<Fft>(edims_[j]));
  // slice at wrapped offsets (dski.cpp:100-114)
  Vec re(static_cast<size_t>(embed_total_)), im(static_cast<size_t>(embed_total_), 0.0);
  std::vector<Index> id(d, 0);
  double off[16];
  for (Index t = 0; t < embed_total_; ++t) {
    for (int j = 0; j < d; ++j) {
      const Index e = edims_[j];
      const Index w = id[j] <= e / 2 ? id[j] : id[j] - e;
      off[j] = static_cast<double>(w) * grid_.spacing[j];
    }
    re[size_t(t)] = profile(off, d);
    for (int j = d - 1; j >= 0; --j) {
      if (++id[j] < edims_[j]) break;
      id[j] = 0;
    }
  }
  fftn(re, im, false);
  spectrum_ = re;  // real part only (dski.cpp:128-132)
}
GridKernelOperator::~GridKernelOperator() = default;
GridKernelOperator::GridKernelOperator(GridKernelOperator&&) noexcept = default;

double GridKernelOperator::min_embedding_eigenvalue() const {
  return *std::min_element(spectrum_.begin(), spectrum_.end());
}

void GridKernelOperator::fftn(std::vector<double>& re, std::vector<double>& im, bool inverse) const {
  const int d = grid_.dim();
  Index inner = 1;
  for (int j = d - 1; j >= 0; --j) {
    const Index e = edims_[j];
    const Index outer = embed_total_ / (e * inner);
    std::vector<double> work(static_cast<size_t>(plans_[j]->work_size()));
    for (Index o = 0; o < outer; ++o)
      for (Index in = 0; in < inner; ++in) {
        const Index base = o * e * inner + in;
        plans_[j]->run(re.data() + base, im.data() + base, inner, inverse, work.data());
      }
    inner *= e;
  }
}

void GridKernelOperator::mvm(const double* v, double* out) const {  // dski.cpp:146-166
  const int d = grid_.dim();
  Vec re(static_cast<size_t>(embed_total_), 0.0), im(static_cast<size_t>(embed_total_), 0.0);
  const Index m = grid_.size();
  std::vector<Index> id(d, 0);
  std::vector<Index> corner(static_cast<size_t>(m));
  for (Index fm = 0; fm < m; ++fm) {  // for_each_corner (dski.cpp:62-77)
    Index fe = 0;
    for (int j = 0; j < d; ++j) fe = fe * edims_[j] + id[j];
    corner[size_t(fm)] = fe;
    for (int j = d - 1; j >= 0; --j) {
      if (++id[j] < grid_.dims[j]) break;
      id[j] = 0;
    }
  }
  for (Index fm = 0; fm < m; ++fm) re[size_t(corner[size_t(fm)])] = v[fm];
  fftn(re, im, false);
  for (Index t = 0; t < embed_total_; ++t) {
    re[size_t(t)] *= spectrum_[size_t(t)];
    im[size_t(t)] *= spectrum_[size_t(t)];
  }
  fftn(re, im, true);
  const double scale = 1.0 / static_cast<double>(embed_total_);
  for (Index fm = 0; fm < m; ++fm) out[fm] = re[size_t(corner[size_t(fm)])] * scale;
}

DskiOperator::DskiOperator(const KernelSpec& k, Grid g, const double* X, Index n, int d,
                           NoiseLevels noise, int order, bool with_gradients)
    : n_(n), d_(d), groups_(with_gradients ? d : 0), grid_(std::move(g)), kernel_(k), noise_(noise),
      interp_(build_interpolation(grid_, X, n, order)), kuu_(grid_, kernel_profile(k)) {
  const int count = order == 0 ? 6 : 4;  // dski.cpp:186-203
  const int width = 2 * count - 1;
  table_dims_.assign(d_, width);
  Index total = 1;
  for (int j = 0; j < d_; ++j) total *= width;
  table_.resize(static_cast<size_t>(total));
  std::vector<int> id(d_, 0);
  double off[16];
  auto profile = kernel_profile(kernel_);
  for (Index t = 0; t < total; ++t) {
    for (int j = 0; j < d_; ++j) off[j] = static_cast<double>(id[j] - (count - 1)) * grid_.spacing[j];
    table_[size_t(t)] = profile(off, d_);
    for (int j = d_ - 1; j >= 0; --j) {
      if (++id[j] < width) break;
      id[j] = 0;
    }
  }
}

Vec DskiOperator::noise_diagonal() const {  // dski.cpp:206-211
  Vec nd(static_cast<size_t>(size()));
  for (Index i = 0; i < size(); ++i)
    nd[size_t(i)] = i < n_ ? noise_.value * noise_.value : noise_.gradient * noise_.gradient;
  return nd;
}

Vec DskiOperator::stacked_transpose_apply(const double* v) const {  // dski.cpp:213-219
  Vec u(static_cast<size_t>(grid_.size()), 0.0);
  interp_.W.tmul_add(v, u.data());
  for (int j = 0; j < groups_; ++j) {
    Vec t(static_cast<size_t>(grid_.size()), 0.0);
    interp_.dW[j].tmul_add(v + n_ * (j + 1), t.data());
    for (size_t a = 0; a < u.size(); ++a) u[a] += t[a];
  }
  return u;
}

Vec DskiOperator::stacked_apply(const double* u) const {  // dski.cpp:221-226
  Vec out(static_cast<size_t>(size()));
  interp_.W.mul(u, out.data());
  for (int j = 0; j < groups_; ++j) interp_.dW[j].mul(u, out.data() + n_ * (j + 1));
  return out;
}

void DskiOperator::mvm(const double* v, double* out) const {  // dski.cpp:228-238
  Vec u = stacked_transpose_apply(v);
  Vec w(static_cast<size_t>(grid_.size()));
  kuu_.mvm(u.data(), w.data());
  Vec o = stacked_apply(w.data());
  const double nv = noise_.value * noise_.value, ng = noise_.gradient * noise_.gradient;
  for (Index i = 0; i < n_; ++i) out[i] = o[size_t(i)] + nv * v[i];
  for (Index i = n_; i < size(); ++i) out[i] = o[size_t(i)] + ng * v[i];
}

Vec DskiOperator::diagonal() const {  // dski.cpp:240-290
  Vec diag(static_cast<size_t>(size()));
  const int count = table_dims_[0] / 2 + 1;
  const Index per_row = interp_.W.ptr[1] - interp_.W.ptr[0];
#pragma omp parallel for schedule(static)
  for (Index i = 0; i < n_; ++i) {
    std::vector<std::array<int, 16>> coords(static_cast<size_t>(per_row));
    Mat wm(per_row, groups_ + 1);
    const Index e0 = interp_.W.ptr[size_t(i)];
    for (Index a = 0; a < per_row; ++a) {
      Index rem = interp_.W.idx[size_t(e0 + a)];
      for (int j = d_ - 1; j >= 0; --j) {
        coords[size_t(a)][j] = static_cast<int>(rem % grid_.dims[j]);
        rem /= grid_.dims[j];
      }
      wm(a, 0) = interp_.W.val[size_t(e0 + a)];
      for (int j = 0; j < groups_; ++j) wm(a, j + 1) = interp_.dW[j].val[size_t(e0 + a)];
    }
    double acc[17] = {0};
    for (Index a = 0; a < per_row; ++a)
      for (Index b = 0; b < per_row; ++b) {
        Index t = 0;
        for (int j = 0; j < d_; ++j)
          t = t * table_dims_[j] + (coords[size_t(a)][j] - coords[size_t(b)][j] + count - 1);
        const double kab = table_[size_t(t)];
        for (int g = 0; g <= groups_; ++g) acc[g] += wm(a, g) * wm(b, g) * kab;
      }
    for (int g = 0; g <= groups_; ++g) diag[size_t(g * n_ + i)] = acc[g];
  }
  const double nv = noise_.value * noise_.value, ng = noise_.gradient * noise_.gradient;
  for (Index i = 0; i < size(); ++i) diag[size_t(i)] += i < n_ ? nv : ng;
  return diag;
}

Vec DskiOperator::row(Index r) const {  // dski.cpp:292-304
  if (r < 0 || r >= size()) throw std::out_of_range("D-SKI row index out of range");
  const Index i = r % n_;
  const int g = static_cast<int>(r / n_);
  Vec b(static_cast<size_t>(grid_.size()), 0.0);
  const Csr& mat = g == 0 ? interp_.W : interp_.dW[g - 1];
  for (Index e = mat.ptr[size_t(i)]; e < mat.ptr[size_t(i + 1)]; ++e) b[size_t(mat.idx[size_t(e)])] = mat.val[size_t(e)];
  Vec w(static_cast<size_t>(grid_.size()));
  kuu_.mvm(b.data(), w.data());
  Vec out = stacked_apply(w.data());
  out[size_t(r)] += g == 0 ? noise_.value * noise_.value : noise_.gradient * noise_.gradient;
  return out;
}

// ============================================================== linalg.cpp
namespace {
double dot(const double* a, const double* b, Index n) {
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double norm(const double* a, Index n) { return std::sqrt(dot(a, a, n)); }

// w -= Q[:, :k] (Q[:, :k]^T w)
void reorth(const Mat& Q, Index k, double* w) {
  const Index n = Q.rows;
  Vec c(static_cast<size_t>(k));
  for (Index j = 0; j < k; ++j) c[size_t(j)] = dot(Q.col(j), w, n);
  for (Index j = 0; j < k; ++j) {
    const double* q = Q.col(j);
    for (Index i = 0; i < n; ++i) w[i] -= q[i] * c[size_t(j)];
  }
}
}  // namespace

LanczosFactor lanczos_from_start(const LinearOperator& op, const Vec& start, Index steps,
                                 std::uint64_t restart_seed) {  // linalg.cpp:17-81
  const Index n = op.size();
  steps = std::min(steps, n);
  LanczosFactor fac;
  fac.Q = Mat(n, steps);
  fac.alpha.assign(static_cast<size_t>(steps), 0.0);
  fac.beta.assign(static_cast<size_t>(steps > 0 ? steps - 1 : 0), 0.0);
  Vec q = start, prev(static_cast<size_t>(n), 0.0), w(static_cast<size_t>(n));
  double beta_prev = 0.0, scale = 0.0;
  std::uint64_t restart_count = 0;
  Index k = 0;
  for (; k < steps; ++k) {
    std::copy(q.begin(), q.end(), fac.Q.col(k));
    op.mvm(q.data(), w.data());
    for (Index i = 0; i < n; ++i) w[size_t(i)] -= beta_prev * prev[size_t(i)];
    const double a = dot(q.data(), w.data(), n);
    fac.alpha[size_t(k)] = a;
    for (Index i = 0; i < n; ++i) w[size_t(i)] -= a * q[size_t(i)];
    for (int pass = 0; pass < 2; ++pass) reorth(fac.Q, k + 1, w.data());
    const double beta = norm(w.data(), n);
    scale = std::max({scale, std::abs(a), beta});
    if (k + 1 >= steps) continue;
    if (beta <= 1e-12 * std::max(scale, 1e-300)) {
      fac.breakdown = true;
      bool found = false;
      for (int attempt = 0; attempt < 8 && !found; ++attempt) {
        Vec r = gaussian_vector(n, mix_seed(restart_seed, 7777 + restart_count++), attempt);
        for (int pass = 0; pass < 2; ++pass) reorth(fac.Q, k + 1, r.data());
        const double rn = norm(r.data(), n);
        if (rn > 1e-8 * std::sqrt(double(n))) {
          for (Index i = 0; i < n; ++i) q[size_t(i)] = r[size_t(i)] / rn;
          found = true;
        }
      }
      if (!found) {
        ++k;
        break;
      }
      fac.beta[size_t(k)] = 0.0;
      std::fill(prev.begin(), prev.end(), 0.0);
      beta_prev = 0.0;
      continue;
    }
    fac.beta[size_t(k)] = beta;
    prev = q;
    for (Index i = 0; i < n; ++i) q[size_t(i)] = w[size_t(i)] / beta;
    beta_prev = beta;
  }
  if (k < steps) {
    Mat Q2(n, k);
    std::copy(fac.Q.a.begin(), fac.Q.a.begin() + n * k, Q2.a.begin());
    fac.Q = std::move(Q2);
    fac.alpha.resize(static_cast<size_t>(k));
    fac.beta.resize(static_cast<size_t>(k > 0 ? k - 1 : 0));
  }
  return fac;
}

CgResult cg(const LinearOperator& A, const double* b, const CgOptions& o, const PrecondApply& M) {
  const Index n = A.size();  // linalg.cpp:85-131
  CgResult res;
  res.x.assign(static_cast<size_t>(n), 0.0);
  const double bnorm = norm(b, n);
  if (bnorm == 0.0) {
    res.converged = true;
    return res;
  }
  Vec r(b, b + n);
  Vec z = M ? M(r) : r;
  Vec p = z;
  double rz = dot(r.data(), z.data(), n);
  Vec Ap(static_cast<size_t>(n));
  double relres = norm(r.data(), n) / bnorm;
  res.residual_history.push_back(relres);
  if (relres <= o.tol) {
    res.converged = true;
    return res;
  }
  for (int it = 0; it < o.max_iterations; ++it) {
    A.mvm(p.data(), Ap.data());
    const double pAp = dot(p.data(), Ap.data(), n);
    if (pAp <= 0.0) break;
    const double alpha = rz / pAp;
    for (Index i = 0; i < n; ++i) res.x[size_t(i)] += alpha * p[size_t(i)];
    for (Index i = 0; i < n; ++i) r[size_t(i)] -= alpha * Ap[size_t(i)];
    res.iterations = it + 1;
    relres = norm(r.data(), n) / bnorm;
    res.residual_history.push_back(relres);
    if (relres <= o.tol) {
      res.converged = true;
      return res;
    }
    z = M ? M(r) : r;
    const double rz_next = dot(r.data(), z.data(), n);
    const double beta = rz_next / rz;
    for (Index i = 0; i < n; ++i) p[size_t(i)] = z[size_t(i)] + beta * p[size_t(i)];
    rz = rz_next;
  }
  return res;
}

PivotedCholeskyFactor pivoted_cholesky(const Vec& diag, const std::function<Vec(Index)>& row_fn,
                                       Index max_rank, double trace_tol) {  // linalg.cpp:133-174
  const Index n = Index(diag.size());
  PivotedCholeskyFactor out;
  if (*std::min_element(diag.begin(), diag.end()) < 0.0)
    throw std::runtime_error("pivoted Cholesky requires a nonnegative diagonal");
  Vec d = diag;
  out.initial_trace = std::accumulate(d.begin(), d.end(), 0.0);
  out.residual_trace = out.initial_trace;
  const double scale = std::max(*std::max_element(diag.begin(), diag.end()), 1e-300);
  max_rank = std::min(max_rank, n);
  out.L = Mat(n, max_rank);
  Index k = 0;
  for (; k < max_rank; ++k) {
    // Eigen maxCoeff(&idx): first index of the maximum
    Index piv = 0;
    double dmax = d[0];
    for (Index i = 1; i < n; ++i)
      if (d[size_t(i)] > dmax) {
        dmax = d[size_t(i)];
        piv = i;
      }
    if (dmax <= 0.0 || out.residual_trace <= trace_tol * out.initial_trace) break;
    Vec col = row_fn(piv);
    if (Index(col.size()) != n) throw std::invalid_argument("pivoted Cholesky row size mismatch");
    if (k > 0) {
      for (Index j = 0; j < k; ++j) {
        const double lp = out.L(piv, j);
        const double* Lj = out.L.col(j);
        for (Index i = 0; i < n; ++i) col[size_t(i)] -= Lj[i] * lp;
      }
    }
    const double sq = std::sqrt(dmax);
    for (Index i = 0; i < n; ++i) col[size_t(i)] /= sq;
    std::copy(col.begin(), col.end(), out.L.col(k));
    out.pivots.push_back(piv);
    double dmin = std::numeric_limits<double>::infinity();
    for (Index i = 0; i < n; ++i) {
      d[size_t(i)] -= col[size_t(i)] * col[size_t(i)];
      dmin = std::min(dmin, d[size_t(i)]);
    }
    if (dmin < -1e-10 * scale)
      throw std::runtime_error("pivoted Cholesky: operator is not positive semidefinite "
                               "(residual diagonal " + std::to_string(dmin) + ")");
    for (auto& v : d) v = std::max(v, 0.0);
    d[size_t(piv)] = 0.0;
    out.residual_trace = std::accumulate(d.begin(), d.end(), 0.0);
  }
  Mat L2(n, k);
  std::copy(out.L.a.begin(), out.L.a.begin() + n * k, L2.a.begin());
  out.L = std::move(L2);
  return out;
}

Preconditioner::Preconditioner(const Mat& F, const Vec& nd) {  // linalg.cpp:176-194
  if (F.rows != Index(nd.size())) throw std::invalid_argument("preconditioner factor and noise sizes differ");
  if (nd.empty() || *std::min_element(nd.begin(), nd.end()) <= 0.0)
    throw std::invalid_argument("preconditioner needs strictly positive noise");
  inv_sqrt_noise_.resize(nd.size());
  for (size_t i = 0; i < nd.size(); ++i) inv_sqrt_noise_[i] = 1.0 / std::sqrt(nd[i]);
  const Index n = F.rows, k = F.cols;
  if (k == 0) throw std::invalid_argument("preconditioner needs a factor of rank at least 1");
  // Householder QR of the stacked (n+k)×k matrix [D^-1/2 F; I]
  const Index R = n + k;
  Mat A(R, k);
  for (Index j = 0; j < k; ++j) {
    for (Index i = 0; i < n; ++i) A(i, j) = inv_sqrt_noise_[size_t(i)] * F(i, j);
    A(n + j, j) = 1.0;
  }
  Vec tau(static_cast<size_t>(k));
  for (Index j = 0; j < k; ++j) {
    // reflector for A(j:, j) (LAPACK/Eigen convention: beta = -sign(a0)*norm)
    double* c = A.col(j);
    double sig = 0.0;
    for (Index i = j + 1; i < R; ++i) sig += c[i] * c[i];
    const double a0 = c[j];
    if (sig == 0.0) {
      tau[size_t(j)] = 0.0;
      continue;
    }
    const double nrm = std::sqrt(a0 * a0 + sig);
    const double beta = a0 <= 0.0 ? nrm : -nrm;
    for (Index i = j + 1; i < R; ++i) c[i] /= (a0 - beta);
    tau[size_t(j)] = (beta - a0) / beta;
    c[j] = beta;
    for (Index jj = j + 1; jj < k; ++jj) {
      double* cc = A.col(jj);
      double s = cc[j];
      for (Index i = j + 1; i < R; ++i) s += c[i] * cc[i];
      s *= tau[size_t(j)];
      cc[j] -= s;
      for (Index i = j + 1; i < R; ++i) cc[i] -= s * c[i];
    }
  }
  // thin Q = H_0 ... H_{k-1} [I_k; 0]
  Mat Q(R, k);
  for (Index j = 0; j < k; ++j) Q(j, j) = 1.0;
  for (Index j = k - 1; j >= 0; --j) {
    const double* v = A.col(j);
    const double t = tau[size_t(j)];
    if (t == 0.0) continue;
    for (Index c = 0; c < k; ++c) {
      double* q = Q.col(c);
      double s = q[j];
      for (Index i = j + 1; i < R; ++i) s += v[i] * q[i];
      s *= t;
      q[j] -= s;
      for (Index i = j + 1; i < R; ++i) q[i] -= s * v[i];
    }
  }
  Q1_ = Mat(n, k);
  for (Index c = 0; c < k; ++c) std::copy(Q.col(c), Q.col(c) + n, Q1_.col(c));
}

Preconditioner::Preconditioner(const Mat& F, double sigma, Index n)
    : Preconditioner(F, Vec(static_cast<size_t>(n), sigma * sigma)) {}

Vec Preconditioner::apply(const Vec& b) const {  // linalg.cpp:200-204
  const Index n = size(), k = rank();
  Vec c(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) c[size_t(i)] = inv_sqrt_noise_[size_t(i)] * b[size_t(i)];
  Vec t(static_cast<size_t>(k));
  for (Index j = 0; j < k; ++j) t[size_t(j)] = dot(Q1_.col(j), c.data(), n);
  Vec y(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < k; ++j) {
    const double* q = Q1_.col(j);
    for (Index i = 0; i < n; ++i) y[size_t(i)] += q[i] * t[size_t(j)];
  }
  for (Index i = 0; i < n; ++i) c[size_t(i)] = inv_sqrt_noise_[size_t(i)] * (c[size_t(i)] - y[size_t(i)]);
  return c;
}

double Preconditioner::quadratic(const Vec& b) const {  // linalg.cpp:210-213
  const Index n = size(), k = rank();
  Vec c(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) c[size_t(i)] = inv_sqrt_noise_[size_t(i)] * b[size_t(i)];
  double t2 = 0.0;
  for (Index j = 0; j < k; ++j) {
    const double t = dot(Q1_.col(j), c.data(), n);
    t2 += t * t;
  }
  return dot(c.data(), c.data(), n) - t2;
}

// Implicit symmetric QL with Wilkinson-type shifts (tql2), eigenvalues
// ascending; eigenvectors accumulated (all rows when evecs != null, else
// the first row only, which is what SLQ's quadrature weights need).
void tridiag_eig(const Vec& alpha, const Vec& beta, Vec& evals, Mat* evecs) {
  // tql2-style implicit QL; replaces Eigen's computeFromTridiagonal
  // (linalg.cpp:231-232,294). Same spectrum/eigenvectors up to roundoff.
  const int n = int(alpha.size());
  Vec dd = alpha;
  Vec e(static_cast<size_t>(n), 0.0);
  for (int i = 0; i + 1 < n; ++i) e[size_t(i)] = beta[size_t(i)];
  Mat Z(n, n);
  for (int i = 0; i < n; ++i) Z(i, i) = 1.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double s = std::abs(dd[size_t(m)]) + std::abs(dd[size_t(m + 1)]);
        if (std::abs(e[size_t(m)]) <= std::numeric_limits<double>::epsilon() * s) break;
      }
      if (m != l) {
        if (++iter > 300) throw std::runtime_error("tridiagonal eigensolver did not converge");
        double g = (dd[size_t(l + 1)] - dd[size_t(l)]) / (2.0 * e[size_t(l)]);
        double r = std::hypot(g, 1.0);
        g = dd[size_t(m)] - dd[size_t(l)] + e[size_t(l)] / (g + (g >= 0 ? r : -r));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[size_t(i)];
          const double b = c * e[size_t(i)];
          r = std::hypot(f, g);
          e[size_t(i + 1)] = r;
          if (r == 0.0) {
            dd[size_t(i + 1)] -= p;
            e[size_t(m)] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = dd[size_t(i + 1)] - p;
          r = (dd[size_t(i)] - g) * s + 2.0 * c * b;
          p = s * r;
          dd[size_t(i + 1)] = g + p;
          g = c * r - b;
          for (int kr = 0; kr < n; ++kr) {
            f = Z(kr, i + 1);
            Z(kr, i + 1) = s * Z(kr, i) + c * f;
            Z(kr, i) = c * Z(kr, i) - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        dd[size_t(l)] -= p;
        e[size_t(l)] = g;
        e[size_t(m)] = 0.0;
      }
    } while (m != l);
  }
  std::vector<int> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return dd[size_t(a)] < dd[size_t(b)]; });
  evals.assign(static_cast<size_t>(n), 0.0);
  Mat sz(n, n);
  for (int j = 0; j < n; ++j) {
    evals[size_t(j)] = dd[size_t(ord[size_t(j)])];
    for (int r = 0; r < n; ++r) sz(r, j) = Z(r, ord[size_t(j)]);
  }
  if (evecs) *evecs = std::move(sz);
}

SlqResult slq_logdet(const LinearOperator& A, const SlqOptions& o) {  // linalg.cpp:215-253
  const Index n = A.size();
  SlqResult out;
  if (o.probes <= 0) return out;
  std::vector<double> est(static_cast<size_t>(o.probes), 0.0);
  std::vector<int> clamps(static_cast<size_t>(o.probes), 0);
#pragma omp parallel for schedule(dynamic)
  for (int p = 0; p < o.probes; ++p) {
    Vec z = rademacher_vector(n, o.seed, std::uint64_t(p));
    const double zn2 = dot(z.data(), z.data(), n);
    const double zn = std::sqrt(zn2);
    Vec start(z);
    for (auto& v : start) v /= zn;
    const Index steps = std::min<Index>(o.lanczos_steps, n);
    LanczosFactor f = lanczos_from_start(A, start, steps, mix_seed(o.seed, 50000 + std::uint64_t(p)));
    Vec ev;
    Mat Z;
    tridiag_eig(f.alpha, f.beta, ev, &Z);
    double e = 0.0;
    for (size_t i = 0; i < ev.size(); ++i) {
      double lambda = ev[i];
      if (lambda < o.eigen_floor) {
        lambda = o.eigen_floor;
        ++clamps[size_t(p)];
      }
      const double w0 = Z(0, Index(i));
      e += w0 * w0 * std::log(lambda);
    }
    est[size_t(p)] = zn2 * e;
  }
  double sum = 0.0;
  for (int p = 0; p < o.probes; ++p) {
    sum += est[size_t(p)];
    out.clamped += clamps[size_t(p)];
  }
  out.logdet = sum / o.probes;
  out.estimates = est;
  return out;
}

double trace_estimate(const LinearOperator& A, const LinearOperator& B, int probes,
                      std::uint64_t seed, const CgOptions& o, const PrecondApply& M) {
  if (A.size() != B.size()) throw std::invalid_argument("trace_estimate: size mismatch");
  const Index n = A.size();  // linalg.cpp:255-279
  if (probes <= 0) return 0.0;
  std::vector<double> est(static_cast<size_t>(probes), 0.0);
  bool failed = false;
#pragma omp parallel for schedule(dynamic)
  for (int p = 0; p < probes; ++p) {
    Vec z = rademacher_vector(n, seed, 1000 + std::uint64_t(p));
    Vec Bz(static_cast<size_t>(n));
    B.mvm(z.data(), Bz.data());
    CgResult s = cg(A, z.data(), o, M);
    if (!s.converged) {
#pragma omp atomic write
      failed = true;
    }
    est[size_t(p)] = dot(s.x.data(), Bz.data(), n);
  }
  if (failed)
    throw std::runtime_error("trace_estimate: CG did not converge within " +
                             std::to_string(o.max_iterations) + " iterations");
  double sum = 0.0;
  for (int p = 0; p < probes; ++p) sum += est[size_t(p)];
  return sum / probes;
}

Mat LanczosFactor::tridiagonal() const {
  const Index r = Index(alpha.size());
  Mat T(r, r);
  for (Index i = 0; i < r; ++i) T(i, i) = alpha[size_t(i)];
  for (Index i = 0; i + 1 < r; ++i) T(i, i + 1) = T(i + 1, i) = beta[size_t(i)];
  return T;
}
Vec LanczosFactor::ritz_values() const {
  Vec ev;
  Mat Z;
  tridiag_eig(alpha, beta, ev, &Z);
  std::reverse(ev.begin(), ev.end());
  return ev;
}
Vec LanczosFactor::apply(const double* v) const {  // linalg.cpp:298-302
  const Index n = Q.rows, r = Q.cols;
  Vec t(static_cast<size_t>(r));
  for (Index j = 0; j < r; ++j) t[size_t(j)] = dot(Q.col(j), v, n);
  Vec Tt(static_cast<size_t>(r), 0.0);
  for (Index j = 0; j < r; ++j) {
    Tt[size_t(j)] = alpha[size_t(j)] * t[size_t(j)];
    if (j > 0) Tt[size_t(j)] += beta[size_t(j - 1)] * t[size_t(j - 1)];
    if (j + 1 < r) Tt[size_t(j)] += beta[size_t(j)] * t[size_t(j + 1)];
  }
  Vec out(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < r; ++j) {
    const double* q = Q.col(j);
    for (Index i = 0; i < n; ++i) out[size_t(i)] += q[i] * Tt[size_t(j)];
  }
  return out;
}
Mat LanczosFactor::dense() const {
  const Index n = Q.rows;
  Mat A(n, n);
  Vec e(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < n; ++j) {
    e[size_t(j)] = 1.0;
    Vec c = apply(e.data());
    std::copy(c.begin(), c.end(), A.col(j));
    e[size_t(j)] = 0.0;
  }
  return A;
}

LanczosFactor lanczos_lowrank(const LinearOperator& op, Index rank, std::uint64_t seed) {
  const Index n = op.size();  // linalg.cpp:306-314
  if (rank <= 0 || rank > n) throw std::invalid_argument("Lanczos rank must lie in [1, N]");
  Vec q = gaussian_vector(n, seed);
  const double qn = norm(q.data(), n);
  for (auto& v : q) v /= qn;
  return lanczos_from_start(op, q, rank, mix_seed(seed, 1));
}

// ============================================================== dskip.cpp
OneDimFactor::OneDimFactor(const KernelSpec& k1, Grid g1, const double* coords, Index n,
                           int direction, int total_dims, bool dlogell)
    : n_(n), d_(total_dims), direction_(direction), grid_(std::move(g1)),
      interp_(build_interpolation(grid_, coords, n, 0)),
      kuu_(grid_, dlogell ? kernel_dlogell_profile(k1) : kernel_profile(k1)) {  // dskip.cpp:40-61
  if (grid_.dim() != 1) throw std::invalid_argument("one-dimensional factor needs a 1-D grid");
  if (direction < -1 || direction >= total_dims)
    throw std::invalid_argument("factor direction out of range");
  table_.resize(11);
  auto prof = dlogell ? kernel_dlogell_profile(k1) : kernel_profile(k1);
  for (int t = 0; t < 11; ++t) {
    double off = static_cast<double>(t - 5) * grid_.spacing[0];
    table_[size_t(t)] = prof(&off, 1);
  }
}

void OneDimFactor::mvm(const double* v, double* out) const {  // dskip.cpp:63-71
  const Index m = grid_.size();
  Vec u(static_cast<size_t>(m), 0.0);
  for (int g = 0; g <= d_; ++g) {
    Vec t(static_cast<size_t>(m), 0.0);
    group_matrix(g).tmul_add(v + g * n_, t.data());
    for (Index a = 0; a < m; ++a) u[size_t(a)] += t[size_t(a)];
  }
  Vec w(static_cast<size_t>(m));
  kuu_.mvm(u.data(), w.data());
  for (int g = 0; g <= d_; ++g) group_matrix(g).mul(w.data(), out + g * n_);
}

Vec OneDimFactor::diagonal() const {  // dskip.cpp:73-99
  Vec diag(static_cast<size_t>(size()));
  for (Index i = 0; i < n_; ++i) {
    const Index e0 = interp_.W.ptr[size_t(i)], e1 = interp_.W.ptr[size_t(i + 1)];
    double aw = 0.0, adw = 0.0;
    for (Index a = e0; a < e1; ++a)
      for (Index b = e0; b < e1; ++b) {
        const double k = table_[size_t(interp_.W.idx[size_t(a)] - interp_.W.idx[size_t(b)] + 5)];
        aw += interp_.W.val[size_t(a)] * interp_.W.val[size_t(b)] * k;
        adw += interp_.dW[0].val[size_t(a)] * interp_.dW[0].val[size_t(b)] * k;
      }
    for (int g = 0; g <= d_; ++g)
      diag[size_t(g * n_ + i)] = (direction_ >= 0 && g == direction_ + 1) ? adw : aw;
  }
  return diag;
}

Vec OneDimFactor::row(Index r) const {  // dskip.cpp:101-113
  if (r < 0 || r >= size()) throw std::out_of_range("factor row index out of range");
  const Index i = r % n_;
  const int g = static_cast<int>(r / n_);
  const Csr& M = group_matrix(g);
  Vec b(static_cast<size_t>(grid_.size()), 0.0);
  for (Index e = M.ptr[size_t(i)]; e < M.ptr[size_t(i + 1)]; ++e) b[size_t(M.idx[size_t(e)])] = M.val[size_t(e)];
  Vec w(static_cast<size_t>(grid_.size()));
  kuu_.mvm(b.data(), w.data());
  Vec out(static_cast<size_t>(size()));
  for (int gg = 0; gg <= d_; ++gg) group_matrix(gg).mul(w.data(), out.data() + gg * n_);
  return out;
}

OneDimFactor build_factor(const KernelSpec& k, const double* X, Index n, int d, int direction,
                          double grid_ratio, int max_grid_nodes, bool dlogell) {  // dskip.cpp:115-130
  if (k.family != SE)
    throw std::invalid_argument("kernel family 'spline' is not separable; the Hadamard "
                                "factorization needs a product kernel");
  if (direction < 0 || direction >= d) throw std::invalid_argument("factor direction out of range");
  KernelSpec k1;
  k1.family = SE;
  k1.ell = k.ell;
  k1.s = std::pow(k.s, 1.0 / d);
  Grid g = grid_cover(X + direction * n, n, 1, k.ell * grid_ratio, 3, max_grid_nodes);
  return OneDimFactor(k1, g, X + direction * n, n, direction, d, dlogell);
}

namespace {
Mat times_tridiagonal(const LanczosFactor& f) {  // dskip.cpp:13-22
  const Index r = f.rank(), n = f.Q.rows;
  Mat QT(n, r);
  for (Index k = 0; k < r; ++k) {
    double* o = QT.col(k);
    const double* q = f.Q.col(k);
    for (Index i = 0; i < n; ++i) o[i] = f.alpha[size_t(k)] * q[i];
    if (k > 0) {
      const double* qm = f.Q.col(k - 1);
      for (Index i = 0; i < n; ++i) o[i] += f.beta[size_t(k - 1)] * qm[i];
    }
    if (k + 1 < r) {
      const double* qp = f.Q.col(k + 1);
      for (Index i = 0; i < n; ++i) o[i] += f.beta[size_t(k)] * qp[i];
    }
  }
  return QT;
}

Vec hadamard_impl(const std::vector<const LanczosFactor*>& fs, size_t at, const double* v) {
  const LanczosFactor& A = *fs[at];  // dskip.cpp:24-36
  if (at + 1 == fs.size()) return A.apply(v);
  Mat QT = times_tridiagonal(A);
  const Index n = A.Q.rows;
  Vec out(static_cast<size_t>(n), 0.0), t(static_cast<size_t>(n));
  for (Index k = 0; k < A.rank(); ++k) {
    const double* q = A.Q.col(k);
    for (Index i = 0; i < n; ++i) t[size_t(i)] = q[i] * v[i];
    Vec u = hadamard_impl(fs, at + 1, t.data());
    const double* qt = QT.col(k);
    for (Index i = 0; i < n; ++i) out[size_t(i)] += qt[i] * u[size_t(i)];
  }
  return out;
}
}  // namespace

Vec hadamard_mvm(const std::vector<const LanczosFactor*>& f, const double* v) {
  if (f.empty()) throw std::invalid_argument("hadamard_mvm needs at least one factor");
  return hadamard_impl(f, 0, v);
}

Vec hadamard_diagonal(const std::vector<const LanczosFactor*>& fs) {
  if (fs.empty()) throw std::invalid_argument("no factors");
  const Index n = fs[0]->Q.rows;
  Vec diag(static_cast<size_t>(n), 1.0);
  for (auto* f : fs) {
    Mat QT = times_tridiagonal(*f);
    for (Index i = 0; i < n; ++i) {
      double s = 0.0;
      for (Index k = 0; k < f->rank(); ++k) s += QT(i, k) * f->Q(i, k);
      diag[size_t(i)] *= s;
    }
  }
  return diag;
}

Vec hadamard_row(const std::vector<const LanczosFactor*>& fs, Index i) {
  if (fs.empty()) throw std::invalid_argument("no factors");
  const Index n = fs[0]->Q.rows;
  if (i < 0 || i >= n) throw std::out_of_range("row index out of range");
  Vec row(static_cast<size_t>(n), 1.0);
  for (auto* f : fs) {
    const Index r = f->rank();
    Vec qi(static_cast<size_t>(r)), ti(static_cast<size_t>(r), 0.0);
    for (Index k = 0; k < r; ++k) qi[size_t(k)] = f->Q(i, k);
    for (Index k = 0; k < r; ++k) {
      ti[size_t(k)] = f->alpha[size_t(k)] * qi[size_t(k)];
      if (k > 0) ti[size_t(k)] += f->beta[size_t(k - 1)] * qi[size_t(k - 1)];
      if (k + 1 < r) ti[size_t(k)] += f->beta[size_t(k)] * qi[size_t(k + 1)];
    }
    for (Index a = 0; a < n; ++a) {
      double s = 0.0;
      for (Index k = 0; k < r; ++k) s += f->Q(a, k) * ti[size_t(k)];
      row[size_t(a)] *= s;
    }
  }
  return row;
}

DskipOperator::DskipOperator(const KernelSpec& k, const double* X, Index n, int d, NoiseLevels noise,
                             const DskipConfig& cfg)
    : n_(n), d_(d), groups_(cfg.with_gradients ? d : 0), noise_(noise), track_(cfg.track_dlogell) {
  const Index N = n_ * (groups_ + 1);  // dskip.cpp:162-234
  const Index rank = std::min(cfg.rank, N);
  if (rank < 1) throw std::invalid_argument("D-SKIP rank must be positive");
  if (k.family != SE)
    throw std::invalid_argument("kernel family 'spline' is not separable; the Hadamard "
                                "factorization needs a product kernel");
  KernelSpec k1;
  k1.family = SE;
  k1.ell = k.ell;
  k1.s = std::pow(k.s, 1.0 / d_);
  for (int j = 0; j < d_; ++j) {
    Grid g1 = grid_cover(X + j * n, n, 1, k.ell * cfg.grid_ratio, 3, cfg.max_grid_nodes);
    const int dir = cfg.with_gradients ? j : -1;
    const int groups = cfg.with_gradients ? d_ : 0;
    OneDimFactor leaf(k1, g1, X + j * n, n, dir, groups);
    factors_.push_back(lanczos_lowrank(leaf, rank, mix_seed(cfg.seed, std::uint64_t(j))));
    if (track_) {
      OneDimFactor dleaf(k1, g1, X + j * n, n, dir, groups, true);
      dlog_factors_.push_back(lanczos_lowrank(dleaf, rank, mix_seed(cfg.seed, 100 + std::uint64_t(j))));
    }
  }
  std::uint64_t merge_id = 1000;
  while (factors_.size() > 2) {
    std::vector<LanczosFactor> next, dnext;
    for (size_t a = 0; a + 1 < factors_.size(); a += 2) {
      const LanczosFactor& A = factors_[a];
      const LanczosFactor& B = factors_[a + 1];
      const Index product_rank = std::min(A.rank() * B.rank(), N);
      if (cfg.rank_policy_error && product_rank > rank)
        throw std::runtime_error("intermediate Hadamard rank " + std::to_string(product_rank) +
                                 " exceeds the cap " + std::to_string(rank));
      std::vector<const LanczosFactor*> pair = {&A, &B};
      CallbackOperator pair_op(N, [&pair, N](const double* x, double* y) {
        Vec r = hadamard_mvm(pair, x);
        std::copy(r.begin(), r.end(), y);
        (void)N;
      });
      next.push_back(lanczos_lowrank(pair_op, rank, mix_seed(cfg.seed, ++merge_id)));
      if (track_) {
        std::vector<const LanczosFactor*> dab = {&dlog_factors_[a], &B};
        std::vector<const LanczosFactor*> adb = {&A, &dlog_factors_[a + 1]};
        CallbackOperator dpair(N, [&dab, &adb, N](const double* x, double* y) {
          Vec r1 = hadamard_mvm(dab, x), r2 = hadamard_mvm(adb, x);
          for (Index i = 0; i < N; ++i) y[i] = r1[size_t(i)] + r2[size_t(i)];
        });
        dnext.push_back(lanczos_lowrank(dpair, rank, mix_seed(cfg.seed, ++merge_id)));
      }
    }
    if (factors_.size() % 2 == 1) {
      next.push_back(factors_.back());
      if (track_) dnext.push_back(dlog_factors_.back());
    }
    factors_ = std::move(next);
    dlog_factors_ = std::move(dnext);
  }
}

Vec DskipOperator::noise_diagonal() const {
  Vec nd(static_cast<size_t>(size()));
  for (Index i = 0; i < size(); ++i)
    nd[size_t(i)] = i < n_ ? noise_.value * noise_.value : noise_.gradient * noise_.gradient;
  return nd;
}

void DskipOperator::mvm(const double* v, double* out) const {  // dskip.cpp:243-250
  std::vector<const LanczosFactor*> fs;
  for (auto& f : factors_) fs.push_back(&f);
  Vec r = hadamard_mvm(fs, v);
  const double nv = noise_.value * noise_.value, ng = noise_.gradient * noise_.gradient;
  for (Index i = 0; i < size(); ++i) out[i] = r[size_t(i)] + (i < n_ ? nv : ng) * v[i];
}

Vec DskipOperator::diagonal() const {
  std::vector<const LanczosFactor*> fs;
  for (auto& f : factors_) fs.push_back(&f);
  Vec dg = hadamard_diagonal(fs);
  const double nv = noise_.value * noise_.value, ng = noise_.gradient * noise_.gradient;
  for (Index i = 0; i < size(); ++i) dg[size_t(i)] += i < n_ ? nv : ng;
  return dg;
}

Vec DskipOperator::row(Index i) const {
  if (i < 0 || i >= size()) throw std::out_of_range("D-SKIP row index out of range");
  std::vector<const LanczosFactor*> fs;
  for (auto& f : factors_) fs.push_back(&f);
  Vec r = hadamard_row(fs, i);
  r[size_t(i)] += (i < n_) ? noise_.value * noise_.value : noise_.gradient * noise_.gradient;
  return r;
}

Vec DskipOperator::dlogell_apply(const double* v) const {  // dskip.cpp:266-274
  if (!track_) throw std::logic_error("D-SKIP operator was built without derivative tracking");
  if (factors_.size() == 1) return dlog_factors_[0].apply(v);
  Vec a = hadamard_mvm({&dlog_factors_[0], &factors_[1]}, v);
  Vec b = hadamard_mvm({&factors_[0], &dlog_factors_[1]}, v);
  for (size_t i = 0; i < a.size(); ++i) a[i] += b[i];
  return a;
}

// ============================================================== gp.cpp glue
GpModel::GpModel(const KernelSpec& k, const double* X, const double* y, const double* dY, Index n,
                 int d, double nv, double ng, const GpConfig& cfg)
    : k_(k), X_(n, d), y_(y, y + n), n_(n), d_(d), nv_(nv), ng_(ng), cfg_(cfg) {
  std::copy(X, X + n * d, X_.a.begin());
  if (dY) {
    dY_ = Mat(n, d);
    std::copy(dY, dY + n * d, dY_.a.begin());
  }
  mean_ = std::accumulate(y_.begin(), y_.end(), 0.0) / double(n);  // gp.cpp:43 (Eigen mean)
}

const LinearOperator& GpModel::op() {  // gp.cpp:66-110
  if (op_) return *op_;
  const bool grads = dY_.rows > 0;
  if (cfg_.backend == 1) {
    Grid g = grid_cover(X_.a.data(), n_, d_, cfg_.grid_ratio * k_.ell, 3, cfg_.max_grid_nodes);
    auto p = std::make_unique<DskiOperator>(k_, g, X_.a.data(), n_, d_, NoiseLevels{nv_, ng_},
                                            cfg_.order, grads);
    dski_ = p.get();
    op_ = std::move(p);
  } else if (cfg_.backend == 2) {
    DskipConfig c;
    c.rank = cfg_.dskip_rank;
    c.grid_ratio = cfg_.dskip_grid_ratio;
    c.max_grid_nodes = cfg_.dskip_max_grid_nodes;
    c.seed = cfg_.seed;
    c.track_dlogell = true;
    c.with_gradients = grads;
    op_ = std::make_unique<DskipOperator>(k_, X_.a.data(), n_, d_, NoiseLevels{nv_, ng_}, c);
  } else {
    throw std::invalid_argument("oracle GpModel: exact backend not restated (dense LLT)");
  }
  return *op_;
}

const Preconditioner* GpModel::preconditioner() {  // gp.cpp:117-141
  if (!cfg_.use_preconditioner) return nullptr;
  if (precond_) return precond_.get();
  const LinearOperator& A = op();
  const Index N = A.size();
  Vec nd(static_cast<size_t>(N));
  for (Index i = 0; i < N; ++i) nd[size_t(i)] = i < n_ ? nv_ * nv_ : ng_ * ng_;
  Vec diag = A.diagonal();
  for (Index i = 0; i < N; ++i) diag[size_t(i)] = std::max(diag[size_t(i)] - nd[size_t(i)], 0.0);
  auto row_fn = [&](Index i) {
    Vec r = A.row(i);
    r[size_t(i)] -= nd[size_t(i)];
    return r;
  };
  factor_ = std::make_unique<PivotedCholeskyFactor>(
      pivoted_cholesky(diag, row_fn, std::min(cfg_.precond_rank, N), 0.0));
  if (factor_->L.cols == 0)
    throw std::runtime_error("pivoted Cholesky produced an empty preconditioner factor");
  precond_ = std::make_unique<Preconditioner>(factor_->L, nd);
  return precond_.get();
}

Vec GpModel::stacked_targets() const {  // observations.hpp:29-35
  const bool grads = dY_.rows > 0;
  Vec t(static_cast<size_t>(n_ * (grads ? d_ + 1 : 1)));
  for (Index i = 0; i < n_; ++i) t[size_t(i)] = y_[size_t(i)] - mean_;
  if (grads)
    for (int j = 0; j < d_; ++j)
      for (Index i = 0; i < n_; ++i) t[size_t(n_ * (j + 1) + i)] = dY_(i, j);
  return t;
}

const Vec& GpModel::alpha() {  // gp.cpp:143-163
  if (alpha_) return *alpha_;
  const LinearOperator& A = op();
  const Preconditioner* M = preconditioner();
  Vec b = stacked_targets();
  last_solve = cg(A, b.data(), cfg_.cg, M ? M->as_apply() : PrecondApply{});
  if (!last_solve.converged)
    throw std::runtime_error("CG did not converge: relative residual " +
                             std::to_string(last_solve.residual_history.back()) + " after " +
                             std::to_string(last_solve.iterations) + " iterations");
  alpha_ = std::make_unique<Vec>(last_solve.x);
  return *alpha_;
}

double GpModel::logdet() {  // gp.cpp:165-179
  const LinearOperator& A = op();
  SlqOptions o;
  o.probes = cfg_.slq_probes;
  o.lanczos_steps = cfg_.slq_steps;
  o.seed = cfg_.seed;
  const double f = dY_.rows > 0 ? std::min(nv_, ng_) : nv_;
  o.eigen_floor = 0.5 * f * f;
  return slq_logdet(A, o).logdet;
}

double GpModel::log_marginal_likelihood() {  // gp.cpp:181-187
  Vec t = stacked_targets();
  const Vec& a = alpha();
  const double fit = dot(t.data(), a.data(), Index(t.size()));
  const double cpx = logdet();
  const double N = double(t.size());
  return -0.5 * (fit + cpx + N * std::log(2.0 * M_PI));
}

Vec GpModel::kernel_part_apply(const double* v) {  // gp.cpp:189-198
  const LinearOperator& A = op();
  const Index N = A.size();
  Vec out(static_cast<size_t>(N));
  A.mvm(v, out.data());
  for (Index i = 0; i < N; ++i) out[size_t(i)] -= (i < n_ ? nv_ * nv_ : ng_ * ng_) * v[i];
  return out;
}

Vec GpModel::dlogell_apply(const double* v) {  // gp.cpp:200-218
  op();
  if (cfg_.backend == 1) {
    // the second grid operator over kernel_dlogell_profile (gp.cpp:212-213)
    if (!kuu_dlogell_)
      kuu_dlogell_ = std::make_unique<GridKernelOperator>(dski_->grid(), kernel_dlogell_profile(k_));
    Vec u = dski_->stacked_transpose_apply(v);
    Vec w(u.size());
    kuu_dlogell_->mvm(u.data(), w.data());
    return dski_->stacked_apply(w.data());
  }
  return static_cast<const DskipOperator&>(*op_).dlogell_apply(v);
}

void GpModel::set_hyperparameters(double ell, double s, double nv, double ng) {  // gp.cpp:46-64
  if (nv <= 0.0) throw std::invalid_argument("value noise must be positive");
  k_.ell = ell;
  k_.s = s;
  nv_ = nv;
  ng_ = ng;
  op_.reset();
  dski_ = nullptr;
  precond_.reset();
  factor_.reset();
  alpha_.reset();
  mean_grid_.reset();
  kuu_dlogell_.reset();
}

// Projected gradient ascent in log-parameter space with a per-restart step
// that grows ×1.4 on acceptance and shrinks ×0.4 on rejection; restarts
// r > 0 jitter the start by U(−0.7, 0.7) from seeded_rng(seed, 31 + r).
GpModel::FitOut GpModel::fit(int max_iterations, int restarts_opt, double initial_step, double min_step,
                             bool optimize_noise, std::uint64_t seed) {
  const bool grads = dY_.rows > 0;
  const int np = grads ? 4 : 3;
  auto encode = [&] {
    Vec p(static_cast<size_t>(np));
    p[0] = std::log(k_.ell);
    p[1] = std::log(k_.s);
    p[2] = std::log(nv_);
    if (grads) p[3] = std::log(ng_);
    return p;
  };
  auto decode = [&](const Vec& p) {
    set_hyperparameters(std::exp(p[0]), std::exp(p[1]), std::exp(p[2]), grads ? std::exp(p[3]) : ng_);
  };
  auto clampv = [](double v, double lo, double hi) { return std::min(std::max(v, lo), hi); };
  auto clamp_params = [&](Vec p) {
    p[0] = clampv(p[0], std::log(1e-4), std::log(1e4));
    p[1] = clampv(p[1], std::log(1e-6), std::log(1e6));
    for (int i = 2; i < np; ++i) p[i] = clampv(p[i], std::log(1e-6), std::log(1e3));
    return p;
  };
  const Vec p0 = encode();
  const int restarts = max_iterations > 0 ? std::max(restarts_opt, 1) : 1;
  FitOut best;
  best.log_marginal = -std::numeric_limits<double>::infinity();
  Vec best_p = p0;
  bool any_ok = false;
  std::string errors;
  for (int r = 0; r < restarts; ++r) {
    FitReport rep;
    Vec p = p0;
    if (r > 0) {
      std::mt19937_64 rng(mix_seed(seed, 31 + std::uint64_t(r)));
      std::uniform_real_distribution<double> jitter(-0.7, 0.7);
      for (int i = 0; i < np; ++i) p[i] += jitter(rng);
      p = clamp_params(p);
    }
    try {
      decode(p);
      double L = log_marginal_likelihood();
      double step = initial_step;
      int it = 0;
      for (; it < max_iterations; ++it) {
        Vec g;
        try {
          g = lml_gradient();
        } catch (const std::exception&) {
          break;
        }
        if (!optimize_noise) {
          g[2] = 0.0;
          if (np == 4) g[3] = 0.0;
        }
        double gn = 0.0;
        for (double v : g) {
          if (!std::isfinite(v)) throw std::runtime_error("non-finite likelihood gradient");
          gn += v * v;
        }
        if (std::sqrt(gn) < 1e-10) break;
        bool accepted = false;
        while (step >= min_step) {
          Vec pt = p;
          for (int i = 0; i < np; ++i) pt[i] = p[i] + clampv(step * g[i], -0.5, 0.5);
          pt = clamp_params(pt);
          decode(pt);
          double Lt;
          try {
            Lt = log_marginal_likelihood();
          } catch (const std::exception&) {
            Lt = -std::numeric_limits<double>::infinity();
          }
          if (std::isfinite(Lt) && Lt > L) {
            p = pt;
            L = Lt;
            step = std::min(step * 1.4, 2.0);
            ++rep.accepted_steps;
            accepted = true;
            break;
          }
          step *= 0.4;
        }
        if (!accepted) break;
      }
      decode(p);
      rep.succeeded = true;
      rep.iterations = it;
      rep.log_marginal = L;
      if (L > best.log_marginal) {
        best.log_marginal = L;
        best_p = p;
      }
      any_ok = true;
    } catch (const std::exception& e) {
      rep.succeeded = false;
      errors += std::string(" [") + e.what() + "]";
    }
    best.restarts.push_back(rep);
  }
  if (!any_ok) throw std::runtime_error("all fit restarts failed:" + errors);
  decode(best_p);
  best.ell = k_.ell;
  best.s = k_.s;
  best.nv = nv_;
  best.ng = ng_;
  return best;
}

Vec GpModel::lml_gradient() {  // gp.cpp:220-292
  const LinearOperator& A = op();
  const Index N = A.size();
  const bool grads = dY_.rows > 0;
  const int nparams = grads ? 4 : 3;
  const Vec a = alpha();
  // dK/dθ over (log ℓ, log s, log σ₁[, log σ₂]) (gp.cpp:229-244)
  auto apply_param = [&](int p, const double* v) {
    Vec out(static_cast<size_t>(N), 0.0);
    if (p == 0) return dlogell_apply(v);
    if (p == 1) {
      out = kernel_part_apply(v);
      for (auto& x : out) x *= 2.0;
    } else if (p == 2) {
      for (Index i = 0; i < n_; ++i) out[size_t(i)] = (2.0 * nv_ * nv_) * v[i];
    } else {
      for (Index i = n_; i < N; ++i) out[size_t(i)] = (2.0 * ng_ * ng_) * v[i];
    }
    return out;
  };
  const Preconditioner* M = preconditioner();
  const PrecondApply precond = M ? M->as_apply() : PrecondApply{};
  CgOptions trace_cg = cfg_.cg;
  trace_cg.tol = std::max(cfg_.cg.tol, 1e-2);  // gp.cpp:281-282
  Vec grad(static_cast<size_t>(nparams));
  for (int p = 0; p < nparams; ++p) {
    Vec Ma = apply_param(p, a.data());
    CallbackOperator Mop(N, [&](const double* x, double* y) {
      Vec r = apply_param(p, x);
      std::copy(r.begin(), r.end(), y);
    });
    const double tr = trace_estimate(A, Mop, cfg_.gradient_probes, cfg_.seed, trace_cg, precond);
    grad[size_t(p)] = 0.5 * (dot(a.data(), Ma.data(), N) - tr);
  }
  return grad;
}

std::pair<Vec, Mat> GpModel::predict_mean_grad(const double* Xt, Index T) {  // gp.cpp:471-496
  op();
  if (!dski_) throw std::logic_error("oracle predict_mean_grad: D-SKI backend only");
  const Vec& a = alpha();
  if (!mean_grid_) {
    Vec u = dski_->stacked_transpose_apply(a.data());
    mean_grid_ = std::make_unique<Vec>(static_cast<size_t>(u.size()));
    dski_->grid_operator().mvm(u.data(), mean_grid_->data());
  }
  const Vec& g = *mean_grid_;
  Vec values(static_cast<size_t>(T));
  Mat grads(T, d_);
  double x[16];
  for (Index t = 0; t < T; ++t) {
    for (int j = 0; j < d_; ++j) x[j] = Xt[j * T + t];
    PointStencil st = point_stencil(dski_->grid(), x, cfg_.order);
    double acc = 0.0, gr[16] = {0};
    for (size_t c = 0; c < st.indices.size(); ++c) {
      acc += st.value[c] * g[size_t(st.indices[c])];
      for (int p = 0; p < d_; ++p) gr[p] += st.derivative(Index(c), p) * g[size_t(st.indices[c])];
    }
    values[size_t(t)] = mean_ + acc;
    for (int p = 0; p < d_; ++p) grads(t, p) = gr[p];
  }
  return {values, grads};
}

Vec GpModel::cross_covariance(const double* x) {  // gp.cpp:406-417 (D-SKI)
  op();
  if (!dski_) throw std::logic_error("oracle cross_covariance: D-SKI backend only");
  PointStencil st = point_stencil(dski_->grid(), x, cfg_.order);
  Vec w(static_cast<size_t>(dski_->grid().size()), 0.0);
  for (size_t c = 0; c < st.indices.size(); ++c) w[size_t(st.indices[c])] = st.value[c];
  Vec kw(w.size());
  dski_->grid_operator().mvm(w.data(), kw.data());
  return dski_->stacked_apply(kw.data());
}

Vec GpModel::solve(const double* b) {  // gp.cpp:143-158 (tol_scale = 1)
  const LinearOperator& A = op();
  const Preconditioner* M = preconditioner();
  CgResult r = cg(A, b, cfg_.cg, M ? M->as_apply() : PrecondApply{});
  if (!r.converged)
    throw std::runtime_error("CG did not converge: relative residual " + std::to_string(r.residual_history.back()) +
                             " after " + std::to_string(r.iterations) + " iterations");
  return r.x;
}

double GpModel::predict_variance_exact(const double* x) {  // gp.cpp:499-502
  Vec q = cross_covariance(x);
  Vec s = solve(q.data());
  return k_eval(k_, x, x, d_) - dot(q.data(), s.data(), Index(q.size()));
}

// gp.cpp:519-547: pivoted-Cholesky base plus an unbiased control-variate
// correction with Rademacher probes over the test points (streams 9000 + p).
Vec GpModel::predict_variance_randomized(const double* Xt, Index T, int probes, std::uint64_t seed) {
  const Preconditioner* M = preconditioner();
  if (!M) throw std::logic_error("randomized variance needs the preconditioner enabled");
  const Index N = op().size();
  std::vector<Vec> Kc(static_cast<size_t>(T));
  Vec base(static_cast<size_t>(T));
  std::vector<double> x(static_cast<size_t>(d_));
  for (Index t = 0; t < T; ++t) {
    for (int j = 0; j < d_; ++j) x[size_t(j)] = Xt[j * T + t];
    Kc[size_t(t)] = cross_covariance(x.data());
    base[size_t(t)] = k_eval(k_, x.data(), x.data(), d_) - M->quadratic(Kc[size_t(t)]);
  }
  if (probes <= 0) return base;
  Vec corr(static_cast<size_t>(T), 0.0);
  for (int p = 0; p < probes; ++p) {
    Vec z = rademacher_vector(T, seed, 9000 + std::uint64_t(p));
    Vec w(static_cast<size_t>(N), 0.0);
    for (Index t = 0; t < T; ++t)
      for (Index i = 0; i < N; ++i) w[size_t(i)] += Kc[size_t(t)][size_t(i)] * z[size_t(t)];
    Vec ex = solve(w.data());
    Vec ap = M->apply(w);
    for (Index t = 0; t < T; ++t) {
      double s = 0.0;
      for (Index i = 0; i < N; ++i) s += Kc[size_t(t)][size_t(i)] * (ex[size_t(i)] - ap[size_t(i)]);
      corr[size_t(t)] += z[size_t(t)] * s;
    }
  }
  for (Index t = 0; t < T; ++t) base[size_t(t)] -= corr[size_t(t)] / double(probes);
  return base;
}

Mat GpModel::cross_covariance_jacobian(const double* x) {  // gp.cpp:431-446 (D-SKI)
  op();
  if (!dski_) throw std::logic_error("oracle cross_covariance_jacobian: D-SKI backend only");
  PointStencil st = point_stencil(dski_->grid(), x, cfg_.order);
  const Index N = dski_->size();
  Mat J(N, d_);
  for (int p = 0; p < d_; ++p) {
    Vec w(static_cast<size_t>(dski_->grid().size()), 0.0);
    for (size_t c = 0; c < st.indices.size(); ++c) w[size_t(st.indices[c])] = st.derivative(c, p);
    Vec kw(w.size());
    dski_->grid_operator().mvm(w.data(), kw.data());
    Vec col = dski_->stacked_apply(kw.data());
    for (Index i = 0; i < N; ++i) J(i, p) = col[size_t(i)];
  }
  return J;
}

double GpModel::predict_variance_pivchol(const double* x) {  // gp.cpp:511-517
  const Preconditioner* M = preconditioner();
  if (!M) throw std::logic_error("pivoted Cholesky variance needs the preconditioner enabled");
  Vec q = cross_covariance(x);
  return k_eval(k_, x, x, d_) - M->quadratic(q);
}

}  // namespace gko
