// gk_oracle.hpp — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's (gradkrig, arXiv 1810.12283) hot path,
// used as the parity checker for the B200 path and as the CPU baseline in
// bench.py. Nothing in the product path (paper_1810_12283_b200/) links or
// calls this code; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs do.
//
// The reference itself cannot be compiled here (needs Eigen3 + FFTW3, both
// absent), so this is a dependency-free port: every
// function cites the reference file:line it restates. Parity of the port is
// pinned by the reference's own known-answer tests and dense-algebra
// identities (tests/test_oracle_*.py), plus numpy/scipy cross-checks.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace gko {

using Index = std::int64_t;
using Vec = std::vector<double>;

// Column-major dense matrix (Eigen default layout).
struct Mat {
  Index rows = 0, cols = 0;
  Vec a;
  Mat() = default;
  Mat(Index r, Index c, double v = 0.0) : rows(r), cols(c), a(size_t(r * c), v) {}
  double& operator()(Index i, Index j) { return a[size_t(j * rows + i)]; }
  double operator()(Index i, Index j) const { return a[size_t(j * rows + i)]; }
  double* col(Index j) { return a.data() + j * rows; }
  const double* col(Index j) const { return a.data() + j * rows; }
};

// ---------------------------------------------------------------- rng.hpp:12-38
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream);
inline std::mt19937_64 seeded_rng(std::uint64_t seed, std::uint64_t stream = 0) {
  return std::mt19937_64(mix_seed(seed, stream));
}
Vec rademacher_vector(Index n, std::uint64_t seed, std::uint64_t stream = 0);
Vec gaussian_vector(Index n, std::uint64_t seed, std::uint64_t stream = 0);

// ---------------------------------------------------------------- kernels (kernels.hpp/.cpp)
enum Family { SE = 0, SPLINE = 1 };
struct KernelSpec {
  int family = SE;
  double ell = 1.0, s = 1.0;
  double spline_a = -1.5, spline_b = 1.0;
  bool spline_even = false;
};
double k_eval(const KernelSpec& k, const double* x, const double* xp, int d);        // kernels.cpp:104-118
void k_eval_grad(const KernelSpec& k, const double* x, const double* xp, int d, double* g);  // :120-136
void k_eval_hess(const KernelSpec& k, const double* x, const double* xp, int d, double* H);  // :138-170 (row-major d×d)
double k_eval_dlogell(const KernelSpec& k, const double* x, const double* xp, int d);        // :172-188
// Dense K∇ in type-major layout (kernels.cpp:242-285); X is n×d col-major.
Mat assemble_dense(const KernelSpec& k, const double* X, Index n, const double* Xp, Index np, int d,
                   bool with_derivatives, Index size_cap = 50'000'000);

// ---------------------------------------------------------------- interpolation
struct Grid {
  std::vector<int> dims;
  Vec origin, spacing;
  int dim() const { return int(dims.size()); }
  Index size() const;
};
struct OutOfGridError : std::runtime_error {
  Index point;
  OutOfGridError(const std::string& w, Index p) : std::runtime_error(w), point(p) {}
};
// interpolation.cpp:117-146 (X n×d col-major)
Grid grid_cover(const double* X, Index n, int d, double target_spacing, int margin, int max_nodes);
void quintic_weights(double t, double w[6], double dw[6]);  // interpolation.cpp:148-158
void cubic_weights(double t, double w[4], double dw[4]);    // interpolation.cpp:160-170

// RowMajor CSR (Eigen::SparseMatrix<double, RowMajor>): columns ascending per row.
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<Index> ptr;
  std::vector<Index> idx;
  Vec val;
  void mul(const double* x, double* y) const;       // y = A x (row-major dot per row)
  void tmul_add(const double* x, double* y) const;  // y += A^T x (rows in order)
};
struct SparseInterpolation {
  Csr W;
  std::vector<Csr> dW;
};
// interpolation.cpp:212-266; order 0 = quintic, 1 = cubic
SparseInterpolation build_interpolation(const Grid& g, const double* X, Index n, int order);
struct PointStencil {
  std::vector<Index> indices;
  Vec value;
  Mat derivative;  // nnz × d
};
PointStencil point_stencil(const Grid& g, const double* x, int order);  // interpolation.cpp:172-210

// ---------------------------------------------------------------- linear operators
class LinearOperator {  // linear_operator.hpp:12-35
 public:
  virtual ~LinearOperator() = default;
  virtual Index size() const = 0;
  virtual void mvm(const double* x, double* y) const = 0;
  virtual bool has_diagonal() const { return false; }
  virtual Vec diagonal() const { throw std::logic_error("operator does not expose its diagonal"); }
  virtual bool has_rows() const { return false; }
  virtual Vec row(Index) const { throw std::logic_error("operator does not expose rows"); }
  Vec apply(const Vec& x) const {
    Vec y(static_cast<size_t>(size()));
    mvm(x.data(), y.data());
    return y;
  }
  Mat dense() const;
};

class DenseOperator final : public LinearOperator {  // linear_operator.hpp:38-56
 public:
  explicit DenseOperator(Mat A) : A_(std::move(A)) {}
  Index size() const override { return A_.rows; }
  void mvm(const double* x, double* y) const override;
  bool has_diagonal() const override { return true; }
  Vec diagonal() const override;
  bool has_rows() const override { return true; }
  Vec row(Index i) const override;
  const Mat& matrix() const { return A_; }

 private:
  Mat A_;
};

class CallbackOperator final : public LinearOperator {  // linear_operator.hpp:60-76
 public:
  using Apply = std::function<void(const double*, double*)>;
  CallbackOperator(Index n, Apply f) : n_(n), f_(std::move(f)) {}
  Index size() const override { return n_; }
  void mvm(const double* x, double* y) const override { f_(x, y); }

 private:
  Index n_;
  Apply f_;
};

// ---------------------------------------------------------------- dski (dski.hpp/.cpp)
// Stationary profile evaluated at an offset vector (dski.cpp:30-40).
using Profile = std::function<double(const double* offset, int d)>;
Profile kernel_profile(const KernelSpec& k);
Profile kernel_dlogell_profile(const KernelSpec& k);

class Fft;  // mixed-radix complex FFT plan (fft.cpp)

class GridKernelOperator {  // dski.cpp:42-172
 public:
  GridKernelOperator(Grid g, const Profile& profile);
  ~GridKernelOperator();
  GridKernelOperator(GridKernelOperator&&) noexcept;
  Index size() const { return grid_.size(); }
  const Grid& grid() const { return grid_; }
  void mvm(const double* v, double* out) const;
  double min_embedding_eigenvalue() const;

 private:
  Grid grid_;
  std::vector<int> edims_;
  Index embed_total_ = 0;
  Vec spectrum_;  // real part of the full embedding spectrum
  std::vector<std::unique_ptr<Fft>> plans_;
  void fftn(std::vector<double>& re, std::vector<double>& im, bool inverse) const;
};

struct NoiseLevels {
  double value = 0.0, gradient = 0.0;
};

class DskiOperator final : public LinearOperator {  // dski.cpp:174-304
 public:
  DskiOperator(const KernelSpec& k, Grid g, const double* X, Index n, int d, NoiseLevels noise,
               int order = 0, bool with_gradients = true);
  Index size() const override { return n_ * (groups_ + 1); }
  void mvm(const double* v, double* out) const override;
  bool has_diagonal() const override { return true; }
  Vec diagonal() const override;
  bool has_rows() const override { return true; }
  Vec row(Index r) const override;
  Index points() const { return n_; }
  int input_dim() const { return d_; }
  int groups() const { return groups_; }
  const Grid& grid() const { return grid_; }
  const SparseInterpolation& interpolation() const { return interp_; }
  const GridKernelOperator& grid_operator() const { return kuu_; }
  Vec noise_diagonal() const;
  Vec stacked_transpose_apply(const double* v) const;  // dski.cpp:213-219
  Vec stacked_apply(const double* u) const;            // dski.cpp:221-226

 private:
  Index n_;
  int d_, groups_;
  Grid grid_;
  KernelSpec kernel_;
  NoiseLevels noise_;
  SparseInterpolation interp_;
  GridKernelOperator kuu_;
  Vec table_;
  std::vector<int> table_dims_;
};

// ---------------------------------------------------------------- linalg (linalg.hpp/.cpp)
struct CgOptions {
  double tol = 1e-4;
  int max_iterations = 1000;
};
struct CgResult {
  Vec x;
  int iterations = 0;
  bool converged = false;
  Vec residual_history;
};
using PrecondApply = std::function<Vec(const Vec&)>;
CgResult cg(const LinearOperator& A, const double* b, const CgOptions& o = {},
            const PrecondApply& M = {});  // linalg.cpp:85-131

struct PivotedCholeskyFactor {
  Mat L;
  std::vector<Index> pivots;
  double initial_trace = 0.0, residual_trace = 0.0;
};
PivotedCholeskyFactor pivoted_cholesky(const Vec& diag, const std::function<Vec(Index)>& row_fn,
                                       Index max_rank, double trace_tol = 0.0);  // :133-174

class Preconditioner {  // linalg.cpp:176-213 (Householder QR of [D^-1/2 F; I])
 public:
  Preconditioner(const Mat& F, const Vec& noise_diag);
  Preconditioner(const Mat& F, double sigma, Index n);
  Vec apply(const Vec& b) const;
  double quadratic(const Vec& b) const;
  PrecondApply as_apply() const {
    return [this](const Vec& b) { return apply(b); };
  }
  Index size() const { return Index(inv_sqrt_noise_.size()); }
  Index rank() const { return Q1_.cols; }
  const Mat& q1() const { return Q1_; }
  const Vec& inv_sqrt_noise() const { return inv_sqrt_noise_; }

 private:
  Vec inv_sqrt_noise_;
  Mat Q1_;
};

struct SlqOptions {
  int probes = 10;
  int lanczos_steps = 50;
  std::uint64_t seed = 0;
  double eigen_floor = 1e-12;
};
struct SlqResult {
  double logdet = 0.0;
  int clamped = 0;
  Vec estimates;  // per-probe (for sharded parity)
};
SlqResult slq_logdet(const LinearOperator& A, const SlqOptions& o = {});  // linalg.cpp:215-253
double trace_estimate(const LinearOperator& A, const LinearOperator& B, int probes,
                      std::uint64_t seed, const CgOptions& o = {}, const PrecondApply& M = {});

struct LanczosFactor {  // linalg.hpp:102-114
  Mat Q;
  Vec alpha, beta;
  bool breakdown = false;
  Index rank() const { return Q.cols; }
  Mat tridiagonal() const;
  Vec ritz_values() const;  // descending
  Vec apply(const double* v) const;
  Mat dense() const;
};
LanczosFactor lanczos_from_start(const LinearOperator& op, const Vec& start, Index steps,
                                 std::uint64_t restart_seed);  // linalg.cpp:17-81
LanczosFactor lanczos_lowrank(const LinearOperator& op, Index rank, std::uint64_t seed);  // :306-314

// Symmetric tridiagonal eigendecomposition (Eigen computeFromTridiagonal
// equivalent): ascending eigenvalues, and the first row of the eigenvector
// matrix (all that SLQ needs) or the full matrix.
void tridiag_eig(const Vec& alpha, const Vec& beta, Vec& evals, Mat* evecs);

// ---------------------------------------------------------------- dskip (dskip.hpp/.cpp)
class OneDimFactor final : public LinearOperator {  // dskip.cpp:40-113
 public:
  OneDimFactor(const KernelSpec& k1, Grid g1, const double* coords, Index n, int direction,
               int total_dims, bool dlogell = false);
  Index size() const override { return n_ * (d_ + 1); }
  void mvm(const double* v, double* out) const override;
  bool has_diagonal() const override { return true; }
  Vec diagonal() const override;
  bool has_rows() const override { return true; }
  Vec row(Index r) const override;
  const Grid& grid() const { return grid_; }

 private:
  const Csr& group_matrix(int g) const {
    return (direction_ >= 0 && g == direction_ + 1) ? interp_.dW[0] : interp_.W;
  }
  Index n_;
  int d_, direction_;
  Grid grid_;
  SparseInterpolation interp_;
  GridKernelOperator kuu_;
  Vec table_;
};
OneDimFactor build_factor(const KernelSpec& k, const double* X, Index n, int d, int direction,
                          double grid_ratio = 0.1, int max_grid_nodes = 512, bool dlogell = false);

Vec hadamard_mvm(const std::vector<const LanczosFactor*>& f, const double* v);  // dskip.cpp:24-36,132-139
Vec hadamard_diagonal(const std::vector<const LanczosFactor*>& f);              // :141-149
Vec hadamard_row(const std::vector<const LanczosFactor*>& f, Index i);          // :151-160

struct DskipConfig {  // dskip.hpp:74-85
  Index rank = 100;
  double grid_ratio = 0.1;
  int max_grid_nodes = 512;
  std::uint64_t seed = 0;
  bool rank_policy_error = false;
  bool track_dlogell = false;
  bool with_gradients = true;
};
class DskipOperator final : public LinearOperator {  // dskip.cpp:162-274
 public:
  DskipOperator(const KernelSpec& k, const double* X, Index n, int d, NoiseLevels noise,
                const DskipConfig& cfg = {});
  // Over given Lanczos factors (e.g. the device build's), for Hadamard-MVM
  // parity with identical factors at full size.
  DskipOperator(Index n, int groups, NoiseLevels noise, std::vector<LanczosFactor> factors)
      : n_(n), d_(groups), groups_(groups), noise_(noise), factors_(std::move(factors)) {}
  Index size() const override { return n_ * (groups_ + 1); }
  void mvm(const double* v, double* out) const override;
  bool has_diagonal() const override { return true; }
  Vec diagonal() const override;
  bool has_rows() const override { return true; }
  Vec row(Index i) const override;
  Vec noise_diagonal() const;
  const std::vector<LanczosFactor>& factors() const { return factors_; }
  Vec dlogell_apply(const double* v) const;

 private:
  Index n_;
  int d_, groups_;
  NoiseLevels noise_;
  std::vector<LanczosFactor> factors_, dlog_factors_;
  bool track_ = false;
};

// ---------------------------------------------------------------- gp glue (gp.cpp:117-187,471-517)
struct GpConfig {
  int backend = 1;  // 0 exact, 1 dski, 2 dskip
  double grid_ratio = 0.2;
  int max_grid_nodes = 128;
  Index dskip_rank = 100;
  double dskip_grid_ratio = 0.1;
  int dskip_max_grid_nodes = 512;
  CgOptions cg{1e-4, 1000};
  bool use_preconditioner = true;
  Index precond_rank = 100;
  int slq_probes = 10, slq_steps = 50;
  std::uint64_t seed = 0;
  int order = 0;
  int gradient_probes = 8;  // gp.hpp:43
};
class GpModel {
 public:
  GpModel(const KernelSpec& k, const double* X, const double* y, const double* dY /*n×d or null*/,
          Index n, int d, double noise_value, double noise_gradient, const GpConfig& cfg);
  const LinearOperator& op();
  const Preconditioner* preconditioner();
  const PivotedCholeskyFactor* pivchol() { preconditioner(); return factor_.get(); }
  Vec stacked_targets() const;
  const Vec& alpha();
  CgResult last_solve;
  double logdet();
  double log_marginal_likelihood();
  std::pair<Vec, Mat> predict_mean_grad(const double* Xtest, Index T);
  double predict_variance_pivchol(const double* x);
  Vec solve(const double* b);                     // gp.cpp:143-158
  Mat cross_covariance_jacobian(const double* x);  // gp.cpp:431-461 (D-SKI)
  double predict_variance_exact(const double* x);  // gp.cpp:499-502
  Vec predict_variance_randomized(const double* Xt /*T×d col-major*/, Index T, int probes, std::uint64_t seed);
  Vec cross_covariance(const double* x);
  double mean() const { return mean_; }
  Vec kernel_part_apply(const double* v);  // gp.cpp:189-198
  Vec dlogell_apply(const double* v);      // gp.cpp:200-218 (D-SKI / D-SKIP branches)
  Vec lml_gradient();                      // gp.cpp:220-292 (stochastic-trace branch)
  void set_gradient_probes(int p) { cfg_.gradient_probes = p; }
  void set_hyperparameters(double ell, double s, double nv, double ng);  // gp.cpp:46-64
  struct FitReport {
    bool succeeded = false;
    double log_marginal = 0.0;
    int iterations = 0, accepted_steps = 0;
  };
  struct FitOut {
    double ell, s, nv, ng, log_marginal;
    std::vector<FitReport> restarts;
  };
  // gp.cpp:294-404 (FitOptions gp.hpp:50-57)
  FitOut fit(int max_iterations, int restarts, double initial_step, double min_step, bool optimize_noise,
             std::uint64_t seed);

 private:
  KernelSpec k_;
  Mat X_;
  Vec y_;
  Mat dY_;
  Index n_;
  int d_;
  double nv_, ng_, mean_ = 0.0;
  GpConfig cfg_;
  std::unique_ptr<LinearOperator> op_;
  DskiOperator* dski_ = nullptr;
  std::unique_ptr<Preconditioner> precond_;
  std::unique_ptr<PivotedCholeskyFactor> factor_;
  std::unique_ptr<Vec> alpha_, mean_grid_;
  std::unique_ptr<GridKernelOperator> kuu_dlogell_;
};

}  // namespace gko
