// gk_oracle_capi.cpp — TEST INFRASTRUCTURE ONLY. extern "C" surface of the
// CPU oracle for ctypes (oracle/__init__.py). Status codes mirror the
// product C-ABI (include/gk_capi.h) so tests can compare error behaviour.
#include <cstring>
#include <string>

#include "gk_oracle.hpp"

using namespace gko;

namespace {
thread_local std::string g_err;
thread_local long long g_err_point = -1;

enum {
  OK = 0, ERR_ARG = 1, ERR_RANGE = 2, ERR_OUT_OF_GRID = 3, ERR_RUNTIME = 4, ERR_LOGIC = 5,
  ERR_LENGTH = 6, ERR_OTHER = 9
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return OK;
  } catch (const OutOfGridError& e) {
    g_err = e.what();
    g_err_point = e.point;
    return ERR_OUT_OF_GRID;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ERR_ARG;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return ERR_RANGE;
  } catch (const std::length_error& e) {
    g_err = e.what();
    return ERR_LENGTH;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ERR_LOGIC;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ERR_OTHER;
  }
}

KernelSpec mk_kernel(int family, double ell, double s, double a, double b, int even) {
  KernelSpec k;
  k.family = family;
  k.ell = ell;
  k.s = s;
  k.spline_a = a;
  k.spline_b = b;
  k.spline_even = even != 0;
  return k;
}

Grid mk_grid(const int* dims, const double* origin, const double* spacing, int d) {
  Grid g;
  g.dims.assign(dims, dims + d);
  g.origin.assign(origin, origin + d);
  g.spacing.assign(spacing, spacing + d);
  return g;
}

void copy_out(const Vec& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

struct Precond {
  std::unique_ptr<Preconditioner> p;
};
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
long long orc_last_error_point() { return g_err_point; }

unsigned long long orc_mix_seed(unsigned long long seed, unsigned long long stream) {
  return mix_seed(seed, stream);
}
void orc_rademacher(long long n, unsigned long long seed, unsigned long long stream, double* out) {
  copy_out(rademacher_vector(n, seed, stream), out);
}
void orc_gaussian(long long n, unsigned long long seed, unsigned long long stream, double* out) {
  copy_out(gaussian_vector(n, seed, stream), out);
}
unsigned long long orc_mt19937_64_nth(unsigned long long seed, long long nth) {
  std::mt19937_64 r(seed);
  unsigned long long v = 0;
  for (long long i = 0; i < nth; ++i) v = r();
  return v;
}

int orc_quintic_weights(double t, double* w, double* dw) {
  return guard([&] { quintic_weights(t, w, dw); });
}
int orc_cubic_weights(double t, double* w, double* dw) {
  return guard([&] { cubic_weights(t, w, dw); });
}

int orc_grid_cover(const double* X, long long n, int d, double target, int margin, int max_nodes,
                   int* dims, double* origin, double* spacing) {
  return guard([&] {
    Grid g = grid_cover(X, n, d, target, margin, max_nodes);
    for (int j = 0; j < d; ++j) {
      dims[j] = g.dims[j];
      origin[j] = g.origin[j];
      spacing[j] = g.spacing[j];
    }
  });
}

int orc_kernel_eval(int family, double ell, double s, double a, double b, int even, const double* x,
                    const double* xp, int d, double* val, double* grad, double* hess, double* dlog) {
  return guard([&] {
    KernelSpec k = mk_kernel(family, ell, s, a, b, even);
    *val = k_eval(k, x, xp, d);
    k_eval_grad(k, x, xp, d, grad);
    k_eval_hess(k, x, xp, d, hess);
    *dlog = k_eval_dlogell(k, x, xp, d);
  });
}

int orc_assemble_dense(int family, double ell, double s, double a, double b, int even,
                       const double* X, long long n, const double* Xp, long long np, int d,
                       int with_der, long long size_cap, double* out) {
  return guard([&] {
    Mat K = assemble_dense(mk_kernel(family, ell, s, a, b, even), X, n, Xp, np, d, with_der != 0,
                           size_cap);
    copy_out(K.a, out);
  });
}

// Dense (rows n, cols m) interpolation matrices [W; dW_1; ...] in type-major
// row blocks, col-major; out has n*(d+1) rows × m cols.
int orc_interp_dense(const int* dims, const double* origin, const double* spacing, int d,
                     const double* X, long long n, int order, double* out) {
  return guard([&] {
    Grid g = mk_grid(dims, origin, spacing, d);
    SparseInterpolation si = build_interpolation(g, X, n, order);
    const long long R = n * (d + 1);
    for (int grp = 0; grp <= d; ++grp) {
      const Csr& A = grp == 0 ? si.W : si.dW[grp - 1];
      for (long long i = 0; i < n; ++i)
        for (long long e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
          out[A.idx[e] * R + grp * n + i] = A.val[e];
    }
  });
}

int orc_point_stencil(const int* dims, const double* origin, const double* spacing, int d,
                      const double* x, int order, long long* idx, double* val, double* der) {
  return guard([&] {
    PointStencil st = point_stencil(mk_grid(dims, origin, spacing, d), x, order);
    for (size_t c = 0; c < st.indices.size(); ++c) {
      idx[c] = st.indices[c];
      val[c] = st.value[c];
    }
    copy_out(st.derivative.a, der);
  });
}

// ---------------------------------------------------------------- operators
void* orc_dense_create(const double* A, long long N) {
  Mat M(N, N);
  std::memcpy(M.a.data(), A, sizeof(double) * N * N);
  return static_cast<LinearOperator*>(new DenseOperator(std::move(M)));
}

void* orc_dski_create(int family, double ell, double s, double a, double b, int even,
                      const int* dims, const double* origin, const double* spacing, int d,
                      const double* X, long long n, double nv, double ng, int order,
                      int with_grad) {
  LinearOperator* out = nullptr;
  int st = guard([&] {
    out = new DskiOperator(mk_kernel(family, ell, s, a, b, even), mk_grid(dims, origin, spacing, d),
                           X, n, d, NoiseLevels{nv, ng}, order, with_grad != 0);
  });
  return st == OK ? out : nullptr;
}

void* orc_dskip_create(int family, double ell, double s, const double* X, long long n, int d,
                       double nv, double ng, long long rank, double grid_ratio, int max_nodes,
                       unsigned long long seed, int track, int with_grad, int policy_error) {
  LinearOperator* out = nullptr;
  int st = guard([&] {
    DskipConfig c;
    c.rank = rank;
    c.grid_ratio = grid_ratio;
    c.max_grid_nodes = max_nodes;
    c.seed = seed;
    c.track_dlogell = track != 0;
    c.with_gradients = with_grad != 0;
    c.rank_policy_error = policy_error != 0;
    out = new DskipOperator(mk_kernel(family, ell, s, 0, 0, 0), X, n, d, NoiseLevels{nv, ng}, c);
  });
  return st == OK ? out : nullptr;
}

void* orc_dskip_from_factors(long long n, int groups, double nv, double ng, int nf, const long long* ranks,
                             const double* const* Q, const double* const* alpha, const double* const* beta) {
  LinearOperator* out = nullptr;
  int st = guard([&] {
    const Index N = n * (groups + 1);
    std::vector<LanczosFactor> fs;
    for (int f = 0; f < nf; ++f) {
      LanczosFactor F;
      const Index r = ranks[f];
      F.Q = Mat(N, r);
      std::copy(Q[f], Q[f] + N * r, F.Q.a.begin());
      F.alpha.assign(alpha[f], alpha[f] + r);
      F.beta.assign(beta[f], beta[f] + std::max<Index>(r - 1, 0));
      fs.push_back(std::move(F));
    }
    out = new DskipOperator(n, groups, NoiseLevels{nv, ng}, std::move(fs));
  });
  return st == OK ? out : nullptr;
}

// Factor data of a D-SKIP operator: number of factors, their ranks, and Q/alpha/beta.
int orc_dskip_factor_count(void* h) {
  auto* op = dynamic_cast<DskipOperator*>(static_cast<LinearOperator*>(h));
  return op ? int(op->factors().size()) : -1;
}
long long orc_dskip_factor_rank(void* h, int f) {
  auto* op = dynamic_cast<DskipOperator*>(static_cast<LinearOperator*>(h));
  return op->factors()[size_t(f)].rank();
}
void orc_dskip_factor_get(void* h, int f, double* Q, double* alpha, double* beta) {
  auto* op = dynamic_cast<DskipOperator*>(static_cast<LinearOperator*>(h));
  const LanczosFactor& F = op->factors()[size_t(f)];
  copy_out(F.Q.a, Q);
  copy_out(F.alpha, alpha);
  copy_out(F.beta, beta);
}
int orc_dskip_dlogell_apply(void* h, const double* v, double* out) {
  return guard([&] {
    auto* op = dynamic_cast<DskipOperator*>(static_cast<LinearOperator*>(h));
    copy_out(op->dlogell_apply(v), out);
  });
}

// OneDimFactor via build_factor (dskip.cpp:115-130).
void* orc_factor_create(int family, double ell, double s, const double* X, long long n, int d,
                        int direction, double grid_ratio, int max_nodes, int dlogell) {
  LinearOperator* out = nullptr;
  guard([&] {
    out = new OneDimFactor(build_factor(mk_kernel(family, ell, s, 0, 0, 0), X, n, d, direction,
                                        grid_ratio, max_nodes, dlogell != 0));
  });
  return out;
}

void orc_op_free(void* h) { delete static_cast<LinearOperator*>(h); }
long long orc_op_size(void* h) { return static_cast<LinearOperator*>(h)->size(); }
int orc_op_mvm(void* h, const double* x, double* y) {
  return guard([&] { static_cast<LinearOperator*>(h)->mvm(x, y); });
}
// Batched: nrhs columns, col-major with leading dimension N. Columns in
// parallel (OpenMP) — the reference runs independent MVMs from parallel
// probe loops (linalg.cpp:222,264).
int orc_op_mvm_batch(void* h, const double* X, double* Y, int nrhs) {
  return guard([&] {
    auto* op = static_cast<LinearOperator*>(h);
    const long long N = op->size();
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < nrhs; ++b) op->mvm(X + b * N, Y + b * N);
  });
}
int orc_op_diagonal(void* h, double* out) {
  return guard([&] { copy_out(static_cast<LinearOperator*>(h)->diagonal(), out); });
}
int orc_op_row(void* h, long long r, double* out) {
  return guard([&] { copy_out(static_cast<LinearOperator*>(h)->row(r), out); });
}
int orc_dski_transpose_apply(void* h, const double* v, double* u) {
  return guard([&] { copy_out(dynamic_cast<DskiOperator&>(*static_cast<LinearOperator*>(h)).stacked_transpose_apply(v), u); });
}
int orc_dski_apply(void* h, const double* u, double* out) {
  return guard([&] { copy_out(dynamic_cast<DskiOperator&>(*static_cast<LinearOperator*>(h)).stacked_apply(u), out); });
}
int orc_dski_grid_mvm(void* h, const double* u, double* w) {
  return guard([&] { dynamic_cast<DskiOperator&>(*static_cast<LinearOperator*>(h)).grid_operator().mvm(u, w); });
}
double orc_dski_min_embedding_eigenvalue(void* h) {
  return dynamic_cast<DskiOperator&>(*static_cast<LinearOperator*>(h)).grid_operator().min_embedding_eigenvalue();
}
long long orc_dski_grid_size(void* h) {
  return dynamic_cast<DskiOperator&>(*static_cast<LinearOperator*>(h)).grid().size();
}

// Standalone grid kernel operator (GridKernelOperator).
void* orc_kuu_create(int family, double ell, double s, double a, double b, int even, int dlogell,
                     const int* dims, const double* origin, const double* spacing, int d) {
  GridKernelOperator* out = nullptr;
  guard([&] {
    KernelSpec k = mk_kernel(family, ell, s, a, b, even);
    out = new GridKernelOperator(mk_grid(dims, origin, spacing, d),
                                 dlogell ? kernel_dlogell_profile(k) : kernel_profile(k));
  });
  return out;
}
void orc_kuu_free(void* h) { delete static_cast<GridKernelOperator*>(h); }
int orc_kuu_mvm(void* h, const double* v, double* out) {
  return guard([&] { static_cast<GridKernelOperator*>(h)->mvm(v, out); });
}
double orc_kuu_min_eig(void* h) { return static_cast<GridKernelOperator*>(h)->min_embedding_eigenvalue(); }

// ---------------------------------------------------------------- solvers
void* orc_precond_create(const double* F, long long n, long long k, const double* nd) {
  Precond* p = nullptr;
  int st = guard([&] {
    Mat M(n, k);
    if (n > 0 && k > 0) std::memcpy(M.a.data(), F, sizeof(double) * n * k);
    Vec d(nd, nd + n);
    p = new Precond{std::make_unique<Preconditioner>(M, d)};
  });
  return st == OK ? p : nullptr;
}
void orc_precond_free(void* p) { delete static_cast<Precond*>(p); }
void orc_precond_apply(void* p, const double* b, double* out) {
  auto* P = static_cast<Precond*>(p)->p.get();
  copy_out(P->apply(Vec(b, b + P->size())), out);
}
double orc_precond_quadratic(void* p, const double* b) {
  auto* P = static_cast<Precond*>(p)->p.get();
  return P->quadratic(Vec(b, b + P->size()));
}
void orc_precond_q1(void* p, double* out) { copy_out(static_cast<Precond*>(p)->p->q1().a, out); }

int orc_cg(void* op, const double* b, double tol, int maxit, void* precond, double* x, int* its,
           int* converged, double* hist, int* hist_len) {
  return guard([&] {
    auto* A = static_cast<LinearOperator*>(op);
    PrecondApply M;
    if (precond) M = static_cast<Precond*>(precond)->p->as_apply();
    CgResult r = cg(*A, b, CgOptions{tol, maxit}, M);
    copy_out(r.x, x);
    *its = r.iterations;
    *converged = r.converged ? 1 : 0;
    if (hist) copy_out(r.residual_history, hist);
    *hist_len = int(r.residual_history.size());
  });
}

// Pivoted Cholesky of op's rows (minus `nd` on the pivot entry when nd is
// non-null: the kernel-part convention of gp.cpp:128-136); diag given.
int orc_pivchol(void* op, const double* diag, const double* nd, long long max_rank, double trace_tol,
                double* L, long long* pivots, long long* rank, double* traces) {
  return guard([&] {
    auto* A = static_cast<LinearOperator*>(op);
    const long long N = A->size();
    Vec dg(diag, diag + N);
    auto row_fn = [&](Index i) {
      Vec r = A->row(i);
      if (nd) r[size_t(i)] -= nd[i];
      return r;
    };
    PivotedCholeskyFactor f = pivoted_cholesky(dg, row_fn, max_rank, trace_tol);
    copy_out(f.L.a, L);
    for (size_t j = 0; j < f.pivots.size(); ++j) pivots[j] = f.pivots[j];
    *rank = f.L.cols;
    traces[0] = f.initial_trace;
    traces[1] = f.residual_trace;
  });
}

int orc_slq(void* op, int probes, int steps, unsigned long long seed, double floor_, double* logdet,
            int* clamped, double* estimates) {
  return guard([&] {
    SlqOptions o;
    o.probes = probes;
    o.lanczos_steps = steps;
    o.seed = seed;
    o.eigen_floor = floor_;
    SlqResult r = slq_logdet(*static_cast<LinearOperator*>(op), o);
    *logdet = r.logdet;
    *clamped = r.clamped;
    if (estimates && !r.estimates.empty()) copy_out(r.estimates, estimates);
  });
}

int orc_trace_estimate(void* A, void* B, int probes, unsigned long long seed, double tol, int maxit,
                       void* precond, double* out) {
  return guard([&] {
    PrecondApply M;
    if (precond) M = static_cast<Precond*>(precond)->p->as_apply();
    *out = trace_estimate(*static_cast<LinearOperator*>(A), *static_cast<LinearOperator*>(B), probes,
                          seed, CgOptions{tol, maxit}, M);
  });
}

// Lanczos from an explicit unit start (slq/probe parity) or seeded (lowrank).
int orc_lanczos(void* op, long long steps, unsigned long long seed, const double* start,
                unsigned long long restart_seed, double* Q, double* alpha, double* beta,
                long long* k, int* breakdown) {
  return guard([&] {
    auto* A = static_cast<LinearOperator*>(op);
    LanczosFactor f = start ? lanczos_from_start(*A, Vec(start, start + A->size()), steps, restart_seed)
                            : lanczos_lowrank(*A, steps, seed);
    copy_out(f.Q.a, Q);
    copy_out(f.alpha, alpha);
    copy_out(f.beta, beta);
    *k = f.rank();
    *breakdown = f.breakdown ? 1 : 0;
  });
}

int orc_tridiag_eig(const double* alpha, const double* beta, long long n, double* evals,
                    double* evecs) {
  return guard([&] {
    Vec ev;
    Mat Z;
    tridiag_eig(Vec(alpha, alpha + n), Vec(beta, beta + (n > 0 ? n - 1 : 0)), ev, &Z);
    copy_out(ev, evals);
    if (evecs) copy_out(Z.a, evecs);
  });
}

// ---------------------------------------------------------------- GP glue
void* orc_gp_create(int family, double ell, double s, const double* X, const double* y,
                    const double* dY, long long n, int d, double nv, double ng, int backend,
                    double grid_ratio, int max_nodes, long long dskip_rank, double dskip_ratio,
                    int dskip_max_nodes, double tol, int maxit, int use_precond,
                    long long precond_rank, int probes, int steps, unsigned long long seed) {
  GpModel* m = nullptr;
  guard([&] {
    GpConfig c;
    c.backend = backend;
    c.grid_ratio = grid_ratio;
    c.max_grid_nodes = max_nodes;
    c.dskip_rank = dskip_rank;
    c.dskip_grid_ratio = dskip_ratio;
    c.dskip_max_grid_nodes = dskip_max_nodes;
    c.cg = CgOptions{tol, maxit};
    c.use_preconditioner = use_precond != 0;
    c.precond_rank = precond_rank;
    c.slq_probes = probes;
    c.slq_steps = steps;
    c.seed = seed;
    m = new GpModel(mk_kernel(family, ell, s, 0, 0, 0), X, y, dY, n, d, nv, ng, c);
  });
  return m;
}
void orc_gp_free(void* m) { delete static_cast<GpModel*>(m); }
int orc_gp_lml(void* m, double* lml, double* logdet, double* fit, int* its) {
  return guard([&] {
    auto* g = static_cast<GpModel*>(m);
    *lml = g->log_marginal_likelihood();
    *logdet = g->logdet();
    Vec t = g->stacked_targets();
    const Vec& a = g->alpha();
    double s = 0.0;
    for (size_t i = 0; i < t.size(); ++i) s += t[i] * a[i];
    *fit = s;
    *its = g->last_solve.iterations;
  });
}
int orc_gp_alpha(void* m, double* out, int* its) {
  return guard([&] {
    auto* g = static_cast<GpModel*>(m);
    copy_out(g->alpha(), out);
    *its = g->last_solve.iterations;
  });
}
int orc_gp_pivots(void* m, long long* piv, long long* k) {
  return guard([&] {
    auto* f = static_cast<GpModel*>(m)->pivchol();
    for (size_t j = 0; j < f->pivots.size(); ++j) piv[j] = f->pivots[j];
    *k = (long long)f->pivots.size();
  });
}
int orc_gp_predict_mean_grad(void* m, const double* Xt, long long T, double* values, double* grads) {
  return guard([&] {
    auto r = static_cast<GpModel*>(m)->predict_mean_grad(Xt, T);
    copy_out(r.first, values);
    copy_out(r.second.a, grads);
  });
}
int orc_gp_lml_gradient(void* m, int probes, double* grad, int* nparams) {
  return guard([&] {
    auto* g = static_cast<GpModel*>(m);
    g->set_gradient_probes(probes);
    Vec r = g->lml_gradient();
    copy_out(r, grad);
    *nparams = int(r.size());
  });
}
// GpModel::fit (gp.cpp:294-404): out = (ℓ, s, σ₁, σ₂, best LML); per
// restart r: reports[3r..3r+2] = (succeeded, iterations, LML).
int orc_gp_fit(void* m, int max_iterations, int restarts, double initial_step, double min_step,
               int optimize_noise, unsigned long long seed, double* out, double* reports) {
  return guard([&] {
    auto r = static_cast<GpModel*>(m)->fit(max_iterations, restarts, initial_step, min_step,
                                           optimize_noise != 0, seed);
    out[0] = r.ell;
    out[1] = r.s;
    out[2] = r.nv;
    out[3] = r.ng;
    out[4] = r.log_marginal;
    for (size_t i = 0; i < r.restarts.size(); ++i) {
      reports[3 * i] = r.restarts[i].succeeded ? 1.0 : 0.0;
      reports[3 * i + 1] = r.restarts[i].iterations;
      reports[3 * i + 2] = r.restarts[i].log_marginal;
    }
  });
}
int orc_gp_set_hyperparameters(void* m, double ell, double s, double nv, double ng) {
  return guard([&] { static_cast<GpModel*>(m)->set_hyperparameters(ell, s, nv, ng); });
}
int orc_gp_dlogell_apply(void* m, const double* v, double* out) {
  return guard([&] { copy_out(static_cast<GpModel*>(m)->dlogell_apply(v), out); });
}
int orc_gp_cross_covariance(void* m, const double* x, double* out) {
  return guard([&] { copy_out(static_cast<GpModel*>(m)->cross_covariance(x), out); });
}
int orc_gp_cross_covariance_jacobian(void* m, const double* x, double* out) {
  return guard([&] { copy_out(static_cast<GpModel*>(m)->cross_covariance_jacobian(x).a, out); });
}
int orc_gp_predict_variance_exact(void* m, const double* x, double* out) {
  return guard([&] { *out = static_cast<GpModel*>(m)->predict_variance_exact(x); });
}
int orc_gp_predict_variance_randomized(void* m, const double* Xt, long long T, int probes, unsigned long long seed,
                                       double* out) {
  return guard([&] { copy_out(static_cast<GpModel*>(m)->predict_variance_randomized(Xt, T, probes, seed), out); });
}
int orc_gp_predict_variance_pivchol(void* m, const double* x, double* out) {
  return guard([&] { *out = static_cast<GpModel*>(m)->predict_variance_pivchol(x); });
}

}  // extern "C"
