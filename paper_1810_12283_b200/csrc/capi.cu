#include <thread>
#include <unistd.h>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
// capi.cu — extern "C" boundary (include/gk_capi.h). Maps C++ exceptions to
// gk_status codes, stages host blocks through the device, converts between
// the reference's external layout and the operators' internal layout.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "gk_kernels.cuh"
#include "solvers.hpp"

extern "C" gk_status gk_sample_test_function_impl(const char* name, int64_t n, std::uint64_t seed, double nv,
                                                  double ng, int with_gradients, int* d, double* X, double* y,
                                                  double* dY);
extern "C" gk_status gk_make_dataset_impl(int config, std::uint64_t seed, int64_t* n, int* d, double* X,
                                          double* y, double* dY);

namespace gk {
std::unique_ptr<Op> make_dski(const gk_kernel& k, const gk_grid& g, const double* X, i64 n, double nv, double ng,
                              int order, int with_grad, int device);
std::unique_ptr<Op> make_exact(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                               int with_grad, int device);
std::unique_ptr<Op> make_dense(const double* A, i64 N, int device);
std::unique_ptr<Op> make_dense_kernel(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                                      int with_grad, i64 size_cap, int device);
void assemble_dense_dev(const gk_kernel& k, const double* dX, i64 n, const double* dXp, i64 np, int d, bool deriv,
                        bool dl, double c, double* out, i64 ld, cudaStream_t s);
void dense_chol_solve(Op& o, const double* dB, double* dX, int nrhs, cudaStream_t s);
double dense_chol_logdet(Op& o);
void dense_exact_lml_gradient(Op& o, const double* alpha_h, double* grad, int* nparams);
std::unique_ptr<Op> make_dskip_from_factors(i64 n, int groups, double nv, double ng, int nf, const i64* ranks,
                                            const double* const* Q, const double* const* alpha,
                                            const double* const* beta, int device);
std::unique_ptr<Op> make_dskip(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                               const gk_dskip_config& cfg, int device);
int64_t dski_grid_size(const Op& o);
int dski_fused_phases(Op& o, int nrhs, i64* out, int max_ctas);
bool dski_fused_split(Op& o, int phase, const double* v, double* u2, double* out, int nrhs, cudaStream_t s);
void dski_cross_cov_dev(Op& o, const double* dXt, i64 nT, int dir, double* dQ, i64 ldq, cudaStream_t s);
void dski_gather_noise(Op& o, const double* W, const double* V, double* out, int nrhs, cudaStream_t s);
gk_grid dski_grid(const Op& o);
double dski_min_embedding_eigenvalue(const Op& o);
std::unique_ptr<Op> make_grid_kernel(int d, const int* dims, const double* slice_ref, int device);
double grid_kernel_min_eig(const Op& o);
std::unique_ptr<Op> make_dski_slices(const gk_grid& g, const double* X, i64 n, double nv, double ng, int order,
                                     int with_grad, int device, const double* slice_ref, const double* offset_table);
void dski_transpose_apply(Op& o, const double* Vi, double* U, int nrhs, cudaStream_t s);
void dski_apply(Op& o, const double* U, double* Oi, int nrhs, cudaStream_t s);
void dski_grid_mvm(Op& o, const double* U, double* W, int nrhs, cudaStream_t s);
void dski_predict(Op& o, const double* alpha_i, double mean, const double* dXt, i64 nT, double* dvals,
                  double* dgrads, int* dbad, cudaStream_t s);
void dski_cross_cov(Op& o, const double* dXt, i64 nT, double* Qi, int* dbad, cudaStream_t s, int dir = -1);
void precond_quadratic(Precond& M, const double* r, int nrhs, double* out_h, cudaStream_t s);
void pivchol_copy_L(const PivChol& f, double* out_host);
int dskip_factor_count(const Op& o);
i64 dskip_factor_rank(const Op& o, int f);
void dskip_factor_get(const Op& o, int f, double* Q, double* a, double* b);
void dskip_dlogell(Op& o, const double* in, double* out, int nrhs, cudaStream_t s);
void dski_dlogell(Op& o, const double* Vi, double* Oi, int nrhs, cudaStream_t s);
double dmma_peak_tflops(int device);
}  // namespace gk

using namespace gk;

namespace {
// Run f(0..n-1) on up to hardware_concurrency host threads (independent items).
template <class F>
void parallel_for(int n, F&& f) {
  const int nt = std::max(1, std::min<int>(n, int(std::thread::hardware_concurrency())));
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (int i = next++; i < n; i = next++) f(i);
    });
  for (auto& th : pool) th.join();
}
}  // namespace

struct gk_precond {
  std::unique_ptr<Precond> impl;
  // cached copies reordered for an operator's internal row order (keyed by
  // Op::uid); the lookup/insert is guarded by reorder_mu (one external-order
  // preconditioner may be bound to several operators from several threads)
  std::mutex reorder_mu;
  std::vector<std::pair<std::uint64_t, std::unique_ptr<Precond>>> reordered;
};
struct gk_pivchol {
  std::unique_ptr<PivChol> impl;
};

namespace {

thread_local std::string g_err;
thread_local i64 g_err_point = -1;

template <class F>
gk_status guard(F&& f) {
  try {
    f();
    return GK_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_point = e.point;
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return GK_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GK_ERR_RUNTIME;
  }
}

Op& O(const gk_op* op) {
  if (!op || !op->impl) fail(GK_ERR_ARG, "null operator handle");
  return *op->impl;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// One C-ABI call's exclusive use of an operator: holds op.mu, orders the
// call's device work after the previous call's (whatever stream that used)
// through op.last_use, and records op.last_use on this call's stream at exit.
// Construct after the DeviceGuard (the event belongs to op.device).
struct OpSession {
  Op& op;
  cudaStream_t s;
  std::unique_lock<std::mutex> lk;
  OpSession(Op& o, cudaStream_t st) : op(o), s(st), lk(o.mu) {
    if (!op.last_use) GK_CUDA(cudaEventCreateWithFlags(&op.last_use, cudaEventDisableTiming));
    else GK_CUDA(cudaStreamWaitEvent(s, op.last_use, 0));
  }
  ~OpSession() { cudaEventRecord(op.last_use, s); }
  OpSession(const OpSession&) = delete;
  OpSession& operator=(const OpSession&) = delete;
};

// Host block (N×nrhs col-major, ld) -> device internal layout.
void upload_internal(Op& op, const double* V, i64 ldv, double* d_ext, double* d_int, int nrhs, cudaStream_t s) {
  GK_CUDA(cudaMemcpy2DAsync(d_ext, sizeof(double) * op.N, V, sizeof(double) * ldv, sizeof(double) * op.N, nrhs,
                            cudaMemcpyHostToDevice, s));
  op.to_internal(d_ext, op.N, d_int, nrhs, s);
}
void download_internal(Op& op, const double* d_int, double* d_ext, double* Out, i64 ldo, int nrhs,
                       cudaStream_t s) {
  op.from_internal(d_int, d_ext, op.N, nrhs, s);
  GK_CUDA(cudaMemcpy2DAsync(Out, sizeof(double) * ldo, d_ext, sizeof(double) * op.N, sizeof(double) * op.N, nrhs,
                            cudaMemcpyDeviceToHost, s));
}

// Precond in the row order of `op`.
Precond& precond_for(const gk_precond* M, const Op& op) {
  auto* mm = const_cast<gk_precond*>(M);
  Precond& base = *mm->impl;
  if (base.N != op.N) fail(GK_ERR_ARG, "preconditioner and operator sizes differ");
  const i64* ext = op.d_ext_of_int();
  if (base.order_uid == op.uid) return base;
  if (base.order_uid == 0 && ext == nullptr) return base;  // both in external order
  if (base.order_uid != 0)
    fail(GK_ERR_UNSUPPORTED, "preconditioner was built for another operator's row order");
  std::lock_guard<std::mutex> rlk(mm->reorder_mu);
  for (auto& pr : mm->reordered)
    if (pr.first == op.uid) return *pr.second;
  // external-ordered preconditioner -> reorder rows for op: new[r] = old[ext[r]]
  auto P = std::make_unique<Precond>();
  P->device = base.device;
  P->N = base.N;
  P->k = base.k;
  P->order_uid = op.uid;
  P->ext_own.alloc(static_cast<size_t>(base.N));
  GK_CUDA(cudaMemcpy(P->ext_own.p, ext, sizeof(i64) * base.N, cudaMemcpyDeviceToDevice));
  P->ext = P->ext_own.p;
  GK_CUDA(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
  P->q1.alloc(static_cast<size_t>(base.N * base.k));
  P->dinv.alloc(static_cast<size_t>(base.N));
  cudaStream_t s = op.stream;
  // q1 is [N][k] row-major == an external "k-column" block transposed; use the
  // generic row map on a k-wide RHS-minor block.
  DevBuf<double> tmp(static_cast<size_t>(base.N * base.k));
  // internal (row-major [N][k]) -> external col-major with identity, then gather by ext
  from_internal(nullptr, base.N, base.q1.p, tmp.p, base.N, int(base.k), s);
  to_internal(ext, base.N, tmp.p, base.N, P->q1.p, int(base.k), s);
  DevBuf<double> tmp1(static_cast<size_t>(base.N));
  from_internal(nullptr, base.N, base.dinv.p, tmp1.p, base.N, 1, s);
  to_internal(ext, base.N, tmp1.p, base.N, P->dinv.p, 1, s);
  GK_CUDA(cudaStreamSynchronize(s));
  mm->reordered.emplace_back(op.uid, std::move(P));
  return *mm->reordered.back().second;
}

}  // namespace

extern "C" {

const char* gk_last_error(void) { return g_err.c_str(); }
int64_t gk_last_error_point(void) { return g_err_point; }
const char* gk_version(void) { return "gk_b200 0.1 (sm_100a)"; }
int64_t gk_kernel_launch_count(void) { return g_launches.load(); }

int gk_set_tuning(const char* key, int value) {
  const std::string k = key ? key : "";
  std::atomic<int>* slot = k == "scatter" ? &g_tuning.scatter
                           : k == "gather" ? &g_tuning.gather
                           : k == "toeplitz" ? &g_tuning.toeplitz
                           : k == "precond" ? &g_tuning.precond
                           : k == "fused" ? &g_tuning.fused
                           : k == "lean" ? &g_tuning.lean
                           : k == "pivchol" ? &g_tuning.pivchol
                           : k == "devbuild" ? &g_tuning.devbuild
                           : k == "fused_prof" ? &g_tuning.fused_prof
                           : k == "pcg_fused" ? &g_tuning.pcg_fused
                           : k == "e2e_chunk" ? &g_tuning.e2e_chunk
                           : k == "e2e_stage" ? &g_tuning.e2e_stage
                           : k == "d3" ? &g_tuning.d3
                           : k == "dskip" ? &g_tuning.dskip
                           : k == "lanczos" ? &g_tuning.lanczos
                           : k == "rng" ? &g_tuning.rng
                           : k == "dskip_e" ? &g_tuning.dskip_e
                           : k == "f2_stc" ? &g_tuning.f2_stc
                           : k == "f2_sl" ? &g_tuning.f2_sl
                           : k == "f2_gtc" ? &g_tuning.f2_gtc
                           : k == "f2_gl" ? &g_tuning.f2_gl
                           : k == "f2_tsplit" ? &g_tuning.f2_tsplit
                           : k == "f2_per_sm" ? &g_tuning.f2_per_sm
                           : k == "f2_skip" ? &g_tuning.f2_skip
                           : k == "f2_warm" ? &g_tuning.f2_warm
                           : k == "f2_twide" ? &g_tuning.f2_twide
                           : k == "f2_grid" ? &g_tuning.f2_grid
                           : k == "f2_rp" ? &g_tuning.f2_rp
                           : k == "f2_smode" ? &g_tuning.f2_smode
                           : k == "f2_gmode" ? &g_tuning.f2_gmode
                           : k == "f2_nspl" ? &g_tuning.f2_nspl
                           : k == "f2_nst" ? &g_tuning.f2_nst
                                             : nullptr;
  if (!slot) return -1;
  g_tuning.gen.fetch_add(1);
  return slot->exchange(value);
}

gk_status gk_grid_cover(const double* X, int64_t n, int d, double target, int margin, int max_nodes,
                        gk_grid* out) {
  return guard([&] {  // interpolation.cpp:117-146
    if (n <= 0) fail(GK_ERR_ARG, "cannot build a grid over no points");
    if (!(target > 0.0)) fail(GK_ERR_ARG, "grid spacing must be positive");
    if (d < 1 || d > 8) fail(GK_ERR_ARG, "grid dimension must be in [1, 8]");
    margin = std::max(margin, 3);
    out->d = d;
    for (int j = 0; j < d; ++j) {
      double lo = X[j * n], hi = X[j * n];
      for (i64 i = 0; i < n; ++i) {
        lo = std::min(lo, X[j * n + i]);
        hi = std::max(hi, X[j * n + i]);
      }
      const double span = std::max(hi - lo, 1e-12);
      double h = target;
      const int interior = static_cast<int>(std::ceil(span / h)) + 1;
      int m = interior + 2 * margin;
      if (m > max_nodes) {
        m = max_nodes;
        h = span / static_cast<double>(m - 1 - 2 * margin);
      }
      if (m < 6 + 2 * margin) m = 6 + 2 * margin;
      out->dims[j] = m;
      out->spacing[j] = h;
      out->origin[j] = lo - margin * h;
    }
  });
}

uint64_t gk_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }
void gk_rademacher_vector(int64_t n, uint64_t seed, uint64_t stream, double* out) { rademacher(n, seed, stream, out); }
void gk_gaussian_vector(int64_t n, uint64_t seed, uint64_t stream, double* out) { gaussian(n, seed, stream, out); }
void gk_uniform_vector(int64_t n, uint64_t seed, uint64_t stream, double a, double b, double* out) {
  uniform(n, seed, stream, a, b, out);
}

gk_status gk_dski_create(const gk_kernel* kernel, const gk_grid* grid, const double* X, int64_t n, double nv,
                         double ng, int order, int with_gradients, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_dski(*kernel, *grid, X, n, nv, ng, order, with_gradients, device);
    *out = h.release();
  });
}

gk_status gk_dskip_create(const gk_kernel* kernel, const double* X, int64_t n, int d, double nv, double ng,
                          const gk_dskip_config* cfg, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_dskip(*kernel, X, n, d, nv, ng, *cfg, device);
    *out = h.release();
  });
}

gk_status gk_dskip_create_from_factors(int64_t n, int groups, double nv, double ng, int nf, const int64_t* ranks,
                                       const double* const* Q, const double* const* alpha,
                                       const double* const* beta, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_dskip_from_factors(n, groups, nv, ng, nf, ranks, Q, alpha, beta, device);
    *out = h.release();
  });
}

gk_status gk_dense_create(const double* A, int64_t N, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_dense(A, N, device);
    *out = h.release();
  });
}

gk_status gk_assemble_dense(const gk_kernel* kernel, const double* X, int64_t n, const double* Xp, int64_t np, int d,
                            int with_derivatives, int dlogell, double derivative_scale, int64_t size_cap, int device,
                            double* out) {
  return guard([&] {
    if (!kernel || !X || !Xp || !out) fail(GK_ERR_ARG, "null argument");
    if (kernel->family != 0 && kernel->family != 1) fail(GK_ERR_ARG, "unknown kernel family");
    if (n < 0 || np < 0 || d < 1) fail(GK_ERR_ARG, "point sets have mismatched dimensions");
    const i64 rows = with_derivatives ? n * (d + 1) : n, cols = with_derivatives ? np * (d + 1) : np;
    if (rows * cols > size_cap)
      fail(GK_ERR_LENGTH, "dense assembly of " + std::to_string(rows) + " x " + std::to_string(cols) +
                              " exceeds the configured size cap");
    if (rows * cols == 0) return;
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    GK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf<double> dX(static_cast<size_t>(n) * d), dXp(static_cast<size_t>(np) * d), K(static_cast<size_t>(rows) * cols);
    dX.upload(X, static_cast<size_t>(n) * d, s);
    dXp.upload(Xp, static_cast<size_t>(np) * d, s);
    assemble_dense_dev(*kernel, dX.p, n, dXp.p, np, d, with_derivatives != 0, dlogell != 0, derivative_scale, K.p, rows, s);
    GK_CUDA(cudaMemcpyAsync(out, K.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
  });
}

gk_status gk_dense_kernel_create(const gk_kernel* kernel, const double* X, int64_t n, int d, double nv, double ng,
                                 int with_gradients, int64_t size_cap, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_dense_kernel(*kernel, X, n, d, nv, ng, with_gradients, size_cap, device);
    *out = h.release();
  });
}

gk_status gk_dense_cholesky_solve(const gk_op* h, const double* B, int64_t ldb, int64_t nrhs, double* X, int64_t ldx) {
  return guard([&] {
    Op& op = O(h);
    if (nrhs < 0 || ldb < op.N || ldx < op.N) fail(GK_ERR_ARG, "solve size mismatch");
    if (nrhs == 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    DevBuf<double> d(static_cast<size_t>(op.N) * nrhs);
    GK_CUDA(cudaMemcpy2DAsync(d.p, sizeof(double) * op.N, B, sizeof(double) * ldb, sizeof(double) * op.N, nrhs,
                              cudaMemcpyHostToDevice, s));
    dense_chol_solve(op, d.p, d.p, int(nrhs), s);
    GK_CUDA(cudaMemcpy2DAsync(X, sizeof(double) * ldx, d.p, sizeof(double) * op.N, sizeof(double) * op.N, nrhs,
                              cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_dense_cholesky_logdet(const gk_op* h, double* logdet) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, op.stream);
    *logdet = dense_chol_logdet(op);
  });
}

gk_status gk_dense_exact_lml_gradient(const gk_op* h, const double* alpha, double* grad, int* nparams) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, op.stream);
    dense_exact_lml_gradient(op, alpha, grad, nparams);
  });
}

gk_status gk_exact_create(const gk_kernel* kernel, const double* X, int64_t n, int d, double nv, double ng,
                          int with_gradients, int device, gk_op** out) {
  return guard([&] {
    auto h = std::make_unique<gk_op>();
    h->impl = make_exact(*kernel, X, n, d, nv, ng, with_gradients, device);
    *out = h.release();
  });
}

void gk_op_destroy(gk_op* op) {
  if (!op) return;
  if (op->impl) {
    DeviceGuard dg(op->impl->device);
    op->impl.reset();
  }
  delete op;
}
int64_t gk_op_size(const gk_op* op) { return op && op->impl ? op->impl->N : -1; }
int gk_op_kind(const gk_op* op) { return op && op->impl ? op->impl->kind : -1; }

// Parallel host copies for the pageable-buffer MVM: a small persistent pool
// (one copy per call is split over the workers and the calling thread). A
// single-threaded memcpy, or the driver's own staging of pageable copies
// (one bounce buffer), moves ~10 GB/s; the copy engines take ~50.
namespace {
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool p;
    return p;
  }
  // copy ncols columns of `rows` doubles, src/dst with their own leading dims
  void copy_cols(double* dst, size_t ldd, const double* src, size_t lds, size_t rows, size_t ncols) {
    const size_t total = rows * ncols;
    // a forked child inherits the pool object but not its threads: copy serially there
    const size_t nw = getpid() == pid_ ? workers_.size() : 0;
    const int parts = int(std::min<size_t>(nw + 1, std::max<size_t>(1, total / (64 * 1024))));
    auto piece = [=](int k) {  // elements [k·total/parts, (k+1)·total/parts) in column-major order
      size_t e = total * size_t(k) / size_t(parts);
      const size_t end = total * size_t(k + 1) / size_t(parts);
      while (e < end) {
        const size_t c = e / rows, r = e - c * rows, len = std::min(rows - r, end - e);
        std::memcpy(dst + c * ldd + r, src + c * lds + r, len * sizeof(double));
        e += len;
      }
    };
    if (parts == 1) {
      piece(0);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);  // one job at a time (operators on other threads)
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = piece;
      nparts_ = parts;
      next_ = 1;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    piece(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == nparts_ - 1; });
  }

 private:
  HostCopyPool() : pid_(getpid()) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const char* env = std::getenv("GK_COPY_THREADS");  // total copy threads incl. the caller (default 8)
    const unsigned want = env ? unsigned(std::max(1, std::atoi(env))) : 8u;
    const int n = int(std::min(want - 1, hw > 1 ? hw - 1 : 0u));
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
  }
  ~HostCopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void run() {
    std::uint64_t seen = 0;
    for (;;) {
      std::function<void(int)> job;
      int k = -1;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < nparts_); });
        if (stop_) return;
        k = next_++;
        job = job_;
        if (next_ >= nparts_) seen = gen_;
      }
      job(k);
      {
        std::lock_guard<std::mutex> lk(mu_);
        ++done_;
      }
      done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)> job_;
  int nparts_ = 0, next_ = 0, done_ = 0;
  std::uint64_t gen_ = 0;
  bool stop_ = false;
  pid_t pid_;
};

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
}  // namespace

gk_status gk_op_mvm(const gk_op* h, const double* V, int64_t ldv, double* Out, int64_t ldo, int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    if (nrhs < 0 || ldv < op.N || ldo < op.N) fail(GK_ERR_ARG, "MVM size mismatch");
    if (nrhs == 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    // Host buffers: column chunks pipelined over five streams, one per
    // resource stage — H2D (copy engine), to-internal permute, MVM,
    // from-internal permute, D2H (the other copy engine). Each stage of chunk
    // j waits only for the previous stage of chunk j, so the copy engines
    // never idle behind a permute and H2D/D2H run in opposite PCIe
    // directions at once. Columns are independent: the result equals the
    // one-shot MVM. Tuning "e2e_chunk": chunk width (0 = nrhs/4 for nrhs >= 16).
    const int pc = g_tuning.e2e_chunk.load();
    int chunk = pc > 0 ? pc : (nrhs >= 16 ? int((nrhs + 3) / 4) : int(nrhs));
    chunk = int(std::min<i64>(std::max(1, chunk), std::min<i64>(nrhs, kMaxRhs)));
    const int nchunks = int((nrhs + chunk - 1) / chunk);
    if (!op.io_in) {
      GK_CUDA(cudaStreamCreateWithFlags(&op.io_in, cudaStreamNonBlocking));
      GK_CUDA(cudaStreamCreateWithFlags(&op.io_out, cudaStreamNonBlocking));
      GK_CUDA(cudaStreamCreateWithFlags(&op.io_pin, cudaStreamNonBlocking));
      GK_CUDA(cudaStreamCreateWithFlags(&op.io_pout, cudaStreamNonBlocking));
    }
    while (int(op.io_events.size()) < 5 * nchunks + 1) {
      cudaEvent_t e;
      GK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      op.io_events.push_back(e);
    }
    const size_t tot = static_cast<size_t>(op.N) * nrhs;
    op.io_ext_in.reserve(tot);
    op.io_int_in.reserve(tot);
    op.io_int_out.reserve(tot);
    op.io_ext_out.reserve(tot);
    // Pageable host buffers (e.g. Eigen storage): chunks go through pinned
    // staging copied by the host pool — chunk j+1 is copied in while the
    // device works on chunk j, and chunk j's result is copied out as soon as
    // its D2H copy has landed — instead of the driver's serial bounce-buffer
    // staging of pageable copies (tuning "e2e_stage" = 1 turns it off).
    const bool stage_in = g_tuning.e2e_stage.load() == 0 && !is_pinned_host(V);
    const bool stage_out = g_tuning.e2e_stage.load() == 0 && !is_pinned_host(Out);
    if (stage_in) op.io_pin_in.reserve(tot);
    if (stage_out) op.io_pin_out.reserve(tot);
    const double* Vsrc = stage_in ? op.io_pin_in.p : V;
    const i64 ldvs = stage_in ? op.N : ldv;
    double* Odst = stage_out ? op.io_pin_out.p : Out;
    const i64 ldos = stage_out ? op.N : ldo;
    HostCopyPool& pool = HostCopyPool::get();
    auto copy_in = [&](int j) {
      const i64 c0 = i64(j) * chunk;
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      pool.copy_cols(op.io_pin_in.p + static_cast<size_t>(op.N) * c0, op.N, V + c0 * ldv, ldv, op.N, nb);
    };
    auto copy_out = [&](int j) {
      const i64 c0 = i64(j) * chunk;
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      GK_CUDA(cudaEventSynchronize(op.io_events[5 * j + 4]));  // chunk j's D2H copy landed
      pool.copy_cols(Out + c0 * ldo, ldo, op.io_pin_out.p + static_cast<size_t>(op.N) * c0, op.N, op.N, nb);
    };
    if (stage_in) copy_in(0);
    // the side streams must not start before earlier work on the compute stream
    cudaEvent_t e0 = op.io_events[5 * nchunks];
    GK_CUDA(cudaEventRecord(e0, s));
    for (cudaStream_t t : {op.io_in, op.io_out, op.io_pin, op.io_pout}) GK_CUDA(cudaStreamWaitEvent(t, e0, 0));
    for (int j = 0; j < nchunks; ++j) {
      const i64 c0 = i64(j) * chunk;
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      const size_t off = static_cast<size_t>(op.N) * c0;
      cudaEvent_t* ev = &op.io_events[5 * j];
      GK_CUDA(cudaMemcpy2DAsync(op.io_ext_in.p + off, sizeof(double) * op.N, Vsrc + c0 * ldvs, sizeof(double) * ldvs,
                                sizeof(double) * op.N, nb, cudaMemcpyHostToDevice, op.io_in));
      GK_CUDA(cudaEventRecord(ev[0], op.io_in));
      GK_CUDA(cudaStreamWaitEvent(op.io_pin, ev[0], 0));
      op.to_internal(op.io_ext_in.p + off, op.N, op.io_int_in.p + off, nb, op.io_pin);
      GK_CUDA(cudaEventRecord(ev[1], op.io_pin));
      GK_CUDA(cudaStreamWaitEvent(s, ev[1], 0));
      op.mvm(op.io_int_in.p + off, op.io_int_out.p + off, nb, s);
      GK_CUDA(cudaEventRecord(ev[2], s));
      GK_CUDA(cudaStreamWaitEvent(op.io_pout, ev[2], 0));
      op.from_internal(op.io_int_out.p + off, op.io_ext_out.p + off, op.N, nb, op.io_pout);
      GK_CUDA(cudaEventRecord(ev[3], op.io_pout));
      GK_CUDA(cudaStreamWaitEvent(op.io_out, ev[3], 0));
      GK_CUDA(cudaMemcpy2DAsync(Odst + c0 * ldos, sizeof(double) * ldos, op.io_ext_out.p + off, sizeof(double) * op.N,
                                sizeof(double) * op.N, nb, cudaMemcpyDeviceToHost, op.io_out));
      GK_CUDA(cudaEventRecord(ev[4], op.io_out));
      if (stage_in && j + 1 < nchunks) copy_in(j + 1);  // overlaps the device work on chunk j
      if (stage_out && j >= 1) copy_out(j - 1);
    }
    if (stage_out) copy_out(nchunks - 1);
    GK_CUDA(cudaStreamSynchronize(op.io_out));
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_op_mvm_dev(const gk_op* h, const double* dV, int64_t ldv, double* dOut, int64_t ldo, int64_t nrhs,
                        void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (nrhs < 0 || ldv < op.N || ldo < op.N) fail(GK_ERR_ARG, "MVM size mismatch");
    if (nrhs == 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = S(stream);
    OpSession ss(op, s);
    const int chunk = int(std::min<i64>(nrhs, kMaxRhs));
    op.scratch_a.reserve(static_cast<size_t>(op.N) * chunk);
    op.scratch_b.reserve(static_cast<size_t>(op.N) * chunk);
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      op.to_internal(dV + c0 * ldv, ldv, op.scratch_a.p, nb, s);
      op.mvm(op.scratch_a.p, op.scratch_b.p, nb, s);
      op.from_internal(op.scratch_b.p, dOut + c0 * ldo, ldo, nb, s);
    }
  });
}

gk_status gk_op_stage_dev(const gk_op* h, int stage, const double* dIn, double* dOut, int64_t nrhs, void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (nrhs < 1 || nrhs > 256) fail(GK_ERR_ARG, "stage: nrhs must be in [1, 256]");
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    op.stage(stage, dIn, dOut, int(nrhs), S(stream));
  });
}

gk_status gk_dski_gather_dev(const gk_op* h, const double* dW, const double* dV, double* dOut, int64_t nrhs,
                             void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (nrhs < 1 || nrhs > 256) fail(GK_ERR_ARG, "gather: nrhs must be in [1, 256]");
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    dski_gather_noise(op, dW, dV, dOut, int(nrhs), S(stream));
  });
}

gk_status gk_dski_fused_split_dev(const gk_op* h, int phase, const double* dV, double* dU2, double* dOut,
                                  int64_t nrhs, void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (phase < 0 || phase > 2) fail(GK_ERR_ARG, "phase must be 0 (scatter), 1 (K_UU + gather) or 2 (query)");
    if (nrhs < 1 || nrhs > kMaxRhs) fail(GK_ERR_ARG, "nrhs out of range");
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    if (!dski_fused_split(op, phase, dV, dU2, dOut, int(nrhs), S(stream)))
      fail(GK_ERR_UNSUPPORTED, "the split one-launch MVM needs a 2-D D-SKI operator with gradients");
  });
}

gk_status gk_dski_cross_covariance_dev(const gk_op* h, const double* dXt, int64_t T, int direction, double* dQ,
                                       int64_t ldq, void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (op.kind != KIND_DSKI) fail(GK_ERR_ARG, "operator is not a D-SKI operator");
    if (T < 1 || T > kMaxRhs) fail(GK_ERR_ARG, "test point count must be in [1, 64]");
    if (ldq < op.N) fail(GK_ERR_ARG, "size mismatch");
    const gk_grid g = dski_grid(op);
    if (direction < -1 || direction >= g.d) fail(GK_ERR_ARG, "direction out of range");
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    dski_cross_cov_dev(op, dXt, T, direction, dQ, ldq, S(stream));
  });
}

gk_status gk_op_to_internal_dev(const gk_op* h, const double* dV, int64_t ldv, double* dI, int64_t nrhs,
                                void* stream) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    op.to_internal(dV, ldv, dI, int(nrhs), S(stream));
  });
}

gk_status gk_op_from_internal_dev(const gk_op* h, const double* dI, double* dV, int64_t ldv, int64_t nrhs,
                                  void* stream) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, S(stream));
    op.from_internal(dI, dV, ldv, int(nrhs), S(stream));
  });
}

gk_status gk_op_diagonal(const gk_op* h, double* out) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    op.scratch_a.reserve(static_cast<size_t>(op.N));
    op.scratch_b.reserve(static_cast<size_t>(op.N));
    op.diagonal(op.scratch_a.p, s);
    op.from_internal(op.scratch_a.p, op.scratch_b.p, op.N, 1, s);
    GK_CUDA(cudaMemcpyAsync(out, op.scratch_b.p, sizeof(double) * op.N, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_op_row(const gk_op* h, int64_t r, double* out) {
  return guard([&] {
    Op& op = O(h);
    if (r < 0 || r >= op.N) fail(GK_ERR_RANGE, "row index out of range");
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    op.scratch_a.reserve(static_cast<size_t>(op.N));
    op.scratch_b.reserve(static_cast<size_t>(op.N));
    op.row(r, op.scratch_a.p, s);
    op.from_internal(op.scratch_a.p, op.scratch_b.p, op.N, 1, s);
    GK_CUDA(cudaMemcpyAsync(out, op.scratch_b.p, sizeof(double) * op.N, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_op_noise_diagonal(const gk_op* h, double* out) {
  return guard([&] {
    Op& op = O(h);
    for (i64 r = 0; r < op.N; ++r) out[r] = r < op.n_value ? op.nv2 : op.ng2;
  });
}

// ---------------------------------------------------------------- D-SKI pieces
int gk_debug_fused_phases(gk_op* h, int nrhs, int64_t* out, int max_ctas) {
  int n = 0;
  guard([&] {
    if (!out || max_ctas < 0) fail(GK_ERR_ARG, "null output");
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, op.stream);
    n = dski_fused_phases(op, nrhs, out, max_ctas);
  });
  return n;
}

gk_status gk_debug_rademacher_dev(int64_t n, uint64_t seed, uint64_t stream, double* out) {
  return guard([&] {
    if (n < 0 || !out) fail(GK_ERR_ARG, "bad arguments");
    DevBuf<double> d(static_cast<size_t>(std::max<int64_t>(n, 1)));
    const std::uint64_t sd = mix_seed(seed, stream);
    rademacher_dev(n, &sd, 1, 1.0, d.p, n, nullptr);
    GK_CUDA(cudaMemcpy(out, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  });
}

gk_status gk_debug_dmma_peak(int device, double* tflops) {
  return guard([&] {
    if (!tflops) fail(GK_ERR_ARG, "null output");
    *tflops = dmma_peak_tflops(device);
  });
}

int64_t gk_dski_grid_size(const gk_op* h) {
  int64_t m = -1;
  guard([&] { m = dski_grid_size(O(h)); });
  return m;
}

gk_status gk_dski_get_grid(const gk_op* h, gk_grid* out) {
  return guard([&] { *out = dski_grid(O(h)); });
}

gk_status gk_dski_min_embedding_eigenvalue(const gk_op* h, double* out) {
  return guard([&] {
    if (!out) fail(GK_ERR_ARG, "null output");
    const Op& op = O(h);
    *out = op.kind == KIND_GRID ? grid_kernel_min_eig(op) : dski_min_embedding_eigenvalue(op);
  });
}

gk_status gk_grid_kernel_create(const gk_grid* grid, const double* slice, int device, gk_op** out) {
  return guard([&] {
    if (!grid || !slice) fail(GK_ERR_ARG, "null argument");
    auto h = std::make_unique<gk_op>();
    h->impl = make_grid_kernel(grid->d, grid->dims, slice, device);
    *out = h.release();
  });
}

gk_status gk_dski_create_from_profile(const gk_grid* grid, const double* X, int64_t n, double nv, double ng,
                                      int order, int with_gradients, const double* slice,
                                      const double* offset_table, int device, gk_op** out) {
  return guard([&] {
    if (!grid) fail(GK_ERR_ARG, "null grid");
    auto h = std::make_unique<gk_op>();
    h->impl = make_dski_slices(*grid, X, n, nv, ng, order, with_gradients, device, slice, offset_table);
    *out = h.release();
  });
}

}  // extern "C"

namespace {
// Generic grid-block helper: host grid blocks (M×nrhs col-major) are
// RHS-minor on device via the identity row map.
template <class F>
void grid_call(Op& op, const double* In, i64 ldi, i64 rows_in, double* Out, i64 ldo, i64 rows_out, i64 nrhs,
               bool in_is_grid, bool out_is_grid, F&& f) {
  DeviceGuard dg(op.device);
  cudaStream_t s = op.stream;
  OpSession ss(op, s);
  const int chunk = int(std::min<i64>(nrhs, kMaxRhs));
  DevBuf<double> ein(static_cast<size_t>(rows_in) * chunk), iin(static_cast<size_t>(rows_in) * chunk), iout(static_cast<size_t>(rows_out) * chunk),
      eout(static_cast<size_t>(rows_out) * chunk);
  for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
    const int nb = int(std::min<i64>(chunk, nrhs - c0));
    GK_CUDA(cudaMemcpy2DAsync(ein.p, sizeof(double) * rows_in, In + c0 * ldi, sizeof(double) * ldi,
                              sizeof(double) * rows_in, nb, cudaMemcpyHostToDevice, s));
    if (in_is_grid) to_internal(nullptr, rows_in, ein.p, rows_in, iin.p, nb, s);
    else op.to_internal(ein.p, rows_in, iin.p, nb, s);
    f(iin.p, iout.p, nb, s);
    if (out_is_grid) from_internal(nullptr, rows_out, iout.p, eout.p, rows_out, nb, s);
    else op.from_internal(iout.p, eout.p, rows_out, nb, s);
    GK_CUDA(cudaMemcpy2DAsync(Out + c0 * ldo, sizeof(double) * ldo, eout.p, sizeof(double) * rows_out,
                              sizeof(double) * rows_out, nb, cudaMemcpyDeviceToHost, s));
  }
  GK_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

extern "C" {

gk_status gk_dski_transpose_apply(const gk_op* h, const double* V, int64_t ldv, double* U, int64_t ldu,
                                  int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    const i64 M = dski_grid_size(op);
    if (ldv < op.N || ldu < M) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    grid_call(op, V, ldv, op.N, U, ldu, M, nrhs, false, true,
              [&](const double* i, double* o, int nb, cudaStream_t s) { dski_transpose_apply(op, i, o, nb, s); });
  });
}

gk_status gk_dski_apply(const gk_op* h, const double* U, int64_t ldu, double* Out, int64_t ldo, int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    const i64 M = dski_grid_size(op);
    if (ldu < M || ldo < op.N) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    grid_call(op, U, ldu, M, Out, ldo, op.N, nrhs, true, false,
              [&](const double* i, double* o, int nb, cudaStream_t s) { dski_apply(op, i, o, nb, s); });
  });
}

gk_status gk_dski_grid_mvm(const gk_op* h, const double* U, int64_t ldu, double* W, int64_t ldw, int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    const i64 M = dski_grid_size(op);
    if (ldu < M || ldw < M) fail(GK_ERR_ARG, "grid kernel MVM size mismatch");
    if (nrhs <= 0) return;
    grid_call(op, U, ldu, M, W, ldw, M, nrhs, true, true,
              [&](const double* i, double* o, int nb, cudaStream_t s) { dski_grid_mvm(op, i, o, nb, s); });
  });
}

gk_status gk_dski_predict_mean_grad(const gk_op* h, const double* alpha, double mean, const double* Xtest,
                                    int64_t T, double* values, double* grads) {
  return guard([&] {
    Op& op = O(h);
    const gk_grid g = dski_grid(op);
    if (T <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    DevBuf<double> ae(static_cast<size_t>(op.N)), ai(static_cast<size_t>(op.N)), xt(static_cast<size_t>(T) * g.d), v(static_cast<size_t>(T)), gr(static_cast<size_t>(T) * g.d);
    DevBuf<int> bad(1);
    const int big = INT_MAX;
    GK_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    ae.upload(alpha, static_cast<size_t>(op.N), s);
    op.to_internal(ae.p, op.N, ai.p, 1, s);
    xt.upload(Xtest, static_cast<size_t>(T) * g.d, s);
    dski_predict(op, ai.p, mean, xt.p, T, v.p, gr.p, bad.p, s);
    int badh = INT_MAX;
    GK_CUDA(cudaMemcpy(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (badh != INT_MAX)
      fail(GK_ERR_OUT_OF_GRID, "test point " + std::to_string(badh) + " lies outside the interior of the grid", badh);
    GK_CUDA(cudaMemcpy(values, v.p, sizeof(double) * T, cudaMemcpyDeviceToHost));
    GK_CUDA(cudaMemcpy(grads, gr.p, sizeof(double) * T * g.d, cudaMemcpyDeviceToHost));
  });
}

// GpModel::cross_covariance_jacobian (gp.cpp:431-461, D-SKI branch) for T test
// points: column t·d + p of J = B K_UU w_p(x_t), w_p the ∂/∂x_p point stencil.
gk_status gk_dski_cross_covariance_jacobian(const gk_op* h, const double* Xtest, int64_t T, double* J, int64_t ldj) {
  return guard([&] {
    Op& op = O(h);
    const gk_grid g = dski_grid(op);
    if (ldj < op.N) fail(GK_ERR_ARG, "size mismatch");
    if (T <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    for (i64 t0 = 0; t0 < T; t0 += kMaxRhs) {
      const i64 nt = std::min<i64>(kMaxRhs, T - t0);
      std::vector<double> xh(static_cast<size_t>(nt) * g.d);
      for (int j = 0; j < g.d; ++j)
        for (i64 i = 0; i < nt; ++i) xh[static_cast<size_t>(j * nt + i)] = Xtest[j * T + t0 + i];
      DevBuf<double> xt(static_cast<size_t>(nt) * g.d), qi(static_cast<size_t>(op.N) * nt), qe(static_cast<size_t>(op.N) * nt);
      DevBuf<int> bad(1);
      xt.upload(xh.data(), xh.size(), s);
      for (int p = 0; p < g.d; ++p) {
        const int big = INT_MAX;
        GK_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
        dski_cross_cov(op, xt.p, nt, qi.p, bad.p, s, p);
        int badh = INT_MAX;
        GK_CUDA(cudaMemcpy(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (badh != INT_MAX)
          fail(GK_ERR_OUT_OF_GRID,
               "test point " + std::to_string(t0 + badh) + " lies outside the interior of the grid", t0 + badh);
        op.from_internal(qi.p, qe.p, op.N, int(nt), s);
        GK_CUDA(cudaMemcpy2DAsync(J + (t0 * g.d + p) * ldj, sizeof(double) * ldj * g.d, qe.p, sizeof(double) * op.N,
                                  sizeof(double) * op.N, nt, cudaMemcpyDeviceToHost, s));
        GK_CUDA(cudaStreamSynchronize(s));
      }
    }
  });
}

gk_status gk_dski_cross_covariance(const gk_op* h, const double* Xtest, int64_t T, double* Q, int64_t ldq) {
  return guard([&] {
    Op& op = O(h);
    const gk_grid g = dski_grid(op);
    if (ldq < op.N) fail(GK_ERR_ARG, "size mismatch");
    if (T <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    for (i64 t0 = 0; t0 < T; t0 += kMaxRhs) {
      const i64 nt = std::min<i64>(kMaxRhs, T - t0);
      std::vector<double> xh(static_cast<size_t>(nt) * g.d);
      for (int j = 0; j < g.d; ++j)
        for (i64 i = 0; i < nt; ++i) xh[static_cast<size_t>(j * nt + i)] = Xtest[j * T + t0 + i];
      DevBuf<double> xt(static_cast<size_t>(nt) * g.d), qi(static_cast<size_t>(op.N) * nt), qe(static_cast<size_t>(op.N) * nt);
      DevBuf<int> bad(1);
      const int big = INT_MAX;
      GK_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
      xt.upload(xh.data(), xh.size(), s);
      dski_cross_cov(op, xt.p, nt, qi.p, bad.p, s);
      int badh = INT_MAX;
      GK_CUDA(cudaMemcpy(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost));
      if (badh != INT_MAX)
        fail(GK_ERR_OUT_OF_GRID, "test point " + std::to_string(t0 + badh) + " lies outside the interior of the grid",
             t0 + badh);
      op.from_internal(qi.p, qe.p, op.N, int(nt), s);
      GK_CUDA(cudaMemcpy2DAsync(Q + t0 * ldq, sizeof(double) * ldq, qe.p, sizeof(double) * op.N,
                                sizeof(double) * op.N, nt, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
    }
  });
}

// ---------------------------------------------------------------- D-SKIP pieces
int gk_dskip_factor_count(const gk_op* h) {
  int c = -1;
  guard([&] { c = dskip_factor_count(O(h)); });
  return c;
}
int64_t gk_dskip_factor_rank(const gk_op* h, int f) {
  int64_t r = -1;
  guard([&] { r = dskip_factor_rank(O(h), f); });
  return r;
}
gk_status gk_dskip_factor_get(const gk_op* h, int f, double* Q, double* alpha, double* beta) {
  return guard([&] { dskip_factor_get(O(h), f, Q, alpha, beta); });
}
gk_status gk_dskip_dlogell_apply(const gk_op* h, const double* V, int64_t ldv, double* Out, int64_t ldo,
                                 int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    if (ldv < op.N || ldo < op.N) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    grid_call(op, V, ldv, op.N, Out, ldo, op.N, nrhs, false, false,
              [&](const double* i, double* o, int nb, cudaStream_t s) { dskip_dlogell(op, i, o, nb, s); });
  });
}

gk_status gk_dski_dlogell_apply(const gk_op* h, const double* V, int64_t ldv, double* Out, int64_t ldo,
                                int64_t nrhs) {
  return guard([&] {
    Op& op = O(h);
    if (ldv < op.N || ldo < op.N) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    grid_call(op, V, ldv, op.N, Out, ldo, op.N, nrhs, false, false,
              [&](const double* i, double* o, int nb, cudaStream_t s) { dski_dlogell(op, i, o, nb, s); });
  });
}

// ---------------------------------------------------------------- solvers
gk_status gk_pcg(const gk_op* h, const gk_precond* M, const double* B, int64_t ldb, int64_t nrhs, double tol,
                 int maxit, double* X, int64_t ldx, int* iterations, int* converged, double* history,
                 int* history_len) {
  return guard([&] {
    Op& op = O(h);
    if (ldb < op.N || ldx < op.N) fail(GK_ERR_ARG, "cg: rhs size mismatch");
    if (nrhs <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    Precond* P = M ? &precond_for(M, op) : nullptr;
    std::unique_lock<std::mutex> plk;
    if (P) plk = std::unique_lock<std::mutex>(P->mu);
    const int chunk = int(std::min<i64>(nrhs, 256));
    // the operator's grow-only scratch (held under op.mu): no per-solve cudaMalloc/cudaFree
    op.scratch_a.reserve(static_cast<size_t>(op.N) * chunk);
    op.scratch_b.reserve(static_cast<size_t>(op.N) * chunk);
    op.scratch_c.reserve(static_cast<size_t>(op.N) * chunk);
    double *e = op.scratch_c.p, *bi = op.scratch_a.p, *xi = op.scratch_b.p;
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      upload_internal(op, B + c0 * ldb, ldb, e, bi, nb, s);
      PcgResult r = pcg_internal(op, P, bi, xi, nb, tol, maxit, history != nullptr, s);
      download_internal(op, xi, e, X + c0 * ldx, ldx, nb, s);
      GK_CUDA(cudaStreamSynchronize(s));
      for (int b = 0; b < nb; ++b) {
        if (iterations) iterations[c0 + b] = r.iterations[static_cast<size_t>(b)];
        if (converged) converged[c0 + b] = r.converged[static_cast<size_t>(b)];
        if (history_len) history_len[c0 + b] = r.hist_len[static_cast<size_t>(b)];
        if (history)
          for (int it = 0; it <= maxit; ++it)
            history[(c0 + b) * (maxit + 1) + it] = r.history[static_cast<size_t>(it) * nb + b];
      }
    }
  });
}

gk_status gk_pcg_dev(const gk_op* h, const gk_precond* M, const double* dB, int64_t ldb, int64_t nrhs, double tol,
                     int maxit, double* dX, int64_t ldx, int* iterations, int* converged, void* stream) {
  return guard([&] {
    Op& op = O(h);
    if (ldb < op.N || ldx < op.N) fail(GK_ERR_ARG, "cg: rhs size mismatch");
    if (nrhs <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = S(stream);
    OpSession ss(op, s);
    Precond* P = M ? &precond_for(M, op) : nullptr;
    std::unique_lock<std::mutex> plk;
    if (P) plk = std::unique_lock<std::mutex>(P->mu);
    const int chunk = int(std::min<i64>(nrhs, 256));
    op.scratch_a.reserve(static_cast<size_t>(op.N) * chunk);
    op.scratch_b.reserve(static_cast<size_t>(op.N) * chunk);
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      op.to_internal(dB + c0 * ldb, ldb, op.scratch_a.p, nb, s);
      PcgResult r = pcg_internal(op, P, op.scratch_a.p, op.scratch_b.p, nb, tol, maxit, false, s);
      op.from_internal(op.scratch_b.p, dX + c0 * ldx, ldx, nb, s);
      for (int b = 0; b < nb; ++b) {
        if (iterations) iterations[c0 + b] = r.iterations[static_cast<size_t>(b)];
        if (converged) converged[c0 + b] = r.converged[static_cast<size_t>(b)];
      }
    }
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_pivoted_cholesky(const gk_op* h, int kernel_part, int64_t max_rank, double trace_tol,
                              gk_pivchol** out) {
  return guard([&] {
    Op& op = O(h);
    DeviceGuard dg(op.device);
    OpSession ss(op, op.stream);
    auto f = std::make_unique<gk_pivchol>();
    f->impl = pivchol_run(op, kernel_part != 0, max_rank, trace_tol);
    *out = f.release();
  });
}
int64_t gk_pivchol_rank(const gk_pivchol* f) { return f && f->impl ? f->impl->k : -1; }
gk_status gk_pivchol_get(const gk_pivchol* f, double* L, int64_t* pivots, double* it, double* rt) {
  return guard([&] {
    if (!f || !f->impl) fail(GK_ERR_ARG, "null factor");
    const PivChol& p = *f->impl;
    DeviceGuard dg(p.device);
    if (L) pivchol_copy_L(p, L);
    if (pivots)
      for (size_t j = 0; j < p.pivots.size(); ++j) pivots[j] = p.pivots[j];
    if (it) *it = p.initial_trace;
    if (rt) *rt = p.residual_trace;
  });
}
void gk_pivchol_destroy(gk_pivchol* f) { delete f; }

gk_status gk_precond_create(const double* F, int64_t N, int64_t k, const double* noise_diag, int device,
                            gk_precond** out) {
  return guard([&] {  // linalg.cpp:176-194
    if (N <= 0) fail(GK_ERR_ARG, "preconditioner needs strictly positive noise");
    for (i64 i = 0; i < N; ++i)
      if (!(noise_diag[i] > 0.0)) fail(GK_ERR_ARG, "preconditioner needs strictly positive noise");
    if (k == 0) fail(GK_ERR_ARG, "preconditioner needs a factor of rank at least 1");
    DeviceGuard dg(device);
    cudaStream_t s;
    GK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf<double> Fd(static_cast<size_t>(N * k)), nd(static_cast<size_t>(N));
    Fd.upload(F, static_cast<size_t>(N * k), s);
    nd.upload(noise_diag, static_cast<size_t>(N), s);
    auto M = std::make_unique<gk_precond>();
    M->impl = precond_build(Fd.p, N, k, nd.p, device, s);
    M->impl->stream = s;
    *out = M.release();
  });
}

gk_status gk_precond_from_pivchol(const gk_op* h, const gk_pivchol* f, gk_precond** out) {
  return guard([&] {
    Op& op = O(h);
    if (!f || !f->impl) fail(GK_ERR_ARG, "null factor");
    const PivChol& p = *f->impl;
    if (p.k == 0) fail(GK_ERR_RUNTIME, "pivoted Cholesky produced an empty preconditioner factor");
    if (p.order_uid != op.uid) fail(GK_ERR_ARG, "pivoted Cholesky factor belongs to another operator");
    DeviceGuard dg(op.device);
    cudaStream_t s;
    GK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    OpSession ss(op, s);
    std::vector<double> nh(static_cast<size_t>(op.N));
    for (i64 r = 0; r < op.N; ++r) nh[static_cast<size_t>(r)] = r < op.n_value ? op.nv2 : op.ng2;
    if (op.nv2 <= 0.0 || (op.N > op.n_value && op.ng2 <= 0.0))
      fail(GK_ERR_ARG, "preconditioner needs strictly positive noise");
    DevBuf<double> nd(static_cast<size_t>(op.N));
    nd.upload(nh.data(), nh.size(), s);  // group structure is order-invariant
    auto M = std::make_unique<gk_precond>();
    M->impl = precond_build(p.L.p, op.N, p.k, nd.p, op.device, s);
    M->impl->stream = s;
    M->impl->order_uid = op.uid;
    if (op.d_ext_of_int()) {
      M->impl->ext_own.alloc(static_cast<size_t>(op.N));
      GK_CUDA(cudaMemcpy(M->impl->ext_own.p, op.d_ext_of_int(), sizeof(i64) * op.N, cudaMemcpyDeviceToDevice));
      M->impl->ext = M->impl->ext_own.p;
    }
    *out = M.release();
  });
}

gk_status gk_precond_apply(const gk_precond* M, const double* B, int64_t ldb, double* Out, int64_t ldo,
                           int64_t nrhs) {
  return guard([&] {
    if (!M || !M->impl) fail(GK_ERR_ARG, "null preconditioner");
    Precond& P = *M->impl;
    if (ldb < P.N || ldo < P.N) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    std::lock_guard<std::mutex> lk(P.mu);
    DeviceGuard dg(P.device);
    cudaStream_t s = P.stream;
    const int chunk = int(std::min<i64>(nrhs, kMaxRhs));
    DevBuf<double> e(static_cast<size_t>(P.N) * chunk), a(static_cast<size_t>(P.N) * chunk), b(static_cast<size_t>(P.N) * chunk);
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      GK_CUDA(cudaMemcpy2DAsync(e.p, sizeof(double) * P.N, B + c0 * ldb, sizeof(double) * ldb, sizeof(double) * P.N,
                                nb, cudaMemcpyHostToDevice, s));
      to_internal(P.ext, P.N, e.p, P.N, a.p, nb, s);
      P.apply(a.p, b.p, nb, s);
      from_internal(P.ext, P.N, b.p, e.p, P.N, nb, s);
      GK_CUDA(cudaMemcpy2DAsync(Out + c0 * ldo, sizeof(double) * ldo, e.p, sizeof(double) * P.N,
                                sizeof(double) * P.N, nb, cudaMemcpyDeviceToHost, s));
    }
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

gk_status gk_precond_quadratic(const gk_precond* M, const double* B, int64_t ldb, int64_t nrhs, double* out) {
  return guard([&] {
    if (!M || !M->impl) fail(GK_ERR_ARG, "null preconditioner");
    Precond& P = *M->impl;
    if (ldb < P.N) fail(GK_ERR_ARG, "size mismatch");
    if (nrhs <= 0) return;
    std::lock_guard<std::mutex> lk(P.mu);
    DeviceGuard dg(P.device);
    cudaStream_t s = P.stream;
    const int chunk = int(std::min<i64>(nrhs, kMaxRhs));
    DevBuf<double> e(static_cast<size_t>(P.N) * chunk), a(static_cast<size_t>(P.N) * chunk);
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      GK_CUDA(cudaMemcpy2DAsync(e.p, sizeof(double) * P.N, B + c0 * ldb, sizeof(double) * ldb, sizeof(double) * P.N,
                                nb, cudaMemcpyHostToDevice, s));
      to_internal(P.ext, P.N, e.p, P.N, a.p, nb, s);
      precond_quadratic(P, a.p, nb, out + c0, s);
    }
  });
}

int64_t gk_precond_rank(const gk_precond* M) { return M && M->impl ? M->impl->k : -1; }

gk_status gk_precond_q1(const gk_precond* M, double* Q1) {
  return guard([&] {
    if (!M || !M->impl) fail(GK_ERR_ARG, "null preconditioner");
    Precond& P = *M->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    DeviceGuard dg(P.device);
    cudaStream_t s = P.stream;
    DevBuf<double> e(static_cast<size_t>(P.N * P.k)), t(static_cast<size_t>(P.N * P.k));
    // q1 rows are internal-ordered [N][k] -> external col-major N×k
    from_internal(P.ext, P.N, P.q1.p, e.p, P.N, int(P.k), s);
    GK_CUDA(cudaMemcpyAsync(Q1, e.p, sizeof(double) * P.N * P.k, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
  });
}

void gk_precond_destroy(gk_precond* M) { delete M; }

gk_status gk_slq_logdet(const gk_op* h, int probes, int steps, uint64_t seed, double floor_, int probe_offset,
                        double* logdet, int* clamped, double* estimates) {
  return guard([&] {  // linalg.cpp:215-253
    Op& op = O(h);
    *logdet = 0.0;
    if (clamped) *clamped = 0;
    if (probes <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    const i64 N = op.N;
    const int chunk = std::min(probes, 64);
    std::vector<double> est(static_cast<size_t>(probes), 0.0);
    std::vector<int> clamps(static_cast<size_t>(probes), 0);
    // An odd probe batch runs one extra (discarded) probe: the batched MVM
    // handles RHS pairs, and an odd count falls to its single-RHS variant.
    const int cap = chunk + 1;
    op.slq_h.reserve(static_cast<size_t>(N) * cap);
    double* hzp = op.slq_h.p;
    op.slq_z.reserve(static_cast<size_t>(N) * cap * 2);
    double* ze_p = op.slq_z.p;
    double* zi_p = op.slq_z.p + static_cast<size_t>(N) * cap;
    const bool prof = std::getenv("GK_SLQ_PROF") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    for (int p0 = 0; p0 < probes; p0 += chunk) {
      const int P = std::min(chunk, probes - p0);
      const int Prun = (P & 1) && N > 1 ? P + 1 : P;
      std::vector<std::uint64_t> rseeds(static_cast<size_t>(Prun));
      auto t0 = now();
      // probe vectors (host mt19937_64 streams, bit-exact with the reference),
      // generated in parallel over probes
      std::vector<double> zn2v(static_cast<size_t>(Prun), 0.0);
      auto gen = [&](int q) {
        const std::uint64_t pid = std::uint64_t(probe_offset + p0 + q);
        double* z = hzp + static_cast<size_t>(q) * N;
        rademacher(N, seed, pid, z);
        double s2 = 0.0;
        for (i64 i = 0; i < N; ++i) s2 += z[i] * z[i];
        zn2v[static_cast<size_t>(q)] = s2;
        const double zn = std::sqrt(s2);
        for (i64 i = 0; i < N; ++i) z[i] /= zn;
        rseeds[static_cast<size_t>(q)] = mix_seed(seed, 50000 + pid);
      };
      if (g_tuning.rng.load() == 0) {  // probes generated on the device (bit-identical streams)
        std::vector<std::uint64_t> sds(static_cast<size_t>(Prun));
        for (int q = 0; q < Prun; ++q) {
          const std::uint64_t pid = std::uint64_t(probe_offset + p0 + q);
          sds[static_cast<size_t>(q)] = mix_seed(seed, pid);
          rseeds[static_cast<size_t>(q)] = mix_seed(seed, 50000 + pid);
          zn2v[static_cast<size_t>(q)] = double(N);  // Σ (±1)² in the host path
        }
        rademacher_dev(N, sds.data(), Prun, 1.0 / std::sqrt(double(N)), ze_p, N, s);
      } else {
        parallel_for(Prun, gen);
      }
      auto t1 = now();
      if (g_tuning.rng.load() != 0)
        GK_CUDA(cudaMemcpyAsync(ze_p, hzp, sizeof(double) * N * Prun, cudaMemcpyHostToDevice, s));
      op.to_internal(ze_p, N, zi_p, Prun, s);
      if (prof) GK_CUDA(cudaStreamSynchronize(s));
      auto t2 = now();
      LanczosBatch lb = lanczos_batch(op, zi_p, Prun, steps, rseeds, nullptr, s);
      auto t3 = now();
      if (prof) std::fprintf(stderr, "slq: probes %.2f ms, upload %.2f ms, lanczos %.2f ms\n", ms(t0, t1), ms(t1, t2), ms(t2, t3));
      for (int q = 0; q < P; ++q) {
        const int len = lb.len[static_cast<size_t>(q)];
        std::vector<double> ev(static_cast<size_t>(len)), Z(static_cast<size_t>(len) * len);
        tridiag_eig(len, lb.alpha[static_cast<size_t>(q)].data(), lb.beta[static_cast<size_t>(q)].data(), ev.data(), Z.data());
        double e = 0.0;
        for (int i = 0; i < len; ++i) {
          double lambda = ev[static_cast<size_t>(i)];
          if (lambda < floor_) {
            lambda = floor_;
            ++clamps[static_cast<size_t>(p0 + q)];
          }
          const double w0 = Z[static_cast<size_t>(i) * len];
          e += w0 * w0 * std::log(lambda);
        }
        est[static_cast<size_t>(p0 + q)] = zn2v[static_cast<size_t>(q)] * e;  // ‖z_p‖² (linalg.cpp:240-243)
      }
    }
    double sum = 0.0;
    int cl = 0;
    for (int p = 0; p < probes; ++p) {
      sum += est[static_cast<size_t>(p)];
      cl += clamps[static_cast<size_t>(p)];
    }
    *logdet = sum / probes;
    if (clamped) *clamped = cl;
    if (estimates) std::copy(est.begin(), est.end(), estimates);
  });
}

gk_status gk_lanczos(const gk_op* h, int64_t steps, uint64_t seed, const double* start, uint64_t restart_seed,
                     double* Q, double* alpha, double* beta, int64_t* k, int* breakdown) {
  return guard([&] {
    Op& op = O(h);
    const i64 N = op.N;
    if (!start && (steps <= 0 || steps > N)) fail(GK_ERR_ARG, "Lanczos rank must lie in [1, N]");
    steps = std::min<i64>(steps, N);
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    std::vector<double> q(static_cast<size_t>(N));
    std::uint64_t rs = restart_seed;
    if (start) {
      std::copy(start, start + N, q.begin());
    } else {  // lanczos_lowrank (linalg.cpp:306-314)
      gaussian(N, seed, 0, q.data());
      double nn = 0.0;
      for (double v : q) nn += v * v;
      nn = std::sqrt(nn);
      for (double& v : q) v /= nn;
      rs = mix_seed(seed, 1);
    }
    DevBuf<double> e(static_cast<size_t>(N)), i1(static_cast<size_t>(N)), Qd(static_cast<size_t>(N) * std::max<i64>(steps, 1));
    e.upload(q.data(), static_cast<size_t>(N), s);
    op.to_internal(e.p, N, i1.p, 1, s);
    LanczosBatch lb = lanczos_batch(op, i1.p, 1, int(steps), {rs}, Qd.p, s);
    const int len = lb.len[0];
    if (Q && len > 0) {
      DevBuf<double> qe(static_cast<size_t>(N) * len);
      // Qd is [steps][N][1] == internal RHS-minor per column: convert each column
      for (int j = 0; j < len; ++j) op.from_internal(Qd.p + (i64)j * N, qe.p + (i64)j * N, N, 1, s);
      GK_CUDA(cudaMemcpyAsync(Q, qe.p, sizeof(double) * N * len, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
    }
    if (alpha) std::copy(lb.alpha[0].begin(), lb.alpha[0].end(), alpha);
    if (beta) std::copy(lb.beta[0].begin(), lb.beta[0].end(), beta);
    *k = len;
    if (breakdown) *breakdown = lb.breakdown[0];
  });
}

gk_status gk_trace_estimate(const gk_op* hA, const gk_op* hB, int probes, uint64_t seed, double tol, int maxit,
                            const gk_precond* M, double* out) {
  return guard([&] {  // linalg.cpp:255-279
    Op& A = O(hA);
    Op& B = O(hB);
    if (A.N != B.N) fail(GK_ERR_ARG, "trace_estimate: size mismatch");
    *out = 0.0;
    if (probes <= 0) return;
    const i64 N = A.N;
    std::vector<double> est(static_cast<size_t>(probes), 0.0);
    bool failed = false;
    const int chunk = std::min(probes, 64);
    std::vector<double> hz(static_cast<size_t>(N) * chunk), hbz(static_cast<size_t>(N) * chunk), hx(static_cast<size_t>(N) * chunk);
    for (int p0 = 0; p0 < probes; p0 += chunk) {
      const int P = std::min(chunk, probes - p0);
      for (int q = 0; q < P; ++q) rademacher(N, seed, 1000 + std::uint64_t(p0 + q), hz.data() + static_cast<size_t>(q) * N);
      gk_status st = gk_op_mvm(hB, hz.data(), N, hbz.data(), N, P);
      if (st != GK_OK) fail(st, g_err);
      std::vector<int> its(static_cast<size_t>(P)), conv(static_cast<size_t>(P));
      st = gk_pcg(hA, M, hz.data(), N, P, tol, maxit, hx.data(), N, its.data(), conv.data(), nullptr, nullptr);
      if (st != GK_OK) fail(st, g_err);
      for (int q = 0; q < P; ++q) {
        if (!conv[static_cast<size_t>(q)]) failed = true;
        double dsum = 0.0;
        for (i64 i = 0; i < N; ++i) dsum += hx[static_cast<size_t>(q) * N + i] * hbz[static_cast<size_t>(q) * N + i];
        est[static_cast<size_t>(p0 + q)] = dsum;
      }
    }
    if (failed)
      fail(GK_ERR_RUNTIME, "trace_estimate: CG did not converge within " + std::to_string(maxit) + " iterations");
    double sum = 0.0;
    for (int p = 0; p < probes; ++p) sum += est[static_cast<size_t>(p)];
    *out = sum / probes;
  });
}

// GpModel::lml_gradient (gp.cpp:220-292), stochastic-trace branch: for
// θ = (log ℓ, log s, log σ₁[, log σ₂]),  ∂LML/∂θ_p = ½(αᵀ M_p α − tr(K⁻¹ M_p)),
// the trace by trace_estimate (linalg.cpp:255-279) with probes z_q =
// rademacher(N, seed, 1000+q) and PCG at tol max(tol, 1e-2). The reference
// re-solves K x = z_q identically for every p; here the probes are solved
// once, as one batched PCG, and each x_q is dotted with every M_p z_q.
gk_status gk_lml_gradient(const gk_op* hA, const gk_precond* M, const double* alpha, int probes, uint64_t seed,
                          double tol, int maxit, double* grad, int* nparams) {
  return guard([&] {
    Op& A = O(hA);
    if (!alpha || !grad || !nparams) fail(GK_ERR_ARG, "null argument");
    if (A.kind != KIND_DSKI && A.kind != KIND_DSKIP)
      fail(GK_ERR_UNSUPPORTED, "lml_gradient: stochastic-trace branch needs a D-SKI or D-SKIP operator");
    const i64 N = A.N, n = A.n_value;
    const int np = N > n ? 4 : 3;
    *nparams = np;
    const double nv2 = A.nv2, ng2 = A.ng2;
    // M_p V for a host block of c columns (gp.cpp:229-244)
    auto apply_param = [&](int p, const double* V, double* Out, i64 c) {
      if (p == 0) {
        const gk_status st = A.kind == KIND_DSKI ? gk_dski_dlogell_apply(hA, V, N, Out, N, c)
                                                 : gk_dskip_dlogell_apply(hA, V, N, Out, N, c);
        if (st != GK_OK) fail(st, g_err);
        return;
      }
      if (p == 1) {
        const gk_status st = gk_op_mvm(hA, V, N, Out, N, c);
        if (st != GK_OK) fail(st, g_err);
        for (i64 q = 0; q < c; ++q)
          for (i64 i = 0; i < N; ++i) {
            const i64 e = q * N + i;
            Out[e] = 2.0 * (Out[e] - (i < n ? nv2 : ng2) * V[e]);
          }
        return;
      }
      for (i64 q = 0; q < c; ++q)
        for (i64 i = 0; i < N; ++i) {
          const i64 e = q * N + i;
          const bool mine = p == 2 ? i < n : i >= n;
          Out[e] = mine ? 2.0 * (p == 2 ? nv2 : ng2) * V[e] : 0.0;
        }
    };
    std::vector<double> data(static_cast<size_t>(np)), Ma(static_cast<size_t>(N));
    for (int p = 0; p < np; ++p) {
      apply_param(p, alpha, Ma.data(), 1);
      double s = 0.0;
      for (i64 i = 0; i < N; ++i) s += alpha[i] * Ma[static_cast<size_t>(i)];
      data[static_cast<size_t>(p)] = s;
    }
    std::vector<double> tr(static_cast<size_t>(np), 0.0);
    if (probes > 0) {
      const double ttol = std::max(tol, 1e-2);  // gp.cpp:281-282
      std::vector<double> Z(static_cast<size_t>(N) * probes), X(Z.size()), MZ(Z.size());
      for (int q = 0; q < probes; ++q) rademacher(N, seed, 1000 + std::uint64_t(q), Z.data() + static_cast<size_t>(q) * N);
      std::vector<int> its(static_cast<size_t>(probes)), conv(static_cast<size_t>(probes));
      gk_status st = gk_pcg(hA, M, Z.data(), N, probes, ttol, maxit, X.data(), N, its.data(), conv.data(), nullptr,
                            nullptr);
      if (st != GK_OK) fail(st, g_err);
      for (int q = 0; q < probes; ++q)
        if (!conv[static_cast<size_t>(q)])
          fail(GK_ERR_RUNTIME, "trace_estimate: CG did not converge within " + std::to_string(maxit) + " iterations");
      for (int p = 0; p < np; ++p) {
        apply_param(p, Z.data(), MZ.data(), probes);
        double sum = 0.0;  // per-probe estimates summed in probe order (linalg.cpp:276-277)
        for (int q = 0; q < probes; ++q) {
          double e = 0.0;
          for (i64 i = 0; i < N; ++i) e += X[static_cast<size_t>(q) * N + i] * MZ[static_cast<size_t>(q) * N + i];
          sum += e;
        }
        tr[static_cast<size_t>(p)] = sum / probes;
      }
    }
    for (int p = 0; p < np; ++p) grad[p] = 0.5 * (data[static_cast<size_t>(p)] - tr[static_cast<size_t>(p)]);
  });
}

// ---------------------------------------------------------------- GpModel glue
}  // extern "C"

namespace {
// GpModel::solve's error text (gp.cpp:151-156).
[[noreturn]] void cg_not_converged(double relres, int its, double tol) {
  fail(GK_ERR_RUNTIME, "CG did not converge: relative residual " + std::to_string(relres) + " after " +
                           std::to_string(its) + " iterations (tol " + std::to_string(tol) + ")");
}
// GpModel::solve (gp.cpp:143-158) on an internal block: PCG, then the
// reference's runtime_error for the first column that did not converge.
void gp_solve_internal(Op& op, Precond* P, const double* Bi, double* Xi, int nb, double tol, int maxit,
                       cudaStream_t s, int* its_out) {
  PcgResult r = pcg_internal(op, P, Bi, Xi, nb, tol, maxit, true, s);
  for (int b = 0; b < nb; ++b) {
    if (its_out) its_out[b] = r.iterations[static_cast<size_t>(b)];
    if (!r.converged[static_cast<size_t>(b)]) {
      const int hl = r.hist_len[static_cast<size_t>(b)];
      const double rr = hl > 0 ? r.history[static_cast<size_t>(hl - 1) * nb + b] : 0.0;
      cg_not_converged(rr, r.iterations[static_cast<size_t>(b)], tol);
    }
  }
}
// Test points [t0, t0+nt) of a T×d col-major host block, re-packed nt×d col-major.
std::vector<double> test_chunk(const double* Xtest, i64 T, int d, i64 t0, i64 nt) {
  std::vector<double> xh(static_cast<size_t>(nt) * d);
  for (int j = 0; j < d; ++j)
    for (i64 i = 0; i < nt; ++i) xh[static_cast<size_t>(j * nt + i)] = Xtest[j * T + t0 + i];
  return xh;
}
// cross_covariance (gp.cpp:412-417) of nt test points into Qi (internal, N×nt).
void cross_cov_chunk(Op& op, const gk_grid& g, const double* Xtest, i64 T, i64 t0, i64 nt, double* Qi,
                     cudaStream_t s) {
  std::vector<double> xh = test_chunk(Xtest, T, g.d, t0, nt);
  DevBuf<double> xt(xh.size());
  DevBuf<int> bad(1);
  const int big = INT_MAX;
  GK_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  xt.upload(xh.data(), xh.size(), s);
  dski_cross_cov(op, xt.p, nt, Qi, bad.p, s);
  int badh = INT_MAX;
  GK_CUDA(cudaMemcpy(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (badh != INT_MAX)
    fail(GK_ERR_OUT_OF_GRID, "test point " + std::to_string(t0 + badh) + " lies outside the interior of the grid",
         t0 + badh);
}
}  // namespace

extern "C" {

gk_status gk_gp_solve(const gk_op* h, const gk_precond* M, const double* B, int64_t ldb, int64_t nrhs, double tol,
                      int maxit, double* X, int64_t ldx, int* iterations) {
  return guard([&] {
    Op& op = O(h);
    if (ldb < op.N || ldx < op.N) fail(GK_ERR_ARG, "cg: rhs size mismatch");
    if (nrhs <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    Precond* P = M ? &precond_for(M, op) : nullptr;
    std::unique_lock<std::mutex> plk;
    if (P) plk = std::unique_lock<std::mutex>(P->mu);
    const int chunk = int(std::min<i64>(nrhs, 256));
    DevBuf<double> e(static_cast<size_t>(op.N) * chunk), bi(e.n), xi(e.n);
    for (i64 c0 = 0; c0 < nrhs; c0 += chunk) {
      const int nb = int(std::min<i64>(chunk, nrhs - c0));
      upload_internal(op, B + c0 * ldb, ldb, e.p, bi.p, nb, s);
      gp_solve_internal(op, P, bi.p, xi.p, nb, tol, maxit, s, iterations ? iterations + c0 : nullptr);
      download_internal(op, xi.p, e.p, X + c0 * ldx, ldx, nb, s);
      GK_CUDA(cudaStreamSynchronize(s));
    }
  });
}

gk_status gk_gp_logdet(const gk_op* h, int probes, int steps, uint64_t seed, double noise_value,
                       double noise_gradient, int has_gradients, double* logdet) {
  const double f2 = has_gradients ? std::min(noise_value, noise_gradient) : noise_value;  // gp.cpp:174-177
  int clamped = 0;
  return gk_slq_logdet(h, probes, steps, seed, 0.5 * f2 * f2, 0, logdet, &clamped, nullptr);
}

gk_status gk_gp_log_marginal_likelihood(const gk_op* h, const gk_precond* M, const double* targets, double tol,
                                        int maxit, int probes, int steps, uint64_t seed, double noise_value,
                                        double noise_gradient, int has_gradients, double* lml, double* fit_term,
                                        double* logdet, double* alpha) {
  return guard([&] {  // gp.cpp:181-187
    Op& op = O(h);
    if (!targets || !lml) fail(GK_ERR_ARG, "null argument");
    std::vector<double> a(static_cast<size_t>(op.N));
    int its = 0;
    gk_status st = gk_gp_solve(h, M, targets, op.N, 1, tol, maxit, a.data(), op.N, &its);
    if (st != GK_OK) fail(st, g_err);
    double fit = 0.0;
    for (i64 i = 0; i < op.N; ++i) fit += targets[i] * a[static_cast<size_t>(i)];
    double ld = 0.0;
    st = gk_gp_logdet(h, probes, steps, seed, noise_value, noise_gradient, has_gradients, &ld);
    if (st != GK_OK) fail(st, g_err);
    const double pi = 3.14159265358979323846;
    *lml = -0.5 * (fit + ld + double(op.N) * std::log(2.0 * pi));
    if (fit_term) *fit_term = fit;
    if (logdet) *logdet = ld;
    if (alpha) std::copy(a.begin(), a.end(), alpha);
  });
}

gk_status gk_dski_predict_variance_exact(const gk_op* h, const gk_precond* M, const double* Xtest, int64_t T,
                                         double prior, double tol, int maxit, double* var) {
  return guard([&] {  // gp.cpp:499-502, batched over test points
    Op& op = O(h);
    const gk_grid g = dski_grid(op);
    if (T <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    Precond* P = M ? &precond_for(M, op) : nullptr;
    std::unique_lock<std::mutex> plk;
    if (P) plk = std::unique_lock<std::mutex>(P->mu);
    const int chunk = int(std::min<i64>(T, kMaxRhs));
    DevBuf<double> Qi(static_cast<size_t>(op.N) * chunk), Si(Qi.n), dots(static_cast<size_t>(chunk)), part;
    std::vector<double> dh(static_cast<size_t>(chunk));
    for (i64 t0 = 0; t0 < T; t0 += chunk) {
      const int nt = int(std::min<i64>(chunk, T - t0));
      cross_cov_chunk(op, g, Xtest, T, t0, nt, Qi.p, s);
      gp_solve_internal(op, P, Qi.p, Si.p, nt, tol, maxit, s, nullptr);
      col_dots_dev(Qi.p, Si.p, op.N, nt, dots.p, part, s);
      GK_CUDA(cudaMemcpyAsync(dh.data(), dots.p, sizeof(double) * nt, cudaMemcpyDeviceToHost, s));
      GK_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i < nt; ++i) var[t0 + i] = prior - dh[static_cast<size_t>(i)];
    }
  });
}

gk_status gk_dski_predict_variance_randomized(const gk_op* h, const gk_precond* M, const double* Xtest, int64_t T,
                                              double prior, int probes, uint64_t seed, double tol, int maxit,
                                              double* var) {
  return guard([&] {  // gp.cpp:519-547
    Op& op = O(h);
    const gk_grid g = dski_grid(op);
    if (!M) fail(GK_ERR_LOGIC, "randomized variance needs the preconditioner enabled");
    if (T <= 0) return;
    DeviceGuard dg(op.device);
    cudaStream_t s = op.stream;
    OpSession ss(op, s);
    Precond* P = &precond_for(M, op);
    std::unique_lock<std::mutex> plk(P->mu);
    const i64 N = op.N;
    const int chunk = int(std::min<i64>(T, kMaxRhs));
    const int nchunks = int((T + chunk - 1) / chunk);
    // K' (N×T) kept on the device as per-chunk internal blocks
    DevBuf<double> Kc(static_cast<size_t>(N) * T);
    std::vector<double> base(static_cast<size_t>(T));
    for (int c = 0; c < nchunks; ++c) {
      const i64 t0 = i64(c) * chunk;
      const int nt = int(std::min<i64>(chunk, T - t0));
      double* Qi = Kc.p + N * t0;
      cross_cov_chunk(op, g, Xtest, T, t0, nt, Qi, s);
      precond_quadratic(*P, Qi, nt, base.data() + t0, s);
      for (int i = 0; i < nt; ++i) base[static_cast<size_t>(t0 + i)] = prior - base[static_cast<size_t>(t0 + i)];
    }
    if (probes <= 0) {
      std::copy(base.begin(), base.end(), var);
      return;
    }
    // z_p = rademacher_vector(T, seed, 9000 + p), row-major Z[t][p]
    std::vector<double> Z(static_cast<size_t>(T) * probes), zc(static_cast<size_t>(T));
    for (int p = 0; p < probes; ++p) {
      rademacher(T, seed, 9000 + std::uint64_t(p), zc.data());
      for (i64 t = 0; t < T; ++t) Z[static_cast<size_t>(t * probes + p)] = zc[static_cast<size_t>(t)];
    }
    std::vector<double> G(static_cast<size_t>(T) * probes);  // G[t][p] = q_tᵀ (K⁻¹ − M⁻¹) w_p
    const int pchunk = std::min(probes, kMaxRhs);
    DevBuf<double> Zd, W(static_cast<size_t>(N) * pchunk), EX(W.n), AP(W.n), Gd(static_cast<size_t>(chunk) * pchunk),
        part;
    std::vector<double> Zsub;
    for (int p0 = 0; p0 < probes; p0 += pchunk) {
      const int np = std::min(pchunk, probes - p0);
      // W = K' Z[:, p0:p0+np], summed over the test-point chunks
      for (int c = 0; c < nchunks; ++c) {
        const i64 t0 = i64(c) * chunk;
        const int nt = int(std::min<i64>(chunk, T - t0));
        Zsub.assign(static_cast<size_t>(nt) * np, 0.0);
        for (int t = 0; t < nt; ++t)
          for (int q = 0; q < np; ++q) Zsub[static_cast<size_t>(t * np + q)] = Z[static_cast<size_t>((t0 + t) * probes + p0 + q)];
        Zd.upload(Zsub.data(), Zsub.size(), s);
        rows_gemm_dev(Kc.p + N * t0, nt, Zd.p, np, N, W.p, c > 0, s);
        GK_CUDA(cudaStreamSynchronize(s));  // Zd reused by the next chunk
      }
      gp_solve_internal(op, P, W.p, EX.p, np, tol, maxit, s, nullptr);
      P->apply(W.p, AP.p, np, s);
      sub_dev(EX.p, AP.p, EX.p, N * np, s);
      for (int c = 0; c < nchunks; ++c) {
        const i64 t0 = i64(c) * chunk;
        const int nt = int(std::min<i64>(chunk, T - t0));
        cross_dev(Kc.p + N * t0, nt, EX.p, np, N, Gd.p, part, s);
        std::vector<double> gh(static_cast<size_t>(nt) * np);
        GK_CUDA(cudaMemcpyAsync(gh.data(), Gd.p, sizeof(double) * gh.size(), cudaMemcpyDeviceToHost, s));
        GK_CUDA(cudaStreamSynchronize(s));
        for (int t = 0; t < nt; ++t)
          for (int q = 0; q < np; ++q) G[static_cast<size_t>((t0 + t) * probes + p0 + q)] = gh[static_cast<size_t>(t * np + q)];
      }
    }
    for (i64 t = 0; t < T; ++t) {
      double corr = 0.0;  // accumulated in probe order (gp.cpp:538-544)
      for (int p = 0; p < probes; ++p) corr += Z[static_cast<size_t>(t * probes + p)] * G[static_cast<size_t>(t * probes + p)];
      var[t] = base[static_cast<size_t>(t)] - corr / double(probes);
    }
  });
}

// ---------------------------------------------------------------- row-sharded preconditioner
gk_status gk_precond_from_q1_dev(const double* dQ1, const double* ddinv, int64_t N, int64_t k, int device,
                                 gk_precond** out) {
  return guard([&] {
    if (N <= 0 || k <= 0 || !dQ1 || !ddinv || !out) fail(GK_ERR_ARG, "bad preconditioner factor");
    DeviceGuard dg(device);
    cudaStream_t s;
    GK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    auto M = std::make_unique<gk_precond>();
    M->impl = precond_from_q1(dQ1, ddinv, N, k, device, s);
    M->impl->stream = s;
    *out = M.release();
  });
}

gk_status gk_precond_project_dev(const gk_precond* M, const double* dR, double* dT, int64_t nrhs, void* stream) {
  return guard([&] {
    if (!M || !M->impl) fail(GK_ERR_ARG, "null preconditioner");
    if (nrhs < 1 || nrhs > 256) fail(GK_ERR_ARG, "nrhs must be in [1, 256]");
    Precond& P = *M->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    DeviceGuard dg(P.device);
    precond_project(P, dR, int(nrhs), dT, S(stream));
  });
}

gk_status gk_precond_finish_dev(const gk_precond* M, const double* dR, const double* dT, double* dZ, int64_t nrhs,
                                void* stream) {
  return guard([&] {
    if (!M || !M->impl) fail(GK_ERR_ARG, "null preconditioner");
    if (nrhs < 1 || nrhs > 256) fail(GK_ERR_ARG, "nrhs must be in [1, 256]");
    Precond& P = *M->impl;
    std::lock_guard<std::mutex> lk(P.mu);
    DeviceGuard dg(P.device);
    precond_finish(P, dR, dT, dZ, int(nrhs), S(stream));
  });
}

gk_status gk_sample_test_function(const char* name, int64_t n, uint64_t seed, double noise_value,
                                  double noise_gradient, int with_gradients, int* d, double* X, double* y,
                                  double* dY) {
  gk_status st = GK_OK;
  try {
    st = gk_sample_test_function_impl(name, n, seed, noise_value, noise_gradient, with_gradients, d, X, y, dY);
    if (st != GK_OK) g_err = std::string("unknown test function '") + (name ? name : "") + "'";
  } catch (const std::exception& e) {
    g_err = e.what();
    st = GK_ERR_RUNTIME;
  }
  return st;
}

gk_status gk_make_dataset(int config, uint64_t seed, int64_t* n, int* d, double* X, double* y, double* dY) {
  gk_status st = GK_OK;
  try {
    st = gk_make_dataset_impl(config, seed, n, d, X, y, dY);
    if (st != GK_OK) g_err = "unknown dataset config";
  } catch (const std::exception& e) {
    g_err = e.what();
    st = GK_ERR_RUNTIME;
  }
  return st;
}

}  // extern "C"
