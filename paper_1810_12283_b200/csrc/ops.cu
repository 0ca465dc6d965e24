// ops.cu — layout conversion shared by all device operators, plus the two
// non-structured operators: the matrix-free exact D-SE operator (the dense
// K∇ of reference kernels.cpp:242-285, never materialised) and an explicit
// dense operator (linear_operator.hpp:38-56) used by solver tests.
#include <cmath>
#include <dlfcn.h>
#include <string>
#include <type_traits>
#include <cusolverDn.h>

#include "gk_kernels.cuh"
#include "solvers.hpp"

namespace gk {

namespace {

// External column-major block (rows N, leading dim ldv) <-> internal RHS-minor
// (I[r*nrhs + b]) with the row map ext[r] (null = identity). 32×32 tiles
// through shared memory keep both sides coalesced.
__global__ void k_to_internal(const double* __restrict__ V, i64 ldv, const i64* __restrict__ ext, i64 N,
                              int nrhs, double* __restrict__ I) {
  __shared__ double tile[32][33];
  const i64 r0 = (i64)blockIdx.x * 32;
  const int b0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 × 8
  for (int k = ty; k < 32; k += 8) {
    const i64 r = r0 + tx;
    const int b = b0 + k;
    if (r < N && b < nrhs) {
      const i64 re = ext ? ext[r] : r;
      tile[k][tx] = V[(i64)b * ldv + re];
    }
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const i64 r = r0 + k;
    const int b = b0 + tx;
    if (r < N && b < nrhs) I[r * nrhs + b] = tile[tx][k];
  }
}

__global__ void k_from_internal(const double* __restrict__ I, const i64* __restrict__ ext, i64 N, int nrhs,
                                double* __restrict__ V, i64 ldv) {
  __shared__ double tile[32][33];
  const i64 r0 = (i64)blockIdx.x * 32;
  const int b0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const i64 r = r0 + k;
    const int b = b0 + tx;
    if (r < N && b < nrhs) tile[tx][k] = I[r * nrhs + b];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const i64 r = r0 + tx;
    const int b = b0 + k;
    if (r < N && b < nrhs) {
      const i64 re = ext ? ext[r] : r;
      V[(i64)b * ldv + re] = tile[k][tx];
    }
  }
}

// Kernel family parameters of the matrix-free exact operator.
struct KParams {
  int family;  // 0 SE, 1 spline
  double s2, ell, ell2, a, b;
  int even;
};

// One (x_i, x_j) pair of K∇ (kernels.cpp:104-170, assembled as :242-285):
// k = eval, dk/dx'_q = g·u_q (u = x_i − x_j; dk/dx_p = −g·u_p), and the
// Hessian block d²k/dx_p dx'_q = α δ_pq + β u_p u_q.
__device__ __forceinline__ void kpair(const KParams& K, double r2, double& k, double& g, double& al, double& be) {
  if (K.family == 0) {  // SeProfile (kernels.cpp:22-27)
    k = K.s2 * exp(-0.5 * r2 / K.ell2);
    g = k / K.ell2;
    al = g;
    be = -g / K.ell2;
    return;
  }
  const double r = sqrt(r2), rho = r / K.ell;
  const double radial = K.even ? (rho > 0 ? rho * rho * log(rho) : 0.0) : rho * rho * rho;
  k = K.s2 * (radial + K.a * rho * rho + K.b);
  if (r == 0.0) {  // analytic limit / convention (kernels.cpp:129, 155-159)
    g = 0.0;
    al = -2.0 * K.a * K.s2 / K.ell2;
    be = 0.0;
  } else if (!K.even) {
    const double c1 = 3.0 * r / (K.ell2 * K.ell) + 2.0 * K.a / K.ell2;
    g = -K.s2 * c1;
    al = g;
    be = -K.s2 * 3.0 / (r * K.ell2 * K.ell);
  } else {
    const double c = (2.0 * log(rho) + 1.0 + 2.0 * K.a) / K.ell2;
    g = -K.s2 * c;
    al = g;
    be = -K.s2 * 2.0 / (K.ell2 * r2);
  }
}

// The same decomposition for ∂/∂log ℓ of the kernel (eval_dlogell,
// eval_grad_dlogell, eval_hess_dlogell, kernels.cpp:172-240).
__device__ __forceinline__ void kpair_dl(const KParams& K, double r2, double& k, double& g, double& al,
                                         double& be) {
  if (K.family == 0) {
    const double kv = K.s2 * exp(-0.5 * r2 / K.ell2), rho2 = r2 / K.ell2;
    k = kv * rho2;
    g = kv / K.ell2 * (rho2 - 2.0);
    al = g;
    be = -kv / (K.ell2 * K.ell2) * (rho2 - 4.0);
    return;
  }
  if (r2 == 0.0) {
    k = 0.0;
    g = 0.0;
    al = 4.0 * K.a * K.s2 / K.ell2;
    be = 0.0;
    return;
  }
  const double r = sqrt(r2), rho2 = r2 / K.ell2, rho = sqrt(rho2);
  if (!K.even) {
    k = K.s2 * (-3.0 * rho * rho2 - 2.0 * K.a * rho2);
    g = K.s2 * (9.0 * r / (K.ell2 * K.ell) + 4.0 * K.a / K.ell2);
    al = g;
    be = K.s2 * 9.0 / (r * K.ell2 * K.ell);
  } else {
    const double lr = log(r / K.ell);
    k = K.s2 * (-2.0 * rho2 * log(rho) - rho2 - 2.0 * K.a * rho2);
    g = 2.0 * K.s2 * (2.0 * lr + 2.0 + 2.0 * K.a) / K.ell2;
    al = g;
    be = 2.0 * K.s2 / K.ell2 * (2.0 / r2);
  }
}

// assemble_dense (kernels.cpp:242-285): K(X, X') in type-major blocks, one
// thread per point pair writing its (d+1)² entries; dl: ∂K/∂log ℓ; scale c
// > 0 multiplies derivative rows and columns (AssemblyOptions, kernels.hpp:83-92).
constexpr int kAsmMaxD = 16;
__global__ void k_assemble_dense(const double* __restrict__ X, i64 n, const double* __restrict__ Xp, i64 np, int d,
                                 KParams K, int with_deriv, int dl, double c, double* __restrict__ out, i64 ld) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n * np; e += (i64)gridDim.x * blockDim.x) {
    const i64 i = e % n, j = e / n;
    double u[kAsmMaxD], r2 = 0.0;
    for (int p = 0; p < d; ++p) {
      u[p] = X[p * n + i] - Xp[p * np + j];
      r2 += u[p] * u[p];
    }
    double k, g, al, be;
    if (dl) kpair_dl(K, r2, k, g, al, be);
    else kpair(K, r2, k, g, al, be);
    out[j * ld + i] = k;
    if (!with_deriv) continue;
    const double cs = c > 0.0 ? c : 1.0;
    for (int p = 0; p < d; ++p) {
      out[((p + 1) * np + j) * ld + i] = cs * g * u[p];   // d/dx'_p columns
      out[j * ld + (p + 1) * n + i] = -cs * g * u[p];     // d/dx_p rows
      for (int q = 0; q < d; ++q)
        out[((q + 1) * np + j) * ld + (p + 1) * n + i] = cs * cs * ((p == q ? al : 0.0) + be * u[p] * u[q]);
    }
  }
}

// Matrix-free exact K∇ (type-major, kernels.cpp:242-285) + noise, SE or
// spline. One thread per (row point i, rhs b) computes all d+1 output
// groups; the column points are streamed through shared memory in tiles.
template <int D, bool GRAD>
__global__ void __launch_bounds__(256) k_exact_mvm(const double* __restrict__ X, i64 n, KParams K,
                                                   const double* __restrict__ v, double* __restrict__ out,
                                                   int nrhs, double nv2, double ng2) {
  constexpr int TILE = 128;
  __shared__ double xs[D][TILE];
  const i64 items = n * nrhs;
  const i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  const bool active = it < items;
  const int b = active ? int(it % nrhs) : 0;
  const i64 i = active ? it / nrhs : 0;
  double xi[D];
#pragma unroll
  for (int p = 0; p < D; ++p) xi[p] = active ? X[p * n + i] : 0.0;
  constexpr int NG = GRAD ? D + 1 : 1;
  double o[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) o[g] = 0.0;
  for (i64 j0 = 0; j0 < n; j0 += TILE) {
    __syncthreads();
    for (int t = threadIdx.x; t < TILE * D; t += blockDim.x) {
      const int p = t / TILE, jj = t % TILE;
      xs[p][jj] = (j0 + jj < n) ? X[p * n + j0 + jj] : 0.0;
    }
    __syncthreads();
    if (!active) continue;
    const int jn = int((n - j0) < TILE ? (n - j0) : TILE);
    for (int jj = 0; jj < jn; ++jj) {
      const i64 j = j0 + jj;
      double u[D], r2 = 0.0;
#pragma unroll
      for (int p = 0; p < D; ++p) {
        u[p] = xi[p] - xs[p][jj];
        r2 += u[p] * u[p];
      }
      double k, gc, al, be;
      kpair(K, r2, k, gc, al, be);
      const double v0 = v[j * nrhs + b];
      o[0] += k * v0;
      if constexpr (GRAD) {
        double vq[D], uv = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          vq[q] = v[((q + 1) * n + j) * nrhs + b];
          o[0] += gc * u[q] * vq[q];  // K(i, (q+1)j) = dk/dx'_q
          uv += u[q] * vq[q];
        }
        // rows (p+1)i: −g u_p v0 + Σ_q (α δ_pq + β u_p u_q) v_q
#pragma unroll
        for (int p = 0; p < D; ++p) o[p + 1] += -gc * u[p] * v0 + al * vq[p] + be * u[p] * uv;
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const i64 idx = ((i64)g * n + i) * nrhs + b;
    out[idx] = o[g] + (g == 0 ? nv2 : ng2) * v[idx];
  }
}

__global__ void k_exact_diag(i64 n, int groups, KParams K, double nv2, double ng2, double* __restrict__ d) {
  const i64 N = n * (groups + 1);
  double k, g, al, be;
  kpair(K, 0.0, k, g, al, be);
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    d[r] = r < n ? k + nv2 : al + ng2;
}

template <int D>
__global__ void k_exact_row(const double* __restrict__ X, i64 n, int groups, KParams K, i64 gi, int gg,
                            double nv2, double ng2, double* __restrict__ out) {
  const i64 N = n * (groups + 1);
  double xi[D];
  for (int p = 0; p < D; ++p) xi[p] = X[p * n + gi];
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x) {
    const int q = int(r / n);  // column group
    const i64 j = r % n;
    double u[D], r2 = 0.0;
    for (int p = 0; p < D; ++p) {
      u[p] = xi[p] - X[p * n + j];
      r2 += u[p] * u[p];
    }
    double k, gc, al, be;
    kpair(K, r2, k, gc, al, be);
    double val;
    if (gg == 0 && q == 0) val = k;
    else if (gg == 0) val = gc * u[q - 1];
    else if (q == 0) val = -gc * u[gg - 1];
    else val = (gg == q ? al : 0.0) + be * u[gg - 1] * u[q - 1];
    if (j == gi && q == gg) val += gg == 0 ? nv2 : ng2;
    out[r] = val;
  }
}

// Explicit dense operator, out = A V (A col-major N×N, V internal RHS-minor).
__global__ void k_dense_mvm(const double* __restrict__ A, i64 N, const double* __restrict__ v,
                            double* __restrict__ out, int nrhs) {
  const i64 items = N * nrhs;
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const int b = int(it % nrhs);
    const i64 r = it / nrhs;
    double acc = 0.0;
    for (i64 c = 0; c < N; ++c) acc += A[c * N + r] * v[c * nrhs + b];
    out[it] = acc;
  }
}
__global__ void k_dense_diag(const double* __restrict__ A, i64 N, double* __restrict__ d) {
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    d[r] = A[r * N + r];
}
__global__ void k_dense_row(const double* __restrict__ A, i64 N, i64 row, double* __restrict__ out) {
  for (i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x; c < N; c += (i64)gridDim.x * blockDim.x)
    out[c] = A[c * N + row];
}

}  // namespace

void to_internal(const i64* ext, i64 N, const double* V, i64 ldv, double* I, int nrhs, cudaStream_t s) {
  dim3 grid(unsigned((N + 31) / 32), unsigned((nrhs + 31) / 32));
  k_to_internal<<<grid, dim3(32, 8), 0, s>>>(V, ldv, ext, N, nrhs, I);
  launched("to_internal");
}

void from_internal(const i64* ext, i64 N, const double* I, double* V, i64 ldv, int nrhs, cudaStream_t s) {
  dim3 grid(unsigned((N + 31) / 32), unsigned((nrhs + 31) / 32));
  k_from_internal<<<grid, dim3(32, 8), 0, s>>>(I, ext, N, nrhs, V, ldv);
  launched("from_internal");
}

void Op::to_internal(const double* V, i64 ldv, double* I, int nrhs, cudaStream_t s) const {
  gk::to_internal(d_ext_of_int(), N, V, ldv, I, nrhs, s);
}

void Op::from_internal(const double* I, double* V, i64 ldv, int nrhs, cudaStream_t s) const {
  gk::from_internal(d_ext_of_int(), N, I, V, ldv, nrhs, s);
}

void Op::mvm_graph(const double* in, double* out, int nrhs, cudaStream_t s) {
  auto drop_stale = [&] {
    for (auto it = graphs.begin(); it != graphs.end();) {
      if (it->epoch != epoch) {
        cudaGraphExecDestroy(it->exec);
        it = graphs.erase(it);
      } else {
        ++it;
      }
    }
  };
  drop_stale();
  for (auto& g : graphs)
    if (g.in == in && g.out == out && g.nrhs == nrhs) {
      GK_CUDA(cudaGraphLaunch(g.exec, s));
      g_launches.fetch_add(g.nodes);
      return;
    }
  if (!cap_stream) init_stream();
  mvm(in, out, nrhs, s);  // warm scratch (allocation must not happen during capture)
  GK_CUDA(cudaStreamSynchronize(s));
  drop_stale();  // the warm call may have grown scratch
  const i64 before = g_launches.load();
  cudaGraph_t graph;
  GK_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
  mvm(in, out, nrhs, cap_stream);
  GK_CUDA(cudaStreamEndCapture(cap_stream, &graph));
  GraphEntry e{in, out, nrhs, nullptr, g_launches.load() - before, epoch};
  g_launches.fetch_sub(e.nodes);
  GK_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
  cudaGraphDestroy(graph);
  if (graphs.size() >= 16) {
    cudaGraphExecDestroy(graphs.front().exec);
    graphs.erase(graphs.begin());
  }
  graphs.push_back(e);
  GK_CUDA(cudaGraphLaunch(e.exec, s));
  g_launches.fetch_add(e.nodes);
}

void Op::stage(int st, const double* in, double* out, int nrhs, cudaStream_t s) {
  if (st == 3) return mvm(in, out, nrhs, s);
  if (st == 4) return mvm_graph(in, out, nrhs, s);
  fail(GK_ERR_ARG, "this operator has no D-SKI stages");
}

// ---------------------------------------------------------------- exact
struct ExactOp final : Op {
  int d = 0, G = 0;
  i64 n = 0;
  KParams K{};
  DevBuf<double> X;
  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {
    const int blocks = int((n * nrhs + 255) / 256);
#define GK_EXACT_CASE(DD)                                                                          \
  case DD:                                                                                         \
    if (G) k_exact_mvm<DD, true><<<blocks, 256, 0, s>>>(X.p, n, K, in, out, nrhs, nv2, ng2); \
    else k_exact_mvm<DD, false><<<blocks, 256, 0, s>>>(X.p, n, K, in, out, nrhs, nv2, ng2); \
    break;
    switch (d) {
      GK_EXACT_CASE(1)
      GK_EXACT_CASE(2)
      GK_EXACT_CASE(3)
      GK_EXACT_CASE(4)
      GK_EXACT_CASE(5)
      GK_EXACT_CASE(6)
      default: fail(GK_ERR_UNSUPPORTED, "exact operator supports 1 <= d <= 6");
    }
#undef GK_EXACT_CASE
    launched("exact mvm");
  }
  void diagonal(double* dd, cudaStream_t s) override {
    k_exact_diag<<<blocks_for(N), 256, 0, s>>>(n, G, K, nv2, ng2, dd);
    launched("exact diag");
  }
  void row(i64 r, double* out, cudaStream_t s) override {
    if (r < 0 || r >= N) fail(GK_ERR_RANGE, "row index out of range");
    const i64 gi = r % n;
    const int gg = int(r / n);
    switch (d) {
#define GK_ROW_CASE(DD) \
  case DD: k_exact_row<DD><<<blocks_for(N), 256, 0, s>>>(X.p, n, G, K, gi, gg, nv2, ng2, out); break;
      GK_ROW_CASE(1)
      GK_ROW_CASE(2)
      GK_ROW_CASE(3)
      GK_ROW_CASE(4)
      GK_ROW_CASE(5)
      GK_ROW_CASE(6)
#undef GK_ROW_CASE
      default: fail(GK_ERR_UNSUPPORTED, "exact operator supports 1 <= d <= 6");
    }
    launched("exact row");
  }
};

std::unique_ptr<Op> make_exact(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                               int with_grad, int device) {
  if (k.family != 0 && k.family != 1) fail(GK_ERR_ARG, "unknown kernel family");
  if (!(k.lengthscale > 0.0)) fail(GK_ERR_ARG, "lengthscale must be > 0");
  if (!(k.outputscale > 0.0)) fail(GK_ERR_ARG, "outputscale must be > 0");
  if (d < 1 || d > 6) fail(GK_ERR_UNSUPPORTED, "exact operator supports 1 <= d <= 6");
  DeviceGuard dg(device);
  auto op = std::make_unique<ExactOp>();
  op->kind = KIND_EXACT;
  op->device = device;
  op->d = d;
  op->G = with_grad ? d : 0;
  op->n = n;
  op->N = n * (op->G + 1);
  op->n_value = n;
  op->nv2 = nv * nv;
  op->ng2 = ng * ng;
  op->K = KParams{k.family, k.outputscale * k.outputscale, k.lengthscale, k.lengthscale * k.lengthscale,
                  k.spline_a, k.spline_b, k.spline_even};
  op->init_stream();
  op->X.upload(X, static_cast<size_t>(n) * d, op->stream);
  GK_CUDA(cudaStreamSynchronize(op->stream));
  return op;
}

// ---------------------------------------------------------------- dense
// cuSOLVER's dense Cholesky (potrf/potrs/potri) for the exact GpModel backend
// (the reference's Eigen LLT, gp.cpp:71-85,146,167,246-276) — not on the
// D-SKI/D-SKIP hot path. Loaded with dlopen on first use by soname, so a
// copy the process already mapped (e.g. torch's) is reused.
struct CusolverApi {
  bool ok = false;
  std::string err;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*potrf_bs)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potrf)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potrs)(cusolverDnHandle_t, cublasFillMode_t, int, int, const double*, int, double*, int,
                            int*) = nullptr;
  cusolverStatus_t (*potri_bs)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potri)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
};
static CusolverApi& cusolver() {
  static CusolverApi api = [] {
    CusolverApi a;
    void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = dlerror();
      return a;
    }
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
    sym(a.create, "cusolverDnCreate");
    sym(a.destroy, "cusolverDnDestroy");
    sym(a.set_stream, "cusolverDnSetStream");
    sym(a.potrf_bs, "cusolverDnDpotrf_bufferSize");
    sym(a.potrf, "cusolverDnDpotrf");
    sym(a.potrs, "cusolverDnDpotrs");
    sym(a.potri_bs, "cusolverDnDpotri_bufferSize");
    sym(a.potri, "cusolverDnDpotri");
    a.ok = a.create && a.destroy && a.set_stream && a.potrf_bs && a.potrf && a.potrs && a.potri_bs && a.potri;
    if (!a.ok) a.err = "cuSOLVER symbols missing";
    return a;
  }();
  if (!api.ok) fail(GK_ERR_CUDA, "cuSOLVER (dense Cholesky of the exact backend) unavailable: " + api.err);
  return api;
}
static void sol_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS) fail(GK_ERR_CUDA, std::string(what) + ": cuSOLVER status " + std::to_string(int(st)));
}

__global__ void k_add_noise_diag(double* __restrict__ A, i64 N, i64 n, double nv2, double ng2) {
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < N; r += (i64)gridDim.x * blockDim.x)
    A[r * N + r] += r < n ? nv2 : ng2;
}
// log det = 2 Σ log L_ii, one block, fixed order (gp.cpp:167-168)
__global__ void k_chol_logdet(const double* __restrict__ L, i64 N, double* __restrict__ out) {
  __shared__ double sm[256];
  double acc = 0.0;
  for (i64 r = threadIdx.x; r < N; r += blockDim.x) acc += log(L[r * N + r]);
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 256; ++k) t += sm[k];
    *out = 2.0 * t;
  }
}
// fill the upper triangle of a lower-stored symmetric matrix
__global__ void k_symmetrize_lower(double* __restrict__ A, i64 N) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < N * N; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e % N, c = e / N;
    if (r < c) A[c * N + r] = A[r * N + c];
  }
}

struct DenseOp final : Op {
  DevBuf<double> A;
  // exact-backend state (make_dense_kernel): the Cholesky factor and the data
  DevBuf<double> L;
  cusolverDnHandle_t sol = nullptr;
  DevBuf<int> info;
  DevBuf<double> work;
  bool kernel_built = false;
  KParams K{};
  DevBuf<double> X;
  i64 n = 0;
  int d = 0, G = 0;
  ~DenseOp() override {
    if (sol) cusolver().destroy(sol);
  }
  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override {
    k_dense_mvm<<<blocks_for(N * nrhs), 256, 0, s>>>(A.p, N, in, out, nrhs);
    launched("dense mvm");
  }
  void diagonal(double* dd, cudaStream_t s) override {
    k_dense_diag<<<blocks_for(N), 256, 0, s>>>(A.p, N, dd);
    launched("dense diag");
  }
  void row(i64 r, double* out, cudaStream_t s) override {
    if (r < 0 || r >= N) fail(GK_ERR_RANGE, "row index out of range");
    k_dense_row<<<blocks_for(N), 256, 0, s>>>(A.p, N, r, out);
    launched("dense row");
  }
};

// assemble_dense(kernel, X, X') on the device into out (rows × cols,
// column-major, leading dimension ld) — shared by gk_assemble_dense and the
// exact backend.
void assemble_dense_dev(const gk_kernel& k, const double* dX, i64 n, const double* dXp, i64 np, int d, bool deriv,
                        bool dl, double c, double* out, i64 ld, cudaStream_t s) {
  if (d > kAsmMaxD) fail(GK_ERR_UNSUPPORTED, "dense assembly supports d <= 16");
  const KParams K{k.family, k.outputscale * k.outputscale, k.lengthscale, k.lengthscale * k.lengthscale,
                  k.spline_a, k.spline_b, k.spline_even};
  k_assemble_dense<<<blocks_for(n * np), 256, 0, s>>>(dX, n, dXp, np, d, K, deriv ? 1 : 0, dl ? 1 : 0, c, out, ld);
  launched("assemble dense");
}

// GpModel's exact operator (gp.cpp:71-85): K = assemble_dense + noise on the
// device and its Cholesky factor; not positive definite -> runtime_error.
std::unique_ptr<Op> make_dense_kernel(const gk_kernel& k, const double* X, i64 n, int d, double nv, double ng,
                                      int with_grad, i64 size_cap, int device) {
  if (k.family != 0 && k.family != 1) fail(GK_ERR_ARG, "unknown kernel family");
  if (!(k.lengthscale > 0.0)) fail(GK_ERR_ARG, "lengthscale must be > 0");
  if (!(k.outputscale > 0.0)) fail(GK_ERR_ARG, "outputscale must be > 0");
  if (n < 1 || d < 1) fail(GK_ERR_ARG, "dense kernel operator needs points");
  const i64 N = with_grad ? n * (d + 1) : n;
  if (N * N > size_cap)
    fail(GK_ERR_LENGTH, "dense assembly of " + std::to_string(N) + " x " + std::to_string(N) +
                            " exceeds the configured size cap");
  if (N >= (i64(1) << 31)) fail(GK_ERR_UNSUPPORTED, "dense operator too large");
  DeviceGuard dg(device);
  auto op = std::make_unique<DenseOp>();
  op->kind = KIND_DENSE;
  op->device = device;
  op->N = N;
  op->n_value = n;
  op->n = n;
  op->d = d;
  op->G = with_grad ? d : 0;
  op->nv2 = nv * nv;
  op->ng2 = ng * ng;
  op->kernel_built = true;
  op->K = KParams{k.family, k.outputscale * k.outputscale, k.lengthscale, k.lengthscale * k.lengthscale,
                  k.spline_a, k.spline_b, k.spline_even};
  op->init_stream();
  cudaStream_t s = op->stream;
  op->X.upload(X, static_cast<size_t>(n) * d, s);
  op->A.alloc(static_cast<size_t>(N) * N);
  assemble_dense_dev(k, op->X.p, n, op->X.p, n, d, with_grad != 0, false, 0.0, op->A.p, N, s);
  k_add_noise_diag<<<blocks_for(N), 256, 0, s>>>(op->A.p, N, n, op->nv2, op->ng2);
  launched("dense noise diagonal");
  auto& api = cusolver();
  sol_check(api.create(&op->sol), "cusolverDnCreate");
  sol_check(api.set_stream(op->sol, s), "cusolverDnSetStream");
  op->L.alloc(static_cast<size_t>(N) * N);
  GK_CUDA(cudaMemcpyAsync(op->L.p, op->A.p, sizeof(double) * N * N, cudaMemcpyDeviceToDevice, s));
  int lwork = 0;
  sol_check(api.potrf_bs(op->sol, CUBLAS_FILL_MODE_LOWER, int(N), op->L.p, int(N), &lwork), "potrf buffer size");
  op->work.alloc(static_cast<size_t>(std::max(1, lwork)));
  op->info.alloc(1);
  sol_check(api.potrf(op->sol, CUBLAS_FILL_MODE_LOWER, int(N), op->L.p, int(N), op->work.p, lwork, op->info.p),
            "potrf");
  int info_h = 0;
  GK_CUDA(cudaMemcpyAsync(&info_h, op->info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  if (info_h != 0) fail(GK_ERR_RUNTIME, "dense kernel matrix is not positive definite");
  return op;
}

static DenseOp& factored(Op& o) {
  if (o.kind != KIND_DENSE || !static_cast<DenseOp&>(o).kernel_built)
    fail(GK_ERR_LOGIC, "operator has no dense Cholesky factor (build it with gk_dense_kernel_create)");
  return static_cast<DenseOp&>(o);
}

// X = K⁻¹ B by the Cholesky factor (llt_->solve, gp.cpp:146); device,
// column-major N × nrhs blocks (in place when dB == dX).
void dense_chol_solve(Op& o, const double* dB, double* dX, int nrhs, cudaStream_t s) {
  DenseOp& op = factored(o);
  auto& api = cusolver();
  if (dB != dX) GK_CUDA(cudaMemcpyAsync(dX, dB, sizeof(double) * op.N * nrhs, cudaMemcpyDeviceToDevice, s));
  sol_check(api.set_stream(op.sol, s), "cusolverDnSetStream");
  sol_check(api.potrs(op.sol, CUBLAS_FILL_MODE_LOWER, int(op.N), nrhs, op.L.p, int(op.N), dX, int(op.N), op.info.p),
            "potrs");
}

double dense_chol_logdet(Op& o) {
  DenseOp& op = factored(o);
  DevBuf<double> out(1);
  k_chol_logdet<<<1, 256, 0, op.stream>>>(op.L.p, op.N, out.p);
  launched("dense logdet");
  double h = 0.0;
  GK_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, op.stream));
  GK_CUDA(cudaStreamSynchronize(op.stream));
  return h;
}

// GpModel::lml_gradient, exact branch (gp.cpp:246-276): Kinv from the
// factor, ∂K/∂log ℓ assembled on the device, traces as fixed-order dots.
void dense_exact_lml_gradient(Op& o, const double* alpha_h, double* grad, int* nparams) {
  DenseOp& op = factored(o);
  auto& api = cusolver();
  cudaStream_t s = op.stream;
  const i64 N = op.N, n = op.n;
  DevBuf<double> Kinv(static_cast<size_t>(N) * N), Mell(static_cast<size_t>(N) * N), a(static_cast<size_t>(N)),
      t(static_cast<size_t>(N)), ones(static_cast<size_t>(N)), dots(8), part;
  GK_CUDA(cudaMemcpyAsync(Kinv.p, op.L.p, sizeof(double) * N * N, cudaMemcpyDeviceToDevice, s));
  int lwork = 0;
  sol_check(api.set_stream(op.sol, s), "cusolverDnSetStream");
  sol_check(api.potri_bs(op.sol, CUBLAS_FILL_MODE_LOWER, int(N), Kinv.p, int(N), &lwork), "potri buffer size");
  op.work.reserve(static_cast<size_t>(std::max(1, lwork)));
  sol_check(api.potri(op.sol, CUBLAS_FILL_MODE_LOWER, int(N), Kinv.p, int(N), op.work.p, lwork, op.info.p), "potri");
  k_symmetrize_lower<<<blocks_for(N * N), 256, 0, s>>>(Kinv.p, N);
  launched("dense symmetrize");
  gk_kernel kk{op.K.family, op.K.ell, std::sqrt(op.K.s2), op.K.a, op.K.b, op.K.even};
  assemble_dense_dev(kk, op.X.p, n, op.X.p, n, op.d, op.G > 0, true, 0.0, Mell.p, N, s);
  a.upload(alpha_h, static_cast<size_t>(N), s);
  // t = Mell a; data_ell = a·t; tr_ell = Σ Kinv ⊙ Mell
  rows_gemm_dev(Mell.p, int(N), a.p, 1, N, t.p, false, s);  // Mell symmetric: row r · a
  col_dots_dev(a.p, t.p, N, 1, dots.p + 0, part, s);
  col_dots_dev(Kinv.p, Mell.p, N * N, 1, dots.p + 1, part, s);
  // Ka = (K − noise) a = A a − nd ⊙ a
  rows_gemm_dev(op.A.p, int(N), a.p, 1, N, t.p, false, s);
  col_dots_dev(a.p, t.p, N, 1, dots.p + 2, part, s);
  std::vector<double> dh(3), diag(static_cast<size_t>(N)), ah(alpha_h, alpha_h + N);
  GK_CUDA(cudaMemcpyAsync(dh.data(), dots.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), Kinv.p, sizeof(double) * (N + 1), sizeof(double), N,
                            cudaMemcpyDeviceToHost, s));
  GK_CUDA(cudaStreamSynchronize(s));
  const double sv2 = op.nv2, sg2 = op.ng2;
  double aKa = dh[2];
  for (i64 r = 0; r < N; ++r) aKa -= (r < n ? sv2 : sg2) * ah[static_cast<size_t>(r)] * ah[static_cast<size_t>(r)];
  double dnd = 0.0, trh = 0.0, trt = 0.0, ah2 = 0.0, at2 = 0.0;
  for (i64 r = 0; r < N; ++r) {
    const double kd = diag[static_cast<size_t>(r)];
    dnd += kd * (r < n ? sv2 : sg2);
    if (r < n) {
      trh += kd;
      ah2 += ah[static_cast<size_t>(r)] * ah[static_cast<size_t>(r)];
    } else {
      trt += kd;
      at2 += ah[static_cast<size_t>(r)] * ah[static_cast<size_t>(r)];
    }
  }
  grad[0] = 0.5 * (dh[0] - dh[1]);
  grad[1] = 0.5 * (2.0 * aKa - 2.0 * (double(N) - dnd));
  grad[2] = 0.5 * (2.0 * sv2 * ah2 - 2.0 * sv2 * trh);
  *nparams = op.G > 0 ? 4 : 3;
  if (op.G > 0) grad[3] = 0.5 * (2.0 * sg2 * at2 - 2.0 * sg2 * trt);
}

std::unique_ptr<Op> make_dense(const double* A, i64 N, int device) {
  if (N < 1) fail(GK_ERR_ARG, "dense operator needs N >= 1");
  DeviceGuard dg(device);
  auto op = std::make_unique<DenseOp>();
  op->kind = KIND_DENSE;
  op->device = device;
  op->N = N;
  op->n_value = N;
  op->init_stream();
  op->A.upload(A, static_cast<size_t>(N) * N, op->stream);
  GK_CUDA(cudaStreamSynchronize(op->stream));
  return op;
}

}  // namespace gk
