// ops.cu — layout conversion shared by all device operators, plus the two
// non-structured operators: the matrix-free exact D-SE operator (the dense
// K∇ of reference kernels.cpp:242-285, never materialised) and an explicit
// dense operator (linear_operator.hpp:38-56) used by solver tests.
#include <cmath>

#include "gk_kernels.cuh"

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
struct DenseOp final : Op {
  DevBuf<double> A;
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
