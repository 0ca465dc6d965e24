// kuu_fft.cu — K_UU = T(κ) for a general stationary profile κ (e.g. the
// spline kernel, kernels.cpp:104-118) on a d ≤ 3 grid, by circulant
// embedding (reference GridKernelOperator, dski.cpp:80-172):
//   w = corner( IFFT( spec · FFT( zero-padded u ) ) ).
// The embedding is the power of two E_j ≥ 2m_j − 1 per axis (the reference
// takes 2(m_j − 1) for FFTW; any E_j ≥ 2m_j − 1 reproduces the same linear
// convolution exactly, and powers of two let one radix-2 kernel serve every
// axis). Right-hand sides go two at a time as the real and imaginary parts
// of one complex field (the spectrum of an even profile slice is real).
//
// FFT: one kernel per axis, a CTA transforms TI lines in shared memory
// (bit-reversed load, log2 E radix-2 butterfly stages, natural-order store);
// for the strided axes the TI lines are adjacent in memory so every load row
// is one coalesced 16·TI-byte segment.
#include <cmath>

#include "kuu_fft.hpp"

namespace gk {

namespace {

constexpr int FFT_THREADS = 256;
constexpr size_t kFftSmem = 64 * 1024;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Lines of one axis pass. A line is (pair p, indices i_k of the axes k < j,
// inner index i over the axes k > j); element t of the line lives at
// p·Etot + Σ_{k<j} i_k·stride_k + t·S + i (S = Π_{k>j} E_k). The axes
// before j are restricted to i_k < lim_k: forward passes run last axis
// first, so those axes still hold the zero-padded input (support m_k);
// inverse passes run first axis first and only the corner i_k < m_k of the
// result is needed. `support` > 0: entries t ≥ support of the line are the
// zero padding and are not read. TI lines per CTA: S == 1 — TI whole lines;
// S > 1 — TI lines adjacent in memory (same outer index, TI | S).
struct AxisPass {
  int L, logL, TI, support, inverse;
  const double* spec;  // non-null: forward FFT, × spec, inverse FFT in one pass (axis 0)
  i64 S, nlines, Etot;
  int j, lim0, lim1;
  i64 st0, st1;  // strides of axes 0 and 1 (elements)
};

__global__ void __launch_bounds__(FFT_THREADS) k_fft_lines(double2* __restrict__ buf, AxisPass a,
                                                           const double2* __restrict__ tw) {
  extern __shared__ double2 sx[];  // [TI][L]
  const int L = a.L, TI = a.TI;
  const i64 g0 = (i64)blockIdx.x * TI;
  const int tid = threadIdx.x;
  auto base = [&](i64 g) -> i64 {
    i64 i = 0, o = g;
    if (a.S > 1) {
      i = g % a.S;
      o = g / a.S;
    }
    i64 off = i;
    if (a.j >= 2) {
      off += (o % a.lim1) * a.st1;
      o /= a.lim1;
    }
    if (a.j >= 1) {
      off += (o % a.lim0) * a.st0;
      o /= a.lim0;
    }
    return o * a.Etot + off;
  };
  const int shift = 32 - a.logL;
  const int sup = a.support > 0 ? a.support : L;
  for (int e = tid; e < TI * L; e += FFT_THREADS) {
    int c, t;
    if (a.S == 1) {
      c = e / L;
      t = e - c * L;
    } else {
      t = e / TI;
      c = e - t * TI;
    }
    const i64 g = g0 + c;
    double2 v = make_double2(0.0, 0.0);
    if (g < a.nlines && t < sup) v = buf[base(g) + (i64)t * a.S];
    const int rt = a.logL ? int(__brev(unsigned(t)) >> shift) : 0;
    sx[c * L + rt] = v;
  }
  __syncthreads();
  const int halfL = L >> 1;
  // radix-2 DIT stages, two at a time in registers (a thread owns the four
  // elements the two stages combine: the same butterflies in the same order
  // as stage-by-stage, half the shared-memory passes and barriers)
  auto stages = [&](int inverse) {
    const double sg = inverse ? -1.0 : 1.0;
    int s = 1;
    if (a.logL & 1) {  // one single stage first when log2 L is odd
      for (int e = tid; e < TI * halfL; e += FFT_THREADS) {
        const int c = e / halfL, jj = e - c * halfL;
        const int i1 = 2 * jj, i2 = i1 + 1;
        const double2 x = sx[c * L + i1], y = sx[c * L + i2];
        sx[c * L + i1] = make_double2(x.x + y.x, x.y + y.y);
        sx[c * L + i2] = make_double2(x.x - y.x, x.y - y.y);
      }
      __syncthreads();
      s = 2;
    }
    const int quarterL = L >> 2;
    for (; s + 1 <= a.logL; s += 2) {
      const int h = 1 << (s - 1);
      const int ts1 = L >> s, ts2 = L >> (s + 1);
      for (int e = tid; e < TI * quarterL; e += FFT_THREADS) {
        const int c = e / quarterL, jj = e - c * quarterL;
        const int pos = jj & (h - 1), grp = jj >> (s - 1);
        const int i0 = grp * 4 * h + pos;
        double2* row = sx + c * L;
        const double2 a0 = row[i0], a1 = row[i0 + h], a2 = row[i0 + 2 * h], a3 = row[i0 + 3 * h];
        double2 w1 = __ldg(tw + pos * ts1), w2 = __ldg(tw + pos * ts2), w3 = __ldg(tw + (pos + h) * ts2);
        w1.y *= sg;
        w2.y *= sg;
        w3.y *= sg;
        const double2 t1 = cmul(w1, a1), t3 = cmul(w1, a3);
        const double2 b0 = make_double2(a0.x + t1.x, a0.y + t1.y), b1 = make_double2(a0.x - t1.x, a0.y - t1.y);
        const double2 b2 = make_double2(a2.x + t3.x, a2.y + t3.y), b3 = make_double2(a2.x - t3.x, a2.y - t3.y);
        const double2 u2 = cmul(w2, b2), u3 = cmul(w3, b3);
        row[i0] = make_double2(b0.x + u2.x, b0.y + u2.y);
        row[i0 + 2 * h] = make_double2(b0.x - u2.x, b0.y - u2.y);
        row[i0 + h] = make_double2(b1.x + u3.x, b1.y + u3.y);
        row[i0 + 3 * h] = make_double2(b1.x - u3.x, b1.y - u3.y);
      }
      __syncthreads();
    }
  };
  stages(a.inverse);
  if (a.spec) {
    // pointwise spectrum multiply (element t of line g sits at spectrum index
    // t·S + inner, the field's own offset), bit-reversal permutation in place,
    // then the inverse transform of the same line
    for (int e = tid; e < TI * L; e += FFT_THREADS) {
      const int c = e / L, t = e - c * L;
      const i64 g = g0 + c;
      if (g < a.nlines) {
        const i64 inner = a.S > 1 ? g % a.S : 0;
        const double sc = __ldg(a.spec + (i64)t * a.S + inner);
        sx[e] = make_double2(sx[e].x * sc, sx[e].y * sc);
      }
    }
    __syncthreads();
    for (int e = tid; e < TI * L; e += FFT_THREADS) {
      const int c = e / L, t = e - c * L;
      const int rt = a.logL ? int(__brev(unsigned(t)) >> shift) : 0;
      if (t < rt) {
        const double2 x = sx[c * L + t];
        sx[c * L + t] = sx[c * L + rt];
        sx[c * L + rt] = x;
      }
    }
    __syncthreads();
    stages(1);
  }
  for (int e = tid; e < TI * L; e += FFT_THREADS) {
    int c, t;
    if (a.S == 1) {
      c = e / L;
      t = e - c * L;
    } else {
      t = e / TI;
      c = e - t * TI;
    }
    const i64 g = g0 + c;
    if (g < a.nlines) buf[base(g) + (i64)t * a.S] = sx[c * L + t];
  }
}

struct Dims3 {
  int m[3], E[3];
};

// zero-padded complex field of RHS pair p: corner node (i0, i1, i2) gets
// u[node][2p] + i·u[node][2p+1]
__global__ void k_fft_load(const double* __restrict__ U, int nrhs, int npairs, Dims3 g, i64 M, i64 Etot,
                           double2* __restrict__ buf) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < M * npairs; e += (i64)gridDim.x * blockDim.x) {
    const int p = int(e / M);
    const i64 node = e - (i64)p * M;
    const int i2 = int(node % g.m[2]);
    const i64 r = node / g.m[2];
    const int i1 = int(r % g.m[1]), i0 = int(r / g.m[1]);
    const i64 ei = ((i64)i0 * g.E[1] + i1) * g.E[2] + i2;
    const int c = 2 * p;
    const double re = U[node * nrhs + c];
    const double im = c + 1 < nrhs ? U[node * nrhs + c + 1] : 0.0;
    buf[(i64)p * Etot + ei] = make_double2(re, im);
  }
}

__global__ void k_fft_store(const double2* __restrict__ buf, int nrhs, int npairs, Dims3 g, i64 M, i64 Etot,
                            double* __restrict__ W) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < M * npairs; e += (i64)gridDim.x * blockDim.x) {
    const int p = int(e / M);
    const i64 node = e - (i64)p * M;
    const int i2 = int(node % g.m[2]);
    const i64 r = node / g.m[2];
    const int i1 = int(r % g.m[1]), i0 = int(r / g.m[1]);
    const i64 ei = ((i64)i0 * g.E[1] + i1) * g.E[2] + i2;
    const double2 v = buf[(i64)p * Etot + ei];
    const int c = 2 * p;
    W[node * nrhs + c] = v.x;
    if (c + 1 < nrhs) W[node * nrhs + c + 1] = v.y;
  }
}

__global__ void k_fft_real_part(const double2* __restrict__ buf, i64 n, double scale, double* __restrict__ out) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x)
    out[e] = buf[e].x * scale;
}

unsigned blocks_of(i64 n) { return static_cast<unsigned>(std::min<i64>((n + 255) / 256, 148 * 32)); }

// All axes of npairs fields, forward (inverse = 0: last axis first, input
// supported on the corner i_k < m_k when `pruned`) or inverse (first axis
// first, only the corner of the result kept when `pruned`); no scaling.
// mode 0 forward, 1 inverse, 2 convolve: forward along axes 2, 1, then axis 0
// forward × spectrum × inverse in one pass, then inverse along axes 1, 2.
void fft_all_axes(const KuuFft& f, double2* buf, int npairs, int mode, bool pruned, cudaStream_t s) {
  const int nsteps = mode == 2 ? 5 : 3;
  for (int step = 0; step < nsteps; ++step) {
    int j, inverse = mode == 1;
    const double* spec = nullptr;
    if (mode == 2) {
      j = step < 3 ? 2 - step : step - 2;  // 2, 1, 0 (conv), 1, 2
      inverse = step > 2;
      if (step == 2) spec = f.spec.p;
    } else {
      j = inverse ? step : 2 - step;
    }
    const int L = f.E[j];
    if (L < 2) continue;
    AxisPass a{};
    a.spec = spec;
    a.L = L;
    a.logL = f.logE[j];
    a.inverse = inverse;
    a.j = j;
    a.Etot = f.Etot;
    a.S = 1;
    for (int k = j + 1; k < 3; ++k) a.S *= f.E[k];
    a.st0 = i64(f.E[1]) * f.E[2];
    a.st1 = f.E[2];
    a.lim0 = pruned ? f.m[0] : f.E[0];
    a.lim1 = pruned ? f.m[1] : f.E[1];
    a.support = pruned && !inverse ? f.m[j] : 0;  // (the convolve pass reads the forward input: pruned support)
    i64 outer = npairs;
    if (j >= 1) outer *= a.lim0;
    if (j >= 2) outer *= a.lim1;
    a.nlines = outer * a.S;
    if (a.S == 1) a.TI = std::max(1, int(kFftSmem / (sizeof(double2) * L)));
    else a.TI = int(std::min<i64>(a.S, std::max<i64>(1, std::min<i64>(16, kFftSmem / (sizeof(double2) * L)))));
    const size_t smem = sizeof(double2) * size_t(a.TI) * L;
    raise_smem_limit((const void*)k_fft_lines, smem);
    k_fft_lines<<<static_cast<unsigned>((a.nlines + a.TI - 1) / a.TI), FFT_THREADS, smem, s>>>(buf, a, f.tw[j].p);
    launched("kuu fft axis");
  }
}

}  // namespace

void KuuFft::init(int dd, const int* dims) {
  d = dd;
  M = 1;
  Etot = 1;
  for (int j = 0; j < 3; ++j) {
    m[j] = j < d ? dims[j] : 1;
    int e = 1, lg = 0;
    if (j < d)
      while (e < 2 * m[j] - 1) {
        e <<= 1;
        ++lg;
      }
    if (e > 8192) fail(GK_ERR_UNSUPPORTED, "grid too large for the circulant-embedding K_UU (E > 8192 per axis)");
    E[j] = e;
    logE[j] = lg;
    M *= m[j];
    Etot *= e;
  }
}

void KuuFft::build(const std::vector<double>& slice, cudaStream_t s) {
  if (static_cast<i64>(slice.size()) != Etot) fail(GK_ERR_ARG, "profile slice size mismatch");
  for (int j = 0; j < 3; ++j) {
    const int L = E[j];
    std::vector<double2> t(static_cast<size_t>(std::max(1, L / 2)));
    for (int k = 0; k < L / 2; ++k) {
      const long double a = -2.0L * 3.14159265358979323846264338327950288L * k / L;
      t[static_cast<size_t>(k)] = make_double2(double(cosl(a)), double(sinl(a)));
    }
    tw[j].upload(t.data(), t.size(), s);
    GK_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<double2> z(static_cast<size_t>(Etot));
  for (i64 e = 0; e < Etot; ++e) z[static_cast<size_t>(e)] = make_double2(slice[static_cast<size_t>(e)], 0.0);
  buf.reserve(static_cast<size_t>(Etot));
  GK_CUDA(cudaMemcpyAsync(buf.p, z.data(), sizeof(double2) * Etot, cudaMemcpyHostToDevice, s));
  fft_all_axes(*this, buf.p, 1, 0, false, s);
  // the slice is even in every axis, so its spectrum is real; the imaginary
  // parts are roundoff and are dropped (as dski.cpp:127-131 does)
  spec.alloc(static_cast<size_t>(Etot));
  k_fft_real_part<<<blocks_of(Etot), 256, 0, s>>>(buf.p, Etot, 1.0 / double(Etot), spec.p);
  launched("kuu fft spectrum");
  GK_CUDA(cudaStreamSynchronize(s));
}

void KuuFft::apply(const double* U, double* W, int nrhs, cudaStream_t s) const {
  const int npairs = (nrhs + 1) / 2;
  buf.reserve(static_cast<size_t>(Etot) * npairs);
  Dims3 g{{m[0], m[1], m[2]}, {E[0], E[1], E[2]}};
  // no zero fill: the pruned forward passes read only the corner they wrote
  k_fft_load<<<blocks_of(M * npairs), 256, 0, s>>>(U, nrhs, npairs, g, M, Etot, buf.p);
  launched("kuu fft load");
  fft_all_axes(*this, buf.p, npairs, 2, true, s);
  k_fft_store<<<blocks_of(M * npairs), 256, 0, s>>>(buf.p, nrhs, npairs, g, M, Etot, W);
  launched("kuu fft store");
}

std::vector<double> slice_from_reference(const KuuFft& f, const std::vector<double>& slice_ref) {
  int Er[3] = {1, 1, 1};
  i64 tot_ref = 1;
  for (int j = 0; j < f.d; ++j) {
    Er[j] = 2 * (f.m[j] - 1);
    tot_ref *= Er[j];
  }
  if (static_cast<i64>(slice_ref.size()) != tot_ref) fail(GK_ERR_ARG, "profile slice size mismatch");
  std::vector<double> out(static_cast<size_t>(f.Etot), 0.0);
  int idx[3] = {0, 0, 0};
  for (i64 t = 0; t < f.Etot; ++t) {
    bool in = true;
    i64 r = 0;
    for (int j = 0; j < f.d; ++j) {
      const int w = f.wrap(j, idx[j]);
      if (w > f.m[j] - 1 || w < -(f.m[j] - 1)) in = false;
      r = r * Er[j] + (w >= 0 ? w : Er[j] + w);
    }
    if (in) out[static_cast<size_t>(t)] = slice_ref[static_cast<size_t>(r)];
    for (int j = f.d - 1; j >= 0; --j) {
      if (++idx[j] < f.E[j]) break;
      idx[j] = 0;
    }
  }
  return out;
}

// GridKernelOperator(grid, profile) (dski.cpp:80-172) at the boundary: the
// caller's profile evaluated on the reference embedding (what dski.cpp:97-114
// computes from the StationaryProfile callback), applied by the FFT route.
struct GridKernelOp final : Op {
  KuuFft f;
  std::vector<double> slice_ref;
  int dims[3] = {1, 1, 1};
  void mvm(const double* in, double* out, int nrhs, cudaStream_t s) override { f.apply(in, out, nrhs, s); }
  void diagonal(double* dd, cudaStream_t s) override {
    std::vector<double> h(static_cast<size_t>(N), slice_ref[0]);  // κ(0) on every node
    GK_CUDA(cudaMemcpyAsync(dd, h.data(), sizeof(double) * N, cudaMemcpyHostToDevice, s));
    GK_CUDA(cudaStreamSynchronize(s));
  }
  void row(i64 r, double* out, cudaStream_t s) override {
    if (r < 0 || r >= N) fail(GK_ERR_RANGE, "grid kernel row index out of range");
    DevBuf<double> e(static_cast<size_t>(N));
    GK_CUDA(cudaMemsetAsync(e.p, 0, sizeof(double) * N, s));
    const double one = 1.0;
    GK_CUDA(cudaMemcpyAsync(e.p + r, &one, sizeof(double), cudaMemcpyHostToDevice, s));
    f.apply(e.p, out, 1, s);
    GK_CUDA(cudaStreamSynchronize(s));
  }
};

std::unique_ptr<Op> make_grid_kernel(int d, const int* dims, const double* slice_ref, int device) {
  if (d < 1 || d > 3) fail(GK_ERR_UNSUPPORTED, "grid kernel operator supports 1 <= d <= 3");
  i64 tot = 1;
  for (int j = 0; j < d; ++j) {
    if (dims[j] < 2) fail(GK_ERR_ARG, "grid needs at least 2 nodes per dimension");
    tot *= 2 * (dims[j] - 1);
  }
  DeviceGuard dg(device);
  auto op = std::make_unique<GridKernelOp>();
  op->kind = KIND_GRID;
  op->device = device;
  op->f.init(d, dims);
  op->N = op->f.M;
  op->n_value = op->N;
  for (int j = 0; j < d; ++j) op->dims[j] = dims[j];
  op->slice_ref.assign(slice_ref, slice_ref + tot);
  op->init_stream();
  op->f.build(slice_from_reference(op->f, op->slice_ref), op->stream);
  return op;
}

double grid_kernel_min_eig(const Op& o) {
  if (o.kind != KIND_GRID) fail(GK_ERR_ARG, "operator is not a grid kernel operator");
  const auto& g = static_cast<const GridKernelOp&>(o);
  return min_embedding_eigenvalue_host(g.f.d, g.dims, g.slice_ref);
}

double min_embedding_eigenvalue_host(int d, const int* dims, const std::vector<double>& slice) {
  // embedding 2(m_j − 1) per axis (dski.cpp:89-95), slice row-major; the
  // even slice's DFT along each axis is a cosine sum (separable)
  int E[3] = {1, 1, 1};
  i64 tot = 1;
  for (int j = 0; j < d; ++j) {
    E[j] = 2 * (dims[j] - 1);
    tot *= E[j];
  }
  if (static_cast<i64>(slice.size()) != tot) fail(GK_ERR_ARG, "embedding slice size mismatch");
  std::vector<long double> a(slice.begin(), slice.end()), b(static_cast<size_t>(tot));
  for (int j = 0; j < d; ++j) {
    const int L = E[j];
    i64 S = 1;
    for (int k = j + 1; k < d; ++k) S *= E[k];
    std::vector<long double> c(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) c[static_cast<size_t>(k)] = cosl(2.0L * 3.14159265358979323846264338327950288L * k / L);
    for (i64 e = 0; e < tot; ++e) {
      const i64 o = e / (S * L), i = e % S;
      const int kk = int((e / S) % L);
      long double acc = 0.0L;
      for (int t = 0; t < L; ++t)
        acc += a[static_cast<size_t>(o * L * S + i + (i64)t * S)] * c[static_cast<size_t>((i64(kk) * t) % L)];
      b[static_cast<size_t>(e)] = acc;
    }
    a.swap(b);
  }
  long double mn = a[0];
  for (const long double v : a) mn = std::min(mn, v);
  return double(mn);
}

}  // namespace gk
