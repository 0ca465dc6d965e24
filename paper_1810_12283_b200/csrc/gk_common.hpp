// gk_common.hpp — shared infrastructure of libgk_b200: error mapping,
// device buffers, launch accounting, the device-operator base class.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gk_capi.h"

namespace gk {

using i64 = std::int64_t;

struct Error : std::runtime_error {
  gk_status code;
  i64 point;
  Error(gk_status c, const std::string& m, i64 p = -1) : std::runtime_error(m), code(c), point(p) {}
};

[[noreturn]] inline void fail(gk_status c, const std::string& msg, i64 point = -1) {
  throw Error(c, msg, point);
}

void cuda_check(cudaError_t e, const char* what);
// Raise (never lower) a kernel's dynamic shared-memory limit: the attribute is
// per function and shared by every plan/operator launching it.
void raise_smem_limit(const void* fn, size_t bytes);
#define GK_CUDA(x) ::gk::cuda_check((x), #x)

// Process-wide kernel-variant knobs (gk_set_tuning); 0 = default.
struct Tuning {
  std::atomic<int> scatter{0}, gather{0}, toeplitz{0}, precond{0}, fused{0}, fused_prof{0}, pcg_fused{0};
  std::atomic<int> devbuild{0};  // 1 = D-SKI point tables built on the host
  std::atomic<int> pivchol{0};  // 1 = host-synchronised pivot loop (3 syncs per pivot)
  std::atomic<int> lean{0};  // lean one-launch 2-D MVM (lean2d.cu): 0 measured policy, 1 never, 2 always
  // fused 2-D MVM decomposition overrides (0 = heuristic)
  std::atomic<int> f2_stc{0}, f2_sl{0}, f2_gtc{0}, f2_gl{0}, f2_tsplit{0}, f2_per_sm{0};
  std::atomic<int> f2_twide{-1};  // one-launch 2-D MVM Toeplitz 16-column items (-1 auto, 0 off, 1 on)  // one-launch 2-D MVM direct gather: RHS per task (4, 8; 0 = plan's RP)
  std::atomic<int> f2_warm{-1};  // one-launch 2-D MVM warm-up passes (bitmask; -1 = default)
  std::atomic<int> f2_skip{0};  // debug: bitmask of phases to skip (1 S, 2 T1, 4 T0, 8 G)
  std::atomic<int> f2_grid{0}, f2_rp{0};
  std::atomic<int> f2_smode{0}, f2_gmode{0};  // 1 staged, 2 direct (0 = default)
  std::atomic<int> f2_nspl{0}, f2_nst{0};
  std::atomic<int> e2e_chunk{0};
  std::atomic<int> e2e_stage{0};  // 1 = pageable host buffers go straight to cudaMemcpyAsync (driver staging)
  // d = 3 MVM A/B bitmask (0 = the measured default; each bit restores the variant it replaced):
  //   1 list-walk merge (k_scatter_merge3), 2 r-fastest gather tasks, 4 CTA-staged push for few RHS,
  //   8 non-persistent Toeplitz modes for M <= 48, 512 runtime RHS count in the gather, 1024 lean
  //   gather, 2048 direct (unstaged) push for few RHS, 4096 one node column per merge CTA, 8192 32-column
  //   Toeplitz tiles at small column counts, 16384 CTA-per-unit gather for few RHS
  std::atomic<int> d3{0};
  // D-SKIP Hadamard kernels: 0 = TMA-ring DMMA (v3, falling back to v2 for odd
  // sizes), 3 = cp.async DMMA (v2), 1 = first generation
  std::atomic<int> dskip{0};
  std::atomic<int> lanczos{0};  // 1 = per-step host-synchronised Lanczos (reference order)
  std::atomic<int> rng{0};      // 1 = SLQ probes generated on the host (else on the device, same streams)
  std::atomic<int> dskip_e{0};  // v3 expand ring: 0 = 8 m × 4 stages, 1 = 16 × 2, 2 = 16 × 4, 3 = 32 × 2
  std::atomic<int> gen{0};  // bumped by every gk_set_tuning call (cached plans rebuild)
};
extern Tuning g_tuning;

// Every kernel launch goes through this so the library can report how many of
// its own kernels ran (bench.py's gpu_launches, smoke()).
extern std::atomic<i64> g_launches;
inline void launched(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cuda_check(cudaGetLastError(), what);
}

// Owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) GK_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  // grow-only reallocation for scratch
  void reserve(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t s = nullptr) {
    reserve(count);
    if (count) GK_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  T* get() const { return p; }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    GK_CUDA(cudaGetDevice(&prev));
    if (prev != dev) GK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Pinned host staging buffer.
struct HostBuf {
  double* p = nullptr;
  size_t n = 0;
  void reserve(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    GK_CUDA(cudaMallocHost(&p, count * sizeof(double)));
    n = count;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

// ---------------------------------------------------------------- host math
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream);
void rademacher(i64 n, std::uint64_t seed, std::uint64_t stream, double* out);
void gaussian(i64 n, std::uint64_t seed, std::uint64_t stream, double* out);
void uniform(i64 n, std::uint64_t seed, std::uint64_t stream, double a, double b, double* out);
// Tridiagonal eigendecomposition, ascending; Z is n×n col-major (may be null
// for values only).
void tridiag_eig(int n, const double* alpha, const double* beta, double* evals, double* Z);
// Dense small Cholesky (upper R, R^T R = A, col-major k×k). Throws on failure.
void cholesky_upper(int k, const double* A, double* R);

// ---------------------------------------------------------------- operators
enum OpKind { KIND_EXACT = 0, KIND_DSKI = 1, KIND_DSKIP = 2, KIND_DENSE = 3, KIND_GRID = 4 };

// Device operator behind gk_op. All compute entry points work on the
// INTERNAL layout: rows in the operator's internal order (D-SKI sorts points
// by stencil cell; others keep the external order), right-hand sides
// innermost ("RHS-minor": element (r, b) at r*nrhs + b).
std::uint64_t next_op_uid();

struct PcgVecPlan;
struct PcgVecArgs;

struct Op {
  Op() : uid(next_op_uid()) {}
  virtual ~Op();
  const std::uint64_t uid;  // identifies the internal row order (never reused)
  int kind = 0;
  int device = 0;
  i64 N = 0;            // logical size
  i64 n_value = 0;      // rows [0, n_value) carry sigma_1^2, the rest sigma_2^2
  double nv2 = 0.0, ng2 = 0.0;
  std::mutex mu;        // serialises host-API calls that use the scratch below
  // Recorded at the end of every C-ABI call on the stream that call used; the
  // next call (any stream: op.stream or a caller's) waits on it first, so
  // device work of successive calls that share op-owned scratch, plans and
  // grid-barrier counters never overlaps (OpSession in capi.cu).
  cudaEvent_t last_use = nullptr;
  cudaStream_t stream = nullptr;  // own stream for host-API calls
  cudaStream_t cap_stream = nullptr;  // private stream used only for CUDA-graph capture
  DevBuf<double> scratch_a, scratch_b, scratch_c;
  // Lanczos / SLQ workspace (grow-only; cudaMalloc/cudaFree of the N×P×steps
  // basis per call cost more than the steps themselves)
  DevBuf<double> lz_ws, slq_z;
  HostBuf slq_h;  // pinned probe staging
  DevBuf<int> lz_wsi;
  HostBuf pinned;
  // PCG workspace, fused-step plan and instantiated iteration graph, reused
  // across solves (solvers.cu PcgCache; type-erased here)
  std::shared_ptr<void> pcg_cache;
  // host-buffer MVM pipeline (gk_op_mvm): copy-in / compute / copy-out streams
  cudaStream_t io_in = nullptr, io_out = nullptr, io_pin = nullptr, io_pout = nullptr;
  std::vector<cudaEvent_t> io_events;
  DevBuf<double> io_ext_in, io_int_in, io_int_out, io_ext_out;
  HostBuf io_pin_in, io_pin_out;  // pinned staging for pageable caller buffers

  virtual void mvm(const double* in, double* out, int nrhs, cudaStream_t s) = 0;
  // diagonal including noise, internal order
  virtual void diagonal(double* d, cudaStream_t s) = 0;
  // row r (EXTERNAL index) including noise, written in internal order
  virtual void row(i64 r_ext, double* out, cudaStream_t s) = 0;
  // Row *d_r_int (INTERNAL index, read from device memory) written in
  // internal order, skipped when *d_active == 0; false = not implemented
  // (callers then use row() with a host round trip).
  virtual bool row_dev(const i64* /*d_r_int*/, const int* /*d_active*/, double* /*out*/, cudaStream_t) {
    return false;
  }
  virtual bool has_row_dev() const { return false; }
  // internal row index -> external row index (device array or null = identity)
  virtual const i64* d_ext_of_int() const { return nullptr; }
  // Persistent PCG (MVM + fused vector step in one cooperative launch, up to
  // `iters` iterations); false when this operator has no such path.
  virtual bool pcg_persist(PcgVecPlan&, const PcgVecArgs&, double* /*P*/, double* /*AP*/, int /*nrhs*/,
                           int /*iters*/, cudaStream_t) {
    return false;
  }
  virtual i64 int_of_ext(i64 r) const { return r; }
  virtual void stage(int st, const double* in, double* out, int nrhs, cudaStream_t s);

  // Whole MVM replayed from a cached CUDA graph (captured once per
  // (in, out, nrhs)): one launch instead of one per kernel.
  void mvm_graph(const double* in, double* out, int nrhs, cudaStream_t s);
  struct GraphEntry {
    const double* in;
    double* out;
    int nrhs;
    cudaGraphExec_t exec;
    i64 nodes;
    std::uint64_t epoch;
  };
  // Bumped whenever scratch memory or launch plans a captured graph may
  // reference are reallocated; cached graphs from older epochs are dropped.
  std::uint64_t epoch = 0;
  std::vector<GraphEntry> graphs;

  void to_internal(const double* V, i64 ldv, double* I, int nrhs, cudaStream_t s) const;
  void from_internal(const double* I, double* V, i64 ldv, int nrhs, cudaStream_t s) const;
  void init_stream();
};

// Blocked host-API MVM helper: copies host blocks in/out through pinned
// memory in chunks of at most kMaxRhs columns.
constexpr int kMaxRhs = 64;

// ---------------------------------------------------------------- reductions
// Deterministic column reductions over RHS-minor blocks (rows × nrhs).
constexpr int kRedBlocks = 296;  // 2 × 148 SMs
constexpr int kRedThreads = 256;

}  // namespace gk

struct gk_op {
  std::unique_ptr<gk::Op> impl;
};
