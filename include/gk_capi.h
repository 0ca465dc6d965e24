/* gk_capi.h — C-ABI of the B200 gradkrig hot path (libgk_b200.so).
 *
 * Drop-in boundary for the reference's core operator/solver API
 * (reference: proj/core/include/gradkrig/{linear_operator,dski,dskip,linalg}.hpp,
 * SPEC.md modules dski/dskip/linalg). Plain pointers and sizes only; no torch,
 * Eigen or CUDA types in the signatures (streams are passed as void*).
 *
 * Conventions (same as the reference):
 *   - X is n×d column-major (Eigen default; X.col(j) contiguous).
 *   - Operator vectors are derivative-type-major [f; d_1 f; ...; d_d f]
 *     (reference kernels.hpp:94-97, observations.hpp:27-35).
 *   - Multi-RHS blocks are column-major N×nrhs with leading dimension ld.
 *   - Host pointers are borrowed for the duration of the call. Handles own
 *     their device memory and are freed by gk_*_destroy.
 *   - Every entry returns a gk_status; gk_last_error() gives the message
 *     (thread-local). Handles are immutable after creation and the const
 *     entry points are safe to call from several host threads (each call
 *     takes the handle's scratch under a mutex, like the reference's FFTW
 *     planner lock dski.cpp:14-17, and runs on its own stream).
 *   - Entry points with the _dev suffix take device pointers and a CUDA
 *     stream (cudaStream_t passed as void*; NULL = legacy default stream) and
 *     are asynchronous with respect to the host.
 */
#ifndef GK_CAPI_H
#define GK_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; each maps to the reference exception named. */
typedef enum {
  GK_OK = 0,
  GK_ERR_ARG = 1,         /* std::invalid_argument (e.g. dski.cpp:230, linalg.cpp:180-181) */
  GK_ERR_RANGE = 2,       /* std::out_of_range (dski.cpp:293, dskip.cpp:260)               */
  GK_ERR_OUT_OF_GRID = 3, /* gradkrig::OutOfGridError (interpolation.cpp:90-95)            */
  GK_ERR_RUNTIME = 4,     /* std::runtime_error (linalg.cpp:165-167, gp.cpp:151-156)       */
  GK_ERR_LOGIC = 5,       /* std::logic_error (linear_operator.cpp:7-13)                   */
  GK_ERR_LENGTH = 6,      /* std::length_error (kernels.cpp:252-255)                       */
  GK_ERR_CUDA = 7,        /* CUDA runtime failure (no reference equivalent)                */
  GK_ERR_NCCL = 8,
  GK_ERR_UNSUPPORTED = 9  /* configuration the B200 path does not implement (reported, never
                             silently routed elsewhere)                                     */
} gk_status;

const char* gk_last_error(void);
/* Index of the offending point after GK_ERR_OUT_OF_GRID, else -1. */
int64_t gk_last_error_point(void);
const char* gk_version(void);
/* Kernel-variant selection for tuning/A-B timing (process-wide). Keys:
 * "scatter", "gather", "toeplitz", "precond" (0 = default choice), "fused"
 * (1 = disable the one-launch 2-D MVM), "pcg_fused" (0/1 = one-launch PCG
 * vector step where supported, 2 = separate kernels, 3 = vector step v1,
 * 5 = persistent MVM + vector step for the 2-D D-SKI operator), "dskip" (D-SKIP Hadamard
 * kernels: 0 = TMA-ring DMMA, 3 = cp.async DMMA, 1 = first generation),
 * "e2e_chunk" (gk_op_mvm host-buffer pipeline chunk, 0 = auto), "e2e_stage"
 * (1 = pageable caller buffers go straight to cudaMemcpyAsync instead of the
 * pinned staging of the host copy pool), "d3" (bitmask restoring earlier d = 3
 * MVM variants, see gk_common.hpp), "fused_prof" and "f2_*" decomposition
 * overrides. Returns the old value. */
int gk_set_tuning(const char* key, int value);
/* Number of CUDA kernels this library has launched in this process. */
int64_t gk_kernel_launch_count(void);

/* ---------------------------------------------------------------- kernel spec
 * KernelSpec (reference kernels.hpp:42-75). family 0 = squared exponential,
 * 1 = spline (kernels.cpp:104-118). D-SKI takes either: the separable SE
 * profile runs as Kronecker–Toeplitz mode products, the spline profile as a
 * circulant embedding with an in-house FFT (dski.cpp:80-172). D-SKIP needs a
 * separable kernel (GK_ERR_ARG for spline, std::invalid_argument at
 * dskip.cpp:118-121); the matrix-free exact operator takes both. */
typedef struct {
  int family;
  double lengthscale;
  double outputscale;
  double spline_a, spline_b;
  int spline_even;
} gk_kernel;

/* Grid (reference interpolation.hpp:13-35); dims/origin/spacing length d. */
typedef struct {
  int d;
  int dims[8];
  double origin[8];
  double spacing[8];
} gk_grid;

/* Grid::cover (interpolation.cpp:117-146). Host-only. */
gk_status gk_grid_cover(const double* X, int64_t n, int d, double target_spacing,
                        int margin_cells, int max_nodes, gk_grid* out);

/* rng.hpp:12-38 (host; identical streams to the reference's libstdc++ build). */
uint64_t gk_mix_seed(uint64_t seed, uint64_t stream);
void gk_rademacher_vector(int64_t n, uint64_t seed, uint64_t stream, double* out);
void gk_gaussian_vector(int64_t n, uint64_t seed, uint64_t stream, double* out);
/* std::uniform_real_distribution<double>(a, b) over seeded_rng(seed, stream)
 * (libstdc++; the restart jitter of GpModel::fit, gp.cpp:328-331). */
void gk_uniform_vector(int64_t n, uint64_t seed, uint64_t stream, double a, double b, double* out);

/* ---------------------------------------------------------------- operators
 * Every structured operator is a gk_op (LinearOperator, linear_operator.hpp:12-35). */
typedef struct gk_op gk_op;

/* Diagnostics for the one-launch 2-D D-SKI MVM: with tuning key "fused_prof"
 * set to 1, each launch records per-CTA %globaltimer stamps (ns) at 8 points:
 * start, scatter done, barrier 1 passed, mode-1 done, barrier 2 passed,
 * mode-0 done, barrier 3 passed, gather done. Copies the stamps of the last
 * launch for `nrhs` into out[cta*8 + k]; returns the CTA count (0 if none). */
int gk_debug_fused_phases(gk_op* op, int nrhs, int64_t* out, int max_ctas);
/* fp64 tensor-core (DMMA m8n8k4) throughput of `device` in TFLOP/s, measured
 * by a register-only kernel (best of 5): the D-SKIP roofline denominator. */
gk_status gk_debug_dmma_peak(int device, double* tflops);
/* rademacher_vector(n, seed, stream) (rng.hpp:23-29) generated by the device
 * mt19937_64 kernel that produces SLQ probes; copied to out[n] (test hook). */
gk_status gk_debug_rademacher_dev(int64_t n, uint64_t seed, uint64_t stream, double* out);

/* DskiOperator(kernel, grid, X, noise, order, with_gradients) (dski.hpp:58-65).
 * order: 0 quintic, 1 cubic. */
gk_status gk_dski_create(const gk_kernel* kernel, const gk_grid* grid, const double* X,
                         int64_t n, double noise_value, double noise_gradient, int order,
                         int with_gradients, int device, gk_op** out);

/* DskipOperator(kernel, X, noise, config) (dskip.hpp:91-94, DskipConfig :74-85). */
typedef struct {
  int64_t rank;
  double grid_ratio;
  int max_grid_nodes;
  uint64_t seed;
  int rank_policy_error;
  int track_dlogell;
  int with_gradients;
} gk_dskip_config;
gk_status gk_dskip_create(const gk_kernel* kernel, const double* X, int64_t n, int d,
                          double noise_value, double noise_gradient, const gk_dskip_config* cfg,
                          int device, gk_op** out);

/* D-SKIP operator from explicit Lanczos factors (one or two; Q_f N×r_f
 * column-major, alpha_f r_f, beta_f r_f-1) — the Hadamard MVM/diagonal/row of
 * dskip.cpp:236-264 over factors built elsewhere (e.g. by the reference). */
gk_status gk_dskip_create_from_factors(int64_t n, int groups, double noise_value, double noise_gradient,
                                       int nfactors, const int64_t* ranks, const double* const* Q,
                                       const double* const* alpha, const double* const* beta, int device,
                                       gk_op** out);

/* DenseOperator(A) (linear_operator.hpp:38-56); A is N×N column-major. */
gk_status gk_dense_create(const double* A, int64_t N, int device, gk_op** out);

/* assemble_dense(kernel, X, X', options) (kernels.cpp:242-285, AssemblyOptions
 * kernels.hpp:83-92): the type-major n(d+1) × n'(d+1) (or n × n') K∇, or
 * ∂K∇/∂log ℓ when dlogell != 0, assembled on `device`; derivative_scale > 0
 * scales derivative rows and columns. Host output, column-major. Above
 * size_cap entries: GK_ERR_LENGTH (std::length_error, kernels.cpp:252-255). */
gk_status gk_assemble_dense(const gk_kernel* kernel, const double* X, int64_t n, const double* Xp, int64_t np, int d,
                            int with_derivatives, int dlogell, double derivative_scale, int64_t size_cap, int device,
                            double* out);
/* GpModel's exact backend (gp.cpp:71-85): DenseOperator over the device-
 * assembled K∇ + noise diagonal, with its dense Cholesky factor (cuSOLVER
 * potrf, loaded on first use; the reference uses Eigen's LLT). Not positive
 * definite: GK_ERR_RUNTIME "dense kernel matrix is not positive definite". */
gk_status gk_dense_kernel_create(const gk_kernel* kernel, const double* X, int64_t n, int d, double noise_value,
                                 double noise_gradient, int with_gradients, int64_t size_cap, int device,
                                 gk_op** out);
/* llt_->solve (gp.cpp:146): X = K⁻¹ B through the factor (host buffers). */
gk_status gk_dense_cholesky_solve(const gk_op* op, const double* B, int64_t ldb, int64_t nrhs, double* X, int64_t ldx);
/* GpModel::logdet exact branch (gp.cpp:167-168): 2 Σ log L_ii. */
gk_status gk_dense_cholesky_logdet(const gk_op* op, double* logdet);
/* GpModel::lml_gradient exact branch (gp.cpp:246-276): traces through K⁻¹ and
 * the assembled ∂K/∂log ℓ. alpha = K⁻¹ targets (host, N). */
gk_status gk_dense_exact_lml_gradient(const gk_op* op, const double* alpha, double* grad, int* nparams);

/* Matrix-free exact D-SE operator: assemble_dense(kernel, X, X) + noise
 * (kernels.cpp:242-285) applied without forming the N×N matrix. */
gk_status gk_exact_create(const gk_kernel* kernel, const double* X, int64_t n, int d,
                          double noise_value, double noise_gradient, int with_gradients,
                          int device, gk_op** out);

void gk_op_destroy(gk_op* op);
int64_t gk_op_size(const gk_op* op);
/* 0 = exact, 1 = dski, 2 = dskip, 3 = dense, 4 = grid kernel (K_UU) */
int gk_op_kind(const gk_op* op);

/* LinearOperator::mvm over nrhs columns: Out = A V (host pointers). */
gk_status gk_op_mvm(const gk_op* op, const double* V, int64_t ldv, double* Out, int64_t ldo,
                    int64_t nrhs);
/* Same with device pointers (external layout) on `stream`. */
gk_status gk_op_mvm_dev(const gk_op* op, const double* dV, int64_t ldv, double* dOut,
                        int64_t ldo, int64_t nrhs, void* stream);
/* LinearOperator::diagonal / row (dski.cpp:240-304, dskip.cpp:252-264). */
gk_status gk_op_diagonal(const gk_op* op, double* out);
gk_status gk_op_row(const gk_op* op, int64_t r, double* out);
/* noise_diagonal() (dski.cpp:206-211). */
gk_status gk_op_noise_diagonal(const gk_op* op, double* out);

/* D-SKI pieces GpModel uses directly (gp.cpp:213,416,445,482):
 * stacked_transpose_apply (dski.cpp:213-219): U(m×nrhs) = B^T V;
 * stacked_apply (dski.cpp:221-226): Out = B U; grid_operator().apply
 * (dski.cpp:146-172): W = K_UU U. */
int64_t gk_dski_grid_size(const gk_op* op);
gk_status gk_dski_get_grid(const gk_op* op, gk_grid* out);
/* GridKernelOperator::min_embedding_eigenvalue (dski.hpp:40-43, dski.cpp:
 * 137-139): the smallest eigenvalue of the reference's circulant embedding
 * (2(m_j − 1) nodes per axis) of the operator's profile, computed on the host
 * (separable cosine sums in long double; O(E·ΣE_j), seconds at C4). */
gk_status gk_dski_min_embedding_eigenvalue(const gk_op* op, double* out);
/* Profile-agnostic forms: the caller evaluates its
 * StationaryProfile where the reference's constructors do and passes the
 * values. slice = the profile on the reference's circulant embedding,
 * 2(m_j − 1) nodes per axis, row-major, entry t at the wrapped offsets
 * (i_j ≤ m_j − 1 ? i_j : i_j − 2(m_j − 1))·h_j (dski.cpp:97-114).
 * GridKernelOperator(grid, profile) (dski.cpp:80-172): K_UU as an operator of
 * size M (mvm, diagonal, row; gk_dski_min_embedding_eigenvalue works on it).
 * D-SKI from a profile: offset_table = the profile at the (2T − 1)^d stencil
 * offsets (i_j − (T − 1))·h_j, row-major (kernel_offset_table_, dski.cpp:
 * 181-203; T = 6 quintic, 4 cubic). Such an operator has no ∂/∂log ℓ. */
gk_status gk_grid_kernel_create(const gk_grid* grid, const double* slice, int device, gk_op** out);
gk_status gk_dski_create_from_profile(const gk_grid* grid, const double* X, int64_t n, double noise_value,
                                      double noise_gradient, int order, int with_gradients, const double* slice,
                                      const double* offset_table, int device, gk_op** out);
gk_status gk_dski_transpose_apply(const gk_op* op, const double* V, int64_t ldv, double* U,
                                  int64_t ldu, int64_t nrhs);
gk_status gk_dski_apply(const gk_op* op, const double* U, int64_t ldu, double* Out, int64_t ldo,
                        int64_t nrhs);
gk_status gk_dski_grid_mvm(const gk_op* op, const double* U, int64_t ldu, double* W, int64_t ldw,
                           int64_t nrhs);

/* D-SKIP factor access (DskipOperator::factors, dskip.hpp:108) and
 * dlogell_apply (dskip.cpp:266-274). */
int gk_dskip_factor_count(const gk_op* op);
int64_t gk_dskip_factor_rank(const gk_op* op, int f);
gk_status gk_dskip_factor_get(const gk_op* op, int f, double* Q, double* alpha, double* beta);
gk_status gk_dskip_dlogell_apply(const gk_op* op, const double* V, int64_t ldv, double* Out,
                                 int64_t ldo, int64_t nrhs);
/* D-SKI ∂K∇/∂log ℓ · V = B (∂K_UU/∂log ℓ) Bᵀ V without noise — the "second
 * grid operator" of GpModel::dlogell_apply (gp.cpp:212-213) built from
 * kernel_dlogell_profile (dski.cpp:36-40); SE only. Host buffers, N × nrhs. */
gk_status gk_dski_dlogell_apply(const gk_op* op, const double* V, int64_t ldv, double* Out, int64_t ldo,
                                int64_t nrhs);

/* Internal-layout stage entry points (device pointers, RHS-minor internal
 * layout; used by the benchmark to time each kernel on its own stream).
 * stage: 0 = scatter (B^T), 1 = grid K_UU, 2 = gather (B, no noise),
 * 3 = whole MVM, 4 = whole MVM replayed from a cached CUDA graph. */
gk_status gk_op_stage_dev(const gk_op* op, int stage, const double* dIn, double* dOut,
                          int64_t nrhs, void* stream);
/* D-SKI gather with the noise term, out = B w + diag(σ1² I, σ2² I) v
 * (internal layout, device pointers): the last stage of a grid-slab sharded
 * MVM whose grid vector w = K_UU Σ_ranks B_rᵀ v_r the caller
 * all-reduced. */
gk_status gk_dski_gather_dev(const gk_op* op, const double* dW, const double* dV, double* dOut,
                             int64_t nrhs, void* stream);
/* The one-launch 2-D MVM split at its first grid barrier (grid-slab sharding,
 * SURVEY §8(e)): phase 0 scatters dV (internal layout) into dU2 = [u; h]
 * (2·M·nrhs doubles: the grid vector and the scatter's segment halo rows);
 * phase 1 applies K_UU to the (all-reduced) dU2 and gathers with noise from
 * dV into dOut. GK_ERR_UNSUPPORTED when the operator has no such plan
 * (callers then use gk_op_stage_dev stages 0/1 and gk_dski_gather_dev);
 * phase 2 only queries that availability for nrhs (no device work). */
gk_status gk_dski_fused_split_dev(const gk_op* op, int phase, const double* dV, double* dU2,
                                  double* dOut, int64_t nrhs, void* stream);
/* Convert external column-major blocks to/from the internal layout. */
gk_status gk_op_to_internal_dev(const gk_op* op, const double* dV, int64_t ldv, double* dI,
                                int64_t nrhs, void* stream);
gk_status gk_op_from_internal_dev(const gk_op* op, const double* dI, double* dV, int64_t ldv,
                                  int64_t nrhs, void* stream);

/* ---------------------------------------------------------------- solvers
 * cg (linalg.cpp:85-131), batched: each of the nrhs columns runs the
 * reference's single-RHS PCG independently (own alpha/beta, own stopping
 * iteration; a column that stops is frozen). Non-convergence is a flag,
 * not an error (linalg.hpp:27-30). residual_history may be NULL; else it
 * holds (max_iterations+1)×nrhs relres values (column-major), and
 * history_len[c] entries are valid for column c. precond may be NULL. */
typedef struct gk_precond gk_precond;
gk_status gk_pcg(const gk_op* op, const gk_precond* precond, const double* B, int64_t ldb,
                 int64_t nrhs, double tol, int max_iterations, double* X, int64_t ldx,
                 int* iterations, int* converged, double* residual_history, int* history_len);
/* Device-pointer variant (external layout), on `stream`. Iteration counts
 * and flags are written to host arrays; the call synchronises `stream`. */
gk_status gk_pcg_dev(const gk_op* op, const gk_precond* precond, const double* dB, int64_t ldb,
                     int64_t nrhs, double tol, int max_iterations, double* dX, int64_t ldx,
                     int* iterations, int* converged, void* stream);

/* pivoted_cholesky (linalg.cpp:133-174) over the operator's own diagonal and
 * rows. kernel_part != 0 factors op - noise_diagonal with the diagonal
 * clamped at 0, exactly as GpModel::preconditioner (gp.cpp:122-136).
 * L (N×max_rank col-major, original row order) and pivots are host outputs;
 * *rank receives the achieved rank. */
typedef struct gk_pivchol gk_pivchol;
gk_status gk_pivoted_cholesky(const gk_op* op, int kernel_part, int64_t max_rank,
                              double trace_tol, gk_pivchol** out);
int64_t gk_pivchol_rank(const gk_pivchol* f);
gk_status gk_pivchol_get(const gk_pivchol* f, double* L /*N×rank or NULL*/,
                         int64_t* pivots /*rank or NULL*/, double* initial_trace,
                         double* residual_trace);
void gk_pivchol_destroy(gk_pivchol* f);

/* Preconditioner(F, noise_diag) (linalg.cpp:176-213): M^{-1}b =
 * D^{-1/2}(c - Q1 Q1^T c), c = D^{-1/2} b, Q1 from a QR of [D^{-1/2}F; I]
 * (CholeskyQR2 on the device; agrees with the reference's Householder Q1 to
 * ≤1e-10 at C4's rank 200, tests/test_gpu_fullsize_parity.py). Any rank:
 * ranks whose projection does not fit shared memory run it in k-column tiles
 * and the apply as S = Q1 T plus a finishing pass (the k×k Cholesky of the
 * Gram matrix runs on the host in long double, O(k³)). */
gk_status gk_precond_create(const double* F, int64_t N, int64_t k, const double* noise_diag,
                            int device, gk_precond** out);
/* From a device-resident pivoted Cholesky factor, with D = op noise diagonal
 * (GpModel::preconditioner, gp.cpp:139). */
gk_status gk_precond_from_pivchol(const gk_op* op, const gk_pivchol* f, gk_precond** out);
gk_status gk_precond_apply(const gk_precond* M, const double* B, int64_t ldb, double* Out,
                           int64_t ldo, int64_t nrhs);
gk_status gk_precond_quadratic(const gk_precond* M, const double* B, int64_t ldb, int64_t nrhs,
                               double* out /*nrhs*/);
int64_t gk_precond_rank(const gk_precond* M);
gk_status gk_precond_q1(const gk_precond* M, double* Q1 /*N×k col-major*/);
void gk_precond_destroy(gk_precond* M);

/* slq_logdet (linalg.cpp:215-253): probes run as one batched Lanczos;
 * probe p uses rademacher_vector(N, seed, p) and restart stream
 * mix_seed(seed, 50000+p); estimates[p] (may be NULL) receives the per-probe
 * value, and *logdet = sum_p estimates[p] / probes summed in probe order.
 * probe_offset lets a rank run probes [probe_offset, probe_offset+probes)
 * of a larger job (probe sharding); *logdet is then the local sum / probes. */
gk_status gk_slq_logdet(const gk_op* op, int probes, int lanczos_steps, uint64_t seed,
                        double eigen_floor, int probe_offset, double* logdet, int* clamped,
                        double* estimates);

/* lanczos_lowrank (linalg.cpp:306-314) / lanczos_from_start (:17-81). Q is
 * N×rank col-major; *k receives the achieved rank. start may be NULL
 * (seeded Gaussian start). */
gk_status gk_lanczos(const gk_op* op, int64_t steps, uint64_t seed, const double* start,
                     uint64_t restart_seed, double* Q, double* alpha, double* beta, int64_t* k,
                     int* breakdown);

/* trace_estimate (linalg.cpp:255-279): E_z[z^T A^{-1} B z], probes batched. */
gk_status gk_trace_estimate(const gk_op* A, const gk_op* B, int probes, uint64_t seed, double tol,
                            int max_iterations, const gk_precond* precond, double* out);
/* GpModel::lml_gradient (gp.cpp:220-292), stochastic-trace branch, for a D-SKI
 * or D-SKIP operator: grad[p] = ½(αᵀ M_p α − tr(K⁻¹ M_p)) over θ = (log ℓ, log s,
 * log σ₁[, log σ₂]) with M_0 = ∂K/∂log ℓ, M_1 = 2(K − noise), M_2/M_3 the
 * noise blocks; traces by trace_estimate with `probes` Rademacher probes
 * (streams 1000+q) and PCG at tol max(tol, 1e-2) preconditioned by M. alpha =
 * K⁻¹ b (host, N). *nparams = 4 with gradient observations, else 3.
 * GK_ERR_RUNTIME if a probe solve does not converge (linalg.cpp:273-275). */
gk_status gk_lml_gradient(const gk_op* op, const gk_precond* M, const double* alpha, int probes, uint64_t seed,
                          double tol, int maxit, double* grad, int* nparams);

/* ---------------------------------------------------------------- GP glue
 * GpModel pieces on the hot path (gp.cpp:117-187,471-517): the operator is
 * built by the caller; these run the batched solve / SLQ / prediction. */
/* predict_mean_grad for D-SKI (gp.cpp:480-495): g = K_UU (B^T alpha) cached in
 * the call; values = mean + W_test g, grads = dW_test g. Xtest T×d col-major. */
gk_status gk_dski_predict_mean_grad(const gk_op* op, const double* alpha, double mean,
                                    const double* Xtest, int64_t T, double* values,
                                    double* grads /*T×d col-major*/);
/* cross_covariance for D-SKI (gp.cpp:412-417), T test points at once:
 * Q (N×T col-major). */
gk_status gk_dski_cross_covariance(const gk_op* op, const double* Xtest, int64_t T, double* Q,
                                   int64_t ldq);
/* Device-pointer cross-covariance for T ≤ 64 test points (dXt T×d col-major
 * on the device): columns B K_UU w(x_t) into dQ (N×T external order, ld
 * ldq), w the value stencil (direction = -1, gp.cpp:412-417) or its ∂/∂x_p
 * (direction = p, gp.cpp:431-461). Used for pivot columns of the
 * grid-slab sharded pivoted Cholesky. Synchronises `stream` once (the
 * out-of-grid check). */
gk_status gk_dski_cross_covariance_dev(const gk_op* op, const double* dXt, int64_t T, int direction,
                                       double* dQ, int64_t ldq, void* stream);
/* GpModel::cross_covariance_jacobian (gp.cpp:431-461, D-SKI branch) for T test
 * points (Xtest T×d col-major): J column t·d + p (leading dimension ldj ≥ N)
 * = ∂q(x_t)/∂x_p = B K_UU w_p(x_t) with w_p the derivative point stencil. */
gk_status gk_dski_cross_covariance_jacobian(const gk_op* op, const double* Xtest, int64_t T, double* J,
                                           int64_t ldj);

/* GpModel::solve (gp.cpp:143-158): PCG over nrhs columns (x0 = 0); a column
 * that does not converge is GK_ERR_RUNTIME with the reference's message
 * "CG did not converge: relative residual R after K iterations (tol T)".
 * iterations (nrhs, may be NULL) receives the per-column counts. */
gk_status gk_gp_solve(const gk_op* op, const gk_precond* precond, const double* B, int64_t ldb,
                      int64_t nrhs, double tol, int max_iterations, double* X, int64_t ldx,
                      int* iterations);
/* GpModel::logdet (gp.cpp:165-179), D-SKI/D-SKIP branch: slq_logdet with the
 * model's eigen floor 0.5·min(σ₁, σ₂)² (0.5·σ₁² without gradients). */
gk_status gk_gp_logdet(const gk_op* op, int probes, int lanczos_steps, uint64_t seed,
                       double noise_value, double noise_gradient, int has_gradients,
                       double* logdet);
/* GpModel::log_marginal_likelihood (gp.cpp:181-187): targets = stacked
 * targets with the mean subtracted (observations.hpp:29-35, gp.cpp:43);
 * alpha = solve(targets) (throws like gk_gp_solve), lml = −½(tᵀα + logdet +
 * N log 2π). fit_term, logdet and alpha (N) may be NULL. */
gk_status gk_gp_log_marginal_likelihood(const gk_op* op, const gk_precond* precond,
                                        const double* targets, double tol, int max_iterations,
                                        int probes, int lanczos_steps, uint64_t seed,
                                        double noise_value, double noise_gradient,
                                        int has_gradients, double* lml, double* fit_term,
                                        double* logdet, double* alpha);
/* GpModel::predict_variance_exact (gp.cpp:499-502) for T test points (Xtest
 * T×d col-major): var[t] = prior − q_tᵀ K⁻¹ q_t; cross-covariances, the
 * batched solve (GpModel::solve semantics) and the dots all on the device. */
gk_status gk_dski_predict_variance_exact(const gk_op* op, const gk_precond* precond,
                                         const double* Xtest, int64_t T, double prior,
                                         double tol, int max_iterations, double* var);
/* GpModel::predict_variance_randomized (gp.cpp:519-547): the pivoted-Cholesky
 * variance minus the control-variate correction over `probes` Rademacher
 * probes z_p = rademacher_vector(T, seed, 9000+p) (accumulated in probe
 * order). K'z, the solves, M⁻¹ and K'ᵀ(·) run on the device. precond is
 * required (std::logic_error → GK_ERR_LOGIC otherwise). */
gk_status gk_dski_predict_variance_randomized(const gk_op* op, const gk_precond* precond,
                                              const double* Xtest, int64_t T, double prior,
                                              int probes, uint64_t seed, double tol,
                                              int max_iterations, double* var);

/* ---------------------------------------------------------------- row-sharded preconditioner
 * SURVEY §8(e) (grid-slab sharding, C4): each rank holds the rows of Q1 and
 * D^{-1/2} for its own rows of the system. The Woodbury apply of
 * Preconditioner::apply (linalg.cpp:200-204) splits into a local projection
 * T_r = Q1_rᵀ D_r^{-1/2} r_r (k×nrhs), an all-reduce T = Σ_r T_r, and a local
 * finish z_r = D_r^{-1/2}(D_r^{-1/2} r_r − Q1_r T). Device pointers; row-
 * minor (RHS innermost) blocks of this rank's rows. */
gk_status gk_precond_from_q1_dev(const double* dQ1 /*N×k col-major*/, const double* dinv_sqrt /*N*/,
                                 int64_t N, int64_t k, int device, gk_precond** out);
gk_status gk_precond_project_dev(const gk_precond* M, const double* dR, double* dT, int64_t nrhs,
                                 void* stream);
gk_status gk_precond_finish_dev(const gk_precond* M, const double* dR, const double* dT, double* dZ,
                                int64_t nrhs, void* stream);

/* ---------------------------------------------------------------- datasets
 * Seeded synthetic workloads C1..C5 (BASELINE.json configs), generated on
 * the host with std::mt19937_64 + libstdc++ distributions like
 * testfns.cpp:355-402. Writes n into *n, X (n×d col-major), y (n), dY (n×d).
 * Pass NULL buffers to query n and d first. */
gk_status gk_make_dataset(int config, uint64_t seed, int64_t* n, int* d, double* X, double* y,
                          double* dY);

/* sample_dataset(test_function_by_name(name), n, Uniform, seed, σ₁, σ₂,
 * with_gradients) (testfns.cpp:355-402) for name "franke" (d = 2,
 * testfns.cpp:67-92) or "friedman" (d = 5, :290-310) — the data of the
 * precond-study tool (cmd_precond_study.cpp:31-34). X n×d col-major, y n,
 * dY n×d (NULL when with_gradients = 0). X = NULL only queries d.
 * Unknown name: GK_ERR_ARG (std::invalid_argument, testfns.cpp:325). */
gk_status gk_sample_test_function(const char* name, int64_t n, uint64_t seed, double noise_value,
                                  double noise_gradient, int with_gradients, int* d, double* X, double* y,
                                  double* dY);

#ifdef __cplusplus
}
#endif
#endif /* GK_CAPI_H */
