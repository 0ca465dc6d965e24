"""Full-size parity with the oracle on BASELINE.json's configurations (north_star
target: "GPU results that match the CPU oracle within the stated tolerances on
all five configs").

- C2: the headline 32-RHS MVM through the exact plan bench.py times
  (stage_dev(3) on the internal layout: the one-launch 2-D kernel), ≤1e-12
  relative per column (reference gate test_dski.cpp:104-116); the 31-probe ×
  30-step SLQ ≤1e-8 per probe (linalg.cpp:215-253).
- C3: the 17-RHS d = 3 MVM (targets + 16 probes), ≤1e-12.
- C4: the 1- and 8-RHS MVMs (400² grid, n = 150,000), ≤1e-12.
- C1: the GpModel pipeline at its stated settings (60² grid, rank-20
  pivoted Cholesky, PCG tol 1e-8, SLQ 8 × 25): pivots bit-exact, the
  reference's own non-convergence reproduced (same exception), early PCG
  history ≤1e-8, log-det ≤1e-8; and at σ = 0.5, where the reference solve
  converges, LML/log-det ≤1e-8 and iterations inside the oracle's band ±1
  (gp.cpp:117-187).
- C5: the 64-RHS Hadamard MVM at full N with identical factors (the device
  build's, evaluated by the oracle's hadamard_mvm, dskip.cpp:24-36), ≤1e-12;
  and the device D-SKIP build pinned step by step (Lanczos α/β of the leaf
  and merge factors, dskip.cpp:162-234) on a problem whose Ritz values have
  not converged.

Inputs come from the oracle's own generators (identical to the product's,
tests/test_capi_host.py)."""
import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu

NOISE = (1e-2, 1e-2)


def rhs(N, y, dY, nprobes):
    """Column 0 = stacked targets, then rademacher_vector(N, 0, 1000+p)."""
    cols = [O.stacked_targets(y, dY, y.mean())] + [O.rademacher_vector(N, 0, 1000 + p) for p in range(nprobes)]
    return np.asfortranarray(np.column_stack(cols))


def col_rel(got, want):
    return np.max(np.linalg.norm(got - want, axis=0) / np.linalg.norm(want, axis=0))


def pair(cfg, ell, nodes):
    X, y, dY = O.make_dataset(cfg, 0)
    og = O.Grid.cover(X, 1e-4, 3, nodes)
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    assert list(grid.dims) == [nodes] * X.shape[1]
    op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, NOISE)
    ref = O.DskiOperator(O.KernelSpec(ell, 1.0), og, X, NOISE)
    return X, y, dY, op, ref


def dev_mvm(op, B, stage=3):
    """The bench's timed step: external block -> internal layout, one
    stage_dev(3) MVM, back to external (all device pointers)."""
    import torch
    nrhs = B.shape[1]
    Vext = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    Vi = torch.empty(op.size() * nrhs, dtype=torch.float64, device="cuda")
    Oi = torch.empty_like(Vi)
    Oe = torch.empty_like(Vext)
    s = torch.cuda.current_stream().cuda_stream
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=s)
    op.stage_dev(stage, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=s)
    op.from_internal_dev(Oi.data_ptr(), Oe.data_ptr(), nrhs, stream=s)
    torch.cuda.synchronize()
    return Oe.cpu().numpy().T


@pytest.fixture(scope="module")
def c2():
    return pair(2, 0.2, 100)


def test_c2_headline_mvm_32rhs(c2):
    X, y, dY, op, ref = c2
    B = rhs(op.size(), y, dY, 31)
    want = ref.mvm(B)
    assert col_rel(dev_mvm(op, B), want) <= 1e-12
    assert col_rel(op.mvm(B), want) <= 1e-12  # host-buffer C-ABI path (gk_op_mvm)


def test_c2_slq_31x30(c2):
    X, y, dY, op, ref = c2
    floor = 0.5 * 1e-4
    got = gk.slq_logdet(op, 31, 30, 0, floor)
    want = O.slq_logdet(ref, 31, 30, 0, floor)
    assert np.max(np.abs(got.estimates - want.estimates) / np.abs(want.estimates)) <= 1e-8
    assert abs(got.logdet - want.logdet) <= 1e-8 * abs(want.logdet)
    assert got.clamped == want.clamped


def test_c3_mvm_17rhs():
    X, y, dY, op, ref = pair(3, 0.3, 48)
    B = rhs(op.size(), y, dY, 16)
    want = ref.mvm(B)
    assert col_rel(op.mvm(B), want) <= 1e-12
    assert col_rel(dev_mvm(op, B), want) <= 1e-12


@pytest.mark.parametrize("nrhs", [1, 8])
def test_c4_mvm(nrhs):
    X, y, dY, op, ref = pair(4, 0.02, 400)
    B = rhs(op.size(), y, dY, nrhs - 1)
    want = ref.mvm(B)
    assert col_rel(dev_mvm(op, B), want) <= 1e-12
    assert col_rel(op.mvm(B), want) <= 1e-12


def c1_models(noise, tol, maxit):
    X, y, dY = O.make_dataset(1, 0)
    kw = dict(noise=noise, backend="dski", grid_ratio=1e-3, max_grid_nodes=60, tol=tol, max_iterations=maxit,
              precond_rank=20, slq_probes=8, slq_steps=25, seed=0)
    return O.GpModel(O.KernelSpec(0.15, 1.0), X, y, dY, **kw), gk.GpModel(gk.KernelSpec(0.15, 1.0), X, y, dY, **kw)


def test_c1_stated_settings():
    """C1 as BASELINE states it (σ = 1e-2, rank 20, tol 1e-8, SLQ 8 × 25). The
    reference algorithm does not reach tol 1e-8 here: the oracle's PCG stops
    at max_iterations with relres ≈ 0.14 and GpModel::solve throws
    (gp.cpp:151-156). Parity: pivots bit-exact, the same exception, the PCG
    residual history of the first 20 iterations ≤1e-8, SLQ log-det with the
    model's floor ½σ² ≤1e-8 per probe."""
    ref, gm = c1_models(NOISE, 1e-8, 2000)
    A = gm.op()
    assert list(A.grid.dims) == [60, 60]
    f = gk.pivoted_cholesky(A, 20, kernel_part=True)
    assert [int(p) for p in f.pivots] == [int(p) for p in ref.pivots(20)]
    with pytest.raises(RuntimeError, match="CG did not converge"):
        ref.alpha()
    with pytest.raises(RuntimeError, match="CG did not converge: relative residual .* after 2000 iterations"):
        gm.alpha()
    t = gm.stacked_targets()
    og = O.Grid(A.grid.dims, A.grid.origin, A.grid.spacing)
    rop = O.DskiOperator(O.KernelSpec(0.15, 1.0), og, gm.X, NOISE)
    fr = O.pivoted_cholesky(rop, 20, noise_diag=rop.noise_diagonal())
    Pr = O.Preconditioner(fr.L, rop.noise_diagonal())
    hr = O.cg(rop, t, 1e-8, 20, Pr).residual_history
    hg = gk.cg(A, t, 1e-8, 20, gm.preconditioner()).residual_history
    assert np.max(np.abs(np.asarray(hg) - hr) / hr) <= 1e-8
    want = O.slq_logdet(rop, 8, 25, 0, 0.5 * 1e-4)
    got = gk.slq_logdet(A, 8, 25, 0, 0.5 * 1e-4)
    assert np.max(np.abs(got.estimates - want.estimates) / np.abs(want.estimates)) <= 1e-8
    assert abs(gm.logdet() - want.logdet) <= 1e-8 * abs(want.logdet)


def test_c1_lml_where_the_solve_converges():
    """The C1 pipeline (data, 60² grid, ℓ, rank-20 preconditioner, SLQ 8 × 25)
    at σ = 0.5, where the reference's PCG converges (tol 1e-10, ~600
    iterations): LML and log-det ≤1e-8, α to the solver tolerance, iteration
    count inside the oracle's own ulp-perturbation band ±1 (CG counts at
    hundreds of iterations move under 1e-16 perturbations of b,
    test_gpu_solvers.oracle_iteration_band)."""
    from test_gpu_solvers import oracle_iteration_band
    ref, gm = c1_models((0.5, 0.5), 1e-10, 3000)
    r = ref.log_marginal_likelihood()
    lml = gm.log_marginal_likelihood()
    assert abs(lml - r["lml"]) <= 1e-8 * abs(r["lml"]), (lml, r["lml"])
    assert abs(gm.logdet() - r["logdet"]) <= 1e-8 * abs(r["logdet"])
    a_ref, its_ref = ref.alpha()
    a = gm.alpha()
    assert np.linalg.norm(a - a_ref) <= 1e-6 * np.linalg.norm(a_ref)
    A, t = gm.op(), gm.stacked_targets()
    og = O.Grid(A.grid.dims, A.grid.origin, A.grid.spacing)
    rop = O.DskiOperator(O.KernelSpec(0.15, 1.0), og, gm.X, (0.5, 0.5))
    fr = O.pivoted_cholesky(rop, 20, noise_diag=rop.noise_diagonal())
    lo, hi = oracle_iteration_band(rop, t, 1e-10, 3000, O.Preconditioner(fr.L, rop.noise_diagonal()), k=2)
    its = gk.cg(A, t, 1e-10, 3000, gm.preconditioner()).iterations
    # ±1 against the oracle GpModel's own solve (measured: 616 vs 616); the
    # band of the free-function oracle PCG (its preconditioner differs from
    # GpModel's at roundoff: 608-609) is accepted as well
    assert abs(its - its_ref) <= 1 or lo - 1 <= its <= hi + 1, (its, its_ref, lo, hi)


def test_c1_gp_solve_raises_reference_error():
    X, y, dY = O.make_dataset(1, 0)
    gm = gk.GpModel(gk.KernelSpec(0.15, 1.0), X, y, dY, noise=NOISE, grid_ratio=1e-3, max_grid_nodes=60,
                    tol=1e-8, max_iterations=3, precond_rank=20)
    with pytest.raises(RuntimeError, match="CG did not converge: relative residual .* after 3 iterations"):
        gm.alpha()


def test_c5_hadamard_full_size_identical_factors():
    X, y, dY = O.make_dataset(5, 0)
    op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, NOISE, rank=30, grid_ratio=0.01, max_grid_nodes=100,
                          seed=0)
    facs = [(f.Q, f.alpha, f.beta) for f in op.factors()]
    assert [f[0].shape[1] for f in facs] == [30, 30]
    ref = O.DskipOperator.from_factors(facs, X.shape[0], 6, NOISE)
    g = gk.DskipOperator.from_factors(facs, X.shape[0], 6, NOISE)
    B = rhs(op.size(), y, dY, 63)
    want = ref.mvm(B)
    assert col_rel(g.mvm(B), want) <= 1e-12
    assert col_rel(op.mvm(B), want) <= 1e-12  # the device-built operator holds the same factors


@pytest.mark.parametrize("d", [2, 4])
def test_dskip_build_pinned_step_by_step(d):
    """Leaf (d = 2: the two factors ARE the leaves) and merge (d = 4: each final
    factor is the Lanczos of a Hadamard merge of two leaves, seed stream
    mix_seed(seed, 1000+k)) factors: α/β of the first 5 Lanczos steps ≤1e-10
    against the oracle build, on data whose leaf operators have numerical rank
    well above the factor rank (no breakdown restarts, Ritz values not yet
    converged)."""
    n, r = 300, 10
    X = np.random.default_rng(40 + d).uniform(0, 1, (n, d))
    kw = dict(rank=r, grid_ratio=0.05, max_grid_nodes=64, seed=3)
    ref = O.DskipOperator(O.KernelSpec(0.12, 1.0), X, NOISE, **kw)
    g = gk.DskipOperator(gk.KernelSpec(0.12, 1.0), X, NOISE, **kw)
    rf, gf = ref.factors(), g.factors()
    assert len(rf) == len(gf) == 2
    for (Qr, ar, br), fg in zip(rf, gf):
        assert fg.alpha.size == ar.size == r
        assert np.max(np.abs(fg.alpha[:5] - ar[:5])) <= 1e-10 * np.max(np.abs(ar))
        assert np.max(np.abs(fg.beta[:5] - br[:5])) <= 1e-10 * np.max(np.abs(ar))
        # and the basis vectors themselves (up to roundoff) for those steps
        assert np.max(np.abs(fg.Q[:, :5] - Qr[:, :5])) <= 1e-9


def test_c4_cholesky_qr2_preconditioner_matches_householder():
    """The preconditioner's Q1 is built by CholeskyQR2 on the device where the
    reference uses Householder QR (linalg.cpp:187-193). At C4's rank 200 and
    σ = 1e-2 (the worst-conditioned [D^{-1/2}L; I] of the configs), M⁻¹b and
    the quadratic form agree with a Householder QR of the same factor (LAPACK
    via numpy) to ≤1e-10."""
    X, y, dY = O.make_dataset(4, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, 400)
    op = gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, NOISE)
    f = gk.pivoted_cholesky(op, 200, kernel_part=True)
    M = gk.Preconditioner.from_pivchol(op, f)
    L = f.L
    nd = np.full(op.size(), NOISE[1] ** 2)
    nd[: X.shape[0]] = NOISE[0] ** 2
    dinv = 1.0 / np.sqrt(nd)
    Q, _ = np.linalg.qr(np.vstack([dinv[:, None] * L, np.eye(L.shape[1])]))  # Householder (LAPACK geqrf)
    Q1 = Q[: op.size()]
    B = np.random.default_rng(4).standard_normal((op.size(), 2))
    B[:, 0] = O.stacked_targets(y, dY, y.mean())
    for j in range(2):
        c = dinv * B[:, j]
        t = Q1.T @ c
        z_ref = dinv * (c - Q1 @ t)
        z = M.apply(B[:, j])
        assert np.linalg.norm(z - z_ref) <= 1e-10 * np.linalg.norm(z_ref)
        q_ref = c @ c - t @ t
        assert abs(M.quadratic(B[:, j]) - q_ref) <= 1e-10 * abs(q_ref)
