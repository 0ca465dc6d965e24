"""GPU hyperparameter-gradient pieces against the oracle (reference
gp.cpp:189-292): the D-SKI ∂K∇/∂log ℓ operator (a second grid operator over
kernel_dlogell_profile, gp.cpp:212-213 — here a sum of d Kronecker-Toeplitz
terms), and GpModel::lml_gradient's stochastic-trace branch with the same
probes, seed, trace tolerance and preconditioner."""
import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu

ELL, NOISE, RATIO, MAXN, RANK = 0.15, (0.05, 0.05), 0.1, 40, 40


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.mark.parametrize("d", [1, 2, 3])
def test_dski_dlogell_matches_oracle(d):
    rng = np.random.default_rng(40 + d)
    n = 300 if d < 3 else 120
    X = rng.uniform(0.1, 0.9, (n, d))
    grid = gk.Grid.cover(X, RATIO * 0.3, 3, 30 if d == 3 else MAXN)
    og = O.Grid(grid.dims, grid.origin, grid.spacing)
    k = gk.KernelSpec(0.3, 1.3)
    op = gk.DskiOperator(k, grid, X, NOISE)
    ref = O.DskiOperator(O.KernelSpec(0.3, 1.3), og, X, NOISE)
    kd = O.GridKernelOperator(O.KernelSpec(0.3, 1.3), og, dlogell=True)
    V = rng.standard_normal((op.size(), 3))
    out = op.dlogell_apply(V)
    for c in range(3):
        want = ref.stacked_apply(kd.mvm(ref.stacked_transpose_apply(V[:, c])))
        assert rel(out[:, c], want) <= 1e-12, c


def make_model(noise, rank=RANK):
    X, y, dY = gk.make_dataset(1, 0)
    X, y, dY = X[:300], y[:300], dY[:300]
    om = O.GpModel(O.KernelSpec(ELL, 1.0), X, y, dY, noise=noise, backend="dski", grid_ratio=RATIO,
                   max_grid_nodes=MAXN, tol=1e-10, max_iterations=5000, precond_rank=rank, seed=3)
    grid = gk.Grid.cover(X, RATIO * ELL, 3, MAXN)
    op = gk.DskiOperator(gk.KernelSpec(ELL, 1.0), grid, X, noise)
    op.test_rank = rank
    return om, op, X, y, dY


@pytest.fixture(scope="module")
def model():
    return make_model(NOISE)


@pytest.fixture(scope="module")
def model_wc():  # well conditioned: every probe solve stops after 5 PCG iterations (oracle)
    return make_model((1.0, 1.0), rank=100)


def test_gp_dlogell_apply_matches_oracle_model(model):
    om, op, X, y, dY = model
    v = np.random.default_rng(9).standard_normal(op.size())
    assert rel(op.dlogell_apply(v), om.dlogell_apply(v)) <= 1e-12


def gpu_gradient(om, op, y, dY, probes):
    b = gk.stacked_targets(y, dY, y.mean())
    P = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, op.test_rank, kernel_part=True))
    sol = gk.cg(op, b, 1e-10, 5000, P)
    assert sol.converged
    return gk.lml_gradient(op, sol.x, probes, seed=3, tol=1e-10, max_iterations=5000, precond=P)


@pytest.mark.parametrize("probes", [8, 20])
def test_lml_gradient_matches_oracle(model_wc, probes):
    """Same probes, seed, preconditioner and trace tolerance (1e-2): with
    identical per-probe PCG iteration counts the gradients agree to roundoff."""
    om, op, X, y, dY = model_wc
    ref = om.lml_gradient(probes)
    g = gpu_gradient(om, op, y, dY, probes)
    assert g.shape == ref.shape == (4,)
    assert np.all(np.abs(g - ref) <= 1e-8 * np.abs(ref) + 1e-8), (g, ref)


def test_lml_gradient_ill_conditioned_within_cg_chaos(model):
    """σ = 0.05: each probe solve takes ~400 PCG iterations to reach the 1e-2
    trace tolerance, and roundoff makes the GPU and oracle runs stop ~10 %
    apart in iteration count (measured per probe: solutions agree to
    3e-5..9e-4). The gradient is held to 1 %."""
    om, op, X, y, dY = model
    ref = om.lml_gradient(8)
    g = gpu_gradient(om, op, y, dY, 8)
    assert np.all(np.abs(g - ref) <= 1e-2 * np.abs(ref)), (g, ref)
