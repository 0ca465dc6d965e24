"""D-SKI with a non-separable stationary profile (the spline kernel,
kernels.cpp:104-118) against the oracle: K_UU by circulant embedding + the
in-house FFT (reference GridKernelOperator, dski.cpp:80-172), MVM / stages /
diagonal / rows ≤1e-12 for d = 1, 2, 3 with and without gradients, both
spline parities; min_embedding_eigenvalue of the reference embedding (SE and
spline); PCG and SLQ on a spline operator."""
import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def abs_scale(op, X, V, order=0):
    """|W| |K_UU| |W|ᵀ |v| per column: the magnitude the MVM's sums run over.
    The spline profile carries a large constant s²·b (positive-definiteness
    calibration, kernels.cpp:42-90) whose contributions cancel in the
    gradient rows, so the output norm understates the roundoff scale: the
    dense float64 product, the oracle and the GPU all differ pairwise by
    ~1e-12 of ‖K v‖ at d = 2, and agree to 1e-13 of this scale."""
    g, k = op.grid, op.kernel
    d = X.shape[1]
    dims = [int(v) for v in g.dims]
    idx = np.stack(np.meshgrid(*[np.arange(m) for m in dims], indexing="ij"), -1).reshape(-1, d)
    pts = idx * np.asarray(g.spacing)
    rho = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)) / k.lengthscale
    with np.errstate(divide="ignore", invalid="ignore"):
        rad = np.where(rho > 0, rho * rho * np.log(np.where(rho > 0, rho, 1.0)), 0.0) if k.spline_even else rho ** 3
    Kuu = np.abs(k.outputscale ** 2 * (rad + k.spline_a * rho ** 2 + k.spline_b))
    W = np.abs(O.interp_dense(O.Grid(g.dims, g.origin, g.spacing), X, order))
    if W.shape[0] != op.size():
        W = W[: op.size()]
    return np.linalg.norm(W @ (Kuu @ (W.T @ np.abs(V))), axis=0)


def spline_pair(d, even, n=300, grad=True, nodes=None, seed=0, noise=(0.2, 0.3), order=0):
    rng = np.random.default_rng(seed + 10 * d)
    X = rng.uniform(0.1, 0.9, (n, d))
    ell = 0.4
    diam = np.sqrt(d) * 0.8 / ell
    a, b = -1.5 * diam, 4.0 * diam ** 3  # SplineConstants::for_domain shape (kernels.cpp:42-90)
    nodes = nodes or {1: 60, 2: 30, 3: 14}[d]
    grid = gk.Grid.cover(X, 0.05, 3, nodes)
    op = gk.DskiOperator(gk.KernelSpec(ell, 1.3, gk.SPLINE, a, b, even), grid, X, noise, order, grad)
    og = O.Grid(grid.dims, grid.origin, grid.spacing)
    ref = O.DskiOperator(O.KernelSpec(ell, 1.3, O.SPLINE, a, b, even), og, X, noise, order, grad)
    return X, op, ref


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("even", [False, True])
@pytest.mark.parametrize("grad", [True, False])
def test_spline_dski_mvm_matches_oracle(d, even, grad):
    X, op, ref = spline_pair(d, even, grad=grad)
    V = np.random.default_rng(1).standard_normal((op.size(), 5))
    got = op.mvm(V)
    scale = abs_scale(op, X, V)
    for c in range(5):
        want = ref.mvm(V[:, c])
        assert rel(got[:, c], want) <= 5e-12, (d, even, grad, c)
        assert np.linalg.norm(got[:, c] - want) <= 1e-12 * scale[c], (d, even, grad, c)
    u = np.random.default_rng(2).standard_normal(op.grid_size())
    assert rel(op.grid_mvm(u), ref.grid_mvm(u)) <= 1e-12


@pytest.mark.parametrize("d", [2, 3])
def test_spline_dski_cubic_and_odd_rhs(d):
    X, op, ref = spline_pair(d, d % 2 == 0, order=1)
    V = np.random.default_rng(3).standard_normal((op.size(), 3))
    got = op.mvm(V)
    scale = abs_scale(op, X, V, order=1)
    for c in range(3):
        assert np.linalg.norm(got[:, c] - ref.mvm(V[:, c])) <= 1e-12 * scale[c]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_spline_dski_diagonal_and_rows(d):
    X, op, ref = spline_pair(d, True, n=120)
    assert rel(op.diagonal(), ref.diagonal()) <= 1e-12
    N = op.size()
    for r in (0, 7, N // 2, N - 1):
        assert rel(op.row(r), ref.row(r)) <= 1e-12, r


@pytest.mark.parametrize("family", ["se", "spline"])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_min_embedding_eigenvalue_matches_oracle(family, d):
    if family == "se":
        rng = np.random.default_rng(5)
        X = rng.uniform(0, 1, (100, d))
        grid = gk.Grid.cover(X, 0.05, 3, {1: 50, 2: 24, 3: 12}[d])
        op = gk.DskiOperator(gk.KernelSpec(0.3, 1.2), grid, X, (0.1, 0.1))
        ref = O.DskiOperator(O.KernelSpec(0.3, 1.2), O.Grid(grid.dims, grid.origin, grid.spacing), X, (0.1, 0.1))
    else:
        _, op, ref = spline_pair(d, d % 2 == 0, n=100)
    got, want = op.min_embedding_eigenvalue(), ref.min_embedding_eigenvalue()
    scale = abs(ref.grid_mvm(np.eye(op.grid_size())[:, 0])[0])  # κ(0): the spectrum's mean value
    assert abs(got - want) <= 1e-10 * max(abs(want), scale), (got, want)


def test_spline_pcg_and_slq_match_oracle():
    X, op, ref = spline_pair(2, True, n=250, noise=(0.5, 0.5))
    b = np.random.default_rng(7).standard_normal(op.size())
    res = gk.cg(op, b, 1e-8, 500)
    want = O.cg(ref, b, 1e-8, 500)
    assert res.converged == want.converged
    assert abs(res.iterations - want.iterations) <= max(1, 0.02 * want.iterations), (res.iterations, want.iterations)
    assert rel(res.x, want.x) <= 1e-6
    got = gk.slq_logdet(op, 4, 20, 0, 1e-12)
    ref_ld = O.slq_logdet(ref, 4, 20, 0, 1e-12)
    assert np.max(np.abs(got.estimates - ref_ld.estimates) / np.abs(ref_ld.estimates)) <= 1e-8


@pytest.mark.parametrize("d", [1, 2, 3, 5])
@pytest.mark.parametrize("even", [False, True])
def test_spline_exact_operator_matches_dense_assembly(d, even):
    """The matrix-free exact K∇ with the spline kernel (eval / eval_grad /
    eval_hess_block, kernels.cpp:104-170, the r = 0 limits included; assembled
    as kernels.cpp:242-285) against the oracle's dense assembly: MVM within
    1e-12 of the |K||v| scale, diagonal and rows ≤1e-12."""
    rng = np.random.default_rng(20 + d)
    n = 150
    X = rng.uniform(0, 1, (n, d))
    X[7] = X[3]  # a coincident pair exercises the r = 0 branches off the diagonal
    ell = 0.5
    a, b, ev = gk.spline_constants_for_domain(np.sqrt(d) / ell, d)
    noise = (0.1, 0.2)
    op = gk.ExactOperator(gk.KernelSpec(ell, 1.1, gk.SPLINE, a, b, even), X, noise)
    K = O.assemble_dense(O.KernelSpec(ell, 1.1, O.SPLINE, a, b, even), X)
    K = K + np.diag(np.concatenate([np.full(n, noise[0] ** 2), np.full(n * d, noise[1] ** 2)]))
    V = rng.standard_normal((op.size(), 4))
    got = op.mvm(V)
    scale = np.linalg.norm(np.abs(K) @ np.abs(V), axis=0)
    assert np.all(np.linalg.norm(got - K @ V, axis=0) <= 1e-12 * scale)
    assert rel(op.diagonal(), np.diag(K)) <= 1e-12
    for r in (0, 3, 7, n + 7, op.size() - 1):
        assert np.linalg.norm(op.row(r) - K[r]) <= 1e-12 * np.linalg.norm(np.abs(K[r])), r


def profile_values(kind, off, ell=0.4, s=1.3, a=-3.0, b=40.0, even=True):
    """κ(offset) of SE / spline as the reference's eval(kernel, offset, 0)."""
    r2 = (np.asarray(off) ** 2).sum(-1)
    if kind == "se":
        return s * s * np.exp(-0.5 * r2 / ell ** 2)
    rho = np.sqrt(r2) / ell
    with np.errstate(divide="ignore", invalid="ignore"):
        rad = np.where(rho > 0, rho * rho * np.log(np.where(rho > 0, rho, 1.0)), 0.0) if even else rho ** 3
    return s * s * (rad + a * rho * rho + b)


@pytest.mark.parametrize("kind", ["se", "spline"])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_grid_kernel_operator_from_profile_slice(kind, d):
    """GridKernelOperator(grid, profile) at the boundary: the caller's profile
    values on the reference embedding; K_UU against the dense profile matrix
    (test_dski.cpp:51-69 analogue) and the oracle's operator; the minimum
    embedding eigenvalue against the oracle's."""
    dims = {1: [40], 2: [20, 16], 3: [10, 9, 8]}[d]
    g = gk.Grid(dims, [0.0] * d, [0.05] * d)
    off = gk.GridKernelOperator.embedding_offsets(g)
    even = d % 2 == 0
    op = gk.GridKernelOperator(g, profile_values(kind, off, even=even))
    idx = np.stack(np.meshgrid(*[np.arange(m) for m in dims], indexing="ij"), -1).reshape(-1, d) * 0.05
    K = profile_values(kind, idx[:, None, :] - idx[None, :, :], even=even)
    u = np.random.default_rng(d).standard_normal((op.size(), 3))
    got = op.mvm(u)
    scale = np.linalg.norm(np.abs(K) @ np.abs(u), axis=0)
    assert np.all(np.linalg.norm(got - K @ u, axis=0) <= 1e-12 * scale)
    ko = O.KernelSpec(0.4, 1.3) if kind == "se" else O.KernelSpec(0.4, 1.3, O.SPLINE, -3.0, 40.0, even)
    ref = O.GridKernelOperator(ko, O.Grid(dims, [0.0] * d, [0.05] * d))
    assert np.linalg.norm(got[:, 0] - ref.mvm(u[:, 0])) <= 1e-12 * scale[0]
    want = ref.min_embedding_eigenvalue()
    assert abs(op.min_embedding_eigenvalue() - want) <= 1e-10 * max(abs(want), abs(K[0, 0]))
    assert np.allclose(op.diagonal(), K[0, 0], rtol=1e-15) and np.linalg.norm(op.row(5) - K[5]) <= 1e-12 * np.abs(K[5]).sum()


def test_dski_from_profile_slices_equals_kernel_build():
    """gk_dski_create_from_profile with the spline profile's embedding slice
    and stencil-offset table reproduces the spline D-SKI operator built from
    the kernel (MVM, diagonal, rows)."""
    X, op, ref = spline_pair(2, True, n=150)
    g = op.grid
    k = op.kernel
    kw = dict(ell=k.lengthscale, s=k.outputscale, a=k.spline_a, b=k.spline_b, even=k.spline_even)
    off = gk.GridKernelOperator.embedding_offsets(g)
    W = 11
    tidx = np.stack(np.meshgrid(np.arange(W), np.arange(W), indexing="ij"), -1).reshape(-1, 2)
    toff = (tidx - 5) * np.asarray(g.spacing)
    pop = gk.DskiOperator.from_profile(g, X, profile_values("spline", off, **kw), profile_values("spline", toff, **kw),
                                       noise=(0.2, 0.3))
    V = np.random.default_rng(4).standard_normal((op.size(), 2))
    # the same operator up to the slice's ulp-level differences (numpy vs libm)
    # and the embedding entries beyond the band (zero here, the profile there)
    assert rel(pop.mvm(V), op.mvm(V)) <= 1e-12
    assert rel(pop.diagonal(), op.diagonal()) <= 1e-13
    assert rel(pop.row(17), op.row(17)) <= 1e-12
    assert abs(pop.min_embedding_eigenvalue() - op.min_embedding_eigenvalue()) <= 1e-10 * abs(op.min_embedding_eigenvalue())
