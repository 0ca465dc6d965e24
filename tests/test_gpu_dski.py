"""GPU parity of the D-SKI operator against the CPU oracle (restated reference).

Mirrors reference proj/tests/test_dski.cpp and SURVEY §8(c): MVM, diagonal,
rows, stacked transpose/apply and the grid kernel MVM must match the
reference algorithm to <= 1e-12 relative (2-norm) on the same seeded inputs.
"""
import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu

TOL = 1e-12  # BASELINE.json north_star: MVM outputs to <= 1e-12 relative in fp64


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def pair(n, d, ell=0.5, s=1.1, spacing=None, max_nodes=24, noise=(0.1, 0.05), order=0, seed=11,
         with_gradients=True, lo=0.0, hi=1.0):
    X = np.random.default_rng(seed).uniform(lo, hi, (n, d))
    grid = gk.Grid.cover(X, spacing or ell / 4, 3, max_nodes)
    g = gk.DskiOperator(gk.KernelSpec(ell, s), grid, X, noise, order, with_gradients)
    r = O.DskiOperator(O.KernelSpec(ell, s), O.Grid(grid.dims, grid.origin, grid.spacing), X, noise,
                       order, with_gradients)
    return g, r, X, grid


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("order", [0, 1])
def test_mvm_matches_oracle(d, order):
    g, r, _, _ = pair(60 if d < 3 else 40, d, order=order, max_nodes=16 if d == 3 else 24)
    rng = np.random.default_rng(30)
    for nrhs in (1, 3, 32):
        V = rng.standard_normal((g.size(), nrhs))
        assert rel(g.mvm(V), r.mvm(V)) <= TOL


def test_mvm_without_gradients_is_plain_ski():
    g, r, _, _ = pair(80, 2, with_gradients=False)
    assert g.size() == 80
    v = np.random.default_rng(1).standard_normal(80)
    assert rel(g.mvm(v), r.mvm(v)) <= TOL


def test_stages_match_oracle():
    g, r, _, grid = pair(120, 2)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(g.size())
    u = rng.standard_normal(grid.size())
    assert rel(g.stacked_transpose_apply(v), r.stacked_transpose_apply(v)) <= TOL
    assert rel(g.stacked_apply(u), r.stacked_apply(u)) <= TOL
    assert rel(g.grid_mvm(u), r.grid_mvm(u)) <= TOL
    assert np.linalg.norm(g.grid_mvm(np.zeros(grid.size()))) == 0.0  # kuu_mvm: zero -> zero


def test_diagonal_and_rows_match_oracle():
    g, r, _, _ = pair(50, 2, s=1.2, noise=(0.1, 0.2), max_nodes=18)  # test_dski.cpp:157-174
    dg, dr = g.diagonal(), r.diagonal()
    assert np.abs(dg - dr).max() <= TOL * dr.max()
    for i in (0, 7, 50, 120, 149):
        row = g.row(i)
        assert rel(row, r.row(i)) <= TOL
        assert abs(row[i] - dg[i]) <= 1e-12 * abs(dg[i])
    with pytest.raises(IndexError):
        g.row(-1)
    with pytest.raises(IndexError):
        g.row(g.size())


def test_diagonal_rows_3d():
    g, r, _, _ = pair(40, 3, max_nodes=14)
    assert np.abs(g.diagonal() - r.diagonal()).max() <= TOL * r.diagonal().max()
    for i in (0, 41, 159):
        assert rel(g.row(i), r.row(i)) <= TOL


def test_size_mismatch_and_out_of_grid():
    g, _, X, grid = pair(30, 2)
    with pytest.raises(ValueError):
        g.mvm(np.zeros(3))  # test_dski.cpp:115
    Xbad = X.copy()
    Xbad[7] = [5.0, 5.0]
    with pytest.raises(gk.OutOfGridError) as e:
        gk.DskiOperator(gk.KernelSpec(0.5, 1.0), grid, Xbad)
    assert e.value.point == 7 and "point 7" in str(e.value)


def test_symmetry_and_psd():
    g, _, _, _ = pair(80, 2, ell=0.4, noise=(0.0, 0.0), max_nodes=24)  # test_dski.cpp:141-155
    rng = np.random.default_rng(60)
    for _ in range(5):
        v = rng.standard_normal(g.size())
        assert v @ g.mvm(v) >= -1e-10 * (v @ v)
    u, v = rng.standard_normal(g.size()), rng.standard_normal(g.size())
    a, b = u @ g.mvm(v), g.mvm(u) @ v
    assert abs(a - b) <= 1e-10 * abs(a)


def test_config_c1_mvm_parity_and_fidelity():
    """C1 (BASELINE configs[0]): 60x60 grid, n=2000, ell=0.15 — MVM parity vs the
    oracle and fidelity vs the exact D-SE K∇ (c02 analogue, ~1e-5)."""
    X, y, dY = gk.make_dataset(1, 0)
    grid = gk.Grid.cover(X, 1e-3, 3, 60)
    assert list(grid.dims) == [60, 60]
    g = gk.DskiOperator(gk.KernelSpec(0.15, 1.0), grid, X, (1e-2, 1e-2))
    r = O.DskiOperator(O.KernelSpec(0.15, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X,
                       (1e-2, 1e-2))
    V = np.random.default_rng(2).standard_normal((g.size(), 9))
    assert rel(g.mvm(V), r.mvm(V)) <= TOL
    ex = gk.ExactOperator(gk.KernelSpec(0.15, 1.0), X, (1e-2, 1e-2))
    E = ex.mvm(V)
    err = np.abs(g.mvm(V) - E).max() / np.abs(E).max()
    # fidelity (interpolation error at ell/h ~ 7.95), not parity: the GPU and
    # the oracle carry the same approximation
    r_err = np.abs(r.mvm(V) - E).max() / np.abs(E).max()
    assert abs(err - r_err) <= 1e-10 and err < 5e-4


def test_exact_operator_matches_dense_assembly():
    X = np.random.default_rng(3).uniform(0, 1, (70, 2))
    k = gk.KernelSpec(0.3, 1.2)
    ex = gk.ExactOperator(k, X, (0.05, 0.02))
    A = O.assemble_dense(O.KernelSpec(0.3, 1.2), X)
    nd = np.r_[np.full(70, 0.05 ** 2), np.full(140, 0.02 ** 2)]
    A = A + np.diag(nd)
    V = np.random.default_rng(4).standard_normal((210, 5))
    assert rel(ex.mvm(V), A @ V) <= TOL
    assert np.abs(ex.diagonal() - np.diag(A)).max() <= 1e-13
    for i in (0, 69, 70, 209):
        assert rel(ex.row(i), A[i]) <= TOL


def test_dense_operator_roundtrip():
    A = np.random.default_rng(5).standard_normal((40, 40))
    op = gk.DenseOperator(A)
    v = np.random.default_rng(6).standard_normal((40, 3))
    assert rel(op.mvm(v), A @ v) <= 1e-14
    assert np.allclose(op.diagonal(), np.diag(A))
    assert np.allclose(op.row(3), A[3])


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("nrhs", [1, 5, 17, 32, 33, 64])
def test_fused_2d_mvm_matches_oracle_and_staged_path(order, nrhs):
    """The one-launch d = 2 MVM (fused2d.cu) against the oracle and against the
    staged scatter / K_UU / gather kernels, over RHS counts that exercise
    partial lanes (5, 17), exactly one chunk (32) and two chunks (33, 64)."""
    g, r, _, _ = pair(700, 2, ell=0.3, order=order, max_nodes=40, seed=3)
    V = np.random.default_rng(nrhs).standard_normal((g.size(), nrhs))
    ref = r.mvm(V)
    launches0 = gk.kernel_launch_count()
    got = g.mvm(V)
    assert rel(got, ref) <= TOL
    prev = gk.set_tuning("fused", 1)
    try:
        staged = g.mvm(V)
    finally:
        gk.set_tuning("fused", prev)
    assert rel(staged, ref) <= TOL
    assert rel(got, staged) <= 1e-13
    assert np.array_equal(got, g.mvm(V))  # deterministic (no atomics)
    assert gk.kernel_launch_count() > launches0


def test_fused_2d_mvm_clustered_points_and_graph_replay():
    """Points piled into a few cells (max cell occupancy >> mean) size the
    staging windows from the data; the graph-replayed MVM equals the direct one."""
    rng = np.random.default_rng(8)
    X = np.concatenate([rng.uniform(0, 1, (300, 2)), 0.5 + 0.004 * rng.standard_normal((400, 2))])
    grid = gk.Grid.cover(X, 0.02, 3, 48)
    g = gk.DskiOperator(gk.KernelSpec(0.25, 1.3), grid, X, (0.05, 0.1))
    r = O.DskiOperator(O.KernelSpec(0.25, 1.3), O.Grid(grid.dims, grid.origin, grid.spacing), X, (0.05, 0.1))
    V = rng.standard_normal((g.size(), 32))
    assert rel(g.mvm(V), r.mvm(V)) <= TOL
    import torch
    dev = torch.device("cuda", 0)
    Vi = torch.empty(g.size() * 32, dtype=torch.float64, device=dev)
    Ve = torch.from_numpy(np.ascontiguousarray(V.T)).to(dev)
    g.to_internal_dev(Ve.data_ptr(), Vi.data_ptr(), 32)
    O1, O2 = torch.empty_like(Vi), torch.empty_like(Vi)
    g.stage_dev(3, Vi.data_ptr(), O1.data_ptr(), 32)
    for _ in range(3):
        g.stage_dev(4, Vi.data_ptr(), O2.data_ptr(), 32)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)


@pytest.mark.parametrize("smode,gmode", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_fused_2d_variants_match_oracle(smode, gmode):
    """Staged (shared-memory rolling) and direct-load scatter/gather variants of
    the one-launch MVM give the same operator; graph replays are refreshed when
    the plan changes."""
    g, r, _, _ = pair(900, 2, ell=0.3, max_nodes=40, seed=21)
    import torch
    prev = (gk.set_tuning("f2_smode", smode), gk.set_tuning("f2_gmode", gmode))
    try:
        for nrhs in (1, 6, 32, 40):
            V = np.random.default_rng(nrhs + smode).standard_normal((g.size(), nrhs))
            assert rel(g.mvm(V), r.mvm(V)) <= TOL
        dev = torch.device("cuda", 0)
        Vi = torch.randn(g.size() * 32, dtype=torch.float64, device=dev)
        O1, O2 = torch.empty_like(Vi), torch.empty_like(Vi)
        g.stage_dev(3, Vi.data_ptr(), O1.data_ptr(), 32)
        g.stage_dev(4, Vi.data_ptr(), O2.data_ptr(), 32)
        torch.cuda.synchronize()
        assert torch.equal(O1, O2)
    finally:
        gk.set_tuning("f2_smode", prev[0])
        gk.set_tuning("f2_gmode", prev[1])


@pytest.mark.parametrize("with_gradients", [True, False])
@pytest.mark.parametrize("order", [0, 1])
def test_d3_tile_scatter_matches_oracle(order, with_gradients):
    """The d = 3 column-tile scatter (k_scatter_tile3; default for 1-2 RHS,
    forced here for every count) against the oracle: points piled onto a few
    z-levels (units that cannot split inside one base cell level), RHS counts
    below, at and above one RHS chunk (36 columns x RC <= 1024 threads), and
    the per-column list scatter it replaces."""
    rng = np.random.default_rng(8)
    X = rng.uniform(0.0, 1.0, (300, 3))
    X[:150, 2] = 0.5 + 1e-3 * rng.standard_normal(150)  # a dense sheet: many entries per (tile, z)
    grid = gk.Grid.cover(X, 0.05, 3, 20)
    g = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (0.1, 0.05), order, with_gradients)
    r = O.DskiOperator(O.KernelSpec(0.3, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X, (0.1, 0.05),
                       order, with_gradients)
    for nrhs in (1, 2, 5, 33):
        V = rng.standard_normal((g.size(), nrhs))
        ref = r.mvm(V)
        prev = gk.set_tuning("scatter", 8)
        try:
            tile = g.mvm(V)
        finally:
            gk.set_tuning("scatter", prev)
        prev = gk.set_tuning("scatter", 6)
        try:
            lists = g.mvm(V)
        finally:
            gk.set_tuning("scatter", prev)
        assert rel(tile, ref) <= TOL
        assert rel(tile, lists) <= 1e-13
        default = g.mvm(V)  # unit push + merge with gradients, ≤ 32 RHS; else tiles / lists
        assert rel(default, ref) <= TOL and rel(default, lists) <= 1e-13


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("nrhs", [1, 2, 5, 6, 8, 16, 17, 21, 33, 64])
def test_d3_unit_paths_bit_identical_and_match_oracle(nrhs, order):
    """The d = 3 unit-push scatter (staged, and the direct variant for
    T*nrhs <= 32), the merge over per-node lists and the gather's 16-column
    task blocks (with the compile-time 16/17-column instantiations) against
    the oracle, and bit for bit against the earlier variants they replaced
    (tuning "d3": 1 list-walk merge, 4 staged push for few RHS, 1024 lean gather, 512 runtime
    RHS count in the gather)."""
    rng = np.random.default_rng(31 + nrhs)
    X = rng.uniform(0.0, 1.0, (700, 3))
    X[:300, 2] = 0.5 + 1e-3 * rng.standard_normal(300)  # a dense sheet: long units, many points per cell
    grid = gk.Grid.cover(X, 0.05, 3, 24)
    g = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (0.1, 0.05), order)
    r = O.DskiOperator(O.KernelSpec(0.3, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X, (0.1, 0.05), order)
    V = rng.standard_normal((g.size(), nrhs))
    ref = r.mvm(V)
    default = g.mvm(V)
    assert rel(default, ref) <= TOL
    prev = gk.set_tuning("d3", 1 | 4 | 512 | 4096 | 16384)
    try:
        old = g.mvm(V)
    finally:
        gk.set_tuning("d3", prev)
    assert np.array_equal(default, old)


@pytest.mark.parametrize("lean", [1, 2])  # 1: fused2d one-launch kernel, 2: lean2d one-launch kernel
@pytest.mark.parametrize("ell,n", [(0.5, 60), (0.4, 80), (0.3, 150)])  # grids 15², 17² (partial last segment), 21²
def test_one_launch_2d_kernels_match_oracle(lean, ell, n):
    g, r, _, _ = pair(n, 2, ell=ell, max_nodes=40)
    rng = np.random.default_rng(n)
    try:
        gk.set_tuning("lean", lean)
        for nrhs in (1, 2, 3, 8, 32, 33, 64):
            V = rng.standard_normal((g.size(), nrhs))
            assert rel(g.mvm(V), r.mvm(V)) <= TOL, nrhs
    finally:
        gk.set_tuning("lean", 0)


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_device_point_tables_bit_identical_to_host_build(cfg):
    """The D-SKI constructor's point tables built on the GPU (stencil weights
    with the host formula's rounding, CUB stable radix sort by base cell, cell
    starts) give bit-identical operators to the host build (tuning "devbuild")."""
    X, *_ = gk.make_dataset(cfg, 0)
    ell, nodes = {1: (0.15, 60), 3: (0.3, 48), 4: (0.02, 400)}[cfg]
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    V = np.random.default_rng(cfg).standard_normal((X.shape[0] * (X.shape[1] + 1), 3))
    try:
        gk.set_tuning("devbuild", 1)
        host = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
        a = host.mvm(V)
        gk.set_tuning("devbuild", 0)
        dev = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
        b = dev.mvm(V)
    finally:
        gk.set_tuning("devbuild", 0)
    assert np.array_equal(a, b)
    assert np.array_equal(host.diagonal(), dev.diagonal())


def test_device_build_reports_out_of_grid_point():
    X = np.random.default_rng(3).uniform(0, 1, (50, 2))
    grid = gk.Grid.cover(X, 0.1, 3, 24)
    X2 = X.copy()
    X2[17, 1] = 5.0  # outside the grid interior
    with pytest.raises(gk.OutOfGridError) as e:
        gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X2, (0.1, 0.1))
    assert e.value.point == 17 and "point 17" in str(e.value)
