"""Grid-slab sharded D-SKI MVM (paper_1810_12283_b200.slab) through NCCL on
the GPU: one rank here (a single GPU per test box; two ranks on one GPU would
wait on each other), so this exercises the code path — partition, local
scatter into the full grid, NCCL all-reduce, K_UU, gather with noise — against
the single-operator MVM and the oracle. The multi-rank logic (slab partition,
halo-free summation) is covered on CPU with gloo in tests/test_sharding_gloo.py."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("nrhs", [1, 8])
def test_slab_sharded_mvm_matches_single_operator_and_oracle(pg, nrhs):
    from paper_1810_12283_b200.slab import SlabShardedDskiOperator
    X, *_ = gk.make_dataset(4, 0)
    X = X[:20000]
    grid = gk.Grid.cover(X, 1e-4, 3, 160)
    k, noise = gk.KernelSpec(0.02, 1.0), (1e-2, 1e-2)
    sop = SlabShardedDskiOperator(k, grid, X, noise)
    full = gk.DskiOperator(k, grid, X, noise)
    V = np.random.default_rng(nrhs).standard_normal((sop.size(), nrhs))
    got = sop.mvm(V)
    ref = full.mvm(V)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    oref = O.DskiOperator(O.KernelSpec(0.02, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X, noise).mvm(V[:, :2])
    assert np.linalg.norm(got[:, :2] - oref) <= 1e-12 * np.linalg.norm(oref)


def test_slab_sharded_solvers_on_gpu_match_oracle(pg):
    """The row-sharded pivoted Cholesky / preconditioner / PCG
    (paper_1810_12283_b200.slab_solver) through the GPU backend — library
    kernels for the slab MVM, cross-covariance columns and the split Woodbury
    apply; NCCL for the all-reduces — against the single-process reference
    algorithms (oracle): pivots bit-exact, M⁻¹b ≤1e-10, PCG iterations equal
    and the solution to tolerance."""
    import torch
    from paper_1810_12283_b200 import slab_solver as S
    from paper_1810_12283_b200.slab import SlabShardedDskiOperator
    X = np.random.default_rng(5).uniform(0, 1, (250, 2))
    grid = gk.Grid.cover(X, 0.3 / 4, 3, 40)
    noise = (0.5, 0.4)
    sop = SlabShardedDskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, noise)
    be = S.GpuSlabBackend(sop)
    f = S.slab_pivoted_cholesky(be, 40)
    M = S.SlabPreconditioner(be, f.L, be.noise_diag())
    og = O.Grid(grid.dims, grid.origin, grid.spacing)
    op = O.DskiOperator(O.KernelSpec(0.3, 1.0), og, X, noise)
    nd = op.noise_diagonal()
    fr = O.pivoted_cholesky(op, 40, noise_diag=nd)
    assert [int(p) for p in f.pivots] == [int(p) for p in fr.pivots]
    Pr = O.Preconditioner(fr.L, nd)
    b = np.random.default_rng(9).standard_normal(op.size())
    bl = torch.from_numpy(b[be.rows].reshape(-1, 1).copy()).to(be.dev)
    z = M.apply(bl).cpu().numpy()[:, 0]
    zr = Pr.apply(b)[be.rows]
    assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr)
    res = S.slab_cg(be, bl, 1e-9, 500, M)
    rr = O.cg(op, b, 1e-9, 500, Pr)
    assert res.iterations[0] == rr.iterations and res.converged[0] == rr.converged
    x = res.X.cpu().numpy()[:, 0]
    assert np.linalg.norm(x - rr.x[be.rows]) <= 1e-8 * np.linalg.norm(rr.x)
