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
