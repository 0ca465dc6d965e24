"""BASELINE.json's five configurations at FULL size, checked through
size-independent properties of K∇ (the oracle cannot run them in seconds):
symmetry uᵀ(Kv) = vᵀ(Ku), linearity, batched vs per-column MVMs, rows and the
diagonal vs unit-vector MVMs, and the noise floor vᵀKv ≥ min(σ)²‖v‖² (the
kernel part is positive semidefinite). Parity with the oracle at these
operators' reduced sizes is in test_gpu_dski.py / test_gpu_dskip.py, and the
full-size C2 solve is pinned by tests/golden/c2_cg.json."""
import numpy as np
import pytest

import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu

NOISE = (1e-2, 1e-2)


def build(cfg):
    X, y, dY = gk.make_dataset(cfg, 0)
    if cfg == 5:  # D-SKIP, product SE ℓ = 0.3, rank 30 on 100-node 1-D grids
        return gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, NOISE, rank=30, grid_ratio=0.01,
                                max_grid_nodes=100, seed=0), X
    ell, nodes = {1: (0.15, 60), 2: (0.2, 100), 3: (0.3, 48), 4: (0.02, 400)}[cfg]
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    return gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, NOISE), X


@pytest.fixture(scope="module", params=[1, 2, 3, 4, 5], ids=lambda c: f"C{c}")
def cfg_op(request):
    op, X = build(request.param)
    return request.param, op, X


def test_full_size(cfg_op):
    cfg, op, X = cfg_op
    N = op.size()
    assert N == X.shape[0] * (X.shape[1] + 1)
    rng = np.random.default_rng(100 + cfg)
    V = rng.standard_normal((N, 4))
    KV = op.mvm(V)
    # batched == per column (columns are independent in every kernel)
    for c in (0, 3):
        assert np.linalg.norm(op.mvm(V[:, c]) - KV[:, c]) <= 1e-13 * np.linalg.norm(KV[:, c])
    # symmetry
    for a, b in ((0, 1), (2, 3)):
        lhs, rhs = V[:, a] @ KV[:, b], V[:, b] @ KV[:, a]
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(V[:, a]) * np.linalg.norm(KV[:, b]), (lhs, rhs)
    # linearity
    comb = op.mvm(2.5 * V[:, 0] - 0.75 * V[:, 1])
    assert np.linalg.norm(comb - (2.5 * KV[:, 0] - 0.75 * KV[:, 1])) <= 1e-13 * np.linalg.norm(comb)
    # noise floor: vᵀKv ≥ min σ² ‖v‖² (kernel part PSD, up to roundoff)
    for c in range(4):
        q = V[:, c] @ KV[:, c]
        assert q >= min(NOISE) ** 2 * (V[:, c] @ V[:, c]) * (1 - 1e-9), (c, q)
    # rows and diagonal against unit-vector MVMs (value and gradient blocks)
    n = X.shape[0]
    idx = [0, n // 2, n + 7, N - 1]
    E = np.zeros((N, len(idx)))
    for j, i in enumerate(idx):
        E[i, j] = 1.0
    KE = op.mvm(E)
    diag = op.diagonal()
    for j, i in enumerate(idx):
        r = op.row(i)
        assert np.linalg.norm(r - KE[:, j]) <= 1e-12 * np.linalg.norm(KE[:, j]), i
        assert abs(diag[i] - KE[i, j]) <= 1e-12 * abs(KE[i, j]), i


def test_c2_probe_sharding_reproduces_single_batch():
    """SURVEY §8(e) probe sharding at full C2 size: the 31 SLQ probes run as one
    batch, or as two shards with probe offsets (what two ranks run), give the
    same per-probe estimates (batch composition only moves roundoff: the
    MVM's decomposition depends on the batch width), and the probe-ordered
    mean reproduces the single-batch log-det."""
    op, X = build(2)
    full = gk.slq_logdet(op, 31, 30, 0, 0.5e-4)
    a = gk.slq_logdet(op, 16, 30, 0, 0.5e-4, probe_offset=0)
    b = gk.slq_logdet(op, 15, 30, 0, 0.5e-4, probe_offset=16)
    est = np.concatenate([a.estimates, b.estimates])
    assert np.allclose(est, full.estimates, rtol=1e-10, atol=0)
    assert abs(np.sum(est) / 31 - full.logdet) <= 1e-10 * abs(full.logdet)
