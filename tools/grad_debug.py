"""Per-probe comparison of the lml_gradient trace solves (GPU vs oracle)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1810_12283_b200 as gk  # noqa: E402

ELL, RATIO, MAXN, RANK = 0.15, 0.1, 40, 40
NOISE = (float(os.environ.get("NOISE", "0.05")),) * 2
X, y, dY = gk.make_dataset(1, 0)
X, y, dY = X[:300], y[:300], dY[:300]
grid = gk.Grid.cover(X, RATIO * ELL, 3, MAXN)
og = O.Grid(grid.dims, grid.origin, grid.spacing)
op = gk.DskiOperator(gk.KernelSpec(ELL, 1.0), grid, X, NOISE)
ref = O.DskiOperator(O.KernelSpec(ELL, 1.0), og, X, NOISE)
nd = ref.noise_diagonal()
F = O.pivoted_cholesky(ref, RANK, noise_diag=nd)
Po = O.Preconditioner(F.L, nd)
P = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, RANK, kernel_part=True))
N = op.size()
Z = np.stack([gk.rademacher_vector(N, 3, 1000 + q) for q in range(8)], 1)
sg = gk.cg(op, Z, 1e-2, 5000, P)
for q in range(8):
    so = O.cg(ref, Z[:, q], 1e-2, 5000, Po)
    hg = np.asarray(sg[q].residual_history) if isinstance(sg, list) else None
    print(q, "its gpu", sg[q].iterations if isinstance(sg, list) else None, "oracle", so.iterations,
          "x rel", np.linalg.norm(sg[q].x - so.x) / np.linalg.norm(so.x) if isinstance(sg, list) else None,
          "hist gpu", None if hg is None else hg[-3:], "oracle", so.residual_history[-3:])
