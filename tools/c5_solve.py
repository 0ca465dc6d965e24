"""C5 solve: rank-100 pivoted Cholesky, PCG over 64 RHS (y + 63 probes), SLQ
64 probes × 50 steps on the D-SKIP operator."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


X, y, dY = gk.make_dataset(5, 0)
op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
N = op.size()
t0 = t()
fac = gk.pivoted_cholesky(op, 100, kernel_part=True)
M = gk.Preconditioner.from_pivchol(op, fac)
t1 = t()
B = np.column_stack([gk.stacked_targets(y, dY, y.mean())] + [gk.rademacher_vector(N, 0, 1000 + p) for p in range(63)])
Vext = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
Xd = torch.empty_like(Vext)
t2 = t()
its, conv = gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), 64, 1e-4, 1000, M)
t3 = t()
r = gk.slq_logdet(op, 64, 50, 0, 0.5e-4)
t4 = t()
print(f"C5 solve: pivchol+precond {t1-t0:.3f} s, PCG(64 RHS, tol 1e-4) {t3-t2:.3f} s its {list(its[:4])}.. max {max(its)} "
      f"conv {sum(conv)}/64, SLQ(64x50) {t4-t3:.3f} s logdet {r.logdet:.6e}", flush=True)
