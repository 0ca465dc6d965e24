"""A few C3 PCG iterations (17 RHS, rank-100 preconditioner) inside
cudaProfilerStart/Stop for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(3, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 100, kernel_part=True))
B = np.column_stack([gk.stacked_targets(y, dY, y.mean())] + [gk.rademacher_vector(N, 0, 1000 + p) for p in range(16)])
Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
Xd = torch.empty_like(Bd)
gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 17, 1e-12, 5, M)
torch.cuda.synchronize()
torch.cuda.profiler.start()
gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 17, 1e-12, 3, M)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
