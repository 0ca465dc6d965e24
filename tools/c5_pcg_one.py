"""A few C5 PCG iterations (64 RHS, rank-100 preconditioner) inside
cudaProfilerStart/Stop for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(5, 0)
op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
N = op.size()
M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 100, kernel_part=True))
B = np.column_stack([gk.rademacher_vector(N, 0, 1000 + p) for p in range(64)])
Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
Xd = torch.empty_like(Bd)
gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 64, 1e-12, 5, M)
torch.cuda.synchronize()
torch.cuda.profiler.start()
gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 64, 1e-12, 3, M)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
