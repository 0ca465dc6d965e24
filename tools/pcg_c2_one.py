"""30 C2 PCG iterations (32 RHS, rank-50 preconditioner) for ncu captures of
the fused vector step (e.g. -k regex:k_pcg_vec2 -s 10 -c 1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 50, kernel_part=True))
B = rhs_block(N, 32, y, dY, 0)
V = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
Xd = torch.empty_like(V)
gk.cg_dev(op, V.data_ptr(), Xd.data_ptr(), 32, 1e-12, 30, M)
torch.cuda.synchronize()
print("ok")
