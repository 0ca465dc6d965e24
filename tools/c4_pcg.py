"""C4 (n = 150,000, N = 450,000, grid 400², ℓ = 0.02): rank-200 pivoted
Cholesky + preconditioner build, and 50 PCG iterations on the targets (1 RHS);
per-iteration time."""
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


X, y, dY = gk.make_dataset(4, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 400)
op = gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
t0 = t()
fac = gk.pivoted_cholesky(op, 200, kernel_part=True)
t1 = t()
M = gk.Preconditioner.from_pivchol(op, fac)
t2 = t()
b = gk.stacked_targets(y, dY, y.mean())
Bd = torch.from_numpy(b).cuda()
Xd = torch.empty_like(Bd)
gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 1, 1e-12, 5, M)
t3 = t()
its, conv = gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 1, 1e-12, 50, M)
t4 = t()
print(f"C4 N={N}: pivchol(200) {t1-t0:.3f} s, precond build {t2-t1:.3f} s, PCG {(t4-t3)/50*1e6:.1f} us/iteration", flush=True)
t5 = t()
its, conv = gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 1, 1e-4, 1000, M)
t6 = t()
print(f"C4 PCG tol 1e-4, its {its[0]}: {(t6-t5)/max(1, its[0])*1e6:.1f} us/iteration", flush=True)
if os.environ.get("PROFILE"):
    torch.cuda.profiler.start()
    gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 1, 1e-12, 3, M)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
