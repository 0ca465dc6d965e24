"""One C3 scatter (17 RHS) inside cudaProfilerStart/Stop (ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(3, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (1e-2, 1e-2))
nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 17
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
for _ in range(3):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
torch.cuda.synchronize()
torch.cuda.profiler.start()
op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
