"""PCG iteration cost on C2 (32 RHS, rank-50 preconditioner): fused vector
step vs the ten-kernel path, fixed iteration count."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N, nrhs = op.size(), 32
M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 50, kernel_part=True))
B = rhs_block(N, nrhs, y, dY, 0)
dev = torch.device("cuda")
Vext = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev)
Xd = torch.empty_like(Vext)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 200
res = {5: [], 1: [], 3: [], 2: []}
for rep in range(int(os.environ.get("REPS", "3"))):
    for fused in (5, 1, 3, 2):
        gk.set_tuning("pcg_fused", fused)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, conv = gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), nrhs, float(os.environ.get("TOL", "1e-12")), its, M)
        torch.cuda.synchronize()
        res[fused].append((time.perf_counter() - t0) / its * 1e6)
for fused in (5, 1, 3, 2):
    print(f"pcg_fused={fused} ({ {5: 'persistent MVM + v2 step', 1: 'graphs: MVM + v2 step', 3: 'graphs: MVM + v1 step', 2: 'separate kernels'}[fused]}): "
          f"{its} iterations, min {min(res[fused]):.1f} us/iteration (all {[round(x, 1) for x in res[fused]]})",
          flush=True)
gk.set_tuning("pcg_fused", 0)
