"""C2 32-RHS one-launch MVM: direct cooperative launch (stage 3) vs the
cached CUDA-graph replay (stage 4), L2 evicted and back-to-back."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.fused_timing import problem, timeit, b2b  # noqa: E402

for cfg, nrhs in [("C2", 32), ("C1", 32), ("C4", 1)]:
    op = problem(cfg)
    V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
    O3, O4 = torch.empty_like(V), torch.empty_like(V)
    t3, t4 = timeit(op, 3, V, O3, nrhs), timeit(op, 4, V, O4, nrhs)
    b3, b4 = b2b(op, 3, V, O3, nrhs), b2b(op, 4, V, O4, nrhs)
    print(f"{cfg} {nrhs}: launch {t3:.2f} us / graph {t4:.2f} us (L2 evicted); b2b {b3:.2f} / {b4:.2f}; "
          f"identical {torch.equal(O3, O4)}", flush=True)
