"""One C2 SLQ (31 probes x 30 Lanczos steps) inside cudaProfilerStart/Stop,
after a warm-up call (for ncu --profile-from-start off)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem  # noqa: E402

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
gk.slq_logdet(op, 31, 30, 0, 0.5e-4)
torch.cuda.synchronize()
t0 = time.perf_counter()
gk.slq_logdet(op, 31, 30, 0, 0.5e-4)
print(f"slq wall {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
torch.cuda.profiler.start()
gk.slq_logdet(op, 31, 30, 0, 0.5e-4)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
