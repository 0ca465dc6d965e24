"""C2 SLQ (31 probes x 30 steps) once warm, then once inside
cudaProfilerStart/Stop for `ncu --profile-from-start off`; prints wall time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY, grid = bench.build_problem()
c = bench.CONFIG
op = gk.DskiOperator(gk.KernelSpec(c["ell"], 1.0), grid, X, (c["noise"], c["noise"]))
r = gk.slq_logdet(op, c["slq_probes"], c["slq_steps"], 0, 0.5e-4)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = gk.slq_logdet(op, c["slq_probes"], c["slq_steps"], 0, 0.5e-4)
torch.cuda.synchronize()
print("slq wall", time.perf_counter() - t0, r.logdet, flush=True)
if os.environ.get("PROFILE"):
    torch.cuda.profiler.start()
    r = gk.slq_logdet(op, c["slq_probes"], c["slq_steps"], 0, 0.5e-4)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
