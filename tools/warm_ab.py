"""A/B of one-launch 2-D MVM tuning keys (default f2_warm, the instruction
warm-up inside the split barriers): event-timed median with L2 evicted,
back-to-back throughput, and bit-identity of the outputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem, timeit, b2b  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "f2_warm"
vals = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
for cfg, nrhs in [("C2", 32), ("C1", 32), ("C2", 1), ("C4", 1)]:
    op = problem(cfg)
    V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
    outs = []
    for v in vals:
        gk.set_tuning(key, v)
        O = torch.empty_like(V)
        t = timeit(op, 3, V, O, nrhs)
        tb = b2b(op, 3, V, O, nrhs)
        outs.append(O.clone())
        print(f"{cfg} nrhs={nrhs} {key}={v}: {t:.2f} us (L2 evicted), {tb:.2f} us back-to-back", flush=True)
    print("   identical:", all(torch.equal(outs[0], o) for o in outs[1:]))
