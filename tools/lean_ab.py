"""A/B of lean2d knobs at C2 32 RHS (phase stamps)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402
from tools.lean_timing import timeit  # noqa: E402

op = problem("C2")
nrhs = 32
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
gk.set_tuning("lean", 2)
for knob in (0, 7):
    gk.set_tuning("f2_nst", knob)
    t = timeit(op, V, O, nrhs)
    gk.set_tuning("fused_prof", 1)
    rows = []
    for _ in range(10):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
        torch.cuda.synchronize()
        st = gk.debug_fused_phases(op, nrhs)
        rows.append(np.median(np.diff(st, axis=1), axis=0) / 1e3)
    gk.set_tuning("fused_prof", 0)
    print(f"knob {knob}: {t:.2f} us; median per-CTA phase us [S b1 T1 b2 T0 b3 G]:",
          np.round(np.median(rows, axis=0), 2), flush=True)
