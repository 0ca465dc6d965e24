"""fused2d one-launch MVM at C2 with phases skipped (tuning f2_skip bitmask:
1 scatter, 2 mode 1, 4 mode 0, 8 gather): kernel time per configuration
(CUDA events, L2 evicted), isolating each phase's cost from barrier skew."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402
from tools.lean_timing import timeit  # noqa: E402

os.environ["GK_FUSED_PLAN_PRINT"] = "1"
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
op = problem(cfg)
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
gk.set_tuning("lean", 1)
names = {0: "all phases", 15: "none (launch + 3 barriers)", 14: "scatter only", 13: "mode1 only", 11: "mode0 only",
         7: "gather only", 1: "all but scatter", 2: "all but mode1", 4: "all but mode0", 8: "all but gather"}
for mask, name in names.items():
    gk.set_tuning("f2_skip", mask)
    print(f"{cfg} nrhs={nrhs} skip={mask:2d} ({name:28s}): {timeit(op, V, O, nrhs):7.2f} us", flush=True)
gk.set_tuning("f2_skip", 0)
