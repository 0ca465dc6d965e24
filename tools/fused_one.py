"""Run the one-launch MVM a few times (for ncu capture): fused_one.py CFG NRHS [knob=value ...]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
for k, v in (a.split("=") for a in sys.argv[3:]):
    gk.set_tuning(k, int(v))
op = problem(cfg)
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
for _ in range(5):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
torch.cuda.synchronize()
print("ok")
