"""fused2d knob sweep at C2 (L2 evicted, CUDA events): GK_SWEEP="knob=v1,v2,..." """
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402
from tools.lean_timing import timeit  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
op = problem(cfg)
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
gk.set_tuning("lean", 1)
for spec in os.environ.get("GK_SWEEP", "f2_tsplit=0,1,2,3,4,6").split(";"):
    knob, vals = spec.split("=")
    for v in vals.split(","):
        old = gk.set_tuning(knob, int(v))
        print(f"{cfg} nrhs={nrhs} {knob}={v}: {timeit(op, V, O, nrhs):7.2f} us", flush=True)
        gk.set_tuning(knob, old)
