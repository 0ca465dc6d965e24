"""gk_op_mvm from pageable host buffers (C2, 32 RHS, the same preallocated
arrays every call, as bench.py's e2e.pageable): pinned staging through the
host copy pool vs the driver's own pageable copies (tuning "e2e_stage" = 1).
GK_COPY_THREADS sets the pool size."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N, nrhs = op.size(), 32
Pin = np.asfortranarray(rhs_block(N, nrhs, y, dY, 0))
Pout = np.zeros_like(Pin, order="F")
for stage in (1, 0, 1, 0):
    gk.set_tuning("e2e_stage", stage)
    gk._check(gk._lib.gk_op_mvm(op.handle, gk._p(Pin), N, gk._p(Pout), N, nrhs))
    ref = Pout.copy()
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        gk._check(gk._lib.gk_op_mvm(op.handle, gk._p(Pin), N, gk._p(Pout), N, nrhs))
        ts.append(time.perf_counter() - t0)
    print(f"threads {os.environ.get('GK_COPY_THREADS', 'default')} e2e_stage {stage}: median {np.median(ts) * 1e6:.1f} us, "
          f"mean {np.mean(ts) * 1e6:.1f} us, identical {np.array_equal(ref, Pout)}", flush=True)
gk.set_tuning("e2e_stage", 0)
