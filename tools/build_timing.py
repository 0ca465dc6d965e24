"""D-SKI operator construction wall time: on-device point tables vs the host build."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

for cfg, ell, nodes in ((2, 0.2, 100), (3, 0.3, 48), (4, 0.02, 400)):
    X, *_ = gk.make_dataset(cfg, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    for knob in (0, 1, 0, 1):
        gk.set_tuning("devbuild", knob)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
        torch.cuda.synchronize()
        print(f"C{cfg} build ({'device tables' if knob == 0 else 'host tables  '}): {(time.perf_counter() - t0) * 1e3:8.2f} ms",
              flush=True)
        del op
    gk.set_tuning("devbuild", 0)
