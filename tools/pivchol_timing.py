"""Pivoted Cholesky (kernel part) wall time: device-resident pivot loop vs the
host-synchronised loop (tuning "pivchol" = 1), C2 rank 50 and C4 rank 200."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

for cfg, ell, nodes, rank in ((2, 0.2, 100, 50), (4, 0.02, 400, 200)):
    X, *_ = gk.make_dataset(cfg, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
    for knob in (0, 1, 0):
        gk.set_tuning("pivchol", knob)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = gk.pivoted_cholesky(op, rank, kernel_part=True)
        torch.cuda.synchronize()
        print(f"C{cfg} rank {rank} {'device loop' if knob == 0 else 'host loop  '}: {(time.perf_counter() - t0) * 1e3:8.2f} ms",
              flush=True)
    gk.set_tuning("pivchol", 0)
