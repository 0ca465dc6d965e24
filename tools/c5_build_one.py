"""Build the C5 D-SKIP operator once (for ncu launch lists of the build)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(5, 0)
op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
torch.cuda.synchronize()
print("ok")
