"""C3 batched MVM (17 RHS) time per scatter variant (tuning "scatter")."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(3, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (1e-2, 1e-2))
N, nrhs = op.size(), 17
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
st = torch.cuda.current_stream().cuda_stream
ref = None
for var in (0, 4, 5, 6, 7, 1, 3):
    gk.set_tuning("scatter", var)
    for _ in range(3):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev:
        a.record()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
        b.record()
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    if ref is None:
        ref = O.clone()
    err = float((O - ref).norm() / ref.norm())
    print(f"scatter variant {var}: MVM {ms*1e3:.1f} us, rel diff vs default {err:.1e}", flush=True)
gk.set_tuning("scatter", 0)
