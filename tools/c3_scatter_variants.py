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
N, m = op.size(), grid.size()
st = torch.cuda.current_stream().cuda_stream


def t(stage, a, b, nrhs):
    for _ in range(3):
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for e0, e1 in ev:
        e0.record()
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
        e1.record()
    torch.cuda.synchronize()
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in ev])) * 1e3


for nrhs in (17, 1, 32):
    V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
    O = torch.empty_like(V)
    U = torch.empty(m * nrhs, dtype=torch.float64, device="cuda")
    ref = uref = None
    for var in (0, 7, 8):
        gk.set_tuning("scatter", var)
        mvm = t(3, V, O, nrhs)
        U.fill_(float("nan"))
        sc = t(0, V, U, nrhs)
        if ref is None:
            ref, uref = O.clone(), U.clone()
        err = float((O - ref).norm() / ref.norm())
        uerr = float((U - uref).norm() / uref.norm())
        print(f"nrhs {nrhs} scatter variant {var}: MVM {mvm:.1f} us, scatter {sc:.1f} us, "
              f"rel diff vs default: MVM {err:.1e}, u {uerr:.1e}", flush=True)
    gk.set_tuning("scatter", 0)
