"""K_UU (stage 1) and whole-MVM times for the spline profile (circulant
embedding + in-house FFT) beside the SE Toeplitz path on the C2/C3/C4 grids."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def tm(fn, reps=20):
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.sum()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


for cfg, ell, nodes, nrhs in [(2, 0.2, 100, 32), (3, 0.3, 48, 17), (4, 0.02, 400, 1)]:
    X, y, dY = gk.make_dataset(cfg, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    d = X.shape[1]
    D = float(np.sqrt(d)) / ell
    a, b, even = gk.spline_constants_for_domain(D, d)
    for name, k in (("se", gk.KernelSpec(ell, 1.0)), ("spline", gk.KernelSpec(ell, 1.0, gk.SPLINE, a, b, even))):
        op = gk.DskiOperator(k, grid, X, (1e-2, 1e-2))
        M, N = op.grid_size(), op.size()
        U = torch.randn(M * nrhs, dtype=torch.float64, device="cuda")
        W = torch.empty_like(U)
        V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
        O = torch.empty_like(V)
        tk = tm(lambda: op.stage_dev(1, U.data_ptr(), W.data_ptr(), nrhs, stream=st))
        tv = tm(lambda: op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st))
        print(f"C{cfg} grid {list(grid.dims)} {nrhs} RHS {name}: K_UU {tk:.1f} us, MVM {tv:.1f} us", flush=True)
