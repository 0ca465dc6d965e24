"""C3 (17 RHS) MVM stages with L2 evicted before each call: scatter, K_UU,
gather (per variant), and the whole MVM; per-unit gather parity vs lean."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(3, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (1e-2, 1e-2))
N, nrhs, M = op.size(), int(sys.argv[1]) if len(sys.argv) > 1 else 17, grid.size()
st = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
U = torch.randn(M * nrhs, dtype=torch.float64, device="cuda")
W = torch.empty_like(U)
O1, O2 = torch.empty_like(V), torch.empty_like(V)


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


res = {}
for var in (0, 3):  # 0: default (cell-line units for d = 3), 3: the previous lean gather
    gk.set_tuning("gather", var)
    res[f"gather[{var}]"] = tm(lambda: op.stage_dev(2, U.data_ptr(), O1.data_ptr() if var == 0 else O2.data_ptr(), nrhs, stream=st))
gk.set_tuning("gather", 0)
err = float((O1 - O2).norm() / O2.norm())
res["scatter"] = tm(lambda: op.stage_dev(0, V.data_ptr(), W.data_ptr(), nrhs, stream=st))
res["kuu"] = tm(lambda: op.stage_dev(1, U.data_ptr(), W.data_ptr(), nrhs, stream=st))
res["mvm"] = tm(lambda: op.stage_dev(3, V.data_ptr(), O1.data_ptr(), nrhs, stream=st))
print(f"C3 nrhs={nrhs}: " + "  ".join(f"{k} {v:.1f} us" for k, v in res.items()) + f"  gather variants rel diff {err:.1e}",
      flush=True)
