"""C4 (n = 150,000, grid 400², 1 RHS) MVM: default path vs staged kernels, per stage (CUDA events, median)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
X, y, dY = gk.make_dataset(4, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 400)
op = gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2))
N, m = op.size(), grid.size()
st = torch.cuda.current_stream().cuda_stream
Vi = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
Oi = torch.empty_like(Vi)
U = torch.empty(m * nrhs, dtype=torch.float64, device="cuda")
W = torch.empty_like(U)
flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def t(fn, reps=50, evict=True):
    for _ in range(5):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if evict:
            flush.sum()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) * 1e3 for a, b in ev]))


print(f"N={N} m={m} nrhs={nrhs}")
c0 = gk.kernel_launch_count()
op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st)
torch.cuda.synchronize()
print("default mvm launches:", gk.kernel_launch_count() - c0)
print(f"default mvm: {t(lambda: op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st)):.1f} us (L2 evicted)")
print(f"default mvm: {t(lambda: op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st), evict=False):.1f} us (warm)")
prev = gk.set_tuning("fused", 1)
for name, s, a, b in (("scatter", 0, Vi, U), ("kuu", 1, U, W), ("gather", 2, W, Oi), ("staged", 3, Vi, Oi)):
    print(f"{name}: {t(lambda: op.stage_dev(s, a.data_ptr(), b.data_ptr(), nrhs, stream=st)):.1f} us")
gk.set_tuning("fused", prev)
prev = gk.set_tuning("fused", 1)
for var in (0, 1, 2, 3):
    gk.set_tuning("scatter", var)
    U.fill_(0.0)
    us = t(lambda: op.stage_dev(0, Vi.data_ptr(), U.data_ptr(), nrhs, stream=st))
    print(f"staged scatter variant {var}: {us:.1f} us, checksum {float(U.sum()):.12e}")
gk.set_tuning("scatter", 0)
gk.set_tuning("fused", prev)
