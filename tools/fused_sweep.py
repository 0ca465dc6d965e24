"""Sweep the fused 2-D MVM decomposition knobs on one config; print phase
medians (max over CTAs) and the end-to-end per-call time."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem, timeit  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
grid = {k: [int(x) for x in v.split(",")] for k, v in (a.split("=") for a in sys.argv[3:])}
op = problem(cfg)
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
keys = list(grid)
for combo in itertools.product(*[grid[k] for k in keys]):
    for k, v in zip(keys, combo):
        gk.set_tuning(k, v)
    gk.set_tuning("fused_prof", 0)
    t = timeit(op, 3, V, O, nrhs)
    gk.set_tuning("fused_prof", 1)
    rows = []
    for _ in range(10):
        if not os.environ.get("NOFLUSH"):
            flush.sum()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
        torch.cuda.synchronize()
        st = gk.debug_fused_phases(op, nrhs)
        t0 = st[:, 0].min()
        rows.append(np.diff([st[:, k].max() - t0 for k in range(8)]) / 1e3)
    r = np.median(np.array(rows), axis=0)
    print(dict(zip(keys, combo)), f"call {t:6.2f} us | S {r[0]:5.2f} b {r[1]:4.2f} T1 {r[2]:5.2f} b {r[3]:4.2f} "
          f"T0 {r[4]:5.2f} b {r[5]:4.2f} G {r[6]:5.2f}", flush=True)
gk.set_tuning("fused_prof", 0)
