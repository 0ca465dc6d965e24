"""Phase breakdown of the one-launch 2-D MVM from per-CTA %globaltimer stamps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402

gk.set_tuning("fused_prof", 1)
for kv in filter(None, os.environ.get("GK_TUNE", "").split(",")):  # e.g. GK_TUNE=f2_tsplit=5
    k, v = kv.split("=")
    gk.set_tuning(k, int(v))
names = ["scatter", "barrier1", "mode1", "barrier2", "mode0", "barrier3", "gather"]
if os.environ.get("SCATTER_STAMPS"):  # a build with -DGK_SCATTER_STAMPS (stamps inside the scatter's first item)
    names = ["cs", "to_row2", "wait", "qrange", "iter0", "rest", "to_exit"]
if os.environ.get("TOEPLITZ_STAMPS"):  # -DGK_TOEPLITZ_STAMPS: slots 0-5 inside mode 1, 6 barrier-1 exit, 7 mode-1 exit
    names = ["seq_wait", "F_table", "issue", "slab_wait", "compute", "to_b1exit", "to_end"]
cases = [("C2", 32), ("C1", 32), ("C2", 1), ("C4", 1)]
if len(sys.argv) > 1:
    cases = [(sys.argv[1], int(sys.argv[2]))]
for cfg, nrhs in cases:
    op = problem(cfg)
    V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
    O = torch.empty_like(V)
    flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rows, durs = [], []
    for rep in range(20):
        if not os.environ.get("NOFLUSH"):
            flush.sum()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs)
        torch.cuda.synchronize()
        st = gk.debug_fused_phases(op, nrhs)
        t0 = st[:, 0].min()
        rows.append([(st[:, k].max() - t0) / 1e3 for k in range(8)])
        durs.append(np.diff(st, axis=1) / 1e3)  # per-CTA duration of each phase
    r = np.median(np.array(rows), axis=0)
    print(f"{cfg} nrhs={nrhs} ctas={len(st)}; cumulative max-over-CTAs (us):",
          " ".join(f"{n}={v:.2f}" for n, v in zip(names, r[1:])), flush=True)
    D = np.concatenate(durs)  # (reps*ctas, 7)
    for k, n in enumerate(names):
        q = np.percentile(D[:, k], [0, 25, 50, 75, 100])
        print(f"   {n:9s} per-CTA us: min {q[0]:6.2f} p25 {q[1]:6.2f} med {q[2]:6.2f} p75 {q[3]:6.2f} max {q[4]:6.2f}")
