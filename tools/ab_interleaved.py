"""Interleaved A/B of a tuning key on the one-launch 2-D MVM: the values
alternate call by call (L2 evicted before each, as bench.py does), so drift
and timer quantisation average out; mean and standard error per value.

  python tools/ab_interleaved.py <key> <v1,v2,...> [C2:32,C4:1,...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402

key = sys.argv[1]
vals = [int(v) for v in sys.argv[2].split(",")]
cases = [(c.split(":")[0], int(c.split(":")[1])) for c in (sys.argv[3] if len(sys.argv) > 3 else "C2:32,C1:32,C2:1,C4:1").split(",")]
reps = int(os.environ.get("REPS", "300"))
st = torch.cuda.current_stream()
flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cfg, nrhs in cases:
    op = problem(cfg)
    V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
    outs = {v: torch.empty_like(V) for v in vals}
    for v in vals:  # plans built, code warm
        gk.set_tuning(key, v)
        for _ in range(3):
            op.stage_dev(3, V.data_ptr(), outs[v].data_ptr(), nrhs, stream=st.cuda_stream)
    torch.cuda.synchronize()
    ts = {v: [] for v in vals}
    for r in range(reps):
        for v in (vals if r % 2 == 0 else vals[::-1]):
            gk.set_tuning(key, v)  # bumps the tuning generation: the next call rebuilds the plan
            op.stage_dev(3, V.data_ptr(), outs[v].data_ptr(), nrhs, stream=st.cuda_stream)  # (untimed)
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            op.stage_dev(3, V.data_ptr(), outs[v].data_ptr(), nrhs, stream=st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            ts[v].append(e0.elapsed_time(e1) * 1000)
    same = all(torch.equal(outs[vals[0]], outs[v]) for v in vals[1:])
    print(f"{cfg} nrhs={nrhs} " + "  ".join(
        f"{key}={v}: {np.mean(ts[v]):.2f}±{np.std(ts[v]) / np.sqrt(len(ts[v])):.2f} us" for v in vals) +
          f"  identical={same}", flush=True)
