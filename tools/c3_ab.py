"""Interleaved A/B of the d = 3 MVM variants (tuning key "d3", a bitmask)
at C3 (17 RHS by default): scatter, gather and the whole MVM per value, L2
evicted before each call, values alternating call by call; outputs compared
bit for bit against the first value.

  python tools/c3_ab.py [d3 values, default 7,0] [nrhs]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

vals = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "7,0").split(",")]
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 17
reps = int(os.environ.get("REPS", "40"))
X, y, dY = gk.make_dataset(3, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (1e-2, 1e-2))
N, M = op.size(), grid.size()
st = torch.cuda.current_stream()
flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda", generator=g)
U = torch.randn(M * nrhs, dtype=torch.float64, device="cuda", generator=g)
stages = {"scatter": (0, V, M), "kuu": (1, U, M), "gather": (2, U, N), "mvm": (3, V, N), "mvm_graph": (4, V, N)}
outs = {(k, v): torch.empty(sz * nrhs, dtype=torch.float64, device="cuda") for k, (_, _, sz) in stages.items()
        for v in vals}
ts = {(k, v): [] for k in stages for v in vals}
for v in vals:
    gk.set_tuning("d3", v)
    for k, (s, x, _) in stages.items():
        for _ in range(2):
            op.stage_dev(s, x.data_ptr(), outs[(k, v)].data_ptr(), nrhs, stream=st.cuda_stream)
torch.cuda.synchronize()
for r in range(reps):
    for v in (vals if r % 2 == 0 else vals[::-1]):
        gk.set_tuning("d3", v)
        for k, (s, x, _) in stages.items():
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            op.stage_dev(s, x.data_ptr(), outs[(k, v)].data_ptr(), nrhs, stream=st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            ts[(k, v)].append(e0.elapsed_time(e1) * 1000)
gk.set_tuning("d3", 0)
for k in stages:
    same = [bool(torch.equal(outs[(k, vals[0])], outs[(k, v)])) for v in vals[1:]]
    diff = [float((outs[(k, vals[0])] - outs[(k, v)]).norm() / outs[(k, vals[0])].norm()) for v in vals[1:]]
    print(f"C3 nrhs={nrhs} {k:8s} " + "  ".join(
        f"d3={v}: {np.median(ts[(k, v)]):7.1f} us" for v in vals) + f"  identical={same} rel={diff}", flush=True)
