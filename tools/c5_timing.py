"""C5: D-SKIP d=6 n=10000 (N=70000), product SE ell=0.3, rank 30 on 100-node
1-D grids, 64 RHS — build time and Hadamard MVM time / DMMA throughput."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

X, y, dY = gk.make_dataset(5, 0)
t0 = time.perf_counter()
op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
torch.cuda.synchronize()
build = time.perf_counter() - t0
N, nrhs = op.size(), 64
dev = torch.device("cuda")
V = torch.randn(N * nrhs, dtype=torch.float64, device=dev)
O = torch.empty_like(V)
st = torch.cuda.current_stream().cuda_stream
def run(knob, ek=0):
    gk.set_tuning("dskip", knob)
    gk.set_tuning("dskip_e", ek)
    for _ in range(3):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        a.record()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])), O.clone()


ranks = [f.Q.shape[1] for f in op.factors()]
flops = 4.0 * N * 30 * 30 * nrhs
res = {}
for knob in (1, 3, 0):
    ms, out = run(knob)
    res[knob] = out
    print(f"C5[dskip={knob}] build {build:.2f} s; MVM {ms*1e3:.1f} us for {nrhs} RHS; "
          f"{N*nrhs/(ms*1e-3)/1e9:.2f} G rows*RHS/s; {flops/(ms*1e-3)/1e12:.2f} TFLOP/s (4 N r^2 B model, r=30); "
          f"factor ranks {ranks}", flush=True)
for ek in (1, 2, 3):
    ms, out = run(0, ek)
    print(f"C5[dskip=0 dskip_e={ek}] MVM {ms*1e3:.1f} us; {flops/(ms*1e-3)/1e12:.2f} TFLOP/s; "
          f"rel diff vs v1 {float((out - res[1]).norm() / res[1].norm()):.2e}", flush=True)
print("v2 vs v1 rel diff", float((res[3] - res[1]).norm() / res[1].norm()))
print("v3 vs v1 rel diff", float((res[0] - res[1]).norm() / res[1].norm()))
