"""D-SKI MVM time vs RHS count (one-launch/fused path, gk_op_stage_dev stage 3)
with L2 evicted before every timed MVM; prints algorithmic bytes
and the fraction of the measured HBM copy bandwidth.
python tools/mvm_sweep.py <config> <nrhs> [<nrhs> ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_12283_b200 as gk  # noqa: E402

cfg = int(sys.argv[1])
X, y, dY = gk.make_dataset(cfg, 0)
ell, nodes = {1: (0.15, 60), 2: (0.2, 100), 3: (0.3, 48), 4: (0.02, 400)}[cfg]
grid = gk.Grid.cover(X, 1e-4, 3, nodes)
op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
N, n, d, m = op.size(), X.shape[0], X.shape[1], grid.size()
try:
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    hbm = 6552.0
flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for nrhs in [int(a) for a in sys.argv[2:]]:
    V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
    O = torch.empty_like(V)
    for _ in range(3):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        flush.sum()
        a.record(st)
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    byts = 8.0 * (3 * N * nrhs if d == 2 else (d + 1) * N // (d + 1) * (d + 1) * nrhs) + 8.0 * (2 * n * d + 4 * m * nrhs)
    byts = 8.0 * (2 * N * nrhs + 2 * n * d + 4 * m * nrhs) + 8.0 * N * nrhs
    print(f"C{cfg} nrhs {nrhs}: {ms * 1e3:.1f} us, {N * nrhs / ms / 1e6:.3e} rows*rhs/s, "
          f"{byts / 1e6:.1f} MB, {byts / ms / 1e6:.0f} GB/s = {byts / ms / 1e6 / hbm:.3f} of HBM", flush=True)
    del V, O
