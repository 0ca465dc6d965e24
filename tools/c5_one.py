"""C5 D-SKIP Hadamard MVMs (64 RHS) inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off`: one per dskip_e value listed.
  python tools/c5_one.py [dskip_knob] [dskip_e,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

knob = int(sys.argv[1]) if len(sys.argv) > 1 else 0
eks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
X, y, dY = gk.make_dataset(5, 0)
op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
gk.set_tuning("dskip", knob)
N, nrhs = op.size(), 64
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for ek in eks:
    gk.set_tuning("dskip_e", ek)
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
