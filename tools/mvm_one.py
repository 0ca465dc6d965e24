"""One batched D-SKI MVM of config C<k> inside cudaProfilerStart/Stop (for
`ncu --profile-from-start off`).  python tools/mvm_one.py <config> <nrhs>"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

for kv in filter(None, os.environ.get("GK_TUNE", "").split(",")):
    k, v = kv.split("=")
    gk.set_tuning(k, int(v))
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 17
X, y, dY = gk.make_dataset(cfg, 0)
ell, nodes = {1: (0.15, 60), 2: (0.2, 100), 3: (0.3, 48), 4: (0.02, 400)}[cfg]
grid = gk.Grid.cover(X, 1e-4, 3, nodes)
op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
torch.cuda.synchronize()
torch.cuda.profiler.start()
op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
