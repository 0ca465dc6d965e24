import os, sys, time, socket
import numpy as np, torch
import torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_1810_12283_b200 as gk
X, y, dY = gk.make_dataset(4, 0)
grid = gk.Grid.cover(X, 1e-4, 3, 400)
op = gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 200, kernel_part=True))
b = gk.stacked_targets(y, dY, y.mean())
Bd = torch.from_numpy(b).cuda(); Xd = torch.empty_like(Bd)
def run(tag):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    its, conv = gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), 1, 1e-4, 300, M)
    torch.cuda.synchronize(); print(tag, (time.perf_counter()-t0)/its[0]*1e6, "us/it", flush=True)
run("before nccl")
run("before nccl 2")
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
U = torch.ones(1000, dtype=torch.float64, device="cuda"); dist.all_reduce(U); torch.cuda.synchronize()
run("after nccl")
run("after nccl 2")
dist.destroy_process_group()
run("after destroy")
