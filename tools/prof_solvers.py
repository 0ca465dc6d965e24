"""Run a short PCG (20 iterations) and SLQ (31 probes x 6 steps) on C2 for kernel launch lists."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk
from bench import build_problem, rhs_block

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N = op.size()
fac = gk.pivoted_cholesky(op, 50, kernel_part=True)
M = gk.Preconditioner.from_pivchol(op, fac)
Bh = rhs_block(N, 32, y, dY, 0)
dev = torch.device('cuda')
Vext = torch.from_numpy(np.ascontiguousarray(Bh.T)).to(dev)
Xd = torch.empty_like(Vext)
st = torch.cuda.current_stream().cuda_stream
gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), 32, 1e-4, 8, M, stream=st)
torch.cuda.synchronize()
t0 = time.perf_counter()
its, conv = gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), 32, 1e-4, 20, M, stream=st)
torch.cuda.synchronize()
t1 = time.perf_counter()
s = gk.slq_logdet(op, 31, 6, 0, 0.5e-4)
t2 = time.perf_counter()
print({'pcg20_s': t1 - t0, 'per_iter_us': (t1 - t0) / 20 * 1e6, 'slq6_s': t2 - t1, 'its': int(its[0])})
