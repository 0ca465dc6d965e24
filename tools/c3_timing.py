"""C3 (d = 3 star surface, n = 25,001, N = 100,004, grid 48³, ℓ = 0.3):
operator build, diagonal, batched MVM (17 RHS), pivoted Cholesky (rank 100),
PCG (tol 1e-6, 17 columns) and SLQ (16 probes × 50 steps) wall times."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


X, y, dY = gk.make_dataset(3, 0)
n, d = X.shape
ell, noise = 0.3, (1e-2, 1e-2)
grid = gk.Grid.cover(X, 1e-4, 3, 48)
t0 = t()
op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, noise)
t1 = t()
dg = op.diagonal()
t2 = t()
N, nrhs = op.size(), 17
V = torch.randn(N * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
for a, b in ev:
    a.record()
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
    b.record()
torch.cuda.synchronize()
mvm_ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
t3 = t()
fac = gk.pivoted_cholesky(op, 100, kernel_part=True)
M = gk.Preconditioner.from_pivchol(op, fac)
t4 = t()
B = np.column_stack([gk.stacked_targets(y, dY, y.mean())] + [gk.rademacher_vector(N, 0, 1000 + p) for p in range(16)])
sol = gk.cg(op, B, 1e-6, 1000, M)
t5 = t()
r = gk.slq_logdet(op, 16, 50, 0, 0.5e-4)
t6 = t()
print(f"C3 n={n} N={N} grid {grid.dims}: build {t1-t0:.3f} s, diagonal {t2-t1:.3f} s, MVM(17 RHS) {mvm_ms*1e3:.1f} us "
      f"({N*nrhs/(mvm_ms*1e-3)/1e9:.2f} G rows*RHS/s), pivchol+precond {t4-t3:.3f} s, "
      f"PCG {t5-t4:.3f} s (its {[s.iterations for s in sol][:4]}..., conv {sum(s.converged for s in sol)}/17), "
      f"SLQ {t6-t5:.3f} s logdet {r.logdet:.6e}", flush=True)
