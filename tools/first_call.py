"""First-call overhead of PCG/SLQ on a fresh operator (C2): times a 1-iteration
PCG, then again, on the first operator and on a second, newly built operator
(what a hyperparameter loop sees after each rebuild)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402


def tm(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, r


X, y, dY, grid = build_problem()
for rep, ell in enumerate((0.2, 0.21)):
    ms_op, op = tm(lambda: gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2)))
    N = op.size()
    ms_pc, M = tm(lambda: gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 50, kernel_part=True)))
    B = rhs_block(N, 32, y, dY, 0)
    V = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    Xd = torch.empty_like(V)
    out = [f"op {rep}: build {ms_op:.1f} ms, precond {ms_pc:.1f} ms"]
    for its in (1, 1, 8, 8, 1000):
        ms, _ = tm(lambda: gk.cg_dev(op, V.data_ptr(), Xd.data_ptr(), 32, 1e-4, its, M))
        out.append(f"pcg{its} {ms:.1f}")
    for _ in range(2):
        ms, _ = tm(lambda: gk.slq_logdet(op, 31, 30, 0, 0.5e-4))
        out.append(f"slq {ms:.1f}")
    print(", ".join(out), flush=True)
