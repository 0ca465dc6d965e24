"""Generate tests/golden/c2_cg.json — TEST INFRASTRUCTURE.

Full-size C2 (bench.py CONFIG: D-SKI d=2, n=10,000, N=30,000, grid 100²,
ℓ=0.2, σ=1e-2) run through the C oracle: the rank-50 pivoted-Cholesky pivot
order (GpModel::preconditioner, gp.cpp:117-141 / linalg.cpp:133-174) and the
PCG relative-residual history of the targets column for 1000 iterations
(linalg.cpp:84-131). At this noise level the reference algorithm does not
reach tol 1e-4 within 1000 iterations; the fixture pins that behaviour.
~25 s on one core.

Run:  python tests/golden/make_c2_cg.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle as O  # noqa: E402

X, y, dY, grid = bench.build_problem()
c = bench.CONFIG
op = O.DskiOperator(O.KernelSpec(c["ell"], 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X,
                    (c["noise"], c["noise"]))
nd = op.noise_diagonal()
F = O.pivoted_cholesky(op, c["precond_rank"], noise_diag=nd)
P = O.Preconditioner(F.L, nd)
b = np.concatenate([y - y.mean()] + [dY[:, j] for j in range(dY.shape[1])])
r = O.cg(op, b, c["pcg_tol"], 1000, P)
out = {"generator": "tests/golden/make_c2_cg.py (C oracle, bench.py CONFIG C2)",
       "pivots": [int(p) for p in F.pivots], "initial_trace": F.initial_trace,
       "residual_trace": F.residual_trace, "iterations": int(r.iterations), "converged": bool(r.converged),
       "residual_history": [float(v) for v in r.residual_history]}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_cg.json"), "w") as f:
    json.dump(out, f)
print("pivots", out["pivots"][:8], "its", out["iterations"], "final", out["residual_history"][-1])
