import json, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1810_12283_b200 as gk
X, y, dY, grid = bench.build_problem(); c = bench.CONFIG
op = gk.DskiOperator(gk.KernelSpec(c["ell"], 1.0), grid, X, (c["noise"], c["noise"]))
fac = gk.pivoted_cholesky(op, c["precond_rank"], kernel_part=True)
b = gk.stacked_targets(y, dY, y.mean())
P = gk.Preconditioner.from_pivchol(op, fac)
out = {}
for pf in (1, 2):
    gk.set_tuning("pcg_fused", pf)
    sol = gk.cg(op, b, c["pcg_tol"], 1000, P)
    out[pf] = [float(v) for v in sol.residual_history]
json.dump(out, open("gpurun_out/c2hist.json", "w"))
