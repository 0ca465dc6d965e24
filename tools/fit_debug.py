"""Compare the device GpModel's LML / gradient with the oracle's along the fit path."""
import numpy as np
import oracle as O
import paper_1810_12283_b200 as gk
X, y, dY = O.sample_test_function("franke", 300, 0, (0.05, 0.05))
kw = dict(noise=(0.05, 0.05), backend="dski", grid_ratio=0.2, max_grid_nodes=40, tol=1e-6,
          max_iterations=1000, precond_rank=30, slq_probes=8, slq_steps=25, seed=0)
for ell, s, nv, ng in [(0.3, 1.0, 0.05, 0.05), (0.25, 1.3, 0.04, 0.06)]:
    ref = O.GpModel(O.KernelSpec(ell, s), X, y, dY, **kw)
    gm = gk.GpModel(gk.KernelSpec(ell, s), X, y, dY, **{**kw, "noise": (nv, ng)})
    ref.set_hyperparameters(ell, s, nv, ng)
    r = ref.log_marginal_likelihood()
    print("params", ell, s, nv, ng)
    print(" lml", gm.log_marginal_likelihood(), r["lml"], " logdet", gm.logdet(), r["logdet"])
    print(" grad", gm.lml_gradient(), ref.lml_gradient(8))
    print(" grid", gm.op().grid.dims, gm.op().grid.spacing)
