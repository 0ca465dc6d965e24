import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1810_12283_b200 as gk
from test_gpu_dski import pair
for kw in (dict(n=60, ell=0.5), dict(n=80, ell=0.4), dict(n=80, ell=0.5), dict(n=60, ell=0.4), dict(n=80, ell=0.4, s=1.0),
           dict(n=80, ell=0.4, noise=(0.1, 0.05))):
    n = kw.pop("n")
    g, r, X, grid = pair(n, 2, **kw)
    v = np.random.default_rng(1).standard_normal((g.size(), 2))
    gk.set_tuning("lean", 1); ref = g.mvm(v)
    gk.set_tuning("lean", 2); out = g.mvm(v)
    want = r.mvm(v)
    e = [float(np.linalg.norm(out[k*n:(k+1)*n] - want[k*n:(k+1)*n]) / np.linalg.norm(want[k*n:(k+1)*n])) for k in range(3)]
    print(n, kw, "dims", list(grid.dims), "lean vs oracle per group", np.round(e, 3),
          "fused vs oracle", float(np.linalg.norm(ref - want) / np.linalg.norm(want)), flush=True)
