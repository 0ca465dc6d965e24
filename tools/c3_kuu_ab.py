"""C3 K_UU (3 Toeplitz mode products, stage 1) per Toeplitz kernel variant:
time with L2 evicted and bit-identity against the default."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.c3_stages import tm, op, U, nrhs, M, st  # noqa: E402

ref = None
for var in [int(v) for v in os.environ.get("VARIANTS", "3,0").split(",")]:
    gk.set_tuning("toeplitz", var)
    W = torch.empty(M * nrhs, dtype=torch.float64, device="cuda")
    t = tm(lambda: op.stage_dev(1, U.data_ptr(), W.data_ptr(), nrhs, stream=st))
    if ref is None:
        ref = W.clone()
    print(f"toeplitz={var}: kuu {t:.1f} us, identical {torch.equal(W, ref)}, max rel {float((W - ref).abs().max() / ref.abs().max()):.1e}",
          flush=True)
