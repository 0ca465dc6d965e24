"""C3 scatter (unit push + merge) with the flattened merge table vs the entry
chain: time (L2 evicted) and bit-identity of u."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.c3_stages import tm, op, V, nrhs, M, st  # noqa: E402

outs = {}
for mv in (1, 0, 2):
    gk.set_tuning("s3merge", mv)
    W = torch.empty(M * nrhs, dtype=torch.float64, device="cuda")
    t = tm(lambda: op.stage_dev(0, V.data_ptr(), W.data_ptr(), nrhs, stream=st))
    O = torch.empty_like(V)
    tmv = tm(lambda: op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st))
    outs[mv] = W.clone()
    print(f"s3merge={mv}: scatter {t:.1f} us, mvm {tmv:.1f} us", flush=True)
print("identical u:", torch.equal(outs[0], outs[1]), torch.equal(outs[2], outs[1]))
