"""Time the one-launch MVM (stage_dev 3) of C2/C1/C4 with the library in
GK_B200_LIB (run once per build to A/B two builds); prints a digest of the
outputs so the two runs can be compared for bit-identity."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.fused_timing import problem, timeit, b2b  # noqa: E402

cases = [("C2", 32), ("C1", 32), ("C2", 1), ("C4", 1), ("C4", 8)]
tag = os.path.basename(os.environ.get("GK_B200_LIB", "libgk_b200.so"))
for cfg, nrhs in cases:
    op = problem(cfg)
    g = torch.Generator(device="cuda").manual_seed(1)
    V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda", generator=g)
    O = torch.empty_like(V)
    t = timeit(op, 3, V, O, nrhs)
    tb = b2b(op, 3, V, O, nrhs)
    dig = hashlib.sha1(O.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{tag} {cfg} nrhs={nrhs}: {t:.2f} us (L2 evicted), {tb:.2f} us back-to-back, out {dig}", flush=True)
