"""Lean one-launch 2-D MVM (lean2d.cu) vs the previous one-launch kernel
(fused2d.cu): median per-call time (CUDA events, L2 evicted before each call)
and max error between the two, for C1/C2 shapes and several RHS counts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timeit(op, V, O, nrhs, reps=50):
    for _ in range(3):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.sum()
        a.record()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st)
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def main():
    cases = [("C2", 32), ("C2", 16), ("C2", 8), ("C2", 2), ("C2", 1), ("C1", 32), ("C1", 9), ("C2", 64), ("C2", 31)]
    if len(sys.argv) > 2:
        cases = [(sys.argv[1], int(sys.argv[2]))]
    for cfg, nrhs in cases:
        op = problem(cfg)
        V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
        O1, O2 = torch.empty_like(V), torch.empty_like(V)
        gk.set_tuning("lean", 2)
        t_lean = timeit(op, V, O1, nrhs)
        gk.set_tuning("lean", 1)
        t_old = timeit(op, V, O2, nrhs)
        gk.set_tuning("lean", 0)
        err = float((O1 - O2).norm() / O2.norm())
        print(f"{cfg} nrhs={nrhs:3d}: lean {t_lean:7.2f} us   fused2d {t_old:7.2f} us   rel diff {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
