"""Fused one-launch d=2 MVM vs the staged kernels on C2 (and C1/C4-shaped
problems): median per-call time with L2 evicted before each call, plus
back-to-back throughput and graph replay."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
REPS = int(os.environ.get("REPS", "100"))


def problem(cfg):
    if cfg == "C2":
        X, y, dY, grid = build_problem()
        return gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
    if cfg == "C1":
        X, *_ = gk.make_dataset(1, 0)
        grid = gk.Grid.cover(X, 1e-3, 3, 60)
        return gk.DskiOperator(gk.KernelSpec(0.15, 1.0), grid, X, (1e-2, 1e-2))
    if cfg == "C4":
        X, *_ = gk.make_dataset(4, 0)
        grid = gk.Grid.cover(X, 1e-4, 3, 400)
        return gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2))


def timeit(op, stage, a, b, nrhs, flush_each=True):
    for _ in range(3):
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
    ts = []
    for _ in range(REPS):
        if flush_each:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    return float(np.median(ts))


def b2b(op, stage, a, b, nrhs, k=200):
    for _ in range(3):
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / k


def main():
  res = {}
  for cfg, rhs_list in (("C2", (32, 64, 1)), ("C1", (32, 8, 1)), ("C4", (1, 8))):
      op = problem(cfg)
      N = op.size()
      for nrhs in rhs_list:
          V = torch.randn(N * nrhs, dtype=torch.float64, device=dev)
          O1, O2 = torch.empty_like(V), torch.empty_like(V)
          row = {}
          for fused in (0, 1):
              gk.set_tuning("fused", fused)
              out = O1 if fused == 0 else O2
              row[f"fused={fused} us"] = round(timeit(op, 3, V, out, nrhs), 2)
              row[f"fused={fused} b2b us"] = round(b2b(op, 3, V, out, nrhs), 2)
              row[f"fused={fused} graph b2b us"] = round(b2b(op, 4, V, out, nrhs), 2)
          gk.set_tuning("fused", 0)
          torch.cuda.synchronize()
          row["rel diff"] = float(torch.linalg.norm(O1 - O2) / torch.linalg.norm(O2))
          res[f"{cfg} nrhs={nrhs}"] = row
          print(cfg, nrhs, row, flush=True)
  print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
