"""gk_op_mvm (host pinned buffers) on C2 with 32 RHS: one-shot vs chunked pipelines."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from bench import build_problem, rhs_block  # noqa: E402

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N, nrhs = op.size(), 32
Bh = rhs_block(N, nrhs, y, dY, 0)
Hin = torch.from_numpy(np.asfortranarray(Bh).T.copy()).pin_memory()
Hout = torch.empty_like(Hin).pin_memory()
pin = ctypes.cast(Hin.data_ptr(), ctypes.POINTER(ctypes.c_double))
pout = ctypes.cast(Hout.data_ptr(), ctypes.POINTER(ctypes.c_double))
ref = None
for chunk in (32, 16, 8, 4, 0):
    gk.set_tuning("e2e_chunk", chunk)
    for _ in range(3):
        gk._check(gk._lib.gk_op_mvm(op.handle, pin, N, pout, N, nrhs))
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        gk._check(gk._lib.gk_op_mvm(op.handle, pin, N, pout, N, nrhs))
        ts.append(time.perf_counter() - t0)
    out = Hout.T.numpy().copy()
    if ref is None:
        ref = out
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    print(f"chunk {({0: 'auto'}).get(chunk, chunk)}: mean {np.mean(ts)*1e6:.1f} us, median {np.median(ts)*1e6:.1f} us per 32-RHS call, "
          f"{N*nrhs/np.median(ts)/1e9:.2f} G rows*RHS/s, rel diff vs one-shot {err:.1e}", flush=True)
gk.set_tuning("e2e_chunk", 0)

# raw PCIe: pinned H2D and D2H of the 32-RHS block, alone and concurrent
dev = torch.device("cuda")
D = torch.empty(Hin.shape, dtype=torch.float64, device=dev)
D2 = torch.empty_like(D)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "both"):
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                D.copy_(Hin, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                Hout.copy_(D2, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = np.median(ts)
    print(f"raw {name}: {t*1e6:.1f} us for {Hin.numel()*8/1e6:.2f} MB -> {Hin.numel()*8/t/1e9:.1f} GB/s", flush=True)
