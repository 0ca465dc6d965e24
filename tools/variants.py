"""A/B timing of kernel variants on the C2 workload (internal layout, CUDA events)."""
import json, os, sys
import numpy as np, torch
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk
from bench import build_problem, rhs_block, CONFIG

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N, m = op.size(), grid.size()
dev = torch.device('cuda')
st = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
res = {}
for nrhs in (32, 1):
    Bh = rhs_block(N, nrhs, y, dY, 0)
    Vext = torch.from_numpy(np.ascontiguousarray(Bh.T)).to(dev)
    Vi = torch.empty(N * nrhs, dtype=torch.float64, device=dev); Oi = torch.empty_like(Vi)
    U = torch.empty(m * nrhs, dtype=torch.float64, device=dev); W = torch.empty_like(U)
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=st)
    ref = None
    def timeit(stage, a, b, reps=int(os.environ.get("REPS", "50"))):
        for _ in range(3): op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
        ts = []
        for _ in range(reps):
            flush.sum(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1000)
        return float(np.median(ts))
    op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st); torch.cuda.synchronize(); ref = Oi.clone()
    for key, stage, a, b in (('scatter', 0, Vi, U), ('toeplitz', 1, U, W), ('gather', 2, W, Oi)):
        for var in (0, 1, 2, 3, 4):
            if key == "gather" and var > 2: continue
            if key == "scatter" and var > 3: continue
            gk.set_tuning(key, var)
            t = timeit(stage, a, b)
            gk.set_tuning(key, 0)
            res[f'{key}[{var}] nrhs={nrhs}'] = round(t, 2)
    for sv, gv, tv in ((0, 0, 0), (1, 1, 1)):
        gk.set_tuning('scatter', sv); gk.set_tuning('gather', gv); gk.set_tuning('toeplitz', tv)
        t = timeit(3, Vi, Oi)
        op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st); torch.cuda.synchronize()
        err = float(torch.linalg.norm(Oi - ref) / torch.linalg.norm(ref))
        res[f'mvm[s{sv} g{gv} t{tv}] nrhs={nrhs}'] = (round(t, 2), err)
    gk.set_tuning('scatter', 0); gk.set_tuning('gather', 0); gk.set_tuning('toeplitz', 0)
print(json.dumps(res, indent=1))
