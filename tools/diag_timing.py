"""Diagnose fixed per-launch overheads: per-call (L2 evicted) vs back-to-back."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk
from bench import build_problem, rhs_block

X, y, dY, grid = build_problem()
op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
N, m = op.size(), grid.size()
dev = torch.device('cuda'); st = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
out = {}
for nrhs in (32, 1):
    Bh = rhs_block(N, nrhs, y, dY, 0)
    Vext = torch.from_numpy(np.ascontiguousarray(Bh.T)).to(dev)
    Vi = torch.empty(N * nrhs, dtype=torch.float64, device=dev); Oi = torch.empty_like(Vi)
    U = torch.empty(m * nrhs, dtype=torch.float64, device=dev); W = torch.empty_like(U)
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=st)
    for name, stage, a, b in (('scatter', 0, Vi, U), ('kuu', 1, U, W), ('gather', 2, W, Oi), ('mvm', 3, Vi, Oi), ('mvm_graph', 4, Vi, Oi)):
        f = lambda: op.stage_dev(stage, a.data_ptr(), b.data_ptr(), nrhs, stream=st)
        for _ in range(5): f()
        torch.cuda.synchronize()
        # (b) back-to-back, warm L2
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200): f()
        e1.record(); torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) * 1000 / 200
        # (c) per-call events with eviction, no host sync
        evs = []
        for _ in range(100):
            flush.sum()
            s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
            s0.record(); f(); s1.record(); evs.append((s0, s1))
        torch.cuda.synchronize()
        pc = float(np.median([x.elapsed_time(y) * 1000 for x, y in evs]))
        # (d) per-call events without eviction
        evs = []
        for _ in range(100):
            s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
            s0.record(); f(); s1.record(); evs.append((s0, s1))
        torch.cuda.synchronize()
        pw = float(np.median([x.elapsed_time(y) * 1000 for x, y in evs]))
        out[f'{name} nrhs={nrhs}'] = {'back_to_back_us': round(b2b, 2), 'per_call_evicted_us': round(pc, 2),
                                     'per_call_warm_us': round(pw, 2)}
print(json.dumps(out, indent=1))
