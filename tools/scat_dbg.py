import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
os.environ["GK_FUSED_PROF_DUMP"] = "gpurun_out/prof_dump.bin"
import paper_1810_12283_b200 as gk
from tools.fused_timing import problem
for k, v in (a.split("=") for a in sys.argv[1:]):
    gk.set_tuning(k, int(v))
gk.set_tuning("fused_prof", 1)
op = problem("C2"); nrhs = 32
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda"); O = torch.empty_like(V)
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for rep in range(5):
    flush.sum(); op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs); torch.cuda.synchronize()
gk.debug_fused_phases(op, nrhs)
h = np.fromfile("gpurun_out/prof_dump.bin", dtype=np.int64)
h = h.reshape(-1, 64)
t0 = h[:, 0].min()
for c in (0, 1, 50, 100):
    r = h[c]
    print(c, "item", (r[8]-t0)/1e3)
    for i in range(5):
        b = 9 + 9 * i
        if r[b] == 0: break
        w = (r[b+1:b+9] - t0) / 1e3
        print(f"   row {i}: ready {(r[b]-t0)/1e3:6.2f}  warps done", " ".join(f"{x:6.2f}" for x in w))
