"""SURVEY §8(a) rows, each measured on the B200 against its roofline, with the
reference algorithm (the C++ oracle restatement, OpenMP where the reference
has it) timed on the same box's host cores beside it.

    python tools/rows_table.py > profiles/r1_rows_table.md

GPU times: wall clock around the public (host-buffer) call with a device
synchronise on both sides, median of reps, unless stated "device" (CUDA
events around the device-pointer call). CPU times: median of a bounded
sample. Roofline: algorithmic bytes (HBM 6552 GB/s, MEASURED_PEAKS.json) or
flops (fp64 DMMA peak measured on the GPU by gk_debug_dmma_peak).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_1810_12283_b200 as gk  # noqa: E402

HBM = float(json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.0)) \
    if os.path.exists(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")) else 6552.0
DMMA = gk.dmma_peak_tflops(0)
CORES = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
rows = []


def gtime(fn, reps=10, warm=2):
    keep = []  # results stay alive until the timing ends (no destructor inside a timed call)
    for _ in range(warm):
        keep.append(fn())
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        keep.append(fn())
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    del keep
    return float(np.median(ts))


def etime(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e-3


def ctime(fn, budget=4.0, max_reps=7):
    keep = [fn()]  # warm
    ts, t_end = [], time.perf_counter() + budget
    while len(ts) < max_reps and (not ts or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        keep.append(fn())
        ts.append(time.perf_counter() - t0)
    del keep
    return float(np.median(ts))


def row(name, ref, cfg, gpu_s, cpu_s, work=None, bound=None, note=""):
    frac = ""
    if work is not None and gpu_s:
        if bound == "hbm":
            ach = work / gpu_s / 1e9
            frac = f"{ach:.0f} GB/s = {ach / HBM:.1%} HBM"
        elif bound == "dmma":
            ach = work / gpu_s / 1e12
            frac = f"{ach:.1f} TF/s = {ach / DMMA:.1%} DMMA"
    sp = f"{cpu_s / gpu_s:.0f}×" if (cpu_s and gpu_s) else "—"
    rows.append((name, ref, cfg, f"{gpu_s * 1e3:.3f}", f"{cpu_s * 1e3:.1f}" if cpu_s else "—", sp, frac, note))
    print(f"  {name}: gpu {gpu_s * 1e3:.3f} ms cpu {cpu_s * 1e3 if cpu_s else float('nan'):.1f} ms {frac}",
          file=sys.stderr, flush=True)


# ---------------------------------------------------------------- C2 D-SKI
X, y, dY, grid = bench.build_problem()
c = bench.CONFIG
n, d = X.shape
og = O.Grid(grid.dims, grid.origin, grid.spacing)
ker, oker, noise = gk.KernelSpec(c["ell"], 1.0), O.KernelSpec(c["ell"], 1.0), (c["noise"], c["noise"])
g_build = gtime(lambda: gk.DskiOperator(ker, grid, X, noise), reps=3, warm=1)
c_build = ctime(lambda: O.DskiOperator(oker, og, X, noise), budget=6.0, max_reps=3)
op = gk.DskiOperator(ker, grid, X, noise)
ref = O.DskiOperator(oker, og, X, noise)
N, B, m = op.size(), c["nrhs"], grid.size()
row("a1–a3, a8 operator build (cover, stencils, point sort)", "dski.cpp:174-204", "C2", g_build, c_build)
Bh = bench.rhs_block(N, B, y, dY, 0)
Vext = torch.from_numpy(np.ascontiguousarray(Bh.T)).cuda()
Vi, Oi = torch.empty(N * B, dtype=torch.float64, device="cuda"), torch.empty(N * B, dtype=torch.float64, device="cuda")
op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), B)
U, W = torch.empty(m * B, dtype=torch.float64, device="cuda"), torch.empty(m * B, dtype=torch.float64, device="cuda")
sb = bench.stage_bytes(N, n, d, m, B)
gk.set_tuning("fused", 1)
t_sc = etime(lambda: op.stage_dev(0, Vi.data_ptr(), U.data_ptr(), B))
t_kuu = etime(lambda: op.stage_dev(1, U.data_ptr(), W.data_ptr(), B))
t_ga = etime(lambda: op.stage_dev(2, W.data_ptr(), Oi.data_ptr(), B))
gk.set_tuning("fused", 0)
t_mvm = etime(lambda: op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), B))
u1 = ref.stacked_transpose_apply(Bh[:, 0])
c_sc = ctime(lambda: [ref.stacked_transpose_apply(Bh[:, j]) for j in range(4)]) * B / 4
c_kuu = ctime(lambda: [ref.grid_mvm(u1) for _ in range(4)]) * B / 4
c_ga = ctime(lambda: [ref.stacked_apply(u1) for _ in range(4)]) * B / 4
c_mvm = ctime(lambda: ref.mvm(Bh))
row("a9 stacked_transpose_apply (scatter Bᵀv)", "dski.cpp:213-219", "C2, 32 RHS, device", t_sc, c_sc,
    sb["scatter"], "hbm", "staged kernel; inside the fused MVM this is phase S")
row("a6/a7 K_UU (grid kernel MVM)", "dski.cpp:146-172", "C2, 32 RHS, device", t_kuu, c_kuu, 2 * sb["kuu_mode"],
    "hbm", "two Kronecker–Toeplitz DMMA modes (reference: circulant FFT)")
row("a10 stacked_apply (gather Bw)", "dski.cpp:221-226", "C2, 32 RHS, device", t_ga, c_ga, sb["gather"], "hbm")
row("a11 D-SKI MVM (one launch)", "dski.cpp:228-238", "C2, 32 RHS, device (L2 warm)", t_mvm, c_mvm,
    bench.dski_bytes(N, n, d, m, B, 198 * 100), "hbm", "bench.py reports it with L2 evicted")
g_diag = gtime(lambda: op.diagonal(), reps=10)
c_diag = ctime(lambda: ref.diagonal())
row("a12 diagonal", "dski.cpp:240-290", "C2", g_diag, c_diag, None, None,
    "host API (includes the N-double copy back)")
ridx = [5, n + 17, 2 * n + 300, N - 1]
g_row = gtime(lambda: [op.row(i) for i in ridx], reps=5) / len(ridx)
c_row = ctime(lambda: [ref.row(i) for i in ridx]) / len(ridx)
row("a13 row", "dski.cpp:292-304", "C2", g_row, c_row, None, None, "per row, host API")
# pivoted Cholesky + preconditioner
g_piv = gtime(lambda: gk.pivoted_cholesky(op, c["precond_rank"], kernel_part=True), reps=3, warm=1)
nd = ref.noise_diagonal()
c_piv = ctime(lambda: O.pivoted_cholesky(ref, c["precond_rank"], noise_diag=nd), budget=6.0, max_reps=3)
row("a21 pivoted_cholesky (rank 50)", "linalg.cpp:133-174, gp.cpp:117-141", "C2", g_piv, c_piv)
fac = gk.pivoted_cholesky(op, c["precond_rank"], kernel_part=True)
F = O.pivoted_cholesky(ref, c["precond_rank"], noise_diag=nd)
g_pb = gtime(lambda: gk.Preconditioner.from_pivchol(op, fac), reps=3, warm=1)
c_pb = ctime(lambda: O.Preconditioner(F.L, nd), budget=4.0, max_reps=3)
row("a22 Preconditioner build (QR of [G; I])", "linalg.cpp:176-193", "C2, k = 50", g_pb, c_pb)
M = gk.Preconditioner.from_pivchol(op, fac)
P = O.Preconditioner(F.L, nd)
Rh = np.asfortranarray(Bh)
g_pa = gtime(lambda: M.apply(Rh), reps=5)
c_pa = ctime(lambda: [P.apply(Bh[:, j]) for j in range(B)])
row("a22 Preconditioner apply", "linalg.cpp:200-204", "C2, k = 50, 32 RHS, host API", g_pa, c_pa, None, None,
    "host API: dominated by the H2D/D2H of the 32 columns; on device it runs inside the PCG step")
# PCG per iteration
Xd = torch.empty_like(Vext)
its = 200
g_cg = gtime(lambda: gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), B, 1e-14, its, M), reps=3, warm=1) / its
c_cg = ctime(lambda: O.cg(ref, Bh[:, 0], 1e-14, 20, P), budget=6.0, max_reps=3) / 20 * B
row("a20 cg, per iteration (MVM + precond + vector ops)", "linalg.cpp:85-131", "C2, 32 RHS, k = 50", g_cg, c_cg,
    142e6, "hbm", "SURVEY §8(d): 142 MB per iteration; CPU: 1-RHS iterations × 32")
g_slq = gtime(lambda: gk.slq_logdet(op, c["slq_probes"], c["slq_steps"], 0, 0.5e-4), reps=3, warm=1)
c_slq = ctime(lambda: O.slq_logdet(ref, 4, c["slq_steps"], 0, 0.5e-4), budget=8.0, max_reps=2) * c["slq_probes"] / 4
row("a23 slq_logdet (31 probes × 30 steps)", "linalg.cpp:215-253", "C2", g_slq, c_slq, None, None,
    "CPU: 4 probes, scaled ×31/4")
# ---------------------------------------------------------------- C1 (dense exact, trace, predict, gradient)
X1, y1, dY1 = gk.make_dataset(1, 0)
N1 = X1.shape[0] * 3
ex = gk.ExactOperator(gk.KernelSpec(0.15, 1.0), X1, (1e-2, 1e-2))
V1 = np.random.default_rng(1).standard_normal((N1, 8))
g_ex = gtime(lambda: ex.mvm(V1), reps=5)
c_ex = ctime(lambda: O.assemble_dense(O.KernelSpec(0.15, 1.0), X1) @ V1, budget=8.0, max_reps=2)
row("a14 exact D-SE K∇ MVM (matrix-free on GPU; reference assembles)", "kernels.cpp:242-285", "C1, 8 RHS",
    g_ex, c_ex, 2.0 * N1 * N1 * 8 * 10, "dmma", "≈10 flops per kernel entry; CPU: assembly + GEMM")
grid1 = gk.Grid.cover(X1, 1e-4, 3, 60)
op1 = gk.DskiOperator(gk.KernelSpec(0.15, 1.0), grid1, X1, (0.1, 0.1))
ref1 = O.DskiOperator(O.KernelSpec(0.15, 1.0), O.Grid(grid1.dims, grid1.origin, grid1.spacing), X1, (0.1, 0.1))
M1 = gk.Preconditioner.from_pivchol(op1, gk.pivoted_cholesky(op1, 20, kernel_part=True))
nd1 = ref1.noise_diagonal()
P1 = O.Preconditioner(O.pivoted_cholesky(ref1, 20, noise_diag=nd1).L, nd1)
g_tr = gtime(lambda: gk.trace_estimate(op1, op1, 8, 3, 1e-6, 5000, M1), reps=3, warm=1)
c_tr = ctime(lambda: O.trace_estimate(ref1, ref1, 8, 3, 1e-6, 5000, P1), budget=8.0, max_reps=2)
row("a24 trace_estimate (8 probes, PCG tol 1e-6)", "linalg.cpp:255-279", "C1, σ = 0.1, k = 20", g_tr, c_tr)
om = O.GpModel(O.KernelSpec(0.15, 1.0), X1, y1, dY1, noise=(0.1, 0.1), backend="dski", grid_ratio=1e-4 / 0.15,
               max_grid_nodes=60, tol=1e-6, max_iterations=5000, precond_rank=20, seed=0)
alpha, _ = om.alpha()
Xt = np.random.default_rng(2).uniform(0.05, 0.95, (10000, 2))
g_pm = gtime(lambda: op1.predict_mean_grad(alpha, y1.mean(), Xt), reps=5)
c_pm = ctime(lambda: om.predict_mean_grad(Xt))
row("(f)1 predict_mean_grad (10,000 test points)", "gp.cpp:471-496", "C1", g_pm, c_pm)
sol = gk.cg(op1, gk.stacked_targets(y1, dY1, y1.mean()), 1e-6, 5000, M1)
g_gr = gtime(lambda: gk.lml_gradient(op1, sol.x, 8, 0, 1e-6, 5000, M1), reps=3, warm=1)
c_gr = ctime(lambda: om.lml_gradient(8), budget=8.0, max_reps=2)
row("(f)2 lml_gradient (4 parameters, 8 probes)", "gp.cpp:220-292", "C1, σ = 0.1", g_gr, c_gr)
# ---------------------------------------------------------------- C5 D-SKIP
X5, y5, dY5 = gk.make_dataset(5, 0)
kw = dict(rank=30, grid_ratio=0.01, max_grid_nodes=100, seed=0)
g_db = gtime(lambda: gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X5, (1e-2, 1e-2), **kw), reps=3, warm=1)
n5c = 2000
c_db = ctime(lambda: O.DskipOperator(O.KernelSpec(0.3, 1.0), X5[:n5c], (1e-2, 1e-2), **kw), budget=10.0,
             max_reps=1)
row("a15–a18 D-SKIP build (leaves + merge tree)", "dskip.cpp:162-234", "C5 (CPU: n = 2,000 of 10,000)", g_db,
    c_db, None, None, "CPU sample is 5× smaller; merge Lanczos is O(N·r²·steps)")
op5 = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X5, (1e-2, 1e-2), **kw)
N5 = op5.size()
V5 = torch.randn(N5 * 64, dtype=torch.float64, device="cuda")
O5 = torch.empty_like(V5)
t_h = etime(lambda: op5.stage_dev(3, V5.data_ptr(), O5.data_ptr(), 64))
ref5 = O.DskipOperator(O.KernelSpec(0.3, 1.0), X5[:n5c], (1e-2, 1e-2), **kw)
Vc = np.random.default_rng(3).standard_normal((ref5.size(), 8))
c_h = ctime(lambda: ref5.mvm(Vc)) * (N5 / ref5.size()) * (64 / 8)
row("a17/a19 D-SKIP Hadamard MVM", "dskip.cpp:24-36,132-139,236-250", "C5, 64 RHS, device", t_h, c_h,
    4.0 * N5 * 30 * 30 * 64, "dmma", "CPU: n = 2,000, 8 RHS, scaled to N and 64 RHS")

print("# r1 — SURVEY §8(a) rows on one B200 vs the reference algorithm on the host\n")
print(f"fp64 DMMA peak (measured, this GPU): {DMMA:.1f} TF/s; HBM {HBM:.0f} GB/s (MEASURED_PEAKS.json); "
      f"host cores used by the CPU oracle: {CORES} (OpenMP where the reference has it).\n")
print("| row | reference | config | GPU ms | CPU ms | speed-up | roofline | note |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(r) + " |")
