#!/usr/bin/env python
"""Benchmark: batched D-SKI K∇ MVM throughput (rows·RHS/s) on BASELINE config C2
(configs[1]: d=2, n=10,000 -> N=30,000, 100x100 grid, SE ell=0.2, 32 RHS =
y + 31 Rademacher probes), plus the PCG+SLQ solve time on the same operator.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One step = one batched K∇ MVM over the 32-RHS block (scatter B^T, K_UU mode
products, gather B + noise) with inputs resident in HBM; L2 is flushed before
every timed step (the C2 working set, ~34 MB, would otherwise sit in the 126 MB
L2). N>1 (torchrun): every rank holds an operator replica and its own 32-RHS
probe shard (weak scaling, no data-path collective); time = max over ranks.
--impl reference times the reference algorithm on the host cores (the C++
oracle port, OpenMP over RHS — the reference cannot be built here, see
DESIGN.md) on the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = {"workload": "C2: D-SKI d=2 n=10000 (N=30000) grid 100x100 SE ell=0.2 s=1 "
                      "sigma=1e-2, 32 RHS (y + 31 Rademacher probes)",
          "config_id": 2, "n": 10000, "d": 2, "N": 30000, "grid": [100, 100], "nrhs": 32,
          "ell": 0.2, "noise": 1e-2, "precond_rank": 50, "pcg_tol": 1e-4, "slq_probes": 31,
          "slq_steps": 30}
METRIC = "K∇ MVM rows·RHS/s"
UNIT = "rows*rhs/s"


def build_problem():
    import paper_1810_12283_b200 as gk
    X, y, dY = gk.make_dataset(2, 0)
    grid = gk.Grid.cover(X, 1e-3, 3, 100)
    assert list(grid.dims) == [100, 100]
    return X, y, dY, grid


def rhs_block(N, nrhs, y, dY, probe_offset):
    """Column 0 = stacked targets (observations.hpp:29-35), the rest Rademacher
    probes rademacher_vector(N, 0, 1000+p) (the trace-estimator streams,
    linalg.cpp:264-266); shard p offsets the probe ids."""
    import paper_1810_12283_b200 as gk
    B = np.empty((N, nrhs), order="F")
    B[:, 0] = gk.stacked_targets(y, dY, y.mean())
    for c in range(1, nrhs):
        B[:, c] = gk.rademacher_vector(N, 0, 1000 + probe_offset + c - 1)
    return B


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.f:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 8:
                continue
            try:
                rows.append((float(p[0]), float(p[1]), float(p[2]), p[3], p[4:8]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [r for r in rows if r[2] > 200.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[4]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in load])),
                "sm_max_mhz": float(max(r[1] for r in rows)), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(load)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def dski_bytes(N, n, d, m, nrhs, Mc):
    """SURVEY §8(d) algorithmic bytes of one batched D-SKI MVM."""
    return 8.0 * (3 * N * nrhs + 2 * n * d + 4 * m * nrhs + Mc)


def stage_bytes(N, n, d, m, nrhs, T=6):
    """Algorithmic bytes per launch of each stage kernel of this implementation
    (per-point stencil record = base ints + d×2×T doubles)."""
    pt = n * (16 + 8 * d * 2 * T)
    return {"scatter": 8.0 * (N * nrhs + m * nrhs) + pt,          # read v, write u
            "kuu_mode": 8.0 * (2 * m * nrhs),                       # read + write one grid block
            "gather": 8.0 * (m * nrhs + 2 * N * nrhs) + pt}         # read w, v; write out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)  # before NCCL init: each rank's communicator on its own GPU
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    import paper_1810_12283_b200 as gk

    X, y, dY, grid = build_problem()
    n, d = X.shape
    ker = gk.KernelSpec(CONFIG["ell"], 1.0)
    noise = (CONFIG["noise"], CONFIG["noise"])
    op = gk.DskiOperator(ker, grid, X, noise, device=local)
    N, nrhs, m = op.size(), CONFIG["nrhs"], grid.size()
    Bh = rhs_block(N, nrhs, y, dY, probe_offset=rank * nrhs)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    # inputs resident in HBM: external (col-major) block -> internal layout once
    Vext = torch.from_numpy(np.ascontiguousarray(Bh.T)).to(dev)  # (nrhs, N) == col-major N×nrhs
    Vi = torch.empty(N * nrhs, dtype=torch.float64, device=dev)
    Oi = torch.empty_like(Vi)
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=sp)
    # L2 eviction buffer: streaming-READ 256 MB (2x L2) before each timed step.
    # (A write-flush would leave ~126 MB of dirty lines whose write-back is then
    # charged to the timed kernel.)
    flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=sp)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # correctness guard on this very data (external round trip vs host API)
    ref_cols = op.mvm(Bh[:, :2])
    Oe = torch.empty_like(Vext)
    op.from_internal_dev(Oi.data_ptr(), Oe.data_ptr(), nrhs, stream=sp)
    torch.cuda.synchronize()
    got = Oe.T.cpu().numpy()[:, :2]
    assert np.linalg.norm(got - ref_cols) <= 1e-13 * np.linalg.norm(ref_cols)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = gk.kernel_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.sum()  # evict L2 (outside the events)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = gk.kernel_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * N * nrhs / (ms * 1e-3)

    # ---- roofline of the dominant kernel. With the one-launch 2-D MVM
    # (fused2d.cu) the step IS one kernel: its algorithmic bytes are SURVEY
    # §8(d)'s per-MVM figure. The staged kernels (gk_set_tuning("fused", 1))
    # are timed alongside for reference.
    Mc = 198 * (198 // 2 + 1)
    mvm_bytes = dski_bytes(N, n, d, m, nrhs, Mc)
    per_step = launches / max(1, args.steps)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    Ui = torch.empty(m * nrhs, dtype=torch.float64, device=dev)
    Wi = torch.empty_like(Ui)
    staged_ms = {}
    reps = max(20, min(args.steps, 200))
    prev = gk.set_tuning("fused", 1)
    try:
        for name, st, a, b in (("scatter", 0, Vi, Ui), ("kuu", 1, Ui, Wi), ("gather", 2, Wi, Oi),
                               ("staged_mvm", 3, Vi, Oi)):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(reps)]
            for s0, e0 in ev:
                flush.sum()
                s0.record(stream)
                op.stage_dev(st, a.data_ptr(), b.data_ptr(), nrhs, stream=sp)
                e0.record(stream)
            torch.cuda.synchronize()
            staged_ms[name] = float(np.mean([s0.elapsed_time(e0) for s0, e0 in ev]))
    finally:
        gk.set_tuning("fused", prev)
    sb = stage_bytes(N, n, d, m, nrhs)
    if per_step == 1:
        dom, dom_bytes, dom_ms = "k_dski_mvm2d (one-launch MVM)", mvm_bytes, ms
    else:
        bytes_per = {"scatter": sb["scatter"], "kuu": 2 * sb["kuu_mode"], "gather": sb["gather"]}
        dom = max(bytes_per, key=lambda k: staged_ms[k])
        dom_bytes, dom_ms = bytes_per[dom], staged_ms[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None  # DRAM bytes per launch of the dominant kernel from the committed ncu capture
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))
        if dom in tj:
            traffic = tj[dom]["dram_bytes_read"] + tj[dom]["dram_bytes_write"]
    except Exception:
        traffic = None

    # ---- end to end through the public API with host (pinned) buffers
    Hin = torch.from_numpy(np.asfortranarray(Bh).T.copy()).pin_memory()  # (nrhs, N) == col-major
    Hout = torch.empty_like(Hin).pin_memory()
    import ctypes
    lib = gk._lib
    pin_in = ctypes.cast(Hin.data_ptr(), ctypes.POINTER(ctypes.c_double))
    pin_out = ctypes.cast(Hout.data_ptr(), ctypes.POINTER(ctypes.c_double))

    def e2e_call():
        gk._check(lib.gk_op_mvm(op.handle, pin_in, N, pin_out, N, nrhs))

    for _ in range(3):
        e2e_call()
    e2e_steps = max(5, min(args.steps, 50))
    if world > 1:
        dist.barrier()
    e2e_ts = []
    for _ in range(e2e_steps):  # each call returns only after its D2H copy landed (host-synchronous API)
        t0 = time.perf_counter()
        e2e_call()
        e2e_ts.append(time.perf_counter() - t0)
    e2e_t = torch.tensor([float(np.median(e2e_ts)), float(np.mean(e2e_ts))], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_med, e2e_mean = [float(v) for v in e2e_t.tolist()]
    e2e_value = world * N * nrhs / e2e_med

    # ---- PCG + SLQ solve (GpModel::preconditioner/solve/logdet on this shard)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fac = gk.pivoted_cholesky(op, CONFIG["precond_rank"], kernel_part=True)
    M = gk.Preconditioner.from_pivchol(op, fac)
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    Xd = torch.empty_like(Vext)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its, conv = gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), nrhs, CONFIG["pcg_tol"], 1000, M,
                          stream=sp)
    torch.cuda.synchronize()
    t_pcg_first = time.perf_counter() - t0
    # the same solve again: steady state (plans, graphs and workspaces cached
    # on the operator), what every later solve of a hyperparameter loop costs
    t0 = time.perf_counter()
    its, conv = gk.cg_dev(op, Vext.data_ptr(), Xd.data_ptr(), nrhs, CONFIG["pcg_tol"], 1000, M,
                          stream=sp)
    torch.cuda.synchronize()
    t_pcg = time.perf_counter() - t0
    t0 = time.perf_counter()
    slq = gk.slq_logdet(op, CONFIG["slq_probes"], CONFIG["slq_steps"], 0, 0.5 * 1e-4,
                        probe_offset=rank * CONFIG["slq_probes"])
    t_slq_first = time.perf_counter() - t0
    t0 = time.perf_counter()
    slq = gk.slq_logdet(op, CONFIG["slq_probes"], CONFIG["slq_steps"], 0, 0.5 * 1e-4,
                        probe_offset=rank * CONFIG["slq_probes"])
    slq_logdet = slq.logdet
    if world > 1:  # global estimate over all ranks' probes, summed in probe order
        from paper_1810_12283_b200 import sharding
        est = sharding.gather_probe_estimates(np.asarray(slq.estimates), rank * CONFIG["slq_probes"],
                                              world * CONFIG["slq_probes"], device=dev)
        slq_logdet = sharding.ordered_mean(est)
    t_slq = time.perf_counter() - t0
    solve = torch.tensor([t_pre, t_pcg, t_slq, t_pcg_first, t_slq_first], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(solve, op=dist.ReduceOp.MAX)
    t_pre, t_pcg, t_slq, t_pcg_first, t_slq_first = [float(v) for v in solve.tolist()]

    c4 = None
    if not args.no_c4:
        try:
            c4 = c4_slab(args, world, rank, local, dist)
        except Exception as e:  # reported, never silently replaced
            c4 = {"error": f"{type(e).__name__}: {e}"}

    c5 = None
    if not args.no_c5:
        try:
            c5 = c5_dskip(args, world, rank, local, dist)
        except Exception as e:  # reported, never silently replaced
            c5 = {"error": f"{type(e).__name__}: {e}"}

    line = None
    if rank == 0:
        cpu = cpu_baseline(args) if world == 1 and not args.no_cpu_baseline else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded C2 generator)",
            "config": dict(CONFIG, parallelism=f"rhs-shard x{world}" if world > 1 else "1 GPU",
                           l2="evicted before every timed step (256 MB streaming read, outside the timed events)",
                           timing="CUDA events per step on the launching stream, max over ranks"),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N * nrhs,
                    "d2h_bytes_per_step": 8 * N * nrhs,
                    "path": "gk_op_mvm (C-ABI, pinned host buffers, permutes + copies timed)",
                    "statistic": f"median of {e2e_steps} host-timed calls, max over ranks",
                    "us_per_call_median": e2e_med * 1e6, "us_per_call_mean": e2e_mean * 1e6},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "traffic_source": "profiles/r1_traffic.json (ncu --set full, one launch)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peaks else "fallback",
                         "bytes_per_launch": dom_bytes, "launch_ms": dom_ms,
                         "bytes_formula": "SURVEY 8(d): 8*(3*N*B + 2*n*d + 4*m*B + M_c)",
                         "staged_kernels_ms": staged_ms},
            "mvm_roofline": {"algorithmic_bytes": mvm_bytes,
                             "achieved_gbs": mvm_bytes / (ms * 1e-3) / 1e9,
                             "frac_hbm": mvm_bytes / (ms * 1e-3) / 1e9 / hbm},
            "solve": {"precond_build_s": t_pre, "pcg_s": t_pcg, "slq_s": t_slq,
                      "pcg_first_call_s": t_pcg_first, "slq_first_call_s": t_slq_first,
                      "timing": "host wall clock around each call with device syncs, max over ranks; "
                                "*_s = second identical call (steady state), *_first_call_s includes "
                                "one-time plan/graph/workspace setup",
                      "pcg_plus_slq_s": t_pcg + t_slq, "pcg_iterations": [int(v) for v in its],
                      "pcg_converged": int(np.sum(conv)), "slq_logdet": slq_logdet,
                      "slq_probes_total": world * CONFIG["slq_probes"],
                      "note": "tol 1e-4, max 1000 iterations: at sigma = 1e-2 the reference algorithm (oracle) "
                              "also stops at 1000 unconverged (relative residual 0.177 for the targets column; "
                              "tests/golden/c2_cg.json, checked by tests/test_gpu_c2_fullsize.py)"},
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "c4_slab": c4,
            "c5_dskip": c5,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def c4_slab(args, world, rank, local, dist):
    """C4 (n = 150,000, d = 2, grid 400², ℓ = 0.02, 1 RHS = the targets):
    the grid-slab sharded MVM — points partitioned by grid
    slab across the ranks, one NCCL all-reduce of the 160,000-node grid vector
    per MVM. Strong scaling (fixed total points). Time = max over ranks."""
    import torch
    import paper_1810_12283_b200 as gk
    from paper_1810_12283_b200.slab import SlabShardedDskiOperator
    if not dist.is_initialized():  # single GPU: a one-rank NCCL group runs the same code path
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    X, y, dY = gk.make_dataset(4, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, 400)
    t0 = time.perf_counter()
    sop = SlabShardedDskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2), device=local)
    build_s = time.perf_counter() - t0
    dev = torch.device("cuda", local)
    nrhs = 1
    b = gk.stacked_targets(y, dY, y.mean())
    rows = sop.local_rows()
    Vext = torch.from_numpy(np.ascontiguousarray(b[rows])).to(dev)
    Vi, Oi = torch.empty_like(Vext), torch.empty_like(Vext)
    st = torch.cuda.current_stream(dev)
    sop.local.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=st.cuda_stream)
    U = torch.empty(sop.M * nrhs, dtype=torch.float64, device=dev)
    W = torch.empty_like(U)
    for _ in range(5):
        sop.mvm_local_dev(Vi, Oi, nrhs, U, W)
    reps = 50
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for e0, e1 in ev:
        e0.record(st)
        sop.mvm_local_dev(Vi, Oi, nrhs, U, W)
        e1.record(st)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b_) for a, b_ in ev]))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    solve = None
    fused = None
    if rank == 0:  # the unsharded single-GPU MVM: the one-launch kernel (fused2d.cu), no all-reduce
        op1 = gk.DskiOperator(gk.KernelSpec(0.02, 1.0), grid, X, (1e-2, 1e-2), device=local)
        bd = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
        V1, O1 = torch.empty_like(bd), torch.empty_like(bd)
        op1.to_internal_dev(bd.data_ptr(), V1.data_ptr(), 1, stream=st.cuda_stream)
        l0 = gk.kernel_launch_count()
        for _ in range(5):
            op1.stage_dev(3, V1.data_ptr(), O1.data_ptr(), 1, stream=st.cuda_stream)
        per_mvm = (gk.kernel_launch_count() - l0) / 5
        ev1 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for e0, e1 in ev1:
            e0.record(st)
            op1.stage_dev(3, V1.data_ptr(), O1.data_ptr(), 1, stream=st.cuda_stream)
            e1.record(st)
        torch.cuda.synchronize()
        ms1 = float(np.median([a.elapsed_time(b_) for a, b_ in ev1]))
        mb = dski_bytes(op1.size(), X.shape[0], 2, grid.size(), 1, 0)
        hbm1 = float(measured_peaks().get("hbm_gbs", 6650.0))
        fused = {"ms_per_mvm": ms1, "value": op1.size() / (ms1 * 1e-3), "unit": UNIT, "gpu_launches_per_mvm": per_mvm,
                 "roofline": {"bound": "hbm", "algorithmic_bytes": mb, "achieved": mb / (ms1 * 1e-3) / 1e9,
                              "peak": hbm1, "unit": "GB/s", "frac": mb / (ms1 * 1e-3) / 1e9 / hbm1,
                              "bytes_formula": "SURVEY 8(d): 8*(3*N*B + 2*n*d + 4*m*B), B = 1"},
                 "timing": "CUDA events per MVM (L2 not evicted), median"}
    if rank == 0 and not args.no_c4_solve:  # BASELINE C4: rank-200 pivoted Cholesky + PCG (one GPU, unsharded)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M = gk.Preconditioner.from_pivchol(op1, gk.pivoted_cholesky(op1, 200, kernel_part=True))
        torch.cuda.synchronize()
        t_pre = time.perf_counter() - t0
        xd = torch.empty_like(bd)
        gk.cg_dev(op1, bd.data_ptr(), xd.data_ptr(), 1, 1e-4, 5, M)  # plans / graphs built outside the timing
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its, conv = gk.cg_dev(op1, bd.data_ptr(), xd.data_ptr(), 1, 1e-4, 1000, M)
        torch.cuda.synchronize()
        t_pcg = time.perf_counter() - t0
        us_it = t_pcg / max(1, int(its[0])) * 1e6
        # HBM roofline of one iteration: the N×200 Woodbury factor Q1 (720 MB,
        # far above L2) is streamed twice (Q1ᵀr, then Q1·c), plus the 1-RHS
        # MVM and ~8 N-vectors of PCG state traffic
        Nn, kk = sop.size(), 200
        it_bytes = 2.0 * 8 * Nn * kk + dski_bytes(Nn, X.shape[0], 2, grid.size(), 1, 0) + 8.0 * 8 * Nn
        peaks = measured_peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        solve = {"precond_build_s": t_pre, "pcg_s": t_pcg, "pcg_iterations": int(its[0]),
                 "pcg_converged": int(conv[0]), "us_per_iteration": us_it,
                 "roofline": {"bound": "hbm", "bytes_per_iteration": it_bytes,
                              "achieved": it_bytes / (us_it * 1e-6) / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": it_bytes / (us_it * 1e-6) / 1e9 / hbm,
                              "bytes_formula": "2*8*N*k (Q1 twice) + MVM bytes (SURVEY 8(d), 1 RHS) + 8*8*N"},
                 "parallelism": "1 GPU (the PCG itself is not slab-sharded)"}
    return {"workload": "C4: D-SKI d=2 n=150000 (N=450000) grid 400x400 SE ell=0.02 sigma=1e-2, 1 RHS", "solve": solve,
            "fused_1gpu": fused,
            "parallelism": f"grid-slab x{world} (NCCL all-reduce of the grid vector per MVM)",
            "scaling": "strong", "ms_per_mvm": ms, "value": sop.size() * nrhs / (ms * 1e-3),
            "unit": UNIT, "local_points": int(sop.mine.size), "build_s": build_s,
            "timing": "CUDA events per MVM on the launching stream (L2 not evicted), median, max over ranks"}


def c5_dskip(args, world, rank, local, dist):
    """C5 (d = 6, n = 10,000, N = 70,000; product SE ℓ = 0.3, rank 30 on
    100-node 1-D grids; 64 RHS per rank): the D-SKIP Hadamard MVM, a DMMA-bound
    Khatri–Rao GEMM pair (4·N·r_A·r_B·B flops). RHS-sharded:
    each rank builds the same operator and owns its own 64 columns (weak)."""
    import torch
    import paper_1810_12283_b200 as gk
    dev = torch.device("cuda", local)
    X, y, dY = gk.make_dataset(5, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = gk.DskipOperator(gk.KernelSpec(0.3, 1.0), X, (1e-2, 1e-2), rank=30, grid_ratio=0.01,
                          max_grid_nodes=100, seed=0, device=local)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    N, nrhs = op.size(), 64
    ranks = [int(f.Q.shape[1]) for f in op.factors()]
    ra, rb = (ranks + [1])[:2]
    g = torch.Generator(device="cpu").manual_seed(1000 + rank)
    V = torch.randn(N * nrhs, dtype=torch.float64, generator=g).to(dev)
    O = torch.empty_like(V)
    flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)
    l0 = gk.kernel_launch_count()
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
    launches = gk.kernel_launch_count() - l0
    for _ in range(3):
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
    reps = 20
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for e0, e1 in ev:
        flush.sum()
        e0.record(st)
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
        e1.record(st)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops = 4.0 * N * ra * rb * nrhs
    peak = gk.dmma_peak_tflops(local)
    # C5 solve (BASELINE: rank-100 pivoted Cholesky, PCG + SLQ with 64 RHS per rank)
    solve = None
    if not args.no_c5_solve:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 100, kernel_part=True))
        torch.cuda.synchronize()
        t_pre = time.perf_counter() - t0
        Bc = np.column_stack([gk.stacked_targets(y, dY, y.mean()) if rank == 0 else
                              gk.rademacher_vector(N, 0, 1000 + rank * nrhs)] +
                             [gk.rademacher_vector(N, 0, 1000 + rank * nrhs + p) for p in range(1, nrhs)])
        Bd = torch.from_numpy(np.ascontiguousarray(Bc.T)).to(dev)
        Xd = torch.empty_like(Bd)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its, conv = gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), nrhs, 1e-4, 1000, M, stream=st.cuda_stream)
        torch.cuda.synchronize()
        t_pcg = time.perf_counter() - t0
        t0 = time.perf_counter()
        slq = gk.slq_logdet(op, nrhs, 50, 0, 0.5e-4, probe_offset=rank * nrhs)
        t_slq = time.perf_counter() - t0
        tt = torch.tensor([t_pre, t_pcg, t_slq], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_pre, t_pcg, t_slq = [float(v) for v in tt.tolist()]
        solve = {"precond_build_s": t_pre, "pcg_s": t_pcg, "slq_s": t_slq, "pcg_plus_slq_s": t_pcg + t_slq,
                 "pcg_iterations_max": int(max(its)), "pcg_converged": int(np.sum(conv)),
                 "slq_probes_per_rank": nrhs, "slq_steps": 50,
                 "note": "tol 1e-4, max 1000 iterations (sigma = 1e-2: the columns do not converge within "
                         "1000, as at C2); times are max over ranks"}
    achieved = world * flops / (ms * 1e-3) / 1e12
    return {"workload": "C5: D-SKIP d=6 n=10000 (N=70000) product SE ell=0.3 sigma=1e-2, rank 30, "
                        "100-node 1-D grids, 64 RHS per rank",
            "parallelism": f"rhs-shard x{world}", "scaling": "weak", "ms_per_mvm": ms,
            "value": world * N * nrhs / (ms * 1e-3), "unit": UNIT, "build_s": build_s,
            "factor_ranks": ranks, "gpu_launches_per_mvm": int(launches), "solve": solve,
            "roofline": {"bound": "tensor (fp64 DMMA)", "achieved": achieved / world, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / world / peak,
                         "flops_per_mvm": flops, "flops_formula": "SURVEY 8(d): 4*N*r_A*r_B*B",
                         "peak_source": "gk_debug_dmma_peak (register-only DMMA m8n8k4 kernel, this GPU, best of 5)"},
            "timing": "CUDA events per MVM on the launching stream, L2 evicted before each (256 MB read), "
                      "median of 20, max over ranks"}


def cpu_baseline(args, full=False):
    """The oracle port of the reference MVM on this host's cores (OpenMP over RHS)."""
    import oracle as O
    X, y, dY, grid = build_problem()
    ref = O.DskiOperator(O.KernelSpec(CONFIG["ell"], 1.0), O.Grid(grid.dims, grid.origin, grid.spacing),
                         X, (CONFIG["noise"], CONFIG["noise"]))
    N, nrhs = ref.size(), CONFIG["nrhs"]
    Bh = rhs_block(N, nrhs, y, dY, 0)
    ref.mvm(Bh[:, :4])  # warm
    reps, times = 0, []
    t_end = time.perf_counter() + (20.0 if full else 10.0)
    while time.perf_counter() < t_end and reps < 50:
        t0 = time.perf_counter()
        ref.mvm(Bh)
        times.append(time.perf_counter() - t0)
        reps += 1
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    med = float(np.median(times))
    return {"value": N * nrhs / med, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{reps} full 32-RHS C2 MVMs (median), OpenMP over RHS columns",
            "ms_per_step": med * 1e3}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle as O
    X, y, dY, grid = build_problem()
    ref = O.DskiOperator(O.KernelSpec(CONFIG["ell"], 1.0), O.Grid(grid.dims, grid.origin, grid.spacing),
                         X, (CONFIG["noise"], CONFIG["noise"]))
    N, nrhs = ref.size(), CONFIG["nrhs"]
    Bh = rhs_block(N, nrhs, y, dY, 0)
    for _ in range(max(args.warmup, 1)):
        ref.mvm(Bh)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.mvm(Bh)
        times.append(time.perf_counter() - t0)
    s = float(np.mean(times))
    value = N * nrhs / s
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded C2 generator)", "config": dict(CONFIG, parallelism="host cores"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full 32-RHS C2 MVMs, OpenMP over RHS columns"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gk", choices=["gk", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 grid-slab sharded MVM measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 D-SKIP MVM measurement")
    ap.add_argument("--no-c5-solve", action="store_true", help="skip the C5 D-SKIP PCG/SLQ solve")
    ap.add_argument("--no-c4-solve", action="store_true", help="skip the C4 rank-200 preconditioned PCG")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    # the contract is ONE JSON line on stdout: everything else any library
    # prints (e.g. NCCL's version banner) goes to stderr at the fd level
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    try:
        if args.impl == "reference":
            line = run_reference(args)
        else:
            line = run_gpu(args)
        try:  # tear NCCL down while stdout still points at stderr
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                dist.destroy_process_group()
        except Exception:
            pass
    finally:
        sys.stdout.flush()
    # write the line on the saved stdout; fd 1 stays on stderr so output at
    # interpreter exit (library teardown banners) cannot follow it
    if line is not None:
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    os.close(json_fd)


if __name__ == "__main__":
    main()
