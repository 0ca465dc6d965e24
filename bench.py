#!/usr/bin/env python
"""Benchmark: batched D-SKI K∇ MVM throughput (rows·RHS/s) on BASELINE config C2
(configs[1]: d=2, n=10,000 -> N=30,000, 100x100 grid, SE ell=0.2, 32 RHS =
y + 31 Rademacher probes), plus the PCG+SLQ solve time on the same operator.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One step = one batched K∇ MVM over the 32-RHS block (scatter B^T, K_UU mode
products, gather B + noise) with inputs resident in HBM; L2 is flushed before
every timed step (the C2 working set, ~34 MB, would otherwise sit in the 126 MB
L2). N>1 (torchrun): every rank holds an operator replica and a slice of the
fixed 32-column batch (strong scaling, no data-path collective; the targets
column on rank 0); time = max over ranks; a weak-scaling figure (32 columns
per rank) is reported beside it. The line also carries the C2 PCG + SLQ solve
(per-iteration rooflines, the reference algorithm's per-iteration cost on the
host cores) and blocks for C1, C3, C4 (grid-slab sharded) and C5 (D-SKIP).
--impl reference times the reference algorithm on the host cores (the C++
oracle port, OpenMP over RHS — the reference cannot be built here, see
DESIGN.md) on the same workload, loading only the oracle library.
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


GRIDS = {1: (0.15, 60), 2: (0.2, 100), 3: (0.3, 48), 4: (0.02, 400)}  # config -> (ℓ, nodes per axis)
NOISE = 1e-2


def make_problem(M, cfg):
    """Seeded config `cfg` from module M (the product `gk` for the GPU arm, the
    oracle `O` for the reference arm: the two generators are bit-identical,
    tests/test_capi_host.py)."""
    X, y, dY = M.make_dataset(cfg, 0)
    grid = M.Grid.cover(X, 1e-4, 3, GRIDS[cfg][1])
    assert [int(x) for x in grid.dims] == [GRIDS[cfg][1]] * X.shape[1]
    return X, y, dY, grid


def build_problem():
    return make_problem(__import__("paper_1810_12283_b200"), 2)


def rhs_cols(M, N, y, dY, cols):
    """Columns of the fixed RHS batch: global column 0 = the stacked targets
    (observations.hpp:29-35), column c >= 1 = rademacher_vector(N, 0, 1000+c-1)
    (the trace-estimator streams, linalg.cpp:264-266)."""
    B = np.empty((N, len(cols)), order="F")
    for j, c in enumerate(cols):
        B[:, j] = M.stacked_targets(y, dY, y.mean()) if c == 0 else M.rademacher_vector(N, 0, 1000 + c - 1)
    return B


def rhs_block(N, nrhs, y, dY, probe_offset):
    import paper_1810_12283_b200 as gk
    return rhs_cols(gk, N, y, dY, [0] + [1 + probe_offset + c for c in range(nrhs - 1)])


def shard(total, world, rank):
    from paper_1810_12283_b200.sharding import shard_range
    return shard_range(total, world, rank)


def ev_time(fn, reps, stream, flush=None):
    """Median device time (ms) of fn() over reps, CUDA events on `stream`,
    optional L2 eviction (outside the events) before each call."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if flush is not None:
            flush.sum()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def wall(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, r


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

    X, y, dY, grid = make_problem(gk, 2)
    n, d = X.shape
    ker = gk.KernelSpec(CONFIG["ell"], 1.0)
    noise = (CONFIG["noise"], CONFIG["noise"])
    op = gk.DskiOperator(ker, grid, X, noise, device=local)
    N, NR, m = op.size(), CONFIG["nrhs"], grid.size()
    # strong scaling: the fixed 32-column batch (targets + 31 probes) is split
    # over the ranks; the targets column lives on rank 0 only
    c0, c1 = shard(NR, world, rank)
    cols = list(range(c0, c1))
    nrhs = len(cols)
    Bh = rhs_cols(gk, N, y, dY, cols)
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
    value = N * NR / (ms * 1e-3)  # the whole fixed batch over the slowest rank's time

    weak = None
    if world > 1:  # weak-scaling figure: every rank runs the full 32-column batch
        Bw = rhs_cols(gk, N, y, dY, [0] + [1 + rank * NR + c for c in range(NR - 1)])
        Vw = torch.from_numpy(np.ascontiguousarray(Bw.T)).to(dev)
        Vwi, Owi = torch.empty(N * NR, dtype=torch.float64, device=dev), torch.empty(N * NR, dtype=torch.float64,
                                                                                     device=dev)
        op.to_internal_dev(Vw.data_ptr(), Vwi.data_ptr(), NR, stream=sp)
        for _ in range(3):
            op.stage_dev(3, Vwi.data_ptr(), Owi.data_ptr(), NR, stream=sp)
        dist.barrier()
        msw = ev_time(lambda: op.stage_dev(3, Vwi.data_ptr(), Owi.data_ptr(), NR, stream=sp), max(args.steps, 10),
                      stream, flush)
        t = torch.tensor([msw], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        weak = {"value": world * N * NR / (float(t.item()) * 1e-3), "unit": UNIT, "ms_per_step": float(t.item()),
                "scaling": "weak", "rhs_per_rank": NR}

    # ---- roofline of the dominant kernel. With the one-launch 2-D MVM the
    # step IS one kernel: its algorithmic bytes are SURVEY §8(d)'s per-MVM
    # figure for this rank's columns.
    Mc = 198 * (198 // 2 + 1)
    mvm_bytes = dski_bytes(N, n, d, m, nrhs, Mc)
    per_step = launches / max(1, args.steps)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    dom, dom_bytes, dom_ms = "one-launch 2-D D-SKI MVM (k_dski_mvm2d / k_lean2d)", mvm_bytes, ms
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None  # DRAM bytes per launch of the dominant kernel from the committed ncu capture
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(f"c2_{nrhs}rhs")
    except Exception:
        traffic = None
    # fp64 work of the step (scatter + gather sum-factorised, two DMMA mode products)
    flops = float(n * nrhs * 348) + 2.0 * m * (int(grid.dims[0]) + int(grid.dims[1])) * nrhs
    dmma_tf = None
    try:
        dmma_tf = gk.dmma_peak_tflops(local)
    except Exception:
        pass

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
    e2e_t = torch.tensor([float(np.mean(e2e_ts)), float(np.median(e2e_ts))], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_mean, e2e_med = [float(v) for v in e2e_t.tolist()]
    e2e_value = N * NR / e2e_mean
    # the same call from pageable (numpy) buffers, as the reference's Eigen
    # callers would pass them (the driver stages the copies)
    Pin = np.asfortranarray(Bh)
    Pout = np.empty_like(Pin, order="F")

    def e2e_pageable():
        gk._check(lib.gk_op_mvm(op.handle, gk._p(Pin), N, gk._p(Pout), N, nrhs))

    e2e_pageable()
    pg = []
    for _ in range(min(e2e_steps, 20)):
        t0 = time.perf_counter()
        e2e_pageable()
        pg.append(time.perf_counter() - t0)
    e2e_pageable_us = float(np.mean(pg)) * 1e6

    solve = c2_solve(gk, op, X, y, dY, cols, world, rank, dev, sp, dist)

    c1 = c3 = c4 = c5 = None
    if rank == 0 and not args.no_c1:
        c1 = guarded(lambda: c1_block(args, gk, dev, stream, flush))
    if rank == 0 and not args.no_c3:
        c3 = guarded(lambda: c3_block(args, gk, dev, stream, flush))
    if not args.no_c4:
        c4 = guarded(lambda: c4_slab(args, world, rank, local, dist))
    if not args.no_c5:
        c5 = guarded(lambda: c5_dskip(args, world, rank, local, dist))

    line = None
    if rank == 0:
        cpu = cpu_baseline(args) if world == 1 and not args.no_cpu_baseline else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded C2 generator)",
            "config": dict(CONFIG, parallelism=f"rhs-shard x{world} (fixed 32-column batch split)" if world > 1
                           else "1 GPU", columns_per_rank=[shard(NR, world, r)[1] - shard(NR, world, r)[0]
                                                           for r in range(world)],
                           l2="evicted before every timed step (256 MB streaming read, outside the timed events)",
                           timing="CUDA events per step on the launching stream, mean of the steps, max over ranks"),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N * nrhs,
                    "d2h_bytes_per_step": 8 * N * nrhs,
                    "path": "gk_op_mvm (C-ABI, pinned host buffers, permutes + copies timed)",
                    "statistic": f"mean of {e2e_steps} host-timed calls, max over ranks",
                    "us_per_call_mean": e2e_mean * 1e6, "us_per_call_median": e2e_med * 1e6,
                    "pageable": {"us_per_call_mean": e2e_pageable_us, "value": N * NR / (e2e_pageable_us * 1e-6),
                                 "path": "gk_op_mvm from pageable numpy buffers (rank 0 of the run, same config)"}},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "traffic_source": "profiles/traffic.json (ncu --set full, one launch)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peaks else "fallback",
                         "bytes_per_launch": dom_bytes, "launch_ms": dom_ms, "launches_per_step": per_step,
                         "bytes_formula": "SURVEY 8(d): 8*(3*N*B + 2*n*d + 4*m*B + M_c)",
                         "fp64": {"flops_per_step": flops, "achieved_tflops": flops / (ms * 1e-3) / 1e12,
                                  "peak_tflops": dmma_tf,
                                  "frac": (flops / (ms * 1e-3) / 1e12 / dmma_tf) if dmma_tf else None,
                                  "flops_formula": "scatter n*B*168 + gather n*B*180 (sum-factorised "
                                                   "stencils) + Toeplitz modes 2*m*(m0+m1)*B (dense DMMA)"}},
            "weak_scaling": weak,
            "solve": solve,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "c1": c1, "c3": c3, "c4_slab": c4, "c5_dskip": c5,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def guarded(fn):
    try:
        return fn()
    except Exception as e:  # reported, never silently replaced
        return {"error": f"{type(e).__name__}: {e}"}


def pcg_iter_bytes(N, n, d, m, nrhs, k, Mc=0):
    """SURVEY §8(d) bytes of one PCG iteration: MVM + preconditioner (Q1 read
    twice, c in/out) + fused CG vector updates."""
    return dski_bytes(N, n, d, m, nrhs, Mc) + 8.0 * (2 * N * k + 2 * N * nrhs) + 8.0 * 9 * N * nrhs


def slq_bytes(N, n, d, m, P, steps, Mc=0):
    """SURVEY §8(d) bytes of a P-probe, s-step SLQ: s batched MVMs plus the
    fused two-pass reorthogonalisation, 8·3·N·j per probe at step j."""
    return steps * dski_bytes(N, n, d, m, P, Mc) + sum(8.0 * 3 * N * j * P for j in range(1, steps + 1))


def c2_solve(gk, op, X, y, dY, cols, world, rank, dev, sp, dist):
    """C2 PCG + SLQ (GpModel::preconditioner/solve/logdet) on this rank's
    columns and probes, with per-iteration rooflines, and the reference
    algorithm's per-iteration cost on the host cores beside it (rank 0, N=1)."""
    import torch
    n, d = X.shape
    N, m = op.size(), op.grid.size()
    k = CONFIG["precond_rank"]
    t_pre, fac = wall(lambda: gk.pivoted_cholesky(op, k, kernel_part=True))
    t_pre2, M = wall(lambda: gk.Preconditioner.from_pivchol(op, fac))
    t_pre += t_pre2
    nrhs = len(cols)
    Bh = rhs_cols(gk, N, y, dY, cols)
    Bd = torch.from_numpy(np.ascontiguousarray(Bh.T)).to(dev)
    Xd = torch.empty_like(Bd)
    t_pcg_first, _ = wall(lambda: gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), nrhs, CONFIG["pcg_tol"], 1000, M,
                                            stream=sp))
    # the same solve again: steady state (plans, graphs and workspaces cached
    # on the operator), what every later solve of a hyperparameter loop costs
    t_pcg, (its, conv) = wall(lambda: gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), nrhs, CONFIG["pcg_tol"], 1000,
                                                M, stream=sp))
    P = CONFIG["slq_probes"]
    p0, p1 = shard(P, world, rank)
    floor = 0.5 * CONFIG["noise"] ** 2
    t_slq_first, _ = wall(lambda: gk.slq_logdet(op, p1 - p0, CONFIG["slq_steps"], 0, floor, probe_offset=p0))
    t_slq, slq = wall(lambda: gk.slq_logdet(op, p1 - p0, CONFIG["slq_steps"], 0, floor, probe_offset=p0))
    slq_logdet = slq.logdet
    if world > 1:  # global estimate over all ranks' probes, summed in probe order
        from paper_1810_12283_b200 import sharding
        est = sharding.gather_probe_estimates(np.asarray(slq.estimates), p0, P, device=dev)
        slq_logdet = sharding.ordered_mean(est)
    tt = torch.tensor([t_pre, t_pcg, t_slq, t_pcg_first, t_slq_first, float(max(its))], device=dev,
                      dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_pre, t_pcg, t_slq, t_pcg_first, t_slq_first, maxit = [float(v) for v in tt.tolist()]
    hbm = float(measured_peaks().get("hbm_gbs", 6650.0))
    it_bytes = pcg_iter_bytes(N, n, d, m, nrhs, k, 198 * 100)
    us_it = t_pcg / max(1.0, maxit) * 1e6
    lz_bytes = slq_bytes(N, n, d, m, p1 - p0, CONFIG["slq_steps"], 198 * 100)
    out = {"precond_build_s": t_pre, "pcg_s": t_pcg, "slq_s": t_slq, "pcg_plus_slq_s": t_pcg + t_slq,
           "pcg_first_call_s": t_pcg_first, "slq_first_call_s": t_slq_first,
           "pcg_iterations_max": int(maxit), "pcg_converged_columns": int(np.sum(conv)),
           "slq_logdet": slq_logdet, "slq_probes_total": P,
           "pcg_iteration": {"us": us_it, "bytes": it_bytes, "achieved_gbs": it_bytes / (us_it * 1e-6) / 1e9,
                             "frac_hbm": it_bytes / (us_it * 1e-6) / 1e9 / hbm,
                             "bytes_formula": "SURVEY 8(d): MVM + 8*(2*N*k + 2*N*B) + 8*9*N*B"},
           "lanczos_step": {"us": t_slq / CONFIG["slq_steps"] * 1e6,
                            "bytes_total": lz_bytes, "achieved_gbs": lz_bytes / t_slq / 1e9,
                            "frac_hbm": lz_bytes / t_slq / 1e9 / hbm,
                            "bytes_formula": "SURVEY 8(d): steps*MVM(P) + sum_j 8*3*N*j*P"},
           "timing": "host wall clock around each call with device syncs, max over ranks; *_s = second "
                     "identical call (steady state); *_first_call_s includes one-time plan/graph setup",
           "note": "tol 1e-4, max 1000 iterations: at sigma = 1e-2 the reference algorithm (oracle) also stops at "
                   "1000 unconverged (relative residual 0.177 for the targets column; tests/golden/c2_cg.json)"}
    if rank == 0 and world == 1:
        out["cpu_reference"] = guarded(lambda: cpu_solver_sample(2, pcg_cols=nrhs, pcg_its=int(maxit),
                                                                 probes=P, steps=CONFIG["slq_steps"],
                                                                 rank_k=k))
    return out


def cpu_solver_sample(cfg, pcg_cols, pcg_its, probes, steps, rank_k, tol=1e-4, sample_its=20, sample_probes=2,
                      sample_steps=None, noise=NOISE):
    """The reference algorithm (oracle port) on this host's cores on bounded
    samples: a `sample_its`-iteration single-RHS PCG (linalg.cpp:85-131) and
    `sample_probes` SLQ probes (linalg.cpp:215-253); full-job CPU times are
    extrapolated per iteration / per probe."""
    import oracle as O
    X, y, dY, grid = make_problem(O, cfg)
    ell = GRIDS[cfg][0]
    ref = O.DskiOperator(O.KernelSpec(ell, 1.0), grid, X, (noise, noise))
    N = ref.size()
    b = O.stacked_targets(y, dY, y.mean())
    t0 = time.perf_counter()
    Pr = None
    if rank_k:
        fr = O.pivoted_cholesky(ref, rank_k, noise_diag=ref.noise_diagonal())
        Pr = O.Preconditioner(fr.L, ref.noise_diagonal())
    t_pre = time.perf_counter() - t0 if rank_k else None
    t0 = time.perf_counter()
    r = O.cg(ref, b, tol, sample_its, Pr)
    t_it = (time.perf_counter() - t0) / max(1, r.iterations)
    ss = sample_steps or steps
    t0 = time.perf_counter()
    O.slq_logdet(ref, sample_probes, ss, 0, 0.5 * noise ** 2)
    t_probe = (time.perf_counter() - t0) / sample_probes * (steps / ss)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"kind": "port", "cores": cores,
            "precond_build_s": t_pre, "pcg_s_per_iteration_per_rhs": t_it,
            "pcg_s_extrapolated": t_it * pcg_cols * pcg_its, "slq_s_per_probe": t_probe,
            "slq_s_extrapolated": t_probe * probes,
            "sample": (f"pivoted Cholesky rank {rank_k} (full); " if rank_k else "no preconditioner (the oracle's "
                       "pivoted Cholesky at this size is minutes of host work); ") +
                      f"{r.iterations} PCG iterations on the targets column; "
                      f"{sample_probes} SLQ probes x {ss} steps; full-job times = per-unit x "
                      f"({pcg_cols} columns x {pcg_its} iterations, {probes} probes x {steps} steps)"}


def c1_block(args, gk, dev, stream, flush):
    """C1 (n = 2,000, 60² grid, ℓ = 0.15, rank 20, tol 1e-8, SLQ 8 × 25): the
    9-column MVM (targets + 8 probes), GpModel at the stated settings (the
    reference's PCG does not reach 1e-8 at σ = 1e-2: max_iterations, not a
    solve), and the whole LML where the solve converges (σ = 0.5, tol 1e-10)
    beside the reference algorithm on the host cores."""
    import torch
    import oracle as O
    X, y, dY, grid = make_problem(gk, 1)
    n = X.shape[0]
    out = {"workload": "C1: D-SKI d=2 n=2000 (N=6000) grid 60x60 SE ell=0.15 sigma=1e-2, rank 20, tol 1e-8, "
                       "SLQ 8x25"}
    op = gk.DskiOperator(gk.KernelSpec(0.15, 1.0), grid, X, (NOISE, NOISE))
    N, nrhs = op.size(), 9
    B = rhs_cols(gk, N, y, dY, list(range(nrhs)))
    Vext = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev)
    Vi, Oi = torch.empty(N * nrhs, dtype=torch.float64, device=dev), torch.empty(N * nrhs, dtype=torch.float64,
                                                                                device=dev)
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=stream.cuda_stream)
    for _ in range(3):
        op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=stream.cuda_stream)
    ms = ev_time(lambda: op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=stream.cuda_stream), 50, stream,
                 flush)
    mb = dski_bytes(N, n, 2, grid.size(), nrhs, 118 * 60)
    hbm = float(measured_peaks().get("hbm_gbs", 6650.0))
    out["mvm"] = {"nrhs": nrhs, "ms": ms, "value": N * nrhs / (ms * 1e-3), "unit": UNIT,
                  "roofline": {"bytes": mb, "achieved_gbs": mb / (ms * 1e-3) / 1e9,
                               "frac_hbm": mb / (ms * 1e-3) / 1e9 / hbm}}
    ref = O.DskiOperator(O.KernelSpec(0.15, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X, (NOISE, NOISE))
    t0 = time.perf_counter()
    ref.mvm(B)
    out["mvm"]["cpu_reference_ms"] = (time.perf_counter() - t0) * 1e3
    kw = dict(backend="dski", grid_ratio=1e-3, max_grid_nodes=60, precond_rank=20, slq_probes=8, slq_steps=25, seed=0)
    # stated settings: PCG to tol 1e-8 stops at max_iterations (as the reference's)
    gm = gk.GpModel(gk.KernelSpec(0.15, 1.0), X, y, dY, noise=(NOISE, NOISE), tol=1e-8, max_iterations=2000, **kw)
    t_pre, M = wall(lambda: gm.preconditioner())
    b = gm.stacked_targets()
    t_pcg, res = wall(lambda: gk.cg(gm.op(), b, 1e-8, 2000, M, history=False))
    t_slq, ld = wall(lambda: gm.logdet())
    out["stated"] = {"precond_build_s": t_pre, "pcg_s": t_pcg, "pcg_iterations": res.iterations,
                     "pcg_converged": bool(res.converged), "pcg_us_per_iteration": t_pcg / max(1, res.iterations) * 1e6,
                     "slq_s": t_slq, "logdet": ld,
                     "note": "the reference algorithm also stops at max_iterations here "
                             "(tests/test_gpu_fullsize_parity.py::test_c1_stated_settings)"}
    # converging variant: the full LML (alpha solve + SLQ), GPU vs the reference on the host cores
    gm2 = gk.GpModel(gk.KernelSpec(0.15, 1.0), X, y, dY, noise=(0.5, 0.5), tol=1e-10, max_iterations=3000, **kw)
    gm2.preconditioner()
    gm2.log_marginal_likelihood()  # plans/graphs built outside the timing
    t_lml, lml = wall(lambda: gm2.log_marginal_likelihood())
    its = gk.cg(gm2.op(), gm2.stacked_targets(), 1e-10, 3000, gm2.preconditioner(), history=False).iterations
    t0 = time.perf_counter()
    rm = O.GpModel(O.KernelSpec(0.15, 1.0), X, y, dY, noise=(0.5, 0.5), tol=1e-10, max_iterations=3000, **kw)
    rl = rm.log_marginal_likelihood()
    t_cpu = time.perf_counter() - t0
    out["lml_converging"] = {"sigma": 0.5, "tol": 1e-10, "gpu_s": t_lml, "pcg_iterations": its, "lml": lml,
                             "cpu_reference_s": t_cpu, "cpu_lml": rl["lml"], "cpu_iterations": rl["iterations"],
                             "cpu_cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
                             "cpu_timing": "oracle GpModel: preconditioner + PCG + SLQ (everything), wall clock",
                             "gpu_timing": "GpModel.log_marginal_likelihood (PCG + SLQ), second call, wall clock"}
    return out


def c3_block(args, gk, dev, stream, flush):
    """C3 (d = 3, n = 25,001, 48³ grid, ℓ = 0.3, rank 100, tol 1e-6, y + 16
    SLQ probes × 50 steps): the 17-column MVM, the PCG on the targets and the
    SLQ, with the reference algorithm's per-unit cost on the host cores."""
    import torch
    import oracle as O
    X, y, dY, grid = make_problem(gk, 3)
    n = X.shape[0]
    op = gk.DskiOperator(gk.KernelSpec(0.3, 1.0), grid, X, (NOISE, NOISE))
    N, nrhs = op.size(), 17
    B = rhs_cols(gk, N, y, dY, list(range(nrhs)))
    Vext = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev)
    Vi, Oi = torch.empty(N * nrhs, dtype=torch.float64, device=dev), torch.empty(N * nrhs, dtype=torch.float64,
                                                                                device=dev)
    sp = stream.cuda_stream
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=sp)
    l0 = gk.kernel_launch_count()
    for _ in range(3):
        op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=sp)
    per = (gk.kernel_launch_count() - l0) / 3
    ms = ev_time(lambda: op.stage_dev(3, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=sp), 20, stream, flush)
    mb = dski_bytes(N, n, 3, grid.size(), nrhs, 94 * 94 * 48)
    hbm = float(measured_peaks().get("hbm_gbs", 6650.0))
    stages = {}
    U = torch.empty(grid.size() * nrhs, dtype=torch.float64, device=dev)
    W = torch.empty_like(U)
    for name, st, a, b in (("scatter", 0, Vi, U), ("kuu", 1, U, W), ("gather", 2, W, Oi)):
        stages[name] = ev_time(lambda: op.stage_dev(st, a.data_ptr(), b.data_ptr(), nrhs, stream=sp), 20, stream,
                               flush)
    # the same MVM replayed from its cached CUDA graph (stage 4: one launch for
    # the six kernels, as the PCG iteration graphs run it)
    ms_graph = ev_time(lambda: op.stage_dev(4, Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=sp), 20, stream, flush)
    out = {"workload": "C3: D-SKI d=3 n=25001 (N=100004) grid 48^3 SE ell=0.3 sigma=1e-2, rank 100, tol 1e-6, "
                       "y + 16 SLQ probes x 50 steps",
           "mvm": {"nrhs": nrhs, "ms": ms, "value": N * nrhs / (ms * 1e-3), "unit": UNIT, "launches": per,
                   "graph_ms": ms_graph, "stages_ms": stages,
                   "roofline": {"bytes": mb, "achieved_gbs": mb / (ms * 1e-3) / 1e9,
                                "frac_hbm": mb / (ms * 1e-3) / 1e9 / hbm,
                                "bytes_formula": "SURVEY 8(d) (C3, B=17: 105.6 MB)"}}}
    t_pre, fac = wall(lambda: gk.pivoted_cholesky(op, 100, kernel_part=True))
    t_pre2, M = wall(lambda: gk.Preconditioner.from_pivchol(op, fac))
    b = gk.stacked_targets(y, dY, y.mean())
    gk.cg(op, b, 1e-6, 5, M, history=False)  # plans / graphs outside the timing
    t_pcg, res = wall(lambda: gk.cg(op, b, 1e-6, 1000, M, history=False))
    t_slq, slq = wall(lambda: gk.slq_logdet(op, 16, 50, 0, 0.5 * NOISE ** 2))
    us_it = t_pcg / max(1, res.iterations) * 1e6
    ib = pcg_iter_bytes(N, n, 3, grid.size(), 1, 100, 94 * 94 * 48)
    out["solve"] = {"precond_build_s": t_pre + t_pre2, "pcg_s": t_pcg, "pcg_iterations": res.iterations,
                    "pcg_converged": bool(res.converged), "pcg_us_per_iteration": us_it,
                    "pcg_iteration_roofline": {"bytes": ib, "achieved_gbs": ib / (us_it * 1e-6) / 1e9,
                                               "frac_hbm": ib / (us_it * 1e-6) / 1e9 / hbm},
                    "slq_s": t_slq, "slq_logdet": slq.logdet, "pcg_plus_slq_s": t_pcg + t_slq}
    ref = O.DskiOperator(O.KernelSpec(0.3, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X, (NOISE, NOISE))
    t0 = time.perf_counter()
    ref.mvm(B)
    t_mvm = time.perf_counter() - t0
    out["cpu_reference"] = {"mvm_ms_17rhs": t_mvm * 1e3,
                            "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "kind": "port"}
    out["cpu_reference"].update(guarded(lambda: cpu_solver_sample(3, 1, res.iterations, 16, 50, None, tol=1e-6,
                                                                  sample_its=3, sample_probes=1, sample_steps=5)))
    return out


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
        if world == 1:  # the reference algorithm for the same 1-RHS MVM on the host cores
            import oracle as O
            ro = O.DskiOperator(O.KernelSpec(0.02, 1.0), O.Grid(grid.dims, grid.origin, grid.spacing), X,
                                (1e-2, 1e-2))
            ro.mvm(b)
            t0 = time.perf_counter()
            for _ in range(3):
                ro.mvm(b)
            fused["cpu_reference"] = {"ms_per_mvm": (time.perf_counter() - t0) / 3 * 1e3, "kind": "port",
                                      "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
                                      "sample": "3 single-RHS C4 MVMs (mean; FFT of the 798² embedding)"}
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
                 "parallelism": "1 GPU, unsharded (the fused single-GPU PCG path)"}
    slab_solve = None
    if not args.no_c4_solve:  # the same solve with rows sharded by grid slab (slab_solver.py)
        from paper_1810_12283_b200 import slab_solver as S
        be = S.GpuSlabBackend(sop)
        t_pc, f = wall(lambda: S.slab_pivoted_cholesky(be, 200))
        t_pb, Ms = wall(lambda: S.SlabPreconditioner(be, f.L, be.noise_diag()))
        bl = torch.from_numpy(np.ascontiguousarray(b[rows]).reshape(-1, 1)).to(dev)
        S.slab_cg(be, bl, 1e-4, 3, Ms)  # warm
        if world > 1:
            dist.barrier()
        t_cg, res = wall(lambda: S.slab_cg(be, bl, 1e-4, 1000, Ms))
        tt = torch.tensor([t_pc, t_pb, t_cg], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_pc, t_pb, t_cg = [float(v) for v in tt.tolist()]
        slab_solve = {"pivchol_s": t_pc, "precond_build_s": t_pb, "pcg_s": t_cg,
                      "pcg_iterations": int(res.iterations[0]), "pcg_converged": bool(res.converged[0]),
                      "us_per_iteration": t_cg / max(1, res.iterations[0]) * 1e6,
                      "parallelism": f"grid-slab x{world}: rows sharded; CG dots, the k x B preconditioner "
                                     "projection and the grid vector all-reduced over NCCL; max-loc pivots",
                      "timing": "host wall clock, max over ranks"}
    return {"workload": "C4: D-SKI d=2 n=150000 (N=450000) grid 400x400 SE ell=0.02 sigma=1e-2, 1 RHS", "solve": solve,
            "slab_solve": slab_solve,
            "fused_1gpu": fused,
            "parallelism": f"grid-slab x{world} (NCCL all-reduce of the grid vector per MVM)",
            "scaling": "strong", "ms_per_mvm": ms, "value": sop.size() * nrhs / (ms * 1e-3),
            "unit": UNIT, "local_points": int(sop.mine.size), "build_s": build_s,
            "timing": "CUDA events per MVM on the launching stream (L2 not evicted), median, max over ranks"}


def c5_dskip(args, world, rank, local, dist):
    """C5 (d = 6, n = 10,000, N = 70,000; product SE ℓ = 0.3, rank 30 on
    100-node 1-D grids; the fixed 64-column batch): the D-SKIP Hadamard MVM, a
    DMMA-bound Khatri–Rao GEMM pair (4·N·r_A·r_B·B flops).
    RHS-sharded (strong scaling): every rank builds the same operator and owns
    a slice of the 64 columns / probes; the targets column lives on rank 0."""
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
    N, NR = op.size(), 64
    c0, c1 = shard(NR, world, rank)
    nrhs = c1 - c0
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
        Bc = rhs_cols(gk, N, y, dY, list(range(c0, c1)))
        Bd = torch.from_numpy(np.ascontiguousarray(Bc.T)).to(dev)
        Xd = torch.empty_like(Bd)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its, conv = gk.cg_dev(op, Bd.data_ptr(), Xd.data_ptr(), nrhs, 1e-4, 1000, M, stream=st.cuda_stream)
        torch.cuda.synchronize()
        t_pcg = time.perf_counter() - t0
        t0 = time.perf_counter()
        slq = gk.slq_logdet(op, nrhs, 50, 0, 0.5e-4, probe_offset=c0)
        t_slq = time.perf_counter() - t0
        tt = torch.tensor([t_pre, t_pcg, t_slq], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_pre, t_pcg, t_slq = [float(v) for v in tt.tolist()]
        solve = {"precond_build_s": t_pre, "pcg_s": t_pcg, "slq_s": t_slq, "pcg_plus_slq_s": t_pcg + t_slq,
                 "pcg_iterations_max": int(max(its)), "pcg_converged": int(np.sum(conv)),
                 "slq_probes_total": NR, "slq_steps": 50,
                 "note": "tol 1e-4, max 1000 iterations (sigma = 1e-2: the columns do not converge within "
                         "1000, as at C2); times are max over ranks"}
    achieved = flops / (ms * 1e-3) / 1e12  # the slowest rank's columns over its time
    return {"workload": "C5: D-SKIP d=6 n=10000 (N=70000) product SE ell=0.3 sigma=1e-2, rank 30, "
                        "100-node 1-D grids, fixed 64-column batch",
            "parallelism": f"rhs-shard x{world}", "scaling": "strong", "ms_per_mvm": ms,
            "value": N * NR / (ms * 1e-3), "unit": UNIT, "build_s": build_s, "columns_on_rank0": nrhs,
            "factor_ranks": ranks, "gpu_launches_per_mvm": int(launches), "solve": solve,
            "roofline": {"bound": "tensor (fp64 DMMA)", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "flops_per_mvm": flops, "flops_formula": "SURVEY 8(d): 4*N*r_A*r_B*B",
                         "peak_source": "gk_debug_dmma_peak (register-only DMMA m8n8k4 kernel, this GPU, best of 5)"},
            "timing": "CUDA events per MVM on the launching stream, L2 evicted before each (256 MB read), "
                      "median of 20, max over ranks"}


def oracle_c2():
    """The C2 workload built by the oracle library alone (no product code
    loaded): its own generator, Grid::cover, stacked targets and probes."""
    import oracle as O
    X, y, dY, grid = make_problem(O, 2)
    ref = O.DskiOperator(O.KernelSpec(CONFIG["ell"], 1.0), grid, X, (CONFIG["noise"], CONFIG["noise"]))
    N, nrhs = ref.size(), CONFIG["nrhs"]
    return ref, N, nrhs, rhs_cols(O, N, y, dY, list(range(nrhs)))


def cpu_baseline(args):
    """The reference algorithm (oracle port) for the C2 MVM on this host's
    cores (OpenMP over RHS), on a bounded sample: ~10 s of steps, mean."""
    ref, N, nrhs, Bh = oracle_c2()
    ref.mvm(Bh)  # warm
    times = []
    t_end = time.perf_counter() + 10.0
    while time.perf_counter() < t_end and len(times) < 50:
        t0 = time.perf_counter()
        ref.mvm(Bh)
        times.append(time.perf_counter() - t0)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    s = float(np.mean(times))
    return {"value": N * nrhs / s, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(times)} full 32-RHS C2 MVMs (mean), OpenMP over RHS columns", "ms_per_step": s * 1e3}


def run_reference(args):
    """--impl reference: the reference algorithm for this path (the oracle port
    of dski.cpp:228-238 — the reference itself cannot be built here,
    DESIGN.md §1) on the host cores, on the same config / metric / unit as the
    GPU arm. Only the oracle library is loaded. Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    ref, N, nrhs, Bh = oracle_c2()
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
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded C2 generator)",
            "config": dict(CONFIG, parallelism="host cores (OpenMP over RHS)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full 32-RHS C2 MVMs (mean), OpenMP over RHS columns"},
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
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 block (MVM, GpModel solve/LML)")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 block (d = 3 MVM, PCG, SLQ)")
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
