"""The gradkrig tool subcommands on the B200 path:
`fit`, `predict`, `benchmark-mvm` and `precond-study`, with the reference's
flags (proj/tools/common.cpp:14-37 and each cmd_*.cpp), file formats
(paper_1810_12283_b200.io) and exit codes (proj/tools/common.hpp:14-18:
0 ok, 2 config error, 3 solver non-convergence, 4 data error;
common.cpp:86-100 classifies exceptions). Run as

    python -m paper_1810_12283_b200 fit --data train.csv --backend dski ...

The operators, solves, log-determinants, gradients and predictions all run in
libgk_b200.so on the GPU; this module is argument parsing, file I/O and the
host control flow of the tools. Differences from the reference tools:
  - benchmark-mvm times "exact" through the matrix-free device operator
    (ExactOperator) instead of an assembled DenseOperator (same product).
  - `--kernel spline` runs on the dski backend (K_UU by circulant embedding
    and an in-house FFT); dskip rejects it like the reference
    (dskip.cpp:118-121, exit 2).
  - GRADKRIG_THREADS is accepted and ignored (no host worker pool).
  - subcommands terrain / active-subspace / bo are out of scope.
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

EXIT_OK, EXIT_CONFIG, EXIT_SOLVER, EXIT_DATA = 0, 2, 3, 4


class ConfigError(ValueError):
    """std::invalid_argument raised by the tool layer (exit 2)."""


def _gk():
    import paper_1810_12283_b200 as gk
    return gk


def _onoff(v: str) -> bool:
    m = {"on": True, "off": False, "1": True, "0": False}
    try:
        return m[v.lower()]
    except KeyError:
        raise argparse.ArgumentTypeError(f"{v} not in {{on, off, 1, 0}}") from None


def add_common_flags(p: argparse.ArgumentParser) -> None:
    """add_common_flags (proj/tools/common.cpp:14-37)."""
    p.add_argument("--kernel", default="se", choices=["se", "spline"], help="kernel family")
    p.add_argument("--backend", default="exact", choices=["exact", "dski", "dskip"],
                   help="kernel operator backend (exact, dski, dskip)")
    p.add_argument("--ell", type=float, default=0.0, help="initial lengthscale (0: heuristic)")
    p.add_argument("--outputscale", type=float, default=0.0, help="initial output scale (0: heuristic)")
    p.add_argument("--noise", type=float, default=1e-2, help="value noise sigma1")
    p.add_argument("--noise-grad", type=float, default=1e-2, help="gradient noise sigma2")
    p.add_argument("--grid-ratio", type=float, default=0.2, help="grid spacing as a fraction of ell")
    p.add_argument("--grid-size", type=int, default=128, help="grid node cap per dimension")
    p.add_argument("--rank", type=int, default=100, help="preconditioner / D-SKIP rank")
    p.add_argument("--tol", type=float, default=1e-4, help="CG relative residual tolerance")
    p.add_argument("--maxit", type=int, default=1000, help="CG iteration cap")
    p.add_argument("--probes", type=int, default=10, help="probe vectors for stochastic estimators")
    p.add_argument("--seed", type=int, default=0, help="random seed")
    p.add_argument("--precond", type=_onoff, default=True, help="preconditioning on/off")
    p.add_argument("--variance", default="pivchol", choices=["exact", "pivchol", "randomized"],
                   help="predictive variance estimator")


def make_gp_config(a):
    """make_gp_config (proj/tools/common.cpp:39-53)."""
    from .io import SolverConfig
    return SolverConfig(backend=a.backend, grid_ratio=a.grid_ratio, max_grid_nodes=a.grid_size, dskip_rank=a.rank,
                        cg_tol=a.tol, cg_maxit=a.maxit, precond=a.precond, precond_rank=a.rank,
                        slq_probes=a.probes, gradient_probes=max(4, a.probes // 2), seed=a.seed)


def make_kernel(a, X):
    """make_kernel (proj/tools/common.cpp:55-72): ℓ defaults to 0.2 × the
    bounding-box diagonal, s to 1."""
    gk = _gk()
    span2 = sum(float(X[:, j].max() - X[:, j].min()) ** 2 for j in range(X.shape[1]))
    diag = math.sqrt(max(span2, 1e-12))
    ell = a.ell if a.ell > 0 else 0.2 * diag
    s = a.outputscale if a.outputscale > 0 else 1.0
    if a.kernel == "spline":  # constants calibrated on the data's scaled diameter (common.cpp:66-69)
        sa, sb, even = gk.spline_constants_for_domain(diag / ell, X.shape[1])
        return gk.KernelSpec(ell, s, gk.SPLINE, sa, sb, even)
    return gk.KernelSpec(ell, s)


def build_model(kernel, X, y, dY, noise_value, noise_gradient, cfg):
    """GpModel(kernel, data, cfg) with the tool's config (gp.cpp:33-44)."""
    gk = _gk()
    return gk.GpModel(kernel, X, y, dY, noise=(noise_value, noise_gradient), backend=cfg.backend,
                      grid_ratio=cfg.grid_ratio, max_grid_nodes=cfg.max_grid_nodes, dskip_rank=cfg.dskip_rank,
                      tol=cfg.cg_tol, max_iterations=cfg.cg_maxit, use_preconditioner=cfg.precond,
                      precond_rank=cfg.precond_rank, slq_probes=cfg.slq_probes, slq_steps=cfg.slq_steps,
                      gradient_probes=cfg.gradient_probes, seed=cfg.seed)


# ------------------------------------------------------------------ fit
def run_fit(a) -> None:
    """run_fit (proj/tools/cmd_fit.cpp:21-61)."""
    from . import io
    t0 = time.monotonic()
    raw = io.read_dataset_csv(a.data)
    if a.no_gradients:
        raw.G = None
    X, y, dY = raw.to_observations(a.noise, a.noise_grad)
    kernel = make_kernel(a, X)
    cfg = make_gp_config(a)
    model = build_model(kernel, X, y, dY, a.noise, a.noise_grad, cfg)
    res = model.fit(max_iterations=a.iters, restarts=a.restarts, seed=a.seed)
    k = res.kernel
    out = io.ModelFile(family="spline" if k.family == 1 else "se", spline_a=k.spline_a, spline_b=k.spline_b,
                       spline_even=bool(k.spline_even), lengthscale=k.lengthscale, outputscale=k.outputscale,
                       noise_value=res.noise_value, noise_gradient=res.noise_gradient, mean=model.mean,
                       backend=cfg.backend, config=cfg, data_path=a.data, with_gradients=dY is not None)
    io.save_model(a.model, out)
    wall = time.monotonic() - t0
    iters = sum(r.iterations for r in res.restarts)
    print(f"fit: n={X.shape[0]} d={X.shape[1]} gradients={'yes' if dY is not None else 'no'} "
          f"backend={cfg.backend}\n"
          f"  ell={res.kernel.lengthscale:.6g} s={res.kernel.outputscale:.6g} sigma1={res.noise_value:.6g} "
          f"sigma2={res.noise_gradient:.6g}\n"
          f"  log-marginal={res.log_marginal:.6g} iterations={iters} wall[s]={wall:.6g}\n"
          f"  model written to {a.model}")


# ------------------------------------------------------------------ predict
def run_predict(a) -> None:
    """run_predict (proj/tools/cmd_predict.cpp:21-75)."""
    from . import io
    gk = _gk()
    m = io.load_model(a.model)
    train = io.read_dataset_csv(m.data_path)
    if not m.with_gradients:
        train.G = None
    X, y, dY = train.to_observations(m.noise_value, m.noise_gradient)
    test = io.read_dataset_csv(a.test, False)
    Xtest = test.X
    if m.projection is not None:
        P = m.projection
        X = np.asfortranarray(X @ P)
        if dY is not None:
            dY = np.asfortranarray(dY @ P)
        Xtest = Xtest @ P
    if m.family == "spline":
        kernel = gk.KernelSpec(m.lengthscale, m.outputscale, gk.SPLINE, m.spline_a, m.spline_b, m.spline_even)
    else:
        kernel = gk.KernelSpec(m.lengthscale, m.outputscale)
    model = build_model(kernel, X, y, dY, m.noise_value, m.noise_gradient, m.config)
    model.set_hyperparameters(kernel, m.noise_value, m.noise_gradient)
    Xtest = np.asfortranarray(Xtest)
    mean, grads = model.predict_mean_grad(Xtest)
    if a.variance == "randomized":
        var = model.predict_variance_randomized(Xtest, a.probes, a.seed)
    elif a.variance == "exact":
        var = model.predict_variance_exact(Xtest)
    else:
        var = model.predict_variance_pivchol(Xtest)
    d = test.dim()
    header = [f"x{j + 1}" for j in range(d)] + ["mean", "variance"]
    if a.gradients:
        header += [f"dmean{j + 1}" for j in range(grads.shape[1])]
    rows = []
    for t in range(Xtest.shape[0]):
        row = list(test.X[t]) + [mean[t], var[t]]
        if a.gradients:
            row += list(grads[t])
        rows.append(row)
    io.write_csv(a.out, header, rows)
    print(f"predict: {Xtest.shape[0]} points, variance={a.variance}, written to {a.out}")


# ------------------------------------------------------------------ benchmark-mvm
def bench_points(n, dim, seed):
    """X (n×dim) uniform on the unit cube from seeded_rng(seed, n), drawn row
    by row (cmd_benchmark_mvm.cpp:49-53)."""
    gk = _gk()
    return np.asfortranarray(gk.uniform_vector(n * dim, seed, n, 0.0, 1.0).reshape(n, dim))


def bench_operator(backend, X, grid_nodes, rank, seed):
    """The operator cmd_benchmark_mvm.cpp:55-80 builds: SE(0.4, 1), noise
    (0.1, 0.1); D-SKI on a fixed grid of grid_nodes per dimension over
    [−0.25, 1.25]; D-SKIP of the given rank; exact = the dense K∇ product
    (here the matrix-free device operator, no noise — DenseOperator(K))."""
    gk = _gk()
    n, dim = X.shape
    ker = gk.KernelSpec(0.4, 1.0)
    if backend == "dski":
        g = gk.Grid([grid_nodes] * dim, [-0.25] * dim, [1.5 / (grid_nodes - 1)] * dim)
        return gk.DskiOperator(ker, g, X, (0.1, 0.1))
    if backend == "dskip":
        return gk.DskipOperator(ker, X, (0.1, 0.1), rank=rank, seed=seed)
    if n * (dim + 1) > 20000:  # AssemblyOptions size_cap = 4e8 entries (cmd_benchmark_mvm.cpp:72-74)
        raise RuntimeError(f"dense K has {(n * (dim + 1)) ** 2} entries, above the cap 400000000")
    return gk.ExactOperator(ker, X, (0.0, 0.0))


def median_mvm_seconds(op, reps, seed, device=False):
    """median_mvm_seconds (cmd_benchmark_mvm.cpp:26-39): one warm-up MVM then
    the median of `reps` timed MVMs of gaussian_vector(N, seed). Host buffers
    through the C-ABI (the reference's call), or with device=True device-
    resident vectors timed with CUDA events."""
    gk = _gk()
    v = gk.gaussian_vector(op.size(), seed)
    if not device:
        op.mvm(v)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            op.mvm(v)
            times.append(time.perf_counter() - t0)
    else:
        import torch
        dv = torch.from_numpy(v).cuda()
        do = torch.empty_like(dv)
        s = torch.cuda.current_stream()
        op.mvm_dev(dv.data_ptr(), do.data_ptr(), 1, stream=s.cuda_stream)
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            op.mvm_dev(dv.data_ptr(), do.data_ptr(), 1, stream=s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
    times.sort()
    return times[len(times) // 2]


def run_benchmark_mvm(a) -> None:
    """run_bench (proj/tools/cmd_benchmark_mvm.cpp:41-102)."""
    from . import io
    backend = io.backend_from_string(a.backend)
    rows, logn, logt = [], [], []
    for n in a.sizes:
        X = bench_points(n, a.dim, a.seed)
        op = bench_operator(backend, X, a.grid_nodes, a.rank, a.seed)
        sec = median_mvm_seconds(op, a.reps, a.seed + 7, a.device_resident)
        rows.append([n, op.size(), sec])
        logn.append(math.log(n))
        logt.append(math.log(sec))
        print(f"n={n} N={op.size()} mvm[s]={sec:.6g}")
    m = float(len(logn))
    sx, sy = sum(logn), sum(logt)
    sxx = sum(v * v for v in logn)
    sxy = sum(x * y for x, y in zip(logn, logt))
    den = m * sxx - sx * sx
    slope = (m * sxy - sx * sy) / den if den != 0 else float("nan")
    print(f"log-log slope: {slope:.6g}")
    io.write_csv(a.out, ["n", "N", "seconds"], rows)
    print(f"timings written to {a.out}")


# ------------------------------------------------------------------ precond-study
def run_precond_study(a) -> None:
    """run_study (proj/tools/cmd_precond_study.cpp:29-98): CG vs PCG iteration
    counts over a log-spaced (ℓ, σ) sweep on Franke (D-SKI) or Friedman
    (D-SKIP) data with normalised targets."""
    from . import io
    gk = _gk()
    use_dskip = a.function == "friedman"
    n = a.n if a.n > 0 else (1000 if use_dskip else 2000)
    X, y, dY = gk.sample_test_function(a.function, n, a.seed)
    yscale = math.sqrt(float(np.mean((y - y.mean()) ** 2)))
    y = (y - y.mean()) / yscale
    dY = dY / yscale
    rows = []
    P = a.sweep_points
    for ei in range(P):
        te = 0.0 if P == 1 else ei / (P - 1)
        ell = 10.0 ** (a.log_ell_lo + te * (a.log_ell_hi - a.log_ell_lo))
        for si in range(P):
            ts = 0.0 if P == 1 else si / (P - 1)
            sigma = 10.0 ** (a.log_sigma_lo + ts * (a.log_sigma_hi - a.log_sigma_lo))
            ker = gk.KernelSpec(ell, 1.0)
            if use_dskip:
                op = gk.DskipOperator(ker, X, (sigma, sigma), rank=a.rank, seed=a.seed)
            else:
                grid = gk.Grid.cover(X, a.grid_ratio * ell, 3, a.grid_size)
                op = gk.DskiOperator(ker, grid, X, (sigma, sigma))
            b = gk.stacked_targets(y, dY, float(y.mean()))
            plain = gk.cg(op, b, a.tol, a.maxit, history=False)
            f = gk.pivoted_cholesky(op, min(a.rank, op.size()), kernel_part=True)
            M = gk.Preconditioner.from_pivchol(op, f)
            pre = gk.cg(op, b, a.tol, a.maxit, M, history=False)
            rows.append([ell, sigma, plain.iterations, 1.0 if plain.converged else 0.0, pre.iterations,
                         1.0 if pre.converged else 0.0])
            print(f"ell={ell:.6g} sigma={sigma:.6g}  CG {plain.iterations}"
                  f"{'' if plain.converged else ' (no convergence)'}  PCG {pre.iterations}"
                  f"{'' if pre.converged else ' (no convergence)'}")
    io.write_csv(a.out, ["ell", "sigma", "cg_iters", "cg_converged", "pcg_iters", "pcg_converged"], rows)
    print(f"study written to {a.out}")


# ------------------------------------------------------------------ main
def _sizes(v: str):
    return [int(t) for t in v.split(",") if t.strip()]


def build_parser() -> argparse.ArgumentParser:
    app = argparse.ArgumentParser(prog="gradkrig-b200",
                                  description="scalable Gaussian process regression with derivatives (B200)")
    sub = app.add_subparsers(dest="command", required=True)

    p = sub.add_parser("fit", help="fit hyperparameters and write a model file")
    p.add_argument("--data", required=True, help="training CSV (x1..xD, y[, g1..gD])")
    p.add_argument("--model", default="model.json", help="output model JSON path")
    p.add_argument("--iters", type=int, default=40, help="optimizer iterations")
    p.add_argument("--restarts", type=int, default=3, help="optimizer restarts")
    p.add_argument("--no-gradients", action="store_true", help="ignore gradient columns even if present")
    add_common_flags(p)
    p.set_defaults(run=run_fit)

    p = sub.add_parser("predict", help="predict mean and variance from a model file")
    p.add_argument("--model", required=True, help="model JSON from 'fit'")
    p.add_argument("--test", required=True, help="test CSV (x1..xD[, y ignored])")
    p.add_argument("--out", default="predictions.csv", help="output CSV path")
    p.add_argument("--variance", default="pivchol", choices=["exact", "pivchol", "randomized"])
    p.add_argument("--probes", type=int, default=64, help="probes for the randomized estimator")
    p.add_argument("--seed", type=int, default=0, help="seed for the randomized estimator")
    p.add_argument("--gradients", action="store_true", help="also write predicted gradient columns")
    p.set_defaults(run=run_predict)

    p = sub.add_parser("benchmark-mvm", help="MVM timings over growing n")
    p.add_argument("--backend", default="dski", choices=["exact", "dski", "dskip"])
    p.add_argument("--sizes", type=_sizes, default=[2000, 4000, 8000, 16000], help="point counts to time")
    p.add_argument("--dim", type=int, default=2, help="input dimension")
    p.add_argument("--reps", type=int, default=7, help="repetitions per size (median reported)")
    p.add_argument("--out", default="mvm_bench.csv", help="output CSV")
    p.add_argument("--seed", type=int, default=0, help="random seed")
    p.add_argument("--grid-nodes", type=int, default=32, help="fixed D-SKI grid nodes per dim")
    p.add_argument("--rank", type=int, default=100, help="D-SKIP rank")
    p.add_argument("--device-resident", action="store_true",
                   help="time device-resident vectors with CUDA events instead of host-buffer calls")
    p.set_defaults(run=run_benchmark_mvm)

    p = sub.add_parser("precond-study", help="CG vs PCG iteration counts over a (ell, sigma) sweep")
    p.add_argument("--function", default="franke", choices=["franke", "friedman"])
    p.add_argument("--n", type=int, default=0, help="training points (default 2000 / 1000)")
    p.add_argument("--out", default="precond_study.csv", help="output CSV")
    p.add_argument("--rank", type=int, default=100, help="pivoted Cholesky rank")
    p.add_argument("--tol", type=float, default=1e-4, help="CG tolerance")
    p.add_argument("--maxit", type=int, default=1000, help="CG iteration cap")
    p.add_argument("--sweep-points", type=int, default=5, help="points per sweep axis")
    p.add_argument("--seed", type=int, default=0, help="random seed")
    p.add_argument("--grid-ratio", type=float, default=0.25, help="D-SKI grid spacing / ell")
    p.add_argument("--grid-size", type=int, default=64, help="D-SKI grid cap per dimension")
    p.set_defaults(run=run_precond_study, log_ell_lo=-1.0, log_ell_hi=1.0, log_sigma_lo=-3.0, log_sigma_hi=0.0)
    return app


def classify_exception(e: BaseException) -> int:
    """classify_exception (proj/tools/common.cpp:86-100)."""
    gk = _gk()
    what = str(e)
    if isinstance(e, gk.OutOfGridError):
        return EXIT_DATA
    if isinstance(e, ValueError):  # std::invalid_argument
        return EXIT_CONFIG
    if "did not converge" in what or "restarts failed" in what:
        return EXIT_SOLVER
    if "malformed" in what or "cannot open" in what or "row" in what:
        return EXIT_DATA
    return EXIT_SOLVER


def main(argv=None) -> int:
    app = build_parser()
    try:
        a = app.parse_args(argv)
    except SystemExit as e:  # argparse: --help exits 0, parse errors exit 2 (kExitConfig)
        return int(e.code or 0)
    try:
        a.run(a)
    except (RuntimeError, ValueError, NotImplementedError) as e:
        print(f"error: {e}", file=sys.stderr)
        if isinstance(e, NotImplementedError):
            return EXIT_CONFIG
        return classify_exception(e)
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
