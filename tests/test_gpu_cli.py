"""The gradkrig tools on the device, against the oracle:
GpModel.fit reproduces the reference optimiser (gp.cpp:294-404) step for step;
`fit` → model JSON → `predict` gives the oracle GpModel's predictive mean,
gradient and variance (cmd_fit.cpp / cmd_predict.cpp); `precond-study`
iteration counts match the oracle's CG/PCG (cmd_precond_study.cpp:29-98);
`benchmark-mvm` times the operator cmd_benchmark_mvm.cpp:55-80 builds."""
import csv
import json

import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk
from paper_1810_12283_b200 import cli
from paper_1810_12283_b200 import io as gio

pytestmark = pytest.mark.gpu

N_PTS = 300
NOISE = 0.05


def _franke():
    X, y, dY = O.sample_test_function("franke", N_PTS, 0, (NOISE, NOISE))
    return X, y, dY


WC = dict(noise=(1.0, 1.0), backend="dski", grid_ratio=0.2, max_grid_nodes=40, tol=1e-10, max_iterations=3000,
          precond_rank=100, slq_probes=8, slq_steps=25, seed=0)


def test_fit_matches_oracle_optimizer():
    """Same trajectory as the oracle's GpModel::fit: every accept/reject
    decision, restart jitter, iteration count and final θ. Well-conditioned
    (σ = 1, rank-100 preconditioner, noise held fixed — FitOptions
    optimize_noise = false): there every 1e-2-tolerance probe solve of the
    stochastic gradient stops at the same PCG iteration on both sides, so the
    gradients agree to ≤1e-8 (tests/test_gpu_gradient.py); in ill-conditioned
    regimes probe iteration counts move under roundoff and the trajectories
    separate, as two runs of the reference on different hardware would."""
    X, y, dY = _franke()
    ref = O.GpModel(O.KernelSpec(0.3, 1.0), X, y, dY, **WC)
    gm = gk.GpModel(gk.KernelSpec(0.3, 1.0), X, y, dY, **WC)
    want = ref.fit(max_iterations=3, restarts=2, optimize_noise=False, seed=0)
    got = gm.fit(max_iterations=3, restarts=2, optimize_noise=False, seed=0)
    assert [(r.succeeded, r.iterations) for r in got.restarts] == [(s, i) for s, i, _ in want["restarts"]]
    assert sum(r.accepted_steps for r in got.restarts) >= 2
    for r, (_, _, L) in zip(got.restarts, want["restarts"]):
        assert abs(r.log_marginal - L) <= 1e-8 * abs(L)
    assert abs(got.kernel.lengthscale - want["ell"]) <= 1e-8 * want["ell"]
    assert abs(got.kernel.outputscale - want["s"]) <= 1e-8 * want["s"]
    # noise is not optimised, but restart jitter moves it (gp.cpp:328-331)
    assert abs(got.noise_value - want["noise_value"]) <= 1e-14 * want["noise_value"]
    assert abs(got.noise_gradient - want["noise_gradient"]) <= 1e-14 * want["noise_gradient"]
    assert abs(got.log_marginal - want["log_marginal"]) <= 1e-8 * abs(want["log_marginal"])
    assert got.log_marginal > gk.GpModel(gk.KernelSpec(0.3, 1.0), X, y, dY, **WC).log_marginal_likelihood()


def test_cli_fit_then_predict_matches_oracle(tmp_path):
    X, y, dY = _franke()
    data = str(tmp_path / "train.csv")
    gio.write_dataset_csv(data, gio.Dataset(X, y, dY))
    model = str(tmp_path / "model.json")
    # --probes 16: slq 16 probes, gradient probes max(4, 16/2) = 8 (common.cpp:49-50)
    # one optimiser iteration from σ = 1 (one well-conditioned gradient, see
    # test_fit_matches_oracle_optimizer), tol 1e-10
    rc = cli.main(["fit", "--data", data, "--model", model, "--backend", "dski", "--ell", "0.3", "--noise", "1",
                   "--noise-grad", "1", "--grid-size", "40", "--rank", "100", "--probes", "16", "--tol", "1e-10",
                   "--maxit", "3000", "--iters", "1", "--restarts", "1"])
    assert rc == 0
    j = json.load(open(model))
    assert j["backend"] == "dski" and j["data"] == {"path": data, "with_gradients": True}
    assert j["solver"]["precond_rank"] == 100 and j["solver"]["slq_probes"] == 16
    ref = O.GpModel(O.KernelSpec(0.3, 1.0), X, y, dY, noise=(1.0, 1.0), backend="dski", grid_ratio=0.2,
                    max_grid_nodes=40, dskip_rank=100, tol=1e-10, max_iterations=3000, precond_rank=100,
                    slq_probes=16, slq_steps=50, seed=0)
    want = ref.fit(max_iterations=1, restarts=1, seed=0)
    assert want["noise_value"] != 1.0  # the step moved every parameter
    for key, w in ((j["kernel"]["lengthscale"], want["ell"]), (j["kernel"]["outputscale"], want["s"]),
                   (j["noise"]["value"], want["noise_value"]), (j["noise"]["gradient"], want["noise_gradient"])):
        assert abs(key - w) <= 1e-8 * w
    assert j["mean"]["value"] == float(np.mean(y)) or abs(j["mean"]["value"] - np.mean(y)) <= 1e-15

    test = str(tmp_path / "test.csv")
    Xt = O.sample_test_function("franke", 7, 9)[0]
    gio.write_csv(test, ["x1", "x2"], Xt.tolist())
    out = str(tmp_path / "pred.csv")
    assert cli.main(["predict", "--model", model, "--test", test, "--out", out, "--gradients"]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["x1", "x2", "mean", "variance", "dmean1", "dmean2"]
    P = np.array(rows[1:], dtype=float)
    assert np.array_equal(P[:, :2], Xt)
    ref.set_hyperparameters(j["kernel"]["lengthscale"], j["kernel"]["outputscale"], j["noise"]["value"],
                            j["noise"]["gradient"])
    mu, g = ref.predict_mean_grad(Xt)
    assert np.max(np.abs(P[:, 2] - mu)) <= 1e-8 * np.max(np.abs(mu))
    assert np.max(np.abs(P[:, 4:] - g)) <= 1e-8 * np.max(np.abs(g))
    var = np.array([ref.predict_variance_pivchol(x) for x in Xt])
    assert np.max(np.abs(P[:, 3] - var)) <= 1e-8 * np.max(np.abs(var))


def test_cli_precond_study_matches_oracle(tmp_path):
    out = str(tmp_path / "study.csv")
    assert cli.main(["precond-study", "--function", "franke", "--n", "300", "--sweep-points", "2", "--rank", "30",
                     "--maxit", "400", "--out", out]) == 0
    rows = np.array(list(csv.reader(open(out)))[1:], dtype=float)
    assert rows.shape == (4, 6)
    X, y, dY = O.sample_test_function("franke", 300, 0)
    ys = np.sqrt(np.mean((y - y.mean()) ** 2))
    y, dY = (y - y.mean()) / ys, dY / ys
    b = O.stacked_targets(y, dY, y.mean())
    for r in rows:
        ell, sigma = r[0], r[1]
        op = O.DskiOperator(O.KernelSpec(ell, 1.0), O.Grid.cover(X, 0.25 * ell, 3, 64), X, (sigma, sigma))
        plain = O.cg(op, b, 1e-4, 400)
        nd = op.noise_diagonal()
        f = O.pivoted_cholesky(op, 30, noise_diag=nd)
        pre = O.cg(op, b, 1e-4, 400, O.Preconditioner(f.L, nd))
        # CG counts at hundreds of iterations move under roundoff (test_gpu_solvers.oracle_iteration_band)
        for its, conv, ref in ((r[2], r[3], plain), (r[4], r[5], pre)):
            assert abs(its - ref.iterations) <= max(2, 0.02 * ref.iterations), (ell, sigma, its, ref.iterations)
            if abs(ref.iterations - 400) > 10:
                assert bool(conv) == ref.converged


@pytest.mark.parametrize("backend", ["dski", "dskip", "exact"])
def test_cli_benchmark_mvm(tmp_path, backend):
    out = str(tmp_path / "bench.csv")
    assert cli.main(["benchmark-mvm", "--backend", backend, "--sizes", "500,1000", "--reps", "3", "--rank", "40",
                     "--out", out]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["n", "N", "seconds"]
    assert [(int(float(r[0])), int(float(r[1]))) for r in rows[1:]] == [(500, 1500), (1000, 3000)]
    assert all(float(r[2]) > 0 for r in rows[1:])


def test_benchmark_operator_is_the_reference_one():
    """cmd_benchmark_mvm.cpp:55-63: SE(0.4, 1) D-SKI on the fixed [−0.25, 1.25]
    grid with noise 0.1 — one MVM against the oracle's ≤1e-12."""
    X = cli.bench_points(800, 2, 0)
    op = cli.bench_operator("dski", X, 32, 100, 0)
    ref = O.DskiOperator(O.KernelSpec(0.4, 1.0), O.Grid([32, 32], [-0.25, -0.25], [1.5 / 31] * 2), X, (0.1, 0.1))
    v = gk.gaussian_vector(op.size(), 7)
    want = ref.mvm(v)
    assert np.linalg.norm(op.mvm(v) - want) <= 1e-12 * np.linalg.norm(want)


def test_cli_spline_kernel_fit_and_predict(tmp_path):
    """--kernel spline on the dski backend (SplineConstants::for_domain
    calibration, K_UU by circulant embedding): fit → model JSON with the
    spline constants → predict; the predictive mean matches the oracle
    D-SKI operator's B K_UU Bᵀ α path (gp.cpp:480-495) through its own K∇."""
    X, y, dY = O.sample_test_function("franke", 150, 3, (0.05, 0.05))
    data = str(tmp_path / "train.csv")
    gio.write_dataset_csv(data, gio.Dataset(X, y, dY))
    model = str(tmp_path / "model.json")
    assert cli.main(["fit", "--data", data, "--model", model, "--kernel", "spline", "--backend", "dski", "--noise", "0.3",
                     "--noise-grad", "0.3", "--grid-size", "40", "--rank", "60", "--tol", "1e-8", "--maxit", "3000",
                     "--probes", "8", "--iters", "1", "--restarts", "1"]) == 0
    j = json.load(open(model))
    assert j["kernel"]["family"] == "spline" and {"spline_a", "spline_b", "spline_even"} <= set(j["kernel"])
    assert j["kernel"]["spline_even"] is True  # d = 2
    test = str(tmp_path / "test.csv")
    gio.write_csv(test, ["x1", "x2"], X[:5].tolist())
    out = str(tmp_path / "pred.csv")
    assert cli.main(["predict", "--model", model, "--test", test, "--out", out]) == 0
    P = np.array(list(csv.reader(open(out)))[1:], dtype=float)
    assert P.shape == (5, 4) and np.all(np.isfinite(P))
    assert np.max(np.abs(P[:, 2] - y[:5])) < 0.5  # the mean interpolates its own (noisy) training values


def test_cli_default_exact_backend(tmp_path):
    """The tools' default backend "exact" (dense K∇ + Cholesky, gp.cpp:71-85):
    fit → JSON → predict with the exact variance equals numpy on the oracle's
    dense assembly at the fitted hyperparameters."""
    X, y, dY = O.sample_test_function("franke", 100, 8, (0.05, 0.05))
    data = str(tmp_path / "train.csv")
    gio.write_dataset_csv(data, gio.Dataset(X, y, dY))
    model = str(tmp_path / "model.json")
    assert cli.main(["fit", "--data", data, "--model", model, "--ell", "0.3", "--noise", "0.2", "--noise-grad", "0.2",
                     "--iters", "2", "--restarts", "1", "--probes", "8"]) == 0
    j = json.load(open(model))
    assert j["backend"] == "exact"
    test = str(tmp_path / "test.csv")
    Xt = O.sample_test_function("franke", 5, 21)[0]
    gio.write_csv(test, ["x1", "x2"], Xt.tolist())
    out = str(tmp_path / "pred.csv")
    assert cli.main(["predict", "--model", model, "--test", test, "--out", out, "--variance", "exact"]) == 0
    P = np.array(list(csv.reader(open(out)))[1:], dtype=float)
    ko = O.KernelSpec(j["kernel"]["lengthscale"], j["kernel"]["outputscale"])
    s1, s2 = j["noise"]["value"], j["noise"]["gradient"]
    K = O.assemble_dense(ko, X) + np.diag(np.concatenate([np.full(100, s1 ** 2), np.full(200, s2 ** 2)]))
    t = O.stacked_targets(y, dY, y.mean())
    Q = O.assemble_dense(ko, X, Xt)[:300, :5]
    mu = y.mean() + Q.T @ np.linalg.solve(K, t)
    var = j["kernel"]["outputscale"] ** 2 - np.einsum("ij,ij->j", Q, np.linalg.solve(K, Q))
    assert np.max(np.abs(P[:, 2] - mu)) <= 1e-9 * np.max(np.abs(mu))
    assert np.max(np.abs(P[:, 3] - var)) <= 1e-9


def test_cli_fit_round_trips_as_a_no_op(tmp_path, capsys):
    """test_cli.cpp:70-96: fit, then refit from the written parameters with
    zero iterations — the same hyperparameters (1e-12); the report has a
    finite log-marginal."""
    X, y, dY = O.sample_test_function("franke", 40, 2, (0.02, 0.02))
    data = str(tmp_path / "toy.csv")
    gio.write_dataset_csv(data, gio.Dataset(X, y, dY))
    m1 = str(tmp_path / "m.json")
    assert cli.main(["fit", "--data", data, "--model", m1, "--iters", "8", "--restarts", "1", "--seed", "1"]) == 0
    report = capsys.readouterr().out
    assert "log-marginal=" in report and "nan" not in report
    j = json.load(open(m1))
    m2 = str(tmp_path / "m2.json")
    assert cli.main(["fit", "--data", data, "--model", m2, "--iters", "0", "--ell", repr(j["kernel"]["lengthscale"]),
                     "--outputscale", repr(j["kernel"]["outputscale"]), "--noise", repr(j["noise"]["value"]),
                     "--noise-grad", repr(j["noise"]["gradient"]), "--seed", "1"]) == 0
    k2 = json.load(open(m2))
    for a, b in ((k2["kernel"]["lengthscale"], j["kernel"]["lengthscale"]),
                 (k2["kernel"]["outputscale"], j["kernel"]["outputscale"]), (k2["noise"]["value"], j["noise"]["value"])):
        assert abs(a - b) <= 1e-12 * abs(b)


def test_cli_predict_pins_training_points_and_is_deterministic(tmp_path):
    """test_cli.cpp:98-141: at low noise the mean pins the training values,
    the pivoted-Cholesky variance never falls below the exact one, and the
    randomized variance is reproducible under a fixed seed."""
    X, y, dY = O.sample_test_function("franke", 60, 7)
    train = str(tmp_path / "train.csv")
    gio.write_dataset_csv(train, gio.Dataset(X, y, dY))
    model = str(tmp_path / "m.json")
    assert cli.main(["fit", "--data", train, "--model", model, "--iters", "0", "--ell", "0.18", "--outputscale", "0.5",
                     "--noise", "1e-3", "--noise-grad", "1e-3", "--rank", "180"]) == 0

    def run(var, name, extra=()):
        out = str(tmp_path / name)
        assert cli.main(["predict", "--model", model, "--test", train, "--out", out, "--variance", var, *extra]) == 0
        return out, np.array(list(csv.reader(open(out)))[1:], dtype=float)

    _, ex = run("exact", "exact.csv")
    _, pc = run("pivchol", "pivchol.csv")
    assert np.all(np.abs(ex[:, 2] - y) < 5e-3)
    # rank 180 = N: M⁻¹ = K⁻¹ up to rounding; at σ = 1e-3 both variances are
    # s² − qᵀ(·)q ≈ 1e-7 from s² = 0.25 with cond(K) ~ 1e11, so each carries
    # ~1e-8 of rounding — the reference's −1e-8 margin sits at that floor
    assert np.all(pc[:, 3] - ex[:, 3] >= -5e-8)
    r1, _ = run("randomized", "r1.csv", ("--probes", "16", "--seed", "9"))
    r2, _ = run("randomized", "r2.csv", ("--probes", "16", "--seed", "9"))
    assert open(r1).read() == open(r2).read()


def test_cli_precond_study_csv_and_pcg_never_behind_cg(tmp_path):
    """test_cli.cpp:194-211."""
    out = str(tmp_path / "study.csv")
    assert cli.main(["precond-study", "--function", "franke", "--n", "300", "--sweep-points", "3", "--rank", "60",
                     "--out", out, "--seed", "4", "--grid-size", "32"]) == 0
    lines = open(out).read().splitlines()
    assert lines[0] == "ell,sigma,cg_iters,cg_converged,pcg_iters,pcg_converged"
    rows = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    assert rows.shape == (9, 6) and np.all(rows[:, 4] <= rows[:, 2] + 2)


def test_cli_benchmark_mvm_timings_grow_with_n(tmp_path):
    """test_cli.cpp:213-228 (host-buffer calls through the C-ABI)."""
    out = str(tmp_path / "bench.csv")
    assert cli.main(["benchmark-mvm", "--backend", "dski", "--sizes", "500,2000,8000", "--reps", "5", "--out", out]) == 0
    secs = [float(ln.split(",")[2]) for ln in open(out).read().splitlines()[1:]]
    assert len(secs) == 3 and secs[2] > secs[0]
