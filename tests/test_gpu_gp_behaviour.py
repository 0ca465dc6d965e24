"""GpModel behaviour on the device, restating the reference's own GP tests
(proj/tests/test_gp.cpp) against this implementation's three backends: the
closed-form LML, exact/D-SKI/D-SKIP agreement, the exact LML gradient, the
fit optimiser, predictive means and gradients, and the exact / pivoted-
Cholesky / randomized variances (gp.cpp:143-547). Data: Franke samples
(testfns.cpp sampling, `sample_test_function`) and draws from a GP prior
through the oracle's dense assembly."""

import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu


def se(ell, s):
    return gk.KernelSpec(ell, s)


def franke(n, seed, grads=True):
    X, y, dY = gk.sample_test_function("franke", n, seed)
    return X, y, (dY if grads else None)


def points(n, d, lo, hi, seed):
    return np.random.default_rng(seed).uniform(lo, hi, (n, d))


def simulate_gp(ell, s, n, d, nv, ng, seed):
    """y, ∇y drawn from the SE prior (dense Cholesky) plus noise."""
    X = points(n, d, 0.0, 1.0, seed)
    K = O.assemble_dense(O.KernelSpec(ell, s), X) + 1e-10 * np.eye(n * (d + 1))
    f = np.linalg.cholesky(K) @ np.random.default_rng(seed + 1).standard_normal(n * (d + 1))
    rng = np.random.default_rng(seed + 2)
    y = f[:n] + nv * rng.standard_normal(n)
    dY = np.column_stack([f[(j + 1) * n:(j + 2) * n] + ng * rng.standard_normal(n) for j in range(d)])
    return X, y, dY


def test_lml_single_noisy_observation_closed_form():
    m = gk.GpModel(se(1.0, 1.0), np.zeros((1, 1)), np.zeros(1), None, noise=(1.0, 1.0), backend="exact")
    want = -0.5 * (np.log(2.0) + np.log(2.0 * np.pi))
    assert abs(m.log_marginal_likelihood() - want) <= 1e-12 * abs(want)


def test_lml_exact_and_dski_agree():
    X, y, dY = franke(100, 3)
    noise = (0.05, 0.05)
    a = gk.GpModel(se(0.4, 0.6), X, y, dY, noise=noise, backend="exact").log_marginal_likelihood()
    b = gk.GpModel(se(0.4, 0.6), X, y, dY, noise=noise, backend="dski", grid_ratio=0.15, tol=1e-8,
                   max_iterations=3000, slq_probes=30, slq_steps=80).log_marginal_likelihood()
    assert abs(a - b) <= 1e-2 * abs(a)


def test_lml_gradient_matches_finite_differences_on_simulated_data():
    X, y, dY = simulate_gp(0.5, 1.2, 40, 2, 0.1, 0.15, 11)
    m = gk.GpModel(se(0.45, 1.0), X, y, dY, noise=(0.1, 0.15), backend="exact")
    g = m.lml_gradient()
    p0 = np.log([0.45, 1.0, 0.1, 0.15])
    h = 1e-5
    for i in range(4):
        def at(delta):
            p = p0.copy()
            p[i] += delta
            m.set_hyperparameters(se(np.exp(p[0]), np.exp(p[1])), np.exp(p[2]), np.exp(p[3]))
            return m.log_marginal_likelihood()
        fd = (at(h) - at(-h)) / (2 * h)
        m.set_hyperparameters(se(0.45, 1.0), 0.1, 0.15)
        assert abs(g[i] - fd) <= 1e-4 * abs(fd), (i, g[i], fd)


def test_noise_gradient_of_the_complexity_term_is_positive():
    X, y, dY = franke(40, 5)

    def logdet_at(s1):
        return gk.GpModel(se(0.4, 1.0), X, y, dY, noise=(s1, 0.05), backend="exact").logdet()

    h = 1e-5
    assert (logdet_at(0.05 * np.exp(h)) - logdet_at(0.05 * np.exp(-h))) / (2 * h) > 0.0


def test_fit_zero_iterations_returns_hyperparameters_unchanged():
    X, y, dY = franke(25, 7)
    m = gk.GpModel(se(0.37, 0.9), X, y, dY, noise=(0.05, 0.05), backend="exact")
    res = m.fit(max_iterations=0)
    assert res.kernel.lengthscale == pytest.approx(0.37) and res.kernel.outputscale == pytest.approx(0.9)
    assert res.noise_value == pytest.approx(0.05)


def test_fit_does_not_decrease_the_likelihood_and_recovers_the_lengthscale():
    rec = []
    for seed in range(10):
        X, y, dY = simulate_gp(0.4, 1.0, 150, 2, 0.05, 0.05, 100 + seed)
        m = gk.GpModel(se(0.8, 0.7), X, y, dY, noise=(0.05, 0.05), backend="exact")  # misplaced start
        L0 = m.log_marginal_likelihood()
        res = m.fit(max_iterations=25, restarts=1)
        assert res.log_marginal >= L0 - 1e-9
        rec.append(res.kernel.lengthscale)
    rec.sort()
    assert abs(0.5 * (rec[4] + rec[5]) - 0.4) <= 0.25 * 0.4


def test_predict_mean_reproduces_training_values_at_vanishing_noise():
    X, y, dY = franke(20, 9)
    m = gk.GpModel(se(0.15, 0.8), X, y, dY, noise=(1e-5, 1e-5), backend="exact")
    assert np.max(np.abs(m.predict_mean(X) - y)) < 1e-6


@pytest.mark.parametrize("backend", ["exact", "dski"])
def test_predicted_gradients_match_finite_differences(backend):
    X, y, dY = franke(60, 15)
    kw = dict(grid_ratio=0.1, tol=1e-10, max_iterations=3000) if backend == "dski" else {}
    m = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=(0.05, 0.05), backend=backend, **kw)
    Xt = points(10, 2, 0.2, 0.8, 16)
    _, grads = m.predict_mean_grad(Xt)
    h = 1e-6
    for p in range(2):
        e = np.zeros(2)
        e[p] = h
        fd = (m.predict_mean(Xt + e) - m.predict_mean(Xt - e)) / (2 * h)
        assert np.all(np.abs(grads[:, p] - fd) <= 1e-5 * np.maximum(np.abs(fd), 1e-3)), (p, grads[:, p], fd)


def test_variance_far_field_is_the_prior_and_training_points_are_pinned():
    X, y, dY = franke(40, 17)
    m = gk.GpModel(se(0.08, 0.9), X, y, dY, noise=(0.01, 0.01), backend="exact")
    assert m.predict_variance_exact(np.array([[40.0, 40.0]]))[0] == pytest.approx(0.81, rel=1e-6)
    assert np.all(m.predict_variance_exact(X[:5]) <= 0.01 ** 2 + 1e-6)


def test_gradient_information_strictly_reduces_the_predictive_variance():
    X, y, dY = franke(50, 19)
    Xt = points(200, 2, 0.05, 0.95, 20)
    vg = gk.GpModel(se(0.35, 0.8), X, y, dY, noise=(0.05, 0.05), backend="exact").predict_variance_exact(Xt)
    vv = gk.GpModel(se(0.35, 0.8), X, y, None, noise=(0.05, 0.05), backend="exact").predict_variance_exact(Xt)
    assert np.all(vv - vg >= 1e-12)


def test_pivoted_cholesky_variance_exact_at_full_rank_biased_up_at_rank_100():
    X, y, dY = franke(120, 21)
    Xt = points(50, 2, 0.1, 0.9, 22)
    full = gk.GpModel(se(0.5, 1.0), X, y, dY, noise=(0.1, 0.1), backend="exact", precond_rank=360)
    ve = full.predict_variance_exact(Xt[:10])
    vp = full.predict_variance_pivchol(Xt[:10])
    # doctest::Approx(v).epsilon(1e-8): |a − b| < 1e-8·(1 + max(|a|, |b|))
    assert np.all(np.abs(vp - ve) <= 1e-8 * (1.0 + np.maximum(np.abs(vp), np.abs(ve))))
    t100 = gk.GpModel(se(0.5, 1.0), X, y, dY, noise=(0.1, 0.1), backend="exact", precond_rank=100)
    assert np.all(t100.predict_variance_pivchol(Xt) - t100.predict_variance_exact(Xt) >= -1e-8)


@pytest.mark.parametrize("backend", ["exact", "dski"])
def test_randomized_variance_with_zero_probes_is_the_pivoted_cholesky_estimate(backend):
    X, y, dY = franke(80, 23)
    kw = dict(grid_ratio=0.1, tol=1e-10, max_iterations=3000) if backend == "dski" else {}
    m = gk.GpModel(se(0.4, 0.9), X, y, dY, noise=(0.1, 0.1), backend=backend, precond_rank=60, **kw)
    Xt = points(20, 2, 0.1, 0.9, 24)
    pv = m.predict_variance_pivchol(Xt)
    assert np.all(np.abs(m.predict_variance_randomized(Xt, 0, 1) - pv) <= 1e-12 * np.abs(pv))


def test_randomized_variance_is_unbiased_around_the_exact_variance():
    X, y, dY = franke(150, 25)
    m = gk.GpModel(se(0.4, 0.9), X, y, dY, noise=(0.1, 0.1), backend="exact", precond_rank=80)
    Xt = points(40, 2, 0.1, 0.9, 26)
    S = np.array([m.predict_variance_randomized(Xt, 1, 1000 + p) for p in range(100)])
    exact = m.predict_variance_exact(Xt)
    se3 = 3.0 * S.std(axis=0, ddof=1) / np.sqrt(100)
    assert np.sum(np.abs(S.mean(axis=0) - exact) <= se3 + 1e-12) >= int(0.85 * 40)


def test_monotone_information_adding_a_point_never_increases_exact_variance():
    X, y, dY = franke(21, 29)
    Xt = points(50, 2, 0.05, 0.95, 30)
    small = gk.GpModel(se(0.4, 0.8), X[:20], y[:20], dY[:20], noise=(0.05, 0.05), backend="exact")
    big = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=(0.05, 0.05), backend="exact")
    assert np.all(big.predict_variance_exact(Xt) <= small.predict_variance_exact(Xt) + 1e-10)


def test_backends_agree_within_tolerances():
    X, y, dY = franke(120, 31)
    Xt = points(60, 2, 0.1, 0.9, 32)
    noise = (0.08, 0.08)
    m0 = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=noise, backend="exact").predict_mean(Xt)
    md = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=noise, backend="dski", grid_ratio=0.125, tol=1e-8,
                    max_iterations=3000).predict_mean(Xt)
    mp = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=noise, backend="dskip", dskip_rank=150, tol=1e-8,
                    max_iterations=3000).predict_mean(Xt)
    scale = np.sqrt(np.mean(m0 ** 2))
    assert np.sqrt(np.mean((md - m0) ** 2)) / scale < 5e-3
    assert np.sqrt(np.mean((mp - m0) ** 2)) / scale < 2e-2


def test_predict_mean_exact_and_dski_agree_on_franke():
    X, y, dY = franke(400, 13)
    Xt = points(300, 2, 0.08, 0.92, 14)
    noise = (0.05, 0.05)
    me = gk.GpModel(se(0.3, 0.7), X, y, dY, noise=noise, backend="exact").predict_mean(Xt)
    md = gk.GpModel(se(0.3, 0.7), X, y, dY, noise=noise, backend="dski", grid_ratio=0.125, tol=1e-8,
                    max_iterations=3000).predict_mean(Xt)
    assert np.sqrt(np.mean((me - md) ** 2)) / np.sqrt(np.mean(me ** 2)) <= 5e-3


def test_dski_rejects_test_points_outside_the_grid_interior():
    X, y, dY = franke(50, 33)
    m = gk.GpModel(se(0.4, 0.8), X, y, dY, noise=(0.05, 0.05), backend="dski")
    m.predict_mean(X[:3])
    with pytest.raises(gk.OutOfGridError):
        m.predict_mean(np.array([[7.0, 7.0]]))
