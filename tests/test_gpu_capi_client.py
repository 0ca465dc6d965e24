"""The C-ABI driven from plain C (tests/capi_client.c, compiled by
__graft_entry__.build_capi_client against include/gk_capi.h only): the
GpModel pipeline a reference-side binding runs matches the
oracle GpModel (gp.cpp:117-187, 471-495) on the same data — MVM ≤1e-12,
pivots bit-exact, α to the solver tolerance, LML/log-det ≤1e-8, predictive
mean and gradient ≤1e-8 — and an out-of-range row is GK_ERR_RANGE
(std::out_of_range, dski.cpp:293)."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _read(path):
    out = {}
    raw = open(path, "rb").read()
    pos = 0
    while pos < len(raw):
        tag = raw[pos:pos + 8].rstrip(b"\0").decode()
        n = int(np.frombuffer(raw, np.int64, 1, pos + 8)[0])
        out[tag] = np.frombuffer(raw, np.float64, n, pos + 16).copy()
        pos += 16 + 8 * n
    return out


def test_capi_client_compiles_against_header_only():
    """CPU: the header is valid C99 and the client links against every
    symbol it uses (no GPU needed to build)."""
    import __graft_entry__ as g
    exe = g.build_capi_client()
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
def test_capi_client_matches_oracle_gp_model(tmp_path):
    import __graft_entry__ as g
    exe = g.build_capi_client() if not os.path.exists(os.path.join(ROOT, "tests", "_bin", "capi_client")) \
        else os.path.join(ROOT, "tests", "_bin", "capi_client")
    out = tmp_path / "out.bin"
    r = subprocess.run([exe, str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    res = _read(out)
    n, d, its, rank = (int(v) for v in res["meta"])

    Xf, yf, dYf = O.make_dataset(1, 0)
    X, y, dY = Xf[:n], yf[:n], dYf[:n]
    ker = O.KernelSpec(0.15, 1.0)
    grid = O.Grid.cover(X, 1e-3, 3, 40)
    op = O.DskiOperator(ker, grid, X, (0.3, 0.3))
    t = O.stacked_targets(y, dY, y.mean())
    want = op.mvm(t)
    assert np.linalg.norm(res["Kt"] - want) <= 1e-12 * np.linalg.norm(want)

    # the oracle GpModel on the same grid (target spacing grid_ratio·ℓ = 1e-3, capped at 40 nodes)
    gm = O.GpModel(ker, X, y, dY, noise=(0.3, 0.3), backend="dski", grid_ratio=1e-3 / 0.15, max_grid_nodes=40,
                   tol=1e-8, max_iterations=2000, precond_rank=60, slq_probes=8, slq_steps=25, seed=0)
    assert [int(p) for p in res["pivots"]] == [int(p) for p in gm.pivots(60)]
    a_ref, its_ref = gm.alpha()
    assert abs(its - its_ref) <= 1, (its, its_ref)
    assert np.linalg.norm(res["alpha"] - a_ref) <= 1e-6 * np.linalg.norm(a_ref)
    lml_ref = gm.log_marginal_likelihood()
    lml, fit, logdet = res["lml"]
    assert abs(logdet - lml_ref["logdet"]) <= 1e-8 * abs(lml_ref["logdet"])
    assert abs(lml - lml_ref["lml"]) <= 1e-8 * abs(lml_ref["lml"])
    Xt = np.column_stack([X[3:53:10, j] for j in range(d)])
    mu_ref, g_ref = gm.predict_mean_grad(Xt)
    assert np.max(np.abs(res["mu"] - mu_ref)) <= 1e-8 * np.max(np.abs(mu_ref))
    assert np.max(np.abs(res["grad"].reshape(d, -1).T - g_ref)) <= 1e-8 * np.max(np.abs(g_ref))
    assert int(res["rowerr"][0]) == 2  # GK_ERR_RANGE
