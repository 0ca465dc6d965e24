"""Full-size C2 (the bench workload) against oracle fixtures
(tests/golden/make_c2_cg.py): the rank-50 pivoted-Cholesky pivot order,
bit-exact, and the PCG residual history of the targets column — including
the reference algorithm's failure to reach tol 1e-4 in 1000 iterations at
this noise level (σ = 1e-2)."""
import json
import os

import numpy as np
import pytest

import bench
import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c2_cg.json")))


@pytest.fixture(scope="module")
def c2():
    X, y, dY, grid = bench.build_problem()
    c = bench.CONFIG
    op = gk.DskiOperator(gk.KernelSpec(c["ell"], 1.0), grid, X, (c["noise"], c["noise"]))
    fac = gk.pivoted_cholesky(op, c["precond_rank"], kernel_part=True)
    b = gk.stacked_targets(y, dY, y.mean())
    return op, fac, b


def test_c2_pivot_order_bit_exact(c2):
    op, fac, b = c2
    assert [int(p) for p in fac.pivots] == FIX["pivots"]
    assert abs(fac.initial_trace - FIX["initial_trace"]) <= 1e-12 * FIX["initial_trace"]
    assert abs(fac.residual_trace - FIX["residual_trace"]) <= 1e-9 * FIX["initial_trace"]


def test_c2_pcg_history_matches_oracle(c2):
    op, fac, b = c2
    P = gk.Preconditioner.from_pivchol(op, fac)
    sol = gk.cg(op, b, bench.CONFIG["pcg_tol"], 1000, P)
    h, ref = np.asarray(sol.residual_history), np.asarray(FIX["residual_history"])
    assert sol.iterations == FIX["iterations"] and sol.converged == FIX["converged"]
    assert h.shape == ref.shape
    # The first 20 iterations agree to 1e-9 (measured); past that, roundoff in
    # this stagnating, ill-conditioned solve makes the two histories diverge
    # chaotically (the fused and separate-kernel GPU paths also differ by up to
    # 0.27 absolute), so the tail is held to its level: the final residual
    # within 25 % and the median |log ratio| over all 1001 entries below 0.1.
    assert np.max(np.abs(h[:20] - ref[:20]) / ref[:20]) <= 1e-8
    assert abs(h[-1] - ref[-1]) <= 0.25 * ref[-1], (h[-1], ref[-1])
    assert np.median(np.abs(np.log(h / ref))) <= 0.1
