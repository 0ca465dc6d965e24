"""Concurrent host threads on one operator (SURVEY §8(b) Threading: the
reference calls op.mvm concurrently from OpenMP threads in slq_logdet and
trace_estimate, linalg.cpp:222,264). Every C-ABI call on a handle is
serialised by the handle's mutex and uses handle-owned scratch; results must
equal the single-threaded ones exactly."""
import threading

import numpy as np
import pytest

import paper_1810_12283_b200 as gk

pytestmark = pytest.mark.gpu


def test_concurrent_mvm_solve_and_slq_on_one_operator():
    X, y, dY = gk.make_dataset(1, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, 60)
    op = gk.DskiOperator(gk.KernelSpec(0.15, 1.0), grid, X, (0.1, 0.1))
    N = op.size()
    rng = np.random.default_rng(7)
    Vs = [rng.standard_normal((N, c)) for c in (1, 4, 7, 32)]
    want_mvm = [op.mvm(V) for V in Vs]
    P = gk.Preconditioner.from_pivchol(op, gk.pivoted_cholesky(op, 20, kernel_part=True))
    b = gk.stacked_targets(y, dY, y.mean())
    want_x = gk.cg(op, b, 1e-8, 2000, P).x
    want_ld = gk.slq_logdet(op, 8, 25, 0, 0.005).logdet
    errors, results = [], {}

    def worker(t):
        try:
            for rep in range(3):
                for i, V in enumerate(Vs):
                    out = op.mvm(V)
                    if not np.array_equal(out, want_mvm[i]):
                        errors.append(("mvm", t, rep, i, float(np.abs(out - want_mvm[i]).max())))
            results[("cg", t)] = gk.cg(op, b, 1e-8, 2000, P).x
            results[("slq", t)] = gk.slq_logdet(op, 8, 25, 0, 0.005).logdet
        except Exception as e:  # surfaced below
            errors.append(("exception", t, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:5]
    for t in range(4):
        assert np.array_equal(results[("cg", t)], want_x)
        assert results[("slq", t)] == want_ld


def test_dev_entry_points_ordered_against_host_calls():
    """device-pointer calls on a caller's side stream (stage_dev /
    mvm_dev, asynchronous) interleaved, without any host synchronisation, with
    host-API calls on the same handle (mvm, diagonal, cg) that reuse the
    handle's scratch, plans and grid-barrier counter. Every call waits on the
    handle's last-use event, so all results equal the serial ones."""
    import torch
    X, y, dY = gk.make_dataset(2, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, 100)
    op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
    N = op.size()
    rng = np.random.default_rng(3)
    B32 = rng.standard_normal((N, 32))
    want32 = op.mvm(B32)
    want_diag = op.diagonal()
    b = gk.stacked_targets(y, dY, y.mean())
    want_x = gk.cg(op, b, 1e-3, 40).x
    side = torch.cuda.Stream()
    Vext = torch.from_numpy(np.ascontiguousarray(B32.T)).cuda()
    Vi = torch.empty(N * 32, dtype=torch.float64, device="cuda")
    outs = [torch.empty_like(Vi) for _ in range(6)]
    Oext = [torch.empty_like(Vext) for _ in range(6)]
    torch.cuda.synchronize()
    s = side.cuda_stream
    op.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), 32, stream=s)
    diags, xs = [], []
    for k in range(6):
        op.stage_dev(3, Vi.data_ptr(), outs[k].data_ptr(), 32, stream=s)  # async on the side stream
        op.from_internal_dev(outs[k].data_ptr(), Oext[k].data_ptr(), 32, stream=s)
        if k % 2 == 0:
            diags.append(op.diagonal())  # host API on the handle's own stream
        else:
            xs.append(gk.cg(op, b, 1e-3, 40).x)
        if k == 5:  # the external-layout device entry point as well
            op.mvm_dev(Vext.data_ptr(), Oext[k].data_ptr(), 32, stream=s)
    side.synchronize()
    for k in range(6):
        got = Oext[k].cpu().numpy().T
        assert np.linalg.norm(got - want32) <= 1e-13 * np.linalg.norm(want32), k
    for d in diags:
        assert np.array_equal(d, want_diag)
    for x in xs:
        assert np.array_equal(x, want_x)


@pytest.mark.gpu
@pytest.mark.parametrize("nrhs", [1, 7, 32, 45])
def test_host_mvm_pageable_staging_matches_pinned_and_direct(nrhs):
    """gk_op_mvm from pageable buffers (pinned staging by the host copy pool,
    chunked, with leading dimensions larger than N) returns exactly what the
    driver's direct pageable copies and pinned buffers return."""
    import torch
    X, y, dY = gk.make_dataset(2, 0)
    X = X[:3000]
    grid = gk.Grid.cover(X, 1e-3, 3, 60)
    op = gk.DskiOperator(gk.KernelSpec(0.2, 1.0), grid, X, (1e-2, 1e-2))
    N = op.size()
    ld = N + 5
    rng = np.random.default_rng(nrhs)
    Vp = np.asfortranarray(rng.standard_normal((ld, nrhs)))
    outs = {}
    for stage in (0, 1):
        prev = gk.set_tuning("e2e_stage", stage)
        try:
            O = np.zeros((ld, nrhs), order="F")
            gk._check(gk._lib.gk_op_mvm(op.handle, gk._p(Vp), ld, gk._p(O), ld, nrhs))
        finally:
            gk.set_tuning("e2e_stage", prev)
        outs[stage] = O[:N].copy()
        assert not O[N:].any()  # rows past N untouched
    Vpin = torch.from_numpy(Vp.T.copy()).pin_memory()  # (nrhs, ld) row-major = column-major (ld, nrhs)
    Opin = torch.zeros_like(Vpin).pin_memory()
    gk._check(gk._lib.gk_op_mvm(op.handle, ctypes_ptr(Vpin), ld, ctypes_ptr(Opin), ld, nrhs))
    pinned = Opin.numpy().T[:N]
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], pinned)


def ctypes_ptr(t):
    import ctypes
    return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))
