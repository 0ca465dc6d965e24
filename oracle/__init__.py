"""CPU oracle for the gradkrig hot path — TEST INFRASTRUCTURE ONLY.

A ctypes view of ``oracle/build/libgk_oracle.so``, the dependency-free C++
restatement of the reference (arXiv 1810.12283 "gradkrig") hot path. Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package, and only
as the checker / CPU baseline — never as the product path.

Layout conventions follow the reference: X is n×d (passed column-major, i.e.
``np.asfortranarray``), vectors are derivative-type-major ``[f; ∂1; …; ∂d]``
(reference kernels.hpp:94-97), matrices column-major.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libgk_oracle.so")

_d = C.c_double
_dp = C.POINTER(C.c_double)
_i64 = C.c_longlong
_i64p = C.POINTER(C.c_longlong)
_ip = C.POINTER(C.c_int)
_u64 = C.c_ulonglong
_vp = C.c_void_p

SE, SPLINE = 0, 1

ERRORS = {1: ValueError, 2: IndexError, 3: "OutOfGrid", 4: RuntimeError, 5: RuntimeError,
          6: OverflowError, 9: RuntimeError}


class OracleOutOfGridError(RuntimeError):
    def __init__(self, msg, point):
        super().__init__(msg)
        self.point = point


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++, no external deps)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_last_error_point": (_i64, []),
            "orc_mix_seed": (_u64, [_u64, _u64]),
            "orc_rademacher": (None, [_i64, _u64, _u64, _dp]),
            "orc_gaussian": (None, [_i64, _u64, _u64, _dp]),
            "orc_mt19937_64_nth": (_u64, [_u64, _i64]),
            "orc_quintic_weights": (C.c_int, [_d, _dp, _dp]),
            "orc_cubic_weights": (C.c_int, [_d, _dp, _dp]),
            "orc_grid_cover": (C.c_int, [_dp, _i64, C.c_int, _d, C.c_int, C.c_int, _ip, _dp, _dp]),
            "orc_kernel_eval": (C.c_int, [C.c_int, _d, _d, _d, _d, C.c_int, _dp, _dp, C.c_int,
                                          _dp, _dp, _dp, _dp]),
            "orc_assemble_dense": (C.c_int, [C.c_int, _d, _d, _d, _d, C.c_int, _dp, _i64, _dp,
                                             _i64, C.c_int, C.c_int, _i64, _dp]),
            "orc_interp_dense": (C.c_int, [_ip, _dp, _dp, C.c_int, _dp, _i64, C.c_int, _dp]),
            "orc_point_stencil": (C.c_int, [_ip, _dp, _dp, C.c_int, _dp, C.c_int, _i64p, _dp, _dp]),
            "orc_dense_create": (_vp, [_dp, _i64]),
            "orc_dski_create": (_vp, [C.c_int, _d, _d, _d, _d, C.c_int, _ip, _dp, _dp, C.c_int,
                                      _dp, _i64, _d, _d, C.c_int, C.c_int]),
            "orc_dskip_create": (_vp, [C.c_int, _d, _d, _dp, _i64, C.c_int, _d, _d, _i64, _d,
                                       C.c_int, _u64, C.c_int, C.c_int, C.c_int]),
            "orc_dskip_factor_count": (C.c_int, [_vp]),
            "orc_dskip_factor_rank": (_i64, [_vp, C.c_int]),
            "orc_dskip_factor_get": (None, [_vp, C.c_int, _dp, _dp, _dp]),
            "orc_dskip_dlogell_apply": (C.c_int, [_vp, _dp, _dp]),
            "orc_factor_create": (_vp, [C.c_int, _d, _d, _dp, _i64, C.c_int, C.c_int, _d,
                                        C.c_int, C.c_int]),
            "orc_op_free": (None, [_vp]),
            "orc_op_size": (_i64, [_vp]),
            "orc_op_mvm": (C.c_int, [_vp, _dp, _dp]),
            "orc_op_mvm_batch": (C.c_int, [_vp, _dp, _dp, C.c_int]),
            "orc_op_diagonal": (C.c_int, [_vp, _dp]),
            "orc_op_row": (C.c_int, [_vp, _i64, _dp]),
            "orc_dski_transpose_apply": (C.c_int, [_vp, _dp, _dp]),
            "orc_dski_apply": (C.c_int, [_vp, _dp, _dp]),
            "orc_dski_grid_mvm": (C.c_int, [_vp, _dp, _dp]),
            "orc_dski_min_embedding_eigenvalue": (_d, [_vp]),
            "orc_dski_grid_size": (_i64, [_vp]),
            "orc_kuu_create": (_vp, [C.c_int, _d, _d, _d, _d, C.c_int, C.c_int, _ip, _dp, _dp,
                                     C.c_int]),
            "orc_kuu_free": (None, [_vp]),
            "orc_kuu_mvm": (C.c_int, [_vp, _dp, _dp]),
            "orc_kuu_min_eig": (_d, [_vp]),
            "orc_precond_create": (_vp, [_dp, _i64, _i64, _dp]),
            "orc_precond_free": (None, [_vp]),
            "orc_precond_apply": (None, [_vp, _dp, _dp]),
            "orc_precond_quadratic": (_d, [_vp, _dp]),
            "orc_precond_q1": (None, [_vp, _dp]),
            "orc_cg": (C.c_int, [_vp, _dp, _d, C.c_int, _vp, _dp, _ip, _ip, _dp, _ip]),
            "orc_pivchol": (C.c_int, [_vp, _dp, _dp, _i64, _d, _dp, _i64p, _i64p, _dp]),
            "orc_slq": (C.c_int, [_vp, C.c_int, C.c_int, _u64, _d, _dp, _ip, _dp]),
            "orc_trace_estimate": (C.c_int, [_vp, _vp, C.c_int, _u64, _d, C.c_int, _vp, _dp]),
            "orc_lanczos": (C.c_int, [_vp, _i64, _u64, _dp, _u64, _dp, _dp, _dp, _i64p, _ip]),
            "orc_tridiag_eig": (C.c_int, [_dp, _dp, _i64, _dp, _dp]),
            "orc_gp_create": (_vp, [C.c_int, _d, _d, _dp, _dp, _dp, _i64, C.c_int, _d, _d,
                                    C.c_int, _d, C.c_int, _i64, _d, C.c_int, _d, C.c_int,
                                    C.c_int, _i64, C.c_int, C.c_int, _u64]),
            "orc_gp_free": (None, [_vp]),
            "orc_gp_lml": (C.c_int, [_vp, _dp, _dp, _dp, _ip]),
            "orc_gp_alpha": (C.c_int, [_vp, _dp, _ip]),
            "orc_gp_pivots": (C.c_int, [_vp, _i64p, _i64p]),
            "orc_gp_predict_mean_grad": (C.c_int, [_vp, _dp, _i64, _dp, _dp]),
            "orc_gp_predict_variance_pivchol": (C.c_int, [_vp, _dp, _dp]),
            "orc_gp_lml_gradient": (C.c_int, [_vp, C.c_int, _dp, C.POINTER(C.c_int)]),
            "orc_gp_predict_variance_exact": (C.c_int, [_vp, _dp, _dp]),
            "orc_gp_cross_covariance_jacobian": (C.c_int, [_vp, _dp, _dp]),
            "orc_gp_cross_covariance": (C.c_int, [_vp, _dp, _dp]),
            "orc_gp_predict_variance_randomized": (C.c_int, [_vp, _dp, C.c_longlong, C.c_int, C.c_ulonglong, _dp]),
            "orc_gp_dlogell_apply": (C.c_int, [_vp, _dp, _dp]),
            "orc_dskip_from_factors": (_vp, [_i64, C.c_int, _d, _d, C.c_int, _i64p, C.POINTER(_dp),
                                             C.POINTER(_dp), C.POINTER(_dp)]),
            "orc_make_dataset": (C.c_int, [C.c_int, _u64, _i64p, _ip, _dp, _dp, _dp]),
            "orc_sample_test_function": (C.c_int, [C.c_char_p, _i64, _u64, _d, _d, C.c_int, _ip, _dp, _dp,
                                                   _dp]),
            "orc_gp_fit": (C.c_int, [_vp, C.c_int, C.c_int, _d, _d, C.c_int, _u64, _dp, _dp]),
            "orc_gp_set_hyperparameters": (C.c_int, [_vp, _d, _d, _d, _d]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _f64(a, fortran=False):
    a = np.asarray(a, dtype=np.float64)
    return np.asfortranarray(a) if fortran else np.ascontiguousarray(a)


def _check(st):
    if st == 0:
        return
    msg = lib().orc_last_error().decode()
    if st == 3:
        raise OracleOutOfGridError(msg, lib().orc_last_error_point())
    raise ERRORS.get(st, RuntimeError)(msg)


# ------------------------------------------------------------------ rng
def mix_seed(seed, stream):
    return lib().orc_mix_seed(seed, stream)


def rademacher_vector(n, seed, stream=0):
    out = np.empty(n)
    lib().orc_rademacher(n, seed, stream, _p(out))
    return out


def gaussian_vector(n, seed, stream=0):
    out = np.empty(n)
    lib().orc_gaussian(n, seed, stream, _p(out))
    return out


def mt19937_64_nth(seed, nth):
    return lib().orc_mt19937_64_nth(seed, nth)


# ------------------------------------------------------------------ workloads
def make_dataset(config, seed=0):
    """Seeded synthetic workload C1..C5 (BASELINE.json configs), generated by the
    oracle library itself (datasets.cpp). Returns X (n×d, col-major), y, dY."""
    n, d = _i64(), C.c_int()
    if lib().orc_make_dataset(int(config), int(seed), C.byref(n), C.byref(d), None, None, None) != 0:
        raise ValueError("unknown dataset config")
    n, d = n.value, d.value
    X = np.empty((n, d), order="F")
    y = np.empty(n)
    dY = np.empty((n, d), order="F")
    lib().orc_make_dataset(int(config), int(seed), None, None, _p(X), _p(y), _p(dY))
    return X, y, dY


def sample_test_function(name, n, seed=0, noise=(0.0, 0.0), with_gradients=True):
    """sample_dataset (testfns.cpp:355-402), uniform sampling, for "franke"
    (d = 2) or "friedman" (d = 5). Returns X (n×d col-major), y, dY (or None)."""
    d = C.c_int()
    if lib().orc_sample_test_function(name.encode(), int(n), int(seed), 0.0, 0.0, 0, C.byref(d), None, None,
                                      None) != 0:
        raise ValueError(f"unknown test function '{name}'")
    X = np.empty((n, d.value), order="F")
    y = np.empty(n)
    dY = np.empty((n, d.value), order="F") if with_gradients else None
    lib().orc_sample_test_function(name.encode(), int(n), int(seed), float(noise[0]), float(noise[1]),
                                   int(with_gradients), C.byref(d), _p(X), _p(y),
                                   _p(dY) if dY is not None else None)
    return X, y, dY


def stacked_targets(y, dY, mean):
    """ObservationSet::stacked_targets (observations.hpp:29-35): [y - mean; ∂1y; …; ∂dy]."""
    parts = [np.asarray(y, dtype=np.float64) - mean]
    if dY is not None:
        dY = np.asarray(dY, dtype=np.float64)
        parts += [dY[:, j] for j in range(dY.shape[1])]
    return np.concatenate(parts)


# ------------------------------------------------------------------ kernels / interpolation
class KernelSpec:
    def __init__(self, ell, s, family=SE, spline_a=-1.5, spline_b=1.0, spline_even=False):
        self.ell, self.s, self.family = float(ell), float(s), int(family)
        self.a, self.b, self.even = float(spline_a), float(spline_b), int(bool(spline_even))

    def args(self):
        return (self.family, self.ell, self.s, self.a, self.b, self.even)


def kernel_eval(k, x, xp):
    x, xp = _f64(x), _f64(xp)
    d = x.size
    v, dl = _d(), _d()
    g = np.empty(d)
    H = np.empty((d, d))
    _check(lib().orc_kernel_eval(*k.args(), _p(x), _p(xp), d, C.byref(v), _p(g), _p(H), C.byref(dl)))
    return v.value, g, H, dl.value


def assemble_dense(k, X, Xp=None, with_derivatives=True, size_cap=50_000_000):
    X = _f64(X, True)
    Xp = X if Xp is None else _f64(Xp, True)
    n, d = X.shape
    npt = Xp.shape[0]
    rows = n * (d + 1) if with_derivatives else n
    cols = npt * (d + 1) if with_derivatives else npt
    if rows * cols > size_cap:
        raise OverflowError("dense assembly exceeds the configured size cap")
    out = np.empty((rows, cols), order="F")
    _check(lib().orc_assemble_dense(*k.args(), _p(X), n, _p(Xp), npt, d, int(with_derivatives),
                                    size_cap, _p(out)))
    return out


def quintic_weights(t):
    w, dw = np.empty(6), np.empty(6)
    _check(lib().orc_quintic_weights(t, _p(w), _p(dw)))
    return w, dw


def cubic_weights(t):
    w, dw = np.empty(4), np.empty(4)
    _check(lib().orc_cubic_weights(t, _p(w), _p(dw)))
    return w, dw


class Grid:
    def __init__(self, dims, origin, spacing):
        self.dims = np.ascontiguousarray(dims, dtype=np.int32)
        self.origin = _f64(origin)
        self.spacing = _f64(spacing)

    @property
    def d(self):
        return int(self.dims.size)

    def size(self):
        return int(np.prod(self.dims.astype(np.int64)))

    def cargs(self):
        return (self.dims.ctypes.data_as(_ip), _p(self.origin), _p(self.spacing), self.d)

    @staticmethod
    def cover(X, target_spacing, margin=3, max_nodes=128):
        X = _f64(X, True)
        n, d = X.shape
        dims = np.empty(d, np.int32)
        o, s = np.empty(d), np.empty(d)
        _check(lib().orc_grid_cover(_p(X), n, d, target_spacing, margin, max_nodes,
                                    dims.ctypes.data_as(_ip), _p(o), _p(s)))
        return Grid(dims, o, s)


def interp_dense(grid, X, order=0):
    X = _f64(X, True)
    n, d = X.shape
    out = np.zeros((n * (d + 1), grid.size()), order="F")
    _check(lib().orc_interp_dense(*grid.cargs(), _p(X), n, order, _p(out)))
    return out


def point_stencil(grid, x, order=0):
    x = _f64(x)
    d = grid.d
    nnz = (6 if order == 0 else 4) ** d
    idx = np.empty(nnz, np.int64)
    val = np.empty(nnz)
    der = np.empty((nnz, d), order="F")
    _check(lib().orc_point_stencil(*grid.cargs(), _p(x), order, idx.ctypes.data_as(_i64p),
                                   _p(val), _p(der)))
    return idx, val, der


# ------------------------------------------------------------------ operators
class Operator:
    def __init__(self, handle, keep=()):
        if not handle:
            _check(9 if not lib().orc_last_error() else _status_from_msg())
        self.h = handle
        self._keep = keep

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_op_free(self.h)
            self.h = None

    def size(self):
        return int(lib().orc_op_size(self.h))

    def mvm(self, x):
        x = _f64(x)
        if x.ndim == 2:
            x = np.asfortranarray(x)
            y = np.empty_like(x, order="F")
            _check(lib().orc_op_mvm_batch(self.h, _p(x), _p(y), x.shape[1]))
            return y
        if x.size != self.size():
            raise ValueError("MVM size mismatch")
        y = np.empty(self.size())
        _check(lib().orc_op_mvm(self.h, _p(x), _p(y)))
        return y

    apply = mvm

    def diagonal(self):
        out = np.empty(self.size())
        _check(lib().orc_op_diagonal(self.h, _p(out)))
        return out

    def row(self, r):
        out = np.empty(self.size())
        _check(lib().orc_op_row(self.h, int(r), _p(out)))
        return out

    def dense(self):
        N = self.size()
        return self.mvm(np.eye(N))


_last_create_status = [0]


def _status_from_msg():
    m = lib().orc_last_error().decode()
    for code, key in ((3, "outside the interior"), (1, ""),):
        if key in m:
            return code
    return 9


class DenseOperator(Operator):
    def __init__(self, A):
        A = _f64(A, True)
        self.A = A
        super().__init__(lib().orc_dense_create(_p(A), A.shape[0]), (A,))


class DskiOperator(Operator):
    def __init__(self, kernel, grid, X, noise=(0.0, 0.0), order=0, with_gradients=True):
        X = _f64(X, True)
        self.n, self.d = X.shape
        self.grid, self.kernel, self.noise = grid, kernel, noise
        h = lib().orc_dski_create(*kernel.args(), *grid.cargs(), _p(X), self.n, noise[0],
                                  noise[1], order, int(with_gradients))
        if not h:
            msg = lib().orc_last_error().decode()
            if "outside the interior" in msg:
                raise OracleOutOfGridError(msg, lib().orc_last_error_point())
            raise ValueError(msg)
        super().__init__(h, (X,))

    def stacked_transpose_apply(self, v):
        v = _f64(v)
        u = np.empty(self.grid.size())
        _check(lib().orc_dski_transpose_apply(self.h, _p(v), _p(u)))
        return u

    def stacked_apply(self, u):
        u = _f64(u)
        out = np.empty(self.size())
        _check(lib().orc_dski_apply(self.h, _p(u), _p(out)))
        return out

    def grid_mvm(self, u):
        u = _f64(u)
        out = np.empty(self.grid.size())
        _check(lib().orc_dski_grid_mvm(self.h, _p(u), _p(out)))
        return out

    def min_embedding_eigenvalue(self):
        return lib().orc_dski_min_embedding_eigenvalue(self.h)

    def noise_diagonal(self):
        N = self.size()
        nd = np.full(N, self.noise[1] ** 2)
        nd[: self.n] = self.noise[0] ** 2
        return nd


class GridKernelOperator:
    def __init__(self, kernel, grid, dlogell=False):
        self.grid = grid
        self.h = lib().orc_kuu_create(*kernel.args(), int(dlogell), *grid.cargs())
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_kuu_free(self.h)

    def mvm(self, v):
        v = _f64(v)
        out = np.empty(self.grid.size())
        _check(lib().orc_kuu_mvm(self.h, _p(v), _p(out)))
        return out

    apply = mvm

    def min_embedding_eigenvalue(self):
        return lib().orc_kuu_min_eig(self.h)


class OneDimFactor(Operator):
    def __init__(self, kernel, X, direction, grid_ratio=0.1, max_grid_nodes=512, dlogell=False):
        X = _f64(X, True)
        n, d = X.shape
        h = lib().orc_factor_create(kernel.family, kernel.ell, kernel.s, _p(X), n, d, direction,
                                    grid_ratio, max_grid_nodes, int(dlogell))
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        super().__init__(h, (X,))


class DskipOperator(Operator):
    def __init__(self, kernel, X, noise=(0.0, 0.0), rank=100, grid_ratio=0.1, max_grid_nodes=512,
                 seed=0, track_dlogell=False, with_gradients=True, rank_policy_error=False):
        X = _f64(X, True)
        self.n, self.d = X.shape
        self.noise = noise
        h = lib().orc_dskip_create(kernel.family, kernel.ell, kernel.s, _p(X), self.n, self.d,
                                   noise[0], noise[1], rank, grid_ratio, max_grid_nodes, seed,
                                   int(track_dlogell), int(with_gradients), int(rank_policy_error))
        if not h:
            msg = lib().orc_last_error().decode()
            raise (ValueError if "separable" in msg or "positive" in msg else RuntimeError)(msg)
        super().__init__(h, (X,))

    @staticmethod
    def from_factors(factors, n, groups, noise=(0.0, 0.0)):
        """Hadamard operator over given factors [(Q, alpha, beta), ...]."""
        op = DskipOperator.__new__(DskipOperator)
        op.n, op.d, op.noise = n, groups, noise
        nf = len(factors)
        Qs = [_f64(f[0], True) for f in factors]
        As = [_f64(f[1]) for f in factors]
        Bs = [_f64(f[2]) if np.asarray(f[2]).size else np.zeros(1) for f in factors]
        ranks = (_i64 * nf)(*[q.shape[1] for q in Qs])
        arr = lambda xs: (_dp * nf)(*[_p(x) for x in xs])  # noqa: E731
        h = lib().orc_dskip_from_factors(n, groups, float(noise[0]), float(noise[1]), nf, ranks, arr(Qs),
                                         arr(As), arr(Bs))
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        Operator.__init__(op, h, (Qs, As, Bs))
        return op

    def factors(self):
        out = []
        N = self.size()
        for f in range(lib().orc_dskip_factor_count(self.h)):
            r = lib().orc_dskip_factor_rank(self.h, f)
            Q = np.empty((N, r), order="F")
            a = np.empty(r)
            b = np.empty(max(r - 1, 0))
            lib().orc_dskip_factor_get(self.h, f, _p(Q), _p(a), _p(b))
            out.append((Q, a, b))
        return out

    def dlogell_apply(self, v):
        v = _f64(v)
        out = np.empty(self.size())
        _check(lib().orc_dskip_dlogell_apply(self.h, _p(v), _p(out)))
        return out

    def noise_diagonal(self):
        N = self.size()
        nd = np.full(N, self.noise[1] ** 2)
        nd[: self.n] = self.noise[0] ** 2
        return nd


# ------------------------------------------------------------------ solvers
class Preconditioner:
    def __init__(self, F, noise_diag):
        F = _f64(F, True)
        if F.ndim == 1:
            F = F.reshape(-1, 1, order="F")
        nd = _f64(noise_diag)
        if np.isscalar(noise_diag) or nd.ndim == 0:
            nd = np.full(F.shape[0], float(noise_diag) ** 2)
        self.n, self.k = F.shape
        self.h = lib().orc_precond_create(_p(F), self.n, self.k, _p(nd))
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_precond_free(self.h)

    def apply(self, b):
        b = _f64(b)
        out = np.empty(self.n)
        lib().orc_precond_apply(self.h, _p(b), _p(out))
        return out

    def quadratic(self, b):
        return lib().orc_precond_quadratic(self.h, _p(_f64(b)))

    def q1(self):
        out = np.empty((self.n, self.k), order="F")
        lib().orc_precond_q1(self.h, _p(out))
        return out


class CgResult:
    def __init__(self, x, iterations, converged, history):
        self.x, self.iterations, self.converged, self.residual_history = x, iterations, converged, history


def cg(op, b, tol=1e-4, max_iterations=1000, precond=None):
    b = _f64(b)
    N = op.size()
    if b.size != N:
        raise ValueError("cg: rhs size mismatch")
    x = np.empty(N)
    hist = np.empty(max_iterations + 1)
    its, conv, hl = C.c_int(), C.c_int(), C.c_int()
    _check(lib().orc_cg(op.h, _p(b), tol, max_iterations, precond.h if precond else None, _p(x),
                        C.byref(its), C.byref(conv), _p(hist), C.byref(hl)))
    return CgResult(x, its.value, bool(conv.value), hist[: hl.value].copy())


class PivotedCholeskyFactor:
    def __init__(self, L, pivots, initial_trace, residual_trace):
        self.L, self.pivots = L, pivots
        self.initial_trace, self.residual_trace = initial_trace, residual_trace


def pivoted_cholesky(op, max_rank, trace_tol=0.0, diag=None, noise_diag=None):
    """Pivoted Cholesky over op's rows (linalg.cpp:133-174). With noise_diag,
    follows GpModel::preconditioner (gp.cpp:128-136): factor the kernel part."""
    N = op.size()
    if diag is None:
        diag = op.diagonal()
        if noise_diag is not None:
            diag = np.maximum(diag - noise_diag, 0.0)
    diag = _f64(diag)
    nd = None if noise_diag is None else _f64(noise_diag)
    kmax = min(max_rank, N)
    L = np.empty((N, max(kmax, 1)), order="F")
    piv = np.empty(max(kmax, 1), np.int64)
    k = _i64()
    tr = np.empty(2)
    _check(lib().orc_pivchol(op.h, _p(diag), _p(nd) if nd is not None else None, kmax, trace_tol,
                             _p(L), piv.ctypes.data_as(_i64p), C.byref(k), _p(tr)))
    k = k.value
    return PivotedCholeskyFactor(np.asfortranarray(L[:, :k]), piv[:k].copy(), tr[0], tr[1])


class SlqResult:
    def __init__(self, logdet, clamped, estimates):
        self.logdet, self.clamped, self.estimates = logdet, clamped, estimates


def slq_logdet(op, probes=10, lanczos_steps=50, seed=0, eigen_floor=1e-12):
    ld, cl = _d(), C.c_int()
    est = np.empty(max(probes, 1))
    _check(lib().orc_slq(op.h, probes, lanczos_steps, seed, eigen_floor, C.byref(ld), C.byref(cl),
                         _p(est)))
    return SlqResult(ld.value, cl.value, est[:probes].copy())


def trace_estimate(A, B, probes, seed, tol=1e-4, max_iterations=1000, precond=None):
    out = _d()
    _check(lib().orc_trace_estimate(A.h, B.h, probes, seed, tol, max_iterations,
                                    precond.h if precond else None, C.byref(out)))
    return out.value


class LanczosFactor:
    def __init__(self, Q, alpha, beta, breakdown):
        self.Q, self.alpha, self.beta, self.breakdown = Q, alpha, beta, breakdown

    def rank(self):
        return self.Q.shape[1]

    def tridiagonal(self):
        r = self.alpha.size
        T = np.diag(self.alpha)
        if r > 1:
            T += np.diag(self.beta, 1) + np.diag(self.beta, -1)
        return T

    def apply(self, v):
        return self.Q @ (self.tridiagonal() @ (self.Q.T @ v))

    def dense(self):
        return self.Q @ self.tridiagonal() @ self.Q.T


def lanczos(op, steps, seed=0, start=None, restart_seed=0):
    N = op.size()
    steps = min(steps, N)
    Q = np.empty((N, steps), order="F")
    a = np.empty(steps)
    b = np.empty(max(steps - 1, 1))
    k = _i64()
    bd = C.c_int()
    st = _f64(start) if start is not None else None
    _check(lib().orc_lanczos(op.h, steps, seed, _p(st) if st is not None else None, restart_seed,
                             _p(Q), _p(a), _p(b), C.byref(k), C.byref(bd)))
    k = k.value
    return LanczosFactor(np.asfortranarray(Q[:, :k]), a[:k].copy(), b[: max(k - 1, 0)].copy(),
                         bool(bd.value))


def lanczos_lowrank(op, rank, seed):
    if rank <= 0 or rank > op.size():
        raise ValueError("Lanczos rank must lie in [1, N]")
    return lanczos(op, rank, seed)


def tridiag_eig(alpha, beta):
    a, b = _f64(alpha), _f64(beta)
    n = a.size
    ev = np.empty(n)
    Z = np.empty((n, n), order="F")
    _check(lib().orc_tridiag_eig(_p(a), _p(b) if b.size else None, n, _p(ev), _p(Z)))
    return ev, Z


# ------------------------------------------------------------------ GP glue
class GpModel:
    BACKENDS = {"exact": 0, "dski": 1, "dskip": 2}

    def __init__(self, kernel, X, y, dY=None, noise=(1e-2, 1e-2), backend="dski", grid_ratio=0.2,
                 max_grid_nodes=128, dskip_rank=100, dskip_grid_ratio=0.1,
                 dskip_max_grid_nodes=512, tol=1e-4, max_iterations=1000, use_preconditioner=True,
                 precond_rank=100, slq_probes=10, slq_steps=50, seed=0):
        self.X = _f64(X, True)
        self.y = _f64(y)
        self.dY = _f64(dY, True) if dY is not None else None
        n, d = self.X.shape
        self.n, self.d = n, d
        self.h = lib().orc_gp_create(kernel.family, kernel.ell, kernel.s, _p(self.X), _p(self.y),
                                     _p(self.dY) if self.dY is not None else None, n, d, noise[0],
                                     noise[1], self.BACKENDS[backend], grid_ratio, max_grid_nodes,
                                     dskip_rank, dskip_grid_ratio, dskip_max_grid_nodes, tol,
                                     max_iterations, int(use_preconditioner), precond_rank,
                                     slq_probes, slq_steps, seed)
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_gp_free(self.h)

    def log_marginal_likelihood(self):
        lml, ld, fit = _d(), _d(), _d()
        its = C.c_int()
        _check(lib().orc_gp_lml(self.h, C.byref(lml), C.byref(ld), C.byref(fit), C.byref(its)))
        return {"lml": lml.value, "logdet": ld.value, "fit": fit.value, "iterations": its.value}

    def alpha(self):
        N = self.n * (self.d + 1 if self.dY is not None else 1)
        out = np.empty(N)
        its = C.c_int()
        _check(lib().orc_gp_alpha(self.h, _p(out), C.byref(its)))
        return out, its.value

    def pivots(self, kmax):
        piv = np.empty(kmax, np.int64)
        k = _i64()
        _check(lib().orc_gp_pivots(self.h, piv.ctypes.data_as(_i64p), C.byref(k)))
        return piv[: k.value].copy()

    def predict_mean_grad(self, Xt):
        Xt = _f64(Xt, True)
        T = Xt.shape[0]
        vals = np.empty(T)
        grads = np.empty((T, self.d), order="F")
        _check(lib().orc_gp_predict_mean_grad(self.h, _p(Xt), T, _p(vals), _p(grads)))
        return vals, grads

    def set_hyperparameters(self, ell, s, noise_value, noise_gradient):
        _check(lib().orc_gp_set_hyperparameters(self.h, ell, s, noise_value, noise_gradient))

    def fit(self, max_iterations=40, restarts=3, initial_step=0.3, min_step=1e-4, optimize_noise=True, seed=0):
        """GpModel::fit (gp.cpp:294-404). Returns dict(ell, s, noise_value,
        noise_gradient, log_marginal, restarts=[(succeeded, iterations, lml)])."""
        out = np.empty(5)
        nrest = max(restarts, 1) if max_iterations > 0 else 1
        rep = np.empty(3 * nrest)
        _check(lib().orc_gp_fit(self.h, int(max_iterations), int(restarts), float(initial_step), float(min_step),
                                int(optimize_noise), int(seed), _p(out), _p(rep)))
        return dict(ell=out[0], s=out[1], noise_value=out[2], noise_gradient=out[3], log_marginal=out[4],
                    restarts=[(bool(rep[3 * i]), int(rep[3 * i + 1]), rep[3 * i + 2]) for i in range(nrest)])

    def lml_gradient(self, probes=8):
        """GpModel::lml_gradient (gp.cpp:220-292): ∂LML/∂(log ℓ, log s, log σ₁[, log σ₂])."""
        g = np.empty(4)
        k = C.c_int()
        _check(lib().orc_gp_lml_gradient(self.h, int(probes), _p(g), C.byref(k)))
        return g[: k.value].copy()

    def dlogell_apply(self, v):
        """GpModel::dlogell_apply (gp.cpp:200-218)."""
        v = _f64(v)
        out = np.empty(v.size)
        _check(lib().orc_gp_dlogell_apply(self.h, _p(v), _p(out)))
        return out

    def cross_covariance(self, x):
        """GpModel::cross_covariance (gp.cpp:406-417, D-SKI): length N."""
        N = self.n * (self.d + 1 if self.dY is not None else 1)
        out = np.empty(N)
        _check(lib().orc_gp_cross_covariance(self.h, _p(_f64(x)), _p(out)))
        return out

    def cross_covariance_jacobian(self, x):
        """GpModel::cross_covariance_jacobian (gp.cpp:431-461, D-SKI): N × d."""
        N = self.n * (self.d + 1 if self.dY is not None else 1)
        out = np.empty(N * self.d)
        _check(lib().orc_gp_cross_covariance_jacobian(self.h, _p(_f64(x)), _p(out)))
        return out.reshape(N, self.d, order="F")

    def predict_variance_exact(self, x):
        """GpModel::predict_variance_exact (gp.cpp:499-502)."""
        out = _d()
        _check(lib().orc_gp_predict_variance_exact(self.h, _p(_f64(x)), C.byref(out)))
        return out.value

    def predict_variance_randomized(self, Xt, probes, seed):
        """GpModel::predict_variance_randomized (gp.cpp:519-547)."""
        Xt = _f64(Xt, True)
        out = np.empty(Xt.shape[0])
        _check(lib().orc_gp_predict_variance_randomized(self.h, _p(Xt), Xt.shape[0], int(probes), int(seed), _p(out)))
        return out

    def predict_variance_pivchol(self, x):
        out = _d()
        _check(lib().orc_gp_predict_variance_pivchol(self.h, _p(_f64(x)), C.byref(out)))
        return out.value
