"""B200-native gradkrig hot path (arXiv 1810.12283): D-SKI / D-SKIP K∇ MVMs,
pivoted-Cholesky preconditioner, batched PCG and SLQ log-det on sm_100a.

This module is a thin Python mirror of the reference's C++ operator API
(proj/core/include/gradkrig/{linear_operator,dski,dskip,linalg}.hpp) over the
C-ABI in ``include/gk_capi.h`` (``_lib/libgk_b200.so``). Every compute call
runs the CUDA kernels of that library; there is no CPU fallback — if the
shared library is missing, importing this package raises.

Conventions follow the reference: X is n×d, operator vectors are
derivative-type-major ``[f; ∂1 f; …; ∂d f]``, multi-RHS blocks are N×nrhs.
"""
from __future__ import annotations

import ctypes as C
import os
import dataclasses
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GK_B200_LIB: an alternative build of the same library (A/B timing of compile-time variants)
LIB_PATH = os.environ.get("GK_B200_LIB") or os.path.join(_HERE, "_lib", "libgk_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

_d = C.c_double
_dp = C.POINTER(C.c_double)
_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_u64 = C.c_uint64
_vp = C.c_void_p


class GkKernel(C.Structure):
    _fields_ = [("family", C.c_int), ("lengthscale", _d), ("outputscale", _d),
                ("spline_a", _d), ("spline_b", _d), ("spline_even", C.c_int)]


class GkGrid(C.Structure):
    _fields_ = [("d", C.c_int), ("dims", C.c_int * 8), ("origin", _d * 8), ("spacing", _d * 8)]


class GkDskipConfig(C.Structure):
    _fields_ = [("rank", _i64), ("grid_ratio", _d), ("max_grid_nodes", C.c_int), ("seed", _u64),
                ("rank_policy_error", C.c_int), ("track_dlogell", C.c_int),
                ("with_gradients", C.c_int)]


_lib = C.CDLL(LIB_PATH)

_SIGS = {
    "gk_last_error": (C.c_char_p, []),
    "gk_last_error_point": (_i64, []),
    "gk_version": (C.c_char_p, []),
    "gk_set_tuning": (C.c_int, [C.c_char_p, C.c_int]),
    "gk_kernel_launch_count": (_i64, []),
    "gk_debug_fused_phases": (C.c_int, [_vp, C.c_int, _i64p, C.c_int]),
    "gk_debug_dmma_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "gk_debug_rademacher_dev": (C.c_int, [_i64, _u64, _u64, _dp]),
    "gk_dski_gather_dev": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "gk_grid_cover": (C.c_int, [_dp, _i64, C.c_int, _d, C.c_int, C.c_int, C.POINTER(GkGrid)]),
    "gk_mix_seed": (_u64, [_u64, _u64]),
    "gk_rademacher_vector": (None, [_i64, _u64, _u64, _dp]),
    "gk_gaussian_vector": (None, [_i64, _u64, _u64, _dp]),
    "gk_dski_create": (C.c_int, [C.POINTER(GkKernel), C.POINTER(GkGrid), _dp, _i64, _d, _d, C.c_int,
                                 C.c_int, C.c_int, C.POINTER(_vp)]),
    "gk_dskip_create": (C.c_int, [C.POINTER(GkKernel), _dp, _i64, C.c_int, _d, _d,
                                  C.POINTER(GkDskipConfig), C.c_int, C.POINTER(_vp)]),
    "gk_dense_create": (C.c_int, [_dp, _i64, C.c_int, C.POINTER(_vp)]),
    "gk_dskip_create_from_factors": (C.c_int, [_i64, C.c_int, _d, _d, C.c_int, _i64p, C.POINTER(_dp),
                                               C.POINTER(_dp), C.POINTER(_dp), C.c_int, C.POINTER(_vp)]),
    "gk_exact_create": (C.c_int, [C.POINTER(GkKernel), _dp, _i64, C.c_int, _d, _d, C.c_int, C.c_int,
                                  C.POINTER(_vp)]),
    "gk_op_destroy": (None, [_vp]),
    "gk_op_size": (_i64, [_vp]),
    "gk_op_kind": (C.c_int, [_vp]),
    "gk_op_mvm": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_op_mvm_dev": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, _vp]),
    "gk_op_diagonal": (C.c_int, [_vp, _dp]),
    "gk_op_row": (C.c_int, [_vp, _i64, _dp]),
    "gk_op_noise_diagonal": (C.c_int, [_vp, _dp]),
    "gk_op_stage_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, _i64, _vp]),
    "gk_op_to_internal_dev": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp]),
    "gk_op_from_internal_dev": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "gk_dski_grid_size": (_i64, [_vp]),
    "gk_dski_get_grid": (C.c_int, [_vp, C.POINTER(GkGrid)]),
    "gk_grid_kernel_create": (C.c_int, [C.POINTER(GkGrid), _dp, C.c_int, C.POINTER(_vp)]),
    "gk_dski_create_from_profile": (C.c_int, [C.POINTER(GkGrid), _dp, _i64, _d, _d, C.c_int, C.c_int, _dp, _dp,
                                              C.c_int, C.POINTER(_vp)]),
    "gk_assemble_dense": (C.c_int, [C.POINTER(GkKernel), _dp, _i64, _dp, _i64, C.c_int, C.c_int, C.c_int, _d, _i64,
                                    C.c_int, _dp]),
    "gk_dense_kernel_create": (C.c_int, [C.POINTER(GkKernel), _dp, _i64, C.c_int, _d, _d, C.c_int, _i64, C.c_int,
                                         C.POINTER(_vp)]),
    "gk_dense_cholesky_solve": (C.c_int, [_vp, _dp, _i64, _i64, _dp, _i64]),
    "gk_dense_cholesky_logdet": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "gk_dense_exact_lml_gradient": (C.c_int, [_vp, _dp, _dp, C.POINTER(C.c_int)]),
    "gk_dski_min_embedding_eigenvalue": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "gk_dski_transpose_apply": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_dski_apply": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_dski_grid_mvm": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_dskip_factor_count": (C.c_int, [_vp]),
    "gk_dskip_factor_rank": (_i64, [_vp, C.c_int]),
    "gk_dskip_factor_get": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp]),
    "gk_dskip_dlogell_apply": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_dski_dlogell_apply": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_pcg": (C.c_int, [_vp, _vp, _dp, _i64, _i64, _d, C.c_int, _dp, _i64, _ip, _ip, _dp, _ip]),
    "gk_pcg_dev": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _d, C.c_int, _vp, _i64, _ip, _ip, _vp]),
    "gk_pivoted_cholesky": (C.c_int, [_vp, C.c_int, _i64, _d, C.POINTER(_vp)]),
    "gk_pivchol_rank": (_i64, [_vp]),
    "gk_pivchol_get": (C.c_int, [_vp, _dp, _i64p, _dp, _dp]),
    "gk_pivchol_destroy": (None, [_vp]),
    "gk_precond_create": (C.c_int, [_dp, _i64, _i64, _dp, C.c_int, C.POINTER(_vp)]),
    "gk_precond_from_pivchol": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "gk_precond_apply": (C.c_int, [_vp, _dp, _i64, _dp, _i64, _i64]),
    "gk_precond_quadratic": (C.c_int, [_vp, _dp, _i64, _i64, _dp]),
    "gk_precond_rank": (_i64, [_vp]),
    "gk_precond_q1": (C.c_int, [_vp, _dp]),
    "gk_precond_destroy": (None, [_vp]),
    "gk_slq_logdet": (C.c_int, [_vp, C.c_int, C.c_int, _u64, _d, C.c_int, _dp, _ip, _dp]),
    "gk_lanczos": (C.c_int, [_vp, _i64, _u64, _dp, _u64, _dp, _dp, _dp, _i64p, _ip]),
    "gk_lml_gradient": (C.c_int, [_vp, _vp, _dp, C.c_int, _u64, C.c_double, C.c_int, _dp, _ip]),
    "gk_trace_estimate": (C.c_int, [_vp, _vp, C.c_int, _u64, _d, C.c_int, _vp, _dp]),
    "gk_dski_predict_mean_grad": (C.c_int, [_vp, _dp, _d, _dp, _i64, _dp, _dp]),
    "gk_dski_cross_covariance_jacobian": (C.c_int, [_vp, _dp, _i64, _dp, _i64]),
    "gk_dski_cross_covariance": (C.c_int, [_vp, _dp, _i64, _dp, _i64]),
    "gk_make_dataset": (C.c_int, [C.c_int, _u64, _i64p, _ip, _dp, _dp, _dp]),
    "gk_uniform_vector": (None, [_i64, _u64, _u64, _d, _d, _dp]),
    "gk_sample_test_function": (C.c_int, [C.c_char_p, _i64, _u64, _d, _d, C.c_int, _ip, _dp, _dp, _dp]),
    "gk_dski_cross_covariance_dev": (C.c_int, [_vp, _vp, _i64, C.c_int, _vp, _i64, _vp]),
    "gk_dski_fused_split_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _i64, _vp]),
    "gk_precond_from_q1_dev": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "gk_precond_project_dev": (C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "gk_precond_finish_dev": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "gk_gp_solve": (C.c_int, [_vp, _vp, _dp, _i64, _i64, _d, C.c_int, _dp, _i64, _ip]),
    "gk_gp_logdet": (C.c_int, [_vp, C.c_int, C.c_int, _u64, _d, _d, C.c_int, _dp]),
    "gk_gp_log_marginal_likelihood": (C.c_int, [_vp, _vp, _dp, _d, C.c_int, C.c_int, C.c_int, _u64, _d, _d,
                                                C.c_int, _dp, _dp, _dp, _dp]),
    "gk_dski_predict_variance_exact": (C.c_int, [_vp, _vp, _dp, _i64, _d, _d, C.c_int, _dp]),
    "gk_dski_predict_variance_randomized": (C.c_int, [_vp, _vp, _dp, _i64, _d, C.c_int, _u64, _d, C.c_int,
                                                      _dp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED_SYMBOLS = tuple(_SIGS)


# ------------------------------------------------------------------ errors
class OutOfGridError(RuntimeError):
    """gradkrig::OutOfGridError (reference interpolation.hpp:37-40)."""

    def __init__(self, msg, point):
        super().__init__(msg)
        self.point = point


class LogicError(RuntimeError):
    """std::logic_error (e.g. linear_operator.cpp:7-13)."""


class CudaError(RuntimeError):
    pass


_ERR = {1: ValueError, 2: IndexError, 4: RuntimeError, 5: LogicError, 6: OverflowError,
        7: CudaError, 8: CudaError, 9: NotImplementedError}


def _check(status):
    if status == 0:
        return
    msg = _lib.gk_last_error().decode()
    if status == 3:
        raise OutOfGridError(msg, int(_lib.gk_last_error_point()))
    raise _ERR.get(status, RuntimeError)(msg)


def _p(a):
    return a.ctypes.data_as(_dp)


def _f64(a, fortran=False):
    a = np.asarray(a, dtype=np.float64)
    return np.asfortranarray(a) if fortran else np.ascontiguousarray(a)


def kernel_launch_count() -> int:
    """Number of libgk_b200 CUDA kernels launched by this process so far."""
    return int(_lib.gk_kernel_launch_count())


def version() -> str:
    return _lib.gk_version().decode()


def set_tuning(key: str, value: int) -> int:
    """Select a kernel variant ("scatter", "gather", "toeplitz", "precond", "fused";
    0 = default; "fused" 1 disables the one-launch d = 2 MVM). Returns the old value."""
    return int(_lib.gk_set_tuning(key.encode(), int(value)))


# ------------------------------------------------------------------ rng (rng.hpp:12-38)
def mix_seed(seed, stream):
    return int(_lib.gk_mix_seed(seed, stream))


def rademacher_vector(n, seed, stream=0):
    out = np.empty(n)
    _lib.gk_rademacher_vector(n, seed, stream, _p(out))
    return out


def gaussian_vector(n, seed, stream=0):
    out = np.empty(n)
    _lib.gk_gaussian_vector(n, seed, stream, _p(out))
    return out


# ------------------------------------------------------------------ kernel / grid
SE, SPLINE = 0, 1


def uniform_vector(n, seed, stream, a, b):
    """std::uniform_real_distribution<double>(a, b) over seeded_rng(seed, stream)."""
    out = np.empty(n)
    _lib.gk_uniform_vector(n, seed, stream, float(a), float(b), _p(out))
    return out


def spline_constants_for_domain(scaled_diameter, dim):
    """SplineConstants::for_domain (kernels.cpp:42-90): a = −1.5·D; b is the
    first of 0.25·D³·2^j (j = 0..12) for which the kernel matrix of a 5-per-
    axis lattice (≤ 3 axes) spanning the scaled diameter D is PSD (min
    eigenvalue ≥ −1e-10 · max), doubled. Returns (a, b, even)."""
    if not scaled_diameter > 0:
        raise ValueError("spline domain diameter must be positive")
    even = dim % 2 == 0
    a = -1.5 * scaled_diameter
    rho3 = scaled_diameter ** 3
    axes = min(dim, 3)
    per_axis = 5
    side = scaled_diameter / np.sqrt(float(axes))
    idx = np.arange(per_axis ** axes)
    P = np.column_stack([side * ((idx // per_axis ** ax) % per_axis) / (per_axis - 1) for ax in range(axes)])
    D = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1))
    with np.errstate(divide="ignore", invalid="ignore"):
        radial = np.where(D > 0, D * D * np.log(np.where(D > 0, D, 1.0)), 0.0) if even else D ** 3
    mult = 0.25
    while mult <= 1024.0:
        b = mult * rho3
        ev = np.linalg.eigvalsh(radial + a * D * D + b)
        if ev.min() >= -1e-10 * ev.max():
            return a, 2.0 * b, even
        mult *= 2.0
    raise RuntimeError("spline constant calibration failed to reach PSD")


@dataclass
class KernelSpec:
    """KernelSpec (kernels.hpp:42-75): family, lengthscale, outputscale."""
    lengthscale: float
    outputscale: float
    family: int = SE
    spline_a: float = -1.5
    spline_b: float = 1.0
    spline_even: bool = False

    def __post_init__(self):
        if not self.lengthscale > 0:
            raise ValueError("lengthscale must be > 0")
        if not self.outputscale > 0:
            raise ValueError("outputscale must be > 0")

    def c(self):
        return GkKernel(self.family, self.lengthscale, self.outputscale, self.spline_a,
                        self.spline_b, int(self.spline_even))


class Grid:
    """Grid (interpolation.hpp:13-35): row-major, last dimension fastest."""

    def __init__(self, dims, origin, spacing):
        self.dims = np.asarray(dims, dtype=np.int64)
        self.origin = _f64(origin)
        self.spacing = _f64(spacing)

    @property
    def d(self):
        return int(self.dims.size)

    def size(self):
        return int(np.prod(self.dims))

    def c(self):
        g = GkGrid()
        g.d = self.d
        for j in range(self.d):
            g.dims[j] = int(self.dims[j])
            g.origin[j] = float(self.origin[j])
            g.spacing[j] = float(self.spacing[j])
        return g

    @staticmethod
    def from_c(g):
        return Grid([g.dims[j] for j in range(g.d)], [g.origin[j] for j in range(g.d)],
                    [g.spacing[j] for j in range(g.d)])

    @staticmethod
    def cover(X, target_spacing, margin_cells=3, max_nodes=128):
        """Grid::cover (interpolation.cpp:117-146)."""
        X = _f64(X, True)
        if X.ndim == 1:
            X = X.reshape(-1, 1, order="F")
        g = GkGrid()
        _check(_lib.gk_grid_cover(_p(X), X.shape[0], X.shape[1], target_spacing, margin_cells,
                                  max_nodes, C.byref(g)))
        return Grid.from_c(g)


# ------------------------------------------------------------------ operators
class LinearOperator:
    """LinearOperator (linear_operator.hpp:12-35) backed by a device gk_op."""

    def __init__(self, handle, device=0):
        self._h = handle
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.gk_op_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self):
        return int(_lib.gk_op_size(self._h))

    def mvm(self, v):
        """y = A v for a vector (N,) or a block (N, nrhs)."""
        v = np.asarray(v, dtype=np.float64)
        N = self.size()
        if v.shape[0] != N:
            raise ValueError("MVM size mismatch")
        if v.ndim == 1:
            out = np.empty(N)
            _check(_lib.gk_op_mvm(self._h, _p(np.ascontiguousarray(v)), N, _p(out), N, 1))
            return out
        V = np.asfortranarray(v)
        out = np.empty_like(V, order="F")
        _check(_lib.gk_op_mvm(self._h, _p(V), N, _p(out), N, V.shape[1]))
        return out

    apply = mvm

    def mvm_dev(self, dV, dOut, nrhs, ldv=None, ldo=None, stream=0):
        """Device-pointer MVM (external layout) on `stream` (raw pointers)."""
        N = self.size()
        _check(_lib.gk_op_mvm_dev(self._h, dV, ldv or N, dOut, ldo or N, nrhs, stream))

    def stage_dev(self, stage, dIn, dOut, nrhs, stream=0):
        _check(_lib.gk_op_stage_dev(self._h, stage, dIn, dOut, nrhs, stream))

    def to_internal_dev(self, dV, dI, nrhs, ldv=None, stream=0):
        _check(_lib.gk_op_to_internal_dev(self._h, dV, ldv or self.size(), dI, nrhs, stream))

    def from_internal_dev(self, dI, dV, nrhs, ldv=None, stream=0):
        _check(_lib.gk_op_from_internal_dev(self._h, dI, dV, ldv or self.size(), nrhs, stream))

    def has_diagonal(self):
        return True

    def diagonal(self):
        out = np.empty(self.size())
        _check(_lib.gk_op_diagonal(self._h, _p(out)))
        return out

    def has_rows(self):
        return True

    def row(self, i):
        out = np.empty(self.size())
        _check(_lib.gk_op_row(self._h, int(i), _p(out)))
        return out

    def noise_diagonal(self):
        out = np.empty(self.size())
        _check(_lib.gk_op_noise_diagonal(self._h, _p(out)))
        return out

    def dense(self):
        """LinearOperator::dense (linear_operator.cpp:15-27), batched."""
        N = self.size()
        out = np.empty((N, N), order="F")
        for c0 in range(0, N, 256):
            nb = min(256, N - c0)
            E = np.zeros((N, nb), order="F")
            E[np.arange(c0, c0 + nb), np.arange(nb)] = 1.0
            out[:, c0:c0 + nb] = self.mvm(E)
        return out


def _create(fn, *args):
    h = _vp()
    _check(fn(*args, C.byref(h)))
    return h


class DskiOperator(LinearOperator):
    """DskiOperator (dski.hpp:58-101): [W; ∂W] K_UU [W; ∂W]^T + noise."""

    def __init__(self, kernel: KernelSpec, grid: Grid, X, noise=(0.0, 0.0), order=0,
                 with_gradients=True, device=0):
        X = _f64(X, True)
        if X.ndim != 2 or X.shape[1] != grid.d:
            raise ValueError("interpolation points do not match grid dimension")
        self.n, self.d = X.shape
        self.kernel, self.grid, self.noise = kernel, grid, tuple(noise)
        k, g = kernel.c(), grid.c()
        super().__init__(_create(_lib.gk_dski_create, C.byref(k), C.byref(g), _p(X), self.n,
                                 float(noise[0]), float(noise[1]), int(order),
                                 int(with_gradients), device), device)

    @classmethod
    def from_profile(cls, grid: Grid, X, slice_ref, offset_table, noise=(0.0, 0.0), order=0, with_gradients=True,
                     device=0):
        """DskiOperator over a caller-evaluated stationary profile: slice_ref on
        the reference embedding (2(m_j − 1) per axis), offset_table at the
        (2T − 1)^d stencil offsets (gk_dski_create_from_profile)."""
        X = _f64(X, True)
        if X.ndim != 2 or X.shape[1] != grid.d:
            raise ValueError("interpolation points do not match grid dimension")
        self = cls.__new__(cls)
        self.n, self.d = X.shape
        self.kernel, self.grid, self.noise = None, grid, tuple(noise)
        g = grid.c()
        sl, ot = _f64(np.ravel(slice_ref)), _f64(np.ravel(offset_table))
        LinearOperator.__init__(self, _create(_lib.gk_dski_create_from_profile, C.byref(g), _p(X), self.n,
                                              float(noise[0]), float(noise[1]), int(order), int(with_gradients),
                                              _p(sl), _p(ot), device), device)
        return self

    def points(self):
        return self.n

    def min_embedding_eigenvalue(self):
        """GridKernelOperator::min_embedding_eigenvalue (dski.hpp:40-43) of the
        reference's 2(m−1) circulant embedding."""
        out = _d()
        _check(_lib.gk_dski_min_embedding_eigenvalue(self.handle, C.byref(out)))
        return out.value

    def grid_size(self):
        return int(_lib.gk_dski_grid_size(self._h))

    def _grid_block(self, fn, a, rows_in, rows_out):
        a = np.asarray(a, dtype=np.float64)
        vec = a.ndim == 1
        A = np.asfortranarray(a.reshape(rows_in, -1) if vec else a)
        if A.shape[0] != rows_in:
            raise ValueError("size mismatch")
        out = np.empty((rows_out, A.shape[1]), order="F")
        _check(fn(self._h, _p(A), rows_in, _p(out), rows_out, A.shape[1]))
        return out[:, 0] if vec else out

    def stacked_transpose_apply(self, v):
        """B^T v (dski.cpp:213-219)."""
        return self._grid_block(_lib.gk_dski_transpose_apply, v, self.size(), self.grid_size())

    def stacked_apply(self, u):
        """B u (dski.cpp:221-226)."""
        return self._grid_block(_lib.gk_dski_apply, u, self.grid_size(), self.size())

    def grid_mvm(self, u):
        """grid_operator().apply(u): K_UU u (dski.cpp:146-172)."""
        return self._grid_block(_lib.gk_dski_grid_mvm, u, self.grid_size(), self.grid_size())

    def predict_mean_grad(self, alpha, mean, Xtest):
        """GpModel::predict_mean_grad for D-SKI (gp.cpp:480-495)."""
        Xt = _f64(Xtest, True)
        T = Xt.shape[0]
        vals = np.empty(T)
        grads = np.empty((T, self.d), order="F")
        _check(_lib.gk_dski_predict_mean_grad(self._h, _p(_f64(alpha)), float(mean), _p(Xt), T,
                                              _p(vals), _p(grads)))
        return vals, grads

    def dlogell_apply(self, v):
        """∂K∇/∂log ℓ · v (no noise) — GpModel::dlogell_apply's D-SKI branch
        (gp.cpp:212-213): a second grid operator over kernel_dlogell_profile."""
        V = _f64(v, True)
        vec = V.ndim == 1
        V = V.reshape(-1, 1, order="F") if vec else V
        out = np.empty_like(V, order="F")
        _check(_lib.gk_dski_dlogell_apply(self._h, _p(V), V.shape[0], _p(out), V.shape[0], V.shape[1]))
        return out[:, 0] if vec else out

    def cross_covariance_dev(self, dXt, T, direction, dQ, ldq=None, stream=0):
        """Device-pointer cross-covariance columns (value stencil for
        direction -1, ∂/∂x_p for direction p), external row order."""
        _check(_lib.gk_dski_cross_covariance_dev(self._h, dXt, int(T), int(direction), dQ, ldq or self.size(),
                                                 stream))

    def fused_split_dev(self, phase, dV, dU2, dOut, nrhs, stream=0):
        """The one-launch MVM split at its first barrier: phase 0 scatters into
        dU2 = [u; h] (2·M·nrhs), phase 1 finishes from an all-reduced dU2.
        Returns False when unsupported for this operator."""
        st = _lib.gk_dski_fused_split_dev(self._h, int(phase), dV, dU2, dOut, int(nrhs), stream)
        if st == 9:
            return False
        _check(st)
        return True

    def gather_dev(self, dW, dV, dOut, nrhs, stream=0):
        """out = B w + noise·v on device pointers (internal layout): the last
        stage of a grid-slab sharded MVM."""
        _check(_lib.gk_dski_gather_dev(self._h, dW, dV, dOut, nrhs, stream))

    def cross_covariance_jacobian(self, Xtest):
        """GpModel::cross_covariance_jacobian (gp.cpp:431-461), batched: array
        (N, T, d) with [:, t, p] = ∂q(x_t)/∂x_p."""
        Xt = _f64(Xtest, True)
        T = Xt.shape[0]
        J = np.empty((self.size(), T * self.d), order="F")
        _check(_lib.gk_dski_cross_covariance_jacobian(self._h, _p(Xt), T, _p(J), self.size()))
        return J.reshape(self.size(), self.d, T, order="F").transpose(0, 2, 1)

    def cross_covariance(self, Xtest):
        """GpModel::cross_covariance for D-SKI (gp.cpp:412-417), one column per test point."""
        Xt = _f64(Xtest, True)
        if Xt.ndim == 1:
            Xt = Xt.reshape(1, -1, order="F")
        T = Xt.shape[0]
        Q = np.empty((self.size(), T), order="F")
        _check(_lib.gk_dski_cross_covariance(self._h, _p(Xt), T, _p(Q), self.size()))
        return Q


class ExactOperator(LinearOperator):
    """Matrix-free exact K∇ + noise, SE or spline kernel (kernels.cpp:104-170, 242-285 without assembly)."""

    def __init__(self, kernel: KernelSpec, X, noise=(0.0, 0.0), with_gradients=True, device=0):
        X = _f64(X, True)
        self.n, self.d = X.shape
        k = kernel.c()
        super().__init__(_create(_lib.gk_exact_create, C.byref(k), _p(X), self.n, self.d,
                                 float(noise[0]), float(noise[1]), int(with_gradients), device),
                         device)


class DenseOperator(LinearOperator):
    """DenseOperator (linear_operator.hpp:38-56) on the device."""

    def __init__(self, A, device=0):
        A = _f64(A, True)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("dense operator must be square")
        super().__init__(_create(_lib.gk_dense_create, _p(A), A.shape[0], device), device)


class GridKernelOperator(LinearOperator):
    """GridKernelOperator(grid, profile) (dski.hpp:20-50, dski.cpp:80-172):
    K_UU over the grid for a stationary profile given as its values on the
    reference's circulant embedding (2(m_j − 1) nodes per axis, wrapped
    offsets, row-major); applied by circulant embedding + FFT on the device."""

    def __init__(self, grid: Grid, slice_ref, device=0):
        self.grid = grid
        g = grid.c()
        sl = _f64(np.ravel(slice_ref))
        super().__init__(_create(_lib.gk_grid_kernel_create, C.byref(g), _p(sl), device), device)

    @staticmethod
    def embedding_offsets(grid: Grid):
        """The wrapped offsets (E' × d, row-major over E'_j = 2(m_j − 1)) at
        which the slice is evaluated (dski.cpp:97-114)."""
        E = [2 * (int(m) - 1) for m in grid.dims]
        idx = np.stack(np.meshgrid(*[np.arange(e) for e in E], indexing="ij"), -1).reshape(-1, grid.d)
        w = np.where(idx <= np.asarray(E) // 2, idx, idx - np.asarray(E))
        return w * np.asarray(grid.spacing)

    def min_embedding_eigenvalue(self):
        out = _d()
        _check(_lib.gk_dski_min_embedding_eigenvalue(self.handle, C.byref(out)))
        return out.value


def assemble_dense(kernel: KernelSpec, X, Xp=None, with_derivatives=True, dlogell=False, derivative_scale=0.0,
                   size_cap=50_000_000, device=0):
    """assemble_dense (kernels.cpp:242-285, AssemblyOptions kernels.hpp:83-92)
    on the device: type-major K∇(X, X') (or ∂K∇/∂log ℓ); OverflowError above
    size_cap entries (std::length_error)."""
    X = _f64(X, True)
    Xp = X if Xp is None else _f64(Xp, True)
    n, d = X.shape
    npt = Xp.shape[0]
    if Xp.shape[1] != d:
        raise ValueError("point sets have mismatched dimensions")
    rows = n * (d + 1) if with_derivatives else n
    cols = npt * (d + 1) if with_derivatives else npt
    out = np.empty((rows, cols), order="F") if rows * cols <= size_cap else np.empty((0, 0))
    k = kernel.c()
    _check(_lib.gk_assemble_dense(C.byref(k), _p(X), n, _p(Xp), npt, d, int(with_derivatives), int(dlogell),
                                  float(derivative_scale), int(size_cap), device, _p(out)))
    return out


class DenseKernelOperator(LinearOperator):
    """GpModel's exact operator (gp.cpp:71-85): the device-assembled K∇ + noise
    as a DenseOperator with its Cholesky factor (solve, logdet, the exact
    LML gradient of gp.cpp:246-276)."""

    def __init__(self, kernel: KernelSpec, X, noise=(1e-2, 1e-2), with_gradients=True, size_cap=50_000_000,
                 device=0):
        X = _f64(X, True)
        self.n, self.d = X.shape
        self.kernel = kernel
        k = kernel.c()
        super().__init__(_create(_lib.gk_dense_kernel_create, C.byref(k), _p(X), self.n, self.d, float(noise[0]),
                                 float(noise[1]), int(with_gradients), int(size_cap), device), device)

    def solve(self, B):
        b = np.asarray(B, dtype=np.float64)
        vec = b.ndim == 1
        Bm = np.asfortranarray(b.reshape(-1, 1) if vec else b)
        X = np.empty_like(Bm, order="F")
        _check(_lib.gk_dense_cholesky_solve(self.handle, _p(Bm), Bm.shape[0], Bm.shape[1], _p(X), X.shape[0]))
        return X[:, 0] if vec else X

    def logdet(self):
        out = _d()
        _check(_lib.gk_dense_cholesky_logdet(self.handle, C.byref(out)))
        return out.value

    def exact_lml_gradient(self, alpha):
        g = np.empty(4)
        k = C.c_int()
        _check(_lib.gk_dense_exact_lml_gradient(self.handle, _p(_f64(alpha)), _p(g), C.byref(k)))
        return g[: k.value].copy()


class DskipOperator(LinearOperator):
    """DskipOperator (dskip.hpp:91-121)."""

    def __init__(self, kernel: KernelSpec, X, noise=(0.0, 0.0), rank=100, grid_ratio=0.1,
                 max_grid_nodes=512, seed=0, rank_policy_error=False, track_dlogell=False,
                 with_gradients=True, device=0):
        X = _f64(X, True)
        self.n, self.d = X.shape
        cfg = GkDskipConfig(rank, grid_ratio, max_grid_nodes, seed, int(rank_policy_error),
                            int(track_dlogell), int(with_gradients))
        k = kernel.c()
        super().__init__(_create(_lib.gk_dskip_create, C.byref(k), _p(X), self.n, self.d,
                                 float(noise[0]), float(noise[1]), C.byref(cfg), device), device)

    @staticmethod
    def from_factors(factors, n, groups, noise=(0.0, 0.0), device=0):
        """D-SKIP operator over given Lanczos factors [(Q, alpha, beta), ...]
        (one or two; e.g. built by the reference/oracle)."""
        op = DskipOperator.__new__(DskipOperator)
        op.n, op.d = n, groups
        nf = len(factors)
        Qs = [np.asfortranarray(np.asarray(f[0], dtype=np.float64)) for f in factors]
        As = [_f64(f[1]) for f in factors]
        Bs = [_f64(f[2]) if np.asarray(f[2]).size else np.zeros(1) for f in factors]
        ranks = (_i64 * nf)(*[q.shape[1] for q in Qs])
        arr = lambda xs: (_dp * nf)(*[_p(x) for x in xs])  # noqa: E731
        h = _vp()
        _check(_lib.gk_dskip_create_from_factors(n, groups, float(noise[0]), float(noise[1]), nf, ranks,
                                                 arr(Qs), arr(As), arr(Bs), device, C.byref(h)))
        LinearOperator.__init__(op, h, device)
        op._keep = (Qs, As, Bs)
        return op

    def factors(self):
        out = []
        N = self.size()
        for f in range(_lib.gk_dskip_factor_count(self._h)):
            r = int(_lib.gk_dskip_factor_rank(self._h, f))
            Q = np.empty((N, r), order="F")
            a = np.empty(r)
            b = np.empty(max(r - 1, 1))
            _check(_lib.gk_dskip_factor_get(self._h, f, _p(Q), _p(a), _p(b)))
            out.append(LanczosFactor(Q, a, b[: max(r - 1, 0)], False))
        return out

    def dlogell_apply(self, v):
        v = np.asarray(v, dtype=np.float64)
        vec = v.ndim == 1
        V = np.asfortranarray(v.reshape(-1, 1) if vec else v)
        out = np.empty_like(V, order="F")
        _check(_lib.gk_dskip_dlogell_apply(self._h, _p(V), V.shape[0], _p(out), V.shape[0], V.shape[1]))
        return out[:, 0] if vec else out


# ------------------------------------------------------------------ solvers
@dataclass
class CgResult:
    """CgResult (linalg.hpp:18-23)."""
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray


def cg(A: LinearOperator, b, tol=1e-4, max_iterations=1000, precond=None, history=True):
    """cg (linalg.cpp:85-131). b may be (N,) or a block (N, nrhs): each column
    runs the reference's single-RHS PCG independently (one batched device
    solve). Returns a CgResult, or a list of them for a block."""
    b = np.asarray(b, dtype=np.float64)
    N = A.size()
    if b.shape[0] != N:
        raise ValueError("cg: rhs size mismatch")
    vec = b.ndim == 1
    B = np.asfortranarray(b.reshape(N, -1) if vec else b)
    nrhs = B.shape[1]
    X = np.empty((N, nrhs), order="F")
    its = np.empty(nrhs, np.int32)
    conv = np.empty(nrhs, np.int32)
    hist = np.empty((max_iterations + 1, nrhs), order="F") if history else None
    hl = np.empty(nrhs, np.int32)
    _check(_lib.gk_pcg(A.handle, precond.handle if precond is not None else None, _p(B), N, nrhs,
                       tol, max_iterations, _p(X), N, its.ctypes.data_as(_ip),
                       conv.ctypes.data_as(_ip), _p(hist) if history else None,
                       hl.ctypes.data_as(_ip)))
    res = [CgResult(X[:, c].copy(), int(its[c]), bool(conv[c]),
                    hist[: hl[c], c].copy() if history else np.empty(0)) for c in range(nrhs)]
    return res[0] if vec else res


def cg_dev(A: LinearOperator, dB, dX, nrhs, tol=1e-4, max_iterations=1000, precond=None, stream=0):
    """Device-pointer batched PCG (external layout). Returns (iterations, converged)."""
    its = np.empty(nrhs, np.int32)
    conv = np.empty(nrhs, np.int32)
    N = A.size()
    _check(_lib.gk_pcg_dev(A.handle, precond.handle if precond is not None else None, dB, N, nrhs,
                           tol, max_iterations, dX, N, its.ctypes.data_as(_ip),
                           conv.ctypes.data_as(_ip), stream))
    return its, conv


class PivotedCholeskyFactor:
    """PivotedCholeskyFactor (linalg.hpp:32-37); device-resident L."""

    def __init__(self, handle, N):
        self._h = handle
        self.N = N

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.gk_pivchol_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def rank(self):
        return int(_lib.gk_pivchol_rank(self._h))

    def _get(self):
        k = self.rank()
        L = np.empty((self.N, k), order="F")
        piv = np.empty(max(k, 1), np.int64)
        it, rt = _d(), _d()
        _check(_lib.gk_pivchol_get(self._h, _p(L) if k else None, piv.ctypes.data_as(_i64p),
                                   C.byref(it), C.byref(rt)))
        return L, piv[:k], it.value, rt.value

    @property
    def L(self):
        return self._get()[0]

    @property
    def pivots(self):
        return self._get()[1]

    @property
    def initial_trace(self):
        return self._get()[2]

    @property
    def residual_trace(self):
        return self._get()[3]


def pivoted_cholesky(A: LinearOperator, max_rank, trace_tol=0.0, kernel_part=False):
    """pivoted_cholesky (linalg.cpp:133-174) over A's diagonal and rows.
    kernel_part=True factors A - noise_diagonal (GpModel::preconditioner,
    gp.cpp:122-136)."""
    h = _vp()
    _check(_lib.gk_pivoted_cholesky(A.handle, int(kernel_part), int(max_rank), float(trace_tol),
                                    C.byref(h)))
    return PivotedCholeskyFactor(h, A.size())


class Preconditioner:
    """Preconditioner (linalg.cpp:176-213): M = D + F F^T applied via Q1."""

    def __init__(self, F=None, noise_diag=None, device=0, _handle=None, size=None):
        if _handle is not None:
            self._h, self.N = _handle, size
            return
        F = _f64(F, True)
        if F.ndim == 1:
            F = F.reshape(-1, 1, order="F")
        N, k = F.shape
        nd = np.asarray(noise_diag, dtype=np.float64)
        if nd.ndim == 0:
            nd = np.full(N, float(noise_diag) ** 2)
        if nd.size != N:
            raise ValueError("preconditioner factor and noise sizes differ")
        self.N = N
        h = _vp()
        _check(_lib.gk_precond_create(_p(F), N, k, _p(_f64(nd)), device, C.byref(h)))
        self._h = h

    @staticmethod
    def from_pivchol(A: LinearOperator, factor: PivotedCholeskyFactor):
        h = _vp()
        _check(_lib.gk_precond_from_pivchol(A.handle, factor.handle, C.byref(h)))
        return Preconditioner(_handle=h, size=A.size())

    @staticmethod
    def from_q1_dev(dQ1, ddinv, N, k, device=0):
        """Preconditioner over an explicit Q1 (N×k col-major) and D^{-1/2} (N),
        device pointers (a rank's rows of a row-sharded preconditioner)."""
        h = _vp()
        _check(_lib.gk_precond_from_q1_dev(dQ1, ddinv, int(N), int(k), int(device), C.byref(h)))
        return Preconditioner(_handle=h, size=int(N))

    def project_dev(self, dR, dT, nrhs, stream=0):
        """T = Q1ᵀ D^{-1/2} r over this preconditioner's rows (RHS-minor r, k×nrhs T)."""
        _check(_lib.gk_precond_project_dev(self._h, dR, dT, int(nrhs), stream))

    def finish_dev(self, dR, dT, dZ, nrhs, stream=0):
        """z = D^{-1/2}(D^{-1/2} r − Q1 T) for a given (all-reduced) T."""
        _check(_lib.gk_precond_finish_dev(self._h, dR, dT, dZ, int(nrhs), stream))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.gk_precond_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def rank(self):
        return int(_lib.gk_precond_rank(self._h))

    def size(self):
        return self.N

    def apply(self, b):
        b = np.asarray(b, dtype=np.float64)
        vec = b.ndim == 1
        B = np.asfortranarray(b.reshape(self.N, -1) if vec else b)
        out = np.empty_like(B, order="F")
        _check(_lib.gk_precond_apply(self._h, _p(B), self.N, _p(out), self.N, B.shape[1]))
        return out[:, 0] if vec else out

    def quadratic(self, b):
        b = np.asarray(b, dtype=np.float64)
        vec = b.ndim == 1
        B = np.asfortranarray(b.reshape(self.N, -1) if vec else b)
        out = np.empty(B.shape[1])
        _check(_lib.gk_precond_quadratic(self._h, _p(B), self.N, B.shape[1], _p(out)))
        return float(out[0]) if vec else out

    def q1(self):
        k = self.rank()
        out = np.empty((self.N, k), order="F")
        _check(_lib.gk_precond_q1(self._h, _p(out)))
        return out


@dataclass
class SlqResult:
    logdet: float
    clamped: int
    estimates: np.ndarray


def slq_logdet(A: LinearOperator, probes=10, lanczos_steps=50, seed=0, eigen_floor=1e-12,
               probe_offset=0):
    """slq_logdet (linalg.cpp:215-253); probes run as one batched Lanczos."""
    ld = _d()
    cl = C.c_int()
    est = np.empty(max(probes, 1))
    _check(_lib.gk_slq_logdet(A.handle, probes, lanczos_steps, seed, eigen_floor, probe_offset,
                              C.byref(ld), C.byref(cl), _p(est)))
    return SlqResult(ld.value, cl.value, est[:probes].copy())


def trace_estimate(A: LinearOperator, B: LinearOperator, probes, seed, tol=1e-4,
                   max_iterations=1000, precond=None):
    """trace_estimate (linalg.cpp:255-279)."""
    out = _d()
    _check(_lib.gk_trace_estimate(A.handle, B.handle, probes, seed, tol, max_iterations,
                                  precond.handle if precond is not None else None, C.byref(out)))
    return out.value


def lml_gradient(A: LinearOperator, alpha, probes=8, seed=0, tol=1e-4, max_iterations=1000, precond=None):
    """GpModel::lml_gradient (gp.cpp:220-292), stochastic-trace branch:
    dLML/d(log ell, log s, log sigma1[, log sigma2]) given alpha = K^-1 b (D-SKI / D-SKIP)."""
    g = np.empty(4)
    k = C.c_int()
    _check(_lib.gk_lml_gradient(A.handle, precond.handle if precond is not None else None, _p(_f64(alpha)),
                                int(probes), int(seed), float(tol), int(max_iterations), _p(g), C.byref(k)))
    return g[: k.value].copy()


def _prior_variance(A):
    k = A.kernel
    if k.family == SE:
        return k.outputscale ** 2  # eval(kernel, x, x) (gp.cpp:464-466)
    return k.outputscale ** 2 * k.spline_b  # spline at ρ = 0: s²·b (kernels.cpp:113-117)


def gp_solve(A: LinearOperator, B, tol=1e-4, max_iterations=1000, precond=None):
    """GpModel::solve (gp.cpp:143-158) for a block of columns: PCG, and the
    reference's RuntimeError when a column does not converge."""
    b = np.asarray(B, dtype=np.float64)
    vec = b.ndim == 1
    Bm = np.asfortranarray(b.reshape(-1, 1) if vec else b)
    X = np.empty_like(Bm, order="F")
    its = np.zeros(Bm.shape[1], np.int32)
    _check(_lib.gk_gp_solve(A.handle, precond.handle if precond is not None else None, _p(Bm), Bm.shape[0],
                            Bm.shape[1], float(tol), int(max_iterations), _p(X), X.shape[0],
                            its.ctypes.data_as(_ip)))
    return X[:, 0] if vec else X


def predict_variance_exact(A: "DskiOperator", Xtest, tol=1e-4, max_iterations=1000, precond=None):
    """GpModel::predict_variance_exact (gp.cpp:499-502) for a batch of test
    points: k(x, x) − q(x)ᵀ K⁻¹ q(x); cross-covariances, the batched solve and
    the dots run on the device (gk_dski_predict_variance_exact)."""
    Xt = _f64(Xtest, True)
    if Xt.ndim == 1:
        Xt = Xt.reshape(1, -1, order="F")
    out = np.empty(Xt.shape[0])
    _check(_lib.gk_dski_predict_variance_exact(A.handle, precond.handle if precond is not None else None, _p(Xt),
                                               Xt.shape[0], _prior_variance(A), float(tol), int(max_iterations),
                                               _p(out)))
    return out


def predict_variance_randomized(A: "DskiOperator", precond, Xtest, probes, seed, tol=1e-4, max_iterations=1000):
    """GpModel::predict_variance_randomized (gp.cpp:519-547): the pivoted-
    Cholesky variance plus an unbiased control-variate correction over
    Rademacher probes (streams 9000 + p) on the test points; all reductions
    on the device (gk_dski_predict_variance_randomized)."""
    if precond is None:
        raise ValueError("randomized variance needs the preconditioner enabled")
    Xt = _f64(Xtest, True)
    out = np.empty(Xt.shape[0])
    _check(_lib.gk_dski_predict_variance_randomized(A.handle, precond.handle, _p(Xt), Xt.shape[0],
                                                    _prior_variance(A), int(probes), int(seed), float(tol),
                                                    int(max_iterations), _p(out)))
    return out


class GpModel:
    """GpModel (gp.hpp:64-145; gp.cpp) over the device operators: the hot-path
    members (op, preconditioner, solve, alpha, logdet, log_marginal_likelihood,
    lml_gradient, predictions, fit). Backends "dski", "dskip" and "exact"
    (the device-assembled dense K∇ with a dense Cholesky factor, gp.cpp:71-85).
    Predictions for the non-D-SKI backends use the assembled cross-covariance
    (gp.cpp:419-461)."""

    def __init__(self, kernel: KernelSpec, X, y, dY=None, noise=(1e-2, 1e-2), backend="dski", grid_ratio=0.2,
                 max_grid_nodes=128, dskip_rank=100, dskip_grid_ratio=0.1, dskip_max_grid_nodes=512, tol=1e-4,
                 max_iterations=1000, use_preconditioner=True, precond_rank=100, slq_probes=10, slq_steps=50,
                 gradient_probes=8, seed=0, interpolation=0, dense_size_cap=50_000_000, device=0):
        if backend not in ("exact", "dski", "dskip"):
            raise ValueError(f"unknown backend '{backend}'")
        self.kernel = kernel
        self.X = _f64(X, True)
        self.y = _f64(y)
        self.dY = _f64(dY, True) if dY is not None else None
        self.n, self.d = self.X.shape
        nv, ng = float(noise[0]), float(noise[1])
        if not nv > 0:  # gp.cpp:38-41
            raise ValueError("value noise must be positive")
        if self.dY is not None and not ng > 0:
            raise ValueError("gradient noise must be positive")
        self.noise = (nv, ng)
        self.backend = backend
        self.cfg = dict(grid_ratio=grid_ratio, max_grid_nodes=max_grid_nodes, dskip_rank=dskip_rank,
                        dskip_grid_ratio=dskip_grid_ratio, dskip_max_grid_nodes=dskip_max_grid_nodes, tol=tol,
                        max_iterations=max_iterations, use_preconditioner=use_preconditioner,
                        precond_rank=precond_rank, slq_probes=slq_probes, slq_steps=slq_steps,
                        gradient_probes=gradient_probes, seed=seed, interpolation=interpolation,
                        dense_size_cap=dense_size_cap)
        self.device = device
        self.mean = float(self.y.mean())  # gp.cpp:43
        self._invalidate()

    def _invalidate(self):  # gp.cpp:55-64
        self._op = self._M = self._alpha = None

    def set_hyperparameters(self, kernel: KernelSpec, noise_value, noise_gradient):
        if not noise_value > 0:
            raise ValueError("value noise must be positive")
        self.kernel, self.noise = kernel, (float(noise_value), float(noise_gradient))
        self._invalidate()

    @property
    def has_gradients(self):
        return self.dY is not None

    def outputs(self):
        return self.n * (self.d + 1 if self.has_gradients else 1)

    def stacked_targets(self):
        return stacked_targets(self.y, self.dY, self.mean)

    def op(self):
        """GpModel::build_operator (gp.cpp:66-110)."""
        if self._op is None:
            c = self.cfg
            if self.backend == "exact":
                self._op = DenseKernelOperator(self.kernel, self.X, self.noise, self.has_gradients,
                                               c["dense_size_cap"], self.device)
            elif self.backend == "dski":
                grid = Grid.cover(self.X, c["grid_ratio"] * self.kernel.lengthscale, 3, c["max_grid_nodes"])
                self._op = DskiOperator(self.kernel, grid, self.X, self.noise, c["interpolation"],
                                        self.has_gradients, self.device)
            else:
                self._op = DskipOperator(self.kernel, self.X, self.noise, c["dskip_rank"], c["dskip_grid_ratio"],
                                         c["dskip_max_grid_nodes"], c["seed"], track_dlogell=True,
                                         with_gradients=self.has_gradients, device=self.device)
        return self._op

    def preconditioner(self):
        """GpModel::preconditioner (gp.cpp:117-141): rank-k pivoted Cholesky of
        the kernel part, noise in D."""
        if not self.cfg["use_preconditioner"]:
            return None
        if self._M is None:
            A = self.op()
            f = pivoted_cholesky(A, min(self.cfg["precond_rank"], A.size()), kernel_part=True)
            if f.rank() == 0:
                raise RuntimeError("pivoted Cholesky produced an empty preconditioner factor")
            self._M = Preconditioner.from_pivchol(A, f)
        return self._M

    def solve(self, b, tol_scale=1.0):
        if self.backend == "exact":  # llt_->solve (gp.cpp:146)
            return self.op().solve(b)
        return gp_solve(self.op(), b, self.cfg["tol"] * tol_scale, self.cfg["max_iterations"],
                        self.preconditioner())

    def alpha(self):
        if self._alpha is None:
            self._alpha = self.solve(self.stacked_targets())
        return self._alpha

    def logdet(self):
        """GpModel::logdet (gp.cpp:165-179): SLQ with floor ½·min(σ₁, σ₂)²
        (exact backend: 2 Σ log L_ii)."""
        if self.backend == "exact":
            return self.op().logdet()
        out = _d()
        _check(_lib.gk_gp_logdet(self.op().handle, int(self.cfg["slq_probes"]), int(self.cfg["slq_steps"]),
                                 int(self.cfg["seed"]), self.noise[0], self.noise[1], int(self.has_gradients),
                                 C.byref(out)))
        return out.value

    def log_marginal_likelihood(self):
        """GpModel::log_marginal_likelihood (gp.cpp:181-187)."""
        if self.backend == "exact":
            t = self.stacked_targets()
            return -0.5 * (float(t @ self.alpha()) + self.logdet() + t.size * np.log(2.0 * np.pi))
        A, M = self.op(), self.preconditioner()
        t = self.stacked_targets()
        lml, fit, ld = _d(), _d(), _d()
        a = np.empty(t.size)
        _check(_lib.gk_gp_log_marginal_likelihood(A.handle, M.handle if M is not None else None, _p(t),
                                                  float(self.cfg["tol"]), int(self.cfg["max_iterations"]),
                                                  int(self.cfg["slq_probes"]), int(self.cfg["slq_steps"]),
                                                  int(self.cfg["seed"]), self.noise[0], self.noise[1],
                                                  int(self.has_gradients), C.byref(lml), C.byref(fit),
                                                  C.byref(ld), _p(a)))
        self._alpha = a
        return lml.value

    def lml_gradient(self):
        """GpModel::lml_gradient (gp.cpp:220-292): exact traces through the
        dense factor (exact backend), else the stochastic-trace branch."""
        if self.backend == "exact":
            return self.op().exact_lml_gradient(self.alpha())
        return lml_gradient(self.op(), self.alpha(), self.cfg["gradient_probes"], self.cfg["seed"],
                            self.cfg["tol"], self.cfg["max_iterations"], self.preconditioner())

    def _assembled_cross(self, Xtest):
        """assemble_dense(X, Xtest) rows of the training outputs: columns t =
        cross_covariance(x_t) (gp.cpp:419-428), columns (p+1)·T + t its
        Jacobian column p (gp.cpp:447-460)."""
        Xt = _f64(np.atleast_2d(Xtest), True)
        K = assemble_dense(self.kernel, self.X, Xt, True, size_cap=self.cfg["dense_size_cap"], device=self.device)
        return K[: self.outputs()], Xt.shape[0]

    def predict_mean_grad(self, Xtest):
        """GpModel::predict_mean_grad (gp.cpp:471-496)."""
        if self.backend == "dski":
            return self.op().predict_mean_grad(self.alpha(), self.mean, Xtest)
        K, T = self._assembled_cross(Xtest)
        a = self.alpha()
        values = self.mean + K[:, :T].T @ a
        grads = np.column_stack([K[:, (p + 1) * T:(p + 2) * T].T @ a for p in range(self.d)])
        return values, grads

    def predict_mean(self, Xtest):
        return self.predict_mean_grad(Xtest)[0]

    def cross_covariance(self, Xtest):
        if self.backend == "dski":
            return self.op().cross_covariance(Xtest)
        K, T = self._assembled_cross(Xtest)
        return np.asfortranarray(K[:, :T])

    def cross_covariance_jacobian(self, Xtest):
        """(N, T, d) array, [:, t, p] = ∂q(x_t)/∂x_p (as DskiOperator's)."""
        if self.backend == "dski":
            return self.op().cross_covariance_jacobian(Xtest)
        K, T = self._assembled_cross(Xtest)
        return np.stack([K[:, (p + 1) * T:(p + 2) * T] for p in range(self.d)], axis=2)

    def prior_variance(self):
        k = self.kernel  # eval(kernel, x, x) (gp.cpp:464-466)
        return k.outputscale ** 2 * (1.0 if k.family == SE else k.spline_b)

    def predict_variance_exact(self, Xtest):
        """GpModel::predict_variance_exact (gp.cpp:506-509)."""
        if self.backend != "dski":
            Q = self.cross_covariance(Xtest)
            S = np.asarray(self.solve(Q)).reshape(Q.shape)
            return self.prior_variance() - np.einsum("ij,ij->j", Q, S)
        return predict_variance_exact(self.op(), Xtest, self.cfg["tol"], self.cfg["max_iterations"],
                                      self.preconditioner())

    def predict_variance_pivchol(self, Xtest):
        """GpModel::predict_variance_pivchol (gp.cpp:506-511)."""
        M = self.preconditioner()
        if M is None:
            raise LogicError("pivoted Cholesky variance needs the preconditioner enabled")
        Q = self.cross_covariance(Xtest)
        return self.prior_variance() - np.asarray(M.quadratic(Q), dtype=np.float64).reshape(Q.shape[1])

    def predict_variance_randomized(self, Xtest, probes, seed):
        M = self.preconditioner()
        if M is None:
            raise LogicError("randomized variance needs the preconditioner enabled")
        if self.backend != "dski":  # gp.cpp:519-547 over the assembled cross-covariance
            Kc = self.cross_covariance(Xtest)
            T = Kc.shape[1]
            base = self.prior_variance() - np.asarray(M.quadratic(Kc), dtype=np.float64).reshape(T)
            if probes <= 0:
                return base
            corr = np.zeros(T)
            for p in range(probes):
                z = rademacher_vector(T, seed, 9000 + p)
                w = Kc @ z
                corr += z * (Kc.T @ (np.asarray(self.solve(w)) - np.asarray(M.apply(w))))
            return base - corr / probes
        return predict_variance_randomized(self.op(), M, Xtest, probes, seed, self.cfg["tol"],
                                           self.cfg["max_iterations"])

    def dlogell_apply(self, v):
        """GpModel::dlogell_apply (gp.cpp:200-218)."""
        if self.backend == "exact":
            M = assemble_dense(self.kernel, self.X, None, self.has_gradients, dlogell=True,
                               size_cap=self.cfg["dense_size_cap"], device=self.device)
            return M @ np.asarray(v, dtype=np.float64)
        return self.op().dlogell_apply(v)

    def fit(self, max_iterations=40, restarts=3, initial_step=0.3, min_step=1e-4, optimize_noise=True, seed=0):
        """GpModel::fit (gp.cpp:294-404, FitOptions gp.hpp:50-57): gradient
        ascent on the LML in log-parameter space θ = (log ℓ, log s, log σ₁[,
        log σ₂]); steps clamped to ±0.5 per coordinate, θ clamped to the
        reference's boxes, step ×1.4 (≤ 2) on an accepted step and ×0.4 on a
        rejected one down to min_step; restart r > 0 jitters the start by
        U(−0.7, 0.7) from seeded_rng(seed, 31 + r). Every LML and gradient
        evaluation runs on the device (log_marginal_likelihood,
        lml_gradient); this loop is host control flow only. Leaves the model
        at the best restart's parameters and returns a FitResult."""
        grads = self.has_gradients
        npar = 4 if grads else 3
        lo = np.array([np.log(1e-4), np.log(1e-6)] + [np.log(1e-6)] * (npar - 2))
        hi = np.array([np.log(1e4), np.log(1e6)] + [np.log(1e3)] * (npar - 2))

        def encode():
            p = [np.log(self.kernel.lengthscale), np.log(self.kernel.outputscale), np.log(self.noise[0])]
            return np.array(p + ([np.log(self.noise[1])] if grads else []))

        def decode(p):
            k = dataclasses.replace(self.kernel, lengthscale=float(np.exp(p[0])), outputscale=float(np.exp(p[1])))
            self.set_hyperparameters(k, float(np.exp(p[2])), float(np.exp(p[3])) if grads else self.noise[1])

        p0 = encode()
        nrest = max(restarts, 1) if max_iterations > 0 else 1
        best = FitResult(self.kernel, self.noise[0], self.noise[1], -np.inf, [])
        best_p, any_ok = p0, False
        for r in range(nrest):
            rep = FitRestartReport()
            p = p0.copy()
            if r > 0:
                p = np.minimum(np.maximum(p + uniform_vector(npar, seed, 31 + r, -0.7, 0.7), lo), hi)
            try:
                decode(p)
                L = self.log_marginal_likelihood()
                step = initial_step
                it = 0
                while it < max_iterations:
                    try:
                        g = self.lml_gradient()
                    except (RuntimeError, ValueError):
                        break  # keep the progress made so far in this restart
                    if not optimize_noise:
                        g[2:] = 0.0
                    if not np.all(np.isfinite(g)):
                        raise RuntimeError("non-finite likelihood gradient")
                    if np.linalg.norm(g) < 1e-10:
                        break
                    accepted = False
                    while step >= min_step:
                        pt = np.minimum(np.maximum(p + np.clip(step * g, -0.5, 0.5), lo), hi)
                        decode(pt)
                        try:
                            Lt = self.log_marginal_likelihood()
                        except (RuntimeError, ValueError):
                            Lt = -np.inf
                        if np.isfinite(Lt) and Lt > L:
                            p, L = pt, Lt
                            step = min(step * 1.4, 2.0)
                            rep.accepted_steps += 1
                            accepted = True
                            break
                        step *= 0.4
                    if not accepted:
                        break
                    it += 1
                decode(p)
                rep.succeeded, rep.iterations, rep.log_marginal = True, it, L
                if L > best.log_marginal:
                    best.log_marginal, best_p = L, p
                any_ok = True
            except (RuntimeError, ValueError) as e:
                rep.succeeded, rep.error = False, str(e)
            best.restarts.append(rep)
        if not any_ok:
            raise RuntimeError("all fit restarts failed:" + "".join(f" [{r.error}]" for r in best.restarts))
        decode(best_p)
        best.kernel, best.noise_value, best.noise_gradient = self.kernel, self.noise[0], self.noise[1]
        return best


@dataclass
class FitRestartReport:
    """FitRestartReport (gp.hpp:59-65)."""
    succeeded: bool = False
    error: str = ""
    log_marginal: float = -np.inf
    iterations: int = 0
    accepted_steps: int = 0


@dataclass
class FitResult:
    """FitResult (gp.hpp:67-73)."""
    kernel: KernelSpec
    noise_value: float
    noise_gradient: float
    log_marginal: float
    restarts: list


class LanczosFactor:
    """LanczosFactor (linalg.hpp:102-114)."""

    def __init__(self, Q, alpha, beta, breakdown):
        self.Q, self.alpha, self.beta, self.breakdown = Q, alpha, beta, breakdown

    def rank(self):
        return self.Q.shape[1]

    def tridiagonal(self):
        T = np.diag(self.alpha)
        if self.alpha.size > 1:
            T = T + np.diag(self.beta, 1) + np.diag(self.beta, -1)
        return T

    def ritz_values(self):
        return np.sort(np.linalg.eigvalsh(self.tridiagonal()))[::-1]

    def apply(self, v):
        return self.Q @ (self.tridiagonal() @ (self.Q.T @ v))

    def dense(self):
        return self.Q @ self.tridiagonal() @ self.Q.T


def lanczos(A: LinearOperator, steps, seed=0, start=None, restart_seed=0):
    N = A.size()
    steps = min(int(steps), N)
    Q = np.empty((N, max(steps, 1)), order="F")
    a = np.empty(max(steps, 1))
    b = np.empty(max(steps, 1))
    k = _i64()
    bd = C.c_int()
    st = _f64(start) if start is not None else None
    _check(_lib.gk_lanczos(A.handle, steps, seed, _p(st) if st is not None else None, restart_seed,
                           _p(Q), _p(a), _p(b), C.byref(k), C.byref(bd)))
    k = k.value
    return LanczosFactor(np.asfortranarray(Q[:, :k]), a[:k].copy(), b[: max(k - 1, 0)].copy(),
                         bool(bd.value))


def lanczos_lowrank(A: LinearOperator, rank, seed):
    """lanczos_lowrank (linalg.cpp:306-314)."""
    if rank <= 0 or rank > A.size():
        raise ValueError("Lanczos rank must lie in [1, N]")
    return lanczos(A, rank, seed)


# ------------------------------------------------------------------ datasets
def make_dataset(config, seed=0):
    """Seeded synthetic workload C1..C5 (BASELINE.json configs). Returns X (n×d), y, dY."""
    n = _i64()
    d = C.c_int()
    _check(_lib.gk_make_dataset(config, seed, C.byref(n), C.byref(d), None, None, None))
    n, d = n.value, d.value
    X = np.empty((n, d), order="F")
    y = np.empty(n)
    dY = np.empty((n, d), order="F")
    _check(_lib.gk_make_dataset(config, seed, None, None, _p(X), _p(y), _p(dY)))
    return X, y, dY


def sample_test_function(name, n, seed=0, noise=(0.0, 0.0), with_gradients=True):
    """sample_dataset (testfns.cpp:355-402), uniform sampling, for the
    precond-study functions "franke" (d = 2) and "friedman" (d = 5).
    Returns X (n×d), y, dY (None without gradients)."""
    d = C.c_int()
    _check(_lib.gk_sample_test_function(name.encode(), int(n), int(seed), 0.0, 0.0, 0, C.byref(d), None, None,
                                        None))
    X = np.empty((n, d.value), order="F")
    y = np.empty(n)
    dY = np.empty((n, d.value), order="F") if with_gradients else None
    _check(_lib.gk_sample_test_function(name.encode(), int(n), int(seed), float(noise[0]), float(noise[1]),
                                        int(with_gradients), C.byref(d), _p(X), _p(y),
                                        _p(dY) if dY is not None else None))
    return X, y, dY


def stacked_targets(y, dY, mean):
    """ObservationSet::stacked_targets (observations.hpp:29-35)."""
    parts = [np.asarray(y) - mean]
    if dY is not None:
        parts += [np.asarray(dY)[:, j] for j in range(np.asarray(dY).shape[1])]
    return np.concatenate(parts)


def rademacher_vector_dev(n, seed, stream=0):
    """rademacher_vector generated by the device mt19937_64 kernel (test hook)."""
    out = np.empty(int(n))
    _check(_lib.gk_debug_rademacher_dev(int(n), int(seed), int(stream), _p(out)))
    return out


def dmma_peak_tflops(device=0):
    """Measured fp64 tensor-core (DMMA) throughput of `device`, TFLOP/s."""
    t = C.c_double(0.0)
    _check(_lib.gk_debug_dmma_peak(int(device), C.byref(t)))
    return t.value


def debug_fused_phases(op, nrhs, max_ctas=4096):
    """Per-CTA phase stamps (ns) of the last one-launch 2-D MVM (tuning
    "fused_prof" = 1): array (ctas, 8) — start, scatter done, barrier 1,
    mode-1 done, barrier 2, mode-0 done, barrier 3, gather done."""
    out = np.zeros((max_ctas, 8), dtype=np.int64)
    n = _lib.gk_debug_fused_phases(op.handle, int(nrhs), out.ctypes.data_as(_i64p), max_ctas)
    return out[:n]
