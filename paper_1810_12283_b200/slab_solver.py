"""Grid-slab sharded solvers for the largest configuration:
PCG, pivoted Cholesky and the Woodbury preconditioner with the system's rows
sharded over ranks by grid slab (one process per GPU, torch.distributed for
the collectives: NCCL on GPUs, gloo in the CPU tests).

Every rank owns the rows of its slab's points (``SlabShardedDskiOperator``:
points partitioned by the first axis of their stencil base cell). Per the
reference algorithms, with the rank-local pieces and the exchanges:

* ``slab_cg`` — cg (linalg.cpp:85-131), each column independent: the MVM is
  the slab MVM (local scatter → all-reduce of the grid vector → K_UU → local
  gather + noise); every dot product and norm is a local partial sum followed
  by one all-reduce of the column vector (fixed rank order inside NCCL/gloo).
* ``slab_pivoted_cholesky`` — pivoted_cholesky (linalg.cpp:133-174) of the
  kernel part (GpModel::preconditioner, gp.cpp:117-141): the pivot is the
  global argmax of the residual diagonal with the LOWEST GLOBAL INDEX on ties
  (Eigen maxCoeff's first maximum) via an all-gather of per-rank (max, index)
  pairs; the pivot's owner broadcasts the pivot point, its derivative group
  and its row of L; each rank forms its rows of the pivot column as
  B_r K_UU w(x_piv) (the cross-covariance of the pivot's stencil).
* ``slab_preconditioner`` — Preconditioner (linalg.cpp:176-213): Q1 is
  row-sharded. The thin QR of [D^{-1/2} L; I] is CholeskyQR2 with the k×k Gram
  matrices all-reduced; apply(b) = D^{-1/2}(c − Q1 (Q1ᵀ c)) is a local
  projection, an all-reduce of the k×B projection, and a local finish.

The algorithms are written once over a per-rank backend: ``GpuSlabBackend``
runs the library's CUDA kernels (libgk_b200: stage kernels, gather, cross-
covariance, preconditioner projection/finish) on device tensors;
``CpuSlabBackend`` (test infrastructure) runs the same rank-local pieces
through the oracle so the multi-rank logic is exercised with gloo on CPU.
Vectors are torch tensors (N_local × B, RHS innermost) in each rank's local
type-major order ``[values; ∂1; …]`` of its own points.
"""
from __future__ import annotations

import math

import numpy as np


def _dist():
    import torch.distributed as dist
    return dist


class SlabSolveError(RuntimeError):
    pass


# ------------------------------------------------------------------ backends
class GpuSlabBackend:
    """Rank-local compute on the GPU through the product library."""

    def __init__(self, sop):
        import torch
        self.sop = sop
        self.torch = torch
        self.dev = sop.dev
        self.local = sop.local  # None on a rank whose slab holds no points
        self.n_loc = int(sop.mine.size)
        self.N_loc = sop.local.size() if sop.local is not None else 0
        self.rows = sop.local_rows()  # global row index of each local row
        self.X_loc = None
        self.noise = tuple(sop.noise)
        self.M = sop.M
        self._U = self._W = None

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64, device=self.dev)

    def mvm(self, P):
        """(N_loc, B) RHS-minor -> K∇ rows of this rank (slab MVM, one all-reduce)."""
        torch = self.torch
        B = P.shape[1]
        st = self._stream()
        if self.local is None:  # empty slab: join the grid all-reduce, no rows
            self.sop.mvm_local_dev(None, None, B)
            return torch.zeros((0, B), dtype=torch.float64, device=self.dev)
        Pc = P.t().contiguous()  # (B, N_loc) == col-major N_loc × B
        Vi = torch.empty(self.N_loc * B, dtype=torch.float64, device=self.dev)
        Oi = torch.empty_like(Vi)
        self.local.to_internal_dev(Pc.data_ptr(), Vi.data_ptr(), B, stream=st)
        if self._U is None or self._U.numel() < self.M * B:
            self._U = torch.empty(self.M * B, dtype=torch.float64, device=self.dev)
            self._W = torch.empty_like(self._U)
        self.sop.mvm_local_dev(Vi, Oi, B, self._U[: self.M * B], self._W[: self.M * B])
        Oe = torch.empty_like(Pc)
        self.local.from_internal_dev(Oi.data_ptr(), Oe.data_ptr(), B, stream=st)
        return Oe.t().contiguous()

    def noise_diag(self):
        nd = np.full(self.N_loc, self.noise[1] ** 2)
        nd[: self.n_loc] = self.noise[0] ** 2
        return self.torch.from_numpy(nd).to(self.dev)

    def diag_kernel(self):
        if self.local is None:
            return self.zeros(0)
        return self.torch.from_numpy(self.local.diagonal()).to(self.dev) - self.noise_diag()

    def point(self, r):
        """(coordinates, derivative group) of local row r."""
        i, g = r % self.n_loc, r // self.n_loc
        if self.X_loc is None:
            self.X_loc = np.asarray(self.sop.X_local, dtype=np.float64)
        return self.X_loc[i], g

    def kernel_column(self, x, g):
        """Local rows of the pivot's kernel column: B_r K_UU w(x), w the
        pivot's value (g = 0) or ∂/∂x_{g-1} stencil, on the device."""
        if self.local is None:
            return self.zeros(0)
        torch = self.torch
        xt = torch.as_tensor(np.asarray(x, dtype=np.float64).reshape(-1), device=self.dev).contiguous()
        col = torch.empty(self.N_loc, dtype=torch.float64, device=self.dev)
        self.local.cross_covariance_dev(xt.data_ptr(), 1, g - 1, col.data_ptr(), self.N_loc, stream=self._stream())
        return col

    def make_precond(self, Q1, dinv):
        from . import Preconditioner
        torch = self.torch
        if self.N_loc == 0:
            return ("empty", Q1.shape[1])
        Qc = Q1.t().contiguous()  # col-major N_loc × k
        di = dinv.contiguous()
        M = Preconditioner.from_q1_dev(Qc.data_ptr(), di.data_ptr(), self.N_loc, Q1.shape[1],
                                       device=self.dev.index or 0)
        torch.cuda.synchronize(self.dev)
        return M

    def precond_project(self, M, R):
        if isinstance(M, tuple):
            return self.zeros(M[1], R.shape[1])
        T = self.torch.empty((M.rank(), R.shape[1]), dtype=self.torch.float64, device=self.dev)
        R = R.contiguous()
        M.project_dev(R.data_ptr(), T.data_ptr(), R.shape[1], stream=self._stream())
        return T

    def precond_finish(self, M, R, T):
        if isinstance(M, tuple):
            return self.torch.empty_like(R)
        R = R.contiguous()
        Z = self.torch.empty_like(R)
        M.finish_dev(R.data_ptr(), T.contiguous().data_ptr(), Z.data_ptr(), R.shape[1], stream=self._stream())
        return Z


class CpuSlabBackend:
    """Rank-local compute through the oracle on CPU (TEST INFRASTRUCTURE: the
    gloo tests of the sharded algorithms). Same contract as GpuSlabBackend."""

    def __init__(self, kernel_o, grid_o, X, noise, mine, group=None):
        import torch
        import oracle as O
        self.O, self.torch, self.group = O, torch, group
        self.dev = torch.device("cpu")
        self.grid = grid_o
        self.X_loc = np.asarray(X, dtype=np.float64)[mine]
        self.n = X.shape[0]
        self.n_loc = self.X_loc.shape[0]
        self.d = X.shape[1]
        self.N_loc = self.n_loc * (self.d + 1)
        self.noise = tuple(noise)
        self.M = grid_o.size()
        self.rows = np.concatenate([g * self.n + np.asarray(mine) for g in range(self.d + 1)])
        self.op = O.DskiOperator(kernel_o, grid_o, self.X_loc, noise) if self.n_loc else None

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64)

    def noise_diag(self):
        nd = np.full(self.N_loc, self.noise[1] ** 2)
        nd[: self.n_loc] = self.noise[0] ** 2
        return self.torch.from_numpy(nd)

    def mvm(self, P):
        torch = self.torch
        Pn = P.numpy()
        B = Pn.shape[1]
        U = np.zeros((self.M, B))
        if self.op is not None:
            for b in range(B):
                U[:, b] = self.op.stacked_transpose_apply(Pn[:, b])
        Ut = torch.from_numpy(U)
        _dist().all_reduce(Ut, group=self.group)
        out = np.zeros((self.N_loc, B))
        if self.op is not None:
            for b in range(B):
                out[:, b] = self.op.stacked_apply(self.op.grid_mvm(Ut[:, b].numpy()))
        return torch.from_numpy(out) + self.noise_diag()[:, None] * P

    def diag_kernel(self):
        if self.op is None:
            return self.zeros(0)
        return self.torch.from_numpy(self.op.diagonal()) - self.noise_diag()

    def point(self, r):
        return self.X_loc[r % self.n_loc], r // self.n_loc

    def kernel_column(self, x, g):
        if self.op is None:
            return self.zeros(0)
        idx, val, der = self.O.point_stencil(self.grid, np.asarray(x, dtype=np.float64))
        w = np.zeros(self.M)
        w[idx] = val if g == 0 else der[:, g - 1]
        return self.torch.from_numpy(self.op.stacked_apply(self.op.grid_mvm(w)))

    def make_precond(self, Q1, dinv):
        return (Q1.clone(), dinv.clone())

    def precond_project(self, M, R):
        Q1, dinv = M
        return Q1.t() @ (dinv[:, None] * R)

    def precond_finish(self, M, R, T):
        Q1, dinv = M
        return dinv[:, None] * (dinv[:, None] * R - Q1 @ T)


# ------------------------------------------------------------------ collectives
def _sum(be, t, group=None):
    _dist().all_reduce(t, group=group)
    return t


def _coldot(be, a, b, group=None):
    """Column dot products Σ_rows a∘b over all ranks (B,)."""
    return _sum(be, (a * b).sum(0), group)


# ------------------------------------------------------------------ pivoted Cholesky
class SlabPivotedCholesky:
    def __init__(self, L, pivots, initial_trace, residual_trace):
        self.L, self.pivots = L, pivots
        self.initial_trace, self.residual_trace = initial_trace, residual_trace

    def rank(self):
        return len(self.pivots)


def slab_pivoted_cholesky(be, max_rank, trace_tol=0.0, group=None):
    """GpModel::preconditioner's pivoted Cholesky of the kernel part
    (gp.cpp:122-136, linalg.cpp:133-174) with rows sharded over ranks."""
    torch = be.torch
    dist = _dist()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    rows = torch.from_numpy(np.asarray(be.rows, dtype=np.int64))
    d = be.diag_kernel().clamp(min=0.0)  # diag.cwiseMax(0.0) (gp.cpp:135)
    N = int(_sum(be, torch.tensor([float(d.numel())], dtype=torch.float64, device=be.dev), group).item())
    initial = float(_sum(be, d.sum().reshape(1), group).item())
    gmax = d.max().reshape(1) if d.numel() else torch.zeros(1, dtype=torch.float64, device=be.dev)
    dist.all_reduce(gmax, op=dist.ReduceOp.MAX, group=group)
    scale = max(float(gmax.item()), 1e-300)
    max_rank = min(int(max_rank), N)
    L = be.zeros(be.N_loc, max(max_rank, 1))
    pivots = []
    residual = initial
    for k in range(max_rank):
        # global argmax, lowest global index on ties (Eigen maxCoeff)
        if d.numel():
            lm = d.max()
            cand = torch.nonzero(d == lm).flatten()
            gi = rows.to(cand.device)[cand].min()
            mine = torch.tensor([float(lm.item()), float(gi.item())], dtype=torch.float64, device=be.dev)
        else:
            mine = torch.tensor([-math.inf, math.inf], dtype=torch.float64, device=be.dev)
        allp = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allp, mine, group=group)
        vals = [(float(p[0].item()), float(p[1].item()), r) for r, p in enumerate(allp)]
        dmax = max(v[0] for v in vals)
        piv, owner = min((v[1], v[2]) for v in vals if v[0] == dmax)
        if dmax <= 0.0 or residual <= trace_tol * initial:
            break
        piv = int(piv)
        # the owner broadcasts the pivot point, its group and its row of L
        buf = torch.zeros(16 + 2 + k, dtype=torch.float64, device=be.dev)
        if me == owner:
            loc = int(np.nonzero(np.asarray(be.rows) == piv)[0][0])
            x, g = be.point(loc)
            buf[0] = float(len(x))
            buf[1] = float(g)
            buf[2:2 + len(x)] = torch.as_tensor(np.asarray(x, dtype=np.float64), device=be.dev)
            if k:
                buf[16 + 2:] = L[loc, :k]
        dist.broadcast(buf, src=owner, group=group)
        dx = int(buf[0].item())
        g = int(buf[1].item())
        x = buf[2:2 + dx].cpu().numpy()
        col = be.kernel_column(x, g)
        if k:
            col = col - L[:, :k] @ buf[16 + 2:]
        col = col / math.sqrt(dmax)
        L[:, k] = col
        pivots.append(piv)
        d = d - col * col
        dmin = d.min().reshape(1) if d.numel() else torch.full((1,), math.inf, dtype=torch.float64, device=be.dev)
        dist.all_reduce(dmin, op=dist.ReduceOp.MIN, group=group)
        if float(dmin.item()) < -1e-10 * scale:
            raise SlabSolveError("pivoted Cholesky: operator is not positive semidefinite "
                                 f"(residual diagonal {float(dmin.item())})")
        d = d.clamp(min=0.0)
        if me == owner:
            d[loc] = 0.0
        residual = float(_sum(be, d.sum().reshape(1), group).item())
    return SlabPivotedCholesky(L[:, : len(pivots)].contiguous(), pivots, initial, residual)


# ------------------------------------------------------------------ preconditioner
class SlabPreconditioner:
    """Row-sharded Preconditioner (linalg.cpp:176-213): Q1 rows of this rank."""

    def __init__(self, be, F, noise_diag, group=None):
        torch = be.torch
        bad = float(bool((noise_diag <= 0).any())) if noise_diag.numel() else 0.0
        if float(_sum(be, torch.tensor([bad], dtype=torch.float64, device=be.dev), group).item()) > 0:
            raise ValueError("preconditioner needs strictly positive noise")  # linalg.cpp:180-181
        k = F.shape[1]
        if k == 0:
            raise ValueError("preconditioner needs a factor of rank at least 1")
        self.be, self.group, self.k = be, group, k
        dinv = 1.0 / torch.sqrt(noise_diag)
        G = dinv[:, None] * F
        Q2 = torch.eye(k, dtype=torch.float64)
        # CholeskyQR2 of [G; I]: two passes, k×k Gram matrices all-reduced
        for _ in range(2):
            gram = _sum(be, (G.t() @ G).contiguous(), group).cpu() + Q2.t() @ Q2
            R = torch.linalg.cholesky(gram).t()  # upper, Rᵀ R = gram
            Rinv = torch.linalg.solve_triangular(R, torch.eye(k, dtype=torch.float64), upper=True)
            G = G @ Rinv.to(G.device)
            Q2 = Q2 @ Rinv
        self.Q1 = G
        self.M = be.make_precond(G, dinv)

    def apply(self, Rv):
        T = self.be.precond_project(self.M, Rv)
        _sum(self.be, T, self.group)
        return self.be.precond_finish(self.M, Rv, T)


# ------------------------------------------------------------------ PCG
class SlabCgResult:
    def __init__(self, X, iterations, converged, history):
        self.X, self.iterations, self.converged, self.residual_history = X, iterations, converged, history


def slab_cg(be, Bm, tol=1e-4, max_iterations=1000, precond=None, group=None):
    """cg (linalg.cpp:85-131) on this rank's rows of a block of right-hand
    sides (N_loc × B), every column with its own α, β and stopping iteration
    (a stopped column is frozen); x0 = 0. The per-column bookkeeping stays on
    the device: one host synchronisation per iteration (the stop test)."""
    torch = be.torch
    B = Bm.shape[1]
    X = torch.zeros_like(Bm)
    bnorm = torch.sqrt(_coldot(be, Bm, Bm, group))
    safe_b = torch.where(bnorm > 0, bnorm, torch.ones_like(bnorm))
    active = bnorm > 0
    conv = ~active  # b = 0: converged with 0 iterations (linalg.cpp:93-96)
    iters = torch.zeros(B, dtype=torch.int64, device=Bm.device)
    R = Bm.clone()
    Z = precond.apply(R) if precond is not None else R.clone()
    P = Z.clone()
    rz = _coldot(be, R, Z, group)
    relres = torch.sqrt(_coldot(be, R, R, group)) / safe_b
    nan = torch.full_like(relres, float("nan"))
    hist = [torch.where(active, relres, nan)]
    done0 = active & (relres <= tol)
    conv = conv | done0
    active = active & ~done0
    for it in range(max_iterations):
        if not bool(active.any()):
            break
        AP = be.mvm(P)
        pAp = _coldot(be, P, AP, group)
        active = active & ~(pAp <= 0)  # loss of positive definiteness: stop unconverged
        a = torch.where(active, rz / torch.where(active, pAp, torch.ones_like(pAp)), torch.zeros_like(pAp))
        X = X + a[None, :] * P
        R = R - a[None, :] * AP
        relres = torch.sqrt(_coldot(be, R, R, group)) / safe_b
        iters = torch.where(active, torch.full_like(iters, it + 1), iters)
        hist.append(torch.where(active, relres, nan))
        done = active & (relres <= tol)
        conv = conv | done
        active = active & ~done
        Z = precond.apply(R) if precond is not None else R.clone()
        rzn = _coldot(be, R, Z, group)
        beta = torch.where(active, rzn / torch.where(active, rz, torch.ones_like(rz)), torch.zeros_like(rz))
        P = torch.where(active[None, :], Z + beta[None, :] * P, P)
        rz = torch.where(active, rzn, rz)
    H = torch.stack(hist).cpu().numpy()
    histories = [[float(v) for v in H[:, b] if v == v] for b in range(B)]
    return SlabCgResult(X, [int(v) for v in iters.cpu().tolist()], [bool(v) for v in conv.cpu().tolist()],
                        histories)
