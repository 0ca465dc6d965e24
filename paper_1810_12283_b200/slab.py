"""Grid-slab point sharding of the D-SKI MVM over ranks (the
largest configuration C4): one process per GPU, points partitioned by the
first axis of their stencil base cell (``sharding.slab_partition``).

Per MVM every rank
  1. scatters its own points into a FULL-size grid vector (Bᵣᵀ vᵣ),
  2. all-reduces the m×B grid vector over NCCL (NVLink/NVSwitch),
  3. applies K_UU to the summed grid vector (redundantly on every rank), and
  4. gathers and adds the noise for its own points (gk_dski_gather_dev).

The linear map is exactly the single-process D-SKI MVM (reference
dski.cpp:228-238); only the order of the grid-vector summation differs
(roundoff-level), which the 1e-12 parity gate covers. The kernels are the
library's own (stages 0 and 1 of gk_op_stage_dev, gk_dski_gather_dev); torch
is used for device memory and the NCCL collective only.
"""
from __future__ import annotations

import numpy as np

from . import DskiOperator
from .sharding import slab_partition


class SlabShardedDskiOperator:
    """The D-SKI operator of all points, with this rank holding one slab."""

    def __init__(self, kernel, grid, X, noise, order=0, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        X = np.asarray(X, dtype=np.float64)
        self.n, self.d = X.shape
        T = 6 if order == 0 else 4
        base0 = np.floor((X[:, 0] - grid.origin[0]) / grid.spacing[0]).astype(np.int64) - (2 if T == 6 else 1)
        nb0 = int(grid.dims[0]) - T + 1
        self.parts = slab_partition(np.clip(base0, 0, nb0 - 1), nb0, self.world)
        self.mine = self.parts[self.rank]
        self.X_local = X[self.mine]
        self.noise = tuple(noise)
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        # a rank whose slab holds no points still joins every all-reduce (with
        # a zero grid vector) and owns no rows
        self.local = (DskiOperator(kernel, grid, self.X_local, noise, order, True, device=self.device)
                      if self.mine.size else None)
        self.M = grid.size()
        self.G = self.d + 1
        # per RHS count: whether every rank can run the split one-launch path
        # (decided collectively: the all-reduced buffers must match)
        self._split = {}
        self._u2buf = None

    def _use_split(self, nrhs):
        import torch
        import torch.distributed as dist
        if nrhs not in self._split:
            ok = 1.0 if self.local is None else float(self.local.fused_split_dev(2, 0, 0, 0, nrhs))
            t = torch.tensor([ok], dtype=torch.float64, device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
            self._split[nrhs] = bool(t.item() > 0.5)
        return self._split[nrhs]

    def _u2(self, nrhs):
        import torch
        need = 2 * self.M * nrhs
        if self._u2buf is None or self._u2buf.numel() < need:
            self._u2buf = torch.empty(need, dtype=torch.float64, device=self.dev)
        return self._u2buf[:need]

    def size(self):
        return self.n * self.G

    def local_rows(self):
        """Global (type-major) row indices this rank owns, in local order."""
        return np.concatenate([g * self.n + self.mine for g in range(self.G)])

    def mvm_local_dev(self, Vi, Oi, nrhs, U=None, W=None):
        """Oi = (K∇ v) on this rank's rows; Vi, Oi are CUDA tensors in the local
        operator's internal layout. U, W: optional M·nrhs scratch tensors."""
        import torch
        import torch.distributed as dist

        st = torch.cuda.current_stream(self.dev).cuda_stream
        U = torch.empty(self.M * nrhs, dtype=torch.float64, device=self.dev) if U is None else U
        W = torch.empty_like(U) if W is None else W
        split = self._use_split(nrhs)
        if self.local is None:  # empty slab: contribute zeros to the grid sum, no rows to gather
            Z = self._u2(nrhs) if split else U
            Z.zero_()
            dist.all_reduce(Z, op=dist.ReduceOp.SUM, group=self.group)
            return
        if split:  # one-launch kernel split at its first barrier: [u; h] all-reduced between the launches
            U2 = self._u2(nrhs)
            self.local.fused_split_dev(0, Vi.data_ptr(), U2.data_ptr(), 0, nrhs, stream=st)
            dist.all_reduce(U2, op=dist.ReduceOp.SUM, group=self.group)
            self.local.fused_split_dev(1, Vi.data_ptr(), U2.data_ptr(), Oi.data_ptr(), nrhs, stream=st)
            return
        self.local.stage_dev(0, Vi.data_ptr(), U.data_ptr(), nrhs, stream=st)   # Bᵣᵀ vᵣ, full grid
        dist.all_reduce(U, op=dist.ReduceOp.SUM, group=self.group)             # Σ_r over NVLink
        self.local.stage_dev(1, U.data_ptr(), W.data_ptr(), nrhs, stream=st)   # K_UU
        self.local.gather_dev(W.data_ptr(), Vi.data_ptr(), Oi.data_ptr(), nrhs, stream=st)

    def mvm(self, V):
        """Host convenience: V (global, type-major, N × nrhs or N) identical on
        every rank; returns the global product on every rank."""
        import torch
        import torch.distributed as dist

        V = np.asarray(V, dtype=np.float64)
        vec = V.ndim == 1
        V2 = V.reshape(-1, 1) if vec else V
        nrhs = V2.shape[1]
        rows = self.local_rows()
        Nl = rows.size
        if self.local is None:
            self.mvm_local_dev(None, None, nrhs)
            out = torch.zeros((nrhs, self.size()), dtype=torch.float64, device=self.dev)
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
            res = out.T.cpu().numpy()
            return res[:, 0] if vec else res
        Vext = torch.from_numpy(np.ascontiguousarray(V2[rows].T)).to(self.dev)  # (nrhs, Nl) = col-major Nl×nrhs
        Vi = torch.empty(Nl * nrhs, dtype=torch.float64, device=self.dev)
        Oi = torch.empty_like(Vi)
        st = torch.cuda.current_stream(self.dev).cuda_stream
        self.local.to_internal_dev(Vext.data_ptr(), Vi.data_ptr(), nrhs, stream=st)
        self.mvm_local_dev(Vi, Oi, nrhs)
        Oe = torch.empty_like(Vext)
        self.local.from_internal_dev(Oi.data_ptr(), Oe.data_ptr(), nrhs, stream=st)
        out = torch.zeros((nrhs, self.size()), dtype=torch.float64, device=self.dev)
        out[:, torch.from_numpy(rows).to(self.dev)] = Oe
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)  # each row owned by one rank
        res = out.T.cpu().numpy()
        return res[:, 0] if vec else res
