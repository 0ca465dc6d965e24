"""Multi-GPU partitioning of the hot path, host side.

Two schemes, both one process per GPU over ``torch.distributed``:

* **RHS / probe sharding** (C2, C5; probes of C1/C3). Columns are
  independent: every rank holds an operator replica and a contiguous slice of
  right-hand sides / SLQ probes. Probe ids are global (rank r's probe p is
  global probe ``offset + p``), so the union is exactly the single-GPU probe
  set, and the only exchange is the final per-probe estimates, summed on the
  host **in probe order** to reproduce ``slq_logdet``'s ordered sum
  (reference linalg.cpp:246-251).
* **Grid-slab point sharding** (C4). Points are partitioned by the first axis
  of their stencil base cell into contiguous slabs; each rank scatters its
  points into a full-size grid vector, the grid vectors are summed with one
  all-reduce per MVM, K_UU is applied redundantly, and each rank gathers its
  own points' outputs.

Nothing here touches the GPU; the functions are exercised on CPU with the
``gloo`` backend in tests/test_sharding_gloo.py.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of ``total`` items for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_probe_estimates(local: np.ndarray, offset: int, total: int, group=None,
                           device=None) -> np.ndarray:
    """All-gather per-probe estimates into global probe order (every rank gets
    the full vector). ``local`` holds probes [offset, offset + len(local)).
    ``device``: where the exchange buffers live (a CUDA device for NCCL, CPU
    for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    buf = torch.zeros(total, dtype=torch.float64, device=device)
    buf[offset:offset + len(local)] = torch.as_tensor(local, dtype=torch.float64, device=device)
    mask = torch.zeros(total, dtype=torch.float64, device=device)
    mask[offset:offset + len(local)] = 1.0
    parts = [torch.zeros_like(buf) for _ in range(world)]
    masks = [torch.zeros_like(mask) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    dist.all_gather(masks, mask, group=group)
    cover = torch.stack(masks).sum(0)
    if not torch.all(cover == 1.0):
        raise RuntimeError("probe shards do not tile the probe range exactly once")
    out = torch.zeros(total, dtype=torch.float64, device=device)
    for p, m in zip(parts, masks):
        out += p * m  # exactly one non-zero contribution per probe: no reordering error
    return out.cpu().numpy()


def ordered_mean(estimates: np.ndarray) -> float:
    """Σ_p est_p / P summed in probe order (linalg.cpp:246-251)."""
    s = 0.0
    for v in estimates:
        s += float(v)
    return s / len(estimates)


def slab_partition(base_rows: np.ndarray, n_rows: int, world: int) -> list[np.ndarray]:
    """Point indices per rank for grid-slab sharding: points are assigned by
    the first coordinate of their stencil base cell, rows split into
    ``world`` contiguous slabs of (nearly) equal point counts."""
    base_rows = np.asarray(base_rows)
    counts = np.bincount(base_rows, minlength=n_rows)
    cum = np.cumsum(counts)
    total = int(cum[-1]) if len(cum) else 0
    # slab boundaries at the row where the cumulative count crosses r*total/world
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cum, r * total / world, side="left")) + 1)
    bounds.append(n_rows)
    bounds = np.maximum.accumulate(np.minimum(bounds, n_rows))
    return [np.nonzero((base_rows >= bounds[r]) & (base_rows < bounds[r + 1]))[0] for r in range(world)]


def allreduce_grid(u_partial, group=None):
    """Sum the ranks' partial grid vectors in place (one all-reduce per MVM);
    a tensor on the rank's device for NCCL, on CPU for gloo."""
    import torch.distributed as dist

    dist.all_reduce(u_partial, op=dist.ReduceOp.SUM, group=group)
    return u_partial
