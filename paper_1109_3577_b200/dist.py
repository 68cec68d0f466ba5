"""Multi-GPU patch scheduling.

Patches are invariant under the optimal dynamics and need no transmission
conditions, so ranks solve disjoint patch sets with no halo exchange; the
only collective is the final gather of v, an element-wise MIN all-reduce
(every rank's non-owned nodes still hold the unreached value, which is >=
the owner's result; target nodes are 0 everywhere).  Patches are placed by
LPT (longest processing time first) on node counts, as north_star asks.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch


def world() -> tuple:
    """(rank, world_size) of the initialised process group, else (0, 1)."""
    import torch.distributed as td

    if td.is_available() and td.is_initialized():
        return td.get_rank(), td.get_world_size()
    return 0, 1


def lpt_assign(sizes: Sequence[int], n_ranks: int,
               weights: Optional[Sequence[float]] = None) -> np.ndarray:
    """Owner rank per patch: largest first onto the least-loaded rank
    (ties -> lowest rank; equal sizes keep patch order).  Empty patches go to
    rank 0 with no load."""
    w = np.asarray(weights if weights is not None else sizes, dtype=float)
    order = sorted(range(len(w)), key=lambda j: (-w[j], j))
    load = np.zeros(n_ranks)
    owner = np.zeros(len(w), dtype=np.int64)
    for j in order:
        r = int(np.argmin(load))
        owner[j] = r
        load[r] += w[j]
    return owner


def load_balance_bound(sizes: Sequence[int], n_ranks: int) -> float:
    """Upper bound on parallel efficiency of an LPT split: sum / (G * max bin)."""
    sizes = np.asarray(sizes, dtype=float)
    owner = lpt_assign(sizes, n_ranks)
    bins = np.bincount(owner, weights=sizes, minlength=n_ranks)
    return float(sizes.sum() / (n_ranks * bins.max())) if bins.max() > 0 else 1.0


def mine_mask(sizes: Sequence[int], rank: int, n_ranks: int, device) -> Optional[torch.Tensor]:
    """uint8 per patch: 1 where this rank sweeps the patch (None = all)."""
    if n_ranks <= 1:
        return None
    owner = lpt_assign(sizes, n_ranks)
    m = (owner == rank) & (np.asarray(sizes) > 0)
    return torch.as_tensor(m.astype(np.uint8), device=device)


def gather_min(t: torch.Tensor) -> torch.Tensor:
    """In-place element-wise MIN over ranks (NCCL over NVLink on GPUs)."""
    import torch.distributed as td

    if td.is_available() and td.is_initialized() and td.get_world_size() > 1:
        td.all_reduce(t, op=td.ReduceOp.MIN)
    return t
