"""Multi-GPU scheduling.

Patches are invariant under the optimal dynamics and need no transmission
conditions, so ranks solve disjoint patch sets with no halo exchange; the
final gather of v is an element-wise MIN all-reduce (every rank's non-owned
nodes still hold the unreached value, which is >= the owner's result; target
nodes are 0 everywhere).  Patches are placed by LPT (longest processing time
first) on node counts, as north_star asks, for the first solve of a patch
map; repeated solves of the same map (the benchmark's steps, parameter
sweeps) weight LPT by the per-patch executed evaluations the previous solve
measured (summed over ranks, so every rank derives the same assignment).

The colour transport (the labelling stage, a third of a step on one GPU) is
split by colour: colours are independent linear fixed points with their own
stopping rule, so each rank transports a disjoint colour set and the
per-node argmax is merged exactly with two all-reduces (MAX of the fp64
value bits -- phi >= 0, so the bit order is the value order -- then MIN of
the colour index, as uint8, among the ranks holding that maximum: the lowest colour
wins ties, as in the single-device running argmax, src/patchy.py:251-256).
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


def mine_mask(sizes: Sequence[int], rank: int, n_ranks: int, device,
              weights: Optional[Sequence[float]] = None) -> Optional[torch.Tensor]:
    """uint8 per patch: 1 where this rank sweeps the patch (None = all).
    LPT on ``weights`` (identical on every rank) when given, else on the
    node counts."""
    if n_ranks <= 1:
        return None
    owner = lpt_assign(sizes, n_ranks, weights)
    m = (owner == rank) & (np.asarray(sizes) > 0)
    return torch.as_tensor(m.astype(np.uint8), device=device)


def gather_min(t: torch.Tensor) -> torch.Tensor:
    """In-place element-wise MIN over ranks (NCCL over NVLink on GPUs)."""
    import torch.distributed as td

    if td.is_available() and td.is_initialized() and td.get_world_size() > 1:
        td.all_reduce(t, op=td.ReduceOp.MIN)
    return t


def colour_owner(n_colors: int, n_ranks: int) -> np.ndarray:
    """Owner rank per colour (round robin: colour costs are not known in
    advance and part sizes say little about them)."""
    return np.arange(n_colors, dtype=np.int64) % max(1, n_ranks)


def my_colours(n_colors: int, rank: int, n_ranks: int) -> np.ndarray:
    """Global indices of the colours this rank transports, ascending."""
    return np.nonzero(colour_owner(n_colors, n_ranks) == rank)[0]


def merge_argmax(best_val: torch.Tensor, best_idx: torch.Tensor, n_colors: int):
    """Exact cross-rank running argmax: per node the maximum value over all
    ranks' colours and the LOWEST global colour index attaining it.
    ``best_val`` (fp64, >= 0) / ``best_idx`` (global colour ids) are this
    rank's local argmax; both are replaced in place."""
    import torch.distributed as td

    if not (td.is_available() and td.is_initialized() and td.get_world_size() > 1):
        return best_val, best_idx
    bits = best_val.view(torch.int64)
    gbits = bits.clone()
    td.all_reduce(gbits, op=td.ReduceOp.MAX)
    # the index reduction in the narrowest type NCCL reduces (uint8 up to 254
    # colours: 1/8 of the bytes of the value reduction)
    idt = torch.uint8 if n_colors < 255 else torch.int32
    cand = torch.where(bits == gbits, best_idx.to(idt),
                       torch.full(bits.shape, n_colors, dtype=idt, device=bits.device))
    td.all_reduce(cand, op=td.ReduceOp.MIN)
    best_val.copy_(gbits.view(torch.float64))
    best_idx.copy_(torch.clamp(cand, max=n_colors - 1).to(best_idx.dtype))
    return best_val, best_idx


def slab_bounds(n_rows: int, n_ranks: int) -> list:
    """Block-row range [begin, end) per rank: equal slabs (the last ones may
    be short or empty), so one all-gather of equal chunks assembles the field."""
    per = (n_rows + n_ranks - 1) // n_ranks
    return [(min(r * per, n_rows), min((r + 1) * per, n_rows)) for r in range(n_ranks)]


def gather_slabs(compute, n_rows: int, row_elems: int, n_total: int, dtype, device):
    """A per-serial field computed by slabs: rank r calls
    ``compute(begin, end, field)`` for its block rows -- it fills
    ``field[begin * row_elems : end * row_elems]`` of the whole (padded) field
    with values >= -1 -- and the slabs are all-gathered in place.  Returns the first
    ``n_total`` elements (entries of other ranks are -1 when there is no
    process group: a patched world() in the one-GPU projection of a share)."""
    import torch.distributed as td

    rank, n_ranks = world()
    bounds = slab_bounds(n_rows, n_ranks)
    per = (n_rows + n_ranks - 1) // n_ranks
    full = torch.full((n_ranks * per * row_elems,), -1, dtype=dtype, device=device)
    b, e = bounds[rank]
    if e > b:
        compute(b, e, full)
    if n_ranks > 1 and td.is_available() and td.is_initialized():
        if full.is_cuda and td.get_backend() != "nccl":
            # gloo has no all-gather of device tensors (the functional
            # two-ranks-on-one-GPU check): the other ranks' entries are -1, the
            # field's values are >= -1, so an element-wise MAX assembles it
            td.all_reduce(full, op=td.ReduceOp.MAX)
        else:
            mine = full[rank * per * row_elems:(rank + 1) * per * row_elems]
            td.all_gather_into_tensor(full, mine.clone())
    return full[:n_total]


def sum_over_ranks(t: torch.Tensor) -> torch.Tensor:
    import torch.distributed as td

    if td.is_available() and td.is_initialized() and td.get_world_size() > 1:
        td.all_reduce(t, op=td.ReduceOp.SUM)
    return t
