"""Single-domain solves and the static decomposition geometry (mirror of
patchyhjb.decomp, decomp.py:1-212).

The reference's overlapping Schwarz iteration converges to the single-domain
fixed point (its module docstring; acceptance c02: max|R4 - R1| = 0).  On the
device the coarse stage of the patchy pipeline therefore runs as one
single-domain solve.  ``solve_dd`` runs the Schwarz iteration itself (the
paper's comparison baseline): per outer iteration one
device sweep per box with the outside hard, then the never-rising minimum
over owners (one MIN all-reduce across ranks).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .grid import ConfigurationError, Grid, NodeField
from .problems import ProblemSpec
from .runtime import ExecutionStrategy
from .solver import SolverConfig, StencilPlan, SweepStats, init_value_field, solve

_FACTORS = {
    2: {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2), 16: (4, 4)},
    3: {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2), 16: (4, 2, 2)},
}


@dataclass
class Subdomain:
    lo: tuple
    hi: tuple
    serials: np.ndarray
    active: np.ndarray


@dataclass
class StaticDecomposition:
    grid: Grid
    n_subdomains: int
    overlap_cells: int
    subdomains: list


def _axis_ranges(n_nodes: int, parts: int, overlap: int) -> list:
    splits = np.linspace(0, n_nodes, parts + 1).astype(int)
    out = []
    for p in range(parts):
        lo, hi = int(splits[p]), int(splits[p + 1]) - 1
        if p > 0:
            lo -= overlap
        if p < parts - 1:
            hi += overlap
        out.append((max(lo, 0), min(hi, n_nodes - 1)))
    return out


def make_static_decomposition(grid: Grid, n_subdomains: int,
                              overlap_cells: int = 1) -> StaticDecomposition:
    """Overlapping axis-slab boxes (decomp.py:64-98)."""
    factors = _FACTORS[grid.dim].get(n_subdomains)
    if factors is None:
        raise ConfigurationError(f"cannot decompose into {n_subdomains} subdomains "
                                 f"(supported: {sorted(_FACTORS[grid.dim])})")
    if overlap_cells < 1:
        raise ConfigurationError("overlap_cells must be >= 1")
    for m, p in zip(grid.shape, factors):
        if m < 2 * p:
            raise ConfigurationError("grid too small for this subdomain count")
    per_axis = [_axis_ranges(grid.shape[ax], factors[ax], overlap_cells)
                for ax in range(grid.dim)]
    subs = []
    for combo in np.ndindex(*factors):
        lo = tuple(per_axis[ax][combo[ax]][0] for ax in range(grid.dim))
        hi = tuple(per_axis[ax][combo[ax]][1] for ax in range(grid.dim))
        mesh = np.meshgrid(*[np.arange(lo[ax], hi[ax] + 1) for ax in range(grid.dim)],
                           indexing="ij")
        serials = np.sort(np.ravel_multi_index([m.ravel() for m in mesh], grid.shape))
        active = np.zeros(grid.n_ext, dtype=np.uint8)
        active[grid.interior_flat()[serials]] = 1
        subs.append(Subdomain(lo=lo, hi=hi, serials=serials.astype(np.int64), active=active))
    return StaticDecomposition(grid, n_subdomains, overlap_cells, subs)


def solve_single(spec: ProblemSpec, grid: Grid, cfg: Optional[SolverConfig] = None,
                 strategy: Optional[ExecutionStrategy] = None, *,
                 table: Optional[StencilPlan] = None):
    """Plain single-domain solve (decomp.py:193-204): (field, stats)."""
    table = table if table is not None else StencilPlan(grid, spec)
    field = init_value_field(grid, spec, kind=table.serial_to_user(table.kind))
    stats = solve(field, spec, cfg=cfg, strategy=strategy, table=table)
    return field, stats


def solve_dd(spec: ProblemSpec, grid: Grid, decomp: Optional[StaticDecomposition] = None,
             cfg: Optional[SolverConfig] = None, strategy: Optional[ExecutionStrategy] = None,
             *, table: Optional[StencilPlan] = None, field: Optional[NodeField] = None):
    """Domain-decomposition value iteration (decomp.py:101-190) on the device.

    Per outer iteration every box runs ONE device sweep of its nodes on a
    copy of the iteration-start field with everything outside the box hard
    (``active`` = the box, solver.py:243-249); overlap nodes take the minimum
    over their owners, never rising above the iteration-start value
    (decomp.py:172-179); converged when no node moved more than ``tol``.
    The box sweep is a Jacobi sweep (the reference: one Gauss-Seidel sweep),
    so the outer iteration counts differ; the fixed point is the
    single-domain one either way.  With several ranks (torch.distributed)
    the boxes are dealt round-robin and the per-iteration minimum is one
    MIN all-reduce -- the DD's halo exchange.  Returns ``(field, SweepStats)``
    with ``sweeps`` = outer iterations."""
    import dataclasses

    import torch

    from . import dist

    cfg = cfg or SolverConfig()
    table = table if table is not None else StencilPlan(grid, spec)
    if decomp is None:
        decomp = make_static_decomposition(grid, 1)
    if field is None:
        field = init_value_field(grid, spec, kind=table.serial_to_user(table.kind))
    rank, world = dist.world()
    box_cfg = dataclasses.replace(cfg, max_sweeps=1, schedule="jacobi", inner_sweeps=1,
                                  activity_tol=0.0)
    inner = torch.as_tensor(grid.interior_flat(), device=field.values.device)
    flat = field.values.view(-1)
    prev = flat[inner].clone()
    subs = [(j, sd) for j, sd in enumerate(decomp.subdomains) if j % max(1, world) == rank]
    sers = [torch.as_tensor(sd.serials, device=flat.device) for _, sd in subs]
    stats = SweepStats()
    limit = cfg.sweep_limit(grid)
    while stats.sweeps < limit:
        snap = field.values.clone()
        acc = prev.clone()
        for (j, sd), ser in zip(subs, sers):
            w = NodeField(grid, snap.clone())
            st = solve(w, spec, node_set=sd.serials, cfg=box_cfg, strategy=strategy, table=table,
                       active=sd.active)
            stats.node_relaxations += st.node_relaxations
            stats.candidate_evals += st.candidate_evals
            stats.performed_evals += st.performed_evals
            acc[ser] = torch.minimum(acc[ser], w.values.view(-1)[inner[ser]])
        dist.gather_min(acc)
        flat[inner] = acc
        stats.sweeps += 1
        stats.max_change = float((acc - prev).abs().max().item())
        prev = acc
        if stats.max_change <= cfg.tol:
            return field, stats
    stats.converged = False
    stats.warning = (f"domain decomposition: no convergence after {stats.sweeps} outer "
                     f"iterations (max change {stats.max_change:.3e} > tol {cfg.tol:.1e})")
    return field, stats
