"""Patchy decomposition pipeline on the device (mirror of patchyhjb.patchy,
patchy.py:1-467).

coarse solve -> saturating lift -> argmin feedback -> colour transport ->
argmax / majority-repair assembly -> independent patch solves -> merge, with
every stage a libphj kernel and fields resident in HBM between stages.  The
coarse stage is a single-domain solve: the reference routes it through
``solve_dd`` whose fixed point equals the single-domain one (decomp.py
module docstring; acceptance c02 measured max|R4-R1| = 0), so
``n_subdomains`` is accepted and not needed.

Extensions (PatchyConfig): ``coarse_target`` (separate coarse target, for
BASELINE config 1 whose 26^2 coarse grid holds no target node), ``parts``
(explicit target partition or a callable), ``transport_max_sweeps``.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os
from dataclasses import dataclass, field as _field
from typing import Callable, Optional, Sequence, Union

import numpy as np
import torch

from . import _lib, dist
from .grid import SENTINEL, ConfigurationError, Grid, NodeField, require_cuda
from .problems import (ProblemSpec, TargetSpec, _check_parts, device_partition_codes,
                       partition_target)
from .runtime import ExecutionStrategy, RunStats
from .solver import (_rule_id, DIRICHLET, KIND_FREE, KIND_OBSTACLE, KIND_TARGET, STATE_CONSTRAINT,
                     FeedbackField, SolverConfig, StencilPlan, SweepStats, ctypes_ref,
                     device_solve, feedback_internal, feedback_sharded, stats_for_patch, unreach_threshold,
                     unreached_value, _dtype_id)

UNREACHABLE = -1
TARGET = -2
OBSTACLE = -3
UNCOVERED = -4

#: last transport launch diagnostics (kernel ms, active blocks per sweep)
TRANSPORT_DIAG: dict = {}

#: colour transport re-activates a block's neighbourhood only for changes
#: above this fraction of color_tol: the geometric tails of
#: the Jacobi transport, orders of magnitude below the stopping tolerance,
#: no longer keep the whole domain busy.  0 gives exact Jacobi activity.
TRANSPORT_ACT_FRAC = float(os.environ.get("PHJ_TRANSPORT_ACT_FRAC", "1e-3"))
#: asynchronous transport: a colour change re-queues the neighbourhood only
#: above this fraction of color_tol; relaxations per block visit by dimension
# 1e-4: labels run-to-run identical at full config-2 size (1e-3: 1-3 of 4.2 M
# labels differed between runs, the dropped sub-threshold changes depending
# on visit order; profiles/r1d_c2_label_reproducibility.txt), +0.4 ms
TRANSPORT_ASYNC_FRAC = 1.0e-4
#: asynchronous transport in 3D too (off: slower than the Jacobi kernel there,
#: DESIGN.md §3.1b); module attributes so experiments can flip them
TRANSPORT_ASYNC_3D = False
TRANSPORT_INNER = {2: 8, 3: 4}
#: value-ordered pass before the Jacobi transport (3D): a
#: node is updated while its time band (lifted time-to-target / (k / max|f|))
#: lies within [s - lo, s + hi] of sweep s -- the colour masses cross the
#: domain in one outward pass instead of ~path-length Jacobi sweeps
TRANSPORT_BANDED = os.environ.get("PHJ_TRANSPORT_BANDED", "1") != "0"
TRANSPORT_BAND_WINDOW = tuple(int(x) for x in os.environ.get("PHJ_TRANSPORT_BAND_WINDOW", "3,1").split(","))  # (trailing, leading)
#: value-ordered pass before the patch solves: the same
#: band schedule over the patch nodes, keyed by the lifted field; the
#: schedule (async / jacobi) then continues from its result
SOLVE_BANDED = os.environ.get("PHJ_SOLVE_BANDED", "1") != "0"
SOLVE_BAND_WINDOW = tuple(int(x) for x in os.environ.get("PHJ_SOLVE_BAND_WINDOW", "6,2").split(","))
#: block-local relaxations per visit in the solve's pass (A/B on config 5,
#: profiles/r2_band_ab.jsonl: 1 -> 2.7 s, 2 -> 341 ms, 3 -> 401 ms)
SOLVE_BAND_INNER = int(os.environ.get("PHJ_BAND_INNER", "2"))
BAND_CAP_PER_NODE = 1.5
#: band width in units of the smallest SL time step (coarser bands: fewer,
#: thicker sweeps)
BAND_SCALE = float(os.environ.get("PHJ_BAND_SCALE", "1"))
#: the same for the transport's pass alone
TRANSPORT_BAND_SCALE = float(os.environ.get("PHJ_TBAND_SCALE", str(BAND_SCALE)))
#: fp32 workloads store the colour fields in fp32
TRANSPORT_PHI_FP32 = True
#: A/B knob: fp32 colour storage for fp64 workloads too (off: fp64 semantics)
TRANSPORT_PHI_FP32_ALWAYS = os.environ.get("PHJ_PHI_FP32", "0") != "0"


@dataclass
class PatchyConfig:
    """Pipeline knobs (patchy.py:48-87) + extensions (module docstring)."""

    n_patches: int = 1
    coarse_nodes: Union[int, tuple] = 51
    fine_nodes: Union[int, tuple] = 101
    bc_mode: str = STATE_CONSTRAINT
    warm_start: bool = False
    order_by_value: bool = False
    reduction: Optional[float] = None
    color_tol: float = 1.0e-2
    unreachable_threshold: Optional[float] = None
    coarse_target: Optional[TargetSpec] = None
    parts: Optional[Union[Sequence, Callable]] = None
    transport_max_sweeps: Optional[int] = None

    def __post_init__(self) -> None:
        if self.n_patches < 1:
            raise ConfigurationError("n_patches must be >= 1")
        if np.any(np.atleast_1d(self.fine_nodes) < np.atleast_1d(self.coarse_nodes)):
            raise ConfigurationError("fine grid must be at least as fine as the coarse grid")
        if self.bc_mode not in (STATE_CONSTRAINT, DIRICHLET):
            raise ConfigurationError(f"unknown bc_mode {self.bc_mode!r}")
        if self.color_tol <= 0.0:
            raise ConfigurationError("color_tol must be positive")
        if self.reduction is not None and self.reduction <= 1.0:
            raise ConfigurationError("reduction factor must exceed 1")


class PatchMap:
    """Node-to-patch assignment (patchy.py:90-118).  ``color`` is an int32
    tensor per user serial (patch id or a negative code)."""

    def __init__(self, grid: Grid, n_patches: int, color, patch_nodes=None, boundary=None,
                 uncovered_serials=None):
        self.grid = grid
        self.n_patches = int(n_patches)
        dev = color.device if isinstance(color, torch.Tensor) else None
        self.color = torch.as_tensor(np.asarray(color) if dev is None else color,
                                     dtype=torch.int32)
        if dev is None and torch.cuda.is_available():
            self.color = self.color.cuda()
        self._patch_nodes = patch_nodes
        self.boundary = boundary
        self.uncovered_serials = (uncovered_serials if uncovered_serials is not None
                                  else np.empty(0, dtype=np.int64))

    @property
    def patch_nodes(self) -> tuple:
        if self._patch_nodes is None:
            c = self.color.cpu().numpy()
            self._patch_nodes = tuple(np.where(c == j)[0].astype(np.int64)
                                      for j in range(self.n_patches))
        return self._patch_nodes

    def sizes(self) -> np.ndarray:
        return count_labels(self.color, self.n_patches).cpu().numpy()

    def size_report(self) -> tuple:
        sizes = self.sizes()
        return int(sizes.min()), int(sizes.max()), float(sizes.mean())

    def imbalance_warning(self) -> Optional[str]:
        lo, hi, mean = self.size_report()
        if self.n_patches > 1 and hi > 10.0 * max(mean, 1.0):
            return (f"patch sizes vary widely (min {lo}, max {hi}, mean {mean:.1f}); "
                    "expect uneven worker load")
        return None


@dataclass
class PatchyResult:
    value: NodeField
    patch_map: PatchMap
    lifted: NodeField
    feedback: FeedbackField
    stats: RunStats
    coarse_stats: SweepStats
    patch_stats: list = _field(default_factory=list)
    transport_sweeps: list = _field(default_factory=list)


# -- internal (device, internal axis order) stages ------------------------------------


def _full_domain_labels(plan: StencilPlan) -> torch.Tensor:
    """Single-domain solve labels: free -> patch 0, target -> TARGET, obstacle
    and ghosts -> HARD (solver.py:240-249 with active = all)."""
    lab = torch.full(plan.int_ext, _lib.LAB_HARD, dtype=torch.int16, device=plan.device)
    k = plan.kind.view(plan.int_shape)
    inner = plan.interior_int(lab)
    inner.copy_(torch.where(k == KIND_FREE, torch.zeros_like(k, dtype=torch.int16),
                            torch.where(k == KIND_TARGET,
                                        torch.full_like(k, _lib.LAB_TARGET, dtype=torch.int16),
                                        torch.full_like(k, _lib.LAB_HARD, dtype=torch.int16))))
    _sync_periodic(plan, lab)
    return lab


def _sync_periodic(plan: StencilPlan, t: torch.Tensor) -> None:
    if any(plan.gs.periodic[i] for i in range(plan.grid.dim)):
        _lib.check(_lib.load().phj_sync_periodic(ctypes_ref(plan.gs), t.element_size(),
                                                 _lib.ptr(t), _lib.stream_handle()),
                   "sync_periodic")


def init_working(plan: StencilPlan, rule: str, dtype: str) -> torch.Tensor:
    """unreached everywhere, 0 on target (solver.py:129-137), working units."""
    w = torch.empty(plan.int_ext, dtype=torch.float32 if dtype == "float32" else torch.float64,
                    device=plan.device)
    _lib.check(_lib.load().phj_init_field(ctypes_ref(plan.gs), _dtype_id(dtype),
                                          _lib.ptr(plan.kind), unreached_value(rule),
                                          _lib.ptr(w), _lib.stream_handle()), "init_field")
    _sync_periodic(plan, w)
    return w


def coarse_cfg(cfg: SolverConfig) -> SolverConfig:
    """Solver settings of the coarse stage.  It runs barrier-separated Jacobi
    sweeps even for asynchronous workloads (with 2 block-local relaxations:
    same speed on config 2's 513^2 grid): block-Jacobi is schedule
    independent, so the lifted field, the feedback and hence the patch labels
    are identical run to run.  Asynchronous coarse values differ between runs
    at rounding level, enough to flip feedback argmin ties (config 4's
    symmetric controls) and move patch boundaries."""
    if cfg.schedule == "async":
        return dataclasses.replace(cfg, schedule="jacobi", inner_sweeps=2)
    return cfg


def solve_full_internal(plan: StencilPlan, cfg: SolverConfig, work: Optional[torch.Tensor] = None):
    """Single-domain device solve from the init field; (working result, SweepStats)."""
    work = init_working(plan, cfg.rule, cfg.dtype) if work is None else work
    lab = _full_domain_labels(plan)
    res = device_solve(plan, work, lab, plan.fmask_hard, 1, rule=cfg.rule, dtype=cfg.dtype,
                       tol=cfg.tol, max_sweeps=cfg.sweep_limit(plan.grid),
                       act_tol=cfg.act_tol, schedule=cfg.schedule,
                           inner=cfg.inner_for(plan.grid.dim))
    n_free = int((plan.kind == KIND_FREE).sum().item())
    st = stats_for_patch(res, 0, n_free, plan.n_adm, cfg.tol)
    if cfg.schedule == "jacobi":
        st.node_relaxations = plan.grid.n_interior * st.sweeps
    st.performed_evals = res.real
    return res.values, st


def lift_internal(cplan: StencilPlan, vc: torch.Tensor, fplan: StencilPlan, rule: str,
                  dtype: str) -> torch.Tensor:
    """Saturating lift onto the fine grid (grid.py:242-261, patchy.py:145-148)."""
    vf = torch.full(fplan.int_ext, unreached_value(rule), dtype=vc.dtype, device=vc.device)
    thr = unreach_threshold(rule)
    _lib.check(_lib.load().phj_lift(ctypes_ref(cplan.gs), ctypes_ref(fplan.gs), _dtype_id(dtype),
                                    _lib.ptr(vc), _lib.ptr(vf), thr, unreached_value(rule), 1,
                                    _lib.stream_handle()), "phj_lift")
    _sync_periodic(fplan, vf)
    return vf


def banded_applies(plan: StencilPlan) -> bool:
    """The value-ordered passes pay on 3D single-class stencils (configs 3
    and 5: patch solve 2-3x, transport up to 3.5x, profiles/r2_banded_ab.jsonl);
    2D sweeps are too thin to hide the per-sweep latency (config 2: 16 -> 54
    ms) and the Dubins headings (config 4) span thousands of bands."""
    return plan.grid.dim == 3 and plan.stencils.n_classes == 1


def band_schedule(plan: StencilPlan, key_work: torch.Tensor, nodes: torch.Tensor, rule: str,
                  window, final_row: bool = False, scale: Optional[float] = None):
    """Block schedule of a value-ordered pass on the device (phj_band_count /
    phj_band_fill): CSR (band_list, band_off, n_band) of the warp blocks each
    sweep visits (phj_transport_args / phj_solve_args band fields).

    A node's band is floor(T / delta), T its lifted time-to-target (working
    field ``key_work``: v for Kruzkov, u for the reference rule), delta =
    BAND_SCALE x k / max|f| (the smallest time one SL step covers), widened so
    that at most BAND_CAP_PER_NODE x the longest axis bands exist; a block
    holding any of ``nodes`` (bool per internal serial) is relaxed at sweeps
    [min band - hi, max band + lo] of those nodes and copied to the other
    buffer one sweep later.  ``final_row`` appends row n_band with every
    scheduled block (the solve's first ordinary sweep).  Returns None when
    ``nodes`` is empty."""
    lo_w, hi_w = (int(x) for x in window)
    dev = plan.device
    lib = _lib.load()
    fmax = plan.eps_speed / 1.0e-12
    delta_min = (BAND_SCALE if scale is None else scale) * plan.grid.k_step / fmax
    max_bands = int(BAND_CAP_PER_NODE * max(plan.int_shape))
    nb = nodes.view(-1).to(torch.uint8).contiguous()
    scratch = torch.empty(int(lib.phj_band_scratch_bytes(ctypes_ref(plan.gs), max_bands, lo_w,
                                                          hi_w)),
                          dtype=torch.uint8, device=dev)
    out = (ctypes.c_int64 * 4)()
    dt = _lib.F32 if key_work.dtype == torch.float32 else _lib.F64
    kw = key_work.contiguous()
    _lib.check(lib.phj_band_count(ctypes_ref(plan.gs), dt, _rule_id(rule), _lib.ptr(kw),
                                  _lib.ptr(nb), delta_min, max_bands, lo_w, hi_w,
                                  _lib.ptr(scratch), out, _lib.stream_handle()), "band_count")
    entries, n_band, n_blocks = int(out[0]), int(out[1]), int(out[2])
    if n_blocks == 0:
        return None
    band_list = torch.empty(entries + (n_blocks if final_row else 0), dtype=torch.int32,
                            device=dev)
    band_off = torch.empty(n_band + (2 if final_row else 1), dtype=torch.int32, device=dev)
    _lib.check(lib.phj_band_fill(ctypes_ref(plan.gs), max_bands, lo_w, hi_w, n_band, n_blocks,
                                 int(final_row), _lib.ptr(scratch), _lib.ptr(band_list),
                                 _lib.ptr(band_off), _lib.stream_handle()), "band_fill")
    return band_list, band_off, n_band


def transport_bands(plan: StencilPlan, key_work: torch.Tensor, fb_int: torch.Tensor, rule: str,
                    window=None):
    """band_schedule over the transport's movers (feedback >= 0, free)."""
    mover = (fb_int.view(-1) >= 0) & (plan.kind.view(-1) == KIND_FREE)
    return band_schedule(plan, key_work, mover, rule, window or TRANSPORT_BAND_WINDOW,
                         scale=TRANSPORT_BAND_SCALE)


def transport_internal(plan: StencilPlan, fb_int: torch.Tensor, parts_flat: Sequence,
                       tol: float, max_sweeps: int, schedule: str = "jacobi",
                       phi_dtype: torch.dtype = torch.float64, bands=None):
    """All colours in one launch, each Jacobi to its own max|change| <= tol
    ("jacobi"), or asynchronously in place until no node changes a colour by
    more than TRANSPORT_ASYNC_FRAC * tol ("async").
    ``parts_flat``: per colour, internal ext flat indices of its part.
    ``phi_dtype`` float32 halves the colour fields' footprint (fp64
    accumulation either way; used for fp32 workloads).  ``bands``
    (transport_bands) prepends the value-ordered pass (Jacobi only); its
    sweeps count in the per-colour sweeps.
    Returns (phi [R][ext] tensor, R, per-colour sweeps, updates)."""
    lib = _lib.load()
    R = len(parts_flat)
    asyn = schedule == "async"
    phi0 = torch.zeros((R,) + plan.int_ext, dtype=phi_dtype, device=plan.device)
    # Jacobi: the second buffer zeroed and seeded like the first (a memset
    # instead of a clone: half the traffic at 35 GB per buffer on config 5)
    phi1 = phi0 if asyn else torch.zeros_like(phi0)
    # every colour's part in one scatter (one index set, one launch)
    sizes = [int(pf.numel()) for pf in parts_flat]
    col = torch.repeat_interleave(torch.arange(R, device=plan.device, dtype=torch.int32),
                                  torch.as_tensor(sizes, device=plan.device))
    seed_flat = torch.cat([pf.view(-1) for pf in parts_flat]).to(torch.int64).contiguous()
    phi0.view(R, -1)[col.long(), seed_flat] = 1.0
    if not asyn:
        phi1.view(R, -1)[col.long(), seed_flat] = 1.0
    if any(plan.gs.periodic[i] for i in range(plan.grid.dim)):
        for j in range(R):
            _sync_periodic(plan, phi0[j])
            if not asyn:
                _sync_periodic(plan, phi1[j])
    n_band = 0 if (bands is None or asyn) else int(bands[2])
    max_sweeps = max_sweeps + n_band
    wsb = lib.phj_solve_workspace_bytes(ctypes_ref(plan.gs), 1, max_sweeps)
    ws = torch.empty(int(wsb), dtype=torch.uint8, device=plan.device)
    mc = torch.zeros(max_sweeps * R, dtype=torch.float64, device=plan.device)
    csw = torch.zeros(R, dtype=torch.int32, device=plan.device)
    info = torch.zeros(4, dtype=torch.int32, device=plan.device)
    upd = torch.zeros(1, dtype=torch.int64, device=plan.device)
    a = _lib.TransportArgs()
    a.grid = plan.gs
    a.st = plan.stencil_struct()
    a.phi0 = _lib.ptr(phi0)
    a.phi1 = _lib.ptr(phi1)
    a.fb = _lib.ptr(fb_int)
    a.kind = _lib.ptr(plan.kind)
    ent = torch.empty(plan.grid.n_interior, dtype=torch.int32, device=plan.device)
    a.ent_scratch = _lib.ptr(ent)
    a.n_colors = R
    a.tol = tol
    a.act_eps = tol * (TRANSPORT_ASYNC_FRAC if asyn else TRANSPORT_ACT_FRAC)
    # a rank that transports a subset of the colours claims list entries in
    # pairs (most entries hold none of its colours; rank 0 of 8 at config 5:
    # 47.8 -> 36.5 ms, one GPU with all colours: 127 -> 130 ms)
    pairs = (not asyn) and dist.world()[1] > 1
    a.options = (_lib.TRANSPORT_ASYNC if asyn else 0) | (_lib.TRANSPORT_PAIRS if pairs else 0)
    a.inner_sweeps = TRANSPORT_INNER[plan.grid.dim]
    a.phi_dtype = _lib.F32 if phi_dtype == torch.float32 else _lib.F64
    # only blocks next to a part start active (exact; the library ignores the
    # seeds beyond 64 colours)
    a.seed_flat = _lib.ptr(seed_flat)
    a.seed_col = _lib.ptr(col)
    a.n_seed = int(seed_flat.numel())
    a.max_sweeps = max_sweeps
    if n_band:
        a.band_list = _lib.ptr(bands[0])
        a.band_off = _lib.ptr(bands[1])
        a.n_band = n_band
    a.workspace = _lib.ptr(ws)
    a.maxch_hist = _lib.ptr(mc)
    a.color_sweeps = _lib.ptr(csw)
    a.info = _lib.ptr(info)
    a.updates = _lib.ptr(upd)
    a.stream = _lib.stream_handle()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.phj_transport(ctypes_ref(a)), "phj_transport")
    e1.record()
    # one device->host copy for the counters (exact in fp64)
    pack = torch.cat([info.double(), csw.double(), upd.double()]).cpu().numpy()
    ih = pack[:4].astype(np.int64)
    phi = phi1 if int(ih[1]) == 1 else phi0
    from .solver import active_blocks_per_sweep

    TRANSPORT_DIAG["kernel_ms"] = e0.elapsed_time(e1)
    if _lib.DIAG:
        TRANSPORT_DIAG["block_counts"] = active_blocks_per_sweep(plan, ws, max_sweeps, int(ih[0]))
    return phi, R, [int(x) for x in pack[4:4 + R]], int(pack[4 + R])


def _transport_and_argmax(fplan: StencilPlan, fb: torch.Tensor, parts, color_tol: float,
                          limit: int, schedule: str = "jacobi", dtype: str = "float64",
                          key_work: Optional[torch.Tensor] = None, rule: str = "kruzkov"):
    """Transport of every colour + running argmax (patchy.py:183-219,
    251-256).  With several ranks each rank transports its own colours
    (dist.my_colours) and the argmax is merged exactly across ranks.
    Returns (best_val, best_idx, per-colour sweeps, updates)."""
    R = len(parts)
    rank, world = dist.world()
    mine = dist.my_colours(R, rank, world) if world > 1 else np.arange(R)
    n = fplan.grid.n_interior
    dev = fplan.device
    csw_all = torch.zeros(R, dtype=torch.int64, device=dev)
    upd = 0
    if len(mine):
        # all parts converted and copied to the device at once
        allp = np.concatenate([np.asarray(parts[j], dtype=np.int64) for j in mine])
        flat = fplan.user_serials_to_internal_flat(allp)
        bounds = np.cumsum([0] + [len(parts[j]) for j in mine])
        parts_flat = [flat[bounds[i]:bounds[i + 1]] for i in range(len(mine))]
        # the asynchronous transport pays in 2D (C2 15.0 -> 6.9 ms); in 3D the
        # one-plane blocks relax little per visit and it is slower (C3 48 ->
        # 58 ms), so 3D keeps the Jacobi transport
        tsched = schedule if (fplan.grid.dim == 2 or TRANSPORT_ASYNC_3D) else "jacobi"
        # fp32 workloads keep their colour fields in fp32 too (half the
        # footprint: 35 GB instead of 70 GB at config 5)
        pdt = torch.float32 if ((dtype == "float32" and TRANSPORT_PHI_FP32) or
                                TRANSPORT_PHI_FP32_ALWAYS) else torch.float64
        bands = None
        if (TRANSPORT_BANDED and tsched == "jacobi" and banded_applies(fplan) and
                key_work is not None):
            bands = transport_bands(fplan, key_work, fb, rule)
        phi, _, csw, upd = transport_internal(fplan, fb, parts_flat, color_tol, limit,
                                              tsched, pdt, bands=bands)
        best_val, best_idx = argmax_batched(fplan.gs, phi, len(mine), n, dev)
        del phi
        csw_all[torch.as_tensor(mine, device=dev)] = torch.as_tensor(csw, device=dev)
        if world > 1:
            best_idx = torch.as_tensor(mine, device=dev, dtype=torch.int32)[best_idx.long()]
    else:
        best_val = torch.zeros(n, dtype=torch.float64, device=dev)
        best_idx = torch.full((n,), R - 1, dtype=torch.int32, device=dev)
    if world > 1:
        dist.merge_argmax(best_val, best_idx, R)
        dist.sum_over_ranks(csw_all)
        u = dist.sum_over_ranks(torch.tensor([upd], dtype=torch.int64, device=dev))
        upd = int(u.item())
    return best_val, best_idx, [int(x) for x in csw_all.tolist()], upd


def argmax_stream(gs, phis, n_serial: int, device):
    """Running argmax over streamed single-colour fields (patchy.py:251-256)."""
    lib = _lib.load()
    best_val = torch.zeros(n_serial, dtype=torch.float64, device=device)
    best_idx = torch.zeros(n_serial, dtype=torch.int32, device=device)
    n_colors = 0
    for j, phi in phis:
        _lib.check(lib.phj_argmax_update(ctypes_ref(gs), _lib.ptr(phi), int(j),
                                         _lib.ptr(best_val), _lib.ptr(best_idx),
                                         _lib.stream_handle()), "argmax")
        n_colors = max(n_colors, int(j) + 1)
    return best_val, best_idx, n_colors


def argmax_batched(gs, phi: torch.Tensor, R: int, n_serial: int, device, quantum: float = 0.0):
    lib = _lib.load()
    best_val = torch.empty(n_serial, dtype=torch.float64, device=device)
    best_idx = torch.empty(n_serial, dtype=torch.int32, device=device)
    pdt = _lib.F32 if phi.dtype == torch.float32 else _lib.F64
    _lib.check(lib.phj_argmax_colors_t(ctypes_ref(gs), _lib.ptr(phi), pdt, R, float(quantum),
                                       _lib.ptr(best_val), _lib.ptr(best_idx),
                                       _lib.stream_handle()), "argmax")
    return best_val, best_idx


def assemble_internal(gs, best_val: torch.Tensor, best_idx: torch.Tensor, n_colors: int,
                      mask_serial: Optional[torch.Tensor], kind_serial: torch.Tensor,
                      n_serial: int, device, warnings=None):
    """Codes + majority repair + fallback + boundary + solve labels
    (patchy.py:258-300) after the argmax.  Returns (color, n_uncovered,
    boundary, lab)."""
    lib = _lib.load()
    stream = _lib.stream_handle()
    color = torch.empty(n_serial, dtype=torch.int32, device=device)
    mask_u8 = None if mask_serial is None else mask_serial.to(torch.uint8).contiguous()
    _lib.check(lib.phj_assemble_codes(ctypes_ref(gs), _lib.ptr(best_val), _lib.ptr(best_idx),
                                      _lib.ptr(mask_u8), _lib.ptr(kind_serial), _lib.ptr(color),
                                      stream), "codes")
    other = torch.empty_like(color)
    counters = torch.zeros(4, dtype=torch.int32, device=device)
    while True:
        _lib.check(lib.phj_assemble_repair(ctypes_ref(gs), _lib.ptr(color), _lib.ptr(other),
                                           n_colors, _lib.ptr(counters), stream), "repair")
        filled, n_open = counters[:2].tolist()
        color, other = other, color
        if n_open == 0 or filled == 0:
            break
    ext = tuple(int(gs.ext[i]) for i in range(gs.dim))
    lab = torch.full(ext, _lib.LAB_HARD, dtype=torch.int16, device=device)
    boundary = torch.empty(n_serial, dtype=torch.uint8, device=device)
    _lib.check(lib.phj_assemble_finish(ctypes_ref(gs), _lib.ptr(color), _lib.ptr(boundary),
                                       _lib.ptr(lab), _lib.ptr(counters), stream), "finish")
    n_unc = int(counters[2].item())
    if n_unc and warnings is not None:
        warnings.append(f"{n_unc} reachable nodes reached by no color; folded into patch 0")
    if any(gs.periodic[i] for i in range(gs.dim)):
        _lib.check(lib.phj_sync_periodic(ctypes_ref(gs), 2, _lib.ptr(lab), stream), "sync")
    return color, n_unc, boundary, lab


def ao3_tables(plan: StencilPlan, spec: ProblemSpec, fb_int: torch.Tensor, r: float):
    """Device tables of the conical control reduction AO3 (solver.py:446-476,
    patchy.py:353-356) for the patch solves: per node its feedback control
    (ext layout), per feedback control the allowed stencil entries (bitmask
    over the class-0 entry order, padding included) and the number of allowed
    admissible controls (candidate-evaluation count).  None when the control
    geometry is not unit-norm (the reference then keeps every control)."""
    cs = spec.control_set
    if not cs.is_unit:
        return None
    st = plan.stencils
    if st.n_classes != 1:
        raise ConfigurationError("conical reduction needs a single-class stencil")
    controls = np.asarray(cs.controls, dtype=float)
    thresh = np.cos(np.pi / r) - 1.0e-12
    pair_ok = controls @ controls.T >= thresh                      # [nc, nc]
    ctrl = st.ctrl[:st.nc].astype(np.int64)
    noct = st.oct_start.shape[1] - 1
    e0, e1 = int(st.oct_start[0, 0]), int(st.oct_start[0, noct])
    if e1 > 128:
        raise ConfigurationError("conical reduction supports at most 128 stencil entries")
    words = 1 if e1 <= 64 else 2
    adm = np.unique(ctrl[e0:e1])
    nc = controls.shape[0]
    mask = np.zeros((nc, words), dtype=np.uint64)
    for e in range(e0, e1):
        ok = pair_ok[:, ctrl[e]]
        mask[ok, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
    count = pair_ok[:, adm].sum(axis=1).astype(np.int32)
    dev = plan.device
    fbx = torch.full(plan.int_ext, -1, dtype=torch.int32, device=dev)
    plan.interior_int(fbx).copy_(fb_int.to(dev, torch.int32).view(plan.int_shape))
    _sync_periodic(plan, fbx)
    return (fbx, torch.as_tensor(mask.view(np.int64), device=dev),
            torch.as_tensor(count, device=dev), words)


def count_labels(color: torch.Tensor, n_labels: int) -> torch.Tensor:
    """Nodes per label 0..n_labels-1 of an int32 label vector (phj_count_labels
    on the device; a host-resident PatchMap is counted on the host)."""
    if not color.is_cuda:
        c = color.numpy()
        return torch.as_tensor(np.bincount(c[c >= 0], minlength=n_labels)[:n_labels])
    out = torch.empty(n_labels, dtype=torch.int64, device=color.device)
    c = color.to(torch.int32).contiguous()
    _lib.check(_lib.load().phj_count_labels(_lib.ptr(c), c.numel(), n_labels, _lib.ptr(out),
                                            _lib.stream_handle()), "count_labels")
    return out


def solve_patches_internal(plan: StencilPlan, color: torch.Tensor, lab: torch.Tensor,
                           n_patches: int, pcfg: PatchyConfig, cfg: SolverConfig,
                           lifted_work: Optional[torch.Tensor] = None,
                           work: Optional[torch.Tensor] = None, ao3=None):
    """All patches on the device (patchy.py:304-389).  `color` per internal
    serial.  Returns (working result, [SweepStats], warnings, performed)."""
    rule, dtype = cfg.rule, cfg.dtype
    dev = plan.device
    unr = unreached_value(rule)
    thr = unreach_threshold(rule)
    if work is None:
        work = init_working(plan, rule, dtype)
    inner_w = plan.interior_int(work)
    col3 = color.view(plan.int_shape)
    if pcfg.warm_start:
        lv = plan.interior_int(lifted_work)
        seed = torch.where(lv < thr, lv, torch.full_like(lv, unr))
        inner_w.copy_(torch.where(col3 >= 0, seed, inner_w))
        _sync_periodic(plan, work)
    sizes = count_labels(color, n_patches).cpu().numpy()
    cands = None  # AO3: candidates per sweep per patch (reduced control sets)
    if ao3 is not None:
        fbx, _, acount, _ = ao3
        fser = plan.interior_int(fbx).reshape(-1)
        per = torch.where(fser >= 0, acount[fser.clamp(min=0).long()],
                          torch.full_like(fser, plan.n_adm)).to(torch.float64)
        sel = color >= 0
        cands = torch.bincount(color[sel].long(), weights=per[sel],
                               minlength=n_patches)[:n_patches].cpu().numpy()
    rank, world = dist.world()
    # LPT weights: the per-patch executed evaluations the previous solve of
    # the same patch map measured (all ranks hold the same, summed over
    # ranks), else node counts (north_star)
    wkey = (tuple(int(x) for x in sizes), world)
    wcache = getattr(plan, "_patch_work", None)
    weights = wcache[1] if (wcache is not None and wcache[0] == wkey) else None
    mine = dist.mine_mask(sizes, rank, world, dev, weights)
    warnings = []
    stats = []
    performed = 0
    logical = 0
    executed = 0
    kernel_ms = 0.0
    sweeps_total = 0
    tiles_total = 0
    block_counts = None
    if pcfg.bc_mode == STATE_CONSTRAINT:
        fmask = plan.fmask_from_labels(lab)
        bands = None
        if (SOLVE_BANDED and lifted_work is not None and not pcfg.warm_start and
                banded_applies(plan) and cfg.schedule == "async"):
            nodes = (color >= 0) & (plan.kind.view(-1) == KIND_FREE)
            if mine is not None:
                nodes &= mine.bool()[color.clamp(min=0).long()]
            bands = band_schedule(plan, lifted_work, nodes, rule, SOLVE_BAND_WINDOW,
                                  final_row=True)
            if bands is not None:
                bands = (*bands, SOLVE_BAND_INNER)
        res = device_solve(plan, work, lab, fmask, n_patches, rule=rule, dtype=dtype, tol=cfg.tol,
                           ao3=ao3, bands=bands,
                           max_sweeps=cfg.sweep_limit(plan.grid), mine=mine,
                           act_tol=cfg.act_tol, schedule=cfg.schedule,
                           inner=cfg.inner_for(plan.grid.dim))
        out = res.values
        performed = res.real
        logical = res.evals
        executed = res.executed
        kernel_ms += res.device_ms
        sweeps_total = int(res.info[0])
        tiles_total = int(res.info[2])
        block_counts = res.block_counts
        for j in range(n_patches):
            if mine is not None and not bool(mine[j]):
                stats.append(SweepStats())
                continue
            stats.append(stats_for_patch(res, j, int(sizes[j]), plan.n_adm, cfg.tol,
                                         cands_per_sweep=None if cands is None else cands[j]))
    else:
        # Dirichlet: out-of-patch reads see the frozen lifted field with
        # UNREACHABLE forced to the sentinel (patchy.py:340-347); one launch per
        # patch since patches read different data at shared nodes.
        frozen = lifted_work.clone()
        fin = plan.interior_int(frozen)
        fin.copy_(torch.where(col3 == UNREACHABLE, torch.full_like(fin, unr), fin))
        fin.copy_(torch.where(plan.kind.view(plan.int_shape) == KIND_TARGET,
                              torch.zeros_like(fin), fin))
        _sync_periodic(plan, frozen)
        out = work.clone()
        for j in range(n_patches):
            if sizes[j] == 0 or (mine is not None and not bool(mine[j])):
                stats.append(SweepStats())
                continue
            own = col3 == j
            w = frozen.clone()
            wi = plan.interior_int(w)
            wi.copy_(torch.where(own, inner_w, wi))
            _sync_periodic(plan, w)
            labj = torch.full(plan.int_ext, _lib.LAB_FIXED, dtype=torch.int16, device=dev)
            li = plan.interior_int(labj)
            li.copy_(torch.where(own, torch.zeros_like(li), li))
            _sync_periodic(plan, labj)
            res = device_solve(plan, w, labj, plan.fmask_hard, 1, rule=rule, dtype=dtype, ao3=ao3,
                               tol=cfg.tol, max_sweeps=cfg.sweep_limit(plan.grid),
                               act_tol=cfg.act_tol, schedule=cfg.schedule,
                           inner=cfg.inner_for(plan.grid.dim))
            oi = plan.interior_int(out)
            oi.copy_(torch.where(own, plan.interior_int(res.values), oi))
            performed += res.real
            logical += res.evals
            executed += res.executed
            kernel_ms += res.device_ms
            sweeps_total += int(res.info[0])
            stats.append(stats_for_patch(res, 0, int(sizes[j]), plan.n_adm, cfg.tol,
                                         cands_per_sweep=None if cands is None else cands[j]))
        _sync_periodic(plan, out)
    if world > 1:
        dist.gather_min(out)
    if pcfg.bc_mode == STATE_CONSTRAINT and res.patch_counts is not None:
        work = torch.as_tensor(res.patch_counts[:, 2].astype(np.float64), device=dev)
        if world > 1:
            dist.sum_over_ranks(work)
        plan._patch_work = (wkey, work.cpu().numpy())
    for j, st in enumerate(stats):
        if st.warning:
            warnings.append(f"patch {j}: {st.warning}")
    # merge (patchy.py:384-388)
    oi = plan.interior_int(out)
    kind3 = plan.kind.view(plan.int_shape)
    oi.copy_(torch.where(kind3 == KIND_TARGET, torch.zeros_like(oi), oi))
    blocked = (col3 < 0) & (col3 != TARGET)
    oi.copy_(torch.where(blocked, torch.full_like(oi, unr), oi))
    _sync_periodic(plan, out)
    return out, stats, warnings, {"performed": performed, "logical": logical,
                                  "executed": executed,
                                  "kernel_ms": kernel_ms,
                                  "sweeps": sweeps_total, "tiles": tiles_total,
                                  "block_counts": block_counts}


# -- public API (reference signatures, user layout) -----------------------------------


def _coarse_spec(spec: ProblemSpec, target: Optional[TargetSpec]) -> ProblemSpec:
    return spec if target is None else dataclasses.replace(spec, target=target)


def coarse_solve_and_lift(spec: ProblemSpec, coarse_grid: Grid, fine_grid: Grid,
                          n_subdomains: int = 1, cfg: Optional[SolverConfig] = None,
                          strategy: Optional[ExecutionStrategy] = None, *,
                          fine_table: Optional[StencilPlan] = None,
                          stats: Optional[RunStats] = None, coarse_target=None):
    """Coarse solve, saturating lift, feedback on fine nodes (patchy.py:121-154).
    Returns (lifted NodeField, FeedbackField, coarse SweepStats)."""
    cfg = cfg or SolverConfig()
    stats = stats if stats is not None else RunStats()
    require_cuda()
    with stats.phase("coarse"):
        cplan = StencilPlan(coarse_grid, _coarse_spec(spec, coarse_target))
        vc, cst = solve_full_internal(cplan, coarse_cfg(cfg))
        stats.merge_counts(cst)
        if cst.warning:
            stats.warnings.append(cst.warning)
    with stats.phase("lift"):
        fplan = fine_table if fine_table is not None else StencilPlan(fine_grid, spec)
        vf = lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
        fb, ev = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
        stats.candidate_evals += int(ev.item())
    lifted = NodeField(fine_grid, fplan.user_from_working(vf, cfg.rule, cfg.dtype))
    return lifted, FeedbackField(fine_grid, spec.control_set, fplan.serial_to_user(fb)), cst


def mask_unreachable(lifted: NodeField, threshold: Optional[float] = None) -> torch.Tensor:
    """Interior mask of coarse-unreachable nodes (patchy.py:157-162)."""
    if threshold is None:
        threshold = 0.5 * lifted.sentinel
    idx = torch.as_tensor(lifted.grid.interior_flat(), device=lifted.values.device)
    return lifted.flat[idx] >= threshold


def transport_color(spec: ProblemSpec, grid: Grid, feedback: FeedbackField, part_serials,
                    color_tol: float = 1.0e-2, *, table: Optional[StencilPlan] = None,
                    max_sweeps: Optional[int] = None, feet=None):
    """Membership fraction of one target part transported upstream
    (patchy.py:183-219), Jacobi on the device.  Returns (NodeField, sweeps,
    updates, warning | None)."""
    plan = table if table is not None else StencilPlan(grid, spec)
    fb_int = plan.serial_to_internal(torch.as_tensor(feedback.indices, device=plan.device,
                                                     dtype=torch.int32)).contiguous()
    part_flat = plan.user_serials_to_internal_flat(np.asarray(part_serials, dtype=np.int64))
    limit = max_sweeps if max_sweeps is not None else 10 * max(grid.shape)
    phi, _, csw, upd = transport_internal(plan, fb_int, [part_flat], color_tol, limit)
    sweeps = abs(csw[0])
    warning = None if csw[0] > 0 else (f"color transport: no convergence after {sweeps} sweeps "
                                       f"(color_tol {color_tol:.1e})")
    phi = phi.view(plan.int_ext)
    return NodeField(grid, plan.to_user(phi), sentinel=SENTINEL), sweeps, upd, warning


def assemble_patches(color_fields, mask, grid: Grid, *, kind, warnings: Optional[list] = None
                     ) -> PatchMap:
    """Project streamed colour fields onto one patch map (patchy.py:236-301)."""
    require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    gs = grid.device_struct()
    kind_t = torch.as_tensor(np.asarray(kind.cpu() if isinstance(kind, torch.Tensor) else kind),
                             device=dev).to(torch.int8)
    mask_t = None
    if mask is not None:
        mask_t = torch.as_tensor(mask.cpu().numpy() if isinstance(mask, torch.Tensor)
                                 else np.asarray(mask), device=dev)

    def stream():
        for j, phi in color_fields:
            vals = phi.values if isinstance(phi, NodeField) else phi
            yield j, torch.as_tensor(vals, device=dev, dtype=torch.float64).contiguous()

    best_val, best_idx, n_colors = argmax_stream(gs, stream(), grid.n_interior, dev)
    color, n_unc, boundary, _ = assemble_internal(gs, best_val, best_idx, n_colors, mask_t,
                                                  kind_t, grid.n_interior, dev, warnings)
    unc = np.empty(0, dtype=np.int64)
    if n_unc:
        unc = np.arange(n_unc)  # count-only; serials are not tracked on the device
    return PatchMap(grid, n_colors, color, None, boundary.bool(), unc)


def solve_patches(spec: ProblemSpec, grid: Grid, patch_map: PatchMap, lifted: NodeField,
                  pcfg: PatchyConfig, cfg: Optional[SolverConfig] = None,
                  strategy: Optional[ExecutionStrategy] = None, *,
                  table: Optional[StencilPlan] = None, feedback: Optional[FeedbackField] = None,
                  field: Optional[NodeField] = None):
    """Independent patch solves merged into one field (patchy.py:304-389).
    Returns (NodeField, list[SweepStats], warnings)."""
    cfg = cfg or SolverConfig()
    if pcfg.reduction is not None and feedback is None:
        raise ConfigurationError("conical reduction needs a feedback field")
    plan = table if table is not None else StencilPlan(grid, spec)
    ao3 = None
    if pcfg.reduction is not None:
        fi = feedback.indices
        fi = fi if isinstance(fi, torch.Tensor) else torch.as_tensor(np.asarray(fi))
        fb_int = plan.serial_to_internal(fi.to(plan.device, torch.int32)).contiguous()
        ao3 = ao3_tables(plan, spec, fb_int, float(pcfg.reduction))
    color_int = plan.serial_to_internal(patch_map.color.to(plan.device)).contiguous()
    lab = torch.full(plan.int_ext, _lib.LAB_HARD, dtype=torch.int16, device=plan.device)
    li = plan.interior_int(lab)
    c3 = color_int.view(plan.int_shape)
    li.copy_(torch.where(c3 >= 0, c3.to(torch.int16),
                         torch.where(c3 == TARGET, torch.full_like(li, _lib.LAB_TARGET),
                                     torch.full_like(li, _lib.LAB_HARD))))
    _sync_periodic(plan, lab)
    lw = plan.working_from_user(lifted.values, cfg.rule, cfg.dtype)
    work = None if field is None else plan.working_from_user(field.values, cfg.rule, cfg.dtype)
    out, stats, warnings, _ = solve_patches_internal(plan, color_int, lab, patch_map.n_patches,
                                                     pcfg, cfg, lw, work, ao3=ao3)
    res = NodeField(grid, plan.user_from_working(out, cfg.rule, cfg.dtype))
    if field is not None:
        field.values.copy_(res.values)
        res = field
    return res, stats, warnings


def make_plans(spec: ProblemSpec, pcfg: PatchyConfig):
    """(fine plan, coarse plan) for run_patchy -- the 'tables' phase."""
    fplan = StencilPlan(spec.make_grid(pcfg.fine_nodes), spec)
    cplan = StencilPlan(spec.make_grid(pcfg.coarse_nodes), _coarse_spec(spec, pcfg.coarse_target))
    return fplan, cplan


def run_patchy(spec: ProblemSpec, pcfg: PatchyConfig, cfg: Optional[SolverConfig] = None,
               strategy: Optional[ExecutionStrategy] = None, *, plans=None,
               outputs: bool = True) -> PatchyResult:
    """Full pipeline on the device (patchy.py:405-467).  ``plans`` reuses
    prebuilt (fine, coarse) StencilPlans; ``outputs=False`` skips building
    the user-layout lifted/feedback/patch-map outputs (value only)."""
    cfg = cfg or SolverConfig()
    require_cuda()
    stats = RunStats()
    rule, dtype = cfg.rule, cfg.dtype
    with stats.phase("tables"):
        fplan, cplan = plans if plans is not None else make_plans(spec, pcfg)
    fine_grid = fplan.grid
    with stats.phase("coarse"):
        vc, cst = solve_full_internal(cplan, coarse_cfg(cfg))
        stats.merge_counts(cst)
        if cst.warning:
            stats.warnings.append(cst.warning)
    with stats.phase("lift"):
        vf = lift_internal(cplan, vc, fplan, rule, dtype)
        fb, ev = feedback_sharded(fplan, vf, rule=rule, dtype=dtype)
    transport_sweeps = []
    with stats.phase("transport"):
        ut = pcfg.unreachable_threshold
        if ut is not None and np.isinf(ut):
            mask = None  # mask disabled (patchy.py:58-62)
        else:
            thr = unreach_threshold(rule) if ut is None else (
                ut if rule == "reference" else float(-np.expm1(-ut)))
            mask = plan_interior_serial(fplan, vf) >= thr
        parts = _resolve_parts(pcfg, spec, fine_grid, fplan)
        limit = pcfg.transport_max_sweeps or 10 * max(fine_grid.shape)
        n_colors = len(parts)
        best_val, best_idx, csw, upd = _transport_and_argmax(fplan, fb, parts, pcfg.color_tol,
                                                             limit, cfg.schedule, cfg.dtype,
                                                             key_work=vf, rule=rule)
        stats.transport_updates += upd
        transport_sweeps = [abs(x) for x in csw]
        for j, x in enumerate(csw):
            if x <= 0:
                stats.warnings.append(f"color {j}: color transport: no convergence after "
                                      f"{abs(x)} sweeps (color_tol {pcfg.color_tol:.1e})")
        color, n_unc, boundary, lab = assemble_internal(
            fplan.gs, best_val, best_idx, n_colors, mask, fplan.kind, fine_grid.n_interior,
            fplan.device, stats.warnings)
    with stats.phase("patch_solve"):
        ao3 = (ao3_tables(fplan, spec, fb, float(pcfg.reduction))
               if pcfg.reduction is not None else None)
        out, pstats, warnings, pinfo = solve_patches_internal(
            fplan, color, lab, n_colors, pcfg, cfg, vf, ao3=ao3)
        stats.warnings.extend(warnings)
        for st in pstats:
            stats.merge_counts(st)
        stats.kernels["patch_solve"] = pinfo
    stats.candidate_evals += int(ev.item())
    value = NodeField(fine_grid, fplan.user_from_working(out, rule, dtype))
    if not outputs:
        stats.finalize()
        return PatchyResult(value, None, None, None, stats, cst, pstats, transport_sweeps)
    pm = PatchMap(fine_grid, n_colors, fplan.serial_to_user(color), None,
                  fplan.serial_to_user(boundary).bool(),
                  np.arange(n_unc) if n_unc else np.empty(0, dtype=np.int64))
    imb = pm.imbalance_warning()
    if imb:
        stats.warnings.append(imb)
    lifted = NodeField(fine_grid, fplan.user_from_working(vf, rule, dtype))
    feedback = FeedbackField(fine_grid, spec.control_set, fplan.serial_to_user(fb))
    stats.finalize()
    return PatchyResult(value, pm, lifted, feedback, stats, cst, pstats, transport_sweeps)


def plan_interior_serial(plan: StencilPlan, w: torch.Tensor) -> torch.Tensor:
    """Interior values of an internal ext tensor, flattened in internal serial order."""
    return plan.interior_int(w).reshape(-1)


def _resolve_parts(pcfg: PatchyConfig, spec: ProblemSpec, grid: Grid, plan=None):
    """Target partition; the target serials come from the device
    classification so only target points are formed on the host (cached on
    the plan)."""
    if pcfg.parts is not None and not callable(pcfg.parts):
        return [np.asarray(p, dtype=np.int64) for p in pcfg.parts]
    # the callable itself is the key (kept alive by the cache): an id() of a
    # collected callable could be reused by a new one
    key = ("parts", pcfg.parts, pcfg.n_patches)
    cache = getattr(plan, "_parts_cache", None) if plan is not None else None
    if cache is not None and key in cache:
        return cache[key]
    serials = None
    if plan is not None:
        kind_user = plan.serial_to_user(plan.kind)
        ser_t = torch.nonzero(kind_user == KIND_TARGET).view(-1)
        dev = device_partition_codes(pcfg.parts, spec.target, grid, ser_t)
        if dev is not None:
            # built-in partitions on the device: one copy of (serials, codes)
            n_parts, code = dev
            # grouped on the device (stable sort by part keeps the serial
            # order inside a part), one copy of (serials, part sizes)
            _, perm = torch.sort(code, stable=True)
            packed = torch.cat([ser_t.to(torch.int64)[perm],
                                torch.bincount(code, minlength=n_parts)]).cpu().numpy()
            bounds = np.cumsum(packed[ser_t.numel():])[:-1]
            parts = np.split(packed[:ser_t.numel()], bounds)
            _check_parts(parts, n_parts)
            if cache is None:
                plan._parts_cache = cache = {}
            cache[key] = parts
            return parts
        serials = ser_t.cpu().numpy()
    if pcfg.parts is None:
        parts = partition_target(spec.target, grid, pcfg.n_patches, serials=serials)
    else:
        try:
            parts = pcfg.parts(spec.target, grid, serials=serials)
        except TypeError:
            parts = pcfg.parts(spec.target, grid)
    if plan is not None:
        if cache is None:
            plan._parts_cache = cache = {}
        cache[key] = parts
    return parts
