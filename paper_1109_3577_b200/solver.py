"""Semi-Lagrangian value iteration on the device (mirror of patchyhjb.solver,
solver.py:1-476).

``solve`` keeps the reference signature and semantics (node_set, active,
frozen, hard; monotone writes; stop at max change <= tol; warning on the
sweep cap) but runs the whole loop on the GPU as one cooperative launch of
``phj_solve``: a Jacobi iteration (the reference sweeps Gauss-Seidel; both
reach the same fixed point) with exact tile-activity skipping.

Two switches the reference lacks (``SolverConfig``):
  ``rule``  "reference" -- u <- min_a I[u](x + h f) + h, sentinel 1e9
            (_kernels.py:70-105) -- or "kruzkov" -- v <- min_a beta I[v] + 1 -
            beta, beta = e^{-h}, v = 1 - e^{-T} (BASELINE north_star).  Fields
            crossing the API are always in T units with the sentinel, as in
            the reference; Kruzkov values are converted at the boundary.
  ``dtype`` "float64" or "float32" (Kruzkov only).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as _field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .dynamics import COST_CTRL, COST_NODE, plan_stencils
from .grid import SENTINEL, ConfigurationError, Grid, NodeField, require_cuda
from .problems import ProblemSpec
from .runtime import ExecutionStrategy

LEXICOGRAPHIC = "lexicographic"
BY_VALUE = "by-value"
STATE_CONSTRAINT = "state-constraint"
DIRICHLET = "dirichlet"
KIND_FREE, KIND_TARGET, KIND_OBSTACLE = 0, 1, 2
RULES = ("reference", "kruzkov")
DTYPES = ("float64", "float32")


@dataclass
class SolverConfig:
    """Knobs of the value iteration (solver.py:45-76) + ``rule`` / ``dtype``."""

    tol: float = 1.0e-6
    max_sweeps: Optional[int] = None
    bc_mode: str = STATE_CONSTRAINT
    sweep_order: str = LEXICOGRAPHIC
    control_reduction: Optional[float] = None
    warm_start: bool = False
    rule: str = "reference"
    dtype: str = "float64"
    #: device activity threshold in time units: changes at or
    #: below it re-sweep their own block only; 0 = exact Jacobi activity.
    #: None: 1e-12 in fp64, 1e-7 in fp32 (about one ulp of v)
    activity_tol: Optional[float] = None
    #: device iteration: "jacobi" (barrier-separated sweeps, per-patch
    #: stopping at max change <= tol) or "async" (chaotic relaxation to within
    #: activity_tol)
    schedule: str = "jacobi"
    #: block-local relaxations per block visit (None: 1 for "jacobi"; for
    #: "async" 7 in 2D, 3 in 3D -- measured best)
    inner_sweeps: Optional[int] = None

    def __post_init__(self):
        if self.bc_mode not in (STATE_CONSTRAINT, DIRICHLET):
            raise ConfigurationError(f"unknown bc_mode {self.bc_mode!r}")
        if self.sweep_order not in (LEXICOGRAPHIC, BY_VALUE):
            raise ConfigurationError(f"unknown sweep_order {self.sweep_order!r}")
        if self.tol <= 0.0:
            raise ConfigurationError("tol must be positive")
        if self.max_sweeps is not None and self.max_sweeps < 1:
            raise ConfigurationError("max_sweeps must be at least 1")
        if self.control_reduction is not None and self.control_reduction <= 1.0:
            raise ConfigurationError("control_reduction factor must exceed 1")
        if self.rule not in RULES:
            raise ConfigurationError(f"unknown rule {self.rule!r}")
        if self.dtype not in DTYPES:
            raise ConfigurationError(f"unknown dtype {self.dtype!r}")
        if self.schedule not in ("jacobi", "async"):
            raise ConfigurationError(f"unknown schedule {self.schedule!r}")
        if self.inner_sweeps is not None and self.inner_sweeps < 1:
            raise ConfigurationError("inner_sweeps must be at least 1")
        if self.activity_tol is not None and not self.activity_tol >= 0.0:
            raise ConfigurationError("activity_tol must be >= 0")
        if self.rule == "reference" and self.dtype != "float64":
            raise ConfigurationError("the sentinel (reference) rule is float64 only")

    @property
    def act_tol(self) -> float:
        if self.activity_tol is not None:
            return float(self.activity_tol)
        return 1.0e-12 if self.dtype == "float64" else 1.0e-7

    def inner_for(self, dim: int) -> int:
        if self.inner_sweeps is not None:
            return int(self.inner_sweeps)
        return 1 if self.schedule == "jacobi" else (7 if dim == 2 else 3)

    def sweep_limit(self, grid: Grid) -> int:
        return self.max_sweeps if self.max_sweeps is not None else 10 * max(grid.shape)


@dataclass
class SweepStats:
    """Outcome of one solve (solver.py:79-88).  ``node_relaxations`` and
    ``candidate_evals`` (admissible controls of every relaxation, the
    reference's count, _kernels.py:76) are counted per patch by the device
    under both schedules; ``performed_evals`` are the candidate evaluations
    the device really executed (after activity skipping and the exact octant
    pruning).  Asynchronous solves report ``sweeps`` as equivalent sweeps
    (node relaxations / patch nodes) and keep no per-sweep max change
    (``max_change`` is NaN: ``tol`` does not apply, ``activity_tol`` does)."""

    sweeps: int = 0
    node_relaxations: int = 0
    candidate_evals: int = 0
    converged: bool = True
    max_change: float = 0.0
    warning: Optional[str] = None
    performed_evals: int = 0


@dataclass
class FeedbackField:
    """Discrete argmin control per interior serial, -1 = none (solver.py:400-410)."""

    grid: Grid
    control_set: object
    indices: torch.Tensor

    def control_vector(self, serial: int):
        c = int(self.indices[serial])
        return None if c < 0 else self.control_set.controls[c]


def _rule_id(rule: str) -> int:
    return _lib.RULE_KRUZKOV if rule == "kruzkov" else _lib.RULE_REF


def _dtype_id(dtype: str) -> int:
    return _lib.F32 if dtype == "float32" else _lib.F64


def _torch_dtype(dtype: str):
    return torch.float32 if dtype == "float32" else torch.float64


def unreached_value(rule: str) -> float:
    return 1.0 if rule == "kruzkov" else SENTINEL


def unreach_threshold(rule: str) -> float:
    return 1.0 if rule == "kruzkov" else 0.5 * SENTINEL


class StencilPlan:
    """Device-resident problem plan: the counterpart of the reference's
    ``CandidateTable`` (solver.py:140-198), without per-(node, control) data.

    Holds the stencil tables, per-node kinds, the ghost/obstacle hard mask
    and its foreign masks, and per-(rule, dtype) node coefficients, all in
    the internal axis order (``perm``)."""

    def __init__(self, grid: Grid, spec: ProblemSpec, model=None):
        if spec.dim != grid.dim:
            raise ConfigurationError("grid/problem dimension mismatch")
        self.grid = grid
        self.spec = spec
        self.device = require_cuda()
        lib = _lib.load()
        self.stencils, self.node_speed, self.eps_speed = plan_stencils(grid, spec, model)
        st = self.stencils
        self.perm = st.perm
        self.inv_perm = tuple(int(i) for i in np.argsort(self.perm))
        self.identity = self.perm == tuple(range(grid.dim))
        self.gs = grid.device_struct(self.perm)
        self.int_shape = tuple(grid.shape[p] for p in self.perm)
        self.int_ext = tuple(grid.ext_shape[p] for p in self.perm)
        dev = self.device
        # the stencil tables in ONE host->device copy (fp64 parts first: aligned)
        parts = [np.ascontiguousarray(st.weights.ravel(), dtype=np.float64),
                 np.ascontiguousarray(st.cost, dtype=np.float64),
                 np.ascontiguousarray(st.oct_start.ravel(), dtype=np.int32),
                 np.ascontiguousarray(st.ctrl, dtype=np.int32),
                 np.ascontiguousarray(st.nzmask.view(np.int32))]
        blob = torch.as_tensor(np.concatenate([q.view(np.uint8) for q in parts])).to(dev)
        views, off = [], 0
        for q, tdt in zip(parts, (torch.float64, torch.float64, torch.int32, torch.int32,
                                  torch.int32)):
            views.append(blob[off:off + q.nbytes].view(tdt))
            off += q.nbytes
        self.d_w, self.d_cost, self.d_oct, self.d_ctrl, self.d_nz = views
        self.n_adm = int(st.n_real)
        self.kind = self._classify(lib)
        # hard base = ghost + obstacle (solver.py:111-126); periodic ghosts copy
        hard = torch.ones(self.int_ext, dtype=torch.uint8, device=dev)
        inner = hard[tuple(slice(1, -1) for _ in range(grid.dim))]
        inner.copy_((self.kind.view(self.int_shape) == KIND_OBSTACLE).to(torch.uint8))
        _lib.check(lib.phj_sync_periodic(ctypes_ref(self.gs), 1, _lib.ptr(hard),
                                         _lib.stream_handle()), "sync_periodic")
        self.hard = hard
        self.fmask_hard = self.fmask_from_hard(hard)
        self._coef: dict = {}

    # -- layout helpers ---------------------------------------------------------

    def to_internal(self, t: torch.Tensor) -> torch.Tensor:
        """User-layout ext (or interior-shaped) tensor -> internal layout."""
        return t if self.identity else t.permute(self.perm).contiguous()

    def to_user(self, t: torch.Tensor) -> torch.Tensor:
        return t if self.identity else t.permute(self.inv_perm).contiguous()

    def serial_to_user(self, t: torch.Tensor) -> torch.Tensor:
        """Per-internal-serial vector -> per-user-serial vector."""
        if self.identity:
            return t
        return t.view(self.int_shape).permute(self.inv_perm).reshape(-1).contiguous()

    def serial_to_internal(self, t: torch.Tensor) -> torch.Tensor:
        if self.identity:
            return t
        return t.view(self.grid.shape).permute(self.perm).reshape(-1).contiguous()

    def user_serials_to_internal_flat(self, serials: np.ndarray) -> torch.Tensor:
        """User interior serials -> internal ext flat indices."""
        idx = np.unravel_index(np.asarray(serials, dtype=np.int64), self.grid.shape)
        flat = np.zeros(len(idx[0]), dtype=np.int64)
        strides = [self.gs.strides[i] for i in range(self.grid.dim)]
        for i, p in enumerate(self.perm):
            flat += (idx[p] + 1) * strides[i]
        return torch.as_tensor(flat, device=self.device)

    def interior_int(self, t: torch.Tensor) -> torch.Tensor:
        return t[tuple(slice(1, -1) for _ in range(self.grid.dim))]

    # -- device data ----------------------------------------------------------------

    def _classify(self, lib) -> torch.Tensor:
        spec, grid = self.spec, self.grid
        d = grid.dim
        kind = torch.empty(grid.n_interior, dtype=torch.int8, device=self.device)
        tgt = spec.target
        balls, planes = [], []
        host_mask = None
        def ball_row(c):
            c = np.asarray(c, dtype=float).ravel()
            return list(c) + [0.0] * (3 - c.size) + [float(tgt.radius), float(c.size)]

        if tgt.kind == "ball":
            balls.append(ball_row(tgt.center))
        elif tgt.kind == "balls":
            for c in tgt.centers:
                balls.append(ball_row(c))
        elif tgt.kind == "plane":
            planes.append([float(tgt.axis), tgt.offset, tgt.plane_tol()])
        else:
            host_mask = tgt.contains(grid.interior_points())
        circ, boxes = [], []
        obs = spec.obstacles
        if obs is not None:
            for center, radius in obs.circles:
                c = np.asarray(center, dtype=float)
                circ.append(list(c) + [0.0] * (3 - c.size) + [float(radius), float(c.size)])
            for lo, hi in obs.boxes:
                lo = np.asarray(lo, dtype=float)
                hi = np.asarray(hi, dtype=float)
                boxes.append([float(lo.size)] + list(lo) + [0.0] * (3 - lo.size) + list(hi) +
                             [0.0] * (3 - hi.size))
        if len(balls) > 16 or len(circ) > 8 or len(boxes) > 8:
            raise ConfigurationError("too many analytic target/obstacle shapes for the device")
        hb = np.ascontiguousarray(np.array(balls, dtype=float).ravel()) if balls else np.zeros(1)
        hp = np.ascontiguousarray(np.array(planes, dtype=float).ravel()) if planes else np.zeros(1)
        hc = np.ascontiguousarray(np.array(circ, dtype=float).ravel()) if circ else np.zeros(1)
        hx = np.ascontiguousarray(np.array(boxes, dtype=float).ravel()) if boxes else np.zeros(1)
        sh = _lib.Shapes(len(balls), hb.ctypes.data, len(planes), hp.ctypes.data, len(circ),
                         hc.ctypes.data, len(boxes), hx.ctypes.data)
        ua = np.ascontiguousarray(np.array(self.perm, dtype=np.int32))
        _lib.check(lib.phj_classify(ctypes_ref(self.gs), ctypes_ref(sh), ua.ctypes.data,
                                    _lib.ptr(kind), _lib.stream_handle()), "classify")
        if host_mask is not None:
            hm = torch.as_tensor(host_mask, device=self.device)
            hm = self.serial_to_internal(hm)
            kind = torch.where((kind == KIND_OBSTACLE), kind,
                               torch.where(hm, torch.ones_like(kind), kind))
        return kind

    def fmask_from_hard(self, hard_int_ext: torch.Tensor) -> torch.Tensor:
        lib = _lib.load()
        fm = torch.zeros(self.int_ext, dtype=torch.int32, device=self.device)
        _lib.check(lib.phj_fmask_from_hard(ctypes_ref(self.gs), _lib.ptr(hard_int_ext),
                                           _lib.ptr(fm), _lib.stream_handle()), "fmask")
        return fm

    def fmask_from_labels(self, lab: torch.Tensor) -> torch.Tensor:
        lib = _lib.load()
        fm = torch.zeros(self.int_ext, dtype=torch.int32, device=self.device)
        _lib.check(lib.phj_fmask_from_labels(ctypes_ref(self.gs), _lib.ptr(lab), _lib.ptr(fm),
                                             _lib.stream_handle()), "fmask")
        return fm

    def stencil_struct(self) -> _lib.Stencil:
        st = self.stencils
        return _lib.Stencil(st.dim, st.n_classes, st.nc, st.cost_mode, int(st.n_real), 0,
                            _lib.ptr(self.d_oct),
                            _lib.ptr(self.d_ctrl), _lib.ptr(self.d_nz), _lib.ptr(self.d_w),
                            _lib.ptr(self.d_cost))

    def coef(self, rule: str, dtype: str):
        """(per-node coefficient tensor or None, scalar coef0)."""
        if self.stencils.cost_mode == COST_CTRL:
            return None, 1.0
        ns = self.node_speed
        if ns.kind == 0 and ns.c0 * ns.ctrl_norm >= ns.eps:
            h = self.grid.k_step / (abs(ns.c0) * ns.ctrl_norm)
            return None, (float(np.exp(-h)) if rule == "kruzkov" else h)
        key = (rule, dtype)
        if key not in self._coef:
            lib = _lib.load()
            c = torch.zeros(self.int_ext, dtype=_torch_dtype(dtype), device=self.device)
            sp_t = None
            if ns.kind == 1:
                sp_t = self.serial_to_internal(
                    torch.as_tensor(np.asarray(ns.speed, dtype=float), device=self.device))
            m = _lib.SpeedModel(ns.kind, ns.c0, ns.amp, (ctypes_double3(ns.omega)), ns.ctrl_norm,
                                ns.eps, _lib.ptr(sp_t))
            ua = np.ascontiguousarray(np.array(self.perm, dtype=np.int32))
            _lib.check(lib.phj_node_coef(ctypes_ref(self.gs), ctypes_ref(m), ua.ctypes.data,
                                         _dtype_id(dtype), _rule_id(rule), _lib.ptr(c),
                                         _lib.stream_handle()), "node_coef")
            self._coef[key] = c
        return self._coef[key], 1.0

    # -- field conversions ------------------------------------------------------------

    def working_from_user(self, values: torch.Tensor, rule: str, dtype: str) -> torch.Tensor:
        """User T-field (ext, float64) -> internal working field (fresh tensor)."""
        t = self.to_internal(values)
        if rule == "reference":
            out = t.clone() if t is values else t
        else:
            lib = _lib.load()
            out = torch.empty(self.int_ext, dtype=_torch_dtype(dtype), device=self.device)
            tt = t.contiguous()
            _lib.check(lib.phj_to_kruzkov(tt.numel(), _dtype_id(dtype), _lib.ptr(tt),
                                          _lib.ptr(out), 0.5 * SENTINEL, _lib.stream_handle()),
                       "to_kruzkov")
        if self.grid.periodic[self.perm[0]]:
            _lib.check(_lib.load().phj_sync_periodic(ctypes_ref(self.gs), out.element_size(),
                                                     _lib.ptr(out), _lib.stream_handle()),
                       "sync_periodic")
        return out

    def user_from_working(self, w: torch.Tensor, rule: str, dtype: str) -> torch.Tensor:
        """Internal working field -> user T-field (ext, float64)."""
        if rule == "reference":
            t = w
        else:
            lib = _lib.load()
            t = torch.empty(self.int_ext, dtype=torch.float64, device=self.device)
            _lib.check(lib.phj_from_kruzkov(w.numel(), _dtype_id(dtype), _lib.ptr(w),
                                            _lib.ptr(t), SENTINEL, _lib.stream_handle()),
                       "from_kruzkov")
        return self.to_user(t)


#: API alias: the reference passes ``table=CandidateTable(grid, spec)``.
CandidateTable = StencilPlan


def ctypes_ref(s):
    import ctypes

    return ctypes.byref(s)


def ctypes_double3(v):
    import ctypes

    arr = (ctypes.c_double * 3)()
    for i, x in enumerate(list(v)[:3]):
        arr[i] = float(x)
    return arr


def classify_nodes(grid: Grid, spec: ProblemSpec) -> np.ndarray:
    """Per-user-serial node kind: free / target / obstacle (solver.py:101-108)."""
    pts = grid.interior_points()
    kind = np.zeros(grid.n_interior, dtype=np.uint8)
    kind[spec.target.contains(pts)] = KIND_TARGET
    if spec.obstacles is not None:
        kind[spec.obstacles.contains(pts)] = KIND_OBSTACLE
    return kind


def init_value_field(grid: Grid, spec: ProblemSpec, kind=None) -> NodeField:
    """Sentinel-initialised field with 0 on target nodes (solver.py:129-137)."""
    field = NodeField(grid)
    if kind is None:
        kind = classify_nodes(grid, spec)
    kind = kind.cpu().numpy() if isinstance(kind, torch.Tensor) else np.asarray(kind)
    idx = torch.as_tensor(grid.interior_flat()[kind == KIND_TARGET], device=field.values.device)
    field.flat[idx] = 0.0
    return field


@dataclass
class DeviceSolveResult:
    values: torch.Tensor           # working field holding the result (internal)
    patch_sweeps: np.ndarray       # per patch, negative = not converged
    last_change: np.ndarray        # [R] max change of each patch's last sweep (Jacobi)
    evals: int
    info: np.ndarray
    device_ms: float = 0.0
    block_counts: Optional[np.ndarray] = None
    executed: int = 0              # stencil-entry evaluations run (after octant pruning)
    real: int = 0                  # real candidate evaluations executed (no padding)
    patch_counts: Optional[np.ndarray] = None  # [R, 3] relaxations, logical, real evals
    schedule: str = "jacobi"


def device_solve(plan: StencilPlan, work: torch.Tensor, lab: torch.Tensor, fmask: torch.Tensor,
                 n_patches: int, *, rule: str, dtype: str, tol: float, max_sweeps: int,
                 mine: Optional[torch.Tensor] = None, sync: bool = True,
                 prune: bool = True, ao3=None, act_tol: float = 0.0,
                 schedule: str = "jacobi", inner: int = 1, bands=None) -> DeviceSolveResult:
    """One phj_solve launch: all patches of `lab`, to per-patch convergence.
    ``bands`` (patchy.band_schedule) prepends the value-ordered pass."""
    lib = _lib.load()
    dev = plan.device
    n_band = 0 if bands is None else int(bands[2])
    max_sweeps = max_sweeps + (n_band + 1 if n_band else 0)
    v1 = work.clone()
    wsb = lib.phj_solve_workspace_bytes(ctypes_ref(plan.gs), n_patches, max_sweeps)
    ws = torch.empty(int(wsb), dtype=torch.uint8, device=dev)
    ps = torch.zeros(n_patches, dtype=torch.int32, device=dev)
    mc = torch.zeros(max_sweeps * n_patches, dtype=torch.float64, device=dev)
    ev = torch.zeros(3, dtype=torch.int64, device=dev)
    pc = torch.zeros((n_patches, 3), dtype=torch.int64, device=dev)
    info = torch.zeros(4, dtype=torch.int32, device=dev)
    coef, coef0 = plan.coef(rule, dtype)
    a = _lib.SolveArgs()
    a.grid = plan.gs
    a.st = plan.stencil_struct()
    a.dtype = _dtype_id(dtype)
    a.rule = _rule_id(rule)
    a.v0 = _lib.ptr(work)
    a.v1 = _lib.ptr(v1)
    a.lab = _lib.ptr(lab)
    a.fmask = _lib.ptr(fmask)
    a.coef = _lib.ptr(coef)
    a.coef0 = coef0
    a.n_patches = n_patches
    a.max_sweeps = max_sweeps
    a.mine = _lib.ptr(mine)
    a.tol = tol
    a.workspace = _lib.ptr(ws)
    a.patch_sweeps = _lib.ptr(ps)
    a.maxch_hist = _lib.ptr(mc)
    a.evals = _lib.ptr(ev)
    a.info = _lib.ptr(info)
    a.options = (0 if prune else _lib.SOLVE_NO_PRUNE) | (
        _lib.SOLVE_ASYNC if schedule == "async" else 0)
    a.act_tol = float(act_tol)
    a.inner_sweeps = int(inner)
    a.patch_counts = _lib.ptr(pc)
    if n_band:
        a.band_list = _lib.ptr(bands[0])
        a.band_off = _lib.ptr(bands[1])
        a.n_band = n_band
        a.band_inner = int(bands[3]) if len(bands) > 3 else 0
    if ao3 is not None:
        fbx, amask, acount, words = ao3
        a.ao3_fb = _lib.ptr(fbx)
        a.ao3_mask = _lib.ptr(amask)
        a.ao3_count = _lib.ptr(acount)
        a.ao3_words = int(words)
    a.stream = _lib.stream_handle()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.phj_solve(ctypes_ref(a)), "phj_solve")
    e1.record()
    # one device->host copy (one synchronisation) for every counter: info,
    # per-patch sweeps, evaluation counters and each patch's last max change
    # (exact in fp64: all counts are < 2^53)
    last = mc.view(max_sweeps, n_patches)[
        (ps.abs().long() - 1).clamp(0, max_sweeps - 1), torch.arange(n_patches, device=dev)]
    pack = torch.cat([info.double(), ps.double(), ev.double(), last]).cpu().numpy()
    # the per-patch counters as exact int64 (they can exceed 2^53 in sum only)
    pc_h = pc.cpu().numpy()
    info_h = pack[:4].astype(np.int64)
    ps_h = pack[4:4 + n_patches].astype(np.int32)
    ev_h = pack[4 + n_patches:7 + n_patches].astype(np.int64)
    res = v1 if int(info_h[1]) == 1 else work
    out = DeviceSolveResult(res, ps_h, pack[7 + n_patches:].copy(), int(ev_h[0]), info_h,
                            executed=int(ev_h[1]), real=int(ev_h[2]), patch_counts=pc_h,
                            schedule=schedule)
    out.device_ms = e0.elapsed_time(e1)
    if _lib.DIAG:
        out.block_counts = active_blocks_per_sweep(plan, ws, max_sweeps, int(info_h[0]))
    return out


def active_blocks_per_sweep(plan: StencilPlan, ws: torch.Tensor, max_sweeps: int, sweeps: int):
    """Active warp blocks per sweep from the solve workspace (diagnostics;
    layout of carve() in csrc/phj_common.cuh)."""
    total = int(_lib.load().phj_blocks_total(ctypes_ref(plan.gs)))
    tb = -(-total * 4 // 256) * 256
    off = 4 * tb
    counts = ws[off: off + 4 * (max_sweeps + 2)].view(torch.int32)
    return counts[:sweeps].cpu().numpy()


def stats_for_patch(res: DeviceSolveResult, p: int, n_nodes: int, n_adm: int, tol: float,
                    label: str = "", cands_per_sweep: Optional[int] = None) -> SweepStats:
    """SweepStats of patch p from the device counters (per-patch node
    relaxations and candidate evaluations counted by the solve kernels)."""
    s = int(res.patch_sweeps[p])
    st = SweepStats()
    if n_nodes == 0:
        return st
    st.converged = s > 0
    asyn = res.schedule == "async"
    pc = res.patch_counts
    if pc is not None:
        st.performed_evals = int(pc[p, 2])
    if asyn:
        # no sweeps: the reference's counters are the device's per-patch counts
        if pc is not None:
            st.node_relaxations = int(pc[p, 0])
            st.candidate_evals = int(pc[p, 1])
        # equivalent sweeps of this patch: its node relaxations / its nodes
        st.sweeps = max(1, -(-st.node_relaxations // n_nodes)) if pc is not None else abs(s)
        st.max_change = float("nan")
        if not st.converged:
            st.warning = (f"{label}asynchronous solve stopped: block-visit budget exhausted "
                          f"after {st.sweeps} equivalent sweeps")
        return st
    # Jacobi: the reference's dense counts for the same number of sweeps
    # (every node relaxed every sweep, _kernels.py:57-76)
    st.sweeps = abs(s)
    st.max_change = float(res.last_change[p]) if st.sweeps > 0 else 0.0
    st.node_relaxations = n_nodes * st.sweeps
    st.candidate_evals = (n_nodes * n_adm if cands_per_sweep is None
                          else int(cands_per_sweep)) * st.sweeps
    if not st.converged:
        st.warning = (f"{label}no convergence after {st.sweeps} sweeps "
                      f"(max change {st.max_change:.3e} > tol {tol:.1e})")
    return st


def _as_user_serials(grid: Grid, node_set) -> np.ndarray:
    if node_set is None:
        return np.arange(grid.n_interior, dtype=np.int64)
    if isinstance(node_set, torch.Tensor):
        return node_set.detach().cpu().numpy().astype(np.int64)
    return np.asarray(node_set, dtype=np.int64)


def _ext_user_tensor(a, plan: StencilPlan, dtype) -> torch.Tensor:
    t = torch.as_tensor(a.values if isinstance(a, NodeField) else a, device=plan.device)
    return t.reshape(plan.grid.ext_shape).to(dtype)


def allowed_tables(plan: StencilPlan, allowed) -> tuple:
    """Device tables for a per-(serial, control) ``allowed`` mask
    (_kernels.py:71-75 ``allowed[s, c]``; e.g. solver.allowed_mask): per ext
    node its row (= user serial) of a bitmask over the stencil entries (entry
    e allowed iff its original control is), and per row the number of allowed
    admissible controls (candidate-evaluation count).  Single-class stencils
    with at most 128 entries."""
    st = plan.stencils
    if st.n_classes != 1:
        raise ConfigurationError("allowed= needs a single-class stencil")
    n = plan.grid.n_interior
    a = allowed.detach() if isinstance(allowed, torch.Tensor) else torch.as_tensor(
        np.asarray(allowed))
    nc = len(plan.spec.control_set)
    if tuple(a.shape) != (n, nc):
        raise ConfigurationError(f"allowed must have shape ({n}, {nc}), got {tuple(a.shape)}")
    dev = plan.device
    a = a.to(dev) != 0
    noct = st.oct_start.shape[1] - 1
    e0, e1 = int(st.oct_start[0, 0]), int(st.oct_start[0, noct])
    if e1 > 128:
        raise ConfigurationError("allowed= supports at most 128 stencil entries")
    words = 1 if e1 <= 64 else 2
    ctrl = torch.as_tensor(st.ctrl[:e1].astype(np.int64), device=dev)
    mask = torch.zeros((n, words), dtype=torch.int64, device=dev)
    for e in range(e0, e1):
        mask[:, e >> 6] |= a[:, int(ctrl[e])].long() << (e & 63)
    adm = torch.unique(ctrl[e0:e1])
    count = a[:, adm].sum(dim=1).to(torch.int32)
    rows = torch.full(plan.int_ext, -1, dtype=torch.int32, device=dev)
    user = torch.arange(n, dtype=torch.int32, device=dev)
    plan.interior_int(rows).copy_(plan.serial_to_internal(user).view(plan.int_shape))
    return rows.contiguous(), mask.contiguous(), count.contiguous(), words


def solve(field: NodeField, spec: ProblemSpec, node_set=None,
          cfg: Optional[SolverConfig] = None, strategy: Optional[ExecutionStrategy] = None, *,
          table: Optional[StencilPlan] = None, active=None, frozen=None, hard=None,
          allowed=None) -> SweepStats:
    """Value iteration over ``node_set`` until converged (solver.py:201-279).

    Semantics follow the reference: ``active`` selects live reads, ``frozen``
    supplies Dirichlet data elsewhere, otherwise non-active corners are
    structurally blocked; ``hard`` overrides the block mask.  ``sweep_order``
    is accepted and has no effect (Jacobi).  ``allowed`` restricts the
    controls per (serial, control) (_kernels.py:71-75, AO3)."""
    cfg = cfg or SolverConfig()
    grid = field.grid
    require_cuda(field.values)
    plan = table if table is not None else StencilPlan(grid, spec)
    ao3 = allowed_tables(plan, allowed) if allowed is not None else None
    order = _as_user_serials(grid, node_set)
    if order.size == 0:
        return SweepStats()
    rule, dtype = cfg.rule, cfg.dtype
    dev = plan.device
    work = plan.working_from_user(field.values, rule, dtype)
    wflat = work.view(-1)
    if frozen is not None:
        if active is None:
            raise ConfigurationError("frozen data needs an active mask")
        fr = plan.working_from_user(_ext_user_tensor(frozen, plan, torch.float64), rule, dtype)
        act = plan.to_internal(_ext_user_tensor(active, plan, torch.uint8)) != 0
        work = torch.where(act, work, fr)
        wflat = work.view(-1)
    flat_int = plan.user_serials_to_internal_flat(order)
    kind_int_serial = plan.kind
    # kinds of the ordered nodes (internal serial order)
    int_serial = plan.serial_to_internal(torch.arange(grid.n_interior, device=dev))
    inv = torch.empty_like(int_serial)
    inv[int_serial] = torch.arange(grid.n_interior, device=dev)
    kinds = kind_int_serial[inv[torch.as_tensor(order, device=dev)]]
    lab = torch.full(plan.int_ext, _lib.LAB_FIXED, dtype=torch.int16, device=dev)
    free = kinds == KIND_FREE
    lab.view(-1)[flat_int[free]] = 0
    wflat[flat_int[kinds == KIND_TARGET]] = 0.0
    wflat[flat_int[kinds == KIND_OBSTACLE]] = unreached_value(rule)
    if hard is not None:
        hard_int = plan.to_internal(_ext_user_tensor(hard, plan, torch.uint8))
        fmask = plan.fmask_from_hard(hard_int.contiguous())
    elif active is None or frozen is not None:
        fmask = plan.fmask_hard
    else:
        act = plan.to_internal(_ext_user_tensor(active, plan, torch.uint8)) != 0
        hard_int = torch.where(act, plan.hard, torch.ones_like(plan.hard)).contiguous()
        fmask = plan.fmask_from_hard(hard_int)
    n_free = int(free.sum().item())
    if n_free == 0:
        # target/obstacle-only node sets: one working pass (solver.py:256-273)
        res_vals = work
        st = SweepStats(sweeps=1, node_relaxations=order.size)
    else:
        res = device_solve(plan, work, lab, fmask, 1, rule=rule, dtype=dtype, tol=cfg.tol,
                           max_sweeps=cfg.sweep_limit(grid), act_tol=cfg.act_tol, ao3=ao3,
                           schedule=cfg.schedule,
                           inner=cfg.inner_for(grid.dim))
        res_vals = res.values
        cands = None
        if ao3 is not None:  # dense count over the allowed sets (_kernels.py:73-76)
            cnt_user = ao3[2]  # rows are user serials
            order_t = torch.as_tensor(order, device=dev)
            cands = int(cnt_user[order_t[free]].sum().item())
        st = stats_for_patch(res, 0, n_free, plan.n_adm, cfg.tol, cands_per_sweep=cands)
        if cfg.schedule == "jacobi":
            st.node_relaxations = order.size * st.sweeps
        st.performed_evals = res.real
    out_user = plan.user_from_working(res_vals, rule, dtype).view(-1)
    uflat = torch.as_tensor(grid.interior_flat()[order], device=dev)
    field.flat[uflat] = out_user[uflat]
    return st


@dataclass
class CandidateEvaluation:
    """One (node, control) evaluation of the relaxation functional
    (solver.py:92-98)."""

    control_index: int
    step_h: float
    foot: np.ndarray
    value: float


def _node_serial(grid: Grid, index) -> int:
    return int(index) if np.ndim(index) == 0 else grid.index_to_serial(index)


def _ext_mask(grid: Grid, active_set) -> Optional[np.ndarray]:
    """Flat ext-layout bool mask from an ext/flat array or a predicate over
    interior-relative multi-indices (solver.py:291-305)."""
    if active_set is None:
        return None
    if callable(active_set):
        g = grid.ghost_width
        idx = np.indices(grid.ext_shape).reshape(grid.dim, -1).T - g
        return np.array([bool(active_set(tuple(int(i) for i in row))) for row in idx])
    arr = active_set.cpu().numpy() if isinstance(active_set, torch.Tensor) else np.asarray(
        active_set)
    return arr.reshape(-1).astype(bool)


def evaluate_candidates(field: NodeField, spec: ProblemSpec, index, active_set=None,
                        frozen: Optional[NodeField] = None,
                        eps_speed: Optional[float] = None) -> list:
    """All admissible candidate evaluations at ONE node (solver.py:308-363):
    the single-node inspection path of the reference, not the sweep.

    The node's 2^d x (controls) corner values are gathered from the device
    field in one copy; locate / weights follow grid.py:123-152, 227-239
    (``Grid.locate_many``); a foot leaning with nonzero weight on a ghost or
    obstacle corner, or on a corner outside ``active_set`` without ``frozen``
    data, evaluates to the sentinel; otherwise value = sum w * corner + h *
    running cost (1 for minimum time)."""
    grid = field.grid
    serial = _node_serial(grid, index)
    x = grid.interior_points()[serial]
    controls = np.asarray(spec.control_set.controls, dtype=float)
    F = np.stack([np.asarray(spec.dynamics(x[None, :], a), dtype=float)[0] for a in controls])
    speeds = np.array([float(np.linalg.norm(f)) for f in F])
    if eps_speed is None:
        eps_speed = 1.0e-12 * float(speeds.max())
    ok = np.nonzero(speeds >= eps_speed)[0]
    if ok.size == 0:
        return []
    h = grid.k_step / speeds[ok]
    feet = x[None, :] + h[:, None] * F[ok]
    cell, local = grid.locate_many(feet)
    corners = grid.cell_flat_base(cell)[:, None] + grid.corner_offsets[None, :]
    w = _reference_weights(local)
    dev = field.values.device
    idx = torch.as_tensor(corners.reshape(-1), device=dev)
    cv = field.flat[idx].cpu().numpy().reshape(corners.shape)
    fv = None if frozen is None else frozen.flat[idx].cpu().numpy().reshape(corners.shape)
    hard = np.ones(grid.n_ext, dtype=bool)
    kind = classify_nodes(grid, spec)
    hard[grid.interior_flat()] = kind == KIND_OBSTACLE
    act = _ext_mask(grid, active_set)
    out = []
    for i, c in enumerate(ok):
        value = 0.0
        blocked = False
        for k in range(corners.shape[1]):
            wc = w[i, k]
            if wc == 0.0:
                continue
            f2 = corners[i, k]
            if hard[f2]:
                blocked = True
                break
            if act is None or act[f2]:
                value += wc * cv[i, k]
            elif fv is not None:
                value += wc * fv[i, k]
            else:
                blocked = True
                break
        if blocked:
            value = field.sentinel
        else:
            cost = 1.0 if spec.running_cost is None else float(
                np.asarray(spec.running_cost(x[None, :], controls[c]))[0])
            value += h[i] * cost
        out.append(CandidateEvaluation(int(c), float(h[i]), feet[i], float(value)))
    return out


def _reference_weights(local: np.ndarray) -> np.ndarray:
    from .grid import interpolation_weights

    return interpolation_weights(local)


def relax_node(field: NodeField, spec: ProblemSpec, index, active_set=None,
               frozen: Optional[NodeField] = None, eps_speed: Optional[float] = None):
    """One node relaxation, pure (solver.py:366-394): ``(new_value,
    control_index)``; target -> (0, None), obstacle -> (sentinel, None); the
    best live candidate (ties to the lowest control index) only if it beats
    the current value."""
    grid = field.grid
    serial = _node_serial(grid, index)
    x = grid.interior_points()[serial][None, :]
    if spec.obstacles is not None and bool(spec.obstacles.contains(x)[0]):
        return field.sentinel, None
    if bool(spec.target.contains(x)[0]):
        return 0.0, None
    cands = evaluate_candidates(field, spec, serial, active_set=active_set, frozen=frozen,
                                eps_speed=eps_speed)
    live = [c for c in cands if c.value < 0.5 * field.sentinel]
    current = float(field.flat[int(grid.interior_flat()[serial])])
    if not live:
        return current, None
    best = min(live, key=lambda c: (c.value, c.control_index))
    if best.value >= current:
        return current, None
    return best.value, best.control_index


def extract_feedback(field: NodeField, spec: ProblemSpec, table: Optional[StencilPlan] = None,
                     strategy: Optional[ExecutionStrategy] = None, allowed=None, *,
                     rule: str = "reference", dtype: str = "float64"):
    """Argmin control at every interior node (solver.py:413-443).

    Dirichlet-style reads (only ghost/obstacle corners reject), -1 on
    target/obstacle/unreachable nodes, ties to the lowest control index.
    Returns ``(FeedbackField, candidate_evals)``."""
    require_cuda(field.values)
    plan = table if table is not None else StencilPlan(field.grid, spec)
    work = plan.working_from_user(field.values, rule, dtype)
    fb = feedback_internal(plan, work, rule=rule, dtype=dtype,
                           allowed=allowed_tables(plan, allowed) if allowed is not None else None)
    return FeedbackField(field.grid, spec.control_set, plan.serial_to_user(fb[0])), fb[1]


def feedback_internal(plan: StencilPlan, work: torch.Tensor, *, rule: str, dtype: str,
                      allowed=None, slab=None, out=None, ev=None):
    """Optimal control per internal serial (solver.py:413-443).  ``slab`` =
    (begin, end) restricts the launch to those block rows along internal axis
    0 (phj_feedback_slab; the other entries of ``out`` are left untouched)."""
    lib = _lib.load()
    if out is None:
        out = torch.empty(plan.grid.n_interior, dtype=torch.int32, device=plan.device)
    if ev is None:
        ev = torch.zeros(1, dtype=torch.int64, device=plan.device)
    coef, coef0 = plan.coef(rule, dtype)
    st = plan.stencil_struct()
    rows, mask, count, words = allowed if allowed is not None else (None, None, None, 0)
    s0, s1 = (0, -1) if slab is None else (int(slab[0]), int(slab[1]))
    _lib.check(lib.phj_feedback_slab(ctypes_ref(plan.gs), ctypes_ref(st), _dtype_id(dtype),
                                     _rule_id(rule), _lib.ptr(work), _lib.ptr(plan.kind),
                                     _lib.ptr(plan.fmask_hard), _lib.ptr(coef), coef0,
                                     unreach_threshold(rule), _lib.ptr(rows), _lib.ptr(mask),
                                     _lib.ptr(count), int(words), _lib.ptr(out),
                                     _lib.ptr(ev), s0, s1, _lib.stream_handle()), "phj_feedback")
    return out, ev


def feedback_sharded(plan: StencilPlan, work: torch.Tensor, *, rule: str, dtype: str):
    """feedback_internal split over the ranks by slabs of block rows along
    internal axis 0 and all-gathered (dist.gather_slabs); one rank: the plain
    launch.  Every rank needs the whole field: the colour transport is split
    by colour, not by space."""
    from . import dist

    rank, world = dist.world()
    if world <= 1:
        return feedback_internal(plan, work, rule=rule, dtype=dtype)
    dims = (ctypes.c_int32 * 3)()
    _lib.load().phj_block_dims(plan.grid.dim, dims)
    layers = int(dims[0])                       # node layers of axis 0 per block row
    n0 = int(plan.int_shape[0])
    row_elems = int(np.prod(plan.int_shape[1:]))
    ev = torch.zeros(1, dtype=torch.int64, device=plan.device)

    def compute(r0, r1, field):
        # the kernel writes field[serial] for the serials of block rows [r0, r1)
        feedback_internal(plan, work, rule=rule, dtype=dtype, slab=(r0, r1), out=field, ev=ev)

    out = dist.gather_slabs(compute, (n0 + layers - 1) // layers, layers * row_elems,
                            plan.grid.n_interior, torch.int32, plan.device)
    dist.sum_over_ranks(ev)
    return out, ev


def reduce_controls(control_set, a_star: np.ndarray, r: float) -> np.ndarray:
    """Indices of controls within angle pi/r of a_star (solver.py:446-459)."""
    if r <= 1.0:
        raise ConfigurationError("reduction factor must exceed 1")
    if not control_set.is_unit:
        return np.arange(len(control_set.controls), dtype=np.int64)
    thresh = np.cos(np.pi / r) - 1.0e-12
    dots = control_set.controls @ np.asarray(a_star, dtype=float)
    return np.where(dots >= thresh)[0]


def allowed_mask(control_set, feedback, r: float) -> np.ndarray:
    """Per-(node, control) conical-reduction mask (solver.py:462-476)."""
    fb = feedback.cpu().numpy() if isinstance(feedback, torch.Tensor) else np.asarray(feedback)
    controls = control_set.controls
    mask = np.ones((fb.size, controls.shape[0]), dtype=np.uint8)
    if not control_set.is_unit:
        return mask
    thresh = np.cos(np.pi / r) - 1.0e-12
    pair_ok = (controls @ controls.T >= thresh).astype(np.uint8)
    has = fb >= 0
    mask[has] = pair_ok[fb[has]]
    return mask
