"""Structured dynamics and node-independent interpolation stencils.

The reference precomputes, per (node, control), the foot cell and local
coordinates of ``x + h f(x, a)`` with ``h = k / |f|`` (solver.py:140-198,
32-40 B per pair; 518 GB for BASELINE config 5).  Whenever the foot
*displacement* ``k f / |f|`` does not depend on the node -- ``f = c(x) a``
(eikonal, fan, configs 1/2/3/5), ``f = f(a)`` (zermelo) -- or depends only on
one coordinate (Dubins heading, config 4), the interpolation weights are a
per-control (per-class) constant.  This module builds those stencils on the
host (tiny) and the per-node step coefficient description; the device reads
only the value grid, a per-node coefficient and a label byte pair.

Stencil convention (include/phj.h): per class, entries sorted by foot
octant; octant bit ax = displacement >= 0 along internal axis ax; the cell
spans offsets {-1,0} (bit 0) or {0,+1} (bit 1) per axis; corner bit ax =
upper face; weights are the reference's snapped multilinear weights
(grid.py:146-152, 227-239).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Union

import numpy as np

from .grid import SNAP_TOL, ConfigurationError, Grid

EPS_SPEED_REL = 1.0e-12  # solver.py:42
COST_NODE, COST_CTRL = 0, 1


@dataclass(frozen=True)
class SinProduct:
    """c(x) = c0 + amp * prod_{ax: omega_ax != 0} sin(omega_ax x_ax)."""

    c0: float
    amp: float
    omega: tuple

    def __call__(self, X: np.ndarray) -> np.ndarray:
        X = np.atleast_2d(X)
        prod = np.ones(X.shape[0])
        for ax, w in enumerate(self.omega):
            if w != 0.0:
                prod = prod * np.sin(w * X[:, ax])
        return self.c0 + self.amp * prod

    def max_bound(self) -> float:
        return abs(self.c0) + abs(self.amp)


@dataclass(frozen=True)
class ScaledSpeed:
    """f(x, a) = c(x) a with a constant, a ``SinProduct`` or a host callable c."""

    speed: Union[float, SinProduct, Callable]

    def dynamics(self) -> Callable:
        sp = self.speed

        def f(X, a):
            X = np.atleast_2d(X)
            c = np.full(X.shape[0], float(sp)) if np.isscalar(sp) else np.asarray(sp(X))
            return c[:, None] * np.asarray(a, dtype=float)[None, :]
        return f


@dataclass(frozen=True)
class Dubins:
    """f = (cos th, sin th, a) on (x, y, th); th is user axis 2 (periodic)."""

    def dynamics(self) -> Callable:
        def f(X, a):
            X = np.atleast_2d(X)
            out = np.empty((X.shape[0], 3))
            out[:, 0] = np.cos(X[:, 2])
            out[:, 1] = np.sin(X[:, 2])
            out[:, 2] = float(np.asarray(a).ravel()[0])
            return out
        return f


@dataclass
class StencilSet:
    """Host-side stencil tables (see module docstring)."""

    dim: int
    n_classes: int
    nc: int
    cost_mode: int
    perm: tuple
    oct_start: np.ndarray  # int32 [ncls, 2^d + 1]
    ctrl: np.ndarray       # int32 [ncls * nc]
    nzmask: np.ndarray     # uint32 [ncls * nc]
    weights: np.ndarray    # float64 [ncls * nc, 2^d]
    cost: np.ndarray       # float64 [ncls * nc]
    disp: np.ndarray       # float64 [ncls, nc, d] internal grid units (diagnostics)
    n_real: int = 0        # admissible controls per class (before padding)


@dataclass
class NodeSpeed:
    """Per-node speed description for COST_NODE plans (phj_speed_model)."""

    kind: int          # 0 constant, 1 array, 2 sin-product
    c0: float = 1.0
    amp: float = 0.0
    omega: tuple = (0.0, 0.0, 0.0)
    ctrl_norm: float = 1.0
    eps: float = 0.0
    speed: Optional[np.ndarray] = None  # kind 1, per USER serial


def _weights_for(disp: np.ndarray):
    """Octant, snapped weights and 3^d nonzero mask for one displacement
    vector (internal axes, grid units, |disp_ax| <= 1)."""
    d = disp.size
    octant = 0
    t = np.empty(d)
    for ax in range(d):
        x = float(disp[ax])
        if x > 1.0:
            x = 1.0
        if x < -1.0:
            x = -1.0
        if x >= 0.0:
            octant |= 1 << ax
            tt = x
        else:
            tt = x + 1.0
        if tt < SNAP_TOL:
            tt = 0.0
        if tt > 1.0 - SNAP_TOL:
            tt = 1.0
        t[ax] = tt
    w = np.ones(2 ** d)
    nz = 0
    for k in range(2 ** d):
        pos = 0
        for ax in range(d):
            up = (k >> ax) & 1
            w[k] *= t[ax] if up else 1.0 - t[ax]
            off = (0 if (octant >> ax) & 1 else -1) + up
            pos = pos * 3 + (off + 1)
        if w[k] != 0.0:
            nz |= 1 << pos
    # Make the left-to-right floating-point sum of the weights exactly 1 (the
    # kernels accumulate corners in this order): I[1] == 1 keeps unreached
    # Kruzkov nodes (v = 1) and pure colour regions (phi = 1) bit-stable, so
    # they never look "changed" to the activity tracking.  The adjustment is
    # at most an ulp of the last nonzero weight.
    last = max(k for k in range(2 ** d) if w[k] != 0.0)
    s = 0.0
    for k in range(last):
        s = s + float(w[k])
    w[last] = 1.0 - s
    return octant, w, nz


def _weights_all(disp: np.ndarray):
    """_weights_for over many displacements at once ([n, d] -> octant [n],
    weights [n, 2^d], nonzero masks [n]); the same IEEE operations in the
    same order, so the results are bit-identical (checked in the tests)."""
    disp = np.asarray(disp, dtype=float)
    n, d = disp.shape
    x = np.clip(disp, -1.0, 1.0)
    up_side = x >= 0.0
    octant = (up_side.astype(np.int64) << np.arange(d)).sum(axis=1)
    t = np.where(up_side, x, x + 1.0)
    t = np.where(t < SNAP_TOL, 0.0, t)
    t = np.where(t > 1.0 - SNAP_TOL, 1.0, t)
    nk = 2 ** d
    w = np.ones((n, nk))
    nz = np.zeros(n, dtype=np.int64)
    for k in range(nk):
        pos = np.zeros(n, dtype=np.int64)
        for ax in range(d):
            up = (k >> ax) & 1
            w[:, k] = w[:, k] * (t[:, ax] if up else 1.0 - t[:, ax])
            off = np.where((octant >> ax) & 1, 0, -1) + up
            pos = pos * 3 + (off + 1)
        nz |= np.where(w[:, k] != 0.0, np.int64(1) << pos, 0)
    # sequential left-to-right sum of the weights before the last nonzero
    # one, which is replaced by 1 - sum (see _weights_for)
    nzw = w != 0.0
    last = nk - 1 - np.argmax(nzw[:, ::-1], axis=1)
    ssum = np.zeros(n)
    for k in range(nk):
        ssum = np.where(k < last, ssum + w[:, k], ssum)
    w[np.arange(n), last] = 1.0 - ssum
    return octant, w, nz


def unroll(dim: int) -> int:
    """Entries per kernel inner-loop iteration (PHJ_UNROLL of the built
    library, include/phj.h)."""
    from . import _lib

    return _lib.unroll(dim)


def build_stencil(disp: np.ndarray, cost: Optional[np.ndarray], admissible: np.ndarray,
                  cost_mode: int, perm: tuple) -> StencilSet:
    """disp [ncls, nc, d] internal grid units; cost [ncls, nc] or None;
    admissible [ncls, nc] bool.  Each octant group is padded to a multiple of
    unroll(d) entries by repeating its last entry (same value, same control
    index: neither the min nor the lowest-index argmin changes)."""
    ncls, nc, d = disp.shape
    noct = 2 ** d
    U = unroll(d)
    per_cls = []
    n_real = 0
    for cls in range(ncls):
        info = []
        adm = np.nonzero(admissible[cls])[0]
        if adm.size:
            oa, wa, nza = _weights_all(disp[cls, adm])
            info = [(int(oa[i]), int(c), wa[i], int(nza[i])) for i, c in enumerate(adm)]
        info.sort(key=lambda e: (e[0], e[1]))  # octant, then original order
        groups = []
        for o in range(noct):
            g = [e for e in info if e[0] == o]
            if g:
                g = g + [g[-1]] * ((-len(g)) % U)
            groups.append(g)
        per_cls.append(groups)
        n_real = max(n_real, len(info))
    # slots >= the control count, so (class, control) -> entry maps index in range
    slots = max(1, nc, max(sum(len(g) for g in groups) for groups in per_cls))
    oct_start = np.zeros((ncls, noct + 1), dtype=np.int32)
    ctrl = np.zeros(ncls * slots, dtype=np.int32)
    nzm = np.zeros(ncls * slots, dtype=np.uint32)
    wts = np.zeros((ncls * slots, noct))
    cst = np.zeros(ncls * slots)
    for cls, groups in enumerate(per_cls):
        pos = cls * slots
        for o in range(noct):
            oct_start[cls, o] = pos
            for (_, c, w, nz) in groups[o]:
                ctrl[pos] = c
                nzm[pos] = nz
                wts[pos] = w
                cst[pos] = cost[cls, c] if cost is not None else 0.0
                pos += 1
        oct_start[cls, noct] = pos
    st = StencilSet(d, ncls, slots, cost_mode, tuple(perm), oct_start, ctrl, nzm, wts, cst,
                    disp.copy())
    st.n_real = n_real
    return st


def _unit_norm(A: np.ndarray) -> float:
    n = np.linalg.norm(A, axis=1)
    if n.min() <= 0.0 or (n.max() - n.min()) > 1e-12 * n.max():
        raise ConfigurationError(
            "f = c(x) a needs controls of one common norm on the device path "
            f"(got |a| in [{n.min()}, {n.max()}])")
    return float(n.mean())


def plan_stencils(grid: Grid, spec, model=None):
    """Return (StencilSet, NodeSpeed | None, eps_speed) for a problem.

    ``model`` defaults to ``spec.model``; without one the dynamics callable
    is sampled once on the host (the reference's CandidateTable does the same
    O(N*Nc) work, solver.py:162-188) and accepted if every control's foot
    displacement is node-independent."""
    model = model if model is not None else getattr(spec, "model", None)
    A = np.atleast_2d(np.asarray(spec.control_set.controls, dtype=float))
    if getattr(spec, "running_cost", None) is not None:
        raise ConfigurationError("running costs are not on the device stencil path")
    k = grid.k_step
    d = grid.dim
    if isinstance(model, ScaledSpeed):
        if A.shape[1] != d:
            raise ConfigurationError("f = c(x) a needs state-dimension controls")
        an = _unit_norm(A)
        disp = (k * (A / an) / grid.spacing[None, :])[None, :, :]
        adm = np.ones((1, A.shape[0]), dtype=bool)
        st = build_stencil(disp, None, adm, COST_NODE, tuple(range(d)))
        sp = model.speed
        if np.isscalar(sp):
            ns = NodeSpeed(kind=0, c0=float(sp), ctrl_norm=an)
            mx = abs(float(sp)) * an
        elif isinstance(sp, SinProduct):
            om = tuple(float(w) for w in sp.omega) + (0.0,) * (3 - len(sp.omega))
            ns = NodeSpeed(kind=2, c0=float(sp.c0), amp=float(sp.amp), omega=om, ctrl_norm=an)
            mx = sp.max_bound() * an
        else:
            arr = np.abs(np.asarray(sp(grid.interior_points()), dtype=float))
            ns = NodeSpeed(kind=1, speed=arr, ctrl_norm=an)
            mx = float(arr.max()) * an
        if mx == 0.0:
            raise ConfigurationError("dynamics vanish identically")
        ns.eps = EPS_SPEED_REL * mx
        return st, ns, ns.eps
    if isinstance(model, Dubins):
        if d != 3 or not grid.periodic[2] or A.shape[1] != 1:
            raise ConfigurationError("Dubins needs a 3D grid with periodic axis 2 and scalar a")
        perm = (2, 0, 1)
        th = grid.axis_nodes(2)
        ncls, nc = th.size, A.shape[0]
        disp = np.empty((ncls, nc, 3))
        cost = np.empty((ncls, nc))
        mx = 0.0
        for j, t in enumerate(th):
            for c in range(nc):
                f = np.array([np.cos(t), np.sin(t), A[c, 0]])
                sp = float(np.sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]))
                mx = max(mx, sp)
                h = k / sp
                du = h * f / grid.spacing
                disp[j, c] = [du[2], du[0], du[1]]
                cost[j, c] = h
        adm = np.ones((ncls, nc), dtype=bool)
        st = build_stencil(disp, cost, adm, COST_CTRL, perm)
        return st, None, EPS_SPEED_REL * mx
    if model is not None:
        raise ConfigurationError(f"unknown dynamics model {model!r}")
    # -- sample the callable (solver.py:162-188) --------------------------------
    X = grid.interior_points()
    nc = A.shape[0]
    speeds = []
    feet = []
    mx = 0.0
    for a in A:
        F = np.asarray(spec.dynamics(X, a), dtype=float)
        sp = np.linalg.norm(F, axis=1)
        mx = max(mx, float(sp.max()))
        speeds.append(sp)
        feet.append(F)
    if mx == 0.0:
        raise ConfigurationError("dynamics vanish identically")
    eps = EPS_SPEED_REL * mx
    S = np.stack(speeds, axis=1)             # [N, nc]
    adm = S >= eps
    disp = np.zeros((1, nc, d))
    adm_c = np.zeros((1, nc), dtype=bool)
    for c in range(nc):
        m = adm[:, c]
        if not m.any():
            continue
        dd = k * feet[c][m] / S[m, c][:, None] / grid.spacing[None, :]
        if np.abs(dd - dd[0]).max() > 1e-9:
            raise ConfigurationError(
                f"control {c}: foot direction varies over the grid; only f = c(x) a, "
                "f = f(a) and Dubins dynamics have node-independent stencils")
        disp[0, c] = dd[0]
        adm_c[0, c] = True
    cost = np.where(adm, k / np.where(adm, S, 1.0), -1.0)
    col = cost[:, adm_c[0]]
    if np.all(np.abs(col - col[0:1]) <= 1e-12 * np.abs(col[0:1])):  # f = f(a): translation
        st = build_stencil(disp, np.where(adm_c, cost[0:1], -1.0), adm_c, COST_CTRL,
                           tuple(range(d)))
        return st, None, eps
    # f = c(x) g(a) with |g(a)| common: node-separable cost
    node_adm = adm.any(axis=1)
    if np.any(adm[node_adm] != adm_c[0][None, :]) or np.any(adm[~node_adm]):
        raise ConfigurationError("per-(node, control) admissibility is not node-separable")
    ref = S[:, adm_c[0]][:, 0:1]
    if not np.all(np.abs(S[:, adm_c[0]] - ref) <= 1e-12 * np.maximum(ref, eps)):
        raise ConfigurationError("step costs are neither per-node nor per-control separable")
    st = build_stencil(disp, None, adm_c, COST_NODE, tuple(range(d)))
    ns = NodeSpeed(kind=1, speed=np.where(node_adm, S[:, np.argmax(adm_c[0])], 0.0),
                   ctrl_norm=1.0, eps=eps)
    return st, ns, eps
