"""Error metrics and greedy-feedback trajectories (mirror of patchyhjb.analysis,
analysis.py:25-139).

``e1`` averages |a - b| over nodes finite (< sentinel/2) in both fields,
``e1_allnodes`` divides the same sum by the interior node count.  The
reduction runs on the device (``phj_error_partials``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import ctypes

from . import _lib
from .grid import NodeField, require_cuda


def ctypes_ref(x):
    return ctypes.byref(x)


@dataclass(frozen=True)
class ErrorReport:
    e1: float
    einf: float
    e1_allnodes: float
    compared_count: int
    excluded_count: int
    against: str = "dd_reference"

    def as_dict(self) -> dict:
        return {"E1": self.e1, "Einf": self.einf, "E1_allnodes": self.e1_allnodes,
                "compared": self.compared_count, "excluded": self.excluded_count}


def _interior_values(field):
    if isinstance(field, NodeField):
        idx = torch.as_tensor(field.grid.interior_flat(), device=field.values.device)
        return field.flat[idx], 0.5 * field.sentinel
    t = torch.as_tensor(np.asarray(field, dtype=float) if not isinstance(field, torch.Tensor)
                        else field, dtype=torch.float64).reshape(-1)
    return t, 0.5 * 1.0e9


def error_report(a, b, against: str = "dd_reference") -> ErrorReport:
    """Compare two fields; nodes unreachable on either side are excluded."""
    va, ha = _interior_values(a)
    vb, hb = _interior_values(b)
    if va.numel() != vb.numel():
        raise ValueError("fields live on different grids")
    n = va.numel()
    dev = require_cuda()
    va = va.to(dev).contiguous()
    vb = vb.to(dev).contiguous()
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().phj_error_partials(n, _lib.ptr(va), _lib.ptr(vb), ha, hb,
                                              _lib.ptr(out), _lib.stream_handle()),
               "error_partials")
    s, mx, cnt = out.cpu().tolist()
    compared = int(round(cnt))
    if compared == 0:
        return ErrorReport(0.0, 0.0, 0.0, 0, n, against)
    return ErrorReport(s / compared, mx, s / n, compared, n - compared, against)


# -- greedy-feedback trajectories (analysis.py:67-139) -------------------------------

REACHED_TARGET = "reached_target"
LEFT_DOMAIN = "left_domain"
STEP_LIMIT = "step_limit"
STALLED = "stalled"


@dataclass(frozen=True)
class Trajectory:
    """Discrete path from a start point; steps have length exactly k."""

    points: np.ndarray
    termination: str

    @property
    def n_steps(self) -> int:
        return self.points.shape[0] - 1

    @property
    def length(self) -> float:
        return float(np.linalg.norm(np.diff(self.points, axis=0), axis=1).sum())


def trace_trajectories(field: NodeField, spec, starts, max_steps=None) -> list:
    """Follow the value function's greedy feedback from many starts at once
    (analysis.py:82-139, batched): each step minimises interpolated value +
    step cost over the controls with |h f| = k; stops on target entry,
    domain exit, the step cap, or when no control has a finite candidate.

    The user's dynamics / target / obstacle callables run on the host for
    all live trajectories at once (they are arbitrary Python); the candidate
    feet of every (trajectory, control) are interpolated on the device
    (``phj_interpolate_points``, bit-exact with the reference's
    interpolate_many) -- the arithmetic around it follows the reference
    operation by operation."""
    grid = field.grid
    X = np.atleast_2d(np.asarray(starts, dtype=float)).copy()
    if X.shape[1] != grid.dim:
        raise ValueError(f"start must be a {grid.dim}-vector")
    if spec.running_cost is not None:
        from .grid import ConfigurationError
        raise ConfigurationError("running costs are not supported")
    if spec.obstacles is not None and np.any(spec.obstacles.contains(X)):
        raise ValueError("trajectory start lies inside an obstacle")
    if max_steps is None:
        max_steps = 10 * int(sum(grid.shape))
    dev = require_cuda(field.values)
    lib = _lib.load()
    gs = grid.device_struct()
    vals = field.values.contiguous()
    dtype_id = _lib.F32 if vals.dtype == torch.float32 else _lib.F64
    sent = float(field.sentinel)
    half = 0.5 * sent
    k = grid.k_step
    controls = np.asarray(spec.control_set.controls, dtype=float)
    nc = controls.shape[0]
    K = X.shape[0]
    per = np.asarray(grid.periodic, dtype=bool)
    paths = [[X[i].copy()] for i in range(K)]
    term = [None] * K
    live = np.arange(K)
    for _ in range(max_steps):
        x = X[live]
        inside = np.asarray(spec.target.contains(x), dtype=bool)
        for i in live[inside]:
            term[i] = REACHED_TARGET
        live, x = live[~inside], x[~inside]
        if live.size == 0:
            break
        F = np.stack([np.asarray(spec.dynamics(x, controls[c]), dtype=float)
                      for c in range(nc)], axis=1)                     # [L, nc, d]
        speeds = np.linalg.norm(F, axis=2)
        eps = 1.0e-12 * np.maximum(speeds.max(axis=1), 1.0)
        ok = speeds >= eps[:, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            h = np.where(ok, k / speeds, 0.0)
        feet = x[:, None, :] + h[:, :, None] * F
        pts = torch.as_tensor(feet.reshape(-1, grid.dim), device=dev).contiguous()
        out = torch.empty(pts.shape[0], dtype=torch.float64, device=dev)
        ood = torch.empty(pts.shape[0], dtype=torch.int8, device=dev)
        _lib.check(lib.phj_interpolate_points(ctypes_ref(gs), dtype_id, _lib.ptr(vals),
                                              _lib.ptr(pts), pts.shape[0], half, sent, 1,
                                              _lib.ptr(out), _lib.ptr(ood),
                                              _lib.stream_handle()), "interpolate_points")
        v = out.cpu().numpy().reshape(live.size, nc)
        bad = ood.cpu().numpy().reshape(live.size, nc) != 0
        ok &= ~bad & (v < half)
        cand = np.where(ok, v + h, np.inf)
        best = np.argmin(cand, axis=1)                                  # lowest index on ties
        found = ok[np.arange(live.size), best]
        for j in np.where(~found)[0]:
            term[live[j]] = STALLED
        keep = np.where(found)[0]
        nx = feet[keep, best[keep]]
        if per.any():  # periodic axes (extension): keep the coordinate in [lo, hi)
            span = grid.hi - grid.lo
            nx[:, per] = grid.lo[per] + np.mod(nx[:, per] - grid.lo[per], span[per])
        X[live[keep]] = nx
        left = np.any((nx < grid.lo) & ~per, axis=1) | np.any((nx > grid.hi) & ~per, axis=1)
        for j, i in enumerate(live[keep]):
            paths[i].append(nx[j].copy())
            if left[j]:
                term[i] = LEFT_DOMAIN
        live = live[keep][~left]
        if live.size == 0:
            break
    for i in range(K):
        if term[i] is None:
            term[i] = STEP_LIMIT
    return [Trajectory(np.array(paths[i]), term[i]) for i in range(K)]


def trace_trajectory(field: NodeField, spec, start, max_steps=None) -> Trajectory:
    """Single-start form (analysis.py:82-139)."""
    x = np.asarray(start, dtype=float)
    if x.shape != (field.grid.dim,):
        raise ValueError(f"start must be a {field.grid.dim}-vector")
    return trace_trajectories(field, spec, x[None, :], max_steps)[0]


# -- exports (analysis.py:140-238): host-side text formatting of one D2H copy --


def _interior_host(field: NodeField) -> np.ndarray:
    g = field.grid
    vals = field.values
    vals = vals.cpu().numpy() if isinstance(vals, torch.Tensor) else np.asarray(vals)
    return vals.reshape(g.ext_shape)[tuple(slice(1, 1 + m) for m in g.shape)]


def _first_axis_fastest(a: np.ndarray) -> np.ndarray:
    return np.asarray(a).ravel(order="F")


def _coordinate_columns(grid) -> list:
    mesh = np.meshgrid(*[grid.axis_nodes(ax) for ax in range(grid.dim)], indexing="ij")
    return [_first_axis_fastest(m) for m in mesh]


def _export_rows(obj):
    """(grid, values first-axis-fastest, value format, column name)."""
    from .patchy import PatchMap

    if isinstance(obj, PatchMap):
        c = obj.color.cpu().numpy() if isinstance(obj.color, torch.Tensor) else obj.color
        return obj.grid, _first_axis_fastest(np.asarray(c).reshape(obj.grid.shape)), "%d", "patch"
    vals = _first_axis_fastest(_interior_host(obj)).copy()
    return obj.grid, vals, "%.9g", "value"


def export_field(obj, path, fmt: str = "csv") -> None:
    """Write a value field or patch map as CSV or legacy ASCII VTK
    (analysis.py:159-174).  CSV: one row per interior node, first coordinate
    fastest, 9 significant digits, unreachable values as ``inf`` (patch maps:
    their integer codes).  VTK: STRUCTURED_POINTS with the raw values."""
    if fmt not in ("csv", "vtk"):
        raise ValueError(f"unknown export format {fmt!r}")
    grid, vals, vfmt, name = _export_rows(obj)
    if fmt == "csv":
        if name == "value":
            vals[vals >= 0.5 * obj.sentinel] = np.inf
        cols = _coordinate_columns(grid)
        header = ",".join(f"x{i + 1}" for i in range(grid.dim)) + f",{name}"
        np.savetxt(path, np.column_stack(cols + [vals]), fmt=["%.9g"] * grid.dim + [vfmt],
                   delimiter=",", header=header, comments="")
        return
    pad = 3 - grid.dim
    dims = list(grid.shape) + [1] * pad
    origin = [float(x) for x in grid.lo] + [0.0] * pad
    spacing = [float(x) for x in grid.spacing] + [1.0] * pad
    scalar = "SCALARS patch int 1" if name == "patch" else "SCALARS value float 1"
    lines = [("%d" % v) if name == "patch" else ("%.9g" % v) for v in vals]
    head = ["# vtk DataFile Version 3.0", "minimum-time value field", "ASCII",
            "DATASET STRUCTURED_POINTS", "DIMENSIONS {} {} {}".format(*dims),
            "ORIGIN {:.9g} {:.9g} {:.9g}".format(*origin),
            "SPACING {:.9g} {:.9g} {:.9g}".format(*spacing), f"POINT_DATA {vals.size}",
            scalar, "LOOKUP_TABLE default"]
    with open(path, "w") as fh:
        fh.write("\n".join(head + lines) + "\n")


def read_field_csv(path, grid=None):
    """Read an exported CSV back (analysis.py:194-211): ``(points, values)``
    without a grid, else a device NodeField with ``inf`` rows at the
    sentinel."""
    data = np.atleast_2d(np.genfromtxt(path, delimiter=",", skip_header=1))
    points, values = data[:, :-1], data[:, -1]
    if grid is None:
        return points, values
    field = NodeField(grid)
    shaped = values.reshape(grid.shape, order="F")
    vals = np.where(np.isfinite(shaped), shaped, field.sentinel).reshape(-1)
    idx = torch.as_tensor(grid.interior_flat(), device=field.values.device)
    field.flat[idx] = torch.as_tensor(vals, dtype=field.values.dtype, device=field.values.device)
    return field
