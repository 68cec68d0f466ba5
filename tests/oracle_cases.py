"""Oracle-side problem builders shared by the tests (test infrastructure).

Each builder restates a reference problem as plain arrays for
``oracle.pipeline.OProblem``; formulas follow
/root/reference/pkg/src/patchyhjb/problems.py (cited per builder).
"""

from __future__ import annotations

import numpy as np

from oracle import pipeline as P


def circle(n: int) -> np.ndarray:  # problems.py:46-51
    ang = 2.0 * np.pi * np.arange(n) / n
    return np.stack([np.cos(ang), np.sin(ang)], axis=1)


def fib_sphere(n: int) -> np.ndarray:  # SURVEY §8d (configs 3/5)
    i = np.arange(n, dtype=float)
    z = 1.0 - (2.0 * i + 1.0) / n
    r = np.sqrt(1.0 - z * z)
    phi = np.pi * (1.0 + np.sqrt(5.0)) * (i + 0.5)
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def eikonal(lo, hi, shape, controls, radius, center=None, periodic=None):
    """f = a, ball target (problems.py:247-249, :111-139)."""
    g = P.OGrid(lo, hi, shape, periodic)
    X = g.interior_points()
    c = np.zeros(g.dim) if center is None else np.asarray(center, dtype=float)
    tgt = np.linalg.norm(X - c, axis=1) <= radius
    return P.OProblem(g, "scaled", controls, tgt, speed=np.ones(g.n_interior))


def c1_fine():
    return eikonal((-2.0, -2.0), (2.0, 2.0), (101, 101), circle(32), 0.1)


def c1_coarse(radius):
    return eikonal((-2.0, -2.0), (2.0, 2.0), (26, 26), circle(32), radius)


def fib3d(n=21, radius=0.25):
    return eikonal((-1.0,) * 3, (1.0,) * 3, (n,) * 3, fib_sphere(48), radius)


def fan(n=41, nc=16):
    """fan2d preset: f = |x1+x2+0.1| a, plane target x1=0 (problems.py:252-255,331-336)."""
    g = P.OGrid((-2.0, -2.0), (2.0, 2.0), (n, n))
    X = g.interior_points()
    tgt = np.abs(X[:, 0] - 0.0) <= 0.0 + 1.0e-9 * (1.0 + 0.0)  # problems.py:140-143
    return P.OProblem(g, "scaled", circle(nc), tgt, speed=np.abs(X.sum(axis=1) + 0.1))


def from_workload(w, which: str = "fine"):
    """OProblem for a paper_1109_3577_b200.configs.Workload (same inputs:
    grid, controls, target / coarse target, speed from the model's numpy
    callable or Dubins)."""
    from paper_1109_3577_b200 import dynamics

    spec, pcfg = w.spec, w.pcfg
    nodes = pcfg.fine_nodes if which == "fine" else pcfg.coarse_nodes
    g = spec.make_grid(nodes)
    og = P.OGrid(g.lo, g.hi, g.shape, g.periodic)
    X = og.interior_points()
    tgt_spec = spec.target if (which == "fine" or pcfg.coarse_target is None) else pcfg.coarse_target
    tgt = tgt_spec.contains(X)
    obs = spec.obstacles.contains(X) if spec.obstacles is not None else None
    model = spec.model
    if isinstance(model, dynamics.Dubins):
        return P.OProblem(og, "dubins", spec.control_set.controls, tgt, obstacle=obs)
    sp = model.speed
    speed = np.full(og.n_interior, float(sp)) if np.isscalar(sp) else np.asarray(sp(X), float)
    return P.OProblem(og, "scaled", spec.control_set.controls, tgt, obstacle=obs, speed=speed)


def zermelo(n=21, nc=16):
    """zermelo2d preset: f = 2.1 a + (2, 0) (problems.py:258-262,337-342)."""
    g = P.OGrid((-2.0, -2.0), (2.0, 2.0), (n, n))
    X = g.interior_points()
    A = circle(nc)
    F = np.stack([np.tile(2.1 * a + np.array([2.0, 0.0]), (X.shape[0], 1)) for a in A],
                 axis=1)
    return P.OProblem(g, "table", A, np.linalg.norm(X, axis=1) <= 0.5, F=F)
