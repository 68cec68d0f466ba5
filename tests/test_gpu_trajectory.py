"""Greedy-feedback trajectories (analysis.py:82-139) through the device
interpolation (phj_interpolate_points) against trajectories of the REAL
reference on the same committed fields (tests/golden/trajectories.npz, made
by tests/golden/make_golden.py traj), plus the reference's own KATs
(test_analysis.py:139-187)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, has_gpu
import oracle_cases as C

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_1109_3577_b200 as phj


def _c1_spec():
    return phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                           dynamics=lambda X, a: np.tile(np.asarray(a, float), (len(X), 1)),
                           control_set=phj.ControlSet(np.asarray(C.circle(32)), "unit-circle"),
                           target=phj.TargetSpec.ball((0.0, 0.0), 0.1),
                           model=phj.ScaledSpeed(1.0))


def _assert_same(tr, pts, term):
    assert tr.termination == str(term)
    assert tr.points.shape == pts.shape
    assert np.abs(tr.points - pts).max() <= 1e-12


def test_c1_trajectories_match_reference_bitwise_batched():
    t = golden("trajectories.npz")
    c = golden("c1_fine.npz")
    spec = _c1_spec()
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    f = phj.NodeField(g, c["u_gs"])
    n = len([k for k in t.files if k.startswith("c1_start_")])
    starts = np.stack([t[f"c1_start_{i}"] for i in range(n)])
    trs = phj.trace_trajectories(f, spec, starts)        # all starts in one batch
    for i, tr in enumerate(trs):
        _assert_same(tr, t[f"c1_points_{i}"], t[f"c1_term_{i}"])
    lim = phj.trace_trajectory(f, spec, (1.5, 1.5), max_steps=3)
    _assert_same(lim, t["c1_limit_points"], t["c1_limit_term"])
    assert lim.termination == phj.STEP_LIMIT and lim.n_steps == 3


def test_fan_trajectories_match_reference_including_stall():
    t = golden("trajectories.npz")
    fa = golden("fan41.npz")
    spec = phj.preset("fan2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    f = phj.NodeField(g, fa["u_gs"])
    for i in range(2):
        tr = phj.trace_trajectory(f, spec, t[f"fan_start_{i}"])
        _assert_same(tr, t[f"fan_points_{i}"], t[f"fan_term_{i}"])
    assert phj.trace_trajectory(f, spec, (-0.2, 0.1)).termination == phj.STALLED


def test_trajectory_kats_on_device_solution():
    # test_analysis.py:139-160 on a device solve
    spec = phj.preset("eikonal2d", controls=32)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    field, _ = phj.solve_single(spec, g)
    tr = phj.trace_trajectory(field, spec, (1.5, 0.0))
    assert tr.termination == phj.REACHED_TARGET
    steps = np.linalg.norm(np.diff(tr.points, axis=0), axis=1)
    assert np.allclose(steps, g.k_step, rtol=1e-9)
    assert tr.length == pytest.approx(1.0, abs=2.0 * g.k_step)
    assert tr.n_steps == 25
    inside = phj.trace_trajectory(field, spec, (0.1, 0.0))
    assert inside.termination == phj.REACHED_TARGET and inside.points.shape == (1, 2)


def test_trajectory_rejects_obstacle_start():
    spec = phj.preset("eikonal2d-obstacles", controls=8)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    field, _ = phj.solve_single(spec, g)
    with pytest.raises(ValueError):
        phj.trace_trajectory(field, spec, (-0.7, 0.7))
