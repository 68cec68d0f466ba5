"""Drop-in API surface beyond the solve path (reference __init__.py:82-140):
single-node relaxation (solver.py:308-394) and CSV/VTK export / import
(analysis.py:140-238), with the reference's own known-answer cases
(pkg/tests/test_solver.py:34-49, pkg/tests/test_analysis.py:77-140)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_1109_3577_b200 as phj


def _eikonal(n=101):
    spec = phj.preset("eikonal2d", controls=32)
    return spec, phj.Grid(spec.box_lo, spec.box_hi, (n, n))


def test_relax_picks_neighbour_on_optimal_ray():
    spec, g = _eikonal()
    f = phj.init_value_field(g, spec)
    f.interior[...] = 0.9
    f.interior[74, 50] = 0.30
    node = (75, 50)  # x = (1, 0); k = 0.04
    cands = phj.evaluate_candidates(f, spec, node)
    assert len(cands) == 32
    assert min(c.value for c in cands if c.control_index != 16) >= 0.38
    value, ctrl = phj.relax_node(f, spec, node)
    assert value == pytest.approx(0.34, abs=1e-12)
    assert ctrl == 16


def test_step_rule_scales_h_by_speed():
    spec = phj.preset("zermelo2d", controls=32)
    g = phj.Grid(spec.box_lo, spec.box_hi, (51, 51))
    f = phj.init_value_field(g, spec)
    x = g.interior_points()[g.index_to_serial((40, 25))]
    for c in phj.evaluate_candidates(f, spec, (40, 25)):
        assert np.linalg.norm(c.foot - x) == pytest.approx(g.k_step, rel=1e-12)


def test_relax_state_constraint_and_targets():
    spec, g = _eikonal(41)
    f = phj.init_value_field(g, spec)
    f.interior[...] = 0.5
    node = (30, 20)
    # every corner outside the active set and no frozen data -> all blocked
    active = np.zeros(g.ext_shape, dtype=bool)
    v, c = phj.relax_node(f, spec, node, active_set=active)
    assert c is None and v == 0.5
    # a frozen field supplies the values instead
    fr = phj.NodeField(g)
    fr.interior[...] = 0.1
    v, c = phj.relax_node(f, spec, node, active_set=active, frozen=fr)
    assert c is not None and v == pytest.approx(0.1 + g.k_step, abs=1e-12)
    tgt = g.index_to_serial((20, 20))  # the origin: a target node
    assert phj.relax_node(f, spec, tgt) == (0.0, None)


def test_relax_agrees_with_the_device_sweep():
    # the single-node path and one device Jacobi sweep give the same value
    spec, g = _eikonal(41)
    f, _ = phj.solve_single(spec, g, phj.SolverConfig(max_sweeps=6, tol=1e-12))
    snap = f.copy()
    g2 = phj.NodeField(g, snap.values.clone())
    phj.solve(g2, spec, cfg=phj.SolverConfig(max_sweeps=1, tol=1e-12))
    # nodes the sweep improved to finite values, and converged finite nodes;
    # relax_node ignores sentinel-mixed candidates (solver.py:384-386) while
    # the sweep writes any improvement (_kernels.py:101), so compare < 10
    before = snap.interior.cpu().numpy()
    after = g2.interior.cpu().numpy()
    moved = np.argwhere((after < before) & (after < 10.0))
    still = np.argwhere((after == before) & (after < 10.0) & (after > 0.0))
    assert len(moved) > 0 and len(still) > 0
    for node in list(map(tuple, moved[:: max(1, len(moved) // 6)])):
        v, c = phj.relax_node(snap, spec, node)
        assert c is not None
        assert float(after[node]) == pytest.approx(v, abs=1e-13)
    for node in list(map(tuple, still[:: max(1, len(still) // 3)])):
        v, c = phj.relax_node(snap, spec, node)
        assert c is None and v == float(before[node])


def test_csv_rows_are_first_axis_fastest(tmp_path):
    g = phj.Grid((0.0, 0.0), (1.0, 1.0), (2, 2))
    f = phj.NodeField(g)
    f.interior[:, :] = torch.tensor([[0.0, 2.0], [1.0, 3.0]], dtype=torch.float64)
    path = tmp_path / "f.csv"
    phj.export_field(f, path)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "x1,x2,value"
    rows = [tuple(float(t) for t in ln.split(",")) for ln in lines[1:]]
    assert rows == [(0.0, 0.0, 0.0), (1.0, 0.0, 1.0), (0.0, 1.0, 2.0), (1.0, 1.0, 3.0)]


def test_csv_round_trip_and_inf(tmp_path):
    spec = phj.preset("fan2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    field, _ = phj.solve_single(spec, g)
    path = tmp_path / "fan.csv"
    phj.export_field(field, path)
    assert "inf" in path.read_text()
    back = phj.read_field_csv(path, g)
    m = field.reachable_mask()
    assert (back.interior[m] - field.interior[m]).abs().max().item() <= 1e-8
    assert torch.equal(back.reachable_mask(), m)
    pts, vals = phj.read_field_csv(path)
    assert pts.shape == (41 * 41, 2) and vals.shape == (41 * 41,)


def test_csv_patch_map_uses_integer_codes(tmp_path):
    res = phj.run_patchy(phj.preset("eikonal2d", controls=8),
                         phj.PatchyConfig(n_patches=2, coarse_nodes=11, fine_nodes=11))
    path = tmp_path / "pm.csv"
    phj.export_field(res.patch_map, path)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "x1,x2,patch"
    codes = {int(ln.split(",")[-1]) for ln in lines[1:]}
    assert codes <= {-4, -3, -2, -1, 0, 1}
    assert -2 in codes and 0 in codes


def test_vtk_header_and_sentinel(tmp_path):
    g = phj.Grid((-1.0, -1.0), (1.0, 1.0), (3, 3))
    f = phj.NodeField(g)
    f.values[...] = 1.0
    f.interior[0, 0] = phj.SENTINEL
    path = tmp_path / "f.vtk"
    phj.export_field(f, path, fmt="vtk")
    lines = path.read_text().splitlines()
    assert lines[3] == "DATASET STRUCTURED_POINTS"
    assert lines[4] == "DIMENSIONS 3 3 1"
    assert lines[5] == "ORIGIN -1 -1 0"
    assert lines[6] == "SPACING 1 1 1"
    assert lines[7] == "POINT_DATA 9"
    assert lines[10] == "1e+09"  # raw sentinel, not inf
    with pytest.raises(ValueError):
        phj.export_field(f, tmp_path / "f.xyz", fmt="xyz")
