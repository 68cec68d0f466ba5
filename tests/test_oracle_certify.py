"""CPU checks of the oracle's full-size certificates (test infrastructure):
the fixed-point residual (og_residual) and the transport residual
(og_transport_residual) against the oracle's own converged pipeline, and the
sparse majority repair against the reference-order dense one."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import pipeline as O
import oracle_cases as C


def _c1_pipeline(rule, tol):
    fine = C.c1_fine()
    coarse = C.c1_coarse(max(0.1, 0.16 * np.sqrt(2.0)))
    X = fine.grid.interior_points()
    ang = np.mod(np.arctan2(X[:, 1], X[:, 0]), 2 * np.pi)
    tgt = np.where(fine.target)[0]
    sec = np.floor(ang[tgt] / (2 * np.pi) * 4).astype(int)
    parts = [tgt[sec == j] for j in range(4)]
    res = O.run_patchy(fine, coarse, parts, rule=rule, tol=tol, color_tol=1e-13)
    return fine, parts, res


@pytest.mark.parametrize("rule", ["kruzkov", "reference"])
def test_residual_of_converged_patch_solve_is_tiny(rule):
    fine, _, res = _c1_pipeline(rule, 1e-14)
    r = O.residual(res.value, fine, res.color, rule=rule)
    assert (r.missed, r.spurious, r.bad_target, r.bad_blocked) == (0, 0, 0, 0)
    assert r.n_certified == int((res.color >= 0).sum())
    assert r.r <= 1e-13, r
    umax = float(res.value[fine.grid.interior_flat()][res.color >= 0].max())
    assert O.contraction_bound(fine, rule, r.r, umax) <= 1e-10


def test_residual_detects_unconverged_and_perturbed_fields():
    fine, _, res = _c1_pipeline("kruzkov", 1e-14)
    v = res.value.copy()
    iflat = fine.grid.interior_flat()
    s = int(np.where(res.color >= 0)[0][500])
    v[iflat[s]] -= 1e-6  # below the fixed point: T(v) - v > 0 somewhere
    r = O.residual(v, fine, res.color, rule="kruzkov")
    assert r.r >= 0.5e-6
    # an unreached node that can be reached is reported as missed
    v = res.value.copy()
    v[iflat[s]] = 1.0
    r = O.residual(v, fine, res.color, rule="kruzkov")
    assert r.missed == 1


def test_contraction_bound_holds_on_a_partial_solve():
    # a field stopped early: its true distance to the fixed point is below
    # the certificate r / (1 - beta_max)
    fine, _, res = _c1_pipeline("kruzkov", 1e-14)
    u, _ = O.solve_patches(fine, res.color, 4, rule="kruzkov", tol=1e-4)
    r = O.residual(u, fine, res.color, rule="kruzkov")
    live = res.color >= 0
    iflat = fine.grid.interior_flat()
    err = np.abs(u[iflat] - res.value[iflat])[live].max()
    assert err > 0
    assert err <= O.contraction_bound(fine, "kruzkov", r.r)


def test_transport_residual_of_converged_colours():
    fine, parts, res = _c1_pipeline("kruzkov", 1e-14)
    feet = O.transport_feet(fine, res.feedback)
    for part in parts:
        phi, _, _, ok = O.transport_color(fine, feet, part, 1e-14)
        assert ok
        r, nm = O.transport_residual(phi, fine, res.feedback)
        assert nm == feet[0].size
        assert r <= 1e-13
    phi, _, _, _ = O.transport_color(fine, feet, parts[0], 1e-2)
    r, _ = O.transport_residual(phi, fine, res.feedback)
    assert r > 1e-6


def test_sparse_assembly_equals_dense_assembly():
    fine, parts, res = _c1_pipeline("kruzkov", 1e-14)
    feet = O.transport_feet(fine, res.feedback)
    fields = []
    for j, part in enumerate(parts):
        phi, _, _, _ = O.transport_color(fine, feet, part, 1e-2)
        fields.append((j, phi))
    mask = res.lifted[fine.grid.interior_flat()] >= 1.0
    kind = fine.kind()
    color, n, unc, _ = O.assemble(iter(fields), mask, fine.grid, kind)
    iflat = fine.grid.interior_flat()
    stack = np.stack([phi[iflat] for _, phi in fields])
    best_idx = np.argmax(stack, axis=0).astype(np.int32)  # lowest index on ties
    best_val = stack.max(axis=0)
    col2, unc2 = O.assemble_sparse(best_val, best_idx, n, mask, fine.grid, kind)
    assert np.array_equal(color, col2)
    assert np.array_equal(unc, unc2)


def test_sparse_assembly_majority_ties_periodic():
    # reference assembly KAT shape (test_patchy.py:226-298): an uncovered
    # stripe between two colours is filled by face-neighbour majority with the
    # lowest colour on count ties; one periodic axis wraps
    g = O.OGrid((0.0, 0.0), (1.0, 1.0), (6, 5), periodic=(True, False))
    best_val = np.zeros(30)
    best_idx = np.zeros(30, dtype=np.int32)
    lab = np.full((6, 5), -1)
    lab[:, :2] = 0
    lab[:, 3:] = 1
    best_val[(lab >= 0).ravel()] = 1.0
    best_idx[:] = np.maximum(lab.ravel(), 0)
    kind = np.zeros(30, dtype=np.uint8)
    col, unc = O.assemble_sparse(best_val, best_idx, 2, None, g, kind)
    fields = [(j, np.where(np.pad((lab == j).astype(float), 1).ravel() > 0, 1.0, 0.0))
              for j in range(2)]
    col_d, _, unc_d, _ = O.assemble(iter(fields), np.zeros(30, dtype=bool), g, kind)
    assert np.array_equal(col, col_d) and unc.size == unc_d.size == 0
    assert np.all(col.reshape(6, 5)[:, 2] == 0)
