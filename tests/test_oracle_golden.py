"""Pin the CPU oracle to the real reference (fixtures from make_golden.py).

In reference-rule Gauss-Seidel mode the oracle must reproduce the shimmed
reference bit for bit; its Jacobi mode must reproduce the reference's own
exact Jacobi mode (active=0, frozen=snapshot) bit for bit.  Everything else
the GPU is checked against rests on these pins.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import pipeline as P
import oracle_cases as C


def _flat(a):
    return np.asarray(a).reshape(-1)


def test_zermelo_gs_and_jacobi_sweep_bit_exact():
    z = golden("zermelo21_sweep.npz")
    pr = C.zermelo()
    order = np.arange(pr.grid.n_interior)
    u = _flat(z["u0"]).copy()
    P.sweep(u, pr, order, rule="reference", mode="gs")
    assert np.array_equal(u, _flat(z["gs"]))
    u = _flat(z["u0"]).copy()
    P.sweep(u, pr, order, rule="reference", mode="jacobi")
    assert np.array_equal(u, _flat(z["jacobi"]))


def test_c1_converged_gs_bit_exact_with_counters():
    c = golden("c1_fine.npz")
    pr = C.c1_fine()
    u = P.init_field(pr, "reference")
    st = P.solve(u, pr, rule="reference", mode="gs", tol=1e-8)
    assert st.sweeps == int(c["sweeps_gs"])
    assert st.candidate_evals == int(c["evals_gs"])
    assert np.array_equal(u, _flat(c["u_gs"]))


def test_c1_jacobi_bit_exact():
    c = golden("c1_fine.npz")
    pr = C.c1_fine()
    u = _flat(c["u0"]).copy()
    P.sweep(u, pr, np.arange(pr.grid.n_interior), rule="reference", mode="jacobi")
    assert np.array_equal(u, _flat(c["jacobi1"]))
    u = P.init_field(pr, "reference")
    st = P.solve(u, pr, rule="reference", mode="jacobi", tol=1e-8)
    assert st.sweeps == int(c["sweeps_jacobi"])
    assert np.array_equal(u, _flat(c["u_jacobi"]))


def test_c1_feedback_bit_exact_and_tie_count():
    c = golden("c1_fine.npz")
    pr = C.c1_fine()
    fb, gaps, _ = P.feedback(_flat(c["u_gs"]), pr, rule="reference")
    assert np.array_equal(fb, c["feedback"])
    # config 1 has 4 free nodes with exact argmin ties
    assert int((gaps < 1e-12).sum()) == 4


def test_c1_patchy_pipeline_stagewise_bit_exact():
    c = golden("c1_patchy.npz")
    pr = C.c1_fine()
    prc = C.c1_coarse(float(c["coarse_radius"]))
    uc = P.init_field(prc, "reference")
    P.solve(uc, prc, rule="reference", mode="gs", tol=1e-8)
    # single-domain coarse == the reference's solve_dd(R=4) (decomp.py docstring)
    assert np.array_equal(uc, _flat(c["coarse"]))
    lf = P.lift(prc, _flat(c["coarse"]), pr, rule="reference")
    assert np.array_equal(lf, _flat(c["lifted"]))
    fb, _, _ = P.feedback(lf, pr, rule="reference")
    assert np.array_equal(fb, c["feedback"])
    feet = P.transport_feet(pr, fb)
    parts = np.split(c["parts"], np.cumsum(c["part_sizes"])[:-1])
    phis = []
    for j, part in enumerate(parts):
        phi, sw, _, ok = P.transport_color(pr, feet, part, 1e-12, mode="gs")
        assert ok and sw == int(c["transport_sweeps"][j])
        assert np.array_equal(phi, _flat(c["phi"][j]))
        phis.append(phi)
    mask = lf[pr.grid.interior_flat()] >= 0.5 * P.SENTINEL
    color, _, unc, bd = P.assemble(list(enumerate(phis)), mask, pr.grid, pr.kind())
    assert np.array_equal(color, c["color"])
    assert np.array_equal(bd, c["boundary"])
    assert unc.size == c["uncovered"].size
    val, pst = P.solve_patches(pr, color, 4, rule="reference", mode="gs", tol=1e-8)
    assert np.array_equal(val, _flat(c["value"]))
    assert [s.sweeps for s in pst] == [int(s) for s in c["patch_sweeps"]]


def test_c1_coarse_solve_dd_bit_exact():
    # the oracle's Schwarz iteration (decomp.py:101-190) reproduces the
    # reference's solve_dd(R=4) coarse field of the fixture bit for bit
    c = golden("c1_patchy.npz")
    prc = C.c1_coarse(float(c["coarse_radius"]))
    u = P.init_field(prc, "reference")
    st = P.solve_dd(u, prc, 4, rule="reference", mode="gs", tol=1e-8)
    assert st.converged and st.sweeps == int(c["coarse_sweeps"])
    assert np.array_equal(u, _flat(c["coarse"]))


def test_c1_jacobi_patchy_within_parity_of_gs():
    # Jacobi (the GPU iteration) reaches the same fixed point within 1e-8
    c = golden("c1_patchy.npz")
    pr = C.c1_fine()
    val, _ = P.solve_patches(pr, c["color"], 4, rule="reference", mode="jacobi", tol=1e-8)
    ref = _flat(c["value"])
    live = ref < 0.5 * P.SENTINEL
    assert np.array_equal(live, val < 0.5 * P.SENTINEL)
    assert np.abs(val[live] - ref[live]).max() <= 1e-8


def test_fib3d_gs_jacobi_feedback_bit_exact():
    f = golden("fib3d_21.npz")
    pr = C.fib3d()
    u = P.init_field(pr, "reference")
    st = P.solve(u, pr, rule="reference", mode="gs", tol=1e-8)
    assert st.sweeps == int(f["sweeps_gs"])
    assert np.array_equal(u, _flat(f["u_gs"]))
    u = _flat(f["u0"]).copy()
    P.sweep(u, pr, np.arange(pr.grid.n_interior), rule="reference", mode="jacobi")
    assert np.array_equal(u, _flat(f["jacobi1"]))
    fb, _, _ = P.feedback(_flat(f["u_gs"]), pr, rule="reference")
    assert np.array_equal(fb, f["feedback"])


def test_fan_degenerate_speed_lift_feedback_bit_exact():
    fa = golden("fan41.npz")
    pr = C.fan()
    assert pr.eps_speed == float(fa["eps_speed"])
    u = P.init_field(pr, "reference")
    st = P.solve(u, pr, rule="reference", mode="gs", tol=1e-8)
    assert st.sweeps == int(fa["sweeps_gs"])
    assert np.array_equal(u, _flat(fa["u_gs"]))
    lf = P.lift(pr, _flat(fa["u_gs"]), pr, rule="reference")
    assert np.array_equal(lf, _flat(fa["lifted"]))
    fb, _, _ = P.feedback(lf, pr, rule="reference")
    assert np.array_equal(fb, fa["feedback"])


def test_relax_kat_0p34():
    # test_solver.py:34-49: left neighbour holds 0.30, k=0.04 -> 0.34 via control 16
    pr = C.eikonal((-2.0, -2.0), (2.0, 2.0), (101, 101), C.circle(32), 0.5)
    g = pr.grid
    u = P.init_field(pr, "reference")
    inner = g.interior(u)
    inner[...] = np.where(g.interior(P.init_field(pr, "reference")) == 0.0, 0.0, 0.9)
    inner[74, 50] = 0.30
    s = 75 * 101 + 50
    P.sweep(u, pr, np.array([s]), rule="reference", mode="jacobi")
    assert g.interior(u)[75, 50] == pytest.approx(0.34, abs=1e-12)
    fb, _, _ = P.feedback(u, pr, rule="reference")


def test_kruzkov_rule_is_monotone_transform_of_reference_at_one_sweep():
    # one Kruzkov relaxation equals 1-exp(-(I[T]+h)) only when I is linear in
    # exp; here we just pin the known-answer: a single neighbour at v and all
    # else unreachable gives beta*v + 1 - beta.
    pr = C.eikonal((-2.0, -2.0), (2.0, 2.0), (101, 101), C.circle(32), 0.5)
    g = pr.grid
    u = P.init_field(pr, "kruzkov")
    inner = g.interior(u)
    inner[74, 50] = 0.25
    s = 75 * 101 + 50
    P.sweep(u, pr, np.array([s]), rule="kruzkov", mode="jacobi")
    beta = np.exp(-g.k_step)
    assert g.interior(u)[75, 50] == pytest.approx(beta * 0.25 + 1.0 - beta, abs=1e-15)


def test_c1_patch_solves_with_conical_reduction_bit_exact():
    """AO3 (solver.py:446-476, patchy.py:353-356): the oracle's reduced patch
    solves reproduce the reference's (r = 3 and 6) bit for bit, with the same
    sweep and candidate-evaluation counts."""
    c = golden("c1_patchy.npz")
    a = golden("c1_patchy_ao3.npz")
    pr = C.c1_fine()
    for r in (3, 6):
        allowed = P.allowed_mask(pr.controls, c["feedback"], float(r))
        val, pst = P.solve_patches(pr, c["color"], 4, rule="reference", mode="gs", tol=1e-8,
                                   allowed=allowed)
        assert np.array_equal(val, _flat(a[f"value_r{r}"]))
        assert [s.sweeps for s in pst] == [int(x) for x in a[f"sweeps_r{r}"]]
        assert [s.candidate_evals for s in pst] == [int(x) for x in a[f"evals_r{r}"]]


def test_c1_patch_solves_dirichlet_and_warm_start_bit_exact():
    """Dirichlet patch boundary condition and AO1 warm start
    (patchy.py:334-347) on the config-1 patch map: bit-exact with the
    reference, same sweep counts."""
    c = golden("c1_patchy.npz")
    b = golden("c1_patchy_bc.npz")
    pr = C.c1_fine()
    lifted = _flat(c["lifted"])
    for key, kw in (("dirichlet", dict(bc_mode="dirichlet")), ("warm", dict(warm_start=True)),
                    ("dirichlet_warm", dict(bc_mode="dirichlet", warm_start=True))):
        val, pst = P.solve_patches(pr, c["color"], 4, rule="reference", mode="gs", tol=1e-8,
                                   lifted=lifted, **kw)
        assert np.array_equal(val, _flat(b[f"value_{key}"])), key
        assert [s.sweeps for s in pst] == [int(x) for x in b[f"sweeps_{key}"]], key
