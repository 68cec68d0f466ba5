"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the golden fixtures of the real reference.

Tolerances (BASELINE north_star): converged v within 1e-8 sup-norm in fp64,
1e-4 in fp32; labels identical except at argmin ties within 1e-12 (counted).
Reference-rule comparisons exclude nodes >= sentinel/2 on either side
(analysis.py:56) plus sentinel-contaminated values (> 1e3).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, has_gpu
from oracle import pipeline as O
import oracle_cases as C

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_1109_3577_b200 as phj
    from paper_1109_3577_b200 import configs


def _flat(a):
    return np.asarray(a).reshape(-1)


def _eik_spec(lo, hi, controls, radius, center=None):
    d = len(lo)
    c = tuple(center) if center is not None else (0.0,) * d
    return phj.ProblemSpec(name="eik", dim=d, box_lo=lo, box_hi=hi,
                           dynamics=lambda X, a: np.tile(np.asarray(a, float), (len(X), 1)),
                           control_set=phj.ControlSet(np.asarray(controls), "unit-circle"
                                                      if d == 2 else "unit-sphere-geodesic"),
                           target=phj.TargetSpec.ball(c, radius), model=phj.ScaledSpeed(1.0))


def _live_close(got, want, tol, contaminated=1e3):
    live = (want < 0.5e9) & (got < 0.5e9)
    assert np.array_equal(want < 0.5e9, got < 0.5e9), "reachability differs"
    m = live & (want < contaminated)
    return float(np.abs(got[m] - want[m]).max()) if m.any() else 0.0


def _to_v(T):
    return np.where(T >= 0.5e9, 1.0, -np.expm1(-T))


# -- single-domain solves -----------------------------------------------------------


def test_c1_reference_rule_matches_golden_and_oracle():
    c = golden("c1_fine.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8))
    assert st.converged
    got = _flat(u.numpy())
    assert _live_close(got, _flat(c["u_jacobi"]), 1e-8) <= 1e-8
    assert _live_close(got, _flat(c["u_gs"]), 1e-8) <= 1e-8
    # Jacobi sweep count equals the reference's exact Jacobi mode (108)
    assert abs(st.sweeps - int(c["sweeps_jacobi"])) <= 1


def test_c1_kruzkov_matches_oracle():
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov"))
    pr = C.c1_fine()
    v = O.init_field(pr, "kruzkov")
    ost = O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-8)
    got = _to_v(_flat(u.numpy()))
    assert np.abs(got - v).max() <= 1e-8
    assert abs(st.sweeps - ost.sweeps) <= 1


def test_c1_kruzkov_fp32_matches_oracle():
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-6, rule="kruzkov",
                                                       dtype="float32"))
    pr = C.c1_fine()
    v = O.init_field(pr, "kruzkov")
    O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-8)
    got = _to_v(_flat(u.numpy()))
    assert np.abs(got - v).max() <= 1e-4


def test_fib3d_reference_rule_matches_golden():
    f = golden("fib3d_21.npz")
    spec = _eik_spec((-1.0,) * 3, (1.0,) * 3, C.fib_sphere(48), 0.25)
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21, 21))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8))
    assert st.converged
    assert _live_close(_flat(u.numpy()), _flat(f["u_gs"]), 1e-8) <= 1e-8


def test_fib3d_kruzkov_matches_oracle():
    spec = _eik_spec((-1.0,) * 3, (1.0,) * 3, C.fib_sphere(48), 0.25)
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21, 21))
    for dtype, tol, bar in (("float64", 1e-8, 1e-8), ("float32", 1e-6, 1e-4)):
        u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=tol, rule="kruzkov", dtype=dtype))
        pr = C.fib3d()
        v = O.init_field(pr, "kruzkov")
        O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-8)
        assert np.abs(_to_v(_flat(u.numpy())) - v).max() <= bar, dtype


def test_fan_variable_speed_with_zero_speed_line_matches_golden():
    fa = golden("fan41.npz")
    spec = phj.preset("fan2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8))
    assert st.converged
    got, want = _flat(u.numpy()), _flat(fa["u_gs"])
    # the fan2d sentinel bleed (acceptance c04) contaminates values;
    # compare the grounded ones
    m = (want < 1e3) & (got < 1e3)
    assert np.abs(got[m] - want[m]).max() <= 1e-8
    assert np.array_equal(want < 0.5e9, got < 0.5e9)


def test_zermelo_translation_stencil_matches_oracle():
    # f = 2.1 a + (2, 0): per-control step cost (COST_CTRL) path
    spec = phj.preset("zermelo2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8))
    pr = C.zermelo(41, 16)
    uo = O.init_field(pr, "reference")
    O.solve(uo, pr, rule="reference", mode="jacobi", tol=1e-8)
    assert _live_close(_flat(u.numpy()), uo, 1e-8) <= 1e-8
    uk, _ = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov"))
    vo = O.init_field(pr, "kruzkov")
    O.solve(vo, pr, rule="kruzkov", mode="jacobi", tol=1e-8)
    assert np.abs(_to_v(_flat(uk.numpy())) - vo).max() <= 1e-8


def test_relax_kat_single_jacobi_pass():
    # test_solver.py:34-49: 0.30 one step left -> 0.34 via control 16
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.5)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    f = phj.init_value_field(g, spec)
    tgt = spec.target.contains(g.interior_points()).reshape(g.shape)
    inner = torch.where(torch.as_tensor(tgt, device=f.values.device),
                        torch.zeros_like(f.interior), torch.full_like(f.interior, 0.9))
    f.interior.copy_(inner)
    f.interior[74, 50] = 0.30
    phj.solve(f, spec, node_set=np.array([75 * 101 + 50]), cfg=phj.SolverConfig(max_sweeps=1))
    assert float(f.interior[75, 50]) == pytest.approx(0.34, abs=1e-12)


def test_empty_and_target_only_node_sets():
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.5)
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21))
    f = phj.init_value_field(g, spec)
    before = f.values.clone()
    st = phj.solve(f, spec, node_set=np.array([], dtype=np.int64))
    assert st.sweeps == 0 and torch.equal(f.values, before)
    targets = np.where(spec.target.contains(g.interior_points()))[0]
    st = phj.solve(f, spec, node_set=targets)
    assert st.sweeps <= 2
    assert torch.all(f.interior.reshape(-1)[torch.as_tensor(targets, device=f.values.device)]
                     == 0.0)


def test_nonconvergence_sets_warning():
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.5)
    g = phj.Grid(spec.box_lo, spec.box_hi, (51, 51))
    f = phj.init_value_field(g, spec)
    st = phj.solve(f, spec, cfg=phj.SolverConfig(max_sweeps=2))
    assert not st.converged and st.warning is not None and st.sweeps == 2


# -- feedback / lift / transport / assembly -------------------------------------------


def test_feedback_matches_golden_except_near_ties():
    c = golden("c1_fine.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u = phj.NodeField(g, c["u_gs"])
    fb, ev = phj.extract_feedback(u, spec)
    got = fb.indices.cpu().numpy()
    _, gaps, _ = O.feedback(_flat(c["u_gs"]), C.c1_fine(), rule="reference")
    diff = got != c["feedback"]
    ties = gaps < 1e-12 * np.maximum(1.0, np.abs(_flat(c["u_gs"])[g.interior_flat()]))
    assert not np.any(diff & ~ties), np.where(diff & ~ties)
    print("feedback tie nodes:", int(ties.sum()), "differing:", int(diff.sum()))


def test_lift_bit_exact_with_golden():
    c = golden("c1_patchy.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    gc = phj.Grid(spec.box_lo, spec.box_hi, (26, 26))
    gf = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    from paper_1109_3577_b200 import patchy as P, solver as S

    cspec = phj.ProblemSpec(**{**spec.__dict__,
                               "target": phj.TargetSpec.ball((0.0, 0.0), float(c["coarse_radius"]))})
    cplan = S.StencilPlan(gc, cspec)
    fplan = S.StencilPlan(gf, spec)
    vc = torch.as_tensor(c["coarse"], device="cuda")
    vf = P.lift_internal(cplan, vc, fplan, "reference", "float64")
    assert np.array_equal(vf.cpu().numpy(), c["lifted"])


def test_c1_patchy_stages_match_golden():
    c = golden("c1_patchy.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    lifted = phj.NodeField(g, c["lifted"])
    fb, _ = phj.extract_feedback(lifted, spec)
    assert np.array_equal(fb.indices.cpu().numpy(), c["feedback"])
    parts = np.split(c["parts"], np.cumsum(c["part_sizes"])[:-1])
    phis = []
    for j, part in enumerate(parts):
        phi, sw, upd, warn = phj.transport_color(spec, g, fb, part, 1e-12)
        assert warn is None
        assert np.abs(phi.numpy() - c["phi"][j]).max() <= 1e-10
        phis.append((j, phi))
    mask = phj.mask_unreachable(lifted)
    kind = phj.solver.classify_nodes(g, spec)
    pm = phj.assemble_patches(phis, mask, g, kind=kind)
    assert np.array_equal(pm.color.cpu().numpy(), c["color"])
    assert np.array_equal(pm.boundary.cpu().numpy(), c["boundary"])
    val, pst, warns = phj.solve_patches(spec, g, pm, lifted, phj.PatchyConfig(n_patches=4),
                                        phj.SolverConfig(tol=1e-8))
    assert _live_close(_flat(val.numpy()), _flat(c["value"]), 1e-8) <= 1e-8
    assert all(s.converged for s in pst)


def test_assembly_kats():
    # patchy test KATs (test_patchy.py:226-298)
    g = phj.Grid((0.0, 0.0), (1.0, 1.0), (5, 5))
    kind = np.zeros(g.n_interior, dtype=np.int8)
    mask = np.zeros(g.n_interior, dtype=bool)

    def phi(entries):
        f = phj.NodeField(g)
        f.values[...] = 0.0
        flat = g.interior_flat()
        for s, v in entries.items():
            f.flat[int(flat[s])] = v
        return f

    pm = phj.assemble_patches([(0, phi({0: 0.8, 1: 0.5, 2: 0.3})),
                               (1, phi({0: 0.2, 1: 0.5, 2: 0.4}))], mask, g, kind=kind)
    col = pm.color.cpu().numpy()
    assert col[0] == 0 and col[1] == 0 and col[2] == 1
    x = g.index_to_serial((2, 2))
    pm = phj.assemble_patches([(1, phi({g.index_to_serial((2, 1)): 0.8})),
                               (2, phi({g.index_to_serial((1, 2)): 0.9,
                                        g.index_to_serial((3, 2)): 0.9,
                                        g.index_to_serial((2, 3)): 0.9}))], mask, g, kind=kind)
    assert int(pm.color[x]) == 2
    g4 = phj.Grid((0.0, 0.0), (1.0, 1.0), (4, 4))
    warns = []
    pm = phj.assemble_patches([(0, phj.NodeField(g4, np.zeros(g4.ext_shape)))],
                              np.zeros(16, bool), g4, kind=np.zeros(16, np.int8), warnings=warns)
    assert warns and np.all(pm.color.cpu().numpy() == 0)


def test_transport_kats_leftflow():
    # test_patchy.py:146-182: band fill, half blend, hole
    def dyn(X, a):
        return np.tile(np.asarray(a, float), (len(np.atleast_2d(X)), 1))

    spec = phj.ProblemSpec(name="leftflow", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                           dynamics=dyn, control_set=phj.discretize_circle(4),
                           target=phj.TargetSpec.plane(axis=0, offset=0.0))
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21))
    idx = torch.full((g.n_interior,), 2, dtype=torch.int32, device="cuda")
    fb = phj.FeedbackField(g, spec.control_set, idx)
    part = np.where(spec.target.contains(g.interior_points()))[0]
    phi, sweeps, upd, warn = phj.transport_color(spec, g, fb, part)
    vals = phi.interior.cpu().numpy()
    assert warn is None
    assert np.array_equal(vals[10:, :], np.ones((11, 21)))
    assert np.array_equal(vals[:10, :], np.zeros((10, 21)))
    idx2 = idx.clone()
    idx2[g.index_to_serial((15, 10))] = -1
    phi, _, _, _ = phj.transport_color(spec, g, phj.FeedbackField(g, spec.control_set, idx2), part)
    v = phi.interior.cpu().numpy()
    assert v[15, 10] == 0.0 and v[16, 10] == 0.0 and v[16, 11] == 1.0


# -- full pipeline vs the oracle pipeline ----------------------------------------------


def _oracle_c1(rule):
    w = configs.c1(rule=rule)
    fine = C.c1_fine()
    coarse = C.c1_coarse(float(w.pcfg.coarse_target.radius))
    parts = phj.partition_target(w.spec.target, w.spec.make_grid(101), 4)
    return w, O.run_patchy(fine, coarse, parts, rule=rule, mode="jacobi", tol=1e-8,
                           color_tol=1e-12)


@pytest.mark.parametrize("rule", ["reference", "kruzkov"])
def test_c1_run_patchy_matches_oracle_pipeline(rule):
    w, ores = _oracle_c1(rule)
    pcfg = w.pcfg
    pcfg.color_tol = 1e-12
    res = phj.run_patchy(w.spec, pcfg, w.cfg)
    g = res.value.grid
    got_fb = res.feedback.indices.cpu().numpy()
    fdiff = got_fb != ores.feedback
    ties = ores.gaps < 1e-12
    assert not np.any(fdiff & ~ties)
    col = res.patch_map.color.cpu().numpy()
    n_lab_diff = int((col != ores.color).sum())
    got = _flat(res.value.numpy())
    if rule == "kruzkov":
        err = np.abs(_to_v(got) - ores.value).max()
    else:
        err = _live_close(got, ores.value, 1e-8)
    print(f"{rule}: label diffs {n_lab_diff}, feedback ties {int(ties.sum())}, err {err:.2e}")
    if not fdiff.any():
        assert n_lab_diff == 0
    assert err <= 1e-8


def test_dubins_small_matches_oracle():
    w = configs.c4(nxy=33, nth=16, cxy=9, cth=8)
    g = w.spec.make_grid(w.pcfg.fine_nodes)
    u, st = phj.solve_single(w.spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov"))
    og = O.OGrid(g.lo, g.hi, g.shape, g.periodic)
    X = og.interior_points()
    pr = O.OProblem(og, "dubins", w.spec.control_set.controls,
                    np.linalg.norm(X[:, :2], axis=1) <= 0.2)
    v = O.init_field(pr, "kruzkov")
    O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-8)
    got = _to_v(_flat(u.numpy()))
    inner = og.interior_flat()
    assert np.abs(got[inner] - v[inner]).max() <= 1e-8


@pytest.mark.parametrize("r", [3, 6])
def test_c1_patch_solves_with_conical_reduction(r):
    """AO3 (solver.py:446-476, patchy.py:353-356) on the config-1 patch map:
    device patch solves with reduction r match the reference's reduced GS
    solves (golden) within the fixed-point bar, and the oracle's reduced
    Jacobi solves; the candidate-evaluation counts follow the reduced
    control sets (fewer than the full solve)."""
    c = golden("c1_patchy.npz")
    a = golden("c1_patchy_ao3.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    lifted = phj.NodeField(g, c["lifted"])
    fb, _ = phj.extract_feedback(lifted, spec)
    pm = phj.PatchMap(g, 4, torch.as_tensor(c["color"]))
    cfg = phj.SolverConfig(tol=1e-8)
    val, pst, _ = phj.solve_patches(spec, g, pm, lifted,
                                    phj.PatchyConfig(n_patches=4, reduction=float(r)), cfg,
                                    feedback=fb)
    got = _flat(val.numpy())
    assert _live_close(got, _flat(a[f"value_r{r}"]), 1e-8) <= 1e-8
    pr = C.c1_fine()
    allowed = O.allowed_mask(pr.controls, c["feedback"], float(r))
    ov, _ = O.solve_patches(pr, c["color"], 4, rule="reference", mode="jacobi", tol=1e-8,
                            allowed=allowed)
    assert _live_close(got, ov, 1e-8) <= 1e-8
    # candidate counts follow the reduced control sets: the reference's GS
    # counts are (its sweeps) x (allowed candidates per sweep); ours use our
    # Jacobi sweep counts, so compare the per-sweep figure
    for j, s in enumerate(pst):
        ref_per_sweep = int(a[f"evals_r{r}"][j]) / int(a[f"sweeps_r{r}"][j])
        assert s.candidate_evals / s.sweeps == ref_per_sweep


@pytest.mark.parametrize("key,kw", [("dirichlet", dict(bc_mode="dirichlet")),
                                    ("warm", dict(warm_start=True)),
                                    ("dirichlet_warm", dict(bc_mode="dirichlet",
                                                            warm_start=True))])
def test_c1_patch_solves_dirichlet_and_warm_start(key, kw):
    """Dirichlet patch BC / AO1 warm start (patchy.py:334-347): device patch
    solves match the reference's (golden, GS) and the oracle's Jacobi solves
    within the fixed-point bar."""
    c = golden("c1_patchy.npz")
    b = golden("c1_patchy_bc.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    lifted = phj.NodeField(g, c["lifted"])
    pm = phj.PatchMap(g, 4, torch.as_tensor(c["color"]))
    val, pst, _ = phj.solve_patches(spec, g, pm, lifted, phj.PatchyConfig(n_patches=4, **kw),
                                    phj.SolverConfig(tol=1e-8))
    got = _flat(val.numpy())
    assert _live_close(got, _flat(b[f"value_{key}"]), 1e-8) <= 1e-8
    ov, _ = O.solve_patches(C.c1_fine(), c["color"], 4, rule="reference", mode="jacobi",
                            tol=1e-8, lifted=_flat(c["lifted"]), **kw)
    assert _live_close(got, ov, 1e-8) <= 1e-8


# -- asynchronous schedule (chaotic relaxation + block-local relaxations) ------------
# Same fixed point as the Jacobi sweeps, reached to within activity_tol; the
# oracle runs to a tight tol so both sides sit at the fixed point.

ASYNC = dict(schedule="async")


def test_async_c1_reference_rule_matches_golden():
    c = golden("c1_fine.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, **ASYNC))
    assert st.converged
    got = _flat(u.numpy())
    assert _live_close(got, _flat(c["u_jacobi"]), 1e-8) <= 1e-8
    assert _live_close(got, _flat(c["u_gs"]), 1e-8) <= 1e-8


@pytest.mark.parametrize("inner", [1, 2, 8])
def test_async_c1_kruzkov_matches_tight_oracle(inner):
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov",
                                                       inner_sweeps=inner, **ASYNC))
    assert st.converged
    pr = C.c1_fine()
    v = O.init_field(pr, "kruzkov")
    O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-14)
    assert np.abs(_to_v(_flat(u.numpy())) - v).max() <= 1e-10


def test_async_fib3d_both_rules_and_fp32():
    spec = _eik_spec((-1.0,) * 3, (1.0,) * 3, C.fib_sphere(48), 0.25)
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21, 21))
    f = golden("fib3d_21.npz")
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, **ASYNC))
    assert st.converged
    assert _live_close(_flat(u.numpy()), _flat(f["u_gs"]), 1e-8) <= 1e-8
    pr = C.fib3d()
    v = O.init_field(pr, "kruzkov")
    O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-14)
    for dtype, bar in (("float64", 1e-10), ("float32", 1e-4)):
        u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov",
                                                           dtype=dtype, **ASYNC))
        assert np.abs(_to_v(_flat(u.numpy())) - v).max() <= bar, dtype


def test_async_zermelo_per_control_cost_matches_oracle():
    spec = phj.preset("zermelo2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    pr = C.zermelo(41, 16)
    u, _ = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, **ASYNC))
    uo = O.init_field(pr, "reference")
    O.solve(uo, pr, rule="reference", mode="jacobi", tol=1e-14)
    assert _live_close(_flat(u.numpy()), uo, 1e-8) <= 1e-8
    uk, _ = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov", **ASYNC))
    vo = O.init_field(pr, "kruzkov")
    O.solve(vo, pr, rule="kruzkov", mode="jacobi", tol=1e-14)
    assert np.abs(_to_v(_flat(uk.numpy())) - vo).max() <= 1e-10


def test_async_dubins_periodic_matches_tight_oracle():
    w = configs.c4(nxy=33, nth=16, cxy=9, cth=8)
    g = w.spec.make_grid(w.pcfg.fine_nodes)
    u, st = phj.solve_single(w.spec, g, phj.SolverConfig(tol=1e-8, rule="kruzkov", **ASYNC))
    og = O.OGrid(g.lo, g.hi, g.shape, g.periodic)
    X = og.interior_points()
    pr = O.OProblem(og, "dubins", w.spec.control_set.controls,
                    np.linalg.norm(X[:, :2], axis=1) <= 0.2)
    v = O.init_field(pr, "kruzkov")
    O.solve(v, pr, rule="kruzkov", mode="jacobi", tol=1e-14)
    inner = og.interior_flat()
    assert np.abs(_to_v(_flat(u.numpy()))[inner] - v[inner]).max() <= 1e-10


def test_async_budget_exhaustion_sets_warning():
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    u, st = phj.solve_single(spec, g, phj.SolverConfig(tol=1e-8, max_sweeps=3, **ASYNC))
    assert not st.converged and st.warning


# -- per-(serial, control) allowed masks on single-domain solves / feedback ----------
# (_kernels.py:71-75: `allowed[s, c] == 0` skips the candidate and is not
# counted; solver.py:446-476 builds such masks for AO3)


def _c1_allowed(kind):
    g = phj.Grid((-2.0, -2.0), (2.0, 2.0), (101, 101))
    rng = np.random.default_rng(1109)
    if kind == "random":
        a = (rng.random((g.n_interior, 32)) < 0.6).astype(np.uint8)
    else:  # conical reduction around the golden feedback, r = 3
        c = golden("c1_fine.npz")
        a = O.allowed_mask(C.circle(32), c["feedback"], 3.0)
    return g, a


@pytest.mark.parametrize("kind", ["random", "conical"])
def test_solve_with_allowed_matches_oracle(kind):
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g, a = _c1_allowed(kind)
    plan = phj.StencilPlan(g, spec)
    u = phj.init_value_field(g, spec, kind=plan.serial_to_user(plan.kind))
    st = phj.solve(u, spec, cfg=phj.SolverConfig(tol=1e-8), table=plan, allowed=a)
    pr = C.c1_fine()
    uo = O.init_field(pr, "reference")
    ost = O.solve(uo, pr, rule="reference", mode="jacobi", tol=1e-8, allowed=a)
    got = _flat(u.numpy())
    assert _live_close(got, uo, 1e-8) <= 1e-8
    # the evaluation count follows the allowed sets (same sweeps on both sides)
    if st.sweeps == ost.sweeps:
        assert st.candidate_evals == ost.candidate_evals


@pytest.mark.parametrize("kind", ["random", "conical"])
def test_feedback_with_allowed_matches_oracle(kind):
    c = golden("c1_fine.npz")
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g, a = _c1_allowed(kind)
    u = phj.NodeField(g, c["u_gs"])
    fb, ev = phj.extract_feedback(u, spec, allowed=a)
    got = fb.indices.cpu().numpy()
    want, gaps, ne = O.feedback(_flat(c["u_gs"]), C.c1_fine(), rule="reference", allowed=a)
    diff = got != want
    ties = gaps < 1e-12 * np.maximum(1.0, np.abs(_flat(c["u_gs"])[g.interior_flat()]))
    assert not np.any(diff & ~ties), np.where(diff & ~ties)
    assert int(ev) == ne
    # every chosen control is an allowed one
    ok = got >= 0
    assert np.all(a[np.where(ok)[0], got[ok]] == 1)


# -- static domain decomposition (decomp.py:101-190, test_decomp.py:96-112) ----------


@pytest.mark.parametrize("R", [1, 4])
def test_solve_dd_reaches_single_domain_fixed_point(R):
    spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.1)
    g = phj.Grid(spec.box_lo, spec.box_hi, (51, 51))
    cfg = phj.SolverConfig(tol=1e-9)
    single, sst = phj.solve_single(spec, g, cfg)
    dd, dst = phj.solve_dd(spec, g, phj.make_static_decomposition(g, R), cfg)
    assert dst.converged and sst.converged
    a, b = _flat(single.numpy()), _flat(dd.numpy())
    assert np.array_equal(a < 0.5e9, b < 0.5e9)
    live = a < 0.5e9
    assert np.abs(a[live] - b[live]).max() <= 1e-8
    # one box = the single-domain Jacobi iteration (same sweep count up to the stop)
    if R == 1:
        assert abs(dst.sweeps - sst.sweeps) <= 1


@pytest.mark.parametrize("R", [2, 4, 8])
def test_solve_dd_matches_oracle_schwarz_iteration(R):
    # the device Schwarz iteration against the oracle's restatement of
    # decomp.py:101-190 with the same (Jacobi) box sweep: identical outer
    # iteration counts, fields equal to rounding; and the oracle's GS form
    # (the reference's box sweep, pinned bit-exact to its solve_dd fixture in
    # tests/test_oracle_golden.py) reaches the same fixed point within 1e-8
    if R == 8:
        pr = C.fib3d(n=17, radius=0.25)
        spec = _eik_spec((-1.0,) * 3, (1.0,) * 3, C.fib_sphere(48), 0.25)
        g = phj.Grid(spec.box_lo, spec.box_hi, (17, 17, 17))
    else:
        pr = C.eikonal((-2.0, -2.0), (2.0, 2.0), (41, 41), C.circle(32), 0.3)
        spec = _eik_spec((-2.0, -2.0), (2.0, 2.0), C.circle(32), 0.3)
        g = phj.Grid(spec.box_lo, spec.box_hi, (41, 41))
    cfg = phj.SolverConfig(tol=1e-9)
    dd, dst = phj.solve_dd(spec, g, phj.make_static_decomposition(g, R), cfg)
    uj = O.init_field(pr, "reference")
    sj = O.solve_dd(uj, pr, R, rule="reference", mode="jacobi", tol=1e-9)
    ug = O.init_field(pr, "reference")
    sg = O.solve_dd(ug, pr, R, rule="reference", mode="gs", tol=1e-9)
    got = _flat(dd.numpy())
    assert dst.converged and sj.converged and sg.converged
    assert dst.sweeps == sj.sweeps, (dst.sweeps, sj.sweeps)
    live = uj < 0.5e9
    assert np.array_equal(got < 0.5e9, live)
    assert np.abs(got[live] - uj[live]).max() <= 1e-12
    assert np.abs(got[live] - ug[live]).max() <= 1e-8
    print(f"R={R}: outer iterations device {dst.sweeps} = oracle Jacobi {sj.sweeps}; "
          f"reference GS {sg.sweeps}")
