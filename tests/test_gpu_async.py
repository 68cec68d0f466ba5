"""Asynchronous schedules against the Jacobi ones on
the same inputs: the in-place chaotic transport converges to the same colour
fields (tight color_tol on both sides), whatever the block-local relaxation
count; the asynchronous patch solve reaches the same fixed point."""

from __future__ import annotations

import pytest
import torch

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    from paper_1109_3577_b200 import configs, patchy

CASES = [("c2", dict(n=129)), ("c3", dict(n=65)),
         ("c4", dict(nxy=41, nth=16, cxy=11, cth=8)), ("c5", dict(n=65, dtype="float64"))]


def _feedback_and_parts(w):
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    cfg = w.cfg
    vc, _ = patchy.solve_full_internal(cplan, cfg)
    vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
    fb, _ = patchy.feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
    parts = patchy._resolve_parts(w.pcfg, w.spec, fplan.grid, fplan)
    pf = [fplan.user_serials_to_internal_flat(p) for p in parts]
    return fplan, fb, pf


@pytest.mark.parametrize("name,kw", CASES)
@pytest.mark.parametrize("inner", [1, 2, 8])
def test_async_transport_matches_jacobi(name, kw, inner, monkeypatch):
    w = configs.CONFIGS[name](**kw)
    fplan, fb, pf = _feedback_and_parts(w)
    # config 4's transport converges slowly (large in-plane weights along the
    # heading axis): a generous cap, tol 1e-11
    limit = 200 * max(fplan.grid.shape)
    pj, _, csj, _ = patchy.transport_internal(fplan, fb, pf, 1e-11, limit, "jacobi")
    monkeypatch.setitem(patchy.TRANSPORT_INNER, fplan.grid.dim, inner)
    pa, _, csa, _ = patchy.transport_internal(fplan, fb, pf, 1e-11, limit, "async")
    err = (pa - pj).abs().max().item()
    print(f"{name} inner={inner}: max|phi_async - phi_jacobi| = {err:.2e}, sweeps jacobi "
          f"{csj[:4]} async {csa[:4]}")
    assert all(c > 0 for c in csj) and all(c > 0 for c in csa)
    assert err <= 1e-9


@pytest.mark.parametrize("name,kw", CASES)
def test_feedback_by_slabs_equals_the_full_launch(name, kw):
    """phj_feedback_slab (the multi-GPU split of the feedback stage,
    solver.feedback_sharded): uneven slabs of block rows fill exactly the
    entries of the full launch, and the evaluation counts add up."""
    import ctypes

    from paper_1109_3577_b200 import _lib, solver

    w = configs.CONFIGS[name](**kw)
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(w.cfg))
    vf = patchy.lift_internal(cplan, vc, fplan, w.cfg.rule, w.cfg.dtype)
    full, ev_full = solver.feedback_internal(fplan, vf, rule=w.cfg.rule, dtype=w.cfg.dtype)
    dims = (ctypes.c_int32 * 3)()
    _lib.load().phj_block_dims(fplan.grid.dim, dims)
    n_rows = (fplan.int_shape[0] + int(dims[0]) - 1) // int(dims[0])
    out = torch.full_like(full, -7)
    ev = torch.zeros(1, dtype=torch.int64, device=full.device)
    cuts = [0, n_rows // 3, n_rows // 3, n_rows - 1, n_rows]  # one empty slab
    for a, b in zip(cuts[:-1], cuts[1:]):
        solver.feedback_internal(fplan, vf, rule=w.cfg.rule, dtype=w.cfg.dtype, slab=(a, b),
                                 out=out, ev=ev)
    assert torch.equal(out, full)
    assert int(ev.item()) == int(ev_full.item())


def test_sharded_feedback_of_two_ranks_assembles_the_full_field(monkeypatch):
    """solver.feedback_sharded as ranks 0 and 1 of 2 (world patched, no
    process group: each call fills its own slab only): the two slabs are
    disjoint, cover every node and equal the single-rank feedback."""
    from paper_1109_3577_b200 import dist, solver

    w = configs.CONFIGS["c5"](n=65, dtype="float64")
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(w.cfg))
    vf = patchy.lift_internal(cplan, vc, fplan, w.cfg.rule, w.cfg.dtype)
    full, ev_full = solver.feedback_internal(fplan, vf, rule=w.cfg.rule, dtype=w.cfg.dtype)
    parts, evs = [], 0
    for r in range(2):
        monkeypatch.setattr(dist, "world", lambda r=r: (r, 2))
        out, ev = solver.feedback_sharded(fplan, vf, rule=w.cfg.rule, dtype=w.cfg.dtype)
        parts.append(out.clone())
        evs += int(ev.item())
    # kind-free nodes without any admissible control also hold -1: compare by slab
    n0 = fplan.int_shape[0]
    row = full.numel() // n0
    cut = ((n0 + 1) // 2) * row
    assert torch.equal(parts[0][:cut], full[:cut]) and torch.equal(parts[1][cut:], full[cut:])
    assert bool((parts[0][cut:] == -1).all()) and bool((parts[1][:cut] == -1).all())
    assert evs == int(ev_full.item())


def test_async_transport_matches_the_reference_golden_colours():
    """The asynchronous (in-place) 2D transport against the colour fields the
    REAL reference produced (tests/golden/c1_patchy.npz, converged at 1e-12)
    -- not only against the device's own Jacobi transport."""
    import os

    import numpy as np

    import paper_1109_3577_b200 as phj
    from paper_1109_3577_b200 import solver as S

    c = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_patchy.npz"))
    spec = phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                           dynamics=lambda X, a: np.tile(np.asarray(a, float), (len(X), 1)),
                           control_set=phj.discretize_circle(32),
                           target=phj.TargetSpec.ball((0.0, 0.0), 0.1),
                           model=phj.ScaledSpeed(1.0))
    g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
    plan = S.StencilPlan(g, spec)
    fb = plan.serial_to_internal(torch.as_tensor(c["feedback"], device=plan.device,
                                                 dtype=torch.int32)).contiguous()
    parts = np.split(c["parts"], np.cumsum(c["part_sizes"])[:-1])
    flat = [plan.user_serials_to_internal_flat(np.asarray(p, dtype=np.int64)) for p in parts]
    for inner in (1, 8):
        patchy.TRANSPORT_INNER[2] = inner
        try:
            phi, R, csw, _ = patchy.transport_internal(plan, fb, flat, 1e-12, 10 * 101, "async")
        finally:
            patchy.TRANSPORT_INNER[2] = 8
        assert all(x > 0 for x in csw)
        for j in range(R):
            got = plan.to_user(phi[j]).cpu().numpy()
            assert np.abs(got - c["phi"][j]).max() <= 1e-9, (inner, j)
