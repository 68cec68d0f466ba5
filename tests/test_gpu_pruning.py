"""Exact octant pruning: the value sweep with pruning must
be bit-identical to evaluating every stencil entry -- same values, same
per-patch sweep counts -- while executing fewer entries.  Runs the fine
patch solves of reduced BASELINE workloads through the C ABI twice
(PHJ_SOLVE_NO_PRUNE on / off) from the same start field and labels."""

from __future__ import annotations

import pytest
import torch

from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    from paper_1109_3577_b200 import configs, patchy
    from paper_1109_3577_b200.solver import device_solve


def _patch_inputs(w):
    """Fine plan, start field and patch labels exactly as run_patchy builds
    them for the patch-solve phase."""
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    cfg = w.cfg
    vc, _ = patchy.solve_full_internal(cplan, cfg)
    vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
    fb, _ = patchy.feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
    parts = patchy._resolve_parts(w.pcfg, w.spec, fplan.grid, fplan)
    pf = [fplan.user_serials_to_internal_flat(p) for p in parts]
    phi, _, _, _ = patchy.transport_internal(fplan, fb, pf, w.pcfg.color_tol,
                                             10 * max(fplan.grid.shape))
    bv, bi = patchy.argmax_batched(fplan.gs, phi, len(parts), fplan.grid.n_interior,
                                   fplan.device)
    thr = patchy.unreach_threshold(cfg.rule)
    mask = patchy.plan_interior_serial(fplan, vf) >= thr
    color, _, _, lab = patchy.assemble_internal(fplan.gs, bv, bi, len(parts), mask, fplan.kind,
                                                fplan.grid.n_interior, fplan.device, [])
    return fplan, vf, lab, len(parts)


@pytest.mark.parametrize("name,kw", [
    ("c2", dict(n=257)),
    ("c3", dict(n=65)),
    ("c5", dict(n=65)),
])
def test_pruning_is_bit_exact(name, kw):
    w = configs.CONFIGS[name](**kw)
    fplan, vf, lab, R = _patch_inputs(w)
    fmask = fplan.fmask_from_labels(lab)
    cfg = w.cfg
    runs = []
    for prune in (True, False):
        res = device_solve(fplan, vf.clone(), lab, fmask, R, rule=cfg.rule, dtype=cfg.dtype,
                           tol=cfg.tol, max_sweeps=cfg.sweep_limit(fplan.grid), prune=prune)
        runs.append(res)
    a, b = runs
    assert torch.equal(a.values, b.values), "pruned sweep differs from the full sweep"
    assert (a.patch_sweeps == b.patch_sweeps).all()
    assert a.evals == b.evals  # same nodes swept, same logical work
    assert a.executed < b.executed, (a.executed, b.executed)
    print(f"{name}: executed {a.executed} of {b.executed} entries "
          f"({a.executed / b.executed:.2f}), sweeps {list(a.patch_sweeps)[:4]}")
