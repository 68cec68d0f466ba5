"""A/B of the value-ordered patch-solve pass on one GPU: patch-solve kernel
time at G=1 and for rank 0 of G=8 (its patch subset alone), per setting of
PHJ_BAND_SCALE / PHJ_SOLVE_BAND_WINDOW / PHJ_BAND_INNER (env, set by caller)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, dist, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.CONFIGS[name](dtype="float64")
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
patchy.run_patchy(spec, pcfg, cfg, plans=(fplan, cplan), outputs=False)
vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
bv, bi, _, _ = patchy._transport_and_argmax(fplan, fb, parts, pcfg.color_tol,
                                             10 * max(fplan.grid.shape), cfg.schedule, cfg.dtype,
                                             key_work=vf, rule=cfg.rule)
mask = patchy.plan_interior_serial(fplan, vf) >= 1.0
color, _, _, lab = patchy.assemble_internal(fplan.gs, bv, bi, len(parts), mask, fplan.kind,
                                            fplan.grid.n_interior, fplan.device)
out = {"config": name, "scale": patchy.BAND_SCALE, "window": patchy.SOLVE_BAND_WINDOW,
       "inner": patchy.SOLVE_BAND_INNER, "twindow": patchy.TRANSPORT_BAND_WINDOW,
       "tscale": patchy.TRANSPORT_BAND_SCALE, "lib": os.path.basename(os.environ.get("PHJ_LIB_PATH", "default"))}
if os.environ.get("PHJ_AB_TRANSPORT_ONLY"):
    real = dist.world
    for G in (1, 8):
        dist.world = lambda G=G: (0, G)
        try:
            for rep in range(2):
                bv, bi, csw, _ = patchy._transport_and_argmax(fplan, fb, parts, pcfg.color_tol,
                                                              10 * max(fplan.grid.shape), cfg.schedule,
                                                              cfg.dtype, key_work=vf, rule=cfg.rule)
        finally:
            dist.world = real
        out[f"G{G}_transport_ms"] = patchy.TRANSPORT_DIAG["kernel_ms"]
        out[f"G{G}_tsweeps"] = [min(map(abs, csw)), max(map(abs, csw))]
    print(json.dumps(out), flush=True)
    sys.exit(0)
real = dist.world
for G in (1, 8):
    dist.world = lambda G=G: (0, G)
    try:
        for rep in range(2):
            patchy._transport_and_argmax(fplan, fb, parts, pcfg.color_tol,
                                         10 * max(fplan.grid.shape), cfg.schedule, cfg.dtype,
                                         key_work=vf, rule=cfg.rule)
    finally:
        dist.world = real
    out[f"G{G}_transport_ms"] = patchy.TRANSPORT_DIAG["kernel_ms"]
for G in (1, 8):
    dist.world = lambda G=G: (0, G)
    try:
        for rep in range(2):
            # node-count LPT on every repetition: a solve stores the work it
            # measured on the plan, and without a process group that is this
            # rank's patches only (weights of the others 0 -> a different,
            # lighter assignment: the G8 figures of earlier A/B files taken
            # with this script are too low for that reason)
            fplan._patch_work = None
            _, pst, _, pinfo = patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg,
                                                             cfg, vf)
    finally:
        dist.world = real
    out[f"G{G}_kernel_ms"] = pinfo["kernel_ms"]
    out[f"G{G}_executed"] = pinfo["performed"]
print(json.dumps(out), flush=True)
