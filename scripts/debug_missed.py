"""Debug: nodes the device leaves unreached although the oracle map reaches
them (certificate 'missed' count), per schedule / pruning."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from oracle import pipeline as O
import oracle_cases as C
from paper_1109_3577_b200 import configs, patchy, solver
from paper_1109_3577_b200.solver import feedback_internal

n = int(sys.argv[1]) if len(sys.argv) > 1 else 129
name = sys.argv[2] if len(sys.argv) > 2 else "c3"
w = configs.CONFIGS[name](n=n)
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
fine = C.from_workload(w, "fine")
fg = fine.grid
vc, cst = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb_i, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
bv, bi, csw, _ = patchy._transport_and_argmax(fplan, fb_i, parts, 1e-12, 10 * max(fg.shape), cfg.schedule, cfg.dtype)
mask_d = patchy.plan_interior_serial(fplan, vf) >= 1.0
color, n_unc, _, lab = patchy.assemble_internal(fplan.gs, bv, bi, len(parts), mask_d, fplan.kind, fg.n_interior, fplan.device)
col = fplan.serial_to_user(color).cpu().numpy()
import dataclasses
for sched, inner, prune in (("async", None, True), ("jacobi", None, True), ("async", 1, True)):
    c2 = dataclasses.replace(cfg, schedule=sched, inner_sweeps=inner)
    val, pst, warns, pinfo = patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg, c2, vf)
    v = fplan.to_user(val).cpu().numpy().reshape(-1)
    r = O.residual(v, fine, col, rule=cfg.rule)
    print(json.dumps({"sched": sched, "inner": inner, "missed": r.missed, "spurious": r.spurious, "r": r.r, "warns": warns}))
    if r.missed:
        ms = r.missed_serials
        fi = fg.interior_flat()
        idx = np.stack(np.unravel_index(ms, fg.shape), 1)
        print("missed:", r.missed, "first idx", idx[:8].tolist(), "labels", col[ms][:8].tolist())
        # neighbourhood labels / values of the first missed node
        s0 = ms[0]
        i0 = np.array(np.unravel_index(s0, fg.shape))
        vv = v.reshape(fg.ext_shape)
        cc = col.reshape(fg.shape)
        for d in np.ndindex(*(3,) * fg.dim):
            j = i0 + np.array(d) - 1
            if np.all(j >= 0) and np.all(j < np.array(fg.shape)):
                print("  nb", (np.array(d) - 1).tolist(), "label", int(cc[tuple(j)]), "v", float(vv[tuple(j + 1)]))
        # block id of the missed node (3D blocks: one plane of 8x8)
