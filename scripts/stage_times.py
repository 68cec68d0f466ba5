"""Per-stage wall times of the transport/assembly phase (diagnostics).

    python scripts/stage_times.py c2
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal, unreach_threshold  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)


def tick(label, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label:28s} {1000 * (t - t0):9.2f} ms", flush=True)
    return t


for rep in range(2):
    print(f"-- rep {rep}")
    t = time.perf_counter()
    vc, cst = patchy.solve_full_internal(cplan, cfg)
    t = tick("coarse solve", t)
    vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
    t = tick("lift", t)
    fb, ev = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
    t = tick("feedback", t)
    mask = patchy.plan_interior_serial(fplan, vf) >= unreach_threshold(cfg.rule)
    t = tick("mask", t)
    parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
    t = tick("parts", t)
    parts_flat = [fplan.user_serials_to_internal_flat(p) for p in parts]
    t = tick("parts_flat", t)
    tsched = cfg.schedule if fplan.grid.dim == 2 else "jacobi"
    phi, R, csw, upd = patchy.transport_internal(fplan, fb, parts_flat, pcfg.color_tol,
                                                 10 * max(fplan.grid.shape), tsched)
    t = tick("transport_internal", t)
    print("   transport kernel ms", patchy.TRANSPORT_DIAG.get("kernel_ms"))
    bv, bi = patchy.argmax_batched(fplan.gs, phi, R, fplan.grid.n_interior, fplan.device)
    t = tick("argmax", t)
    color, n_unc, boundary, lab = patchy.assemble_internal(
        fplan.gs, bv, bi, R, mask, fplan.kind, fplan.grid.n_interior, fplan.device, [])
    t = tick("assemble", t)
    out, pst, warns, pinfo = patchy.solve_patches_internal(fplan, color, lab, R, pcfg, cfg, vf)
    t = tick("patch solve", t)
    print("   patch kernel ms", pinfo["kernel_ms"], "uncovered", n_unc)
