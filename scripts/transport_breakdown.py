"""Host-timed breakdown of the transport phase (sync around every call)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.patchy import solve_full_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
cfg, pcfg, spec = w.cfg, w.pcfg, w.spec


def T(label, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn(*a, **k)
    torch.cuda.synchronize()
    print(f"  {label:28s} {1000 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return r


for step in range(4):
    print("step", step)
    vc, cst = T("coarse", solve_full_internal, cplan, cfg)
    vf = T("lift", patchy.lift_internal, cplan, vc, fplan, cfg.rule, cfg.dtype)
    fb, ev = T("feedback", patchy.feedback_internal, fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
    thr = patchy.unreach_threshold(cfg.rule)
    mask = T("mask", lambda: patchy.plan_interior_serial(fplan, vf) >= thr)
    parts = T("parts", patchy._resolve_parts, pcfg, spec, fplan.grid, fplan)
    pf = T("parts_flat", lambda: [fplan.user_serials_to_internal_flat(p) for p in parts])
    limit = pcfg.transport_max_sweeps or 10 * max(fplan.grid.shape)
    phi, _, csw, upd = T("transport_internal", patchy.transport_internal, fplan, fb, pf,
                         pcfg.color_tol, limit)
    bv, bi = T("argmax", patchy.argmax_batched, fplan.gs, phi, len(parts), fplan.grid.n_interior,
               fplan.device)
    del phi
    warn = []
    T("assemble", patchy.assemble_internal, fplan.gs, bv, bi, len(parts), mask, fplan.kind,
      fplan.grid.n_interior, fplan.device, warn)
