"""Colour-transport labels of the C2 workload under different stops, against
the converged labels (Jacobi to color_tol 1e-12): how far is each stop from
the fixed point's argmax, and what does it cost."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
cfg = w.cfg
vc, _ = patchy.solve_full_internal(cplan, cfg)
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(w.pcfg, w.spec, fplan.grid, fplan)
pf = [fplan.user_serials_to_internal_flat(p) for p in parts]
n = fplan.grid.n_interior
limit = 40 * max(fplan.grid.shape)


def labels(tol, sched, frac=1e-3):
    patchy.TRANSPORT_ASYNC_FRAC = frac
    for _ in range(2):
        phi, R, csw, upd = patchy.transport_internal(fplan, fb, pf, tol, limit, sched)
        torch.cuda.synchronize()
    ms = patchy.TRANSPORT_DIAG["kernel_ms"]
    bv, bi = patchy.argmax_batched(fplan.gs, phi, R, n, fplan.device)
    return bv, bi, ms


rv, ri, rms = labels(1e-12, "jacobi")
live = rv > 0
print(json.dumps({"ref": "jacobi color_tol 1e-12", "kernel_ms": rms, "nodes_with_mass": int(live.sum())}))
for tol, sched, frac in [(1e-2, "jacobi", 1e-3), (1e-2, "async", 1e-3), (1e-2, "async", 1e-2),
                         (1e-2, "async", 1e-1), (1e-2, "async", 1.0), (1e-3, "jacobi", 1e-3)]:
    bv, bi, ms = labels(tol, sched, frac)
    d = int(((bi != ri) & live).sum())
    print(json.dumps({"color_tol": tol, "schedule": sched, "async_frac": frac, "kernel_ms": ms,
                      "label_diffs_vs_converged": d}), flush=True)
