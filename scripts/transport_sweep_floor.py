"""Per-sweep fixed cost of the 3D transport's value-ordered pass: the same
pass (all ~630 sweeps of the band schedule) with 1, 2, 4, 8, 16, 32 colours --
kernel time vs colour count separates the per-sweep floor from the per-colour
work."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.CONFIGS[name](dtype="float64")
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
bands = patchy.transport_bands(fplan, vf, fb, cfg.rule)
for nc in (1, 2, 4, 8, 16, 32):
    sel = list(range(nc))
    flat = [fplan.user_serials_to_internal_flat(np.asarray(parts[j], dtype=np.int64)) for j in sel]
    for rep in range(2):
        phi, _, csw, upd = patchy.transport_internal(fplan, fb, flat, pcfg.color_tol,
                                                     10 * max(fplan.grid.shape), "jacobi",
                                                     torch.float64, bands=bands)
        del phi
    print(json.dumps({"colours": nc, "kernel_ms": round(patchy.TRANSPORT_DIAG["kernel_ms"], 2),
                      "sweeps": [int(min(map(abs, csw))), int(max(map(abs, csw)))],
                      "mover_updates": int(upd)}), flush=True)
