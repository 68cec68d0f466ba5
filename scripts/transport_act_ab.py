"""Transport activity-threshold A/B (config 5): kernel time and label
differences against the default threshold's labels."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

w = configs.c5(dtype="float64")
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
ref = None
for frac in (1e-3, 1e-2, 1e-1, 1e-4):
    patchy.TRANSPORT_ACT_FRAC = frac
    for rep in range(2):
        bv, bi, csw, upd = patchy._transport_and_argmax(fplan, fb, parts, pcfg.color_tol,
                                                         10 * max(fplan.grid.shape), cfg.schedule,
                                                         cfg.dtype, key_work=vf, rule=cfg.rule)
    ms = patchy.TRANSPORT_DIAG["kernel_ms"]
    if ref is None:
        ref = bi.clone()
    diff = int((bi != ref).sum().item())
    print(json.dumps({"act_frac": frac, "transport_ms": ms, "label_diffs_vs_1e-3": diff,
                      "updates": upd, "sweeps": [min(csw), max(csw)]}), flush=True)
