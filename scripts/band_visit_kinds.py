"""Outcome of the visits of the value-ordered patch-solve pass (diagnostic
build with -DPHJ_TIMING, PHJ_LIB_PATH): how many visits changed nothing, only
below the activity threshold, above it, or were copy visits.  (The cleanup's
~2 M visits land in the same counters.)"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import _lib, configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.CONFIGS[name](dtype="float64")
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
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
lib = _lib.load()
kinds = (ctypes.c_ulonglong * 4)()
lib.phj_dbg_visit_kinds.argtypes = [ctypes.c_void_p]
lib.phj_dbg_visit_kinds(kinds)  # reset
_, _, _, pinfo = patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg, cfg, vf)
torch.cuda.synchronize()
lib.phj_dbg_visit_kinds(kinds)
print(json.dumps({"config": name, "kernel_ms_timing_build": pinfo["kernel_ms"], "tiles": pinfo["tiles"],
                  "visits": {"unchanged": kinds[0], "below_threshold": kinds[1],
                             "changed": kinds[2], "copy": kinds[3]}}))
