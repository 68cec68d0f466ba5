"""Per-phase cycle split of the asynchronous transport (needs a -DPHJ_TIMING
build): PHJ_LIB_PATH=.../libphj_timing.so python scripts/transport_phases.py c2"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import _lib, configs, patchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
cfg = w.cfg
vc, _ = patchy.solve_full_internal(cplan, cfg)
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = patchy.feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(w.pcfg, w.spec, fplan.grid, fplan)
pf = [fplan.user_serials_to_internal_flat(p) for p in parts]
lib = _lib.load()
fn = lib.phj_dbg_phase_cycles
fn.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 12)()
names = ["pop", "stage", "-", "relax", "writeback", "-", "mark_release"]
for i in range(2):
    fn(buf)
    _, _, csw, upd = patchy.transport_internal(fplan, fb, pf, w.pcfg.color_tol,
                                               10 * max(fplan.grid.shape), "async")
    torch.cuda.synchronize()
    fn(buf)
tot = sum(buf)
print(json.dumps({"config": name, "kernel_ms": patchy.TRANSPORT_DIAG.get("kernel_ms"),
                  "sweeps": csw[:2], "updates": upd,
                  "frac": {n: round(buf[i] / tot, 4) for i, n in enumerate(names) if n != "-"}}))
