"""Per-phase cycle split (-DPHJ_TIMING build) of the patch-solve kernels at
G=1 and for rank 0 of G=8 (its patches alone): where a sweep of the
value-ordered pass spends its time.

    PHJ_LIB_PATH=.../libphj_timing.so python scripts/band_phases.py c5
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import _lib, configs, dist, patchy  # noqa: E402
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
fn = lib.phj_dbg_phase_cycles
fn.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 12)()
names = ["sweep_prologue", "fetch", "labels", "eval", "store", "maxch", "mark", "post_sweep",
         "sweep_flush", "cta_wait", "grid_sync", "-"]
real = dist.world
for G in (1, 8):
    dist.world = lambda G=G: (0, G)
    try:
        patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg, cfg, vf)
        fn(buf)
        _, _, _, pinfo = patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg, cfg, vf)
        torch.cuda.synchronize()
        fn(buf)
    finally:
        dist.world = real
    tot = sum(buf)
    print(json.dumps({"G": G, "kernel_ms": pinfo["kernel_ms"], "sweeps": pinfo["sweeps"],
                      "frac": {n: round(buf[i] / tot, 4) for i, n in enumerate(names)}}), flush=True)
