"""Visits per 20 us of the asynchronous transport and patch solve (needs a
-DPHJ_TIMING build): concurrency over time, tail length.

    PHJ_LIB_PATH=.../libphj_timing.so python scripts/visit_timeline.py c2
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1109_3577_b200 import _lib, configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
cfg = w.cfg
lib = _lib.load()
fn = lib.phj_dbg_timeline
fn.argtypes = [ctypes.c_void_p]
bins = (ctypes.c_uint * 4096)()


def report(label):
    b = np.frombuffer(bins, dtype=np.uint32).copy()
    nz = np.nonzero(b)[0]
    last = int(nz[-1]) + 1 if nz.size else 0
    b = b[:last]
    tot = int(b.sum())
    cum = np.cumsum(b) / max(tot, 1)
    t50, t90, t99 = [int(np.searchsorted(cum, q)) * 20 for q in (0.5, 0.9, 0.99)]
    print(json.dumps({"kernel": label, "visits": tot, "span_us": last * 20,
                      "t50_us": t50, "t90_us": t90, "t99_us": t99,
                      "visits_per_20us_profile": [int(x) for x in b[:: max(1, last // 40)]]}))


vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(w.pcfg, w.spec, fplan.grid, fplan)
pf = [fplan.user_serials_to_internal_flat(p) for p in parts]
for _ in range(2):
    fn(bins)
    phi, R, csw, upd = patchy.transport_internal(fplan, fb, pf, w.pcfg.color_tol,
                                                 10 * max(fplan.grid.shape), "async")
    torch.cuda.synchronize()
    fn(bins)
report("transport_async")
bv, bi = patchy.argmax_batched(fplan.gs, phi, R, fplan.grid.n_interior, fplan.device)
mask = patchy.plan_interior_serial(fplan, vf) >= patchy.unreach_threshold(cfg.rule)
color, _, _, lab = patchy.assemble_internal(fplan.gs, bv, bi, R, mask, fplan.kind,
                                            fplan.grid.n_interior, fplan.device, [])
kinds = (ctypes.c_ulonglong * 4)()
lib.phj_dbg_visit_kinds.argtypes = [ctypes.c_void_p]
for _ in range(2):
    fn(bins)
    lib.phj_dbg_visit_kinds(kinds)
    patchy.solve_patches_internal(fplan, color, lab, R, w.pcfg, cfg, vf)
    torch.cuda.synchronize()
    fn(bins)
    lib.phj_dbg_visit_kinds(kinds)
report("patch_solve_async")
print(json.dumps({"solve_visits_by_outcome": {"unchanged": kinds[0], "below_threshold": kinds[1],
                                              "changed": kinds[2]}}))
