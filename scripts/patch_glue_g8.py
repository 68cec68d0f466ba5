"""Wall-clock split of solve_patches_internal for rank 0 of G ranks on one GPU
(full feedback / labels, dist.world patched): kernel vs host-side glue."""
import functools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, dist, patchy, solver  # noqa: E402
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
acc = {}


def wrap(obj, fn):
    f = getattr(obj, fn)

    @functools.wraps(f)
    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            torch.cuda.synchronize()
            acc[fn] = acc.get(fn, 0.0) + 1000 * (time.perf_counter() - t0)

    setattr(obj, fn, g)


for fn in ("band_schedule", "device_solve", "count_labels", "init_working"):
    wrap(patchy, fn)
wrap(type(fplan), "fmask_from_labels")
real = dist.world
for G in (1, 8):
    dist.world = lambda G=G: (0, G)
    try:
        for rep in range(3):
            acc.clear()
            fplan._patch_work = None  # node-count LPT (see scripts/band_ab.py)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, _, pinfo = patchy.solve_patches_internal(fplan, color, lab, len(parts), pcfg, cfg, vf)
            torch.cuda.synchronize()
            wall = 1000 * (time.perf_counter() - t0)
    finally:
        dist.world = real
    print(json.dumps({"G": G, "wall_ms": round(wall, 2), "kernel_ms": round(pinfo["kernel_ms"], 2),
                      "split_ms": {k: round(v, 2) for k, v in acc.items()}}), flush=True)
