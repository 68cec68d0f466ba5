"""Stage-by-stage GPU bring-up probe (prints progress, dumps tracebacks on stall)."""
import faulthandler
import os
import sys
import time

faulthandler.dump_traceback_later(45, repeat=True)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t0 = time.time()


def log(*a):
    print(f"[{time.time() - t0:7.2f}s]", *a, flush=True)


import numpy as np  # noqa: E402
import torch  # noqa: E402

log("torch", torch.__version__, torch.cuda.is_available())
import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import _lib, patchy, solver  # noqa: E402

lib = _lib.load()
log("lib loaded, sms", lib.phj_num_sms())
spec = phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                       dynamics=lambda X, a: np.tile(np.asarray(a, float), (len(X), 1)),
                       control_set=phj.discretize_circle(32),
                       target=phj.TargetSpec.ball((0.0, 0.0), 0.1), model=phj.ScaledSpeed(1.0))
g = phj.Grid(spec.box_lo, spec.box_hi, (101, 101))
plan = solver.StencilPlan(g, spec)
torch.cuda.synchronize()
log("plan ok; kinds", torch.bincount(plan.kind.long()).tolist())
cfg = phj.SolverConfig(tol=1e-8, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 3)
work = patchy.init_working(plan, cfg.rule, cfg.dtype)
lab = patchy._full_domain_labels(plan)
torch.cuda.synchronize()
log("init ok")
res = solver.device_solve(plan, work, lab, plan.fmask_hard, 1, rule=cfg.rule, dtype=cfg.dtype,
                          tol=cfg.tol, max_sweeps=cfg.max_sweeps)
torch.cuda.synchronize()
log("solve ok", res.patch_sweeps, res.info, res.evals, res.device_ms)
cfg2 = phj.SolverConfig(tol=1e-8)
res = solver.device_solve(plan, patchy.init_working(plan, "reference", "float64"), lab,
                          plan.fmask_hard, 1, rule="reference", dtype="float64", tol=1e-8,
                          max_sweeps=1010)
torch.cuda.synchronize()
log("full solve ok", res.patch_sweeps, res.info, res.evals, res.device_ms)
faulthandler.cancel_dump_traceback_later()
