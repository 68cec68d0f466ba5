"""Coarse (513^2) and fine C2 solve time vs cooperative grid size
(PHJ_MAX_BLOCKS), plus the empty-sweep cost at each size."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
from paper_1109_3577_b200 import configs, patchy
from paper_1109_3577_b200.solver import device_solve
from paper_1109_3577_b200.patchy import init_working
w = configs.c2()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
cfg = w.cfg
for name, plan in (("coarse", cplan),):
    lab = patchy._full_domain_labels(plan)
    for rep in range(3):
        work = init_working(plan, cfg.rule, cfg.dtype)
        res = device_solve(plan, work, lab, plan.fmask_hard, 1, rule=cfg.rule, dtype=cfg.dtype,
                           tol=cfg.tol, max_sweeps=cfg.sweep_limit(plan.grid))
    sw = int(res.info[0])
    work = init_working(plan, cfg.rule, cfg.dtype)
    res2 = device_solve(plan, work, lab, plan.fmask_hard, 1, rule=cfg.rule, dtype=cfg.dtype,
                        tol=-1.0, max_sweeps=sw + 2000)
    print(name, "sweeps", sw, "ms", round(res.device_ms, 3), "empty-sweep us",
          round(1000 * (res2.device_ms - res.device_ms) / 2000, 2), flush=True)
''' % ROOT
for cap in ("37", "74", "148", "222", "296"):
    env = dict(os.environ, PHJ_MAX_BLOCKS=cap)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("CTAs", cap, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
