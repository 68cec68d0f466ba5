"""Fixed per-sweep cost of the solve kernel at full occupancy: the fine C2
grid solved as one domain with tol < 0 (never converges); once the active
set has died out every extra sweep is pure overhead (barrier, start-up)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import device_solve  # noqa: E402
from paper_1109_3577_b200.patchy import init_working  # noqa: E402

w = configs.c2(n=int(sys.argv[1]) if len(sys.argv) > 1 else 2049)
plan = patchy.make_plans(w.spec, w.pcfg)[0]
cfg = w.cfg
lab = patchy._full_domain_labels(plan)
res0 = None
for sweeps in (6000, 9000, 12000):
    work = init_working(plan, cfg.rule, cfg.dtype)
    res = device_solve(plan, work, lab, plan.fmask_hard, 1, rule=cfg.rule, dtype=cfg.dtype,
                       tol=-1.0, max_sweeps=sweeps)
    bc = res.block_counts
    print("sweeps", int(res.info[0]), "ms", round(res.device_ms, 3),
          "last-1000 mean blocks", float(bc[-1000:].mean()), flush=True)
