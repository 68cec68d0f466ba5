"""Small asynchronous / Jacobi patchy runs for compute-sanitizer (memcheck,
racecheck, synccheck): reduced config 2 (2D, async solve + async transport)
and reduced config 4 (3D Dubins, periodic heading, async solve, Jacobi
transport), plus a config-5-shaped 3D run.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs  # noqa: E402

which = sys.argv[1:] or ["c2", "c4", "c5"]
for name in which:
    if name == "c2":
        w = configs.c2(n=129)
    elif name == "c4":
        w = configs.c4(nxy=33, nth=16, cxy=9, cth=8)
    else:
        w = configs.c5(n=33, dtype="float64")
    for sched in ("async", "jacobi"):
        cfg = w.cfg
        cfg.schedule = sched
        cfg.inner_sweeps = None
        res = phj.run_patchy(w.spec, w.pcfg, cfg)
        torch.cuda.synchronize()
        ok = res.coarse_stats.converged and all(s.converged for s in res.patch_stats)
        print(f"{name} {sched}: converged={ok} transport_sweeps={res.transport_sweeps[:4]}",
              flush=True)
        assert ok
print("SANITIZE_RUN_OK")
