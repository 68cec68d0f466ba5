"""Coarse-stage (block-Jacobi) time against the cooperative CTA count
(PHJ_MAX_BLOCKS is read at every launch)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402

w = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
ccfg = patchy.coarse_cfg(w.cfg)
for cap in ("296", "222", "148", "111", "74", "37"):
    os.environ["PHJ_MAX_BLOCKS"] = cap
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vc, st = patchy.solve_full_internal(cplan, ccfg)
        torch.cuda.synchronize()
        ts.append(1000 * (time.perf_counter() - t0))
    print(cap, "CTAs: coarse ms", sorted(ts)[2], "sweeps", st.sweeps, flush=True)
