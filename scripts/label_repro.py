"""Run-to-run reproducibility of the full-size C2 pipeline: labels and v over
several runs (the asynchronous kernels' visit order varies)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

w = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
plans = patchy.make_plans(w.spec, w.pcfg)
ref = None
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    r = phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans)
    T = r.value.values.double()
    v = torch.where(T < 1e8, -torch.expm1(-T), torch.ones_like(T))
    col = r.patch_map.color.clone()
    if ref is None:
        ref = (v.clone(), col)
        continue
    print(f"run {i}: label diffs {int((col != ref[1]).sum())}, max|dv| "
          f"{float((v - ref[0]).abs().max()):.2e}", flush=True)
