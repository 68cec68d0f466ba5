"""Label reproducibility and transport time of the 2D asynchronous transport
against its activity fraction (x color_tol)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

w = configs.c2()
plans = patchy.make_plans(w.spec, w.pcfg)
for frac in (1e-3, 1e-4, 1e-5, 1e-6):
    patchy.TRANSPORT_ASYNC_FRAC = frac
    ref, diffs, ms = None, [], []
    for i in range(5):
        r = phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans)
        ms.append(patchy.TRANSPORT_DIAG["kernel_ms"])
        col = r.patch_map.color.clone()
        if ref is None:
            ref = col
        else:
            diffs.append(int((col != ref).sum()))
    print(f"frac {frac:g}: transport kernel ms {sorted(ms)[2]:.2f}, label diffs vs run 0 {diffs}",
          flush=True)
