"""3D colour transport: Jacobi kernel vs the asynchronous tiled kernel
(seeded, fp32 fields for fp32 workloads) -- kernel time and labels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

name = sys.argv[1]
w = configs.CONFIGS[name]()
plans = patchy.make_plans(w.spec, w.pcfg)
ref = None
for mode, inner in (("jacobi", 0), ("async", 2), ("async", 4)):
    patchy.TRANSPORT_ASYNC_3D = mode == "async"
    if inner:
        patchy.TRANSPORT_INNER[3] = inner
    for _ in range(2):
        r = phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans)
        torch.cuda.synchronize()
    col = r.patch_map.color.clone()
    if ref is None:
        ref = col
    print(name, mode, inner, "transport kernel ms %.1f" % patchy.TRANSPORT_DIAG["kernel_ms"],
          "phase %.1f" % r.stats.phases_ms()["transport"],
          "label diffs vs jacobi", int((col != ref).sum()), flush=True)
