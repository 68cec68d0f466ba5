"""One full patchy step of a BASELINE workload (for ncu launch lists / captures).

    python scripts/profile_step.py c2 [float64|float32] [steps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import _lib, configs, patchy  # noqa: E402

_lib.DIAG = True

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = configs.CONFIGS[name](dtype=dtype)
plans = patchy.make_plans(w.spec, w.pcfg)
for i in range(steps):
    t0 = time.perf_counter()
    res = phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans, outputs=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    pk = dict(res.stats.kernels.get("patch_solve", {}))
    bc = pk.pop("block_counts", None)
    if bc is not None and len(bc):
        import numpy as np

        q = np.percentile(bc, [10, 50, 90, 99]).round().tolist()
        pk["blocks_per_sweep"] = {"mean": float(bc.mean()), "max": int(bc.max()),
                                  "p10_50_90_99": q, "sweeps_below_296": int((bc < 296).sum())}
    td = dict(patchy.TRANSPORT_DIAG)
    tb = td.pop("block_counts", None)
    if tb is not None and len(tb):
        import numpy as np

        td["blocks_per_sweep"] = {"mean": float(tb.mean()), "max": int(tb.max()),
                                  "p10_50_90_99": np.percentile(tb, [10, 50, 90, 99]).round().tolist()}
    print(json.dumps({"transport_kernel": td,"config": name, "dtype": dtype, "wall_ms": 1000 * dt,
                      "phases_ms": res.stats.phases_ms(),
                      "coarse_sweeps": res.coarse_stats.sweeps,
                      "transport_sweeps": res.transport_sweeps,
                      "patch_sweeps": [s.sweeps for s in res.patch_stats],
                      "patch_kernel": pk,
                      "performed": res.stats.performed_evals,
                      "dense": res.stats.candidate_evals}), flush=True)
