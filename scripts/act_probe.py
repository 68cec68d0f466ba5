"""Schedule / threshold probe: phase times, patch-solve kernel stats, max
|v - v_base| and label differences for SolverConfig variants (first = base).

    python scripts/act_probe.py c2 float64 jacobi:0 async:1e-12:8 async:1e-12:8:1e-8:1e-3:8

variant = schedule:activity_tol[:inner[:tol[:transport_frac[:transport_inner]]]]
"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

name, dtype = sys.argv[1], sys.argv[2]
acts = sys.argv[3:] or ["jacobi:0"]
w = configs.CONFIGS[name](dtype=dtype)
plans = patchy.make_plans(w.spec, w.pcfg)
ref = ref_col = None
for a in acts:
    sched, act, *rest = a.split(":")
    cfg = dataclasses.replace(w.cfg, activity_tol=float(act), schedule=sched,
                              inner_sweeps=int(rest[0]) if rest else None,
                              tol=float(rest[1]) if len(rest) > 1 else w.cfg.tol)
    if len(rest) > 2:
        patchy.TRANSPORT_ASYNC_FRAC = float(rest[2])
    if len(rest) > 3:
        patchy.TRANSPORT_INNER[w.spec.dim] = int(rest[3])
    for rep in range(2):
        res = phj.run_patchy(w.spec, w.pcfg, cfg, plans=plans)
        torch.cuda.synchronize()
    v = res.value.values.double()
    col = res.patch_map.color.clone()
    if ref is None:
        ref, ref_col = v.clone(), col
    fin = (ref < 1e8) & (v < 1e8)
    pk = res.stats.kernels.get("patch_solve", {})
    print(json.dumps({"config": name, "variant": a, "patch_ms": pk.get("kernel_ms"),
                      "transport_kernel_ms": patchy.TRANSPORT_DIAG.get("kernel_ms"),
                      "tiles": pk.get("tiles"), "sweeps": pk.get("sweeps"),
                      "executed": pk.get("executed"),
                      "transport_sweeps": res.transport_sweeps[:4],
                      "phases": res.stats.phases_ms(),
                      "max_diff": float((v - ref)[fin].abs().max()),
                      "label_diff": int((col != ref_col).sum()),
                      "mismatch_finite": int(((ref < 1e8) != (v < 1e8)).sum())}), flush=True)
