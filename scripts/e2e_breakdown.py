"""Where the public-API (e2e) step spends time beyond the device pipeline
(bench.py's e2e loop: run_patchy from the problem description, value copied
into a pinned host buffer)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name](dtype="float64") if name == "c5" else configs.CONFIGS[name]()
r = phj.run_patchy(w.spec, w.pcfg, w.cfg)
host = torch.empty(r.value.values.shape, dtype=r.value.values.dtype, pin_memory=True)


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"  {label:34s} {1000 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return out


for i in range(3):
    print("step", i)
    plans = t("make_plans", lambda: patchy.make_plans(w.spec, w.pcfg))
    t("run_patchy(plans, outputs=False)", lambda: phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans,
                                                                outputs=False))
    t("run_patchy(plans, outputs=True)", lambda: phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans))
    r = t("run_patchy(public)", lambda: phj.run_patchy(w.spec, w.pcfg, w.cfg))
    t("value -> pinned host", lambda: host.copy_(r.value.values))
    print("  phases", {k: round(v, 2) for k, v in r.stats.phases_ms().items()})
