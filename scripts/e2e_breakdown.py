"""Where the public-API (e2e) step spends time beyond the device pipeline."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.CONFIGS[name]()


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"  {label:30s} {1000 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return r


for i in range(4):
    print("step", i)
    plans = t("make_plans", lambda: patchy.make_plans(w.spec, w.pcfg))
    t("run_patchy(plans, outputs=False)", lambda: phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans,
                                                                outputs=False))
    r = t("run_patchy(public, outputs)", lambda: phj.run_patchy(w.spec, w.pcfg, w.cfg))
    t("value D2H", lambda: r.value.values.cpu())
    print("  phases", {k: round(v, 1) for k, v in r.stats.phases_ms().items()})
