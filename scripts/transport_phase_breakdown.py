"""Wall-time split of run_patchy's transport phase (synchronising wrappers
around its stages; the public API path, fresh plans each step)."""
import functools
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

acc = {}


def timed(mod, name):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + 1000 * (time.perf_counter() - t0)
        return r
    setattr(mod, name, g)


for n in ("_resolve_parts", "transport_internal", "argmax_batched", "assemble_internal",
          "plan_interior_serial", "_transport_and_argmax"):
    timed(patchy, n)
w = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
for i in range(3):
    acc.clear()
    r = phj.run_patchy(w.spec, w.pcfg, w.cfg)
    torch.cuda.synchronize()
    print({k: round(v, 2) for k, v in acc.items()}, "kernel",
          round(patchy.TRANSPORT_DIAG.get("kernel_ms", 0), 2), flush=True)
