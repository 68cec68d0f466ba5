"""Compare fp32 and fp64 pipelines stage by stage (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65
mk = configs.CONFIGS[name]
out = {}
for dt in ("float64", "float32"):
    w = mk(n=n, dtype=dt)
    w.pcfg.color_tol = 1e-12
    r = phj.run_patchy(w.spec, w.pcfg, w.cfg)
    out[dt] = r
    print(dt, "coarse sweeps", r.coarse_stats.sweeps, r.coarse_stats.converged,
          "patch sweeps", [s.sweeps for s in r.patch_stats][:8], r.stats.warnings[:3])
a, b = out["float64"], out["float32"]
la, lb = a.lifted.numpy(), b.lifted.numpy()
fin = np.isfinite(la) & (la < 1e8)
print("lifted max diff", np.abs(la - lb)[fin].max(), "reach mismatch", int(((la < 1e8) != (lb < 1e8)).sum()))
fa, fb = a.feedback.indices.cpu().numpy(), b.feedback.indices.cpu().numpy()
print("feedback diffs", int((fa != fb).sum()), "of", fa.size)
ca, cb = a.patch_map.color.cpu().numpy(), b.patch_map.color.cpu().numpy()
print("label diffs", int((ca != cb).sum()))
va, vb = a.value.numpy(), b.value.numpy()
d = np.abs(va - vb)
d[(va > 1e8) | (vb > 1e8)] = 0
i = np.unravel_index(np.argmax(d), d.shape)
print("value max diff (T)", d.max(), "at", i, va[i], vb[i],
      "unreach mismatch", int(((va > 1e8) != (vb > 1e8)).sum()))
