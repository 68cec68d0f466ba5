"""Debug: C4 nodes the device reaches but the oracle map (under the device's
patch map) cannot -- candidate by candidate for the first such node."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from oracle import pipeline as O
import oracle_cases as C
from paper_1109_3577_b200 import configs, patchy
from paper_1109_3577_b200.solver import feedback_internal

nxy = int(sys.argv[1]) if len(sys.argv) > 1 else 257
w = configs.c4(nxy=nxy, nth=max(16, (nxy - 1) // 2))
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
pcfg.color_tol = 1e-8
res = patchy.run_patchy(spec, pcfg, cfg)
fine = C.from_workload(w, "fine")
g = fine.grid
v = res.value.numpy().reshape(-1)
v = np.where(v >= 0.5e9, 1.0, -np.expm1(-v))
col = res.patch_map.color.cpu().numpy()
r = O.residual(v, fine, col, rule="kruzkov")
print("missed", r.missed, "spurious", r.spurious, "r", r.r)
sp = r.spurious_serials
print("spurious serials", sp[:10], "idx", [np.unravel_index(s, g.shape) for s in sp[:5]])
s0 = int(sp[0])
i0 = np.array(np.unravel_index(s0, g.shape))
iflat = g.interior_flat()
print("node", i0.tolist(), "label", col[s0], "v", v[iflat[s0]])
cc = col.reshape(g.shape)
vv = v.reshape(g.ext_shape)
for d in np.ndindex(3, 3, 3):
    j = i0 + np.array(d) - 1
    j[2] %= g.shape[2]
    if 0 <= j[0] < g.shape[0] and 0 <= j[1] < g.shape[1]:
        print("  nb", (np.array(d) - 1).tolist(), "label", int(cc[tuple(j)]), "v", float(vv[tuple(j + 1)]))
X = g.interior_points()[s0]
print("X", X)
for c, a in enumerate(spec.control_set.controls):
    F = np.array([np.cos(X[2]), np.sin(X[2]), a[0]])
    h = g.k_step / np.linalg.norm(F)
    P = X + h * F
    t = (P - g.ext_lo) / g.spacing
    cell = np.floor(t).astype(int); loc = t - cell
    loc[loc < 1e-12] = 0; loc[loc > 1 - 1e-12] = 1
    print(" ctrl", c, "cell-node offset", (cell - (i0 + 1)).tolist(), "loc", loc.round(6).tolist())
