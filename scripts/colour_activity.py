"""How many colours a warp block of the 3D transport holds above a threshold
(the sticky colour masks of the value-ordered pass grow with every colour
whose change exceeded act_eps once): histogram per block, from the colour
fields of one transport."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.CONFIGS[name](dtype="float64")
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg))
vf = patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype)
fb, _ = feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype)
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
R = len(parts)
allp = np.concatenate([np.asarray(parts[j], dtype=np.int64) for j in range(R)])
flat = fplan.user_serials_to_internal_flat(allp)
bounds = np.cumsum([0] + [len(parts[j]) for j in range(R)])
parts_flat = [flat[bounds[i]:bounds[i + 1]] for i in range(R)]
bands = patchy.transport_bands(fplan, vf, fb, cfg.rule)
phi, _, csw, upd = patchy.transport_internal(fplan, fb, parts_flat, pcfg.color_tol,
                                             10 * max(fplan.grid.shape), "jacobi",
                                             torch.float64, bands=bands)
out = {"config": name, "kernel_ms": patchy.TRANSPORT_DIAG["kernel_ms"], "mover_updates": int(upd),
       "band_entries": int(bands[0].numel()), "n_band": int(bands[2]),
       "sweeps": [int(min(map(abs, csw))), int(max(map(abs, csw)))]}
M = fplan.int_shape
for thr in (1e-12, 1e-7, 1e-5, 1e-4, 1e-3, 1e-2):
    cnt = None
    for j in range(R):
        a = fplan.interior_int(phi[j])
        pad = [0, (-M[2]) % 8, 0, (-M[1]) % 8]
        a = torch.nn.functional.pad(a, pad)
        blk = a.view(M[0], a.shape[1] // 8, 8, a.shape[2] // 8, 8).amax(dim=(2, 4)) > thr
        cnt = blk.to(torch.int32) if cnt is None else cnt + blk
    h = torch.bincount(cnt.view(-1), minlength=9)[:9].tolist()
    out[f"thr{thr:g}"] = {"mean_colours_reached_blocks": float(cnt[cnt > 0].float().mean()),
                          "hist0_8": h, "max": int(cnt.max())}
print(json.dumps(out), flush=True)
