"""Where a two-rank run (gloo, both ranks on cuda:0) differs from the
single-rank run: labels, values, and the oracle's fixed-point residual of
both results under their own patch maps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as td  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
torch.cuda.set_device(0)
w = configs.CONFIGS[name](n=n, dtype="float64")
r1 = phj.run_patchy(w.spec, w.pcfg, w.cfg)
single = r1.value.values.clone()
col1 = r1.patch_map.color.clone()
r1b = phj.run_patchy(w.spec, w.pcfg, w.cfg)
rep = float((r1b.value.values - single)[single < 1e8].abs().max())
td.init_process_group("gloo")
rank = td.get_rank()
w = configs.CONFIGS[name](n=n, dtype="float64")
res = phj.run_patchy(w.spec, w.pcfg, w.cfg)
v = res.value.values
col = res.patch_map.color
fin = (single < 1e8) & (v < 1e8)
d = (v - single).abs()
d[~fin] = 0
imax = int(d.argmax())
if rank == 0:
    print(f"single repeat diff {rep:.3e}; multi-single max {float(d.max()):.3e} at {imax} "
          f"(v_multi {float(v.view(-1)[imax]):.12f}, v_single {float(single.view(-1)[imax]):.12f}, "
          f"label multi {int(col.view(-1)[imax])} single {int(col1.view(-1)[imax])}); "
          f"nodes > 1e-9: {int((d > 1e-9).sum())}; label diffs {int((col != col1).sum())}", flush=True)
    from oracle import pipeline as O
    import oracle_cases as C
    fine = C.from_workload(w, "fine")
    for tag, vv, cc in (("single", single, col1), ("multi", v, col)):
        x = vv.cpu().numpy().reshape(-1)
        x = np.where(x >= 0.5e9, 1.0, -np.expm1(-x))
        r = O.residual(x, fine, cc.cpu().numpy().reshape(-1), rule="kruzkov")
        print(tag, "residual", r.r, "bound", O.contraction_bound(fine, "kruzkov", r.r),
              (r.missed, r.spurious), flush=True)
td.barrier()
td.destroy_process_group()
