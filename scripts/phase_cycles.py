"""Per-phase cycle split of the solve kernel (needs a -DPHJ_TIMING build):

    PHJ_LIB_PATH=.../libphj_timing.so python scripts/phase_cycles.py c2

Counts are summed over warps (lane 0 of each warp) for one full patchy step
(coarse + patch solves)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import _lib, configs, patchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
w = configs.CONFIGS[name](dtype=dtype)
plans = patchy.make_plans(w.spec, w.pcfg)
lib = _lib.load()
fn = lib.phj_dbg_phase_cycles
fn.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 12)()
names = ["sweep_prologue", "fetch", "labels", "eval", "store", "maxch", "mark", "post_sweep",
         "sweep_flush", "cta_wait", "grid_sync", "-"]
for i in range(2):
    fn(buf)
    phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans, outputs=False)
    torch.cuda.synchronize()
    fn(buf)
tot = sum(buf)
print(json.dumps({"config": name, "dtype": dtype, "frac": {n: round(buf[i] / tot, 4) for i, n in enumerate(names)},
                  "cycles": {n: buf[i] for i, n in enumerate(names)}}))
