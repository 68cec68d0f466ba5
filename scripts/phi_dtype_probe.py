"""C5 (fp32) step with fp32 vs fp64 colour fields: phases and transport kernel time."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs, patchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.CONFIGS[name](dtype="float32")
plans = patchy.make_plans(w.spec, w.pcfg)
for fp32 in (True, False, True):
    patchy.TRANSPORT_PHI_FP32 = fp32
    for _ in range(2):
        res = phj.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans, outputs=False)
        torch.cuda.synchronize()
    print(json.dumps({"phi_fp32": fp32, "phases": res.stats.phases_ms(),
                      "transport_kernel_ms": patchy.TRANSPORT_DIAG.get("kernel_ms"),
                      "max_mem_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    torch.cuda.reset_peak_memory_stats()
