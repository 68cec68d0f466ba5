"""Functional check of the multi-rank path on ONE GPU (no kernel waits on
another rank's kernel: ranks only meet in host-issued collectives).  Both
ranks run on cuda:0 with the gloo backend (NCCL refuses two ranks on one
device); the result must equal the single-rank run.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
        scripts/multi_rank_check.py c2 257
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as td  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
KW = dict(nxy=n, nth=16, cxy=(n - 1) // 4 + 1, cth=8) if name == "c4" else dict(n=n)
if name == "c5":
    KW["dtype"] = "float64"  # (its default is the fp32 workload; the 1e-9 bar below is fp64)
torch.cuda.set_device(0)
w = configs.CONFIGS[name](**KW)
single = phj.run_patchy(w.spec, w.pcfg, w.cfg).value.values.clone()
single_col = None
td.init_process_group("gloo")
rank = td.get_rank()
w = configs.CONFIGS[name](**KW)
res = phj.run_patchy(w.spec, w.pcfg, w.cfg)
v = res.value.values
fin = (single < 1e8) & (v < 1e8)
d = float((v - single)[fin].abs().max()) if fin.any() else 0.0
same_reach = bool(torch.equal(single < 1e8, v < 1e8))
print(f"rank {rank}: schedule {w.cfg.schedule} max|v_multi - v_single| = {d:.3e}, "
      f"reachability equal {same_reach}, patches {[s.sweeps for s in res.patch_stats][:8]}",
      flush=True)
ok = torch.tensor([1 if (d <= 1e-9 and same_reach) else 0])
td.all_reduce(ok, op=td.ReduceOp.MIN)
td.destroy_process_group()
if rank == 0:
    print("MULTI-RANK", "OK" if int(ok) == 1 else "MISMATCH")
sys.exit(0 if int(ok) == 1 else 1)
