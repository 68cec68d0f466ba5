"""Host-side profile (cProfile) of the public-API step run_patchy(spec, pcfg, cfg)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1109_3577_b200 as phj  # noqa: E402
from paper_1109_3577_b200 import configs  # noqa: E402

w = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
for _ in range(3):
    phj.run_patchy(w.spec, w.pcfg, w.cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    r = phj.run_patchy(w.spec, w.pcfg, w.cfg)
    torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr).sort_stats("tottime")
st.print_stats(25)
