"""Fine-grained wall-clock split of one pipeline step (synchronised before and
after every wrapped internal function, so host glue counts): where the time
outside the two dominant kernels goes."""
import functools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1109_3577_b200 import configs, patchy, solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
w = configs.CONFIGS[name](dtype=dtype)
acc = {}
depth = [0]


def wrap(mod, fn):
    f = getattr(mod, fn)

    @functools.wraps(f)
    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        depth[0] += 1
        try:
            return f(*a, **k)
        finally:
            depth[0] -= 1
            torch.cuda.synchronize()
            key = "  " * depth[0] + fn
            acc[key] = acc.get(key, 0.0) + 1000 * (time.perf_counter() - t0)

    setattr(mod, fn, g)


for fn in ("solve_full_internal", "lift_internal", "band_schedule", "transport_internal",
           "argmax_batched", "assemble_internal", "solve_patches_internal", "_resolve_parts",
           "_transport_and_argmax", "init_working", "count_labels", "plan_interior_serial"):
    wrap(patchy, fn)
for fn in ("device_solve", "feedback_internal"):
    wrap(solver, fn)
    if hasattr(patchy, fn):
        wrap(patchy, fn)
plans = patchy.make_plans(w.spec, w.pcfg)
fake = os.environ.get("PHJ_FAKE_WORLD")  # "rank,world": this rank's share, no collectives
if fake:
    from paper_1109_3577_b200 import dist
    fr, fw = (int(x) for x in fake.split(","))
    dist.world = lambda: (fr, fw)
for step in range(3):
    acc.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    patchy.run_patchy(w.spec, w.pcfg, w.cfg, plans=plans, outputs=False)
    torch.cuda.synchronize()
    total = 1000 * (time.perf_counter() - t0)
    out = {"config": name, "dtype": dtype, "step": step, "fake_world": fake, "total_ms": round(total, 2),
           "transport_kernel_ms": round(patchy.TRANSPORT_DIAG.get("kernel_ms", 0.0), 2),
           "split_ms": {k: round(v, 2) for k, v in acc.items()}}
    print(json.dumps(out), flush=True)
