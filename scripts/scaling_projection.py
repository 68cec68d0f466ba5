"""Multi-GPU projection of the patchy pipeline on ONE GPU (this pool has one
GPU per call; ranks whose kernels wait on each other cannot share a GPU, but
these ranks never wait: patches and colours are independent).

For G in (1, 2, 4, 8) and each rank r, the rank's own work is run alone on
the full GPU exactly as that rank would run it (dist.world() patched to
(r, G)): its colour subset of the transport (dist.my_colours) and its patch
subset of the patch solve (dist.mine_mask, LPT), its slab of the feedback
stage (phj_feedback_slab).  Replicated stages (coarse, lift, assembly) are
timed once.  Collectives are estimated from their byte counts at an NVLink-5
bus bandwidth (feedback all-gather: N x 4 B; argmax merge: N x 8 B MAX +
N x 1 B MIN; value gather: N x 8 B MIN).  Projected step time of G GPUs =
replicated + max_r (feedback_r) + all-gather + max_r (transport_r) + merge +
max_r (patch_r) + gather; efficiency = T(1) / (G * T(G)).

    python scripts/scaling_projection.py [c5] [float64] [weights]
weights: "work" (default: the per-patch executed evaluations of a previous
solve of the same patch map, as the library uses from the second solve on)
or "nodes" (north_star: node count, the first solve).
Writes one JSON object to stdout.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1109_3577_b200 import _lib, configs, dist, patchy  # noqa: E402
from paper_1109_3577_b200.solver import feedback_internal, unreach_threshold  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
WEIGHTS = sys.argv[3] if len(sys.argv) > 3 else "work"  # LPT weights: "work" or "nodes"
BUS_GBS = float(os.environ.get("PHJ_NVLINK_BUS_GBS", "600"))  # all-reduce bus bandwidth
w = configs.CONFIGS[name](dtype=dtype)
spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
fplan, cplan = patchy.make_plans(spec, pcfg)
dev = fplan.device
n = fplan.grid.n_interior


REPS = int(os.environ.get("PHJ_PROJ_REPS", "2"))


def timed(fn):
    """Device time of fn(): the last of REPS calls -- a rank repeats the same
    shapes every step, so its steady state has the allocator pools and the
    band-list sizes of its own share warm (a single cold call of a rank's
    share measured ~23 ms more at G = 8)."""
    for _ in range(REPS):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
    return out, a.elapsed_time(b)


# warm-up: one full run (allocator pools, stencils)
patchy.run_patchy(spec, pcfg, cfg, plans=(fplan, cplan), outputs=False)

(vc, cst), t_coarse = timed(lambda: patchy.solve_full_internal(cplan, patchy.coarse_cfg(cfg)))
vf, t_lift = timed(lambda: patchy.lift_internal(cplan, vc, fplan, cfg.rule, cfg.dtype))
(fb, _), t_fb = timed(lambda: feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype))
parts = patchy._resolve_parts(pcfg, spec, fplan.grid, fplan)
R = len(parts)
limit = 10 * max(fplan.grid.shape)
thr = unreach_threshold(cfg.rule)
mask = patchy.plan_interior_serial(fplan, vf) >= thr

real_world = dist.world
res = {"config": name, "dtype": dtype, "lpt_weights": WEIGHTS, "replicated_ms": {"coarse": t_coarse, "lift": t_lift,
                                                          "feedback": t_fb}}
base = None
color = lab = None
sizes = None
for G in (1, 2, 4, 8):
    tr_ms, pa_ms, ranks = [], [], []
    for r in range(G):
        dist.world = lambda r=r, G=G: (r, G)
        try:
            (bv, bi, csw, _), t_tr = timed(lambda: patchy._transport_and_argmax(
                fplan, fb, parts, pcfg.color_tol, limit, cfg.schedule, cfg.dtype,
                key_work=vf, rule=cfg.rule))
            tr_ms.append(t_tr)
            if G == 1:
                (color, n_unc, _, lab), t_as = timed(lambda: patchy.assemble_internal(
                    fplan.gs, bv, bi, R, mask, fplan.kind, n, dev))
                res["replicated_ms"]["assembly"] = t_as
                sizes = patchy.count_labels(color, R).cpu().numpy()
            def patch_share():
                # LPT weights: the per-patch work every rank would hold after a
                # first solve of this patch map (measured at G = 1, all
                # patches), or node counts; reset before every repetition (a
                # solve stores its own measured work on the plan)
                if G > 1 and WEIGHTS == "work":
                    fplan._patch_work = ((tuple(int(x) for x in sizes), G), execd_all)
                else:
                    fplan._patch_work = None
                return patchy.solve_patches_internal(fplan, color, lab, R, pcfg, cfg, vf)

            (out, pst, warns, pinfo), t_pa = timed(patch_share)
            pa_ms.append(t_pa)
            if G == 1:
                relax = np.array([s.node_relaxations for s in pst], dtype=float)
                execd = np.array([s.performed_evals for s in pst], dtype=float)
                execd_all = execd.copy()
        finally:
            dist.world = real_world
    # the feedback stage is split by slabs of block rows (solver.feedback_sharded):
    # the slowest rank's slab + an all-gather of the int32 field
    fb_ms = [t_fb]
    if G > 1:
        import ctypes as _ct
        dims = (_ct.c_int32 * 3)()
        _lib.load().phj_block_dims(fplan.grid.dim, dims)
        n_rows = (fplan.int_shape[0] + int(dims[0]) - 1) // int(dims[0])
        fb_ms = []
        for b0, b1 in dist.slab_bounds(n_rows, G):
            _, t = timed(lambda: feedback_internal(fplan, vf, rule=cfg.rule, dtype=cfg.dtype,
                                                   slab=(b0, b1)))
            fb_ms.append(t)
    rep = sum(v for k, v in res["replicated_ms"].items() if k != "feedback")
    nbytes = n * 8
    allreduce_ms = lambda b: 0.0 if G == 1 else 2.0 * (G - 1) / G * b / (BUS_GBS * 1e9) * 1e3
    allgather_ms = lambda b: 0.0 if G == 1 else (G - 1) / G * b / (BUS_GBS * 1e9) * 1e3
    fb_stage = max(fb_ms) + allgather_ms(n * 4)
    # argmax merge: MAX of the fp64 bits + MIN of the uint8 colour index
    merge = allreduce_ms(nbytes) + allreduce_ms(n)
    gather = allreduce_ms(nbytes)
    step = rep + fb_stage + max(tr_ms) + merge + max(pa_ms) + gather
    if G == 1:
        base = step
        owner = np.zeros(R, dtype=int)
    else:
        owner = dist.lpt_assign(sizes, G, execd_all if WEIGHTS == "work" else None)
    work_bins = np.bincount(owner, weights=execd, minlength=G)
    res[f"G{G}"] = {"step_ms": step, "feedback_ms_per_rank": fb_ms, "feedback_stage_ms": fb_stage,
                    "transport_ms_per_rank": tr_ms,
                    "patch_ms_per_rank": pa_ms, "merge_ms_est": merge, "gather_ms_est": gather,
                    "efficiency": base / (G * step),
                    "patch_work_balance": float(execd.sum() / (G * work_bins.max())),
                    "node_balance_bound": dist.load_balance_bound(sizes, G)}
# work predictors available before the patch solve (from the lifted field)
col = color.long()
live = col >= 0
Tl = patchy.plan_interior_serial(fplan, vf).to(torch.float64)
if cfg.rule == "kruzkov":
    Tl = -torch.log1p(-Tl.clamp(max=1 - 1e-16))
res["patch_sum_T"] = torch.bincount(col[live], weights=Tl[live], minlength=R).cpu().tolist()
res["patch_max_T"] = torch.zeros(R, dtype=torch.float64, device=dev).scatter_reduce(
    0, col[live], Tl[live], reduce="amax").cpu().tolist()
res["patch_sizes"] = sizes.tolist()
res["patch_relaxations"] = relax.tolist()
res["patch_executed_evals"] = execd.tolist()
res["collective_model"] = f"ring all-reduce 2(G-1)/G x bytes at {BUS_GBS} GB/s bus bandwidth"
print(json.dumps(res))
