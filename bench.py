"""Benchmark: SL node-updates/s and time-to-converge of the patchy pipeline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--dtype float64|float32]

One step = one full patchy solve of the workload (coarse solve -> lift ->
feedback -> colour transport -> assembly -> patch solves) to convergence,
i.e. the time-to-converge (``time_to_converge_ms``, the figure to compare
across schedules).  The workloads use the asynchronous device schedule
(DESIGN.md §3.1c): the patch solves stop when no node can change by more
than activity_tol (1e-12 in time units) -- a tighter stop than the
reference's per-sweep max change <= tol (1e-8); the coarse stage is
deterministic block-Jacobi.  Units = candidate evaluations (node x control
x sweep, ``candidate_evals`` of _kernels.py:76) the value solves actually
performed (coarse + patch solves) -- a work rate, so a schedule that wastes
fewer evaluations can score lower while converging sooner; the reference's
dense count is reported beside it.

* ``value``  -- device-resident: plans (stencils, node kinds, coefficients)
  built before timing, each step timed with CUDA events, L2 flushed between
  steps (256 MiB write, untimed).
* ``e2e``    -- through the public API ``run_patchy(spec, pcfg, cfg)`` from
  host inputs (problem description -> device tables: H2D) to the value field
  in a pinned host buffer (D2H), all inside the timed region; wall clock over
  max(5, min(K, 10)) steps after W untimed calls.
* ``roofline`` -- dominant kernel = the fine patch solve launch; algorithmic
  FP64 (FP32) flops per candidate 2*2^d + 1 x candidates the
  kernel executed (after exact octant pruning) / its CUDA-event duration,
  against the FP pipe peak measured here with ``phj_peak_flops``
  (MEASURED_PEAKS.json has no FP64/FP32 figure); ``logical_tflops`` counts
  every admissible control of every swept node instead.
* ``cpu_baseline`` -- the C oracle port (oracle/phj_oracle.c, reference
  update rule, OpenMP over all host cores) timed on Jacobi sweeps of the same
  fine grid (bounded sample), rank 0 at N=1.

``--impl reference`` runs that CPU port alone (rank 0; others exit 0).
Multi-GPU: one process per GPU (torchrun), patches LPT-split across ranks,
one MIN all-reduce gathers v; time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SL node-updates/sec (nodes x controls x iters/s)"
UNIT = "node-updates/s"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--dtype", default="float64")
    p.add_argument("--rule", default="kruzkov")
    p.add_argument("--cpu-sweeps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def _workload(args):
    from paper_1109_3577_b200 import configs

    kw = {"rule": args.rule, "dtype": args.dtype}
    return configs.CONFIGS[args.config](**kw)


def _flops_per_candidate(dim: int) -> int:
    return 2 * 2 ** dim + 1


# -- CPU port (oracle) ------------------------------------------------------------------


def cpu_port_rate(w, sweeps: int, threads: int):
    """Jacobi sweeps of the C oracle over the fine grid of workload w
    (reference update rule, on-the-fly feet).  Returns (updates/s, evals,
    seconds, sample description)."""
    from oracle import pipeline as O
    from paper_1109_3577_b200 import dynamics

    spec = w.spec
    g = spec.make_grid(w.pcfg.fine_nodes)
    og = O.OGrid(g.lo, g.hi, g.shape, g.periodic)
    X = og.interior_points()
    tgt = spec.target.contains(X)
    model = spec.model
    if isinstance(model, dynamics.Dubins):
        pr = O.OProblem(og, "dubins", spec.control_set.controls, tgt)
    else:
        sp = model.speed
        speed = np.full(og.n_interior, float(sp)) if np.isscalar(sp) else np.asarray(sp(X))
        pr = O.OProblem(og, "scaled", spec.control_set.controls, tgt, speed=speed)
    u = O.init_field(pr, "reference")
    order = np.arange(og.n_interior, dtype=np.int64)
    O.sweep(u, pr, order[: min(order.size, 4096)], rule="reference", mode="jacobi",
            nthreads=threads)  # warm (page-in)
    t0 = time.perf_counter()
    ev = 0
    for _ in range(sweeps):
        _, _, ne = O.sweep(u, pr, order, rule="reference", mode="jacobi", nthreads=threads)
        ev += ne
    dt = time.perf_counter() - t0
    sample = (f"{sweeps} Jacobi sweeps of the {'x'.join(map(str, g.shape))} fine grid, "
              f"{pr.nc} controls, reference rule, oracle/phj_oracle.c OpenMP")
    return ev / dt, ev, dt, sample


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# -- clocks ---------------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -- GPU arm ------------------------------------------------------------------------------


def measure_peak(dtype: str) -> float:
    """FP pipe peak (TFLOP/s) from phj_peak_flops: 8 x SMs CTAs x 256 threads
    x 8 independent FMA chains."""
    import torch

    from paper_1109_3577_b200 import _lib

    lib = _lib.load()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    did = _lib.F32 if dtype == "float32" else _lib.F64
    iters = 2000
    for _ in range(2):
        _lib.check(lib.phj_peak_flops(did, iters, _lib.ptr(sink), _lib.stream_handle()), "peak")
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.phj_peak_flops(did, iters, _lib.ptr(sink), _lib.stream_handle()), "peak")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        flops = 8 * lib.phj_num_sms() * 256 * iters * 16 * 8 * 2.0
        best = max(best, flops / (ms * 1e-3) / 1e12)
    return best


def run_ours(args):
    import torch
    import torch.distributed as td

    import paper_1109_3577_b200 as phj
    from paper_1109_3577_b200 import _lib, patchy

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        # PHJ_DIST_BACKEND=gloo: two ranks on one GPU for functional checks of
        # the multi-rank bench path (NCCL needs one device per rank)
        backend = os.environ.get("PHJ_DIST_BACKEND", "nccl")
        if backend == "nccl":
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            td.init_process_group(backend)
    lib = _lib.load()
    w = _workload(args)
    spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
    dim = spec.dim

    fplan, cplan = patchy.make_plans(spec, pcfg)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def step(timed: bool):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        res = phj.run_patchy(spec, pcfg, cfg, plans=(fplan, cplan), outputs=False)
        b.record()
        torch.cuda.synchronize()
        return res, a.elapsed_time(b)

    for _ in range(args.warmup):
        step(False)
    if world > 1:
        td.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    l0 = lib.phj_launch_count()
    tot_ms, perf, dense, kern_ms, kern_evals, patch_sweeps = 0.0, 0, 0, 0.0, 0, 0
    kern_exec = 0
    res = None
    for _ in range(args.steps):
        res, ms = step(True)
        tot_ms += ms
        perf += res.stats.performed_evals
        dense += res.stats.candidate_evals
        k = res.stats.kernels.get("patch_solve", {})
        kern_ms += k.get("kernel_ms", 0.0)
        kern_evals += k.get("performed", 0)
        kern_exec += k.get("executed", 0)
        patch_sweeps = k.get("sweeps", 0)
    launches = lib.phj_launch_count() - l0
    clocks = clk.stop()
    torch.cuda.synchronize()
    if world > 1:
        td.barrier()
        t = torch.tensor([tot_ms, kern_ms], device="cuda", dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        tot_ms_max, kern_ms_max = t.tolist()
        c = torch.tensor([perf, dense, kern_evals, kern_exec, launches], device="cuda",
                         dtype=torch.float64)
        td.all_reduce(c, op=td.ReduceOp.SUM)
        perf, dense, kern_evals, kern_exec, launches = [int(x) for x in c.tolist()]
    else:
        tot_ms_max, kern_ms_max = tot_ms, kern_ms
    value = perf / (tot_ms_max * 1e-3)

    # -- e2e: public API from host inputs, D2H of the value field ----------------
    e2e_val, h2d, d2h = None, 0, 0
    # wall-clock timed: at least 5 steps (host jitter), after the same number
    # of untimed public-API warm-up calls as the device loop (the first calls
    # with fresh plans grow the allocator's pools)
    e2e_steps = max(5, min(args.steps, 10))
    # the result lands in a pinned host buffer (allocated once, like a
    # caller's output array); the copy itself is inside the timed region
    r = phj.run_patchy(spec, pcfg, cfg)
    host = torch.empty(r.value.values.shape, dtype=r.value.values.dtype, pin_memory=True)
    for _ in range(max(0, args.warmup)):
        r = phj.run_patchy(spec, pcfg, cfg)
        host.copy_(r.value.values)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_perf = 0
    for _ in range(e2e_steps):
        r = phj.run_patchy(spec, pcfg, cfg)
        host.copy_(r.value.values)
        e_perf += r.stats.performed_evals
    torch.cuda.synchronize()
    e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e_dt], device="cuda", dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        e_dt = float(t.item())
        c = torch.tensor([e_perf], device="cuda", dtype=torch.float64)
        td.all_reduce(c, op=td.ReduceOp.SUM)
        e_perf = int(c.item())
    e2e_val = e_perf / e_dt
    d2h = host.numel() * host.element_size()
    st = fplan.stencils
    h2d = int(st.oct_start.nbytes + st.ctrl.nbytes + st.nzmask.nbytes + st.weights.nbytes +
              st.cost.nbytes) * 2 + 8 * 64

    if rank != 0:
        td.destroy_process_group()
        return
    peak = measure_peak(args.dtype)
    fl = _flops_per_candidate(dim)
    # hardware work: stencil entries the kernel really evaluated (after octant
    # pruning, incl. padding and masked lanes); the logical rate (every
    # admissible control of every swept node) is reported beside it
    achieved = kern_exec * fl / (kern_ms_max * 1e-3) / 1e12 if kern_ms_max > 0 else 0.0
    logical = kern_evals * fl / (kern_ms_max * 1e-3) / 1e12 if kern_ms_max > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        thr = host_threads()
        rate, ev, dt, sample = cpu_port_rate(w, args.cpu_sweeps, thr)
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample,
               "seconds": dt}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.dtype == "float64" else "f32", "data": "synthetic",
        "config": {"workload": w.description, "name": w.name, "fine": list(w.fine_shape),
                   "coarse": list(w.coarse_shape), "controls": int(len(spec.control_set)),
                   "patches": pcfg.n_patches, "rule": args.rule, "tol": cfg.tol,
                   "color_tol": pcfg.color_tol, "l2": "flushed between steps (256 MiB write)",
                   "schedule": cfg.schedule, "inner_sweeps": cfg.inner_for(dim),
                   "activity_tol": cfg.act_tol,
                   "parallelism": f"patch-lpt{world}"},
        "time_to_converge_ms": tot_ms_max / args.steps,
        "dense_equivalent_updates_per_s": dense / (tot_ms_max * 1e-3),
        "performed_updates_per_step": perf // args.steps,
        "patch_solve_sweeps": patch_sweeps,
        "phases_ms": {k: round(v, 3) for k, v in res.stats.phases_ms().items()},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": {"bound": "fp64" if args.dtype == "float64" else "fp32",
                     "kernel": ("solve_async_kernel (fine patch solve, one persistent launch)"
                                if cfg.schedule == "async" else
                                "solve_kernel (fine patch solve, one cooperative launch)"),
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "flops_per_candidate": fl,
                     "executed_candidates": kern_exec // max(1, args.steps),
                     "logical_candidates": kern_evals // max(1, args.steps),
                     "logical_tflops": logical,
                     "peak_source": "measured here: phj_peak_flops FMA-chain probe"},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": int(launches // max(1, world) * world),
    }
    print(json.dumps(out))
    if world > 1:
        td.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = _workload(args)
    thr = host_threads()
    from oracle import pipeline as O

    O.build_oracle()
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_port_rate(w, 1, thr)
    rates, secs = [], 0.0
    sample = ""
    for _ in range(args.steps):
        r, ev, dt, sample = cpu_port_rate(w, 1, thr)
        rates.append(r)
        secs += dt
    value = float(np.mean(rates))
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": int(os.environ.get(
           "WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": w.description, "name": w.name, "fine": list(w.fine_shape),
                      "controls": int(len(w.spec.control_set)), "rule": "reference"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
