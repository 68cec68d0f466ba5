"""Benchmark: SL node-updates/s and time-to-converge of the patchy pipeline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c5] [--dtype float64|float32]

Default workload: BASELINE.json configs[4] ("c5": 513^3, 96 Fibonacci
controls, 32 seeded-random patches, Kruzkov fp64) -- the configuration the
metric ("at 1/2/4/8 B200") is quoted on; the other configs are parity cases
and extra bench lines (``--config c2`` etc.).

One step = one full patchy solve of the workload (coarse solve -> lift ->
feedback -> colour transport -> assembly -> patch solves) to convergence;
``time_to_converge_ms`` is its device time.  The patch solves use the
asynchronous schedule (stop when no node can change by more
than activity_tol = 1e-12 in time units), the coarse stage deterministic
block-Jacobi.

* ``value``  -- node-updates/s = candidate evaluations (node x control, one
  interpolation + min each: ``candidate_evals`` of _kernels.py:76) the value
  solves EXECUTED (coarse once + patch solves of every rank; real controls
  only, after activity skipping and the exact octant pruning) / device
  time-to-converge.  ``logical_updates_per_s`` counts every admissible
  control of every node relaxation instead (what a prune-free kernel would
  evaluate for the same relaxations).  Plans are built before timing, each
  step timed with CUDA events, L2 flushed between steps (256 MiB write).
* ``e2e``    -- the same executed count through the public API
  ``run_patchy(spec, pcfg, cfg)`` from host inputs (problem description ->
  device tables: H2D) to the value field in a pinned host buffer (D2H), all
  inside the wall-clock timed region, over max(5, min(K, 10)) steps after W
  untimed calls.
* ``roofline`` -- dominant kernel = the fine patch-solve launch; algorithmic
  FP64 (FP32) flops per candidate 2*2^d + 1 x real candidates it
  executed / its CUDA-event duration, against the FP pipe peak measured in
  the same run with ``phj_peak_flops`` (MEASURED_PEAKS.json has no FP64/FP32
  figure); ``traffic`` = DRAM bytes per launch from the committed ncu capture.
* ``cpu_baseline`` -- the C oracle port (oracle/phj_oracle.c, reference
  update rule, OpenMP over all host cores) on Jacobi sweeps of a bounded slab
  of the same fine grid (~10 s), rank 0 at N=1; ``time_to_converge_est_s`` =
  the dense work of a Jacobi CPU solve to the same tol (per-patch Jacobi sweep
  counts measured on the device's Jacobi schedule x patch nodes x controls,
  + coarse) / that rate.

``--impl reference`` runs that CPU port alone (rank 0; others exit 0), one
bounded slab sample per step.  Multi-GPU: one process per GPU (torchrun),
patches LPT-split across ranks, one MIN all-reduce gathers v; time = max
over ranks.
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
    p.add_argument("--config", default="c5")
    p.add_argument("--dtype", default="float64")
    p.add_argument("--rule", default="kruzkov")
    p.add_argument("--cpu-seconds", type=float, default=10.0,
                   help="target CPU seconds of the bounded cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def _workload(args):
    from paper_1109_3577_b200 import configs

    kw = {"rule": args.rule, "dtype": args.dtype}
    return configs.CONFIGS[args.config](**kw)


def _config(w, args, world: int) -> dict:
    """The workload description shared by both arms."""
    cfg, pcfg = w.cfg, w.pcfg
    return {"workload": w.description, "name": w.name, "fine": list(w.fine_shape),
            "coarse": list(w.coarse_shape), "controls": int(len(w.spec.control_set)),
            "patches": pcfg.n_patches, "rule": args.rule, "tol": cfg.tol,
            "color_tol": pcfg.color_tol, "l2": "flushed between steps (256 MiB write)",
            "schedule": cfg.schedule, "inner_sweeps": cfg.inner_for(w.spec.dim),
            "activity_tol": cfg.act_tol, "parallelism": f"patch-lpt{world}"}


def _flops_per_candidate(dim: int) -> int:
    return 2 * 2 ** dim + 1


# -- CPU port (oracle) ------------------------------------------------------------------


class CpuPort:
    """The C oracle on the fine grid of workload w (reference update rule,
    on-the-fly feet, Jacobi; test infrastructure used as the CPU baseline)."""

    def __init__(self, w, threads: int):
        from oracle import pipeline as O
        from paper_1109_3577_b200 import dynamics

        self.O = O
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
        del X
        self.pr, self.g, self.threads = pr, g, threads
        self.u = O.init_field(pr, "reference")
        self.u_in = self.u.copy()           # Jacobi input, allocated once
        self.kind = pr.kind()
        self.hard = pr.hard_base()
        self.n = og.n_interior
        self.rate = None

    def sweep(self, lo: int, hi: int):
        """One Jacobi sweep of serials [lo, hi) (og_sweep, _kernels.py:18-106
        semantics); returns (evals, seconds)."""
        import ctypes

        O = self.O
        L = O.lib()
        order = np.arange(lo, hi, dtype=np.int64)
        mc, nr, ne = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        t0 = time.perf_counter()
        L.og_sweep(ctypes.byref(self.pr.grid.struct), ctypes.byref(self.pr._dyn),
                   self.u.ctypes.data, self.u_in.ctypes.data, order.ctypes.data, order.size,
                   self.kind.ctypes.data, None, None, self.hard.ctypes.data, None,
                   O.SENTINEL, O.RULE_REF, self.threads, ctypes.byref(mc), ctypes.byref(nr),
                   ctypes.byref(ne))
        return ne.value, time.perf_counter() - t0

    def sample(self, seconds: float):
        """A slab of consecutive serials in the middle of the grid sized for
        about `seconds` of CPU work (calibrated on a small slab first).
        Returns (updates/s, evals, seconds, description)."""
        mid = self.n // 2
        if self.rate is None:
            m = min(self.n, 1 << 15)
            self.sweep(mid - m // 2, mid + m // 2)  # page-in / thread start
            ne, dt = self.sweep(mid - m // 2, mid + m // 2)
            self.rate = ne / max(dt, 1e-9)
            self.per_node = ne / max(m // 2 * 2, 1)
        nodes = int(min(self.n, max(1 << 12, seconds * self.rate / max(self.per_node, 1.0))))
        lo = max(0, mid - nodes // 2)
        ne, dt = self.sweep(lo, lo + nodes)
        self.rate = ne / dt
        desc = (f"1 Jacobi sweep of {nodes} consecutive serials (mid-grid slab) of the "
                f"{'x'.join(map(str, self.g.shape))} fine grid, {self.pr.nc} controls, "
                f"reference rule, oracle/phj_oracle.c OpenMP, {self.threads} threads")
        return ne / dt, ne, dt, desc


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


def _counts(res):
    """(executed, logical) candidate evaluations of one run_patchy result,
    split into (coarse, patch solves): the coarse stage is replicated on
    every rank and is counted once; patch solves are summed over ranks."""
    k = res.stats.kernels.get("patch_solve", {})
    cst = res.coarse_stats
    return (int(cst.performed_evals), int(cst.candidate_evals),
            int(k.get("performed", 0)), int(k.get("logical", 0)))


def jacobi_patch_work(phj, patchy, spec, pcfg, cfg, plans):
    """Dense work of a Jacobi solve to the workload tol: per-patch Jacobi
    sweep counts from the device's Jacobi schedule x patch nodes x admissible
    controls, + the coarse stage's dense count (for the CPU estimate)."""
    import dataclasses

    jcfg = dataclasses.replace(cfg, schedule="jacobi", inner_sweeps=None)
    r = phj.run_patchy(spec, pcfg, jcfg, plans=plans, outputs=False)
    dense = sum(int(st.candidate_evals) for st in r.patch_stats)
    sweeps = [int(st.sweeps) for st in r.patch_stats]
    return dense + int(r.coarse_stats.candidate_evals), sweeps


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
        # NCCL's init lines (ranks, NVLink/NVLS transport) in the run log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            td.init_process_group(backend)
    lib = _lib.load()
    w = _workload(args)
    spec, pcfg, cfg = w.spec, w.pcfg, w.cfg
    dim = spec.dim

    plans = patchy.make_plans(spec, pcfg)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def step():
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        res = phj.run_patchy(spec, pcfg, cfg, plans=plans, outputs=False)
        b.record()
        torch.cuda.synchronize()
        return res, a.elapsed_time(b)

    for _ in range(args.warmup):
        step()
    if world > 1:
        td.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    l0 = lib.phj_launch_count()
    tot_ms, kern_ms, kern_hw = 0.0, 0.0, 0
    cnt = np.zeros(4, dtype=np.int64)  # coarse exec, coarse logical, patch exec, patch logical
    res = None
    for _ in range(args.steps):
        res, ms = step()
        tot_ms += ms
        cnt += np.array(_counts(res), dtype=np.int64)
        k = res.stats.kernels.get("patch_solve", {})
        kern_ms += k.get("kernel_ms", 0.0)
        kern_hw += k.get("executed", 0)
    launches = lib.phj_launch_count() - l0
    clocks = clk.stop()
    torch.cuda.synchronize()
    patch_stats = res.patch_stats
    if world > 1:
        td.barrier()
        t = torch.tensor([tot_ms, kern_ms], device="cuda", dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        tot_ms_max, kern_ms_max = t.tolist()
        # coarse counted once (replicated on every rank), patch work summed
        c = torch.tensor([0, 0, cnt[2], cnt[3], kern_hw, launches], device="cuda",
                         dtype=torch.float64)
        td.all_reduce(c, op=td.ReduceOp.SUM)
        cnt = np.array([cnt[0], cnt[1], c[2].item(), c[3].item()], dtype=np.int64)
        kern_hw, launches = int(c[4].item()), int(c[5].item())
    else:
        tot_ms_max, kern_ms_max = tot_ms, kern_ms
    executed = int(cnt[0] + cnt[2])
    logical = int(cnt[1] + cnt[3])
    value = executed / (tot_ms_max * 1e-3)

    # -- e2e: public API from host inputs, D2H of the value field ----------------
    e2e_steps = max(5, min(args.steps, 10))
    # the result lands in a pinned host buffer (allocated once, like a
    # caller's output array); the copy itself is inside the timed region
    r = phj.run_patchy(spec, pcfg, cfg)
    host = torch.empty(r.value.values.shape, dtype=r.value.values.dtype, pin_memory=True)
    del r
    for _ in range(max(0, args.warmup)):
        r = phj.run_patchy(spec, pcfg, cfg)
        host.copy_(r.value.values)
    torch.cuda.synchronize()
    if world > 1:
        td.barrier()
    t0 = time.perf_counter()
    ecnt = np.zeros(4, dtype=np.int64)
    for _ in range(e2e_steps):
        r = phj.run_patchy(spec, pcfg, cfg)
        host.copy_(r.value.values)
        ecnt += np.array(_counts(r), dtype=np.int64)
    torch.cuda.synchronize()
    e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e_dt], device="cuda", dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        e_dt = float(t.item())
        c = torch.tensor([float(ecnt[2])], device="cuda", dtype=torch.float64)
        td.all_reduce(c, op=td.ReduceOp.SUM)
        ecnt[2] = int(c.item())
    e2e_val = float(ecnt[0] + ecnt[2]) / e_dt
    d2h = host.numel() * host.element_size()
    st = plans[0].stencils
    h2d = int(st.oct_start.nbytes + st.ctrl.nbytes + st.nzmask.nbytes + st.weights.nbytes +
              st.cost.nbytes) * 2 + 8 * 64
    jac = None
    if world == 1 and not args.no_cpu_baseline:
        jac = jacobi_patch_work(phj, patchy, spec, pcfg, cfg, plans)

    if rank != 0:
        td.destroy_process_group()
        return
    peak = measure_peak(args.dtype)
    fl = _flops_per_candidate(dim)
    # algorithmic work of the patch-solve launch: real candidates it executed
    # (after octant pruning) x flops per candidate
    kern_real = int(cnt[2])
    achieved = kern_real * fl / (kern_ms_max * 1e-3) / 1e12 if kern_ms_max > 0 else 0.0
    issued = kern_hw * fl / (kern_ms_max * 1e-3) / 1e12 if kern_ms_max > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            ent = json.load(open(prof)).get(f"{args.config}_{args.dtype}", {})
            traffic = ent.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        thr = host_threads()
        port = CpuPort(w, thr)
        rate, ev, dt, sample = port.sample(args.cpu_seconds)
        dense, jsweeps = jac
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample,
               "seconds": dt,
               "time_to_converge_est_s": dense / rate,
               "time_to_converge_est_basis": (
                   f"{dense:.4g} dense candidate evaluations of a Jacobi solve to tol "
                   f"{cfg.tol:g} (device Jacobi schedule: per-patch sweeps "
                   f"{min(jsweeps)}..{max(jsweeps)} x patch nodes x controls, + coarse) / "
                   f"the measured CPU rate; the reference's Gauss-Seidel may need fewer "
                   f"sweeps")}
    ttc = tot_ms_max / args.steps
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ttc,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.dtype == "float64" else "f32", "data": "synthetic",
        "config": _config(w, args, world),
        "time_to_converge_ms": ttc,
        "value_counts": "executed candidate evaluations (real controls, after octant pruning) "
                        "of the coarse (once) + patch solves per second of time-to-converge",
        "executed_updates_per_step": executed // args.steps,
        "logical_updates_per_s": logical / (tot_ms_max * 1e-3),
        "logical_updates_per_step": logical // args.steps,
        "patch_equivalent_sweeps": [int(s.sweeps) for s in patch_stats],
        "phases_ms": {k: round(v, 3) for k, v in res.stats.phases_ms().items()},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "ms_per_step": 1000.0 * e_dt / e2e_steps},
        "roofline": {"bound": "fp64" if args.dtype == "float64" else "fp32",
                     "kernel": ("fine patch solve: value-ordered pass (solve_kernel) + asynchronous "
                                "relaxation (solve_async_kernel), one phj_solve call"
                                if cfg.schedule == "async" else
                                "solve_kernel (fine patch solve, one cooperative launch)"),
                     "limiter": "shared-memory (LSU) wavefronts + latency, not the FP64 pipe: ncu of "
                                "the C5 fp64 pass: LSU data pipe 65 % of peak, FP64 pipe 38 %, DRAM "
                                "0.44 TB/s (profiles/r2ae_c5f64_solve_banded_ncu.txt, DESIGN.md §5)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "flops_per_candidate": fl,
                     "kernel_ms": kern_ms_max / args.steps,
                     "executed_candidates": kern_real // max(1, args.steps),
                     "issued_entry_tflops": issued,
                     "peak_source": "measured here: phj_peak_flops FMA-chain probe"},
        "cpu_baseline": cpu,
        "process_group": ({"backend": td.get_backend(), "world_size": td.get_world_size()}
                          if world > 1 else None),
        "clocks": clocks,
        "gpu_launches": int(launches),
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
    port = CpuPort(w, thr)
    # each step: one bounded slab sample (the whole run stays within minutes)
    per_step = float(os.environ.get("PHJ_REF_STEP_SECONDS", "5"))
    for _ in range(max(0, min(args.warmup, 1))):
        port.sample(min(per_step, 2.0))
    evs, secs = 0, 0.0
    sample = ""
    for _ in range(args.steps):
        r, ev, dt, sample = port.sample(per_step)
        evs += ev
        secs += dt
    value = evs / secs
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": int(os.environ.get(
           "WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": _config(w, args, int(os.environ.get("WORLD_SIZE", "1"))),
           "cpu_update_rule": "reference (u <- min I[u] + h, _kernels.py:98): the "
                              "reference's own arithmetic; same candidate work",
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
