"""Generate golden fixtures from the REAL reference (run in the build container).

    python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only; numba
cache redirected to /tmp) and applies the arity shim documented in SURVEY.md
§0.2: the shipped ``_kernels.sweep_batch`` declares an unused ``value_reject``
parameter at position 13 (/root/reference/pkg/src/patchyhjb/_kernels.py:19-21,
never read in :52-106) that both call sites omit (solver.py:258-263,
decomp.py:156-161).  The wrapper inserts ``False`` there; the parameter is
dead, so semantics are unchanged.

Every fixture is produced through the reference's own public API and stock
code path, reference update rule, lexicographic Gauss-Seidel (or its exact
Jacobi mode ``active=0, frozen=snapshot``, solver.py:240-249).  The fixtures
are committed; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_phj")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import patchyhjb
    import patchyhjb._kernels as K

    if not getattr(K.sweep_batch, "_phj_shim", False):
        orig = K.sweep_batch

        def sweep_batch(*args):
            a = list(args)
            a.insert(13, False)  # value_reject (dead parameter)
            return orig(*a)

        sweep_batch._phj_shim = True
        K.sweep_batch = sweep_batch
    return patchyhjb


def fib_sphere(n: int) -> np.ndarray:
    """Fibonacci directions (BASELINE configs 3/5; formula in SURVEY §8d)."""
    i = np.arange(n, dtype=float)
    z = 1.0 - (2.0 * i + 1.0) / n
    r = np.sqrt(1.0 - z * z)
    phi = np.pi * (1.0 + np.sqrt(5.0)) * (i + 0.5)
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def eikonal_dyn(X, a):
    X = np.atleast_2d(X)
    return np.tile(np.asarray(a, dtype=float), (X.shape[0], 1))


def jacobi_sweep(phj, field, spec, table):
    """Exact Jacobi sweep through the public API (active=0, frozen=snapshot)."""
    g = field.grid
    snap = field.flat.copy()
    st = phj.solve(field, spec, cfg=phj.SolverConfig(max_sweeps=1), table=table,
                   active=np.zeros(g.n_ext, dtype=np.uint8), frozen=snap,
                   hard=table.hard_base)
    return st


def noisy_field(phj, spec, g, seed):
    f = phj.init_value_field(g, spec)
    rng = np.random.default_rng(seed)
    noise = rng.uniform(0.5, 2.5, size=g.shape)
    noise[rng.random(g.shape) < 0.2] = phj.SENTINEL
    keep = spec.target.contains(g.interior_points()).reshape(g.shape)
    f.interior[...] = np.where(keep, 0.0, noise)
    return f


def main():
    phj = import_reference()
    out = {}

    # -- G1: zermelo 21^2, 16 controls: one GS sweep + one Jacobi sweep from
    #        the seeded noisy field of test_solver.py:158-175 (seed 7)
    spec = phj.preset("zermelo2d", controls=16)
    g = phj.Grid(spec.box_lo, spec.box_hi, (21, 21))
    table = phj.CandidateTable(g, spec)
    f0 = noisy_field(phj, spec, g, 7)
    fgs = f0.copy()
    phj.solve(fgs, spec, cfg=phj.SolverConfig(max_sweeps=1), table=table)
    fj = f0.copy()
    jacobi_sweep(phj, fj, spec, table)
    np.savez_compressed(os.path.join(OUT, "zermelo21_sweep.npz"),
                        u0=f0.values, gs=fgs.values, jacobi=fj.values)

    # -- G2: config-1 fine problem (eikonal, 32 circle controls, 101^2,
    #        ball r=0.1): converged GS solve at tol 1e-8 + feedback, and one
    #        Jacobi sweep from a seeded noisy field
    spec1 = phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                            dynamics=eikonal_dyn,
                            control_set=phj.discretize_circle(32),
                            target=phj.TargetSpec.ball((0.0, 0.0), 0.1))
    g1 = phj.Grid(spec1.box_lo, spec1.box_hi, (101, 101))
    t1 = phj.CandidateTable(g1, spec1)
    cfg = phj.SolverConfig(tol=1e-8)
    u1, st1 = phj.solve_single(spec1, g1, cfg=cfg, table=t1)
    fb1, _ = phj.extract_feedback(u1, spec1, table=t1)
    n1 = noisy_field(phj, spec1, g1, 11)
    j1 = n1.copy()
    jacobi_sweep(phj, j1, spec1, t1)
    # exact Jacobi iteration to tol 1e-8 through the public API
    uj = phj.init_value_field(g1, spec1)
    sweeps_j = 0
    while True:
        st = jacobi_sweep(phj, uj, spec1, t1)
        sweeps_j += 1
        if st.max_change <= 1e-8 or sweeps_j > 2000:
            break
    np.savez_compressed(os.path.join(OUT, "c1_fine.npz"), u_gs=u1.values,
                        sweeps_gs=st1.sweeps, evals_gs=st1.candidate_evals,
                        feedback=fb1.indices, u0=n1.values, jacobi1=j1.values,
                        u_jacobi=uj.values, sweeps_jacobi=sweeps_j)

    # -- G3: config-1 patchy pipeline at function level (the
    #        26^2 coarse grid holds no target node, so the coarse stage uses a
    #        ball of radius max(0.1, k_c*sqrt(2)); same code path as
    #        patchy.py:121-154).  Transport converged (color_tol 1e-12).
    gc = phj.Grid(spec1.box_lo, spec1.box_hi, (26, 26))
    rc = max(0.1, gc.k_step * np.sqrt(2.0))
    spec1c = phj.ProblemSpec(name="c1c", dim=2, box_lo=spec1.box_lo,
                             box_hi=spec1.box_hi, dynamics=eikonal_dyn,
                             control_set=spec1.control_set,
                             target=phj.TargetSpec.ball((0.0, 0.0), rc))
    dec = phj.make_static_decomposition(gc, 4)
    uc, stc = phj.solve_dd(spec1c, gc, dec, cfg)
    lifted = phj.NodeField(g1, sentinel=uc.sentinel)
    lifted.flat[g1.interior_flat()] = phj.interpolate_many(uc, g1.interior_points())
    fbl, _ = phj.extract_feedback(lifted, spec1, table=t1)
    mask = phj.mask_unreachable(lifted)
    parts = phj.partition_target(spec1.target, g1, 4)
    phis = []
    tsweeps = []
    for j, part in enumerate(parts):
        phi, sw, _, warn = phj.transport_color(spec1, g1, fbl, part, 1e-12, table=t1)
        phis.append(phi.values.copy())
        tsweeps.append(sw)
    pm = phj.assemble_patches(list(enumerate(
        [phj.NodeField(g1, p) for p in phis])), mask, g1, kind=t1.kind)
    pcfg = phj.PatchyConfig(n_patches=4, coarse_nodes=26, fine_nodes=101)
    val, pst, _ = phj.solve_patches(spec1, g1, pm, lifted, pcfg, cfg, table=t1)
    np.savez_compressed(
        os.path.join(OUT, "c1_patchy.npz"), coarse=uc.values, coarse_radius=rc,
        coarse_sweeps=stc.sweeps, lifted=lifted.values, feedback=fbl.indices,
        phi=np.stack(phis), transport_sweeps=np.array(tsweeps),
        parts=np.concatenate(parts), part_sizes=np.array([p.size for p in parts]),
        color=pm.color, boundary=pm.boundary, uncovered=pm.uncovered_serials,
        value=val.values, patch_sweeps=np.array([s.sweeps for s in pst]))

    # -- G4: 3D, 48 Fibonacci controls (config 3/5 control rule), 21^3 on
    #        [-1,1]^3, ball r=0.25: converged GS + feedback + a Jacobi sweep
    spec3 = phj.ProblemSpec(name="fib3", dim=3, box_lo=(-1.0,) * 3, box_hi=(1.0,) * 3,
                            dynamics=eikonal_dyn,
                            control_set=phj.ControlSet(fib_sphere(48), "unit-sphere-geodesic"),
                            target=phj.TargetSpec.ball((0.0,) * 3, 0.25))
    g3 = phj.Grid(spec3.box_lo, spec3.box_hi, (21, 21, 21))
    t3 = phj.CandidateTable(g3, spec3)
    u3, st3 = phj.solve_single(spec3, g3, cfg=cfg, table=t3)
    fb3, _ = phj.extract_feedback(u3, spec3, table=t3)
    n3 = noisy_field(phj, spec3, g3, 5)
    j3 = n3.copy()
    jacobi_sweep(phj, j3, spec3, t3)
    np.savez_compressed(os.path.join(OUT, "fib3d_21.npz"), u_gs=u3.values,
                        sweeps_gs=st3.sweeps, feedback=fb3.indices, u0=n3.values,
                        jacobi1=j3.values)

    # -- G5: fan2d 41^2, 16 controls (variable speed with a zero-speed line):
    #        converged GS, saturating lift at equal resolution, feedback
    specf = phj.preset("fan2d", controls=16)
    gf = phj.Grid(specf.box_lo, specf.box_hi, (41, 41))
    tf = phj.CandidateTable(gf, specf)
    uf, stf = phj.solve_single(specf, gf, cfg=cfg, table=tf)
    lf, fbf, _ = phj.coarse_solve_and_lift(specf, gf, gf, 1, cfg, fine_table=tf)
    np.savez_compressed(os.path.join(OUT, "fan41.npz"), u_gs=uf.values,
                        sweeps_gs=stf.sweeps, lifted=lf.values, feedback=fbf.indices,
                        eps_speed=tf.eps_speed)

    # -- G6: partition_target outputs (problems.py:147-193)
    parts_out = {}
    for name, n, R in (("eikonal2d", 41, 4), ("zermelo2d", 31, 4), ("fan2d", 31, 4),
                       ("eikonal3d", 15, 4), ("eikonal2d", 101, 8)):
        sp = phj.preset(name)
        gg = phj.Grid(sp.box_lo, sp.box_hi, (n,) * sp.dim)
        ps = phj.partition_target(sp.target, gg, R)
        parts_out[f"{name}_{n}_{R}"] = np.concatenate(
            [np.full(p.size, j, dtype=np.int64) for j, p in enumerate(ps)])
        parts_out[f"{name}_{n}_{R}_serials"] = np.concatenate(ps)
    np.savez_compressed(os.path.join(OUT, "partitions.npz"), **parts_out)

    print("wrote fixtures to", OUT)
    print("c1 GS sweeps", st1.sweeps, "jacobi sweeps", sweeps_j,
          "coarse outer", stc.sweeps, "patch sweeps", [s.sweeps for s in pst],
          "transport", tsweeps)


def main_ao3():
    """G7: conical control reduction (AO3, solver.py:446-476, patchy.py:353-356)
    on the config-1 patch map of G3: state-constrained patch solves with
    ``reduction`` r = 3 and 6 (reference rule, GS, tol 1e-8)."""
    phj = import_reference()
    spec1 = phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                            dynamics=eikonal_dyn,
                            control_set=phj.discretize_circle(32),
                            target=phj.TargetSpec.ball((0.0, 0.0), 0.1))
    g1 = phj.Grid(spec1.box_lo, spec1.box_hi, (101, 101))
    t1 = phj.CandidateTable(g1, spec1)
    cfg = phj.SolverConfig(tol=1e-8)
    c = np.load(os.path.join(OUT, "c1_patchy.npz"))
    lifted = phj.NodeField(g1, c["lifted"].copy(), sentinel=1e9)
    fbl = phj.FeedbackField(g1, spec1.control_set, c["feedback"].copy())
    mask = phj.mask_unreachable(lifted)
    pm = phj.assemble_patches(list(enumerate([phj.NodeField(g1, p.copy()) for p in c["phi"]])),
                              mask, g1, kind=t1.kind)
    assert np.array_equal(pm.color, c["color"])
    out = {}
    for r in (3.0, 6.0):
        pcfg = phj.PatchyConfig(n_patches=4, coarse_nodes=26, fine_nodes=101, reduction=r)
        val, pst, _ = phj.solve_patches(spec1, g1, pm, lifted, pcfg, cfg, table=t1,
                                        feedback=fbl)
        key = f"r{int(r)}"
        out[f"value_{key}"] = val.values
        out[f"sweeps_{key}"] = np.array([s.sweeps for s in pst])
        out[f"evals_{key}"] = np.array([s.candidate_evals for s in pst])
        print("ao3", r, "sweeps", [s.sweeps for s in pst], "evals",
              [s.candidate_evals for s in pst])
    np.savez_compressed(os.path.join(OUT, "c1_patchy_ao3.npz"), **out)

    # -- G8: Dirichlet patch boundary condition and AO1 warm start
    #        (patchy.py:334-347) on the same patch map
    out = {}
    for key, kw in (("dirichlet", dict(bc_mode="dirichlet")),
                    ("warm", dict(warm_start=True)),
                    ("dirichlet_warm", dict(bc_mode="dirichlet", warm_start=True))):
        pcfg = phj.PatchyConfig(n_patches=4, coarse_nodes=26, fine_nodes=101, **kw)
        val, pst, _ = phj.solve_patches(spec1, g1, pm, lifted, pcfg, cfg, table=t1)
        out[f"value_{key}"] = val.values
        out[f"sweeps_{key}"] = np.array([s.sweeps for s in pst])
        print(key, "sweeps", [s.sweeps for s in pst])
    np.savez_compressed(os.path.join(OUT, "c1_patchy_bc.npz"), **out)


def main_traj():
    """G9: greedy-feedback trajectories (analysis.py:82-139) on committed
    fields: config-1 fine field (u_gs of c1_fine.npz) from several starts
    (target reached, trivial start inside the target, step limit) and the
    fan2d field (zero-speed line: stalled)."""
    phj = import_reference()
    out = {}
    spec1 = phj.ProblemSpec(name="c1", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                            dynamics=eikonal_dyn,
                            control_set=phj.discretize_circle(32),
                            target=phj.TargetSpec.ball((0.0, 0.0), 0.1))
    g1 = phj.Grid(spec1.box_lo, spec1.box_hi, (101, 101))
    f1 = phj.NodeField(g1, np.load(os.path.join(OUT, "c1_fine.npz"))["u_gs"])
    starts = [(1.5, 0.0), (-1.3, 0.9), (0.05, 0.0), (1.9, -1.9), (0.7, 0.23), (-0.4, -1.7)]
    for i, st in enumerate(starts):
        tr = phj.trace_trajectory(f1, spec1, st)
        out[f"c1_start_{i}"] = np.asarray(st, dtype=float)
        out[f"c1_points_{i}"] = tr.points
        out[f"c1_term_{i}"] = np.array(tr.termination)
    tr = phj.trace_trajectory(f1, spec1, (1.5, 1.5), max_steps=3)
    out["c1_limit_points"] = tr.points
    out["c1_limit_term"] = np.array(tr.termination)
    specf = phj.preset("fan2d", controls=16)
    gf = phj.Grid(specf.box_lo, specf.box_hi, (41, 41))
    ff = phj.NodeField(gf, np.load(os.path.join(OUT, "fan41.npz"))["u_gs"])
    for i, st in enumerate([(-0.2, 0.1), (0.6, -0.5)]):
        tr = phj.trace_trajectory(ff, specf, st)
        out[f"fan_start_{i}"] = np.asarray(st, dtype=float)
        out[f"fan_points_{i}"] = tr.points
        out[f"fan_term_{i}"] = np.array(tr.termination)
    for k, v in out.items():
        if "term" in k:
            print(k, v)
    np.savez_compressed(os.path.join(OUT, "trajectories.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ao3":
        main_ao3()
    elif len(sys.argv) > 1 and sys.argv[1] == "traj":
        main_traj()
    else:
        main()
        main_ao3()
        main_traj()
