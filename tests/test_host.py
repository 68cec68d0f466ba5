"""CPU tests of the host side: C ABI exports, stencil planning, partitions,
configs and configuration validation (no device needed)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

import paper_1109_3577_b200 as phj
from paper_1109_3577_b200 import _lib, configs, dist, dynamics, problems


def _header_functions():
    src = open(os.path.join(ROOT, "include", "phj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(phj_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 20
    for n in names:
        getattr(lib, n)  # raises AttributeError if missing
    assert set(names) <= set(_lib.EXPORTS) | {"phj_num_sms"}


def test_library_reports_errors_without_device_work():
    lib = _lib.load()
    # a NULL argument is rejected with a message, no CUDA work is issued
    assert lib.phj_solve(None) == 1
    assert b"missing" in lib.phj_last_error()
    assert lib.phj_launch_count() >= 0


def test_stencil_weights_exact_sum_and_octants():
    for n in (8, 32, 64):
        A = phj.discretize_circle(n).controls
        disp = (A / np.linalg.norm(A, axis=1, keepdims=True))[None]
        st = dynamics.build_stencil(disp, None, np.ones((1, n), bool), dynamics.COST_NODE, (0, 1))
        for e in range(st.oct_start[0, 0], st.oct_start[0, -1]):
            s = 0.0
            for w in st.weights[e]:
                s = s + float(w)
            assert s == 1.0  # kernel accumulation order sums to exactly 1
            assert np.all(st.weights[e] >= 0.0)
        # every control appears, octant groups padded to a multiple of 4
        assert set(st.ctrl[st.oct_start[0, 0]: st.oct_start[0, -1]]) == set(range(n))
        for o in range(4):
            assert (st.oct_start[0, o + 1] - st.oct_start[0, o]) % 4 == 0


def test_stencil_matches_reference_interpolation_weights():
    # node-independent weights == the reference's snapped multilinear weights
    # (grid.py:146-152, 227-239) at an interior node, up to the exact-sum ulp
    A = problems.fibonacci_sphere(48).controls
    g = phj.Grid((-1.0,) * 3, (1.0,) * 3, (21, 21, 21))
    disp = (g.k_step * A / g.spacing)[None]
    st = dynamics.build_stencil(disp, None, np.ones((1, 48), bool), dynamics.COST_NODE,
                                (0, 1, 2))
    x = g.interior_points()[g.index_to_serial((10, 10, 10))]
    for pos in range(st.oct_start[0, 0], st.oct_start[0, -1]):
        c = st.ctrl[pos]
        cell, loc = g.locate_many((x + g.k_step * A[c])[None])
        w_ref = phj.grid.interpolation_weights(loc)[0]
        # map reference corners (absolute cell) to octant corners
        base = np.array(g.locate_many(x[None])[0][0])
        got = {}
        octant = 0
        for ax in range(3):
            if disp[0, c, ax] >= 0:
                octant |= 1 << ax
        for k in range(8):
            pos3 = tuple((0 if (octant >> ax) & 1 else -1) + ((k >> ax) & 1) for ax in range(3))
            got[pos3] = st.weights[pos][k]
        want = {}
        for k in range(8):
            pos3 = tuple(int(cell[0][ax] + ((k >> ax) & 1) - base[ax]) for ax in range(3))
            want[pos3] = want.get(pos3, 0.0) + w_ref[k]
        for key, v in want.items():
            if v != 0.0:
                assert got.get(key, 0.0) == pytest.approx(v, abs=1e-12)


def test_plan_detects_dynamics_structure():
    # zermelo: translation (per-control cost); fan: scaled with a zero-speed
    # line; lqr (double integrator): rejected
    g = phj.Grid((-2.0, -2.0), (2.0, 2.0), (21, 21))
    st, ns, eps = dynamics.plan_stencils(g, phj.preset("zermelo2d", controls=16))
    assert st.cost_mode == dynamics.COST_CTRL and ns is None
    fan = phj.preset("fan2d", controls=16)
    fan_generic = phj.ProblemSpec(**{**fan.__dict__, "model": None})
    st, ns, eps = dynamics.plan_stencils(g, fan_generic)
    assert st.cost_mode == dynamics.COST_NODE and ns.kind == 1
    assert eps == pytest.approx(1e-12 * np.abs(g.interior_points().sum(1) + 0.1).max())
    with pytest.raises(phj.ConfigurationError):
        dynamics.plan_stencils(phj.Grid((-1, -1), (1, 1), (11, 11)), phj.preset("lunar2d"))
    with pytest.raises(phj.ConfigurationError):
        dynamics.plan_stencils(phj.Grid((-1, -1), (1, 1), (11, 11)), phj.preset("lqr2d"))


def test_dubins_stencils_per_heading():
    w = configs.c4(nxy=33, nth=16)
    g = w.spec.make_grid(w.pcfg.fine_nodes)
    st, ns, eps = dynamics.plan_stencils(g, w.spec)
    assert st.perm == (2, 0, 1) and st.n_classes == 16 and st.cost_mode == dynamics.COST_CTRL
    # |h f| = k for every heading/control (solver.py:180)
    for j in range(16):
        for c in range(5):
            d = st.disp[j, c] * np.array([g.spacing[2], g.spacing[0], g.spacing[1]])
            assert np.linalg.norm(d) == pytest.approx(g.k_step, rel=1e-12)


@pytest.mark.parametrize("name,n,R", [("eikonal2d", 41, 4), ("zermelo2d", 31, 4),
                                      ("fan2d", 31, 4), ("eikonal3d", 15, 4),
                                      ("eikonal2d", 101, 8)])
def test_partition_target_matches_reference(name, n, R):
    gp = golden("partitions.npz")
    spec = phj.preset(name)
    g = phj.Grid(spec.box_lo, spec.box_hi, (n,) * spec.dim)
    parts = phj.partition_target(spec.target, g, R)
    assert np.array_equal(np.concatenate(parts), gp[f"{name}_{n}_{R}_serials"])
    # the same through the pre-classified-serials fast path
    serials = np.where(spec.target.contains(g.interior_points()))[0]
    parts2 = phj.partition_target(spec.target, g, R, serials=serials)
    assert all(np.array_equal(a, b) for a, b in zip(parts, parts2))


def test_partition_errors():
    spec = phj.preset("eikonal2d")
    with pytest.raises(phj.ConfigurationError):
        phj.partition_target(spec.target, phj.Grid((-2, -2), (2, 2), (5, 5)), 4)


def test_config_partitions_are_disjoint_covers():
    for w, nparts in ((configs.c2(n=257), 8), (configs.c3(n=65), 8), (configs.c5(n=65), 32),
                      (configs.c4(nxy=33, nth=16), 16)):
        g = w.spec.make_grid(w.pcfg.fine_nodes)
        parts = w.pcfg.parts(w.spec.target, g)
        assert len(parts) == nparts and all(p.size > 0 for p in parts)
        allp = np.concatenate(parts)
        assert allp.size == np.unique(allp).size
        assert set(allp) == set(np.where(w.spec.target.contains(g.interior_points()))[0])


def test_c1_coarse_target_dilation():
    w = configs.c1()
    gc = w.spec.make_grid(w.pcfg.coarse_nodes)
    # 0 coarse target nodes at r=0.1, 4 after dilation
    assert w.spec.target.contains(gc.interior_points()).sum() == 0
    assert w.pcfg.coarse_target.contains(gc.interior_points()).sum() == 4


def test_invalid_configs_rejected():
    for kw in ({"tol": 0.0}, {"max_sweeps": 0}, {"bc_mode": "neumann"},
               {"sweep_order": "random"}, {"control_reduction": 0.5}, {"rule": "x"},
               {"dtype": "float16"}, {"dtype": "float32"}):
        with pytest.raises(phj.ConfigurationError):
            phj.SolverConfig(**kw)
    phj.SolverConfig(rule="kruzkov", dtype="float32")
    for kw in ({"n_patches": 0}, {"coarse_nodes": 101, "fine_nodes": 51},
               {"bc_mode": "neumann"}, {"color_tol": 0.0}, {"reduction": 1.0}):
        with pytest.raises(phj.ConfigurationError):
            phj.PatchyConfig(**kw)


def test_grid_periodic_and_layout():
    g = phj.Grid((0.0, 0.0, 0.0), (1.0, 1.0, 2 * np.pi), (5, 5, 8),
                 periodic=(False, False, True))
    assert g.spacing[2] == pytest.approx(2 * np.pi / 8)
    s = g.device_struct((2, 0, 1))
    assert s.periodic[0] == 1 and s.shape[0] == 8 and s.ext[1] == 7
    assert s.strides[0] == 7 * 7 and s.strides[2] == 1


def test_lpt_assignment_and_bound():
    sizes = [26098, 665, 5000, 9000, 12000, 700, 800, 3000]
    owner = dist.lpt_assign(sizes, 4)
    bins = np.bincount(owner, weights=sizes, minlength=4)
    assert owner[0] != owner[4] and bins.max() == 26098
    assert dist.load_balance_bound(sizes, 4) == pytest.approx(sum(sizes) / (4 * 26098))
    assert dist.load_balance_bound([10] * 8, 8) == 1.0
    assert dist.mine_mask(sizes, 0, 1, "cpu") is None


def test_schedule_options_validated_and_resolved():
    for kw in ({"schedule": "gauss-seidel"}, {"inner_sweeps": 0}, {"activity_tol": -1.0}):
        with pytest.raises(phj.ConfigurationError):
            phj.SolverConfig(**kw)
    c = phj.SolverConfig(rule="kruzkov", schedule="async")
    assert (c.inner_for(2), c.inner_for(3)) == (7, 3)
    assert phj.SolverConfig().inner_for(2) == 1  # Jacobi default: plain sweeps
    assert phj.SolverConfig(inner_sweeps=5).inner_for(3) == 5
    assert phj.SolverConfig().act_tol == 1e-12
    assert phj.SolverConfig(rule="kruzkov", dtype="float32").act_tol == 1e-7
    assert phj.SolverConfig(activity_tol=0.0).act_tol == 0.0


def test_coarse_stage_is_deterministic_block_jacobi():
    from paper_1109_3577_b200 import patchy

    a = patchy.coarse_cfg(phj.SolverConfig(rule="kruzkov", schedule="async", tol=1e-8))
    assert a.schedule == "jacobi" and a.inner_sweeps == 2 and a.tol == 1e-8
    j = phj.SolverConfig(rule="kruzkov")
    assert patchy.coarse_cfg(j) is j
    # BASELINE workloads: all asynchronous
    assert [configs.CONFIGS[n]().cfg.schedule for n in ("c1", "c2", "c3", "c4", "c5")] == \
        ["async"] * 5


def _header_fields(struct: str):
    """Field names of a struct typedef in include/phj.h, in order."""
    import re

    src = open(os.path.join(ROOT, "include", "phj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    body = src[src.index(f"typedef struct {struct} {{"):]
    body = body[body.index("{") + 1:body.index(f"}} {struct};")]
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if decl:
            names.append(re.findall(r"([A-Za-z_][A-Za-z0-9_]*)\s*(?:\[[^\]]*\])?$", decl)[0])
    return names


def test_solve_args_layout_matches_header():
    # the ctypes mirrors carry every field of the C structs in header order
    assert [f[0] for f in _lib.SolveArgs._fields_] == _header_fields("phj_solve_args")
    assert [f[0] for f in _lib.TransportArgs._fields_] == _header_fields("phj_transport_args")


def test_vectorised_stencil_weights_bit_identical():
    rng = np.random.default_rng(3577)
    for d in (2, 3):
        disp = rng.uniform(-1.0, 1.0, size=(300, d))
        disp[::7] = np.round(disp[::7])      # axis-aligned feet (snapped weights)
        disp[::11, 0] = 1.0e-13              # below the snap tolerance
        o, w, nz = dynamics._weights_all(disp)
        for i in range(disp.shape[0]):
            o1, w1, nz1 = dynamics._weights_for(disp[i])
            assert o1 == o[i] and nz1 == nz[i] and np.array_equal(w1, w[i])


def test_device_partition_codes_match_numpy_partitions():
    # the built-in partitions computed with torch ops (device path of
    # patchy._resolve_parts; run here on CPU tensors) equal the numpy forms
    import torch

    for w in (configs.c2(n=257), configs.c3(n=65), configs.c5(n=65), configs.c5(n=129)):
        g = w.spec.make_grid(w.pcfg.fine_nodes)
        ser = np.nonzero(w.spec.target.contains(g.interior_points()))[0]
        want = w.pcfg.parts(w.spec.target, g, serials=ser)
        n, code = problems.device_partition_codes(w.pcfg.parts, w.spec.target, g,
                                                  torch.as_tensor(ser))
        code = code.numpy()
        got = [ser[code == j] for j in range(n)]
        assert len(got) == len(want)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_transport_band_schedule():
    # the pass visits a block at sweeps [min band - hi, max band + lo] of its
    # nodes, then once more as a copy (-b-1); reference construction of the
    # rows the device builds (phj_band_count / phj_band_fill, tested against
    # it in tests/test_gpu_bands.py)
    import torch

    from band_reference import schedule_rows

    shape = (3, 9, 17)  # internal (planes, rows, nodes): blocks 1 x 8 x 8
    k = 0.125
    T = torch.zeros(shape, dtype=torch.float64) + torch.arange(shape[2], dtype=torch.float64) * k
    nodes = torch.ones(shape, dtype=torch.bool)
    nodes.view(-1)[0] = False  # not scheduled
    rows, n_band, delta = schedule_rows(T, nodes, shape, (1, 8, 8), k, 100, (2, 1))
    visits = {}
    for s, entries in rows.items():
        for e in entries:
            visits.setdefault(e, []).append(s)
    n1, n2 = 2, 3
    b = (0 * n1 + 0) * n2 + 2  # plane 0, rows 0-7, nodes 16 -> band 16
    assert visits[b] == list(range(15, 19)) and visits[-b - 1] == [19]
    b = (1 * n1 + 1) * n2 + 0  # plane 1, rows 8, nodes 0-7 -> bands 0..7
    assert visits[b] == list(range(0, 10)) and visits[-b - 1] == [10]
    assert n_band == 20 and delta == k
    for s, entries in rows.items():  # one visit per block and sweep
        ids = [e if e >= 0 else -e - 1 for e in entries]
        assert len(set(ids)) == len(ids)
    # the band cap widens delta: at most max_bands bands
    rows, n_band, delta = schedule_rows(T, nodes, shape, (1, 8, 8), k, 4, (2, 1))
    assert delta == 16 * k / 4 and n_band <= 4 + 2 + 1 + 1
