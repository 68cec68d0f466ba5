"""The device schedule of the value-ordered passes (phj_band_count /
phj_band_fill, csrc/phj_bands.cu) equals the reference construction
(tests/band_reference.py) row by row on a real lifted field."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from band_reference import schedule_rows
from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    from paper_1109_3577_b200 import _lib, configs, patchy


@pytest.mark.parametrize("final_row", [False, True])
def test_device_schedule_equals_reference(final_row):
    w = configs.c5(n=65, dtype="float64")
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(w.cfg))
    vf = patchy.lift_internal(cplan, vc, fplan, w.cfg.rule, w.cfg.dtype)
    inner = patchy.plan_interior_serial(fplan, vf)
    nodes = (inner < 1.0) & (fplan.kind.view(-1) == 0)
    nodes[::7] = False
    band_list, band_off, n_band = patchy.band_schedule(fplan, vf, nodes, "kruzkov", (6, 2),
                                                       final_row=final_row)
    T = -torch.log1p(-inner.double().clamp(max=1 - 1e-16))
    dims = (__import__("ctypes").c_int32 * 3)()
    _lib.load().phj_block_dims(3, dims)
    fmax = fplan.eps_speed / 1e-12
    rows, n_ref, _ = schedule_rows(T.cpu(), nodes.cpu(), fplan.int_shape, tuple(dims),
                                   patchy.BAND_SCALE * fplan.grid.k_step / fmax,
                                   int(patchy.BAND_CAP_PER_NODE * max(fplan.int_shape)), (6, 2),
                                   final_row=final_row)
    assert n_band == n_ref
    lst = band_list.cpu().numpy()
    off = band_off.cpu().numpy()
    assert off.size == n_band + (2 if final_row else 1)
    for s in range(off.size - 1):
        assert sorted(lst[off[s]:off[s + 1]].tolist()) == rows.get(s, []), s


def test_device_schedule_equals_reference_2d():
    """The 2D instance of the schedule kernels (Morton fill over block rows x
    block columns) on config 2's lifted field."""
    w = configs.c2(n=257)
    fplan, cplan = patchy.make_plans(w.spec, w.pcfg)
    vc, _ = patchy.solve_full_internal(cplan, patchy.coarse_cfg(w.cfg))
    vf = patchy.lift_internal(cplan, vc, fplan, w.cfg.rule, w.cfg.dtype)
    inner = patchy.plan_interior_serial(fplan, vf)
    nodes = (inner < 1.0) & (fplan.kind.view(-1) == 0)
    nodes[::5] = False
    band_list, band_off, n_band = patchy.band_schedule(fplan, vf, nodes, "kruzkov", (3, 1),
                                                       final_row=True)
    T = -torch.log1p(-inner.double().clamp(max=1 - 1e-16))
    dims = (__import__("ctypes").c_int32 * 3)()
    _lib.load().phj_block_dims(2, dims)
    fmax = fplan.eps_speed / 1e-12
    rows, n_ref, _ = schedule_rows(T.cpu(), nodes.cpu(), fplan.int_shape, tuple(dims)[:2],
                                   patchy.BAND_SCALE * fplan.grid.k_step / fmax,
                                   int(patchy.BAND_CAP_PER_NODE * max(fplan.int_shape)), (3, 1),
                                   final_row=True)
    assert n_band == n_ref
    lst = band_list.cpu().numpy()
    off = band_off.cpu().numpy()
    for s in range(off.size - 1):
        assert sorted(lst[off[s]:off[s + 1]].tolist()) == rows.get(s, []), s
