"""Error metrics (mirror of patchyhjb.analysis.error_report, analysis.py:25-63).

``e1`` averages |a - b| over nodes finite (< sentinel/2) in both fields,
``e1_allnodes`` divides the same sum by the interior node count.  The
reduction runs on the device (``phj_error_partials``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import NodeField, require_cuda


@dataclass(frozen=True)
class ErrorReport:
    e1: float
    einf: float
    e1_allnodes: float
    compared_count: int
    excluded_count: int
    against: str = "dd_reference"

    def as_dict(self) -> dict:
        return {"E1": self.e1, "Einf": self.einf, "E1_allnodes": self.e1_allnodes,
                "compared": self.compared_count, "excluded": self.excluded_count}


def _interior_values(field):
    if isinstance(field, NodeField):
        idx = torch.as_tensor(field.grid.interior_flat(), device=field.values.device)
        return field.flat[idx], 0.5 * field.sentinel
    t = torch.as_tensor(np.asarray(field, dtype=float) if not isinstance(field, torch.Tensor)
                        else field, dtype=torch.float64).reshape(-1)
    return t, 0.5 * 1.0e9


def error_report(a, b, against: str = "dd_reference") -> ErrorReport:
    """Compare two fields; nodes unreachable on either side are excluded."""
    va, ha = _interior_values(a)
    vb, hb = _interior_values(b)
    if va.numel() != vb.numel():
        raise ValueError("fields live on different grids")
    n = va.numel()
    dev = require_cuda()
    va = va.to(dev).contiguous()
    vb = vb.to(dev).contiguous()
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().phj_error_partials(n, _lib.ptr(va), _lib.ptr(vb), ha, hb,
                                              _lib.ptr(out), _lib.stream_handle()),
               "error_partials")
    s, mx, cnt = out.cpu().tolist()
    compared = int(round(cnt))
    if compared == 0:
        return ErrorReport(0.0, 0.0, 0.0, 0, n, against)
    return ErrorReport(s / compared, mx, s / n, compared, n - compared, against)
