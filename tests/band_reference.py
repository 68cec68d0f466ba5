"""Reference (test-only) construction of the value-ordered pass schedule,
with torch ops on any device: the semantics phj_band_count / phj_band_fill
implement on the GPU.  Returns rows as sorted lists."""

from __future__ import annotations

import numpy as np
import torch


def schedule_rows(T: torch.Tensor, nodes: torch.Tensor, shape, block_dims, delta_min: float,
                  max_bands: int, window, final_row: bool = False):
    """T, nodes per internal serial (time-to-target, bool); shape = internal
    interior shape; block_dims = (planes, rows, nodes) per warp block."""
    lo_w, hi_w = window
    T = T.to(torch.float64).view(-1).clamp(min=0.0)
    nodes = nodes.view(-1).bool()
    t_max = float(T[nodes].max()) if bool(nodes.any()) else 0.0
    delta = max(delta_min, t_max / max_bands)
    band = torch.floor(T / delta).clamp(max=max_bands).to(torch.int64)
    d = len(shape)
    ser = torch.nonzero(nodes).view(-1)
    if d == 3:
        i0 = ser // (shape[1] * shape[2])
        i1 = (ser // shape[2]) % shape[1]
        i2 = ser % shape[2]
        n1 = -(-shape[1] // block_dims[1])
        n2 = -(-shape[2] // block_dims[2])
        bid = (i0 * n1 + i1 // block_dims[1]) * n2 + i2 // block_dims[2]
        total = shape[0] * n1 * n2
    else:
        i0 = ser // shape[1]
        i1 = ser % shape[1]
        n1 = -(-shape[1] // block_dims[1])
        bid = (i0 // block_dims[0]) * n1 + i1 // block_dims[1]
        total = -(-shape[0] // block_dims[0]) * n1
    bm = band[ser]
    kmin = torch.full((total,), 1 << 40, dtype=torch.int64).scatter_reduce(0, bid.cpu(), bm.cpu(),
                                                                           reduce="amin")
    kmax = torch.full((total,), -1, dtype=torch.int64).scatter_reduce(0, bid.cpu(), bm.cpu(),
                                                                      reduce="amax")
    rows = {}
    blocks = torch.nonzero(kmax >= 0).view(-1).tolist()
    n_band = 0
    for b in blocks:
        lo = max(0, int(kmin[b]) - hi_w)
        hi = int(kmax[b]) + lo_w
        for s in range(lo, hi + 1):
            rows.setdefault(s, []).append(b)
        rows.setdefault(hi + 1, []).append(-b - 1)
        n_band = max(n_band, hi + 2)
    if final_row:
        rows[n_band] = list(blocks)
    return {s: sorted(v) for s, v in rows.items()}, n_band, delta
