"""X-slab geometry of the multi-GPU decomposition.

The global cell grid is cut along x into slabs of whole cell columns [x0_k, x1_k), one per
rank (the reference's Slices geometry, engines/kernels.py:230-323, balance.py:46-88, with
particle-count or measured-time balanced bounds).  The stepper is ``dslab.DeviceSlabSim``;
the torch restatement of the decomposition that the CPU (gloo) tests run lives in
tests/slab_torch_reference.py.
"""
from __future__ import annotations

import numpy as np
import torch

# ------------------------------------------------------------------ geometry helpers
def columns_of(x: torch.Tensor, origin_x: float, cell_size: float, nx: int) -> torch.Tensor:
    """Cell x-column of float32 coordinates, exactly as assign_cells (grid.py:87-89)."""
    c = torch.floor((x.double() - origin_x) / cell_size).to(torch.int64)
    return torch.clamp(c, max=nx - 1)


def balanced_bounds(col_counts: np.ndarray, nranks: int, min_width: int) -> np.ndarray:
    """Slab bounds over cell columns with ~equal particle counts, each >= min_width wide."""
    nx = col_counts.shape[0]
    if nx < nranks * min_width:
        raise ValueError("fewer cell columns than slabs x halo width")
    cum = np.concatenate([[0], np.cumsum(col_counts, dtype=np.float64)])
    total = cum[-1]
    b = np.zeros(nranks + 1, dtype=np.int64)
    b[-1] = nx
    for k in range(1, nranks):
        b[k] = int(np.searchsorted(cum, total * k / nranks, side="left"))
    return enforce_min_width(b, min_width)


def enforce_min_width(b: np.ndarray, w: int) -> np.ndarray:
    b = b.copy()
    n = b.size - 1
    for k in range(1, n):
        b[k] = max(b[k], b[k - 1] + w)
    for k in range(n - 1, 0, -1):
        b[k] = min(b[k], b[k + 1] - w)
    return b


def rebalance_slices(bounds, times) -> np.ndarray:
    """Equal-time quantiles of the piecewise-linear cumulative cost, whole columns, width >= 1
    (the reference's slab rebalancer, engines/balance.py:53-88, restated)."""
    bounds = np.asarray(bounds, dtype=np.int64)
    times = np.asarray(times, dtype=np.float64)
    ns = bounds.size - 1
    if times.size != ns:
        raise ValueError("one time per slice required")
    if np.any(times <= 0):
        raise ValueError("slice times must be positive")
    if int(bounds[-1] - bounds[0]) < ns:
        raise ValueError("fewer cells than slices")
    widths = np.diff(bounds).astype(np.float64)
    cum = np.concatenate(([0.0], np.cumsum(times)))
    new = bounds.copy()
    for k in range(1, ns):
        target = cum[-1] * k / ns
        s = min(int(np.searchsorted(cum, target, side="right") - 1), ns - 1)
        new[k] = int(round(bounds[s] + (target - cum[s]) / times[s] * widths[s]))
    return enforce_min_width(new, 1)


__all__ = ["columns_of", "balanced_bounds", "enforce_min_width", "rebalance_slices"]
