"""The reference's neighbour-list module (sphbench/grid.py) on the B200.

Same types, signatures, results and errors as grid.py:22-224; the work runs in libsphb200
(K1 cell keys, the stable radix sort, K4 per-cell ranges, k_build_ranges).  Host numpy arrays
in, host numpy arrays out, so a loop written against the reference (or the reference's own
``run_simulation`` with these functions patched into ``sphbench.sim``) runs its NL on the GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import Workspace, _ptr, _stream, cellbits_of, new_ctrl, require_cuda
from .physics import grid_desc, grid_dims

OUT_OF_DOMAIN = -1


@dataclass
class CellGrid:
    cell_size: float
    dims: np.ndarray            # (3,) int64: cells per axis
    origin: np.ndarray          # (3,) float64: domain_min
    cell_of: np.ndarray         # (n,) int64 linear cell index, -1 outside
    sort_perm: np.ndarray | None = None  # new index -> old index, set by reorder

    @property
    def ncells(self) -> int:
        return int(self.dims[0] * self.dims[1] * self.dims[2])

    @property
    def out_of_domain(self) -> np.ndarray:
        return np.nonzero(self.cell_of == OUT_OF_DOMAIN)[0]


@dataclass
class CellBeginEnd:
    """Per-cell half-open [begin, end) particle ranges into sorted arrays."""

    begin: np.ndarray  # (ncells,) int64
    end: np.ndarray    # (ncells,) int64


@dataclass
class CellIndex:
    """Dual-list cell ranges with global particle indices (boundary block first)."""

    fluid: CellBeginEnd
    boundary: CellBeginEnd


@dataclass
class InteractionRanges:
    begin: np.ndarray  # (ncells, nranges) int64
    end: np.ndarray    # (ncells, nranges) int64
    n_subdiv: int

    @property
    def nranges(self) -> int:
        return self.begin.shape[1]


@dataclass
class DualRanges:
    fluid: InteractionRanges
    boundary: InteractionRanges


def ranges_per_cell(n_subdiv: int) -> int:
    if n_subdiv not in (1, 2):
        raise ValueError("interaction ranges support n_subdiv in {1, 2} only")
    return (2 * n_subdiv + 1) ** 2


def _dev():
    require_cuda()
    return torch.device("cuda")


def assign_cells(positions: np.ndarray, params) -> CellGrid:
    """grid.py:77-93 with K1: f64-exact cell of every particle, -1 outside (never clamped;
    the upper domain face belongs to the last cell)."""
    dev = _dev()
    pos = np.ascontiguousarray(positions, np.float32).reshape(-1, 3)
    n = pos.shape[0]
    cs, dims = grid_dims(params)
    ncells = int(np.prod(dims))
    posp = torch.zeros((max(n, 1), 4), dtype=torch.float32, device=dev)
    if n:
        posp[:n, :3] = torch.as_tensor(pos).to(dev)
    keys = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cell = torch.empty_like(keys)
    ws = Workspace(max(n, 1), ncells)
    ctrl = new_ctrl(dev)
    _lib.check(_lib.lib().sphb_cell_keys(ws.handle, _lib.ref(grid_desc(params)), _ptr(posp), n, 0,
                                         _ptr(keys), _ptr(cell), _ptr(ctrl), _stream()),
               "sphb_cell_keys")
    cell_of = cell[:n].cpu().numpy().astype(np.int64)
    return CellGrid(cell_size=float(cs), dims=np.asarray(dims, np.int64),
                    origin=np.asarray(params.domain_min, np.float64).copy(), cell_of=cell_of)


def _stable_perm(cell_of: np.ndarray, nb: int, ncells: int) -> np.ndarray:
    """The per-list stable argsort (grid.py:107-109) by the device radix sort."""
    dev = _dev()
    n = int(cell_of.shape[0])
    if n == 0:
        return np.zeros(0, np.int64)
    cellbits = cellbits_of(ncells)
    key = np.asarray(cell_of, np.int64) | (np.arange(n) >= nb).astype(np.int64) << cellbits
    keys = torch.as_tensor(key.astype(np.uint32).view(np.int32)).to(dev)
    ksort = torch.empty_like(keys)
    perm = torch.empty_like(keys)
    g = _lib.GridDesc()
    # the sort needs only the cell count (its key width): a 1-D grid of ncells cells
    g.cell_size = 1.0
    g.dims[0], g.dims[1], g.dims[2] = int(ncells), 1, 1
    g.domain_max[0] = float(ncells)
    g.reach, g.tx0, g.tx1 = 1, 0, int(ncells)
    ws = Workspace(n, ncells)
    ctrl = new_ctrl(dev)
    _lib.check(_lib.lib().sphb_sort(ws.handle, _lib.ref(g), _ptr(keys), n, _ptr(ksort), _ptr(perm),
                                    _ptr(ctrl), _stream()), "sphb_sort")
    return perm.cpu().numpy().astype(np.int64)


def reorder(system, grid: CellGrid, extra_arrays: tuple = ()):
    """grid.py:96-120: stable sort by cell, boundary and fluid lists separately; mutates the
    system (and ``extra_arrays``) in place, records ``grid.sort_perm`` and returns
    (system, inverse) with inverse[old] = new."""
    if np.any(grid.cell_of == OUT_OF_DOMAIN):
        raise ValueError("cannot reorder with out-of-domain particles present")
    perm = _stable_perm(grid.cell_of, int(system.count_boundary), grid.ncells)
    for name in ("pos", "vel", "rho", "ptype", "id"):
        setattr(system, name, getattr(system, name)[perm])
    for arr in extra_arrays:
        arr[:] = arr[perm]
    grid.cell_of = grid.cell_of[perm]
    grid.sort_perm = perm
    inverse = np.empty_like(perm)
    inverse[perm] = np.arange(system.n)
    return system, inverse


def _ranges_from_sorted(cell_sorted: np.ndarray, nb: int, dims) -> tuple[np.ndarray, np.ndarray]:
    """K4 over a sorted (boundary block, fluid block) cell array: beg/end of both lists."""
    dev = _dev()
    ncells = int(np.prod(dims))
    n = int(cell_sorted.shape[0])
    g = _lib.GridDesc()
    g.cell_size = 1.0
    g.dims[0], g.dims[1], g.dims[2] = int(dims[0]), int(dims[1]), int(dims[2])
    g.domain_max[0], g.domain_max[1], g.domain_max[2] = float(dims[0]), float(dims[1]), float(dims[2])
    g.reach, g.tx0, g.tx1 = 1, 0, int(dims[0])
    cells = torch.as_tensor(np.ascontiguousarray(cell_sorted, np.int32)).to(dev) if n else \
        torch.zeros(1, dtype=torch.int32, device=dev)
    beg = torch.empty(2 * ncells, dtype=torch.int32, device=dev)
    end = torch.empty_like(beg)
    ws = Workspace(max(n, 1), ncells)
    _lib.check(_lib.lib().sphb_cell_ranges_from_sorted(ws.handle, _lib.ref(g), _ptr(cells), n, nb,
                                                       _ptr(beg), _ptr(end), _stream()),
               "sphb_cell_ranges_from_sorted")
    return beg.cpu().numpy().astype(np.int64), end.cpu().numpy().astype(np.int64)


def build_cell_begin_end(cell_of_sorted: np.ndarray, ncells: int) -> CellBeginEnd:
    """grid.py:123-134 (one list, indices from 0)."""
    cells = np.asarray(cell_of_sorted, dtype=np.int64)
    if cells.size and np.any(np.diff(cells) < 0):
        raise ValueError("cell_of must be nondecreasing")
    b, e = _ranges_from_sorted(cells, int(cells.size), (int(ncells), 1, 1))
    return CellBeginEnd(begin=b[:ncells], end=e[:ncells])


def build_cell_index(system, grid: CellGrid) -> CellIndex:
    """grid.py:137-144: both lists' ranges over the reordered system (global indices)."""
    nb = int(system.count_boundary)
    b, e = _ranges_from_sorted(grid.cell_of, nb, grid.dims)
    nc = grid.ncells
    return CellIndex(fluid=CellBeginEnd(begin=b[nc:], end=e[nc:]),
                     boundary=CellBeginEnd(begin=b[:nc], end=e[:nc]))


def forward_offsets(reach: int = 1) -> np.ndarray:
    """grid.py:147-156: the lexicographically positive half of the (2 reach + 1)^3 stencil."""
    offs = []
    for dz in range(0, reach + 1):
        for dy in range(-reach if dz > 0 else 0, reach + 1):
            for dx in range(-reach if (dz > 0 or dy > 0) else 1, reach + 1):
                offs.append((dx, dy, dz))
    return np.array(offs, dtype=np.int64)


def forward_cells(coords, dims, reach: int = 1) -> np.ndarray:
    """grid.py:159-167: forward neighbour cells of ``coords``, clipped to the grid."""
    cells = forward_offsets(reach) + np.array([int(coords[0]), int(coords[1]), int(coords[2])])
    ok = np.all((cells >= 0) & (cells < np.asarray(dims)), axis=1)
    return cells[ok]


def build_ranges(cbe: CellBeginEnd, dims, n_subdiv: int) -> InteractionRanges:
    """grid.py:170-200 with k_build_ranges: the (2n+1)^2 row ranges of every cell's block."""
    nr = ranges_per_cell(n_subdiv)
    nx, ny, nz = int(dims[0]), int(dims[1]), int(dims[2])
    ncells = nx * ny * nz
    if cbe.begin.shape[0] != ncells:
        raise ValueError("cell ranges inconsistent with grid dims")
    dev = _dev()
    beg = torch.as_tensor(np.ascontiguousarray(cbe.begin, np.int32)).to(dev)
    end = torch.as_tensor(np.ascontiguousarray(cbe.end, np.int32)).to(dev)
    rb = torch.empty((ncells, nr), dtype=torch.int64, device=dev)
    re = torch.empty_like(rb)
    _lib.check(_lib.lib().sphb_build_ranges(_ptr(beg), _ptr(end), nx, ny, nz, int(n_subdiv),
                                            _ptr(rb), _ptr(re), _stream()), "sphb_build_ranges")
    return InteractionRanges(begin=rb.cpu().numpy(), end=re.cpu().numpy(), n_subdiv=n_subdiv)


def build_dual_ranges(cindex: CellIndex, dims, n_subdiv: int) -> DualRanges:
    return DualRanges(fluid=build_ranges(cindex.fluid, dims, n_subdiv),
                      boundary=build_ranges(cindex.boundary, dims, n_subdiv))


def search_volume_ratio(n_subdiv: float) -> float:
    """grid.py:216-220: candidate-to-true volume ratio (2 + 1/n)^3 / (4/3 pi)."""
    return (2.0 + 1.0 / n_subdiv) ** 3 / (4.0 / 3.0 * math.pi)


__all__ = ["OUT_OF_DOMAIN", "CellGrid", "CellBeginEnd", "CellIndex", "InteractionRanges",
           "DualRanges", "ranges_per_cell", "assign_cells", "reorder", "build_cell_begin_end",
           "build_cell_index", "forward_offsets", "forward_cells", "build_ranges",
           "build_dual_ranges", "search_volume_ratio"]
