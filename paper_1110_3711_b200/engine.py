"""The drop-in force engine: ``make_engine(cfg).compute(...) -> ForceOutput``.

Same protocol as the reference engines (sphbench/engines/__init__.py:30-48,
gather.py:42-110): takes the caller's sorted frame (system, derived, grid, cindex,
params) as host arrays, runs the B200 interaction kernels (csrc/interact.cu), and
returns f64 numpy arrays plus StepStats with the reference's counter definitions.
This is the per-call ("partial GPU") boundary; ``run_simulation``
keeps the state resident instead.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .config import (DERIVED_RECOMPUTED, ENGINE_GATHER, GATHER_FAST_HALF, NEIGHBOR_BYTES,
                     EngineConfig, ForceOutput)
from .device import Workspace, _ptr, _stream, new_ctrl, read_ctrl, require_cuda
from .model import StepStats
from .physics import grid_desc, grid_dims, params_desc

PRECISION_CODE = {"fp32": _lib.SPHB_FP32, "fp64": _lib.SPHB_FP64}


class B200Engine:
    """Device gather engine; holds its device buffers across calls (resized on demand)."""

    def __init__(self, config: EngineConfig, pi_block="auto", pi_kernel="gather"):
        """``pi_block``: targets per FP32 interaction block (128, 256, 384, 512) or "auto", the
        production rule of run_simulation (sim.initial_pi_block of the frame's particle count
        and n_subdiv), so the engine path runs the same interaction build as the stepper.
        ``pi_kernel``: "gather", "symmetric" (pair evaluation once per unordered pair, the
        reactions scattered, 384-target blocks; cell-order variants only) or "paired" (the
        gather with two targets per lane on 512-target bricks)."""
        self.config = config.validated()
        if pi_block not in (128, 256, 384, 512, "auto"):
            raise ValueError("pi_block must be 128, 256, 384, 512 or 'auto'")
        if pi_kernel not in ("gather", "symmetric", "paired"):
            raise ValueError("pi_kernel must be 'gather', 'symmetric' or 'paired'")
        self.pi_block = pi_block
        self.pi_kernel = pi_kernel
        self.last_pi_block = None
        self._buf = None
        self._ws = None
        self.last_kernel_ms = None

    @property
    def tag(self) -> str:
        return self.config.tag

    def _buffers(self, n: int, ncells: int):
        if self._buf is None or self._buf["n"] < n or self._buf["ncells"] < ncells:
            dev = torch.device("cuda")
            m = max(n, 1)
            self._buf = dict(
                n=n, ncells=ncells,
                host=torch.empty((3, m, 4), dtype=torch.float32, pin_memory=True),
                hcell=torch.empty(m, dtype=torch.int32, pin_memory=True),
                dev4=torch.empty((3, m, 4), dtype=torch.float32, device=dev),
                cell=torch.empty(m, dtype=torch.int32, device=dev),
                beg=torch.empty(2 * ncells, dtype=torch.int32, device=dev),
                end=torch.empty(2 * ncells, dtype=torch.int32, device=dev),
                acc=torch.empty((m, 3), dtype=torch.float64, device=dev),
                drho=torch.empty(m, dtype=torch.float64, device=dev),
                visc=torch.empty(m, dtype=torch.float64, device=dev),
                acc64=torch.empty((m, 3), dtype=torch.float64, device=dev),
                drho64=torch.empty(m, dtype=torch.float64, device=dev),
                visc64=torch.empty(m, dtype=torch.float64, device=dev),
                out=torch.empty((m, 5), dtype=torch.float64, pin_memory=True),
            )
            self._ws = Workspace(n, ncells)
        return self._buf

    def compute(self, system, derived, grid, cindex, params, ranges=None) -> ForceOutput:
        require_cuda()
        cfg = self.config
        n, nb = int(system.n), int(system.count_boundary)
        cell_of = np.asarray(grid.cell_of)
        if cell_of.shape[0] != n:
            raise ValueError("grid/system length mismatch")
        need = cfg.required_n_subdiv()
        if need is not None and params.n_subdiv != need:
            raise ValueError(f"gather variant {cfg.gather_variant} needs "
                             f"n_subdiv={need}, got {params.n_subdiv}")
        if cfg.engine == ENGINE_GATHER and cfg.gather_variant == GATHER_FAST_HALF and ranges is None:
            raise ValueError("fastcellshalf requires precomputed interaction ranges")
        reach = cfg.device_reach(params.n_subdiv)
        g = grid_desc(params, reach)
        _, dims = grid_dims(params)
        ncells = int(np.prod(dims))
        prm = params_desc(params, system.mass_fluid, system.mass_boundary, cfg.device_order(),
                          PRECISION_CODE[cfg.precision], cfg.device_counters())
        b = self._buffers(n, ncells)
        if n:
            # pack the caller's frame as K3 lays it out: posp = (pos, prrho), velr = (vel, rho),
            # aux = (press, csound, tensil, list mass)
            h = b["host"]
            h[0, :n, :3] = torch.from_numpy(np.ascontiguousarray(system.pos, np.float32))
            h[0, :n, 3] = torch.from_numpy(np.ascontiguousarray(derived.prrho, np.float32))
            h[1, :n, :3] = torch.from_numpy(np.ascontiguousarray(system.vel, np.float32))
            h[1, :n, 3] = torch.from_numpy(np.ascontiguousarray(system.rho, np.float32))
            h[2, :n, 0] = torch.from_numpy(np.ascontiguousarray(derived.press, np.float32))
            h[2, :n, 1] = torch.from_numpy(np.ascontiguousarray(derived.csound, np.float32))
            h[2, :n, 2] = torch.from_numpy(np.ascontiguousarray(derived.tensil, np.float32))
            h[2, :nb, 3] = float(np.float32(system.mass_boundary))
            h[2, nb:n, 3] = float(np.float32(system.mass_fluid))
            b["hcell"][:n] = torch.from_numpy(cell_of.astype(np.int32))
            b["dev4"][:, :n].copy_(h[:, :n], non_blocking=True)
            b["cell"][:n].copy_(b["hcell"][:n], non_blocking=True)
        if self.pi_block == "auto":
            from .sim import initial_pi_block
            blk = initial_pi_block(n, params.n_subdiv)
        else:
            blk = int(self.pi_block)
        kern = {"gather": _lib.SPHB_PI_GATHER, "symmetric": _lib.SPHB_PI_SYMMETRIC,
                "paired": _lib.SPHB_PI_PAIRED}[self.pi_kernel]
        if self.pi_kernel != "gather":  # the builds' own blockings (pi384s / pi512p)
            blk = 384 if self.pi_kernel == "symmetric" else 512
        self._ws.set_pi_block(blk)
        self._ws.set_pi_kernel(kern)
        self.last_pi_block = blk
        ctrl = new_ctrl(torch.device("cuda"))
        L, s = _lib.lib(), _stream()
        d4 = b["dev4"]
        _lib.check(L.sphb_cell_ranges_from_sorted(self._ws.handle, _lib.ref(g), _ptr(b["cell"]), n, nb,
                                                  _ptr(b["beg"]), _ptr(b["end"]), s),
                   "sphb_cell_ranges_from_sorted")
        _lib.check(L.sphb_step_begin(_ptr(ctrl), s), "sphb_step_begin")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.sphb_interact(self._ws.handle, _lib.ref(prm), _lib.ref(g), n, nb, _ptr(d4[0]), _ptr(d4[1]),
                                   _ptr(d4[2]), _ptr(b["cell"]), _ptr(b["beg"]), _ptr(b["end"]),
                                   _ptr(b["acc"]), _ptr(b["drho"]), _ptr(b["visc"]), _ptr(ctrl), s),
                   "sphb_interact")
        e1.record()
        out = b["out"]
        if n:
            # the kernel's force layout (FP32: float4 + float, include/sphb200.h) widened to the
            # ForceOutput f64 arrays (exact)
            _lib.check(L.sphb_forces_f64(_lib.ref(prm), n, _ptr(b["acc"]), _ptr(b["drho"]),
                                         _ptr(b["visc"]), _ptr(b["acc64"]), _ptr(b["drho64"]),
                                         _ptr(b["visc64"]), s), "sphb_forces_f64")
            out[:n, :3].copy_(b["acc64"][:n], non_blocking=True)
            out[:n, 3].copy_(b["drho64"][:n], non_blocking=True)
            out[:n, 4].copy_(b["visc64"][:n], non_blocking=True)
        c = read_ctrl(ctrl)  # synchronises
        self.last_kernel_ms = e0.elapsed_time(e1)
        o = out[:n].numpy()
        accel = np.ascontiguousarray(o[:, :3])
        raw = [int(v) for v in c["counters"]]  # raw[1]: ordered hits (either counter mode)
        stats = StepStats(candidate_pairs=raw[0], true_pairs=raw[1] // 2, force_evals=raw[2],
                          ff_force_evals=raw[3], engine_tag=self.tag,
                          neighbor_bytes=NEIGHBOR_BYTES[cfg.derived_mode])
        return ForceOutput(accel=accel, drho_dt=np.ascontiguousarray(o[:, 3]),
                           visc_dt=np.ascontiguousarray(o[:, 4]), stats=stats)


def make_engine(config: EngineConfig, pi_block="auto", pi_kernel="gather") -> B200Engine:
    """engines/__init__.py:30-34 -- every validated config runs on the B200."""
    return B200Engine(config.validated(), pi_block=pi_block, pi_kernel=pi_kernel)


def compute_forces_gather(system, derived, grid, cindex, ranges, params,
                          config: EngineConfig) -> ForceOutput:
    """engines/__init__.py:43-48."""
    return B200Engine(config).compute(system, derived, grid, cindex, params, ranges=ranges)


def compute_forces_cellpairs(system, derived, grid, cindex, params,
                             config: EngineConfig) -> ForceOutput:
    """engines/__init__.py:37-40 (executed by the device gather traversal)."""
    return B200Engine(config).compute(system, derived, grid, cindex, params)
