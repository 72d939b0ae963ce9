"""Physics constants handed to the device (the reference's ``pack_params``,
sphbench/physics.py:149-180) and the cubic-spline value used for W(dp).

The pair math itself only exists on the device (csrc/interact.cu); the values here are
computed with the reference's own f64 expressions so the FP64 kernel instantiation is
bit-identical to the reference (tests/test_host.py pins them against tests/golden).
"""
from __future__ import annotations

import math

import numpy as np

from . import _lib

PP_NAMES = ("sup2", "h", "invh", "kc", "eta2", "alpha", "invwdp", "c0", "rho0", "gamma",
            "mass_fluid", "mass_boundary")


def kernel_norm(h: float, kernel: str = "cubic") -> float:
    """3-D normalisation kc: cubic 1/(pi h^3) (physics.py:25-33), Wendland C2 21/(16 pi h^3)."""
    if kernel == "wendland":
        return 21.0 / (16.0 * math.pi * h ** 3)
    return 1.0 / (math.pi * h ** 3)


def kernel_w(r, h: float, kernel: str = "cubic"):
    """W(r) with support 2h: the reference's cubic spline (physics.py:25-33) or the Wendland
    C2 kernel kc (1 - q/2)^4 (2q + 1) (extension)."""
    q = np.asarray(r, dtype=np.float64) / h
    kc = kernel_norm(h, kernel)
    if kernel == "wendland":
        t = np.maximum(1.0 - 0.5 * q, 0.0)
        w = kc * t ** 4 * (2.0 * q + 1.0)
    else:
        w = np.where(q < 1.0, kc * (1.0 - 1.5 * q * q + 0.75 * q ** 3),
                     np.where(q < 2.0, 0.25 * kc * (2.0 - q) ** 3, 0.0))
    return w if w.ndim else float(w)


def kernel_of(params) -> str:
    return getattr(params, "kernel", "cubic")


def pack_params(params, mass_fluid: float, mass_boundary: float) -> np.ndarray:
    """The 12 f64 constants of the pair loop, in the reference's order (kc and 1/W(dp) of the
    selected kernel; the cubic values are the reference's)."""
    sup = params.support_radius
    k = kernel_of(params)
    return np.array([sup * sup, params.h, 1.0 / params.h, kernel_norm(params.h, k),
                     params.eta2, params.alpha, 1.0 / kernel_w(params.dp, params.h, k), params.c0,
                     params.rho0, params.gamma, mass_fluid, mass_boundary], dtype=np.float64)


def params_desc(params, mass_fluid: float, mass_boundary: float, order: int = 0,
                precision: int = _lib.SPHB_FP32, counters: int = 0) -> "_lib.ParamsDesc":
    d = _lib.ParamsDesc()
    for name, v in zip(PP_NAMES, pack_params(params, mass_fluid, mass_boundary)):
        setattr(d, name, float(v))
    d.tait_b = float(params.tait_b)
    for k in range(3):
        d.g[k] = float(np.asarray(params.g, np.float64)[k])
    d.cfl = float(params.cfl)
    d.dt_min = float(params.dt_min)
    d.dt_max = float(params.dt_max)
    d.verlet_stride = int(params.verlet_corrector_stride)
    d.order = int(order)
    d.precision = int(precision)
    d.counters = int(counters)  # SPHB_COUNTERS_GATHER / _SYMMETRIC (EngineConfig.device_counters)
    d.kernel = _lib.SPHB_KERNEL_WENDLAND if kernel_of(params) == "wendland" else _lib.SPHB_KERNEL_CUBIC
    d.integrator = (_lib.SPHB_INT_SYMPLECTIC if getattr(params, "integrator", "verlet") == "symplectic"
                    else _lib.SPHB_INT_VERLET)
    pm = getattr(params, "piston", None)
    if pm is not None:
        d.piston_id0, d.piston_id1 = int(pm.id0), int(pm.id1)
        d.piston_x0, d.piston_stroke, d.piston_period = float(pm.x0), float(pm.stroke), float(pm.period)
    bf = getattr(params, "boundary_force", None)
    if bf is not None:
        d.wall_d, d.wall_r0 = float(bf.d), float(bf.r0)
        d.wall_p1, d.wall_p2 = int(bf.p1), int(bf.p2)
    return d


def grid_dims(params):
    """Cell side and dims exactly as assign_cells computes them (grid.py:81-84)."""
    cs = params.cell_size
    extent = np.asarray(params.domain_max, np.float64) - np.asarray(params.domain_min, np.float64)
    dims = np.maximum(np.ceil(extent / cs - 1e-12).astype(np.int64), 1)
    return cs, dims


def grid_desc(params, reach: int | None = None, target_cols=None) -> "_lib.GridDesc":
    cs, dims = grid_dims(params)
    g = _lib.GridDesc()
    for k in range(3):
        g.origin[k] = float(np.asarray(params.domain_min, np.float64)[k])
        g.domain_max[k] = float(np.asarray(params.domain_max, np.float64)[k])
        g.dims[k] = int(dims[k])
    g.cell_size = float(cs)
    g.reach = int(params.n_subdiv if reach is None else reach)
    g.tx0, g.tx1 = (0, int(dims[0])) if target_cols is None else (int(target_cols[0]), int(target_cols[1]))
    return g
