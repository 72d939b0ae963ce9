"""Synthetic dam-break input: ``Scenario``, ``make_params``, ``build_dam_break``.

Host-side generator of the step's inputs (not part of the timed path).  It reproduces
the reference's generator (sphbench/sim.py:46-190) value for value -- same lattice order,
same f64 arithmetic before the float32 cast, same hydrostatic density profile -- so the
same ``Scenario`` yields bit-identical particle arrays here and in the reference
(tests/test_host.py pins this against tests/golden).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .model import ParticleKind, ParticleSystem, PistonMotion, SimParams, validate


@dataclass
class Scenario:
    """A water column (fill box) inside an open-top tank (sim.py:46-113)."""

    tank_min: np.ndarray = field(default_factory=lambda: np.zeros(3))
    tank_size: np.ndarray = field(default_factory=lambda: np.array([0.3, 0.2, 0.24]))
    fill_offset: np.ndarray = field(default_factory=lambda: np.zeros(3))
    fill_size: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.2, 0.15]))
    dp: float = 0.01
    hydrostatic: bool = True

    def __post_init__(self):
        for name in ("tank_min", "tank_size", "fill_offset", "fill_size"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64))

    @property
    def tank_max(self):
        return self.tank_min + self.tank_size

    @property
    def fill_min(self):
        return self.tank_min + self.fill_offset

    @property
    def fill_max(self):
        return self.fill_min + self.fill_size

    @property
    def fill_height(self) -> float:
        return float(self.fill_size[2])

    def lattice_counts(self):
        return np.maximum(np.round(self.fill_size / self.dp).astype(np.int64), 0)

    def wall_counts(self):
        return np.maximum(np.round(self.tank_size / self.dp).astype(np.int64), 1)

    @property
    def fluid_count(self) -> int:
        return int(np.prod(self.lattice_counts()))

    @property
    def boundary_count(self) -> int:
        nx, ny, nz = (int(v) for v in self.wall_counts())
        return (nx + 1) * (ny + 1) + nz * 2 * (nx + ny)

    def validate(self) -> "Scenario":
        if self.dp <= 0:
            raise ValueError("dp must be positive")
        if np.any(self.dp > self.tank_size) or np.any(self.dp > self.fill_size):
            raise ValueError("dp larger than a box dimension")
        inside = (np.all(self.fill_min >= self.tank_min) and np.all(self.fill_max <= self.tank_max)
                  and float(np.prod(self.fill_size)) < float(np.prod(self.tank_size)))
        if not inside:
            raise ValueError("fill box must lie strictly inside the tank")
        if self.fluid_count <= 0 or self.boundary_count <= 0:
            raise ValueError("scenario produces no particles")
        return self


def make_params(scenario: Scenario, hdp: float = 2.0, n_subdiv: int = 1, cfl: float = 0.3,
                alpha: float = 0.25, gamma: float = 7.0, rho0: float = 1000.0,
                c0: float | None = None, gravity: float = 9.81, **overrides) -> SimParams:
    """sim.py:116-134: h = hdp*dp, c0 = 10 sqrt(g H) unless given, domain = tank padded by
    4h (and 8h more headroom above)."""
    h = hdp * scenario.dp
    if c0 is None:
        c0 = 10.0 * math.sqrt(gravity * scenario.fill_height)
    pad = 2.0 * 2.0 * h
    lo = scenario.tank_min - pad
    hi = scenario.tank_max + pad
    hi[2] += 2.0 * pad
    return validate(SimParams(h=h, dp=scenario.dp, rho0=rho0, c0=c0, gamma=gamma, alpha=alpha,
                              g=np.array([0.0, 0.0, -gravity]), cfl=cfl, domain_min=lo,
                              domain_max=hi, n_subdiv=n_subdiv, **overrides))


def _boundary_positions(scenario: Scenario) -> np.ndarray:
    """Floor lattice (x-major), then per height level k the four wall rows y=0, y=max,
    x=0 (interior y), x=max (interior y) -- the reference's emission order."""
    dp = scenario.dp
    nx, ny, nz = (int(v) for v in scenario.wall_counts())
    x0, y0, z0 = (float(v) for v in scenario.tank_min)
    gi, gj = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="ij")
    parts = [np.stack([x0 + gi.ravel() * dp, y0 + gj.ravel() * dp, np.full(gi.size, z0)], axis=1)]
    xs = np.arange(nx + 1) * dp + x0
    ys = np.arange(1, ny) * dp + y0
    for k in range(1, nz + 1):
        z = z0 + k * dp
        parts.append(np.stack([xs, np.full(nx + 1, y0), np.full(nx + 1, z)], axis=1))
        parts.append(np.stack([xs, np.full(nx + 1, y0 + ny * dp), np.full(nx + 1, z)], axis=1))
        parts.append(np.stack([np.full(ny - 1, x0), ys, np.full(ny - 1, z)], axis=1))
        parts.append(np.stack([np.full(ny - 1, x0 + nx * dp), ys, np.full(ny - 1, z)], axis=1))
    return np.concatenate(parts, axis=0)


def _fluid_positions(scenario: Scenario) -> np.ndarray:
    dp = scenario.dp
    fx, fy, fz = (int(v) for v in scenario.lattice_counts())
    ii, jj, kk = np.meshgrid(np.arange(fx), np.arange(fy), np.arange(fz), indexing="ij")
    lo = scenario.fill_min
    return np.stack([lo[0] + (ii.ravel() + 0.5) * dp, lo[1] + (jj.ravel() + 0.5) * dp,
                     lo[2] + (kk.ravel() + 0.5) * dp], axis=1)


def build_dam_break(scenario: Scenario, params: SimParams) -> ParticleSystem:
    """sim.py:137-190: deterministic lattice fill + one boundary layer on floor and walls."""
    scenario.validate()
    bound = _boundary_positions(scenario)
    fluid = _fluid_positions(scenario)
    nb, nf = bound.shape[0], fluid.shape[0]
    pos = np.concatenate([bound, fluid], axis=0).astype(np.float32)
    if scenario.hydrostatic:
        depth = np.maximum(scenario.fill_max[2] - pos[:, 2].astype(np.float64), 0.0)
        gmag = float(np.linalg.norm(params.g))
        rho = params.rho0 * (1.0 + params.rho0 * gmag * depth / params.tait_b) ** (1.0 / params.gamma)
    else:
        rho = np.full(nb + nf, params.rho0, dtype=np.float64)
    mass = params.rho0 * params.dp ** 3
    ptype = np.concatenate([np.full(nb, ParticleKind.BOUNDARY, np.uint8),
                            np.full(nf, ParticleKind.FLUID, np.uint8)])
    system = ParticleSystem(count_fluid=nf, count_boundary=nb, pos=pos,
                            vel=np.zeros((nb + nf, 3), np.float32), rho=rho.astype(np.float32),
                            mass_fluid=mass, mass_boundary=mass, ptype=ptype,
                            id=np.arange(nb + nf, dtype=np.int64))
    return system.validate()


# ---------------------------------------------------------------- wave tank (C5, extension)
@dataclass
class WaveTank(Scenario):
    """Piston-type wavemaker flume (SURVEY.md §8(d) C5 suggestion; no reference counterpart):
    a full-length water layer in a long tank whose x = tank_min wall (above the floor) is a
    piston moving as x0 + stroke/2 (1 - cos(2 pi t / period))."""

    tank_size: np.ndarray = field(default_factory=lambda: np.array([2.4, 0.3, 0.5]))
    fill_size: np.ndarray = field(default_factory=lambda: np.array([2.4, 0.3, 0.3]))
    dp: float = 0.02
    stroke: float = 0.1
    period: float = 1.0

    def __post_init__(self):
        super().__post_init__()
        # the water starts one dp in front of the piston and one dp before the far wall
        self.fill_offset = np.array([0.5 * self.dp, 0.0, 0.0])
        self.fill_size = np.array([self.tank_size[0] - self.dp, self.fill_size[1], self.fill_size[2]])


def piston_mask(scenario: Scenario, bound_pos: np.ndarray) -> np.ndarray:
    """Boundary particles of the x = tank_min wall above the floor (the piston)."""
    x0, z0 = float(scenario.tank_min[0]), float(scenario.tank_min[2])
    return (np.abs(bound_pos[:, 0] - x0) < 0.25 * scenario.dp) & (bound_pos[:, 2] > z0 + 0.5 * scenario.dp)


def make_wave_tank_params(scenario: "WaveTank", **kw) -> SimParams:
    """make_params for the flume plus its PistonMotion (piston particles get ids [0, np))."""
    bound = _boundary_positions(scenario)
    npist = int(piston_mask(scenario, bound).sum())
    pm = PistonMotion(id0=0, id1=npist, x0=float(scenario.tank_min[0]), stroke=float(scenario.stroke),
                      period=float(scenario.period))
    return make_params(scenario, piston=pm, **kw)


def build_wave_tank(scenario: "WaveTank", params: SimParams) -> ParticleSystem:
    """Same lattice generator as build_dam_break (hydrostatic rho, one boundary layer), with
    the piston particles moved to the front of the boundary list so they hold ids
    [0, params.piston.id1)."""
    system = build_dam_break(scenario, params)
    nb = system.count_boundary
    m = piston_mask(scenario, system.pos[:nb].astype(np.float64))
    order = np.concatenate([np.nonzero(m)[0], np.nonzero(~m)[0], np.arange(nb, system.n)])
    system.pos = np.ascontiguousarray(system.pos[order])
    system.vel = np.ascontiguousarray(system.vel[order])
    system.rho = np.ascontiguousarray(system.rho[order])
    system.id = np.arange(system.n, dtype=np.int64)
    pm = getattr(params, "piston", None)
    if pm is not None and (pm.id0, pm.id1) != (0, int(m.sum())):
        raise ValueError("params.piston ids do not match this wave tank (use make_wave_tank_params)")
    return system.validate()


# Named configurations of BASELINE.json / SURVEY.md §8 (C1-C4; C5 is builder-defined).
FULL_TANK = dict(tank_size=np.array([1.6, 0.67, 0.6]), fill_size=np.array([0.4, 0.67, 0.3]))
CONFIGS = {
    "c1": dict(dp=0.006),            # 22,399 particles
    "c2": dict(dp=0.00144),          # 1,142,622
    "c3": dict(dp=0.00068),          # 10,200,478
    "c4_1": dict(dp=0.002003, **FULL_TANK),   # 10.97M (weak scaling, 1 GPU)
    "c4_2": dict(dp=0.00159, **FULL_TANK),    # 21.55M
    "c4_4": dict(dp=0.001262, **FULL_TANK),   # 42.45M
    "c4_8": dict(dp=0.001, **FULL_TANK),      # 84.20M
    # weak-scaling family in C3's own tank (SURVEY.md §8 table note): ~10M particles per GPU
    "c3w_2": dict(dp=0.00054),       # 20.06M
    "c3w_4": dict(dp=0.00043),       # 39.44M
    "c3w_8": dict(dp=0.00034),       # 78.83M
}


WAVE_CONFIGS = {
    "c5": dict(dp=0.00175),          # 40,060,170 fluid (2.4 x 0.3 x 0.3 m layer)
    "c5_small": dict(dp=0.02),       # test size
}


def named_scenario(name: str) -> Scenario:
    if name in WAVE_CONFIGS:
        return WaveTank(**WAVE_CONFIGS[name])
    return Scenario(**CONFIGS[name])
