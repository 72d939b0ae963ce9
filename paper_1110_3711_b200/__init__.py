"""paper_1110_3711_b200 -- B200-native SPH step hot path (arXiv 1110.3711).

Drop-in for the reference package's step API (sphbench/__init__.py:5-18):
``EngineConfig``, ``ForceOutput``, ``make_engine``, the model types, ``Scenario``,
``build_dam_break``, ``make_params`` and ``run_simulation`` -- with every NL/PI/SU FLOP
executed by hand-written sm_100a kernels in libsphb200.so (csrc/, include/sphb200.h).
There is no CPU fallback: without the CUDA library and a GPU the compute entry points
raise.
"""
from .config import EngineConfig, ForceOutput
from .engine import B200Engine, compute_forces_cellpairs, compute_forces_gather, make_engine
from .model import (BoundaryForce, DerivedQuantities, ParticleKind, ParticleSystem, PistonMotion, SimParams,
                    StepStats, validate)
from .scenario import (Scenario, WaveTank, build_dam_break, build_wave_tank, make_params,
                       make_wave_tank_params, named_scenario)
from . import grid
from .sim import DivergenceError, VerletState, compute_derived, compute_dt, run_simulation, verlet_update

__version__ = "0.1.0"

__all__ = [
    "EngineConfig", "ForceOutput", "make_engine", "B200Engine", "compute_forces_gather",
    "compute_forces_cellpairs", "DerivedQuantities", "ParticleKind", "ParticleSystem",
    "SimParams", "StepStats", "validate", "Scenario", "build_dam_break", "make_params",
    "named_scenario", "run_simulation", "DivergenceError", "compute_derived", "__version__",
    "PistonMotion", "BoundaryForce", "WaveTank", "build_wave_tank", "make_wave_tank_params",
    "VerletState", "compute_dt", "verlet_update", "grid",
]
