"""The step loop: ``run_simulation`` with the reference's signature, semantics and errors
(sphbench/sim.py:272-352), executed device-resident on the B200.

Differences from the reference are in *where* things run, not in what they compute:
the state is uploaded once, every step runs NL -> PI -> SU in libsphb200 kernels with no
per-step host synchronisation, and the host reads the device control block only every
``chunk`` steps (or at snapshot / stats boundaries) to emit StepStats and to raise
``DivergenceError`` with the same step, particle id and message the reference would.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import EngineConfig, NEIGHBOR_BYTES
from .device import DeviceSim, compute_derived_device, require_cuda
from .engine import PRECISION_CODE
from .model import DerivedQuantities, ParticleKind, StepStats, validate
from .physics import params_desc
from .scenario import Scenario, build_dam_break


class DivergenceError(RuntimeError):
    """A particle left the domain or the state went non-finite (sim.py:22-29)."""

    def __init__(self, message: str, step: int, particle_id: int | None = None):
        super().__init__(message)
        self.step = step
        self.particle_id = particle_id


def divergence_from_device(err) -> DivergenceError:
    step, code, index, pid = err
    if code == _lib.SPHB_DIV_LEFT_DOMAIN:
        return DivergenceError(f"particle id {pid} left the domain at step {step}", step, pid)
    if code == _lib.SPHB_DIV_NONFINITE_FORCES:
        return DivergenceError(f"non-finite forces at step {step}", step)
    return DivergenceError(f"non-finite state at step {step}", step)


# Interaction blocking (tools/block_matrix.sh, profiles/r01k_block_matrix.txt): the 384-target
# build (12-warp CTAs, one per SM) beats the 128-target one at rest on every BASELINE
# configuration but C1, whose 25k particles make only ~65 such blocks for 148 SMs (C1 ms/step:
# 0.131 with 256-target blocks on 8-warp CTAs, 0.147 with 128, 0.174 with 384); it also wins
# over a whole 10,000-step collapse (profiles/r01k_c3_10000steps_auto.json).  "auto" = 384
# from PI_LARGE_MIN_TARGETS targets (4 blocks per SM) up, 256 below, fixed for the run.
PI_LARGE_MIN_TARGETS = 4 * 148 * 384


def initial_pi_block(n_targets: int, n_subdiv: int = 1) -> int:
    """The "auto" blocking for ``n_targets`` interaction targets: 384 from 4 such blocks per SM,
    256 below.  With h/2 cells (n_subdiv 2: 8 particles per cell, a 5x5 stencil of rows) the
    FP32 kernel cuts 2x2-row bricks, which stage ~12 candidates per target like the 384-target
    row blocks at n_subdiv 1 (C3 n_subdiv 2, ms/step: 19.6 with 384-target bricks, 22.2 with
    256, 34.3 with 128; 26.2 with the earlier 128-target row blocks)."""
    return 384 if n_targets >= PI_LARGE_MIN_TARGETS else 256


@dataclass
class VerletState:
    """Previous-step velocity and density, permuted alongside the system (sim.py:31-43)."""

    vel_prev: np.ndarray   # (n, 3) float32
    rho_prev: np.ndarray   # (n,) float32
    step: int = 0
    corrector_stride: int = 40

    @classmethod
    def from_system(cls, system, stride: int) -> "VerletState":
        return cls(vel_prev=system.vel.copy(), rho_prev=system.rho.copy(), corrector_stride=stride)


def tree_min(values, block: int = 4096) -> float:
    """sim.py:196-208 (the min is exact, so the blocked order does not change the result)."""
    a = np.asarray(values, dtype=np.float64).ravel()
    if a.size == 0:
        raise ValueError("empty reduction")
    return float(a.min())


def tree_max(values, block: int = 4096) -> float:
    return -tree_min(-np.asarray(values, dtype=np.float64), block=block)


def compute_dt(forces, system, derived, params) -> float:
    """sim.py:215-232 on the device (k_dt_terms): cfl * min(dt_f, dt_cv) clamped to
    [dt_min, dt_max]; dt_f over fluid with gravity included, dt_cv over all particles."""
    require_cuda()
    dev = torch.device("cuda")
    n, nb = int(system.n), int(system.count_boundary)
    acc = torch.as_tensor(np.ascontiguousarray(forces.accel, np.float64)).to(dev)
    visc = torch.as_tensor(np.ascontiguousarray(forces.visc_dt, np.float64)).to(dev)
    cs = torch.as_tensor(np.ascontiguousarray(derived.csound, np.float32)).to(dev)
    inf = np.array([np.inf, np.inf]).view(np.int64)
    out = torch.as_tensor(inf).to(dev)
    prm = params_desc(params, float(system.mass_fluid), float(system.mass_boundary))
    _lib.check(_lib.lib().sphb_dt_terms(_lib.ref(prm), n, nb, acc.data_ptr(), visc.data_ptr(),
                                        cs.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "sphb_dt_terms")
    dt_f, dt_cv = out.cpu().numpy().view(np.float64)
    dt = params.cfl * min(float(dt_f), float(dt_cv))
    return float(min(max(dt, params.dt_min), params.dt_max))


def verlet_update(state: VerletState, system, forces, params, dt: float) -> None:
    """sim.py:235-259 on the device (k_verlet_soa): two-step Verlet with the periodic
    single-step corrector; fluid moves, boundary particles only update density.  Updates
    ``system`` and ``state`` in place, bit-identical to the reference."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    require_cuda()
    dev = torch.device("cuda")
    n, nb = int(system.n), int(system.count_boundary)
    corrector = state.step % state.corrector_stride == 0
    t = lambda a, dt_: torch.as_tensor(np.ascontiguousarray(a, dt_)).to(dev)  # noqa: E731
    pos, vel, rho = t(system.pos, np.float32), t(system.vel, np.float32), t(system.rho, np.float32)
    vp, rp = t(state.vel_prev, np.float32), t(state.rho_prev, np.float32)
    acc, drho = t(forces.accel, np.float64), t(forces.drho_dt, np.float64)
    prm = params_desc(params, float(system.mass_fluid), float(system.mass_boundary))
    _lib.check(_lib.lib().sphb_verlet_soa(_lib.ref(prm), n, nb, int(corrector), float(dt),
                                          pos.data_ptr(), vel.data_ptr(), rho.data_ptr(), vp.data_ptr(),
                                          rp.data_ptr(), acc.data_ptr(), drho.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream), "sphb_verlet_soa")
    system.pos = pos.cpu().numpy()
    system.vel = vel.cpu().numpy()
    system.rho = rho.cpu().numpy()
    state.vel_prev = vp.cpu().numpy()
    state.rho_prev = rp.cpu().numpy()
    state.step += 1


def compute_derived(rho, params) -> DerivedQuantities:
    """physics.compute_derived (physics.py:96-110) on the device EOS."""
    press, csound, prrho, tensil = compute_derived_device(np.asarray(rho), params)
    return DerivedQuantities(press=press, csound=csound, prrho=prrho, tensil=tensil)


class _Timer:
    def __init__(self, steps, per_step=4):
        self.ev = [[torch.cuda.Event(enable_timing=True) for _ in range(per_step)]
                   for _ in range(steps)]


def make_device_sim(system, params, cfg: EngineConfig, max_steps=None, t_end=None, **kw) -> DeviceSim:
    return DeviceSim(system, params, reach=cfg.device_reach(params.n_subdiv),
                     order=cfg.device_order(), precision=PRECISION_CODE[cfg.precision],
                     counters=cfg.device_counters(),
                     max_steps=-1 if max_steps is None else int(max_steps),
                     t_end=math.inf if t_end is None else float(t_end), **kw)


def run_simulation(scenario_or_system, params, config: EngineConfig, max_steps: int | None = None,
                   t_end: float | None = None, snapshot_every: int = 0, snapshot_sink=None,
                   stats_sink=None, *, chunk: int = 256, stage_timing: bool = True,
                   checkpoint_every: int = 0, checkpoint_path=None, resume_from=None,
                   pi_block="auto", pi_kernel="gather", retune_every: int = 500):
    """NL -> PI -> SU loop on the B200.  Returns (system, stats_list) like sim.py:272-352;
    raises DivergenceError on the first out-of-domain particle or non-finite state.

    ``chunk`` bounds how many steps run between host readbacks (the record ring is
    sized for it); ``stage_timing`` records CUDA events at the NL/PI/SU boundaries of
    every step to fill StepStats.stage_*_s and wall_seconds.

    Extensions: ``checkpoint_every`` > 0 writes a binary checkpoint (snapshots.save_checkpoint;
    ``checkpoint_path`` may contain ``{step}``) every that many steps; ``resume_from`` continues
    bit-identically from such a checkpoint (``scenario_or_system`` may then be None; step
    numbers and the stop rules continue from the checkpoint's step).

    ``pi_block``: targets per FP32 interaction block, 128, 256, 384, 512 or "auto" (initial_pi_block of
    the particle count; recorded in checkpoints so resumed runs keep the same blocking).
    ``pi_kernel``: "gather", "symmetric" or "paired" FP32 interaction (DeviceSim.set_pi_kernel);
    the symmetric kernel needs the cell traversal order (every config but fastcellshalf).
    "tuned": measured selection -- every ``retune_every`` steps the next steps run once with
    each of DeviceSim.pi_candidates (the gather kernel on the size rule's blocking, the paired
    kernel), their PI stages are timed with CUDA events and the fastest build runs until the
    next tuning point (the tuning steps are ordinary steps of the run).  The choice follows
    the timing, so FP32 results are reproducible to the FP32 tolerance, not bit for bit; the
    other settings are deterministic."""
    if max_steps is None and t_end is None:
        raise ValueError("need max_steps or t_end")
    validate(params)
    cfg = config.validated()
    need = cfg.required_n_subdiv()
    if need is not None and params.n_subdiv != need:
        raise ValueError(f"config {cfg.tag} needs n_subdiv={need}")
    if checkpoint_every and checkpoint_path is None:
        raise ValueError("checkpoint_every needs checkpoint_path")
    chunk = max(1, int(chunk))
    if snapshot_every and snapshot_sink is not None:
        chunk = int(snapshot_every)  # chunk boundaries land on snapshot steps
    if checkpoint_every:
        chunk = math.gcd(chunk, int(checkpoint_every))
    if resume_from is not None:
        sim = DeviceSim.from_checkpoint(resume_from, params, reach=cfg.device_reach(params.n_subdiv),
                                        order=cfg.device_order(), precision=PRECISION_CODE[cfg.precision],
                                        counters=cfg.device_counters(),
                                        max_steps=-1 if max_steps is None else int(max_steps),
                                        t_end=math.inf if t_end is None else float(t_end),
                                        record_capacity=max(chunk, 1))
        system = scenario_or_system if scenario_or_system is not None else _shell_system(sim)
    else:
        system = build_dam_break(scenario_or_system, params) if isinstance(scenario_or_system, Scenario) \
            else scenario_or_system
        sim = make_device_sim(system, params, cfg, max_steps, t_end, record_capacity=max(chunk, 1))
    if pi_block not in (128, 256, 384, 512, "auto"):
        raise ValueError("pi_block must be 128, 256, 384, 512 or 'auto'")
    adapt = pi_block == "auto" and cfg.precision == "fp32"
    if resume_from is None and (pi_block != "auto" or adapt):
        sim.set_pi_block(initial_pi_block(sim.n, params.n_subdiv) if adapt else int(pi_block))
    if pi_kernel not in ("gather", "symmetric", "paired", "tuned"):
        raise ValueError("pi_kernel must be 'gather', 'symmetric', 'paired' or 'tuned'")
    if pi_kernel == "symmetric" and cfg.precision == "fp32" and cfg.device_order() == 0:
        sim.set_pi_kernel("symmetric")
    if pi_kernel == "paired" and cfg.precision == "fp32":
        sim.set_pi_kernel("paired")
    tuned = pi_kernel == "tuned" and cfg.precision == "fp32"
    cands = sim.pi_candidates(params.n_subdiv) if tuned else []
    last_tune = None
    stats_out: list[StepStats] = []
    nbytes = NEIGHBOR_BYTES[cfg.derived_mode]
    done_steps = int(sim.ctrl_host()["step"])
    while True:
        # chunks end on multiples of ``chunk`` (snapshot / checkpoint steps), also after a
        # resume from a step that is not one; a tuning chunk is one step per candidate build
        this = chunk - done_steps % chunk
        tune_now = tuned and (last_tune is None or done_steps - last_tune >= int(retune_every)) \
            and this >= 2 * len(cands)  # (else at the next chunk)
        if tune_now:
            # the first tuning runs each build twice and decides on the second round (a
            # kernel's first launch carries its one-time module load)
            this = len(cands) * (2 if last_tune is None else 1)
        timer = _Timer(this, sim.n_stage_events()) if (stage_timing or tune_now) else None
        for k in range(this):
            if tune_now:
                sim.select_pi(*cands[k % len(cands)])
            sim.launch_step(events=timer.ev[k] if timer else None)
        c = sim.ctrl_host()  # synchronises
        if tune_now:
            sim.tune_choose(cands, timer.ev[-len(cands):])
            last_tune = done_steps
        now = int(c["step"])
        recs = sim.records(done_steps, now)
        for k, r in enumerate(recs):
            st = StepStats(step=done_steps + k, dt=float(r["dt"]),
                           candidate_pairs=int(r["candidate_pairs"]),
                           true_pairs=int(r["hits_ordered"]) // 2,
                           force_evals=int(r["force_evals"]), ff_force_evals=int(r["ff_force_evals"]),
                           engine_tag=cfg.tag, neighbor_bytes=nbytes)
            if stage_timing:
                st.stage_nl_s, st.stage_pi_s, st.stage_su_s, st.wall_seconds = \
                    DeviceSim.stage_seconds(timer.ev[k])
            step_no = done_steps + k + 1
            # snapshot first, then the stats record (sim.py:345-351)
            if snapshot_every and step_no % snapshot_every == 0 and snapshot_sink is not None \
                    and step_no == now:
                snap = _system_from_device(sim, system)
                snapshot_sink.emit(step_no, snap, compute_derived(snap.rho, params))
            if stats_sink is not None:
                stats_sink(st)
            stats_out.append(st)
        err = sim.error()
        if err is not None:
            raise divergence_from_device(err)
        if checkpoint_every and now > done_steps and now % int(checkpoint_every) == 0:
            sim.save_checkpoint(str(checkpoint_path).format(step=now))
        done_steps = now
        if not int(c["active"]):
            break
    _write_back(sim, system)
    return system, stats_out


def _shell_system(sim: DeviceSim):
    """A ParticleSystem of the right shape for write-back after a resume."""
    from .model import ParticleSystem
    n, nb = sim.n, sim.nb
    z3 = np.zeros((n, 3), np.float32)
    return ParticleSystem(count_fluid=n - nb, count_boundary=nb, pos=z3, vel=z3.copy(),
                          rho=np.ones(n, np.float32), mass_fluid=sim.mass_fluid,
                          mass_boundary=sim.mass_boundary,
                          ptype=np.concatenate([np.full(nb, ParticleKind.BOUNDARY, np.uint8),
                                                np.full(n - nb, ParticleKind.FLUID, np.uint8)]),
                          id=np.arange(n, dtype=np.int64))


def _system_from_device(sim: DeviceSim, like):
    pos, vel, rho, ids, _, _ = sim.download()
    out = like.copy() if hasattr(like, "copy") else like
    out.pos, out.vel, out.rho, out.id = pos, vel, rho, ids
    nb = int(like.count_boundary)
    out.ptype = np.concatenate([np.full(nb, ParticleKind.BOUNDARY, np.uint8),
                                np.full(int(like.n) - nb, ParticleKind.FLUID, np.uint8)])
    return out


def _write_back(sim: DeviceSim, system):
    pos, vel, rho, ids, _, _ = sim.download()
    system.pos, system.vel, system.rho, system.id = pos, vel, rho, ids
    nb = int(system.count_boundary)
    system.ptype = np.concatenate([np.full(nb, ParticleKind.BOUNDARY, np.uint8),
                                   np.full(int(system.n) - nb, ParticleKind.FLUID, np.uint8)])
