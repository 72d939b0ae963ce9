"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package (sphbench, /root/reference/pkg/src) in the dev container.

This script is the only place that imports the reference.  It never runs on the
GPU box (the reference does not exist there); its outputs are committed as
small compressed .npz files that pin both the CPU oracle (oracle/) and the
CUDA path.

Run:  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
      python tests/golden/make_golden.py [--skip-long]

Fixture catalogue (every array keeps the reference dtype):
  frame_*.npz      one sorted frame + its NL outputs + gather ForceOutput(s)
  eos.npz          compute_derived on edge/random densities
  traj_*.npz       run_simulation trajectories (per-step dt/counters + states)
  drift_c1.npz     1000-step C1 energy/mass diagnostics (survey §8(d))
  io_small.npz     the reference's snapshot CSV text and stats JSON lines of a short run
                   (bench/snapshots.py write_snapshot / stats_line), for the I/O surface
"""
from __future__ import annotations

import argparse
import copy
import os
import sys
import time
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

import sphbench  # noqa: E402
from sphbench import EngineConfig, Scenario, build_dam_break, make_params, run_simulation  # noqa: E402
from sphbench import physics  # noqa: E402
from sphbench.engines import make_engine  # noqa: E402
from sphbench.grid import assign_cells, build_cell_index, build_dual_ranges, reorder  # noqa: E402
from sphbench.model import ParticleKind, ParticleSystem  # noqa: E402
from sphbench.sim import VerletState, compute_dt, verlet_update  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NTHREADS = min(8, os.cpu_count() or 1)


def params_dict(p):
    return dict(
        p_h=p.h, p_dp=p.dp, p_rho0=p.rho0, p_c0=p.c0, p_gamma=p.gamma, p_alpha=p.alpha,
        p_g=np.asarray(p.g, np.float64), p_cfl=p.cfl,
        p_domain_min=np.asarray(p.domain_min, np.float64),
        p_domain_max=np.asarray(p.domain_max, np.float64),
        p_n_subdiv=p.n_subdiv, p_verlet_corrector_stride=p.verlet_corrector_stride,
        p_dt_min=p.dt_min, p_dt_max=p.dt_max)


def system_dict(s, prefix=""):
    return {prefix + "pos": s.pos.copy(), prefix + "vel": s.vel.copy(),
            prefix + "rho": s.rho.copy(), prefix + "id": s.id.copy(),
            prefix + "ptype": s.ptype.copy(),
            prefix + "nb": s.count_boundary, prefix + "nf": s.count_fluid,
            prefix + "mass_fluid": s.mass_fluid, prefix + "mass_boundary": s.mass_boundary}


def gather_cfg(variant, threads=NTHREADS, dmode="precomputed"):
    return EngineConfig(engine="gather", symmetry=False, gather_variant=variant,
                        thread_count=threads, derived_mode=dmode)


def frame_fixture(name, system_unsorted, params, variants, extra=None):
    """NL from the unsorted state, then gather forces for each variant."""
    out = {}
    out.update(params_dict(params))
    out.update(system_dict(system_unsorted, "in_"))
    sysn = system_unsorted.copy()
    grid = assign_cells(sysn.pos, params)
    out["cell_of_unsorted"] = grid.cell_of.copy()
    out["dims"] = np.asarray(grid.dims, np.int64)
    out["cell_size"] = grid.cell_size
    reorder(sysn, grid)
    out["sort_perm"] = grid.sort_perm.copy()
    out["cell_of"] = grid.cell_of.copy()
    cindex = build_cell_index(sysn, grid)
    out["fbeg"] = cindex.fluid.begin
    out["fend"] = cindex.fluid.end
    out["bbeg"] = cindex.boundary.begin
    out["bend"] = cindex.boundary.end
    out.update(system_dict(sysn, "s_"))
    derived = physics.compute_derived(sysn.rho, params)
    out["press"], out["csound"] = derived.press, derived.csound
    out["prrho"], out["tensil"] = derived.prrho, derived.tensil
    ranges = build_dual_ranges(cindex, grid.dims, params.n_subdiv) if params.n_subdiv in (1, 2) else None
    if ranges is not None and name.startswith("small"):
        out["rng_fbeg"], out["rng_fend"] = ranges.fluid.begin, ranges.fluid.end
        out["rng_bbeg"], out["rng_bend"] = ranges.boundary.begin, ranges.boundary.end
    for v in variants:
        eng = make_engine(gather_cfg(v))
        f = eng.compute(sysn, derived, grid, cindex, params, ranges=ranges)
        st = f.stats
        out[f"{v}_accel"] = f.accel
        out[f"{v}_drho"] = f.drho_dt
        out[f"{v}_visc"] = f.visc_dt
        out[f"{v}_counters"] = np.array([st.candidate_pairs, st.true_pairs,
                                         st.force_evals, st.ff_force_evals], np.int64)
        dt = compute_dt(f, sysn, derived, params)
        out[f"{v}_dt"] = dt
        # one Verlet step from this frame (step 0 -> corrector branch), history = current
        s1 = sysn.copy()
        state = VerletState.from_system(s1, params.verlet_corrector_stride)
        verlet_update(state, s1, f, params, dt)
        out[f"{v}_step1_pos"], out[f"{v}_step1_vel"], out[f"{v}_step1_rho"] = s1.pos, s1.vel, s1.rho
        # non-corrector branch with a synthetic history (prev = current - 1 ulp-ish shift)
        s2 = sysn.copy()
        st2 = VerletState.from_system(s2, params.verlet_corrector_stride)
        st2.vel_prev = (s2.vel * np.float32(0.5)).astype(np.float32)
        st2.rho_prev = (s2.rho - np.float32(0.25)).astype(np.float32)
        out[f"{v}_hist_vel_prev"], out[f"{v}_hist_rho_prev"] = st2.vel_prev.copy(), st2.rho_prev.copy()
        st2.step = 1
        verlet_update(st2, s2, f, params, dt)
        out[f"{v}_step1nc_pos"], out[f"{v}_step1nc_vel"], out[f"{v}_step1nc_rho"] = s2.pos, s2.vel, s2.rho
    if extra:
        out.update(extra)
    path = os.path.join(OUT, f"frame_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: n={system_unsorted.n} {os.path.getsize(path)/1e6:.2f} MB", flush=True)


def mid_collapse(dp, steps):
    sc = Scenario(dp=dp)
    params = make_params(sc)
    system, _ = run_simulation(sc, params, gather_cfg("slowcellsh"), max_steps=steps)
    return sc, params, system


def uniform_fluid(n, box=1.0, h=0.05, seed=7, vel_scale=0.1, n_subdiv=1, rho0=1000.0, c0=20.0):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, box, size=(n, 3)).astype(np.float32)
    vel = rng.normal(0.0, vel_scale, size=(n, 3)).astype(np.float32)
    rho = rng.uniform(0.98 * rho0, 1.02 * rho0, size=n).astype(np.float32)
    dp = h / 2.0
    system = ParticleSystem(
        count_fluid=n, count_boundary=0, pos=pos, vel=vel, rho=rho,
        mass_fluid=rho0 * dp ** 3, mass_boundary=rho0 * dp ** 3,
        ptype=np.full(n, ParticleKind.FLUID, dtype=np.uint8),
        id=np.arange(n, dtype=np.int64))
    params = make_params(Scenario(dp=dp), hdp=h / dp, n_subdiv=n_subdiv, c0=c0)
    params = replace(params, domain_min=np.zeros(3) - 1e-6, domain_max=np.full(3, box) + 1e-6)
    return system, params


def eos_fixture():
    sc = Scenario(dp=0.006)
    params = make_params(sc)
    rng = np.random.default_rng(11)
    rho = np.concatenate([
        np.array([params.rho0, 999.0, 1001.0, 950.0, 1100.0, 1000.0001, 500.0, 2000.0], np.float32),
        rng.uniform(900, 1100, 20000).astype(np.float32),
        (params.rho0 + rng.normal(0, 0.01, 2000)).astype(np.float32),
    ]).astype(np.float32)
    d = physics.compute_derived(rho, params)
    out = dict(rho=rho, press=d.press, csound=d.csound, prrho=d.prrho, tensil=d.tensil)
    out.update(params_dict(params))
    # pack_params constants (physics.py:165-180)
    out["pp"] = physics.pack_params(params, 1.0e-3, 2.0e-3)
    np.savez_compressed(os.path.join(OUT, "eos.npz"), **out)
    print("wrote eos.npz", flush=True)


def trajectory_fixture(name, sc, params, cfg, steps, keep_states=(), hydro=None):
    seen = []
    snaps = {}

    class Sink:
        def emit(self, step, system, derived):
            if step in keep_states:
                snaps[step] = system

    t0 = time.perf_counter()
    final, stats = run_simulation(sc, params, cfg, max_steps=steps, snapshot_every=1,
                                  snapshot_sink=Sink(), stats_sink=seen.append)
    el = time.perf_counter() - t0
    out = {}
    out.update(params_dict(params))
    out["scenario"] = np.array(list(sc.tank_min) + list(sc.tank_size) + list(sc.fill_offset)
                               + list(sc.fill_size) + [sc.dp, float(sc.hydrostatic)])
    out["dt"] = np.array([s.dt for s in stats])
    out["counters"] = np.array([[s.candidate_pairs, s.true_pairs, s.force_evals, s.ff_force_evals]
                                for s in stats], np.int64)
    for k, s in snaps.items():
        out.update(system_dict(s, f"st{k}_"))
    out.update(system_dict(final, "final_"))
    out["engine_tag"] = cfg.validated().tag
    out["wall_s"] = el
    np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), **out)
    print(f"wrote traj_{name}.npz ({steps} steps, {el:.1f}s)", flush=True)


def energy_terms(system, params):
    """Survey §8(d) functional: KE, PE (gravity), Tait internal energy rel. rho0."""
    m = np.where(system.ptype == ParticleKind.FLUID, system.mass_fluid, system.mass_boundary)
    fl = system.ptype == ParticleKind.FLUID
    v = system.vel.astype(np.float64)
    ke = 0.5 * float((m[fl] * (v[fl] ** 2).sum(1)).sum())
    g = float(np.linalg.norm(params.g))
    pe = float((m[fl] * g * system.pos[fl, 2].astype(np.float64)).sum())
    B, g7, r0 = params.tait_b, params.gamma, params.rho0
    rho = system.rho.astype(np.float64)

    def u(r):
        return B / (g7 - 1.0) * r ** (g7 - 1.0) / r0 ** g7 + B / r
    ie = float((m * (u(rho) - u(r0))).sum())
    return ke, pe, ie, float(rho[fl].mean()), float(rho.mean())


def drift_fixture(steps=1000, every=10):
    sc = Scenario(dp=0.006)
    params = make_params(sc)
    rows = []

    class Sink:
        def emit(self, step, system, derived):
            rows.append((step,) + energy_terms(system, params))

    system0 = build_dam_break(sc, params)
    rows.append((0,) + energy_terms(system0, params))
    t0 = time.perf_counter()
    final, stats = run_simulation(sc, params, gather_cfg("slowcellsh"), max_steps=steps,
                                  snapshot_every=every, snapshot_sink=Sink())
    out = dict(diag=np.array(rows), dt=np.array([s.dt for s in stats]),
               true_pairs=np.array([s.true_pairs for s in stats], np.int64),
               wall_s=time.perf_counter() - t0)
    out.update(params_dict(params))
    out.update(system_dict(final, "final_"))
    np.savez_compressed(os.path.join(OUT, "drift_c1.npz"), **out)
    print(f"wrote drift_c1.npz ({out['wall_s']:.1f}s)", flush=True)


def io_fixture():
    """Snapshot CSV + stats lines exactly as the reference writes them (3 steps, dp=0.03)."""
    import tempfile

    from sphbench.bench.snapshots import snapshot_of, stats_line, write_snapshot
    sc = Scenario(dp=0.03)
    params = make_params(sc)
    captured = {}

    class Sink:
        def emit(self, step, system, derived):
            with tempfile.NamedTemporaryFile("r", suffix=".csv", delete=False) as fh:
                path = fh.name
            write_snapshot(path, snapshot_of(system, derived))
            captured[step] = open(path).read()
            os.unlink(path)

    lines = []
    system, stats = run_simulation(sc, params, gather_cfg("slowcellsh"), max_steps=3,
                                   snapshot_every=3, snapshot_sink=Sink(),
                                   stats_sink=lambda st: lines.append(stats_line(st)))
    s0 = build_dam_break(sc, params)
    init_csv_path = os.path.join(OUT, "_tmp_init.csv")
    write_snapshot(init_csv_path, snapshot_of(s0, physics.compute_derived(s0.rho, params)))
    init_csv = open(init_csv_path).read()
    os.unlink(init_csv_path)
    out = dict(csv_step3=np.array(captured[3]), csv_init=np.array(init_csv),
               stats_lines=np.array(lines), **system_dict(s0, "init_"), **system_dict(system, "final_"),
               **params_dict(params))
    np.savez_compressed(os.path.join(OUT, "io_small.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-long", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None

    def want(k):
        return only is None or k in only

    if want("eos"):
        eos_fixture()
    if want("small"):
        for n in (1, 2):
            sc = Scenario(dp=0.02)
            params = make_params(sc, n_subdiv=n)
            s = build_dam_break(sc, params)
            variants = ["slowcellsh"] if n == 1 else ["slowcellshalf", "fastcellshalf"]
            frame_fixture(f"small_n{n}", s, params, variants)
    if want("mid"):
        sc, params, s = mid_collapse(0.01, 80)
        for n in (1, 2):
            prm = replace(params, n_subdiv=n)
            variants = ["slowcellsh"] if n == 1 else ["slowcellshalf"]
            frame_fixture(f"mid5k_n{n}", s, prm, variants)
    if want("uniform"):
        for n in (1, 2):
            s, params = uniform_fluid(3000, h=0.05, seed=7, n_subdiv=n)
            variants = ["slowcellsh"] if n == 1 else ["slowcellshalf"]
            frame_fixture(f"uniform3k_n{n}", s, params, variants)
    if want("c1"):
        sc = Scenario(dp=0.006)
        params = make_params(sc)
        s = build_dam_break(sc, params)
        frame_fixture("c1_n1", s, params, ["slowcellsh"])
    if want("c1mid"):
        sc, params, s = mid_collapse(0.006, 60)
        frame_fixture("c1mid_n1", s, params, ["slowcellsh"])
    if want("traj"):
        sc = Scenario(dp=0.025)
        params = make_params(sc)
        trajectory_fixture("dp025_g", sc, params, gather_cfg("slowcellsh"), 45, keep_states=(1, 2, 40, 41))
        sc = Scenario(dp=0.02)
        params = make_params(sc, n_subdiv=2)
        trajectory_fixture("dp02_n2_g", sc, params, gather_cfg("slowcellshalf"), 12, keep_states=(1,))
    if want("trajc1") and not a.skip_long:
        sc = Scenario(dp=0.006)
        params = make_params(sc)
        trajectory_fixture("c1_g100", sc, params, gather_cfg("slowcellsh"), 100, keep_states=(1, 10))
    if want("drift") and not a.skip_long:
        drift_fixture()
    if want("io"):
        io_fixture()


if __name__ == "__main__":
    main()
