"""Parity of the CUDA path (through the package -> libsphb200 C ABI) with the reference.

Anchors: golden vectors produced by the reference itself (tests/golden), the C oracle
pinned to them (oracle/, tests/test_oracle.py), and reference-measured counts at full size
(SURVEY.md Appendix A.9).  Bars (SURVEY.md §8(a')):
  * NL (cell ids, sort permutation, per-cell ranges) and neighbour counters: bit-exact;
  * forces / density rates / visc_dt: FP64 instantiation bit-exact; FP32 rel_linf <= 1e-5;
  * one-step state rel_linf <= 1e-5 (FP32), dt rel <= 1e-6; FP64 trajectories bit-exact;
  * 1000-step drift vs the reference within the tolerances stated in DESIGN.md.
"""
import types

import numpy as np
import torch
import pytest

import oracle
from conftest import golden, initial_state, scenario_from_npz

pytestmark = pytest.mark.gpu

sph = pytest.importorskip("paper_1110_3711_b200")
from paper_1110_3711_b200 import device as D  # noqa: E402

FRAMES = [("frame_small_n1.npz", "slowcellsh"), ("frame_small_n2.npz", "slowcellshalf"),
          ("frame_small_n2.npz", "fastcellshalf"), ("frame_mid5k_n1.npz", "slowcellsh"),
          ("frame_mid5k_n2.npz", "slowcellshalf"), ("frame_uniform3k_n1.npz", "slowcellsh"),
          ("frame_uniform3k_n2.npz", "slowcellshalf"), ("frame_c1_n1.npz", "slowcellsh"),
          ("frame_c1mid_n1.npz", "slowcellsh")]
FP32_TOL = 1e-5


def frame_objects(z):
    prm = oracle.params_from_npz(z)
    nb, nf = int(z["s_nb"]), int(z["s_nf"])
    system = sph.ParticleSystem(count_fluid=nf, count_boundary=nb, pos=z["s_pos"], vel=z["s_vel"],
                                rho=z["s_rho"], mass_fluid=float(z["s_mass_fluid"]),
                                mass_boundary=float(z["s_mass_boundary"]), ptype=z["s_ptype"],
                                id=z["s_id"])
    derived = sph.DerivedQuantities(press=z["press"], csound=z["csound"], prrho=z["prrho"],
                                    tensil=z["tensil"])
    grid = types.SimpleNamespace(cell_of=z["cell_of"], dims=z["dims"])
    cindex = types.SimpleNamespace()
    return system, derived, grid, cindex, prm


def gather_cfg(variant, precision):
    return sph.EngineConfig(engine="gather", symmetry=False, gather_variant=variant,
                            precision=precision)


# ------------------------------------------------------------------ EOS / NL
def test_device_eos_bit_exact():
    z = golden("eos.npz")
    prm = oracle.params_from_npz(z)
    d = sph.compute_derived(z["rho"], prm)
    for f in ("press", "csound", "prrho", "tensil"):
        assert np.array_equal(getattr(d, f), z[f]), f


@pytest.mark.parametrize("name", sorted({f for f, _ in FRAMES}))
def test_device_nl_bit_exact(name):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    out = D.nl_frame(z["in_pos"], int(z["in_nb"]), prm)
    assert out["error"] is None
    for k in ("cell_of_unsorted", "sort_perm", "cell_of", "fbeg", "fend", "bbeg", "bend"):
        assert np.array_equal(out[k], z[k]), k


@pytest.mark.parametrize("name", ["frame_small_n1.npz", "frame_mid5k_n2.npz"])
def test_device_nl_build_one_call(name):
    """sphb_nl_build (K1 + K2 + K4 in one call) equals the reference's NL outputs."""
    from paper_1110_3711_b200 import _lib
    from paper_1110_3711_b200.physics import grid_desc, grid_dims
    z = golden(name)
    prm = oracle.params_from_npz(z)
    nb = int(z["in_nb"])
    pos = np.asarray(z["in_pos"], np.float32)
    n = pos.shape[0]
    _, dims = grid_dims(prm)
    ncells = int(np.prod(dims))
    posp = torch.zeros((n, 4), dtype=torch.float32, device="cuda")
    posp[:, :3] = torch.as_tensor(pos).cuda()
    i32 = lambda m: torch.empty(m, dtype=torch.int32, device="cuda")  # noqa: E731
    keys, ksort, perm = i32(n), i32(n), i32(n)
    beg, end = i32(2 * ncells), i32(2 * ncells)
    ws = D.Workspace(n, ncells)
    ctrl = D.new_ctrl(torch.device("cuda"))
    g = grid_desc(prm, prm.n_subdiv)
    L = _lib.lib()
    _lib.check(L.sphb_nl_build(ws.handle, _lib.ref(g), posp.data_ptr(), n, nb, keys.data_ptr(),
                               ksort.data_ptr(), perm.data_ptr(), beg.data_ptr(), end.data_ptr(),
                               ctrl.data_ptr(), torch.cuda.current_stream().cuda_stream), "nl_build")
    assert np.array_equal(perm.cpu().numpy().astype(np.int64), z["sort_perm"])
    b, e = beg.cpu().numpy().astype(np.int64), end.cpu().numpy().astype(np.int64)
    for got, key in ((b[:ncells], "bbeg"), (e[:ncells], "bend"), (b[ncells:], "fbeg"), (e[ncells:], "fend")):
        assert np.array_equal(got, z[key]), key


def _grid_params(cell=0.5, n_subdiv=1):
    h = cell * n_subdiv / 2.0
    return oracle.Params(h=h, dp=h / 2, rho0=1000.0, c0=20.0, gamma=7.0, alpha=0.25,
                         g=np.zeros(3), cfl=0.3, domain_min=np.zeros(3), domain_max=np.ones(3),
                         n_subdiv=n_subdiv)


def test_device_cell_known_answers():
    """pkg/tests/test_grid.py:34-62 restated against the device K1."""
    prm = _grid_params()
    pts = np.array([[0.6, 0.1, 0.1], [0.5, 0.1, 0.1], [1.0, 1.0, 1.0], [0.1, 0.6, 0.1],
                    [0.1, 0.1, 0.6], [0.2, 0.2, 0.2]], np.float32)
    out = D.nl_frame(pts, 0, prm)
    assert list(out["cell_of_unsorted"]) == [1, 1, 7, 2, 4, 0]
    out = D.nl_frame(np.array([[0.2, 0.2, 0.2], [-0.1, 0.0, 0.0], [0.3, 0.3, 0.3],
                               [2.0, 0.1, 0.1]], np.float32), 0, prm)
    assert list(out["cell_of_unsorted"]) == [0, -1, 0, -1]
    step, code, index = out["error"]
    assert (step, code, index) == (0, 1, 1)  # first offending index


def test_device_sort_stable_and_lists_segregated():
    """test_grid.py:75-115: stability ([1,2,0]) and per-list sorting."""
    prm = _grid_params()
    out = D.nl_frame(np.array([[0.6, 0.1, 0.1], [0.1, 0.1, 0.1], [0.11, 0.1, 0.1]], np.float32), 0, prm)
    assert list(out["sort_perm"]) == [1, 2, 0]
    rng = np.random.default_rng(6)
    pos = rng.uniform(0, 1, (20000, 3)).astype(np.float32)
    prm = _grid_params(cell=0.05)
    out = D.nl_frame(pos, 8000, prm)
    cell, _, _ = oracle.assign_cells(pos, prm)
    perm = oracle.sort_perm(cell, 8000)
    assert np.array_equal(out["sort_perm"], perm)
    ncells = int(np.prod(out["dims"]))
    fb, fe, bb, be = oracle.cell_index(cell[perm], 8000, ncells)
    assert np.array_equal(out["fbeg"], fb) and np.array_equal(out["bend"], be)


def test_device_nl_empty_and_single():
    prm = _grid_params()
    out = D.nl_frame(np.zeros((0, 3), np.float32), 0, prm)
    assert out["sort_perm"].size == 0 and np.all(out["fbeg"] == 0) and np.all(out["bend"] == 0)
    out = D.nl_frame(np.array([[0.7, 0.7, 0.7]], np.float32), 0, prm)
    assert list(out["sort_perm"]) == [0] and out["fend"][-1] == 1


# ------------------------------------------------------------------ forces
@pytest.mark.parametrize("name,variant", FRAMES)
def test_interact_fp64_bit_exact(name, variant):
    z = golden(name)
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(gather_cfg(variant, "fp64"))
    out = eng.compute(system, derived, grid, cindex, prm, ranges=object())
    assert np.array_equal(out.accel, z[f"{variant}_accel"])
    assert np.array_equal(out.drho_dt, z[f"{variant}_drho"])
    assert np.array_equal(out.visc_dt, z[f"{variant}_visc"])
    c = z[f"{variant}_counters"]
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(c)


@pytest.mark.parametrize("name,variant", FRAMES)
def test_interact_fp32_within_tolerance(name, variant):
    z = golden(name)
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(gather_cfg(variant, "fp32"))
    out = eng.compute(system, derived, grid, cindex, prm, ranges=object())
    nb = system.count_boundary
    assert np.all(out.accel[:nb] == 0.0)
    assert oracle.rel_linf(out.accel, z[f"{variant}_accel"]) <= FP32_TOL
    assert oracle.rel_linf(out.drho_dt, z[f"{variant}_drho"]) <= FP32_TOL
    assert oracle.rel_linf(out.visc_dt, z[f"{variant}_visc"]) <= FP32_TOL
    c = z[f"{variant}_counters"]
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(c)
    out.stats.validate()


@pytest.mark.parametrize("block", [128, 256, 384, 512])
@pytest.mark.parametrize("name,variant", FRAMES)
def test_interact_fp32_each_blocking_vs_reference(name, variant, block):
    """Every FP32 interaction build (pi128 / pi256 / pi384: 4-, 8-, 12-warp CTAs), selected
    through the engine's ``pi_block``, against the reference's own gather output: forces within
    1e-5, counters bit-exact.  The n2 frames run reach 2 (25 stencil rows), where the larger
    blocks stage their candidates in several batches with partial drains."""
    z = golden(name)
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(gather_cfg(variant, "fp32"), pi_block=block)
    out = eng.compute(system, derived, grid, cindex, prm, ranges=object())
    assert eng.last_pi_block == block
    nb = system.count_boundary
    assert np.all(out.accel[:nb] == 0.0)
    for a, f in ((out.accel, "accel"), (out.drho_dt, "drho"), (out.visc_dt, "visc")):
        assert oracle.rel_linf(a, z[f"{variant}_{f}"]) <= FP32_TOL, f
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(z[f"{variant}_counters"])


@pytest.mark.parametrize("name,variant", FRAMES)
def test_paired_kernel_vs_reference(name, variant):
    """The FP32 gather with two targets per lane (k_interact_v12, 512-target bricks; row blocks
    for the ranges order) against the reference's own gather output on every golden frame
    (n1 / n2, all three variants): forces within 1e-5, counters bit-exact."""
    z = golden(name)
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(gather_cfg(variant, "fp32"), pi_kernel="paired")
    out = eng.compute(system, derived, grid, cindex, prm, ranges=object())
    assert eng.last_pi_block == 512
    nb = system.count_boundary
    assert np.all(out.accel[:nb] == 0.0)
    for a, f in ((out.accel, "accel"), (out.drho_dt, "drho"), (out.visc_dt, "visc")):
        assert oracle.rel_linf(a, z[f"{variant}_{f}"]) <= FP32_TOL, f
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(z[f"{variant}_counters"])


CELL_FRAMES = [(f, v) for f, v in FRAMES if v != "fastcellshalf"]


@pytest.mark.parametrize("name,variant", CELL_FRAMES)
def test_symmetric_kernel_vs_reference_gather(name, variant):
    """The symmetric FP32 kernel (each unordered pair evaluated once, the reaction scattered to
    the partner) reproduces the reference's gather output: counters bit-exact (the hit set is
    the same), forces within 1e-5 (summation order only)."""
    z = golden(name)
    system, derived, grid, cindex, prm = frame_objects(z)
    out = sph.make_engine(gather_cfg(variant, "fp32"), pi_kernel="symmetric").compute(
        system, derived, grid, cindex, prm)
    nb = system.count_boundary
    assert np.all(out.accel[:nb] == 0.0)
    for a, f in ((out.accel, "accel"), (out.drho_dt, "drho"), (out.visc_dt, "visc")):
        assert oracle.rel_linf(a, z[f"{variant}_{f}"]) <= FP32_TOL, f
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(z[f"{variant}_counters"])


SYM_FRAMES = ["small_n1", "small_n2", "mid5k_n1", "mid5k_n2", "uniform3k_n1", "c1mid_n1"]


@pytest.mark.parametrize("name", SYM_FRAMES)
@pytest.mark.parametrize("precision,kernel", [("fp32", "symmetric"), ("fp32", "gather"),
                                              ("fp64", "gather")])
def test_cellpairs_symmetric_config_vs_reference(name, precision, kernel):
    """EngineConfig(symmetry=True) -- the reference's CellPairsEngine with run_cells_symmetric --
    reports the symmetric traversal's StepStats (half-stencil candidates, force_evals = unordered
    pairs, unordered ff; cellpairs.py:92-99) whichever device kernel runs; forces within 1e-5
    (FP32) / 1e-12 (FP64: the one-sided sums differ from the symmetric ones in order only) of
    the reference's own output (tests/golden/make_golden_sym.py)."""
    z = golden(f"frame_{name}.npz")
    g = golden(f"sym_{name}.npz")
    system, derived, grid, cindex, prm = frame_objects(z)
    cfg = sph.EngineConfig(symmetry=True, precision=precision)
    out = sph.make_engine(cfg, pi_kernel=kernel).compute(system, derived, grid, cindex, prm)
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(g["sym1_counters"])
    tol = FP32_TOL if precision == "fp32" else 1e-12
    for a, f in ((out.accel, "accel"), (out.drho_dt, "drho"), (out.visc_dt, "visc")):
        assert oracle.rel_linf(a, g[f"sym1_{f}"]) <= tol, f
    assert out.stats.engine_tag.startswith("b200-cellpairs-on")


@pytest.mark.parametrize("name", SYM_FRAMES)
def test_cellpairs_asymmetric_config_vs_reference(name):
    """EngineConfig(symmetry=False): run_cells_asymmetric's counters and (FP64) its forces bit
    for bit -- the one-sided cell traversal accumulates in the gather kernels' order."""
    z = golden(f"frame_{name}.npz")
    g = golden(f"sym_{name}.npz")
    system, derived, grid, cindex, prm = frame_objects(z)
    out = sph.make_engine(sph.EngineConfig(symmetry=False, precision="fp64")).compute(
        system, derived, grid, cindex, prm)
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(g["asym1_counters"])
    assert np.array_equal(out.accel, g["asym1_accel"]) and np.array_equal(out.drho_dt, g["asym1_drho"])
    assert np.array_equal(out.visc_dt, g["asym1_visc"])


def test_engine_auto_blocking_is_the_run_rule():
    z = golden("frame_c1_n1.npz")
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(gather_cfg("slowcellsh", "fp32"))
    eng.compute(system, derived, grid, cindex, prm)
    assert eng.last_pi_block == sph.sim.initial_pi_block(system.n, prm.n_subdiv)
    with pytest.raises(ValueError, match="pi_block"):
        sph.make_engine(gather_cfg("slowcellsh", "fp32"), pi_block=64)


def test_interact_deterministic_and_momentum():
    z = golden("frame_uniform3k_n1.npz")  # fluid only
    system, derived, grid, cindex, prm = frame_objects(z)
    eng = sph.make_engine(sph.EngineConfig(engine="b200", symmetry=False))
    a = eng.compute(system, derived, grid, cindex, prm)
    b = eng.compute(system, derived, grid, cindex, prm)
    assert np.array_equal(a.accel, b.accel) and np.array_equal(a.drho_dt, b.drho_dt)
    m = system.mass_fluid
    total = (m * a.accel).sum(axis=0)
    assert np.abs(total).max() <= 1e-3 * (m * np.abs(a.accel)).sum()


def test_engine_errors_match_reference():
    z = golden("frame_small_n1.npz")
    system, derived, grid, cindex, prm = frame_objects(z)
    bad = types.SimpleNamespace(cell_of=grid.cell_of[:-1])
    with pytest.raises(ValueError, match="mismatch"):
        sph.make_engine(sph.EngineConfig()).compute(system, derived, bad, cindex, prm)
    with pytest.raises(ValueError, match="n_subdiv"):
        sph.make_engine(gather_cfg("fastcellshalf", "fp32")).compute(system, derived, grid, cindex, prm)


# ------------------------------------------------------------------ trajectories
TRAJ = [("traj_dp025_g.npz", "slowcellsh"), ("traj_dp02_n2_g.npz", "slowcellshalf"),
        ("traj_c1_g100.npz", "slowcellsh")]


@pytest.mark.parametrize("name,variant", TRAJ)
def test_run_simulation_fp64_bit_exact(name, variant):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    sc = scenario_from_npz(z)
    steps = z["dt"].shape[0]
    system, stats = sph.run_simulation(sc, prm, gather_cfg(variant, "fp64"), max_steps=steps)
    assert np.array_equal(np.array([s.dt for s in stats]), z["dt"])
    got = np.array([[s.candidate_pairs, s.true_pairs, s.force_evals, s.ff_force_evals] for s in stats])
    assert np.array_equal(got, z["counters"])
    for f in ("id", "pos", "vel", "rho"):
        assert np.array_equal(getattr(system, f), z["final_" + f]), f


def test_run_simulation_fp32_one_step_and_short_trajectory():
    z = golden("traj_c1_g100.npz")
    prm = oracle.params_from_npz(z)
    sc = scenario_from_npz(z)
    cfg = gather_cfg("slowcellsh", "fp32")
    s1, st1 = sph.run_simulation(sc, prm, cfg, max_steps=1)
    assert abs(st1[0].dt - z["dt"][0]) <= 1e-6 * z["dt"][0]
    assert np.array_equal(s1.id, z["st1_id"])
    for f in ("pos", "vel", "rho"):
        assert oracle.rel_linf(getattr(s1, f), z["st1_" + f]) <= FP32_TOL, f
    s10, st10 = sph.run_simulation(sc, prm, cfg, max_steps=10)
    order = np.argsort(s10.id)
    ref_order = np.argsort(z["st10_id"])
    for f in ("pos", "vel", "rho"):
        assert oracle.rel_linf(getattr(s10, f)[order], z["st10_" + f][ref_order]) <= 1e-4, f
    dts = np.array([s.dt for s in st10])
    np.testing.assert_allclose(dts, z["dt"][:10], rtol=1e-5)


@pytest.mark.parametrize("pi_block,pi_kernel", [("auto", "gather"), (384, "gather"),
                                               (384, "symmetric"), ("auto", "paired")])
def test_drift_1000_steps_fp32_vs_reference(pi_block, pi_kernel):
    """SURVEY.md §8(d) drift bar: E = KE + PE + IE; tolerances stated in DESIGN.md.  Run with
    the size rule's build (C1: pi256) and with the production 384-target build forced."""
    z = golden("drift_c1.npz")
    prm = oracle.params_from_npz(z)
    sc = sph.Scenario(dp=0.006)
    rows = []

    class Sink:
        def emit(self, step, system, derived):
            rows.append((step,) + oracle.energy_terms(system.pos, system.vel, system.rho,
                                                      system.count_boundary, system.mass_fluid,
                                                      system.mass_boundary, prm))

    system, stats = sph.run_simulation(sc, prm, gather_cfg("slowcellsh", "fp32"), max_steps=1000,
                                       snapshot_every=10, snapshot_sink=Sink(), stage_timing=False,
                                       pi_block=pi_block, pi_kernel=pi_kernel)
    got = np.array(rows)
    ref = z["diag"][1:]
    assert got.shape == ref.shape and np.array_equal(got[:, 0], ref[:, 0])
    emech0 = z["diag"][0][2] + z["diag"][0][3]  # PE0 + IE0 (KE0 = 0)
    e_got = got[:, 1] + got[:, 2] + got[:, 3]
    e_ref = ref[:, 1] + ref[:, 2] + ref[:, 3]
    assert np.max(np.abs(e_got - e_ref)) / emech0 <= 1e-4
    ke_ref = ref[:, 1]
    mask = ke_ref > 1e-3 * ke_ref.max()
    assert np.max(np.abs(got[mask, 1] - ke_ref[mask]) / ke_ref[mask]) <= 1e-3
    assert np.max(np.abs(got[:, 4] - ref[:, 4])) / prm.rho0 <= 1e-5
    sdt = np.sum([s.dt for s in stats])
    assert abs(sdt - z["dt"].sum()) / z["dt"].sum() <= 1e-4
    assert system.n == int(z["final_nb"]) + int(z["final_nf"])


# ------------------------------------------------------------------ divergence
def test_divergence_escaped_particle():
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    system.pos[-1] = prm.domain_max.astype(np.float32) + np.float32(1.0)
    with pytest.raises(sph.DivergenceError) as err:
        sph.run_simulation(system, prm, sph.EngineConfig(), max_steps=1)
    assert err.value.step == 0
    assert err.value.particle_id == int(system.id[-1])
    assert "left the domain" in str(err.value)


@pytest.mark.parametrize("chunk", [1, 256])
def test_particle_escaping_during_the_final_step_ends_normally(chunk):
    """The reference checks the stop rule before assign_cells (sim.py:302-315): a particle that
    leaves the domain during the last step does not raise; one more step does."""
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    dmax = np.asarray(prm.domain_max, np.float64)
    system.pos[-1] = (dmax - 1e-6).astype(np.float32)
    system.vel[-1] = np.float32(5.0)
    pid = int(system.id[-1])
    out, stats = sph.run_simulation(system.copy(), prm, sph.EngineConfig(), max_steps=1, chunk=chunk)
    assert len(stats) == 1
    assert np.any(out.pos[out.id == pid] > dmax.astype(np.float32))
    with pytest.raises(sph.DivergenceError) as err:
        sph.run_simulation(system.copy(), prm, sph.EngineConfig(), max_steps=2, chunk=chunk)
    assert err.value.step == 1 and err.value.particle_id == pid


def test_divergence_nonfinite_state():
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    system.vel[-1, 0] = np.float32(np.nan)
    with pytest.raises(sph.DivergenceError) as err:
        sph.run_simulation(system, prm, sph.EngineConfig(), max_steps=1)
    assert err.value.step == 0


def test_run_zero_steps_and_t_end():
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc)
    expect = sph.build_dam_break(sc, prm)
    system, stats = sph.run_simulation(sc, prm, sph.EngineConfig(), max_steps=0)
    assert stats == [] and np.array_equal(system.pos, expect.pos)
    _, stats = sph.run_simulation(sc, prm, sph.EngineConfig(), t_end=1e-3)
    assert sum(s.dt for s in stats) >= 1e-3 and sum(s.dt for s in stats[:-1]) < 1e-3


def test_stage_times_cover_the_step():
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    _, stats = sph.run_simulation(sc, prm, sph.EngineConfig(), max_steps=8)
    for s in stats[2:]:
        assert s.stage_nl_s >= 0 and s.stage_pi_s > 0 and s.stage_su_s >= 0
        staged = s.stage_nl_s + s.stage_pi_s + s.stage_su_s
        assert staged <= s.wall_seconds * 1.001


def test_snapshots_and_stats_sink():
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc)
    seen, lines = [], []

    class Sink:
        def emit(self, step, system, derived):
            seen.append((step, system.n))

    sph.run_simulation(sc, prm, sph.EngineConfig(), max_steps=6, snapshot_every=2,
                       snapshot_sink=Sink(), stats_sink=lines.append)
    assert [s[0] for s in seen] == [2, 4, 6] and len(lines) == 6


def test_graph_capture_matches_eager():
    z = golden("traj_dp025_g.npz")
    prm = oracle.params_from_npz(z)
    pos, vel, rho, ids, nb, mf, mb = initial_state(z)
    s = sph.ParticleSystem(count_fluid=pos.shape[0] - nb, count_boundary=nb, pos=pos, vel=vel,
                           rho=rho, mass_fluid=mf, mass_boundary=mb,
                           ptype=np.r_[np.zeros(nb, np.uint8), np.ones(pos.shape[0] - nb, np.uint8)],
                           id=ids)
    sim = D.DeviceSim(s, prm, reach=1, precision=1)
    sim.capture(5)
    for _ in range(9):
        sim.run_graph()
    p, v, r, i, _, _ = sim.download()
    assert int(sim.ctrl_host()["step"]) == 45
    assert np.array_equal(i, z["final_id"]) and np.array_equal(p, z["final_pos"])
    assert np.array_equal(v, z["final_vel"]) and np.array_equal(r, z["final_rho"])


def test_movers_only_sort_matches_radix():
    """sphb_step's movers-only sort (nl.cu k_mv_*) gives the radix sort's permutation
    (grid.py:107-109 stable order) at every step; cap -1 forces the radix path, a small cap
    mixes both paths from step to step."""
    sc = sph.named_scenario("c1")
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    sims = []
    for cap in (None, -1, 40):
        sim = D.DeviceSim(system, prm, reach=1, precision=0)
        if cap is not None:
            sim.ws.set_mover_cap(cap)
        sims.append(sim)
    modes = {0: [], 1: [], 2: []}
    for step in range(60):
        for k, sim in enumerate(sims):
            sim.launch_step()
            modes[k].append(sim.ws.sort_info())
        a = sims[0]
        for b in sims[1:]:
            assert np.array_equal(a.perm[:a.n].cpu().numpy(), b.perm[:b.n].cpu().numpy()), step
            assert np.array_equal(a.keys_sorted[:a.n].cpu().numpy(), b.keys_sorted[:b.n].cpu().numpy())
            assert np.array_equal(a.beg.cpu().numpy(), b.beg.cpu().numpy())
        ks = a.keys_sorted[:a.n].cpu().numpy().view(np.uint32)
        assert np.all(ks[1:] >= ks[:-1])
    assert modes[0][0][1] == 1  # first step after upload: no previous order -> radix
    assert all(m == 0 for _, m in modes[0][1:]) and sum(mv for mv, _ in modes[0]) > 0
    assert all(m == 1 for _, m in modes[1])
    assert all(m == int(mv > 40) for mv, m in modes[2][1:])  # the cap decides per step
    fa, fb = sims[0].download(), sims[1].download()
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)


def test_movers_only_sort_rejects_an_inconsistent_previous_order():
    """sphb_sort_ranges trusts keys_sorted / beg / end only after checking them on the device:
    corrupted, the step falls back to the radix passes and still sorts correctly."""
    sc = sph.named_scenario("c1")
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    a = D.DeviceSim(system, prm, reach=1, precision=0)
    b = D.DeviceSim(system, prm, reach=1, precision=0)
    b.ws.set_mover_cap(-1)
    for _ in range(5):
        a.launch_step()
        b.launch_step()
    n = a.n
    for corrupt in ("swap", "range"):
        if corrupt == "swap":  # keys_sorted no longer ascending
            ks = a.keys_sorted[:n].clone()
            a.keys_sorted[:1] = ks[n - 1:n]
            a.keys_sorted[n - 1:n] = ks[:1]
        else:  # a present key's old range shifted by one row
            nz = torch.nonzero(a.end - a.beg > 1).flatten()
            a.beg[int(nz[len(nz) // 2])] += 1
        a.launch_step()
        b.launch_step()
        assert a.ws.sort_info()[1] == 1, corrupt  # radix fallback
        assert np.array_equal(a.perm[:n].cpu().numpy(), b.perm[:n].cpu().numpy()), corrupt
        a.launch_step()
        b.launch_step()
        assert a.ws.sort_info()[1] == 0  # the fallback re-established the order
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)


def test_state_soa_round_trip():
    """sphb_state_to_soa / sphb_state_from_soa: the reference's (pos, vel, rho, vel_prev,
    rho_prev) arrays <-> the step rows, bit for bit, by row ranges."""
    from paper_1110_3711_b200 import _lib
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    sim = D.DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1)
    for _ in range(3):
        sim.launch_step()
    n = sim.n
    L, s = _lib.lib(), torch.cuda.current_stream().cuda_stream
    soa = [torch.empty((n, 3), device="cuda"), torch.empty((n, 3), device="cuda"),
           torch.empty(n, device="cuda"), torch.empty((n, 3), device="cuda"), torch.empty(n, device="cuda")]
    ptrs = [t.data_ptr() for t in soa]
    _lib.check(L.sphb_state_to_soa(0, n, sim.posp.data_ptr(), sim.velr.data_ptr(), sim.prev.data_ptr(),
                                   *ptrs, s), "to_soa")
    p, v, r, _, vp, rp = sim.download()
    for got, want in zip(soa, (p, v, r, vp, rp)):
        assert np.array_equal(got.cpu().numpy(), want)
    before = [t.clone() for t in (sim.posp, sim.velr, sim.prev)]
    for t in (sim.posp, sim.velr, sim.prev):
        t.zero_()
    half = n // 2  # two row ranges, as the chunked copies use them
    for lo, hi in ((0, half), (half, n)):
        _lib.check(L.sphb_state_from_soa(lo, hi - lo, *ptrs, sim.posp.data_ptr(), sim.velr.data_ptr(),
                                         sim.prev.data_ptr(), s), "from_soa")
    torch.cuda.synchronize()
    assert torch.equal(sim.posp[:n, :3], before[0][:n, :3]) and torch.all(sim.posp[:n, 3] == 0)
    assert torch.equal(sim.velr[:n], before[1][:n]) and torch.equal(sim.prev[:n], before[2][:n])
    assert L.sphb_state_from_soa(-1, 1, *ptrs, 0, 0, 0, s) == _lib.SPHB_E_INVALID


@pytest.mark.parametrize("variant", ["match", "mismatch"])
def test_interact_plan_side_stream_equals_inline(monkeypatch, variant):
    """The interaction's block list built on the workspace's side stream during K3
    (sphb_interact_plan, taken by the next sphb_interact) gives the same steps as the list built
    in line; a plan that does not match the call (the build changed in between) is waited for
    and rebuilt."""
    from paper_1110_3711_b200 import _lib
    sc = sph.named_scenario("c2")  # >= 2^19 rows: the side-stream plan is active
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    L = _lib.lib()
    real = L.sphb_interact_plan
    blk = 384 if variant == "match" else 256
    out = []
    for plan in (True, False):
        sim = D.DeviceSim(system, prm, reach=1, record_capacity=16)
        sim.set_pi_block(blk)
        if not plan:
            monkeypatch.setattr(L, "sphb_interact_plan", lambda *args: 0)
        elif variant == "mismatch":  # planned for 384, then the 256-target build runs
            def planned_other(*args, sim=sim):
                sim.set_pi_block(384)
                rc = real(*args)
                sim.set_pi_block(256)
                return rc
            monkeypatch.setattr(L, "sphb_interact_plan", planned_other)
        for _ in range(3):
            sim.launch_step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
        torch.cuda.synchronize()
        monkeypatch.setattr(L, "sphb_interact_plan", real)
        recs = sim.records(0, 3)
        out.append((sim.download(), recs["candidate_pairs"], recs["hits_ordered"]))
    (a_state, a_cand, a_hits), (b_state, b_cand, b_hits) = out
    assert np.array_equal(a_cand, b_cand) and np.array_equal(a_hits, b_hits)
    for x, y in zip(a_state, b_state):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("shuffle", [False, True])
def test_upload_keep_order_equals_reset(shuffle):
    """A host round trip of the state (sphb_state_to_soa -> host -> sphb_state_from_soa) and
    first_keys_resync(keep_order=True) (sphb_workspace_clear_hist / trust_order) sorts the next
    step by the movers-only path, and the steps equal those after a full reset (radix sort);
    with the rows shuffled inside each list before the upload too (every row is then a mover)."""
    from paper_1110_3711_b200 import _lib
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    a = D.DeviceSim(system, prm, reach=1)
    b = D.DeviceSim(system, prm, reach=1)
    for _ in range(3):
        a.launch_step()
        b.launch_step()
    n, nb = a.n, a.nb
    L, s = _lib.lib(), torch.cuda.current_stream().cuda_stream
    shapes = [(n, 3), (n, 3), (n,), (n, 3), (n,)]
    soa = [torch.empty(sh, device="cuda") for sh in shapes]
    ptrs = [t.data_ptr() for t in soa]
    _lib.check(L.sphb_state_to_soa(0, n, a.posp.data_ptr(), a.velr.data_ptr(), a.prev.data_ptr(),
                                   *ptrs, s), "to_soa")
    ids = a.id[:n].clone()
    if shuffle:
        g = torch.Generator(device="cpu").manual_seed(7)
        perm = torch.cat([torch.randperm(nb, generator=g), nb + torch.randperm(n - nb, generator=g)]).cuda()
        soa = [t[perm].contiguous() for t in soa]
        ptrs = [t.data_ptr() for t in soa]
        ids = ids[perm]
    host = [t.cpu() for t in soa]  # the round trip through host memory
    for sim, keep in ((a, True), (b, False)):
        dev = [t.cuda() for t in host]
        _lib.check(L.sphb_state_from_soa(0, n, *[t.data_ptr() for t in dev], sim.posp.data_ptr(),
                                         sim.velr.data_ptr(), sim.prev.data_ptr(), s), "from_soa")
        sim.id[:n].copy_(ids)
        sim.first_keys_resync(keep_order=keep)
        sim.launch_step()
        torch.cuda.synchronize()
        movers, mode = sim.ws.sort_info()
        assert mode == (0 if keep else 1), (keep, mode, movers)
        if keep:
            assert (movers > n // 2) if shuffle else (movers < n // 100)
        sim.launch_step()
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("block", [256, 384, "symmetric", "paired"])
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_pi_block_matches_128(name, block):
    """The 256- and 384-target blockings (pi256 / pi384: 8- / 12-warp CTAs) gives the 128-target one's counters
    exactly and its forces within the FP32 tolerance, step after step."""
    sc = sph.named_scenario(name)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    a = D.DeviceSim(system, prm, reach=1, precision=0)
    b = D.DeviceSim(system, prm, reach=1, precision=0)
    if block in ("symmetric", "paired"):
        b.set_pi_kernel(block)
    else:
        b.set_pi_block(block)
    for step in range(4):
        a.launch_step()
        b.launch_step()
        ra, rb = a.records(step, step + 1), b.records(step, step + 1)
        if block in ("symmetric", "paired") and step > 0:
            # the reactions (symmetric) / the pair sums (paired) add in another order: after one
            # step positions differ in
            # the last bit, the lattice's pairs sitting exactly at r = 2h may flip and the two
            # runs are no longer the same state (same-frame parity: the C2 / C3 / collapsed
            # oracle tests and the golden frames)
            for f in ("hits_ordered", "force_evals", "ff_force_evals"):
                assert abs(int(ra[f][0]) - int(rb[f][0])) <= 1e-6 * int(ra[f][0]), f
            continue
        for f in ("candidate_pairs", "hits_ordered", "force_evals", "ff_force_evals"):
            assert int(ra[f][0]) == int(rb[f][0]), f
        for x, y in zip(a.forces(), b.forces()):
            assert oracle.rel_linf(x.cpu().numpy(), y.cpu().numpy()) <= FP32_TOL
        assert abs(float(ra["dt"][0]) / float(rb["dt"][0]) - 1.0) <= 1e-6
    assert 0.0 < b.pi_lane_use() <= 1.0 and int(b.ctrl_host()["nblk"][0]) < int(a.ctrl_host()["nblk"][0])


def test_run_simulation_tuned_policy():
    """pi_kernel="tuned": tuning chunks run one step per candidate build (gather on the size
    rule's blocking, paired), the faster build runs on; the run equals the gather run within
    the FP32 tolerance (the first step's counters exactly: same state) and tunes at the start
    and every ``retune_every`` steps."""
    sc = sph.named_scenario("c2")
    prm = sph.make_params(sc)
    cfg = gather_cfg("slowcellsh", "fp32")
    sa, sta = sph.run_simulation(sc, prm, cfg, max_steps=24, chunk=8, pi_kernel="gather")
    sb, stb = sph.run_simulation(sc, prm, cfg, max_steps=24, chunk=8, pi_kernel="tuned",
                                 retune_every=8)
    assert len(stb) == 24 and [s.step for s in stb] == list(range(24))
    assert (sta[0].candidate_pairs, sta[0].true_pairs, sta[0].force_evals) == \
        (stb[0].candidate_pairs, stb[0].true_pairs, stb[0].force_evals)
    for a, b in zip(sta, stb):
        assert abs(a.true_pairs - b.true_pairs) <= 1e-5 * a.true_pairs
        assert abs(a.dt / b.dt - 1.0) <= 1e-4
    oa, ob = np.argsort(sa.id), np.argsort(sb.id)
    for f in ("pos", "vel", "rho"):
        assert oracle.rel_linf(getattr(sb, f)[ob], getattr(sa, f)[oa]) <= 1e-4, f
    sim = D.DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, precision=0)
    t = sim.tune_pi(sim.pi_candidates(1))
    assert set(t) == {"gather/384", "paired/512"} and all(v > 0 for v in t.values())
    assert (sim.pi_kernel, sim.pi_block) in (("gather", 384), ("paired", 512))


def test_run_simulation_auto_blocking_follows_the_size_rule():
    """pi_block="auto" = sim.initial_pi_block(n) for the whole run (256 below 4 large blocks
    per SM); explicit 384 on a small case agrees with 128 (counters exact, FP32 tolerance)."""
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    cfg = sph.EngineConfig(engine="gather", symmetry=False, gather_variant="slowcellsh")
    s_auto, st_auto = sph.run_simulation(sc, prm, cfg, max_steps=20, chunk=10)
    s_256, st_256 = sph.run_simulation(sc, prm, cfg, max_steps=20, chunk=10, pi_block=256)
    s_128, st_128 = sph.run_simulation(sc, prm, cfg, max_steps=20, chunk=10, pi_block=128)
    s_384, st_384 = sph.run_simulation(sc, prm, cfg, max_steps=20, chunk=10, pi_block=384)
    assert s_auto.n < sph.sim.PI_LARGE_MIN_TARGETS
    assert [x.true_pairs for x in st_auto] == [x.true_pairs for x in st_256]
    for f in ("pos", "vel", "rho"):
        assert np.array_equal(getattr(s_auto, f), getattr(s_256, f)), f
    assert [x.true_pairs for x in st_384[:5]] == [x.true_pairs for x in st_128[:5]]
    for f in ("pos", "vel", "rho"):
        assert oracle.rel_linf(getattr(s_384, f), getattr(s_128, f)) <= 1e-4, f
    with pytest.raises(ValueError, match="pi_block"):
        sph.run_simulation(sc, prm, cfg, max_steps=1, pi_block=64)


# ------------------------------------------------------------------ full sizes
def _sorted_frame(system, prm):
    """The device-NL-sorted frame of ``system`` with its derived quantities."""
    nl = D.nl_frame(system.pos, system.count_boundary, prm)
    perm = nl["sort_perm"]
    ss = sph.ParticleSystem(count_fluid=system.count_fluid, count_boundary=system.count_boundary,
                            pos=system.pos[perm], vel=system.vel[perm], rho=system.rho[perm],
                            mass_fluid=system.mass_fluid, mass_boundary=system.mass_boundary,
                            ptype=system.ptype[perm], id=system.id[perm])
    return ss, sph.compute_derived(ss.rho, prm), nl


def _oracle_frame(system, prm):
    """Oracle NL (numpy restatement of grid.py, pinned to the reference) + the oracle C gather
    (bit-exact to the reference's gather kernels) on ``system``'s sorted frame."""
    cell, dims, _ = oracle.assign_cells(system.pos, prm)
    perm = oracle.sort_perm(cell, system.count_boundary)
    cidx = oracle.cell_index(cell[perm], system.count_boundary, int(np.prod(dims)))
    ref = oracle.gather(system.pos[perm], system.vel[perm], system.rho[perm], system.count_boundary,
                        system.mass_fluid, system.mass_boundary, cell[perm], dims, cidx, prm,
                        variant="slowcellsh" if prm.n_subdiv == 1 else "slowcellshalf")
    return cell, perm, cidx, ref


def _check_vs_oracle(out, ref, tol=FP32_TOL):
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(ref["counters"])
    for a, b, f in ((out.accel, ref["accel"], "accel"), (out.drho_dt, ref["drho_dt"], "drho"),
                    (out.visc_dt, ref["visc_dt"], "visc")):
        assert oracle.rel_linf(a, b) <= tol, f


@pytest.fixture(scope="module")
def c2_frames():
    cache = {}

    def get(n_subdiv):
        if n_subdiv not in cache:
            sc = sph.named_scenario("c2")
            prm = sph.make_params(sc, n_subdiv=n_subdiv)
            system = sph.build_dam_break(sc, prm)
            ss, der, nl = _sorted_frame(system, prm)
            cache[n_subdiv] = (system, prm, ss, der, nl, _oracle_frame(system, prm))
        return cache[n_subdiv]
    return get


def _device_counters(name, n_subdiv, precision="fp32"):
    sc = sph.named_scenario(name)
    prm = sph.make_params(sc, n_subdiv=n_subdiv)
    system = sph.build_dam_break(sc, prm)
    nl = D.nl_frame(system.pos, system.count_boundary, prm)
    perm = nl["sort_perm"]
    ss = sph.ParticleSystem(count_fluid=system.count_fluid, count_boundary=system.count_boundary,
                            pos=system.pos[perm], vel=system.vel[perm], rho=system.rho[perm],
                            mass_fluid=system.mass_fluid, mass_boundary=system.mass_boundary,
                            ptype=system.ptype[perm], id=system.id[perm])
    der = sph.compute_derived(ss.rho, prm)
    grid = types.SimpleNamespace(cell_of=nl["cell_of"])
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    out = sph.make_engine(gather_cfg(variant, precision)).compute(ss, der, grid, None, prm)
    return ss, der, nl, prm, out


@pytest.mark.slow
@pytest.mark.parametrize("n_subdiv", [1, 2])
def test_c2_symmetric_kernel_vs_oracle(c2_frames, n_subdiv):
    """C2 through the symmetric FP32 kernel: gather counters bit-exact and forces within 1e-5 of
    the oracle gather; and the cellpairs-symmetric config's counters equal the oracle's
    symmetric traversal (oracle.cellpairs, bit-exact to the reference's)."""
    system, prm, ss, der, nl, (cell, perm, cidx, ref) = c2_frames(n_subdiv)
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    grid = types.SimpleNamespace(cell_of=nl["cell_of"])
    out = sph.make_engine(gather_cfg(variant, "fp32"), pi_kernel="symmetric").compute(ss, der, grid, None, prm)
    _check_vs_oracle(out, ref)
    sym = oracle.cellpairs(ss.pos, ss.vel, ss.rho, ss.count_boundary, ss.mass_fluid, ss.mass_boundary,
                           cell_dims(prm), cidx, prm, symmetric=True, threads=16)
    outs = sph.make_engine(sph.EngineConfig(symmetry=True), pi_kernel="symmetric").compute(
        ss, der, grid, None, prm)
    _check_vs_oracle(outs, sym)


def cell_dims(prm):
    from paper_1110_3711_b200.physics import grid_dims
    return grid_dims(prm)[1]


@pytest.mark.slow
@pytest.mark.parametrize("n_subdiv,block", [(1, 128), (1, 256), (1, 384), (1, "paired"), (2, 128),
                                            (2, 384), (2, "paired")])
def test_c2_each_blocking_vs_oracle(c2_frames, n_subdiv, block):
    """C2 (1,142,622 particles) through the engine with each FP32 build forced: counters
    bit-exact and forces within 1e-5 of the oracle gather (bit-exact to the reference).  At
    n_subdiv 2 (reach 2, 25 stencil rows of h-cells) the larger blocks need several staging
    batches per block."""
    system, prm, ss, der, nl, (cell, perm, cidx, ref) = c2_frames(n_subdiv)
    assert np.array_equal(nl["sort_perm"], perm)
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    eng = sph.make_engine(gather_cfg(variant, "fp32"), pi_block=512 if block == "paired" else block,
                          pi_kernel="paired" if block == "paired" else "gather")
    out = eng.compute(ss, der, types.SimpleNamespace(cell_of=nl["cell_of"]), None, prm)
    assert eng.last_pi_block == (512 if block == "paired" else block)
    _check_vs_oracle(out, ref)


@pytest.mark.slow
def test_c3_10m_production_build_vs_oracle():
    """C3 (10,200,478 particles, the bench workload), initial frame, the production FP32 build
    (engine "auto" = pi384 at this size, the build bench.py times) against the oracle gather
    on the oracle's own NL: counters bit-exact, accel / drho_dt / visc_dt within 1e-5."""
    sc = sph.named_scenario("c3")
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    ss, der, nl = _sorted_frame(system, prm)
    cell, perm, cidx, ref = _oracle_frame(system, prm)
    assert np.array_equal(nl["sort_perm"], perm)
    eng = sph.make_engine(gather_cfg("slowcellsh", "fp32"))
    out = eng.compute(ss, der, types.SimpleNamespace(cell_of=nl["cell_of"]), None, prm)
    assert eng.last_pi_block == 384
    _check_vs_oracle(out, ref)
    for kern in ("symmetric", "paired"):
        out = sph.make_engine(gather_cfg("slowcellsh", "fp32"), pi_kernel=kern).compute(
            ss, der, types.SimpleNamespace(cell_of=nl["cell_of"]), None, prm)
        _check_vs_oracle(out, ref)


@pytest.mark.slow
def test_collapsed_c2_production_build_vs_fp64():
    """A collapsed frame (C2 after 2,000 FP32 steps, t ~ 0.14 s: the column is falling, cells
    hold 30-100 particles): the production FP32 build against the FP64 kernel, which is
    bit-identical to the reference's gather, and against the oracle gather on the oracle NL."""
    sc = sph.named_scenario("c2")
    prm = sph.make_params(sc)
    cfg = gather_cfg("slowcellsh", "fp32")
    system, _ = sph.run_simulation(sc, prm, cfg, max_steps=2000, stage_timing=False)
    ss, der, nl = _sorted_frame(system, prm)
    grid = types.SimpleNamespace(cell_of=nl["cell_of"])
    counts = np.bincount(nl["cell_of"][ss.count_boundary:])
    assert counts.max() > 64  # no longer the lattice
    o64 = sph.make_engine(gather_cfg("slowcellsh", "fp64")).compute(ss, der, grid, None, prm)
    cell, perm, cidx, ref = _oracle_frame(system, prm)
    assert np.array_equal(nl["sort_perm"], perm)
    assert np.array_equal(o64.accel, ref["accel"]) and np.array_equal(o64.drho_dt, ref["drho_dt"])
    for block in (384, 128):
        eng = sph.make_engine(cfg, pi_block=block)
        out = eng.compute(ss, der, grid, None, prm)
        _check_vs_oracle(out, ref)
    for kern in ("symmetric", "paired"):
        out = sph.make_engine(cfg, pi_kernel=kern).compute(ss, der, grid, None, prm)
        _check_vs_oracle(out, ref)


@pytest.mark.slow
def test_c2_1m_parity_vs_oracle():
    """C2 (1,142,622 particles), initial frame: device NL bit-exact vs the oracle; FP32 forces
    vs the oracle C gather (bit-exact to the reference) within 1e-5; counters bit-exact;
    FP64 forces bit-exact."""
    ss, der, nl, prm, out = _device_counters("c2", 1)
    sc = sph.named_scenario("c2")
    system = sph.build_dam_break(sc, prm)
    cell, dims, _ = oracle.assign_cells(system.pos, prm)
    perm = oracle.sort_perm(cell, system.count_boundary)
    assert np.array_equal(nl["cell_of_unsorted"], cell) and np.array_equal(nl["sort_perm"], perm)
    cidx = oracle.cell_index(cell[perm], system.count_boundary, int(np.prod(dims)))
    for k, a in zip(("fbeg", "fend", "bbeg", "bend"), cidx):
        assert np.array_equal(nl[k], a), k
    ref = oracle.gather(ss.pos, ss.vel, ss.rho, ss.count_boundary, ss.mass_fluid,
                        ss.mass_boundary, cell[perm], dims, cidx, prm)
    assert [out.stats.candidate_pairs, out.stats.true_pairs, out.stats.force_evals,
            out.stats.ff_force_evals] == list(ref["counters"])
    for a, b in ((out.accel, ref["accel"]), (out.drho_dt, ref["drho_dt"]), (out.visc_dt, ref["visc_dt"])):
        assert oracle.rel_linf(a, b) <= FP32_TOL
    grid = types.SimpleNamespace(cell_of=nl["cell_of"])
    out64 = sph.make_engine(gather_cfg("slowcellsh", "fp64")).compute(ss, der, grid, None, prm)
    assert np.array_equal(out64.accel, ref["accel"]) and np.array_equal(out64.drho_dt, ref["drho_dt"])
    assert np.array_equal(out64.visc_dt, ref["visc_dt"])


@pytest.mark.slow
@pytest.mark.parametrize("n_subdiv,cand", [(1, 16_164_890_622), (2, 9_401_964_162)])
def test_c3_10m_counters_match_reference_measurement(n_subdiv, cand):
    """C3 (10,200,478 particles): the reference's own counts at its second step (SURVEY.md
    Appendix A.9), reproduced by the bit-exact FP64 device trajectory.  (Lattice pairs sit
    exactly on the 2h cutoff, so step-1 counts are only reproducible with bit-identical
    step-0 motion.)"""
    sc = sph.named_scenario("c3")
    prm = sph.make_params(sc, n_subdiv=n_subdiv)
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    _, stats = sph.run_simulation(sc, prm, gather_cfg(variant, "fp64"), max_steps=2,
                                  stage_timing=False)
    st = stats[1]
    assert st.true_pairs == 1_210_590_160
    assert st.force_evals == 2_421_180_320
    assert st.ff_force_evals == 2_373_133_760
    assert st.candidate_pairs == cand


# ------------------------------------------------------------------ X-slab decomposition
@pytest.mark.parametrize("nslabs,precision", [(2, 1), (3, 1), (3, 0)])
def test_device_virtual_slabs_match_single_domain(nslabs, precision):
    """k virtual slabs on one GPU (LoopbackComm; the same exchange code as the NCCL path)
    against the single-domain device run: step 0 identical, 20 steps close (id-aligned)."""
    import slab_torch_reference as tslab
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    steps = 20
    sim = tslab.device_slab_simulation(system, prm, nslabs, precision=precision)
    sim.run(steps)
    cfg = gather_cfg("slowcellsh", "fp64" if precision == 1 else "fp32")
    ref, stats = sph.run_simulation(sph.build_dam_break(sc, prm), prm, cfg, max_steps=steps,
                                    stage_timing=False)
    st0 = sim.ranks[0].stats[0]
    assert st0["dt"] == stats[0].dt
    assert [st0["candidate_pairs"], st0["true_pairs"], st0["force_evals"], st0["ff_force_evals"]] \
        == [stats[0].candidate_pairs, stats[0].true_pairs, stats[0].force_evals,
            stats[0].ff_force_evals]
    pos, vel, rho, ids, _ = sim.gather_host()
    assert np.array_equal(np.sort(ids), np.sort(ref.id))
    a, b = np.argsort(ids), np.argsort(ref.id)
    tol = 1e-9 if precision == 1 else 1e-5
    assert oracle.rel_linf(pos[a], ref.pos[b]) <= tol
    assert oracle.rel_linf(vel[a], ref.vel[b]) <= max(tol, 1e-4 if precision == 0 else tol)
    assert oracle.rel_linf(rho[a], ref.rho[b]) <= tol


def test_device_slabs_c2_fp32_counters_match_single_domain():
    """C2 (1.14M particles) on three virtual X slabs in FP32: the ranks' windows are large
    enough for the 384-target build's hybrid brick / row blocking and the count-pass
    candidate counter, over edge and interior grids -- the first step's counters (candidates
    from the cell tables, exact hits) and dt equal the single-domain step's."""
    from paper_1110_3711_b200 import dslab
    sc = sph.named_scenario("c2")
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    sim = dslab.DeviceSlabSim(system, prm, dslab.DevLoopbackComm(3), precision=0)
    sim.run(2)
    got = sim.records(0, 2)
    one = D.DeviceSim(system, prm, reach=1, record_capacity=8)
    one.set_pi_block(384)
    for _ in range(2):
        one.launch_step()
    torch.cuda.synchronize()
    want = one.records(0, 2)
    for k in ("candidate_pairs", "hits_ordered", "force_evals", "ff_force_evals"):
        assert int(got[k][0]) == int(want[k][0]), k
    assert got["dt"][0] == want["dt"][0]


@pytest.mark.parametrize("nslabs,precision", [(1, 1), (2, 1), (3, 0), (4, 1)])
def test_device_resident_slabs_match_single_domain(nslabs, precision):
    """The production multi-GPU stepper (dslab.DeviceSlabSim: device classify/scatter/unpack,
    one host sync per step) on k virtual ranks vs the single-domain run: every step's dt and
    counters identical, 20-step state close (id-aligned), no particle lost or duplicated."""
    from paper_1110_3711_b200 import dslab
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    steps = 20
    sim = dslab.DeviceSlabSim(system, prm, dslab.DevLoopbackComm(nslabs), precision=precision)
    sim.run(steps)
    cfg = gather_cfg("slowcellsh", "fp64" if precision == 1 else "fp32")
    ref, stats = sph.run_simulation(sph.build_dam_break(sc, prm), prm, cfg, max_steps=steps,
                                    stage_timing=False)
    recs = sim.records(0, steps)
    if precision == 1:  # FP64: identical hit sets and dt every step
        assert np.array_equal(recs["dt"], np.array([s.dt for s in stats]))
        got = np.stack([recs["candidate_pairs"], recs["hits_ordered"] // 2, recs["force_evals"],
                        recs["ff_force_evals"]], 1).astype(np.int64)
        want = np.array([[s.candidate_pairs, s.true_pairs, s.force_evals, s.ff_force_evals]
                         for s in stats], np.int64)
        assert np.array_equal(got, want)
    else:
        assert recs["dt"][0] == stats[0].dt
        assert int(recs["hits_ordered"][0]) // 2 == stats[0].true_pairs
    pos, vel, rho, ids, fl = sim.gather_host()
    assert np.array_equal(ids, np.sort(ref.id))
    b = np.argsort(ref.id)
    tol = 1e-9 if precision == 1 else 1e-5
    assert oracle.rel_linf(pos, ref.pos[b]) <= tol
    assert oracle.rel_linf(vel, ref.vel[b]) <= max(tol, 1e-4 if precision == 0 else tol)
    assert oracle.rel_linf(rho, ref.rho[b]) <= tol
    assert int(fl.sum()) == system.count_fluid


@pytest.mark.parametrize("transport", ["copy", "peer"])
def test_device_slabs_two_processes(tmp_path, transport):
    """DeviceSlabSim with DevDistComm across two real processes (torchrun, gloo: they share
    this box's GPU; NCCL only changes the transport): every step's dt and counters equal the
    single-domain FP64 run's, the id set is conserved and the 20-step state matches."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = tmp_path / "mp.npz"
    steps = 20
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    proc = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                           str(port), os.path.join(root, "tests", "slab_mp_worker.py"), str(out),
                           str(steps), transport], capture_output=True, text=True, timeout=600, cwd=root)
    assert proc.returncode == 0, proc.stderr[-3000:]
    z = np.load(out)
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    ref, stats = sph.run_simulation(sph.build_dam_break(sc, prm), prm, gather_cfg("slowcellsh", "fp64"),
                                    max_steps=steps, stage_timing=False)
    assert len(z["bounds"]) == 3
    assert np.array_equal(z["dt"], np.array([s.dt for s in stats]))
    got = np.stack([z["cand"], z["hits"] // 2, z["evals"], z["ff"]], 1).astype(np.int64)
    want = np.array([[s.candidate_pairs, s.true_pairs, s.force_evals, s.ff_force_evals] for s in stats])
    assert np.array_equal(got, want)
    b = np.argsort(ref.id)
    assert np.array_equal(z["id"], ref.id[b])
    for f in ("pos", "vel", "rho"):
        assert oracle.rel_linf(z[f], getattr(ref, f)[b]) <= 1e-9, f


def test_device_slabs_regrow_mid_step(monkeypatch):
    """Row capacities with no headroom: arrivals outgrow a rank's arrays in the middle of a step
    (DevRank._grow_mid_step: new primary arrays and workspace while this step's sorted arrays
    are still being read) -- the FP64 run still matches the single domain at every step."""
    from paper_1110_3711_b200 import dslab
    monkeypatch.setattr(dslab.DevRank, "CAP_FACTOR", 1.0)
    monkeypatch.setattr(dslab.DevRank, "CAP_SLACK", 0)
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    steps = 12
    sim = dslab.DeviceSlabSim(sph.build_dam_break(sc, prm), prm, dslab.DevLoopbackComm(3), precision=1)
    caps0 = [r.cap for r in sim.ranks]
    sim.run(steps)
    assert any(r.cap > c for r, c in zip(sim.ranks, caps0))  # a rank did regrow
    ref, stats = sph.run_simulation(sph.build_dam_break(sc, prm), prm, gather_cfg("slowcellsh", "fp64"),
                                    max_steps=steps, stage_timing=False)
    recs = sim.records(0, steps)
    assert np.array_equal(recs["dt"], np.array([s.dt for s in stats]))
    assert np.array_equal(recs["hits_ordered"].astype(np.int64) // 2,
                          np.array([s.true_pairs for s in stats], np.int64))
    pos, vel, rho, ids, fl = sim.gather_host()
    assert np.array_equal(ids, np.sort(ref.id))
    b = np.argsort(ref.id)
    assert oracle.rel_linf(pos, ref.pos[b]) <= 1e-9 and oracle.rel_linf(rho, ref.rho[b]) <= 1e-9


def test_device_slabs_rebalance_keeps_results():
    """Time-balanced slab bounds (DeviceSlabSim.rebalance): forced uneven times move the
    bounds by several columns (multi-hop settle), a measured rebalance runs every 6 steps; ids
    are conserved and the FP64 run still matches the single domain at every step."""
    from paper_1110_3711_b200 import dslab
    sc = sph.Scenario(dp=0.006)
    prm = sph.make_params(sc)
    system = sph.build_dam_break(sc, prm)
    steps = 18
    sim = dslab.DeviceSlabSim(system, prm, dslab.DevLoopbackComm(3), precision=1, rebalance_every=6)
    b0 = sim.bounds.copy()
    sim.run(4)
    new = sim.rebalance(times=[1.0, 1.0, 8.0])  # slab 2 slow: columns move two slabs left
    assert not np.array_equal(new, b0) and np.all(np.diff(new) >= 1)
    sim.run(steps - 4)
    cfg = gather_cfg("slowcellsh", "fp64")
    ref, stats = sph.run_simulation(sph.build_dam_break(sc, prm), prm, cfg, max_steps=steps,
                                    stage_timing=False)
    recs = sim.records(0, steps)
    assert np.array_equal(recs["dt"], np.array([s.dt for s in stats]))
    assert np.array_equal(recs["hits_ordered"].astype(np.int64) // 2,
                          np.array([s.true_pairs for s in stats], np.int64))
    pos, vel, rho, ids, fl = sim.gather_host()
    assert np.array_equal(ids, np.sort(ref.id))
    b = np.argsort(ref.id)
    assert oracle.rel_linf(pos, ref.pos[b]) <= 1e-9 and oracle.rel_linf(rho, ref.rho[b]) <= 1e-9
