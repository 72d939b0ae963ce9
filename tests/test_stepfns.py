"""The reference's module-level NL and SU functions on the device (paper_1110_3711_b200.grid,
sim.compute_dt / verlet_update) against the reference's own outputs (tests/golden) and the
hand examples of its tests (test_grid.py)."""
import types

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu

sph = pytest.importorskip("paper_1110_3711_b200")
G = sph.grid

FRAMES = ["frame_small_n1.npz", "frame_small_n2.npz", "frame_mid5k_n1.npz", "frame_mid5k_n2.npz",
          "frame_uniform3k_n1.npz"]


def _system(z, prefix="in_"):
    nb = int(z[prefix + "nb"]) if prefix + "nb" in z.files else int(z["s_nb"])
    pos = z[prefix + "pos"]
    n = pos.shape[0]
    return sph.ParticleSystem(count_fluid=n - nb, count_boundary=nb, pos=pos.copy(),
                              vel=np.zeros_like(pos), rho=np.full(n, 1000.0, np.float32),
                              mass_fluid=1.0, mass_boundary=1.0,
                              ptype=np.r_[np.zeros(nb, np.uint8), np.ones(n - nb, np.uint8)],
                              id=np.arange(n, dtype=np.int64))


@pytest.mark.parametrize("name", FRAMES)
def test_grid_functions_match_reference(name):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    system = _system(z)
    grid = G.assign_cells(system.pos, prm)
    assert np.array_equal(grid.cell_of, z["cell_of_unsorted"])
    assert np.array_equal(grid.dims, z["dims"]) and grid.cell_size == float(z["cell_size"])
    system, inverse = G.reorder(system, grid)
    assert np.array_equal(grid.sort_perm, z["sort_perm"])
    assert np.array_equal(inverse[grid.sort_perm], np.arange(system.n))
    assert np.array_equal(grid.cell_of, z["cell_of"])
    cidx = G.build_cell_index(system, grid)
    for got, key in ((cidx.fluid.begin, "fbeg"), (cidx.fluid.end, "fend"),
                     (cidx.boundary.begin, "bbeg"), (cidx.boundary.end, "bend")):
        assert np.array_equal(got, z[key]), key
    if "rng_fbeg" in z.files:
        dr = G.build_dual_ranges(cidx, grid.dims, prm.n_subdiv)
        assert np.array_equal(dr.fluid.begin, z["rng_fbeg"]) and np.array_equal(dr.fluid.end, z["rng_fend"])
        assert np.array_equal(dr.boundary.begin, z["rng_bbeg"]) and np.array_equal(dr.boundary.end, z["rng_bend"])
        assert dr.fluid.nranges == G.ranges_per_cell(prm.n_subdiv)


def test_grid_known_answers_and_errors():
    # CellBeginEnd hand example (test_grid.py:127-130)
    cbe = G.build_cell_begin_end(np.array([0, 0, 2, 2, 2]), 4)
    assert cbe.begin.tolist() == [0, 2, 2, 5] and cbe.end.tolist() == [2, 2, 5, 5]
    empty = G.build_cell_begin_end(np.zeros(0, np.int64), 3)
    assert empty.begin.tolist() == [0, 0, 0] and empty.end.tolist() == [0, 0, 0]
    with pytest.raises(ValueError, match="nondecreasing"):
        G.build_cell_begin_end(np.array([1, 0]), 2)
    with pytest.raises(ValueError, match="n_subdiv"):
        G.ranges_per_cell(3)
    assert len(G.forward_offsets(1)) == 13 and len(G.forward_offsets(2)) == 62
    assert G.forward_cells((0, 0, 0), (3, 3, 3)).shape == (7, 3)
    assert abs(G.search_volume_ratio(1) - 27 / (4 / 3 * np.pi)) < 1e-15
    # reorder refuses out-of-domain particles (grid.py:104-105)
    z = golden("frame_small_n1.npz")
    prm = oracle.params_from_npz(z)
    system = _system(z)
    system.pos[3] = np.float32(1e3)
    grid = G.assign_cells(system.pos, prm)
    assert grid.cell_of[3] == G.OUT_OF_DOMAIN and grid.out_of_domain.tolist() == [3]
    with pytest.raises(ValueError, match="out-of-domain"):
        G.reorder(system, grid)


@pytest.mark.parametrize("name,variant", [("frame_small_n1.npz", "slowcellsh"),
                                          ("frame_mid5k_n1.npz", "slowcellsh"),
                                          ("frame_small_n2.npz", "fastcellshalf")])
def test_compute_dt_and_verlet_match_reference(name, variant):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    nb, nf = int(z["s_nb"]), int(z["s_nf"])
    mk = lambda: sph.ParticleSystem(count_fluid=nf, count_boundary=nb, pos=z["s_pos"].copy(),  # noqa: E731
                                    vel=z["s_vel"].copy(), rho=z["s_rho"].copy(),
                                    mass_fluid=float(z["s_mass_fluid"]),
                                    mass_boundary=float(z["s_mass_boundary"]), ptype=z["s_ptype"],
                                    id=z["s_id"])
    forces = types.SimpleNamespace(accel=z[f"{variant}_accel"], drho_dt=z[f"{variant}_drho"],
                                   visc_dt=z[f"{variant}_visc"])
    system = mk()
    derived = sph.compute_derived(system.rho, prm)
    dt = sph.compute_dt(forces, system, derived, prm)
    assert dt == float(z[f"{variant}_dt"])
    # step 0: the corrector branch
    st = sph.VerletState.from_system(system, prm.verlet_corrector_stride)
    sph.verlet_update(st, system, forces, prm, dt)
    assert np.array_equal(system.pos, z[f"{variant}_step1_pos"])
    assert np.array_equal(system.vel, z[f"{variant}_step1_vel"])
    assert np.array_equal(system.rho, z[f"{variant}_step1_rho"])
    assert st.step == 1 and np.array_equal(st.vel_prev, z["s_vel"]) and np.array_equal(st.rho_prev, z["s_rho"])
    # step 1: the leapfrog branch from the recorded history
    system = mk()
    st = sph.VerletState(vel_prev=z[f"{variant}_hist_vel_prev"].copy(),
                         rho_prev=z[f"{variant}_hist_rho_prev"].copy(), step=1,
                         corrector_stride=prm.verlet_corrector_stride)
    sph.verlet_update(st, system, forces, prm, dt)
    assert np.array_equal(system.pos, z[f"{variant}_step1nc_pos"])
    assert np.array_equal(system.vel, z[f"{variant}_step1nc_vel"])
    assert np.array_equal(system.rho, z[f"{variant}_step1nc_rho"])
    with pytest.raises(ValueError, match="dt must be positive"):
        sph.verlet_update(st, system, forces, prm, 0.0)


def test_reference_loop_structure_with_device_functions():
    """sim.py:300-350's loop written with this package's module-level functions and engine
    (FP64) reproduces the reference's own 45-step trajectory bit for bit (dt per step, final
    state): the parity trick of SURVEY.md §8(b) on the GPU box, where the reference is absent."""
    from conftest import initial_state
    z = golden("traj_dp025_g.npz")
    prm = oracle.params_from_npz(z)
    pos, vel, rho, ids, nb, mf, mb = initial_state(z)
    n = pos.shape[0]
    system = sph.ParticleSystem(count_fluid=n - nb, count_boundary=nb, pos=pos.copy(), vel=vel.copy(),
                                rho=rho.copy(), mass_fluid=mf, mass_boundary=mb,
                                ptype=np.r_[np.zeros(nb, np.uint8), np.ones(n - nb, np.uint8)],
                                id=ids.copy())
    state = sph.VerletState.from_system(system, prm.verlet_corrector_stride)
    engine = sph.make_engine(sph.EngineConfig(engine="gather", symmetry=False,
                                              gather_variant="slowcellsh", precision="fp64"))
    dts = []
    for step in range(int(z["dt"].shape[0])):
        grid = G.assign_cells(system.pos, prm)
        assert grid.out_of_domain.size == 0
        G.reorder(system, grid, extra_arrays=(state.vel_prev, state.rho_prev))
        cindex = G.build_cell_index(system, grid)
        derived = sph.compute_derived(system.rho, prm)
        forces = engine.compute(system, derived, grid, cindex, prm)
        dt = sph.compute_dt(forces, system, derived, prm)
        sph.verlet_update(state, system, forces, prm, dt)
        dts.append(dt)
    assert np.array_equal(np.array(dts), z["dt"])
    for f, key in (("pos", "final_pos"), ("vel", "final_vel"), ("rho", "final_rho"), ("id", "final_id")):
        assert np.array_equal(getattr(system, f), z[key]), f
