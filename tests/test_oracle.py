"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

Every check is bit equality: the oracle restates the reference's numpy NL/SU
exactly and its numba pair loop in C with the same f64 operation order.
"""
import numpy as np
import pytest

import oracle
from conftest import golden, initial_state

FRAMES = [("frame_small_n1.npz", ["slowcellsh"]),
          ("frame_small_n2.npz", ["slowcellshalf", "fastcellshalf"]),
          ("frame_mid5k_n1.npz", ["slowcellsh"]),
          ("frame_mid5k_n2.npz", ["slowcellshalf"]),
          ("frame_uniform3k_n1.npz", ["slowcellsh"]),
          ("frame_uniform3k_n2.npz", ["slowcellshalf"]),
          ("frame_c1_n1.npz", ["slowcellsh"]),
          ("frame_c1mid_n1.npz", ["slowcellsh"])]


def test_pack_params_bit_exact():
    z = golden("eos.npz")
    prm = oracle.params_from_npz(z)
    assert np.array_equal(oracle.pack_params(prm, 1.0e-3, 2.0e-3), z["pp"])


def test_derived_bit_exact():
    z = golden("eos.npz")
    prm = oracle.params_from_npz(z)
    press, cs, prrho, ten = oracle.derived(z["rho"], prm)
    for got, want in ((press, z["press"]), (cs, z["csound"]), (prrho, z["prrho"]), (ten, z["tensil"])):
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name,variants", FRAMES)
def test_nl_bit_exact(name, variants):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    cell_of, dims, cs = oracle.assign_cells(z["in_pos"], prm)
    assert np.array_equal(cell_of, z["cell_of_unsorted"])
    assert np.array_equal(dims, z["dims"]) and cs == float(z["cell_size"])
    nb = int(z["in_nb"])
    perm = oracle.sort_perm(cell_of, nb)
    assert np.array_equal(perm, z["sort_perm"])
    assert np.array_equal(cell_of[perm], z["cell_of"])
    fbeg, fend, bbeg, bend = oracle.cell_index(cell_of[perm], nb, int(np.prod(dims)))
    for got, key in ((fbeg, "fbeg"), (fend, "fend"), (bbeg, "bbeg"), (bend, "bend")):
        assert np.array_equal(got, z[key]), key
    if "rng_fbeg" in z.files:
        rb, re = oracle.build_ranges(fbeg, fend, dims, prm.n_subdiv)
        assert np.array_equal(rb, z["rng_fbeg"]) and np.array_equal(re, z["rng_fend"])
        rb, re = oracle.build_ranges(bbeg, bend, dims, prm.n_subdiv)
        assert np.array_equal(rb, z["rng_bbeg"]) and np.array_equal(re, z["rng_bend"])


@pytest.mark.parametrize("name,variants", FRAMES)
def test_gather_forces_dt_verlet_bit_exact(name, variants):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    nb = int(z["s_nb"])
    cidx = (z["fbeg"], z["fend"], z["bbeg"], z["bend"])
    for v in variants:
        out = oracle.gather(z["s_pos"], z["s_vel"], z["s_rho"], nb, float(z["s_mass_fluid"]),
                            float(z["s_mass_boundary"]), z["cell_of"], z["dims"], cidx, prm,
                            variant=v, nthreads=4)
        assert np.array_equal(out["accel"], z[f"{v}_accel"]), v
        assert np.array_equal(out["drho_dt"], z[f"{v}_drho"]), v
        assert np.array_equal(out["visc_dt"], z[f"{v}_visc"]), v
        assert np.array_equal(out["counters"], z[f"{v}_counters"]), v
        dt = oracle.compute_dt(out["accel"], out["visc_dt"], out["derived"][1], nb, prm)
        assert dt == float(z[f"{v}_dt"])
        p, vv, r, _, _ = oracle.verlet_update(0, z["s_pos"], z["s_vel"], z["s_rho"], z["s_vel"],
                                              z["s_rho"], out["accel"], out["drho_dt"], nb, prm, dt)
        assert np.array_equal(p, z[f"{v}_step1_pos"])
        assert np.array_equal(vv, z[f"{v}_step1_vel"])
        assert np.array_equal(r, z[f"{v}_step1_rho"])
        p, vv, r, _, _ = oracle.verlet_update(1, z["s_pos"], z["s_vel"], z["s_rho"],
                                              z[f"{v}_hist_vel_prev"], z[f"{v}_hist_rho_prev"],
                                              out["accel"], out["drho_dt"], nb, prm, dt)
        assert np.array_equal(p, z[f"{v}_step1nc_pos"])
        assert np.array_equal(vv, z[f"{v}_step1nc_vel"])
        assert np.array_equal(r, z[f"{v}_step1nc_rho"])


def test_gather_thread_count_independent():
    z = golden("frame_mid5k_n1.npz")
    prm = oracle.params_from_npz(z)
    cidx = (z["fbeg"], z["fend"], z["bbeg"], z["bend"])
    outs = [oracle.gather(z["s_pos"], z["s_vel"], z["s_rho"], int(z["s_nb"]),
                          float(z["s_mass_fluid"]), float(z["s_mass_boundary"]), z["cell_of"],
                          z["dims"], cidx, prm, nthreads=t) for t in (1, 3)]
    assert np.array_equal(outs[0]["accel"], outs[1]["accel"])


def test_recomputed_derived_mode_bitwise_equal():
    """physics.py:238-243: the in-loop recomputation gives the same bits (test_engines.py:201-207)."""
    z = golden("frame_small_n1.npz")
    prm = oracle.params_from_npz(z)
    cidx = (z["fbeg"], z["fend"], z["bbeg"], z["bend"])
    args = (z["s_pos"], z["s_vel"], z["s_rho"], int(z["s_nb"]), float(z["s_mass_fluid"]),
            float(z["s_mass_boundary"]), z["cell_of"], z["dims"], cidx, prm)
    a = oracle.gather(*args, dmode=0)
    b = oracle.gather(*args, dmode=1)
    assert np.array_equal(a["accel"], b["accel"]) and np.array_equal(a["drho_dt"], b["drho_dt"])


@pytest.mark.parametrize("name,variant", [("traj_dp025_g.npz", "slowcellsh"),
                                          ("traj_dp02_n2_g.npz", "slowcellshalf"),
                                          ("traj_c1_g100.npz", "slowcellsh")])
def test_trajectory_bit_exact(name, variant):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    steps = z["dt"].shape[0]
    pos, vel, rho, ids, nb, mf, mb = initial_state(z)
    p, v, r, i, stats = oracle.run_simulation(pos, vel, rho, ids, nb, mf, mb, prm, steps,
                                              variant=variant, nthreads=8)
    assert np.array_equal(np.array([s["dt"] for s in stats]), z["dt"])
    assert np.array_equal(np.array([s["counters"] for s in stats]), z["counters"])
    assert np.array_equal(i, z["final_id"])
    assert np.array_equal(p, z["final_pos"])
    assert np.array_equal(v, z["final_vel"])
    assert np.array_equal(r, z["final_rho"])


def test_energy_functional_matches_generator():
    z = golden("drift_c1.npz")
    prm = oracle.params_from_npz(z)
    e = oracle.energy_terms(z["final_pos"], z["final_vel"], z["final_rho"], int(z["final_nb"]),
                            float(z["final_mass_fluid"]), float(z["final_mass_boundary"]), prm)
    np.testing.assert_allclose(e, z["diag"][-1][1:], rtol=1e-12)


def test_brute_force_agrees_with_gather():
    z = golden("frame_mid5k_n1.npz")
    prm = oracle.params_from_npz(z)
    bf = oracle.brute_force(z["s_pos"], z["s_vel"], z["s_rho"], int(z["s_nb"]),
                            float(z["s_mass_fluid"]), float(z["s_mass_boundary"]), prm)
    assert bf["true_pairs"] == int(z["slowcellsh_counters"][1])
    assert oracle.rel_linf(bf["accel"], z["slowcellsh_accel"]) < 1e-4
    assert oracle.rel_linf(bf["drho_dt"], z["slowcellsh_drho"]) < 1e-4


# ------------------------------------------------------------------ cell-pair engines
SYM_FRAMES = ["small_n1", "small_n2", "mid5k_n1", "mid5k_n2", "uniform3k_n1", "c1mid_n1"]


@pytest.mark.parametrize("name", SYM_FRAMES)
@pytest.mark.parametrize("tag,symmetric,threads", [("sym1", True, 1), ("symT", True, 4),
                                                   ("asym1", False, 1)])
def test_cellpairs_bit_exact(name, tag, symmetric, threads):
    """oracle.cellpairs == the reference's CellPairsEngine (run_cells_symmetric /
    run_cells_asymmetric, private-accumulator threading at T = 4), bit for bit, on the
    frames' sorted state (tests/golden/make_golden_sym.py ran the reference)."""
    z = golden(f"frame_{name}.npz")
    g = golden(f"sym_{name}.npz")
    prm = oracle.params_from_npz(z)
    out = oracle.cellpairs(z["s_pos"], z["s_vel"], z["s_rho"], int(z["s_nb"]),
                           float(z["s_mass_fluid"]), float(z["s_mass_boundary"]), z["dims"],
                           (z["fbeg"], z["fend"], z["bbeg"], z["bend"]), prm,
                           symmetric=symmetric, threads=threads, block_of_cells=10)
    assert np.array_equal(out["counters"], g[f"{tag}_counters"])
    assert np.array_equal(out["accel"], g[f"{tag}_accel"])
    assert np.array_equal(out["drho_dt"], g[f"{tag}_drho"])
    assert np.array_equal(out["visc_dt"], g[f"{tag}_visc"])


@pytest.mark.parametrize("name", SYM_FRAMES)
def test_symmetric_counters_relate_to_gather(name):
    """The reference's counter contract between traversals: same unordered true pairs,
    symmetric evals = true (each pair evaluated once), ff halves (ordered -> unordered)."""
    g = golden(f"sym_{name}.npz")
    s, a = g["sym1_counters"], g["asym1_counters"]
    assert s[1] == a[1] and s[2] == s[1] and a[2] == 2 * a[1] and 2 * s[3] == a[3]
    assert np.array_equal(g["symT_counters"], s)
