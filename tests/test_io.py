"""CPU tests of the I/O surface (snapshots.py) and the host side of the extensions.

The snapshot CSV text and the stats JSON lines are pinned byte-for-byte against what the
reference itself wrote (tests/golden/io_small.npz, make_golden.py io_fixture)."""
import json

import numpy as np
import pytest

from conftest import golden

sph = pytest.importorskip("paper_1110_3711_b200")
from paper_1110_3711_b200 import snapshots as S  # noqa: E402
from paper_1110_3711_b200.model import PistonMotion, validate  # noqa: E402


def _system(z, prefix):
    return sph.ParticleSystem(count_fluid=int(z[prefix + "nf"]), count_boundary=int(z[prefix + "nb"]),
                              pos=z[prefix + "pos"], vel=z[prefix + "vel"], rho=z[prefix + "rho"],
                              mass_fluid=float(z[prefix + "mass_fluid"]),
                              mass_boundary=float(z[prefix + "mass_boundary"]),
                              ptype=z[prefix + "ptype"], id=z[prefix + "id"])


def _press(rho, z):
    """Tait EOS in the reference's f64 order, rounded to f32 (physics.py:119-121)."""
    b = float(z["p_c0"]) ** 2 * float(z["p_rho0"]) / float(z["p_gamma"])
    return (b * ((rho.astype(np.float64) / float(z["p_rho0"])) ** float(z["p_gamma"]) - 1.0)).astype(np.float32)


@pytest.mark.parametrize("prefix,key", [("init_", "csv_init"), ("final_", "csv_step3")])
def test_snapshot_text_matches_reference(prefix, key):
    z = golden("io_small.npz")
    s = _system(z, prefix)
    snap = S.Snapshot(id=s.id, ptype=s.ptype, pos=s.pos, vel=s.vel, rho=s.rho,
                      press=_press(s.rho, z))
    assert S.format_snapshot(snap) == str(z[key])


def test_snapshot_round_trip_and_compare(tmp_path):
    z = golden("io_small.npz")
    s = _system(z, "final_")
    snap = S.Snapshot(id=s.id, ptype=s.ptype, pos=s.pos, vel=s.vel, rho=s.rho, press=_press(s.rho, z))
    p = tmp_path / "a.csv"
    S.write_snapshot(p, snap)
    back = S.read_snapshot(p)
    for f in ("id", "ptype", "pos", "vel", "rho", "press"):
        assert np.array_equal(getattr(back, f), getattr(snap, f)), f
    rep = S.compare_snapshots(snap, back)
    assert rep.passed and rep.worst().max_rel == 0.0
    shuffled = S.Snapshot(**{f: getattr(back, f)[::-1].copy() for f in ("id", "ptype", "pos", "vel", "rho", "press")})
    assert S.compare_snapshots(snap, shuffled).passed
    worse = S.Snapshot(**{f: getattr(back, f).copy() for f in ("id", "ptype", "pos", "vel", "rho", "press")})
    worse.pos[3, 0] += np.float32(0.1)
    assert not S.compare_snapshots(snap, worse).passed
    with pytest.raises(ValueError, match="counts differ"):
        S.compare_snapshots(snap, S.Snapshot(**{f: getattr(back, f)[1:] for f in
                                                ("id", "ptype", "pos", "vel", "rho", "press")}))
    (tmp_path / "bad.csv").write_text("x,y\n1,2\n")
    with pytest.raises(ValueError, match="unexpected snapshot header"):
        S.read_snapshot(tmp_path / "bad.csv")


def test_stats_lines_match_reference():
    z = golden("io_small.npz")
    for line in z["stats_lines"]:
        rec = json.loads(str(line))
        st = sph.StepStats(step=rec["step"], dt=rec["dt"], candidate_pairs=rec["candidate_pairs"],
                           true_pairs=rec["true_pairs"], force_evals=rec["force_evals"],
                           wall_seconds=rec["wall_s"], stage_nl_s=rec["stage_nl_s"],
                           stage_pi_s=rec["stage_pi_s"], stage_su_s=rec["stage_su_s"])
        assert S.stats_line(st) == str(line)
        assert tuple(rec) == S.STATS_KEYS


def test_dir_sink_background_writer(tmp_path):
    z = golden("io_small.npz")
    s = _system(z, "final_")
    derived = sph.DerivedQuantities(press=_press(s.rho, z), csound=s.rho, prrho=s.rho, tensil=s.rho)
    with S.DirSink(str(tmp_path)) as sink:
        sink.emit(3, s, derived)
        sink.emit(6, s, derived)
    assert open(tmp_path / "snapshot_000003.csv").read() == str(z["csv_step3"])
    assert (tmp_path / "snapshot_000006.csv").exists()


# ------------------------------------------------------------------ extension host logic
def test_wave_tank_builder_piston_ids():
    sc = sph.named_scenario("c5_small")
    prm = sph.make_wave_tank_params(sc)
    s = sph.build_wave_tank(sc, prm)
    pm = prm.piston
    ny, nz = int(sc.wall_counts()[1]), int(sc.wall_counts()[2])
    assert (pm.id0, pm.id1) == (0, (ny + 1) * nz)
    assert np.all(s.pos[pm.id0:pm.id1, 0] == np.float32(sc.tank_min[0]))
    assert np.all(s.pos[pm.id0:pm.id1, 2] > sc.tank_min[2])
    rest = s.pos[pm.id1:s.count_boundary]
    assert not np.any((rest[:, 0] == np.float32(sc.tank_min[0])) & (rest[:, 2] > sc.tank_min[2]))
    assert np.array_equal(s.id, np.arange(s.n))
    fl = s.pos[s.count_boundary:]
    assert fl[:, 0].min() == np.float32(sc.tank_min[0] + sc.dp)  # one dp in front of the piston
    assert s.count_fluid == sc.fluid_count
    # C5 size: ~40M fluid
    assert sph.named_scenario("c5").fluid_count == 40060170


def test_piston_law_and_extension_validation():
    pm = PistonMotion(id0=0, id1=10, x0=0.5, stroke=0.2, period=2.0)
    assert pm.x(0.0) == 0.5 and abs(pm.x(1.0) - 0.7) < 1e-15 and abs(pm.v(0.5) - 0.1 * np.pi) < 1e-12
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    assert (prm.kernel, prm.integrator, prm.piston) == ("cubic", "verlet", None)
    for bad, msg in ((dict(kernel="quintic"), "kernel"), (dict(integrator="rk4"), "integrator"),
                     (dict(piston=PistonMotion(0, 1, 0.0, 0.1, 0.0)), "piston")):
        with pytest.raises(ValueError, match=msg):
            sph.make_params(sc, **bad)
    p = sph.make_params(sc, kernel="wendland")
    from paper_1110_3711_b200.physics import kernel_w, pack_params
    pp = pack_params(p, 1.0, 1.0)
    assert pp[3] == 21.0 / (16.0 * np.pi * p.h ** 3)
    assert pp[6] == 1.0 / kernel_w(p.dp, p.h, "wendland")
    # normalisation: integral of W over its support is 1 (both kernels)
    r = np.linspace(0.0, 2.0 * p.h, 200001)
    for k in ("cubic", "wendland"):
        integral = np.trapezoid(4.0 * np.pi * r * r * kernel_w(r, p.h, k), r)
        assert abs(integral - 1.0) < 1e-6, k
    validate(p)


def test_symplectic_restatement_free_motion():
    """No neighbours and no gravity: both stages reduce to exact free flight r += dt v."""
    import oracle
    pos = np.array([[0.1, 0.1, 0.1], [0.5, 0.5, 0.5]], np.float32)
    vel = np.array([[0.0, 0.0, 0.0], [1.0, -2.0, 0.5]], np.float32)
    rho = np.full(2, 1000.0, np.float32)
    z3 = np.zeros((2, 3))
    prm = sph.make_params(sph.Scenario(dp=0.02))
    prm = sph.SimParams(h=prm.h, dp=prm.dp, rho0=prm.rho0, c0=prm.c0, gamma=prm.gamma, alpha=prm.alpha,
                        g=np.zeros(3), cfl=prm.cfl, domain_min=prm.domain_min, domain_max=prm.domain_max)
    dt = 1e-3
    p1, v1, r1, vp, rp = oracle.symplectic_stage(0, pos, vel, rho, vel, rho, z3, np.zeros(2), 1, prm, dt)
    p2, v2, r2, _, _ = oracle.symplectic_stage(1, p1, v1, r1, vp, rp, z3, np.zeros(2), 1, prm, dt)
    assert np.array_equal(v2, vel) and np.array_equal(r2, rho)
    np.testing.assert_allclose(p2[1], pos[1] + dt * vel[1], rtol=0, atol=1e-7)
    assert np.array_equal(p2[0], pos[0])  # boundary row untouched


def test_boundary_force_validation_and_restatement():
    import oracle
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    for bad in (sph.BoundaryForce(d=0.0, r0=0.01), sph.BoundaryForce(d=1.0, r0=3 * prm.h),
                sph.BoundaryForce(d=1.0, r0=0.01, p1=4, p2=4)):
        with pytest.raises(ValueError, match="boundary force"):
            sph.make_params(sc, boundary_force=bad)
    from paper_1110_3711_b200.physics import params_desc
    d = params_desc(sph.make_params(sc, boundary_force=sph.BoundaryForce(d=2.0, r0=0.01)), 1.0, 1.0, 0, 0)
    assert (d.wall_d, d.wall_r0, d.wall_p1, d.wall_p2) == (2.0, 0.01, 12, 4)
    assert params_desc(prm, 1.0, 1.0, 0, 0).wall_d == 0.0  # off by default: the reference
    # one pair at r = 0.8 r0 along x: analytic Lennard-Jones magnitude, repulsive (+x)
    pos = np.array([[0.0, 0.0, 0.0], [0.008, 0.0, 0.0]], np.float32)
    a = oracle.wall_accel(pos, 1, 0.01, 2.0)
    r = float(np.float32(0.008))
    assert a[0].tolist() == [0.0, 0.0, 0.0]
    assert abs(a[1, 0] - 2.0 * ((0.01 / r) ** 12 - (0.01 / r) ** 4) / r) < 1e-9 * a[1, 0] and a[1, 0] > 0
    bf = sph.BoundaryForce(d=2.0, r0=0.01)
    assert abs(bf.accel(np.array([r, 0.0, 0.0]), np.array(r * r))[0] - a[1, 0]) < 1e-9 * a[1, 0]
