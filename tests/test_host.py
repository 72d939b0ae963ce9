"""Host-side logic (no GPU): scenario builder, constants, config rules, and the C ABI
(library loads, exports every symbol include/sphb200.h declares, struct layouts match)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden
import paper_1110_3711_b200 as sph
from paper_1110_3711_b200 import _lib
from paper_1110_3711_b200.physics import grid_dims, pack_params


@pytest.mark.parametrize("name,dp", [("frame_small_n1.npz", 0.02), ("frame_c1_n1.npz", 0.006)])
def test_build_dam_break_bit_exact(name, dp):
    z = golden(name)
    sc = sph.Scenario(dp=dp)
    prm = sph.make_params(sc)
    s = sph.build_dam_break(sc, prm)
    assert s.count_boundary == int(z["in_nb"]) and s.count_fluid == int(z["in_nf"])
    for f in ("pos", "vel", "rho", "id", "ptype"):
        assert np.array_equal(getattr(s, f), z["in_" + f]), f
    assert s.mass_fluid == float(z["in_mass_fluid"])
    for k in ("h", "dp", "rho0", "c0", "gamma", "alpha", "cfl"):
        assert getattr(prm, k) == float(z["p_" + k])
    assert np.array_equal(prm.domain_min, z["p_domain_min"])
    assert np.array_equal(prm.domain_max, z["p_domain_max"])


def test_named_config_sizes():
    """particle counts of the named configurations."""
    want = {"c1": 22_399, "c2": 1_142_622, "c3": 10_200_478}
    for k, n in want.items():
        sc = sph.named_scenario(k)
        assert sc.fluid_count + sc.boundary_count == n


def test_pack_params_bit_exact():
    z = golden("eos.npz")
    prm = oracle.params_from_npz(z)
    assert np.array_equal(pack_params(prm, 1.0e-3, 2.0e-3), z["pp"])


@pytest.mark.parametrize("name", ["frame_small_n1.npz", "frame_small_n2.npz", "frame_c1_n1.npz"])
def test_grid_dims(name):
    z = golden(name)
    prm = oracle.params_from_npz(z)
    cs, dims = grid_dims(prm)
    assert cs == float(z["cell_size"]) and np.array_equal(dims, z["dims"])


def test_params_validate_messages():
    sc = sph.Scenario(dp=0.02)
    prm = sph.make_params(sc)
    from dataclasses import replace
    with pytest.raises(ValueError, match="cfl"):
        sph.validate(replace(prm, cfl=1.5))
    with pytest.raises(ValueError, match="dt bounds"):
        sph.validate(replace(prm, dt_min=1.0, dt_max=0.5))


# ------------------------------------------------------------- config (test_engines.py:19-46)
def test_config_rules_match_reference():
    with pytest.raises(ValueError, match="symmetry"):
        sph.EngineConfig(engine="gather", symmetry=True).validated()
    with pytest.raises(ValueError, match="requires symmetry"):
        sph.EngineConfig(symmetry=False, threading="symmetric").validated()
    assert sph.EngineConfig(symmetry=True, threading="asymmetric").validated().symmetry is False
    for bad in (dict(engine="cuda"), dict(lane_batch=2), dict(threading="farm"),
                dict(thread_count=0), dict(block_of_cells=0), dict(derived_mode="live"),
                dict(engine="gather", symmetry=False, gather_variant="fastcellsh"),
                dict(precision="fp16")):
        with pytest.raises(ValueError):
            sph.EngineConfig(**bad).validated()
    cfg = sph.EngineConfig(engine="gather", symmetry=False, gather_variant="slowcellsh")
    assert cfg.required_n_subdiv() == 1 and cfg.device_reach(1) == 1 and cfg.device_order() == 0
    cfg = sph.EngineConfig(engine="gather", symmetry=False, gather_variant="fastcellshalf")
    assert cfg.required_n_subdiv() == 2 and cfg.device_order() == 1
    assert sph.EngineConfig(engine="b200", symmetry=False).device_reach(2) == 2


def test_run_simulation_argument_checks_before_device():
    sc = sph.Scenario(dp=0.025)
    prm = sph.make_params(sc, n_subdiv=1)
    with pytest.raises(ValueError, match="max_steps or t_end"):
        sph.run_simulation(sc, prm, sph.EngineConfig())
    with pytest.raises(ValueError, match="n_subdiv"):
        sph.run_simulation(sc, prm, sph.EngineConfig(engine="gather", symmetry=False), max_steps=1)


# ------------------------------------------------------------- C ABI
HEADER = os.path.join(ROOT, "include", "sphb200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sphb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.sphb_version().decode().startswith("sphb200")


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout and "sm_90" not in out.stdout


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sphb200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sphb_grid_t),'
                   ' sizeof(sphb_params_t), sizeof(sphb_ctrl_t), sizeof(sphb_step_record_t),'
                   ' sizeof(sphb_state_t), offsetof(sphb_ctrl_t, err), offsetof(sphb_ctrl_t, active));}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.GridDesc), ctypes.sizeof(_lib.ParamsDesc), None,
            _lib.REC_DTYPE.itemsize, ctypes.sizeof(_lib.StateDesc),
            _lib.CTRL_DTYPE.fields["err"][1], _lib.CTRL_DTYPE.fields["active"][1]]
    assert got[0] == want[0] and got[1] == want[1] and got[3] == want[3] and got[4] == want[4]
    assert got[2] <= _lib.CTRL_BYTES and got[2] == _lib.CTRL_DTYPE.itemsize
    assert got[5] == want[5] and got[6] == want[6]


def test_abi_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call, so it is testable on CPU."""
    L = _lib.lib()
    g = _lib.GridDesc()
    g.cell_size = 1.0
    g.dims[0] = g.dims[1] = g.dims[2] = 0  # invalid
    rc = L.sphb_sort(None, ctypes.byref(g), None, 0, None, None, None, None)
    assert rc == _lib.SPHB_E_INVALID
    assert b"null" in L.sphb_last_error() or b"dims" in L.sphb_last_error()
    rc = L.sphb_interact(None, None, None, 0, 0, None, None, None, None, None, None, None, None,
                         None, None, None)
    assert rc == _lib.SPHB_E_INVALID


def test_auto_interaction_blocking_policy():
    """sim.initial_pi_block: 384-target blocks once there are >= 4 per SM, 256 below (the
    blockings' parity: test_pi_block_matches_128 on the GPU)."""
    from paper_1110_3711_b200 import sim as S
    assert S.PI_LARGE_MIN_TARGETS == 4 * 148 * 384
    assert S.initial_pi_block(25_000) == 256            # C1: ~65 large blocks for 148 SMs
    assert S.initial_pi_block(1_180_000) == 384         # C2
    assert S.initial_pi_block(10_200_478) == 384        # C3
    assert S.initial_pi_block(S.PI_LARGE_MIN_TARGETS) == 384
    assert S.initial_pi_block(S.PI_LARGE_MIN_TARGETS - 1) == 256
    assert S.initial_pi_block(10_200_478, n_subdiv=2) == 384  # h/2 cells: 2x2-row bricks
