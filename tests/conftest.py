import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def gold():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = golden(name)
        return cache[name]
    return get


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def scenario_from_npz(z):
    """Rebuild the Scenario a trajectory fixture was generated from (make_golden.py)."""
    from paper_1110_3711_b200 import Scenario
    s = np.asarray(z["scenario"], np.float64)
    return Scenario(tank_min=s[0:3], tank_size=s[3:6], fill_offset=s[6:9], fill_size=s[9:12],
                    dp=float(s[12]), hydrostatic=bool(s[13]))


def initial_state(z):
    """(pos, vel, rho, id, nb, mass_fluid, mass_boundary) of build_dam_break for a fixture."""
    import oracle
    from paper_1110_3711_b200 import build_dam_break
    prm = oracle.params_from_npz(z)
    s = build_dam_break(scenario_from_npz(z), prm)
    return s.pos, s.vel, s.rho, s.id, s.count_boundary, s.mass_fluid, s.mass_boundary
