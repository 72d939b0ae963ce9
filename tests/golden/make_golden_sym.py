"""Golden fixtures for the reference's cell-pair engines (symmetric pair evaluation), made by
running the UNMODIFIED reference (sphbench, /root/reference/pkg/src) on the sorted frames
already committed by make_golden.py.

Run:  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
      python tests/golden/make_golden_sym.py

For each frame_<name>.npz it writes sym_<name>.npz with ForceOutputs of
  * ``sym1``   EngineConfig(symmetry=True)                          -- run_cells_symmetric,
               single thread (kernels.py:121-175 + eval_scatter 29-68, cellpairs.py:59-69)
  * ``symT``   EngineConfig(symmetry=True, threading="symmetric", thread_count=4,
               block_of_cells=10) -- private accumulators merged in thread order
               (cellpairs.py:132-164, balance.py:12-43)
  * ``asym1``  EngineConfig(symmetry=False)                         -- run_cells_asymmetric
(accel, drho, visc, counters), the references for oracle.symmetric and the device K5s.
"""
from __future__ import annotations

import os
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from sphbench import EngineConfig  # noqa: E402
from sphbench.engines import make_engine  # noqa: E402
from sphbench.grid import CellBeginEnd, CellIndex  # noqa: E402
from sphbench.model import DerivedQuantities, ParticleSystem, SimParams  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FRAMES = ["small_n1", "small_n2", "mid5k_n1", "mid5k_n2", "uniform3k_n1", "c1mid_n1"]
CONFIGS = {
    "sym1": EngineConfig(symmetry=True),
    "symT": EngineConfig(symmetry=True, threading="symmetric", thread_count=4, block_of_cells=10),
    "asym1": EngineConfig(symmetry=False),
}


def load(name):
    z = np.load(os.path.join(OUT, f"frame_{name}.npz"))
    p = SimParams(h=float(z["p_h"]), dp=float(z["p_dp"]), rho0=float(z["p_rho0"]),
                  c0=float(z["p_c0"]), gamma=float(z["p_gamma"]), alpha=float(z["p_alpha"]),
                  g=np.asarray(z["p_g"]), cfl=float(z["p_cfl"]),
                  domain_min=np.asarray(z["p_domain_min"]), domain_max=np.asarray(z["p_domain_max"]),
                  n_subdiv=int(z["p_n_subdiv"]),
                  verlet_corrector_stride=int(z["p_verlet_corrector_stride"]),
                  dt_min=float(z["p_dt_min"]), dt_max=float(z["p_dt_max"]))
    s = ParticleSystem(count_fluid=int(z["s_nf"]), count_boundary=int(z["s_nb"]), pos=z["s_pos"],
                       vel=z["s_vel"], rho=z["s_rho"], mass_fluid=float(z["s_mass_fluid"]),
                       mass_boundary=float(z["s_mass_boundary"]), ptype=z["s_ptype"], id=z["s_id"])
    d = DerivedQuantities(press=z["press"], csound=z["csound"], prrho=z["prrho"], tensil=z["tensil"])
    dims = tuple(int(v) for v in z["dims"])
    grid = types.SimpleNamespace(cell_of=z["cell_of"], dims=dims, ncells=int(np.prod(dims)))
    cidx = CellIndex(fluid=CellBeginEnd(begin=z["fbeg"], end=z["fend"]),
                     boundary=CellBeginEnd(begin=z["bbeg"], end=z["bend"]))
    return s, d, grid, cidx, p


def main():
    for name in FRAMES:
        s, d, grid, cidx, p = load(name)
        out = {}
        for tag, cfg in CONFIGS.items():
            f = make_engine(cfg).compute(s, d, grid, cidx, p)
            st = f.stats
            out[f"{tag}_accel"], out[f"{tag}_drho"], out[f"{tag}_visc"] = f.accel, f.drho_dt, f.visc_dt
            out[f"{tag}_counters"] = np.array([st.candidate_pairs, st.true_pairs, st.force_evals,
                                               st.ff_force_evals], np.int64)
            out[f"{tag}_tag"] = np.array(st.engine_tag)
        path = os.path.join(OUT, f"sym_{name}.npz")
        np.savez_compressed(path, **out)
        print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    main()
