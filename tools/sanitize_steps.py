"""A few steps of a small dam break through every kernel family, for compute-sanitizer:
FP32 (pi128, pi256 and pi384 interaction builds -- the last with the hybrid brick / row
blocking --, the candidate counter, movers-only + radix sorts, the upload resync, symplectic,
wall force, energy, SoA state conversion) and FP64.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_steps.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import _lib  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

sc = sph.Scenario(dp=0.02)
prm = sph.make_params(sc, boundary_force=sph.BoundaryForce(d=5.0 * 9.81 * sc.fill_height, r0=sc.dp))
system = sph.build_dam_break(sc, prm)
for precision, block, integ in ((0, 128, "verlet"), (0, 256, "verlet"), (0, 384, "verlet"), (1, 128, "verlet"),
                                (0, 128, "symplectic"), (0, "paired", "verlet"), (0, "symmetric", "verlet")):
    p = sph.make_params(sc, integrator=integ,
                        boundary_force=sph.BoundaryForce(d=5.0 * 9.81 * sc.fill_height, r0=sc.dp))
    sim = DeviceSim(system, p, reach=1, precision=precision)
    if isinstance(block, str):
        sim.set_pi_kernel(block)
    else:
        sim.set_pi_block(block)
    for _ in range(4):
        sim.launch_step()
    sim.energy()
    n = sim.n
    soa = [torch.empty((n, 3), device="cuda"), torch.empty((n, 3), device="cuda"),
           torch.empty(n, device="cuda"), torch.empty((n, 3), device="cuda"), torch.empty(n, device="cuda")]
    L, s = _lib.lib(), torch.cuda.current_stream().cuda_stream
    _lib.check(L.sphb_state_to_soa(0, n, sim.posp.data_ptr(), sim.velr.data_ptr(), sim.prev.data_ptr(),
                                   *[t.data_ptr() for t in soa], s), "to_soa")
    _lib.check(L.sphb_state_from_soa(0, n, *[t.data_ptr() for t in soa], sim.posp.data_ptr(),
                                     sim.velr.data_ptr(), sim.prev.data_ptr(), s), "from_soa")
    sim.first_keys_resync(keep_order=True)  # the upload path (clear_hist / trust_order)
    sim.launch_step()
    torch.cuda.synchronize()
    assert sim.error() is None, sim.error()
    print("ok", precision, block, integ, sim.ws.sort_info(), flush=True)

# the X-slab exchange kernels (slab.cu) through two virtual ranks on this GPU
from paper_1110_3711_b200 import dslab  # noqa: E402

# (the slab stepper has no wall-force extension), edge bands + dead-bin sort, then a re-settle
ds = dslab.DeviceSlabSim(system, sph.make_params(sc), dslab.DevLoopbackComm(2), precision=0)
for _ in range(4):
    ds.step()
ds.rebalance(times=[1.0, 3.0])
for _ in range(2):
    ds.step()
ds.check()
torch.cuda.synchronize()
print("ok slabs", ds.bounds, flush=True)

# the module-level step functions (stepfn.cu, grid.py)
import types  # noqa: E402

import numpy as np  # noqa: E402

s2 = sph.build_dam_break(sc, prm)
g2 = sph.grid.assign_cells(s2.pos, prm)
s2, _ = sph.grid.reorder(s2, g2)
ci = sph.grid.build_cell_index(s2, g2)
sph.grid.build_dual_ranges(ci, g2.dims, 1)
f2 = types.SimpleNamespace(accel=np.zeros((s2.n, 3)), drho_dt=np.zeros(s2.n), visc_dt=np.zeros(s2.n))
dt2 = sph.compute_dt(f2, s2, sph.compute_derived(s2.rho, prm), prm)
sph.verlet_update(sph.VerletState.from_system(s2, 40), s2, f2, prm, dt2)
torch.cuda.synchronize()
print("ok step functions", flush=True)
