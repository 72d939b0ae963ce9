"""C5 (BASELINE.json config 5): piston wave tank, 1000 steps, energy / mass drift from the
device diagnostics (sphb_energy), on one GPU.  Writes a JSON summary (argv[2]).

  python tools/wave_tank_drift.py [c5|c5_small] [out.json] [steps] [every] [128|384|auto]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
out = sys.argv[2] if len(sys.argv) > 2 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
every = int(sys.argv[4]) if len(sys.argv) > 4 else 50
blocking = sys.argv[5] if len(sys.argv) > 5 else "auto"
t0 = time.time()
sc = sph.named_scenario(name)
prm = sph.make_wave_tank_params(sc)
system = sph.build_wave_tank(sc, prm)
t_build = time.time() - t0
sim = DeviceSim(system, prm, reach=1, record_capacity=steps + 8)
if blocking == "auto":
    sim.set_pi_block(sph.sim.initial_pi_block(sim.n, prm.n_subdiv))
if blocking != "auto":
    sim.set_pi_block(int(blocking))
rows = []
e = sim.energy()
rows.append(dict(step=0, t=0.0, **e))
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
gpu_ms = 0.0
done = 0
while done < steps:
    k = min(every, steps - done)
    ev0.record()
    for _ in range(k):
        sim.launch_step()
    ev1.record()
    torch.cuda.synchronize()
    gpu_ms += ev0.elapsed_time(ev1)
    done += k
    c = sim.ctrl_host()
    err = sim.error()
    if err is not None:
        raise SystemExit(f"diverged: {err}")
    rows.append(dict(step=done, t=float(c["t_sim"]), **sim.energy()))
recs = sim.records(0, steps)
pm = prm.piston
e0 = rows[0]
emech0 = e0["pe"] + e0["ie"]
final = rows[-1]
summary = dict(
    config=name, particles=system.n, fluid=system.count_fluid, boundary=system.count_boundary,
    piston_particles=pm.id1 - pm.id0, piston=dict(stroke=pm.stroke, period=pm.period),
    steps=steps, blocking=blocking, pi_block_final=sim.pi_block, t_end=final["t"], host_build_s=t_build, gpu_ms_per_step=gpu_ms / steps,
    particle_steps_per_s=system.n * steps / (gpu_ms * 1e-3),
    mean_true_pairs=float(np.mean(recs["hits_ordered"])) / 2,
    energy0=e0, energy_final=final,
    rel_energy_change=(final["ke"] + final["pe"] + final["ie"] - e0["ke"] - e0["pe"] - e0["ie"]) / emech0,
    mean_fluid_rho_drift=(final["rho_fluid"] - e0["rho_fluid"]) / prm.rho0,
    piston_x_final=float(pm.x(final["t"])), series=rows,
    note="FP32, verlet, 1 GPU; energy = KE + PE + Tait IE (device f64 reduction); the piston "
         "injects work, so E is not conserved -- the series shows the injected energy and the "
         "density drift; particle count is exact by construction")
print(json.dumps({k: v for k, v in summary.items() if k != "series"}, indent=1))
if out:
    json.dump(summary, open(out, "w"), indent=1)
