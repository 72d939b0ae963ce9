"""C3 dam break over a long run on one GPU: how the step cost evolves as the column collapses
(cells fill unevenly, more rows change cell per step), with the energy diagnostics.

  python tools/dam_break_long.py [c3] [out.json] [steps] [every] [128|384|auto|tuned] [n_subdiv]

("tuned": run_simulation(pi_kernel="tuned")'s policy -- at every window start one step of each
of DeviceSim.pi_candidates, the faster build runs the window.)

Per window of ``every`` steps: mean ms/step and NL / PI / SU stage means (CUDA events), the
movers-only sort's mover count and path on the window's last step, t_sim, KE/PE/IE.
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
out = sys.argv[2] if len(sys.argv) > 2 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
every = int(sys.argv[4]) if len(sys.argv) > 4 else 500
blocking = sys.argv[5] if len(sys.argv) > 5 else "auto"
n_subdiv = int(sys.argv[6]) if len(sys.argv) > 6 else 1
t0 = time.time()
sc = sph.named_scenario(name)
prm = sph.make_params(sc, n_subdiv=n_subdiv)
system = sph.build_dam_break(sc, prm)
sim = DeviceSim(system, prm, reach=n_subdiv, record_capacity=steps + 8)
if blocking in ("auto", "tuned"):
    sim.set_pi_block(sph.sim.initial_pi_block(sim.n, prm.n_subdiv))
else:
    sim.set_pi_block(int(blocking))
n = sim.n
rows = []
e0 = sim.energy()
done = 0
while done < steps:
    if blocking == "tuned" and steps - done > every:
        sim.tune_pi(sim.pi_candidates(prm.n_subdiv))  # (ordinary steps of the run)
        done += 2
    k = min(every, steps - done)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(sim.n_stage_events())] for _ in range(k)]
    for i in range(k):
        sim.launch_step(evs[i])
    torch.cuda.synchronize()
    st = np.array([DeviceSim.stage_seconds(e) for e in evs]) * 1e3  # nl, pi, su, wall [ms]
    done += k
    err = sim.error()
    if err is not None:
        raise SystemExit(f"diverged at step {done}: {err}")
    movers, mode = sim.ws.sort_info()
    c = sim.ctrl_host()
    e = sim.energy()
    nblk = int(c["nblk"][0])
    lane = sim.pi_lane_use(c)
    block_now = f"{sim.pi_kernel}/{sim.pi_block}"
    rows.append(dict(step=done, t_sim=float(c["t_sim"]), ms_per_step=float(st[:, 3].mean()),
                     pi_block=block_now, pi_blocks=nblk, lane_use=lane,
                     nl_ms=float(st[:, 0].mean()), pi_ms=float(st[:, 1].mean()),
                     su_ms=float(st[:, 2].mean()),
                     particle_steps_per_s=n / (float(st[:, 3].mean()) * 1e-3),
                     movers_last_step=movers, sort_path="movers" if mode == 0 else "radix", **e))
    print(json.dumps(rows[-1]), flush=True)
recs = sim.records(0, steps)
summary = dict(config=name, blocking=blocking, particles=n, steps=steps, wall_s=time.time() - t0, energy0=e0,
               mean_particle_steps_per_s=n / (np.mean([r["ms_per_step"] for r in rows]) * 1e-3),
               true_pairs_first=int(recs["hits_ordered"][0]) // 2,
               true_pairs_last=int(recs["hits_ordered"][-1]) // 2, windows=rows)
if out:
    json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "windows"}))
