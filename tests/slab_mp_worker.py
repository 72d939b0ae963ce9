"""Worker of test_device_slabs_two_processes: one rank of dslab.DeviceSlabSim over
torch.distributed (gloo: the processes share the box's one GPU), launched by torchrun.

  python -m torch.distributed.run --nproc-per-node 2 ... tests/slab_mp_worker.py OUT.npz STEPS [copy|peer]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import dslab  # noqa: E402

out, steps = sys.argv[1], int(sys.argv[2])
transport = sys.argv[3] if len(sys.argv) > 3 else "copy"
dist.init_process_group("gloo")
torch.cuda.set_device(0)
sc = sph.Scenario(dp=0.006)
prm = sph.make_params(sc)
system = sph.build_dam_break(sc, prm)
# "copy": bands staged through gloo; "peer": written into the neighbour's memory (CUDA IPC)
comm = dslab.DevPeerComm(cap_rows=256) if transport == "peer" else dslab.DevDistComm()
sim = dslab.DeviceSlabSim(system, prm, comm, precision=1)
sim.run(steps)
torch.cuda.synchronize()
mine = sim.gather_host()
parts = [None] * dist.get_world_size()
dist.gather_object(mine, parts if dist.get_rank() == 0 else None, dst=0)
recs = sim.records(0, steps)  # collective: the counters are summed over the ranks here
if dist.get_rank() == 0:
    pos, vel, rho, ids, fl = (np.concatenate([p[k] for p in parts]) for k in range(5))
    o = np.argsort(ids)
    np.savez(out, pos=pos[o], vel=vel[o], rho=rho[o], id=ids[o], fl=fl[o], dt=recs["dt"],
             cand=recs["candidate_pairs"], hits=recs["hits_ordered"], evals=recs["force_evals"],
             ff=recs["ff_force_evals"], bounds=np.array(sim.bounds))
if transport == "peer":
    comm.close()
dist.barrier()
dist.destroy_process_group()
