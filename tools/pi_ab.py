"""PI ms of several interaction builds on the same advancing C3 run: at rest (step 5) and after K
steps (collapsed column), at n_subdiv N.
  python tools/pi_ab.py N K M build[,build...]     build = kernel/block, e.g. gather/384,paired/512"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

N, K, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
builds = [(b.split("/")[0], int(b.split("/")[1])) for b in sys.argv[4].split(",")]
sc = sph.named_scenario("c3")
prm = sph.make_params(sc, n_subdiv=N)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=N, record_capacity=K + 40 * M + 64)
sim.set_pi_block(384)


def measure(tag):
    for rep in range(2):
        for kern, blk in builds:
            sim.select_pi(kern, blk)
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(M)]
            for e in evs:
                sim.launch_step(e)
            torch.cuda.synchronize()
            st = np.array([DeviceSim.stage_seconds(e) for e in evs]) * 1e3
            if rep:
                print(f"n{N} {tag} {kern}/{blk}: pi {st[:, 1].mean():.3f} ms lane {sim.pi_lane_use():.3f}",
                      flush=True)


for _ in range(5):
    sim.launch_step()
measure("rest")
for _ in range(K):
    sim.launch_step()
torch.cuda.synchronize()
measure(f"step{K}")
