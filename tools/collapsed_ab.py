"""C3 after K steps (collapsed column): PI ms of each interaction build over M steps each, on the
same advancing run.  python tools/collapsed_ab.py [K] [M]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sc = sph.named_scenario("c3")
prm = sph.make_params(sc)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, record_capacity=K + 16 * M + 8)
sim.set_pi_block(384)
for _ in range(K):
    sim.launch_step()
torch.cuda.synchronize()
for rep in range(2):
    for kern, blk in (("gather", 256), ("gather", 384), ("gather", 512), ("paired", 512)):
        sim.select_pi(kern, blk)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(M)]
        for e in evs:
            sim.launch_step(e)
        torch.cuda.synchronize()
        st = np.array([DeviceSim.stage_seconds(e) for e in evs]) * 1e3
        print(f"after {K} steps {kern}/{blk}: pi {st[:, 1].mean():.3f} ms lane {sim.pi_lane_use():.3f}",
              flush=True)
