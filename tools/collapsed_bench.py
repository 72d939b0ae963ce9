"""C3 after K steps (collapsed column): mean ms/step and PI ms over M more steps, for A/B of
the interaction builds.  python tools/collapsed_bench.py [K] [M] [128|384]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 200
block = int(sys.argv[3]) if len(sys.argv) > 3 else 384
sc = sph.named_scenario("c3")
prm = sph.make_params(sc)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, record_capacity=K + M + 8)
sim.set_pi_block(block)
for _ in range(K):
    sim.launch_step()
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(M)]
for e in evs:
    sim.launch_step(e)
torch.cuda.synchronize()
st = np.array([DeviceSim.stage_seconds(e) for e in evs]) * 1e3
print(f"block {block} after {K} steps: ms/step {st[:, 3].mean():.3f} pi {st[:, 1].mean():.3f} "
      f"lane {sim.pi_lane_use():.3f}")
