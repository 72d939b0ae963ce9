"""Run C3 for K steps (the column collapses), then one profiled step (for ncu
--profile-from-start off):  python tools/collapsed_profile.py [steps] [128|384]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
block = int(sys.argv[2]) if len(sys.argv) > 2 else 128
sc = sph.named_scenario("c3")
prm = sph.make_params(sc)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, record_capacity=steps + 8)
sim.set_pi_block(block)
for _ in range(steps):
    sim.launch_step()
torch.cuda.synchronize()
print("lane use", sim.pi_lane_use(), "t_sim", float(sim.ctrl_host()["t_sim"]), flush=True)
torch.cuda.profiler.start()
sim.launch_step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
