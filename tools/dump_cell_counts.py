import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph
from paper_1110_3711_b200.device import DeviceSim
sc = sph.named_scenario("c3"); prm = sph.make_params(sc)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, record_capacity=7000)
for _ in range(6000):
    sim.launch_step()
torch.cuda.synchronize()
b = sim.beg.cpu().numpy().astype(np.int64); e = sim.end.cpu().numpy().astype(np.int64)
cnt = (e - b).astype(np.int16)
np.savez_compressed(sys.argv[1], cnt=cnt, dims=np.array(sim.grid.dims[:3]))
print("saved", cnt.shape, cnt.max())
