"""Per-step overhead of the X-slab machinery on one GPU: the same C3 system stepped by
DeviceSim (single domain) and by SlabSimulation with k virtual slabs (LoopbackComm)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import slab  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sc = sph.named_scenario(name)
prm = sph.make_params(sc)
system = sph.build_dam_break(sc, prm)
sim = DeviceSim(system, prm, reach=1)
for _ in range(3):
    sim.launch_step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(steps):
    sim.launch_step()
torch.cuda.synchronize()
single = (time.perf_counter() - t) / steps * 1e3
print(f"single-domain DeviceSim: {single:.2f} ms/step")
for k in (1, 2):
    s = slab.device_slab_simulation(system, prm, k)
    for _ in range(3):
        s.step()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        s.step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / steps * 1e3
    print(f"slabs={k} (loopback, one GPU): {ms:.2f} ms/step  overhead vs single {ms - single:.2f} ms")
