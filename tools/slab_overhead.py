"""Per-step overhead of the X-slab machinery on one GPU: the same system stepped by DeviceSim
(single domain), by the torch SlabSimulation (tests/, --legacy) and by the device-resident DeviceSlabSim with k
virtual slabs (loopback comms)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import dslab  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
legacy = "--legacy" in sys.argv
sc = sph.named_scenario(name)
prm = sph.make_params(sc)
system = sph.build_dam_break(sc, prm)


def timed(stepper):
    for _ in range(3):
        stepper()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        stepper()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e3


sim = DeviceSim(system, prm, reach=1)
single = timed(sim.launch_step)
print(f"single-domain DeviceSim: {single:.2f} ms/step")
del sim
for k in (1, 2, 4):
    d = dslab.DeviceSlabSim(system, prm, dslab.DevLoopbackComm(k))
    ms = timed(d.step)
    print(f"DeviceSlabSim slabs={k} (loopback, one GPU): {ms:.2f} ms/step, vs single +{ms - single:.2f} ms")
    del d
    torch.cuda.empty_cache()
if legacy:  # the torch restatement (test infrastructure)
    sys.path.insert(0, "tests")
    import slab_torch_reference as tslab  # noqa: E402
    s = tslab.device_slab_simulation(system, prm, 1)
    ms = timed(s.step)
    print(f"torch SlabSimulation slabs=1: {ms:.2f} ms/step, vs single +{ms - single:.2f} ms")
