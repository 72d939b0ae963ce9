"""Where the eager step loses time vs graph replay at C3: 30 steps timed eagerly with and without
the per-stage events (and with each single event), and as one CUDA graph (the paired kernel)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import _lib  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim, _ptr, _stream  # noqa: E402

sc = sph.named_scenario("c3")
prm = sph.make_params(sc)
system = sph.build_dam_break(sc, prm)
sim = DeviceSim(system, prm, reach=1)
sim.select_pi("paired", 512)
N = 30
Ev = lambda t=True: torch.cuda.Event(enable_timing=t)  # noqa: E731


def timed(fn):
    torch.cuda.synchronize()
    a, b = Ev(), Ev()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / N


class Rec:
    """An events list that records only the listed positions."""
    def __init__(self, keep, timing=True):
        self.e = [Ev(timing) for _ in range(4)]
        self.keep = keep

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(4))]
        ev, keep = self.e[k], k in self.keep

        class R:
            def record(self):
                if keep:
                    ev.record()
        return R()

    def __len__(self):
        return 4


for _ in range(3):
    sim.launch_step()
for label, keep, timing in (("all 4 events", {0, 1, 2, 3}, True), ("none", set(), True),
                            ("start only", {0}, True), ("after NL", {1}, True),
                            ("after PI", {2}, True), ("after SU", {3}, True),
                            ("all 4, no timing", {0, 1, 2, 3}, False), ("all 4 events", {0, 1, 2, 3}, True)):
    evs = [Rec(keep, timing) for _ in range(N)]
    print("eager, %-18s %.3f ms/step" % (label, timed(lambda: [sim.launch_step(events=e) for e in evs])),
          flush=True)
sim.capture(N)
print("graph replay               %.3f ms/step" % timed(sim.run_graph))
