"""Timeline of bench.py's e2e loop (C3, host round trip of the reference-layout state every
step): per steady-state step, when the H2D chunks land, the conversions and the step end, and
when the D2H chunks land, relative to the step's first H2D chunk.
  python tools/e2e_timeline.py [steps] [chunks]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1110_3711_b200 as sph  # noqa: E402
from paper_1110_3711_b200 import _lib  # noqa: E402
from paper_1110_3711_b200.device import DeviceSim  # noqa: E402

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 8
NCH = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sc = sph.named_scenario("c3")
prm = sph.make_params(sc)
sim = DeviceSim(sph.build_dam_break(sc, prm), prm, reach=1, record_capacity=4096)
sim.select_pi("paired", 512)
for _ in range(4):
    sim.launch_step()
torch.cuda.synchronize()

L = _lib.lib()
n = sim.n
names = ("pos", "vel", "rho", "vel_prev", "rho_prev")
width = {"pos": 3, "vel": 3, "rho": 1, "vel_prev": 3, "rho_prev": 1}
offs, off = {"id": 0}, 8 * n
for k in names:
    off = (off + 15) // 16 * 16
    offs[k] = off
    off += 4 * width[k] * n
nbytes = off
hbuf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
dbuf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dsoa = {"id": dbuf[:8 * n].view(torch.int64)}
for k in names:
    a = dbuf[offs[k]:offs[k] + 4 * width[k] * n].view(torch.float32)
    dsoa[k] = a.view(n, width[k]) if width[k] > 1 else a
ptr = lambda t: t.data_ptr()  # noqa: E731
cs = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def to_soa():
    _lib.check(L.sphb_state_to_soa(0, n, ptr(sim.posp), ptr(sim.velr), ptr(sim.prev),
                                   *[ptr(dsoa[k]) for k in names], cs()), "to_soa")
    dsoa["id"].copy_(sim.id[:n])


def from_soa():
    _lib.check(L.sphb_state_from_soa(0, n, *[ptr(dsoa[k]) for k in names], ptr(sim.posp),
                                     ptr(sim.velr), ptr(sim.prev), cs()), "from_soa")
    sim.id[:n].copy_(dsoa["id"])


to_soa()
hbuf.copy_(dbuf)
bounds = [(nbytes * c // NCH, nbytes * (c + 1) // NCH) for c in range(NCH)]
comp = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ev = [{"in": [E() for _ in bounds], "out": [E() for _ in bounds], "packed": E(),
       "conv": E(), "keys": E(), "step": E(), "st": [E() for _ in range(4)]} for _ in range(STEPS)]
t0 = E()
torch.cuda.synchronize()
t0.record()
s_in.wait_stream(comp)
with torch.cuda.stream(s_in):
    for c, (lo, hi) in enumerate(bounds):
        dbuf[lo:hi].copy_(hbuf[lo:hi], non_blocking=True)
        ev[0]["in"][c].record(s_in)
for k in range(STEPS):
    e = ev[k]
    comp.wait_event(e["in"][-1])
    from_soa()
    e["conv"].record(comp)
    sim.first_keys_resync(keep_order=True)
    e["keys"].record(comp)
    sim.launch_step(e["st"])
    e["step"].record(comp)
    to_soa()
    e["packed"].record(comp)
    with torch.cuda.stream(s_out):
        s_out.wait_event(e["packed"])
        for c, (lo, hi) in enumerate(bounds):
            hbuf[lo:hi].copy_(dbuf[lo:hi], non_blocking=True)
            e["out"][c].record(s_out)
    if k + 1 < STEPS:
        with torch.cuda.stream(s_in):
            for c, (lo, hi) in enumerate(bounds):
                s_in.wait_event(e["out"][c])
                dbuf[lo:hi].copy_(hbuf[lo:hi], non_blocking=True)
                ev[k + 1]["in"][c].record(s_in)
comp.wait_stream(s_out)
torch.cuda.synchronize()
T = lambda x: t0.elapsed_time(x)  # noqa: E731
rows = []
for k in range(1, STEPS - 1):
    e, nx = ev[k], ev[k + 1]
    base = T(e["in"][0])
    rows.append([T(e["in"][-1]) - base, T(e["conv"]) - base, T(e["keys"]) - base, T(e["step"]) - base,
                 T(e["packed"]) - base, T(e["out"][0]) - base, T(e["out"][-1]) - base,
                 T(nx["in"][0]) - base])
r = np.mean(rows, axis=0)
print(f"chunks {NCH}: per step (ms from the step's first H2D chunk landing): last H2D chunk {r[0]:.2f}, "
      f"converted {r[1]:.2f}, keys {r[2]:.2f}, step done {r[3]:.2f}, packed {r[4]:.2f}, "
      f"first D2H chunk {r[5]:.2f}, last D2H chunk {r[6]:.2f}, next step's first H2D chunk {r[7]:.2f}")
st = np.mean([DeviceSim.stage_seconds(ev[k]["st"]) for k in range(1, STEPS - 1)], axis=0) * 1e3
print(f"  stages NL {st[0]:.3f} PI {st[1]:.3f} SU {st[2]:.3f} ms")
print(f"  => e2e {n / (r[7] * 1e-3) / 1e6:.1f}M particle-steps/s; step alone {r[3] - r[2]:.2f} ms")
