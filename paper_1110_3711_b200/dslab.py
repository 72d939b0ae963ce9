"""Device-resident X-slab decomposition: the production multi-GPU stepper.

Same decomposition as ``slab.SlabSimulation`` (whose torch implementation is kept as the
host-logic restatement the CPU / gloo tests run), but the state never leaves the engine's SoA
arrays: per step and per rank

  1. NL of the assembled arrays (owned rows + halo rows with id < 0) on the sort keys that
     travelled with the rows (K7 wrote them; K1 only on upload), interaction of the owned
     target columns [x0, x1) only;
  2. device all-reduces of the two dt minima (MIN) and the four counters (SUM);
  3. K7 into the primary arrays (sphb_integrate);
  4. ``sphb_slab_count``: per-category tile counts + totals on the device;
  5. ONE host synchronisation: an all-gather of every rank's 10 totals and error word;
  6. ``sphb_slab_scatter``: kept rows straight into the next step's arrays, migrants and halo
     copies into one packed buffer per neighbour;
  7. NCCL send/recv of exact byte counts, ``sphb_slab_unpack`` into the next arrays.

The next step's layout per rank is [boundary: kept | migrants from left | from right | halo
from left | from right][fluid: same]; the K2 sort regroups by cell anyway.  Comms:
``DevLoopbackComm`` (k virtual ranks on one GPU, device copies) and ``DevDistComm``
(torch.distributed / NCCL, one rank per process).
"""
from __future__ import annotations

import collections
import ctypes
import math

import numpy as np
import torch

from . import _lib
from .device import Workspace, _ptr, _stream, decode_err, new_ctrl, read_ctrl
from .physics import grid_desc, grid_dims, params_desc
from .slab import balanced_bounds, columns_of, enforce_min_width, rebalance_slices

ROW_WORDS = 16  # packed exchange row: 64 B (posp, velr, prev float4, int64 id, u32 key, pad)
NCAT = 10
KEEP_B, KEEP_F, MIGL_B, MIGL_F, MIGR_B, MIGR_F, HALOL_B, HALOL_F, HALOR_B, HALOR_F = range(10)


# ------------------------------------------------------------------ comms
class DevLoopbackComm:
    """k virtual ranks in one process on one device."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.local_ranks = list(range(nranks))

    def allreduce(self, tensors, op: str):
        red = {"min": lambda t: t.min(0).values, "max": lambda t: t.max(0).values,
               "sum": lambda t: t.sum(0)}[op](torch.stack(tensors))
        for t in tensors:
            t.copy_(red)

    def allgather(self, tensors):
        g = torch.stack(tensors)
        return [g for _ in tensors]

    def sendrecv(self, items):
        """items[r] = dict(send_l=(buf, rows), send_r=(...), recv_l=(buf, rows), recv_r=(...))"""
        n = self.nranks
        for r in range(n):
            if r > 0:
                buf, rows = items[r]["recv_l"]
                src, srows = items[r - 1]["send_r"]
                assert rows == srows
                if rows:
                    buf[:rows].copy_(src[:rows])
            if r < n - 1:
                buf, rows = items[r]["recv_r"]
                src, srows = items[r + 1]["send_l"]
                assert rows == srows
                if rows:
                    buf[:rows].copy_(src[:rows])


class DevDistComm:
    """One rank per process over torch.distributed.  NCCL (the production transport) moves the
    device buffers directly; over gloo (several processes sharing one GPU, the multi-process
    test on a single-GPU box) the same calls stage through host memory."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self.local_ranks = [self.rank]
        self.host = dist.get_backend() != "nccl"

    def allreduce(self, tensors, op: str):
        d = self.dist
        rop = {"min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX, "sum": d.ReduceOp.SUM}[op]
        t = tensors[0]
        if self.host:
            h = t.cpu()
            d.all_reduce(h, op=rop)
            t.copy_(h)
        else:
            d.all_reduce(t, op=rop)

    def allgather(self, tensors):
        t = tensors[0].contiguous()
        if self.host:
            h = t.cpu()
            parts = [torch.empty_like(h) for _ in range(self.nranks)]
            self.dist.all_gather(parts, h)
            return [torch.stack(parts).to(t.device)]
        out = torch.empty((self.nranks,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t)
        return [out]

    def sendrecv(self, items):
        d, r, n = self.dist, self.rank, self.nranks
        it = items[0]
        ops, landing = [], []
        for side, peer, ok in (("l", r - 1, r > 0), ("r", r + 1, r < n - 1)):
            if not ok:
                continue
            buf, rows = it["send_" + side]
            if rows:
                src = buf[:rows].cpu() if self.host else buf[:rows]
                ops.append(d.P2POp(d.isend, src, peer))
            buf, rows = it["recv_" + side]
            if rows:
                if self.host:
                    tmp = torch.empty(buf[:rows].shape, dtype=buf.dtype)
                    landing.append((buf, rows, tmp))
                    ops.append(d.P2POp(d.irecv, tmp, peer))
                else:
                    ops.append(d.P2POp(d.irecv, buf[:rows], peer))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        for buf, rows, tmp in landing:
            buf[:rows].copy_(tmp)


# ------------------------------------------------------------------ one rank
class _Arrays:
    def __init__(self, cap, dev):
        self.posp = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.velr = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.prev = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.id = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.key = torch.zeros(cap, dtype=torch.int32, device=dev)  # K7's sort key, carried


class DevRank:
    """A slab's arrays and engine scratch on one device."""

    def __init__(self, rank, bounds, params, prm, reach, dev, n_hint):
        self.rank = rank
        self.bounds = (int(bounds[0]), int(bounds[1]))
        self.params, self.prm, self.reach, self.dev = params, prm, int(reach), dev
        self.grid = grid_desc(params, reach, target_cols=self.bounds)
        _, dims = grid_dims(params)
        self.ncells = int(np.prod(dims))
        self.ctrl = new_ctrl(dev)
        self.rec_cap = 4096
        self.rec = torch.zeros(self.rec_cap * _lib.REC_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.totals = torch.zeros(NCAT, dtype=torch.int32, device=dev)
        self.send = [torch.zeros((1, ROW_WORDS), dtype=torch.float32, device=dev) for _ in range(2)]
        self.recv = [torch.zeros((1, ROW_WORDS), dtype=torch.float32, device=dev) for _ in range(2)]
        self.n = self.nb = 0
        self.cap = self.cap_ab = 0
        # (start, end) of the recent interaction launches (since the last rebalance, at most 64)
        self.pi_events = collections.deque(maxlen=64)
        self._grow(n_hint)

    def _grow(self, n):
        """Capacity of the state arrays (a: current, b: next) and the engine scratch."""
        if n > self.cap_ab:
            cap = int(n * 1.2) + 4096
            old_a, old_b = getattr(self, "a", None), getattr(self, "b", None)
            self.a, self.b = _Arrays(cap, self.dev), _Arrays(cap, self.dev)
            for old, new in ((old_a, self.a), (old_b, self.b)):
                if old is not None and self.n:  # keep the current rows (a) during an exchange
                    for f in ("posp", "velr", "prev", "id", "key"):
                        getattr(new, f)[: self.n].copy_(getattr(old, f)[: self.n])
            self.cap_ab = cap
        self._ensure_engine(n)

    def _ensure_engine(self, n):
        """Engine scratch for n rows (keys / tiles are rebuilt by K1 + count every step, except
        between sphb_slab_count and the scatter: keep them when growing then)."""
        if n <= self.cap:
            return
        cap = int(n * 1.2) + 4096
        dev = self.dev
        f4 = lambda: torch.zeros((cap, 4), dtype=torch.float32, device=dev)  # noqa: E731
        i32 = lambda m: torch.zeros(m, dtype=torch.int32, device=dev)  # noqa: E731
        old_keys, old_tiles = getattr(self, "keys", None), getattr(self, "tiles", None)
        self.posp_s, self.velr_s, self.prev_s, self.aux = f4(), f4(), f4(), f4()
        self.id_s = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.keys, self.keys_sorted, self.perm, self.cell_s = i32(cap), i32(cap), i32(cap), i32(cap)
        self.beg, self.end = i32(2 * self.ncells), i32(2 * self.ncells)
        self.acc = torch.zeros((cap, 3), dtype=torch.float64, device=dev)
        self.drho = torch.zeros(cap, dtype=torch.float64, device=dev)
        self.visc = torch.zeros(cap, dtype=torch.float64, device=dev)
        self.tiles = torch.zeros(NCAT * int(_lib.lib().sphb_slab_tiles(cap)) + NCAT,
                                 dtype=torch.int32, device=dev)
        if old_keys is not None:
            self.keys[: old_keys.shape[0]].copy_(old_keys)
            self.tiles[: old_tiles.shape[0]].copy_(old_tiles)
        self.ws = Workspace(cap, self.ncells)
        if getattr(self, "pi_block", None):  # a regrown workspace keeps the chosen blocking
            self.ws.set_pi_block(self.pi_block)
        self.cap = cap

    def _buf(self, which, side, rows):
        lst = self.send if which == "send" else self.recv
        if lst[side].shape[0] < rows:
            lst[side] = torch.zeros((int(rows * 1.3) + 1024, ROW_WORDS), dtype=torch.float32,
                                    device=self.dev)
        return lst[side]

    # -------------------------------------------------------------- upload
    def upload(self, pos, vel, rho, ids, nb):
        n = int(pos.shape[0])
        self._grow(n)
        a = self.a
        a.posp[:n, :3] = pos
        a.posp[:n, 3] = 0
        a.velr[:n, :3] = vel
        a.velr[:n, 3] = rho
        a.prev[:n, :3] = vel
        a.prev[:n, 3] = rho
        a.id[:n] = ids
        self.n, self.nb = n, int(nb)

    # -------------------------------------------------------------- step phases
    def nl_pi(self):
        L, s, ws = _lib.lib(), _stream(), self.ws.handle
        g, p, n, nb, a = _lib.ref(self.grid), _lib.ref(self.prm), self.n, self.nb, self.a
        self.ws.reset()
        # the keys travelled with the rows (K7 of the previous step, on whichever rank owned
        # the row): only the per-cell histogram is rebuilt, no K1 pass over the positions
        _lib.check(L.sphb_cell_hist(ws, g, _ptr(a.key), n, _ptr(self.ctrl), s), "sphb_cell_hist")
        _lib.check(L.sphb_step_begin(_ptr(self.ctrl), s), "sphb_step_begin")
        _lib.check(L.sphb_sort(ws, g, _ptr(a.key), n, _ptr(self.keys_sorted), _ptr(self.perm),
                               _ptr(self.ctrl), s), "sphb_sort")
        _lib.check(L.sphb_reorder(p, g, n, _ptr(self.perm), _ptr(self.keys_sorted), _ptr(a.posp),
                                  _ptr(a.velr), _ptr(a.prev), _ptr(a.id), _ptr(self.posp_s),
                                  _ptr(self.velr_s), _ptr(self.prev_s), _ptr(self.id_s),
                                  _ptr(self.aux), _ptr(self.cell_s), _ptr(self.ctrl), s), "sphb_reorder")
        _lib.check(L.sphb_cell_ranges(ws, g, _ptr(self.beg), _ptr(self.end), _ptr(self.ctrl), s),
                   "sphb_cell_ranges")
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        _lib.check(L.sphb_interact(ws, p, g, n, nb, _ptr(self.posp_s), _ptr(self.velr_s),
                                   _ptr(self.aux), _ptr(self.cell_s), _ptr(self.beg), _ptr(self.end),
                                   _ptr(self.acc), _ptr(self.drho), _ptr(self.visc), _ptr(self.ctrl),
                                   s), "sphb_interact")
        ev[1].record()
        self.pi_events.append(ev)

    def dt_words(self):
        return self.ctrl.view(torch.int64)[5:7]

    def counter_words(self):
        return self.ctrl.view(torch.int64)[8:12]

    def su_and_count(self):
        L, s, ws = _lib.lib(), _stream(), self.ws.handle
        g, p, n, nb, a = _lib.ref(self.grid), _lib.ref(self.prm), self.n, self.nb, self.a
        _lib.check(L.sphb_integrate(ws, p, g, n, nb, _ptr(self.posp_s), _ptr(self.velr_s),
                                    _ptr(self.prev_s), _ptr(self.id_s), _ptr(self.acc),
                                    _ptr(self.drho), _ptr(a.posp), _ptr(a.velr), _ptr(a.prev),
                                    _ptr(a.id), _ptr(self.keys), _ptr(self.ctrl), s), "sphb_integrate")
        _lib.check(L.sphb_step_end(_ptr(self.ctrl), p, _ptr(self.rec), self.rec_cap, s), "sphb_step_end")
        x0, x1 = self.bounds
        _lib.check(L.sphb_slab_count(g, n, nb, _ptr(self.keys), _ptr(a.id), x0, x1, _ptr(self.tiles),
                                     _ptr(self.totals), s), "sphb_slab_count")

    def status_words(self):
        """10 totals + the error word, int64, for the one all-gather of the step."""
        return torch.cat([self.totals.to(torch.int64), self.ctrl.view(torch.int64)[7:8]])

    def scatter(self, layout):
        L, s = _lib.lib(), _stream()
        g, n, nb, a, b = _lib.ref(self.grid), self.n, self.nb, self.a, self.b
        x0, x1 = self.bounds
        kb = (ctypes.c_int64 * 2)(*layout["keep_bases"])
        sec = (ctypes.c_int64 * 6)(*layout["sections"])
        sl = self._buf("send", 0, layout["send_rows"][0])
        sr = self._buf("send", 1, layout["send_rows"][1])
        _lib.check(L.sphb_slab_scatter(g, n, nb, _ptr(self.keys), _ptr(a.id), x0, x1, _ptr(self.tiles),
                                       _ptr(a.posp), _ptr(a.velr), _ptr(a.prev), kb, _ptr(b.posp),
                                       _ptr(b.velr), _ptr(b.prev), _ptr(b.id), _ptr(b.key), _ptr(sl), _ptr(sr),
                                       sec, s),
                   "sphb_slab_scatter")

    def unpack(self, layout):
        L, s, b = _lib.lib(), _stream(), self.b
        for side in (0, 1):
            buf = self.recv[side]
            for r0, cnt, dst in layout["unpack"][side]:
                if cnt:
                    _lib.check(L.sphb_slab_unpack(_ptr(buf), r0, cnt, dst, _ptr(b.posp), _ptr(b.velr),
                                                  _ptr(b.prev), _ptr(b.id), _ptr(b.key), s),
                               "sphb_slab_unpack")
        self.a, self.b = self.b, self.a
        self.n, self.nb = layout["n_next"], layout["nb_next"]


def rank_layout(tab, r, nranks):
    """Next-step layout of rank r from every rank's 10 totals (tab[k][c])."""
    t = tab[r]
    left = tab[r - 1] if r > 0 else np.zeros(NCAT, np.int64)
    right = tab[r + 1] if r < nranks - 1 else np.zeros(NCAT, np.int64)
    # rows arriving from the left neighbour = its right-side sends, and vice versa
    in_l = [int(left[MIGR_B]), int(left[MIGR_F]), int(left[HALOR_B]), int(left[HALOR_F])]
    in_r = [int(right[MIGL_B]), int(right[MIGL_F]), int(right[HALOL_B]), int(right[HALOL_F])]
    keep_b, keep_f = int(t[KEEP_B]), int(t[KEEP_F])
    nb_next = keep_b + in_l[0] + in_r[0] + in_l[2] + in_r[2]
    nf_next = keep_f + in_l[1] + in_r[1] + in_l[3] + in_r[3]
    # boundary block: kept | mig L | mig R | halo L | halo R ; fluid block likewise at nb_next
    dst = {
        ("L", "migB"): keep_b, ("R", "migB"): keep_b + in_l[0],
        ("L", "haloB"): keep_b + in_l[0] + in_r[0], ("R", "haloB"): keep_b + in_l[0] + in_r[0] + in_l[2],
        ("L", "migF"): nb_next + keep_f, ("R", "migF"): nb_next + keep_f + in_l[1],
        ("L", "haloF"): nb_next + keep_f + in_l[1] + in_r[1],
        ("R", "haloF"): nb_next + keep_f + in_l[1] + in_r[1] + in_l[3],
    }
    unpack = []
    for side, cnts in (("L", in_l), ("R", in_r)):
        r0 = 0
        ops = []
        for k, name in enumerate(("migB", "migF", "haloB", "haloF")):
            ops.append((r0, cnts[k], dst[(side, name)]))
            r0 += cnts[k]
        unpack.append(ops)
    send_l = [int(t[MIGL_B]), int(t[MIGL_F]), int(t[HALOL_B]), int(t[HALOL_F])]
    send_r = [int(t[MIGR_B]), int(t[MIGR_F]), int(t[HALOR_B]), int(t[HALOR_F])]
    sections = [send_l[0], send_l[0] + send_l[1], send_l[0] + send_l[1] + send_l[2],
                send_r[0], send_r[0] + send_r[1], send_r[0] + send_r[1] + send_r[2]]
    return dict(keep_bases=(0, nb_next), sections=sections, n_next=nb_next + nf_next,
                nb_next=nb_next, send_rows=(sum(send_l), sum(send_r)),
                recv_rows=(sum(in_l), sum(in_r)), unpack=unpack)


# ------------------------------------------------------------------ the stepper
class DeviceSlabSim:
    """X-slab stepper of the local ranks of ``comm`` (all on this process's current device)."""

    def __init__(self, system, params, comm, reach: int | None = None, precision: int = 0,
                 bounds=None, order: int = 0, rebalance_every: int = 0):
        self.params = params
        self.rebalance_every = int(rebalance_every)
        self.comm = comm
        self.reach = int(params.n_subdiv if reach is None else reach)
        cs, dims = grid_dims(params)
        nx = int(dims[0])
        pos = torch.as_tensor(np.ascontiguousarray(system.pos, np.float32))
        col = columns_of(pos[:, 0], float(np.asarray(params.domain_min, np.float64)[0]), cs, nx).numpy()
        if bounds is None:
            bounds = balanced_bounds(np.bincount(col, minlength=nx), comm.nranks, max(self.reach, 1))
        self.bounds = np.asarray(bounds, np.int64)
        self.prm = params_desc(params, float(system.mass_fluid), float(system.mass_boundary), order,
                               precision)
        dev = torch.device("cuda", torch.cuda.current_device())
        nb = int(system.count_boundary)
        self.n_total = int(system.n)
        self.ranks = []
        for k in comm.local_ranks:
            x0, x1 = int(self.bounds[k]), int(self.bounds[k + 1])
            sel = (col >= x0) & (col < x1)
            ib, iff = np.nonzero(sel[:nb])[0], np.nonzero(sel[nb:])[0] + nb
            idx = np.concatenate([ib, iff])
            r = DevRank(k, (x0, x1), params, self.prm, self.reach, dev, int(idx.size * 1.1) + 1024)
            t = lambda v: torch.as_tensor(np.ascontiguousarray(v)).to(dev)  # noqa: E731
            r.upload(t(system.pos[idx]), t(system.vel[idx]), t(system.rho[idx]),
                     t(np.asarray(system.id)[idx].astype(np.int64)), ib.size)
            self.ranks.append(r)
        self.step_index = 0
        self._halos_built = False

    def _exchange(self):
        """Phases 4-7 (the counts already computed by su_and_count / prime()); returns the
        all-gathered totals table (ranks x 10)."""
        gathered = self.comm.allgather([r.status_words() for r in self.ranks])
        tab = gathered[0].cpu().numpy()  # the step's one host synchronisation
        errs = tab[:, NCAT].astype(np.uint64)
        if np.any(errs != np.uint64(_lib.ERR_NONE)):
            k = int(np.argmax(errs != np.uint64(_lib.ERR_NONE)))
            raise RuntimeError(f"slab rank {k} diverged: {decode_err(errs[k])}")
        tots = tab[:, :NCAT]
        items, layouts = [], []
        for r in self.ranks:
            lay = rank_layout(tots, r.rank, self.comm.nranks)
            r._grow(lay["n_next"])
            r.scatter(lay)
            rl = r._buf("recv", 0, lay["recv_rows"][0])
            rr = r._buf("recv", 1, lay["recv_rows"][1])
            items.append(dict(send_l=(r.send[0], lay["send_rows"][0]), send_r=(r.send[1], lay["send_rows"][1]),
                              recv_l=(rl, lay["recv_rows"][0]), recv_r=(rr, lay["recv_rows"][1])))
            layouts.append(lay)
        self.comm.sendrecv(items)
        for r, lay in zip(self.ranks, layouts):
            r.unpack(lay)
        return tots

    def _count_resident(self):
        """K1 keys + category counts of the current (assembled) arrays."""
        L, s = _lib.lib(), _stream()
        for r in self.ranks:
            r.ws.reset()
            _lib.check(L.sphb_cell_keys(r.ws.handle, _lib.ref(r.grid), _ptr(r.a.posp), r.n, r.nb,
                                        _ptr(r.keys), None, _ptr(r.ctrl), s), "sphb_cell_keys")
            x0, x1 = r.bounds
            _lib.check(L.sphb_slab_count(_lib.ref(r.grid), r.n, r.nb, _ptr(r.keys), _ptr(r.a.id), x0, x1,
                                         _ptr(r.tiles), _ptr(r.totals), s), "sphb_slab_count")

    def measured_pi_ms(self) -> np.ndarray:
        """Mean interaction time per rank since the last rebalance (all ranks, gathered)."""
        torch.cuda.synchronize()
        mine = []
        for r in self.ranks:
            ts = [a.elapsed_time(b) for a, b in r.pi_events]
            mine.append(torch.tensor([float(np.mean(ts)) if ts else 1.0], dtype=torch.float64,
                                     device=r.dev))
            r.pi_events.clear()
        return self.comm.allgather(mine)[0].reshape(-1).cpu().numpy()

    def set_bounds(self, bounds):
        """Move the slab bounds and re-settle: repeat classify + exchange until no particle
        sits outside its slab (multi-column moves take several neighbour hops); the last round
        rebuilds the halos for the new bounds."""
        bounds = np.asarray(bounds, np.int64)
        self.bounds = bounds
        for r in self.ranks:
            r.bounds = (int(bounds[r.rank]), int(bounds[r.rank + 1]))
            r.grid = grid_desc(self.params, self.reach, target_cols=r.bounds)
        for _ in range(self.comm.nranks + 1):
            self._count_resident()
            tots = self._exchange()
            if not np.any(tots[:, MIGL_B:MIGR_F + 1]):
                break

    def rebalance(self, times=None):
        """Equal-time slab bounds (slab.rebalance_slices, the reference's balance.py:53-88
        restated) from the measured (or given) per-rank interaction times; width >= reach."""
        t = self.measured_pi_ms() if times is None else np.asarray(times, np.float64)
        new = enforce_min_width(rebalance_slices(self.bounds, t), max(self.reach, 1))
        if not np.array_equal(new, self.bounds):
            self.set_bounds(new)
        return new

    def prime(self):
        """Initial halos: classify the uploaded owned rows (keys from K1) and exchange."""
        L, s = _lib.lib(), _stream()
        for r in self.ranks:
            r.ws.reset()
            _lib.check(L.sphb_cell_keys(r.ws.handle, _lib.ref(r.grid), _ptr(r.a.posp), r.n, r.nb,
                                        _ptr(r.keys), None, _ptr(r.ctrl), s), "sphb_cell_keys")
            x0, x1 = r.bounds
            _lib.check(L.sphb_slab_count(_lib.ref(r.grid), r.n, r.nb, _ptr(r.keys), _ptr(r.a.id), x0, x1,
                                         _ptr(r.tiles), _ptr(r.totals), s), "sphb_slab_count")
        self._exchange()
        self._halos_built = True

    def step(self):
        if not self._halos_built:
            self.prime()
        if self.rebalance_every and self.step_index and self.step_index % self.rebalance_every == 0:
            self.rebalance()
        for r in self.ranks:
            r.nl_pi()
        # the step's dt is global (min over ranks) and needed now; the counters stay per rank in
        # each rank's record ring and are summed over ranks only when read (records())
        self.comm.allreduce([r.dt_words() for r in self.ranks], "min")
        for r in self.ranks:
            r.su_and_count()
        self._exchange()
        self.step_index += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()

    # -------------------------------------------------------------- readback
    def records(self, first, last):
        """StepStats records [first, last): dt (the same on every rank) and the counters summed
        over the ranks (one all-reduce per read instead of one per step)."""
        words = _lib.REC_DTYPE.itemsize // 8
        cnt = [r.rec.view(torch.int64).reshape(-1, words)[:, 1:].clone() for r in self.ranks]
        self.comm.allreduce(cnt, "sum")
        r = self.ranks[0]
        host = r.rec.cpu().numpy().view(_lib.REC_DTYPE).copy()
        summed = cnt[0].cpu().numpy().view(np.uint64)
        for k, f in enumerate(("candidate_pairs", "hits_ordered", "force_evals", "ff_force_evals")):
            host[f] = summed[:, k]
        return host[np.arange(first, last) % r.rec_cap]

    def ctrl_host(self):
        return read_ctrl(self.ranks[0].ctrl)

    def gather_host(self):
        """Owned particles of the local ranks (pos, vel, rho, id, is_fluid) as numpy, id-sorted."""
        pos, vel, rho, ids, fl = [], [], [], [], []
        for r in self.ranks:
            n, nb = r.n, r.nb
            i = r.a.id[:n].cpu().numpy()
            own = i >= 0
            pos.append(r.a.posp[:n, :3].cpu().numpy()[own])
            vel.append(r.a.velr[:n, :3].cpu().numpy()[own])
            rho.append(r.a.velr[:n, 3].cpu().numpy()[own])
            ids.append(i[own])
            fl.append((np.arange(n) >= nb)[own])
        pos, vel, rho, ids, fl = (np.concatenate(v) for v in (pos, vel, rho, ids, fl))
        o = np.argsort(ids)
        return pos[o], vel[o], rho[o], ids[o], fl[o]

    @property
    def n_owned_max(self) -> int:
        return max(int((r.a.id[: r.n] >= 0).sum().item()) for r in self.ranks)

    def choose_pi_block(self, large_min) -> list[int]:
        """Per rank, run_simulation's rule: 384-target blocks when the rank owns at least
        ``large_min`` targets, else 256; 128 when ``large_min`` is None (h/2 cells); returns
        each local rank's blocking."""
        out = []
        for r in self.ranks:
            owned = int((r.a.id[: r.n] >= 0).sum().item())
            blk = 128 if large_min is None else 384 if owned >= large_min else 256
            r.pi_block = blk
            r.ws.set_pi_block(blk)
            out.append(blk)
        return out

    def launches_per_step(self) -> int:
        return int(_lib.lib().sphb_step_launch_count(_lib.ref(self.ranks[0].grid), self.ranks[0].n)) + 4


def estimate_steps_per_sync() -> int:
    """Host synchronisations per step of DeviceSlabSim (the totals all-gather)."""
    return 1


__all__ = ["DeviceSlabSim", "DevLoopbackComm", "DevDistComm", "rank_layout", "math"]
