"""Device-resident X-slab decomposition: the production multi-GPU stepper.

The global cell grid is cut along x into slabs of whole cell columns [x0_k, x1_k), one per
rank (the reference's Slices geometry, engines/kernels.py:230-323 / balance.py:46-88, with
particle-count or measured-time balanced bounds, ``slab.py``).  A rank's arrays hold its owned
rows plus read-only halo copies (id < 0) of the neighbours' rows within ``reach`` columns, so
every pair its targets need is present; rows stay in place from step to step.

One step per rank, edge bands first so the exchange overlaps the interior interaction:

  1. NL (movers-only sort: the rows arrive in the previous sorted order; rows that left the
     slab and the old halo copies carry the dead key and sort to the tail), K3 reorder;
     ``sphb_band_count``: sizes of the two edge bands (the W = reach + 1 owned columns next
     to each neighbour) and the host-read info words (live rows, boundary rows, band rows);
  2. interaction of the edge-band targets; the host reads the info words meanwhile (the GPU
     still has the edge interaction queued: no idle gap), exchanges the band sizes with its
     neighbours on the host and packs each band row's sorted state + forces
     (``sphb_band_pack``, 96-B rows);
  3. the band buffers move on a high-priority comm stream (NCCL send/recv over NVLink) while
     the interior targets' interaction runs on the compute stream;
  4. device all-reduce (MIN) of the two dt minima (global dt);
  5. K7 on the live rows (rows that left the slab -> dead key: the neighbour integrates them
     from the band it received), then ``sphb_band_integrate`` on each received band with the
     same arithmetic and dt: rows landing in this slab are migrants (owned), rows within reach
     columns outside it are the next step's halo copies, the rest are dropped; they are
     appended after the live rows and the dead bin's end is moved (``sphb_slab_tail``).

A band row of the sender at step k becomes, integrated by the receiver, exactly the halo copy /
migrant the receiver needs at step k + 1 (|column change| <= 1 per step, flagged otherwise), so
the only per-step traffic is the bands, and it travels while the interior targets compute.
Counters stay per rank in the record ring and are summed over ranks when read.

Re-placing the bounds (rebalance) and the initial halos use the full re-layout exchange
(``sphb_slab_count`` / ``sphb_slab_scatter`` / ``sphb_slab_unpack``).

Comms: ``DevLoopbackComm`` (k virtual ranks on one GPU, device copies, stream-ordered) and
``DevDistComm`` (torch.distributed: NCCL, or gloo with host staging when several processes
share one GPU; band sizes and error words over a host (gloo) group).
"""
from __future__ import annotations

import collections
import ctypes

import numpy as np
import torch

from . import _lib
from .device import Workspace, _ptr, _stream, cellbits_of, decode_err, new_ctrl, read_ctrl
from .physics import grid_desc, grid_dims, params_desc
from .slab import balanced_bounds, columns_of, enforce_min_width, rebalance_slices

ROW_WORDS = 16  # re-layout exchange row: 64 B (posp, velr, prev float4, int64 id, u32 key, pad)
BAND_WORDS = 24  # edge-band row: 96 B (include/sphb200.h SPHB_BAND_ROW_BYTES)
NCAT = 10
KEEP_B, KEEP_F, MIGL_B, MIGL_F, MIGR_B, MIGR_F, HALOL_B, HALOL_F, HALOR_B, HALOR_F = range(10)
INFO_WORDS = 8  # sphb_band_count: live rows, boundary rows, band rows L / R, err, active, step


# ------------------------------------------------------------------ comms
class DevLoopbackComm:
    """k virtual ranks in one process on one device (stream-ordered device copies)."""

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

    def host_allgather(self, rows):
        """rows[local] = int64 vector -> (nranks, k) table of every rank's vector."""
        return np.stack([np.asarray(r, np.int64) for r in rows])

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

    def band_sendrecv(self, items, ready_events):
        """The band exchange; returns per local rank the event the receiver waits on (None:
        already ordered on the compute stream)."""
        self.sendrecv(items)
        return [None] * len(items)


class DevDistComm:
    """One rank per process over torch.distributed.  NCCL (the production transport) moves the
    device buffers directly, the band exchange on a high-priority comm stream; over gloo
    (several processes sharing one GPU, the multi-process test on a single-GPU box) the same
    calls stage through host memory.  Small host vectors (band sizes, error words) go over a
    gloo group."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self.local_ranks = [self.rank]
        self.host = dist.get_backend() != "nccl"
        self.cpu_group = None if self.host else dist.new_group(backend="gloo")
        self.band_group = None
        self.cstream = None
        if not self.host:
            self.cstream = torch.cuda.Stream(priority=-1)
            try:  # the band exchange's NCCL kernels ahead of the interior interaction's CTAs
                from torch.distributed import ProcessGroupNCCL
                opts = ProcessGroupNCCL.Options()
                opts.is_high_priority_stream = True
                self.band_group = dist.new_group(backend="nccl", pg_options=opts)
            except Exception:  # noqa: BLE001 -- older torch: the default group's stream
                self.band_group = None

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

    def host_allgather(self, rows):
        h = torch.as_tensor(np.asarray(rows[0], np.int64))
        parts = [torch.empty_like(h) for _ in range(self.nranks)]
        self.dist.all_gather(parts, h, group=self.cpu_group)
        return torch.stack(parts).numpy()

    def _ops(self, it, group):
        d, r, n = self.dist, self.rank, self.nranks
        ops, landing = [], []
        for side, peer, ok in (("l", r - 1, r > 0), ("r", r + 1, r < n - 1)):
            if not ok:
                continue
            buf, rows = it["send_" + side]
            if rows:
                src = buf[:rows].cpu() if self.host else buf[:rows]
                ops.append(d.P2POp(d.isend, src, peer, group=group))
            buf, rows = it["recv_" + side]
            if rows:
                if self.host:
                    tmp = torch.empty(buf[:rows].shape, dtype=buf.dtype)
                    landing.append((buf, rows, tmp))
                    ops.append(d.P2POp(d.irecv, tmp, peer, group=group))
                else:
                    ops.append(d.P2POp(d.irecv, buf[:rows], peer, group=group))
        return ops, landing

    def sendrecv(self, items):
        ops, landing = self._ops(items[0], None)
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for buf, rows, tmp in landing:
            buf[:rows].copy_(tmp)

    def band_sendrecv(self, items, ready_events):
        if self.host:  # host-staged: the .cpu() of the send buffers waits for the pack
            self.sendrecv(items)
            return [None]
        done = torch.cuda.Event()
        with torch.cuda.stream(self.cstream):
            self.cstream.wait_event(ready_events[0])
            ops, _ = self._ops(items[0], self.band_group)
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()  # the comm stream waits for the NCCL kernels
            done.record(self.cstream)
        return [done]


class DevPeerComm(DevDistComm):
    """DevDistComm whose edge bands travel by peer-memory stores instead of NCCL: each rank's
    band kernel (sphb_band_put) writes its rows straight into the neighbours' receive buffers
    -- CUDA IPC mappings of the neighbours' device memory, NVLink P2P stores on a multi-GPU
    box -- and releases a step tag into their flag words; a receiver's stream waits for its
    flags (sphb_band_wait) before integrating.  Pack and send are one kernel, on a
    high-priority comm stream with 32 CTAs, next to the interior interaction.  Receive buffers
    are double-buffered by the tag's parity (a sender cannot run two steps ahead: it needs the
    receiver's band of the step in between).  The control plane (band sizes, dt all-reduce,
    re-layouts) stays on torch.distributed.  Several processes may share one GPU (the CPU-side
    control then runs over gloo): IPC handles of one device open in another process."""

    transport = "peer"

    def __init__(self, cap_rows: int = 1 << 16):
        super().__init__()
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.pstream = torch.cuda.Stream(priority=-1)
        self.done = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.flags = torch.zeros(2, dtype=torch.int64, device=self.dev)  # from left, from right
        self.tag = 0
        self.cap = 0
        self.put_ev = torch.cuda.Event()
        self._share(int(cap_rows))

    def _share(self, cap):
        """(Re)allocate the receive buffers and map the neighbours' (collective)."""
        from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor
        torch.cuda.synchronize()
        self.cap = cap
        self.recv = [torch.zeros((2, cap, BAND_WORDS), dtype=torch.float32, device=self.dev)
                     for _ in range(2)]
        mine = [reduce_tensor(t)[1] for t in (self.recv[0], self.recv[1], self.flags)]
        allh = [None] * self.nranks
        self.dist.all_gather_object(allh, mine, group=self.cpu_group)
        r, n = self.rank, self.nranks
        self.peer, self.peer_flag = [None, None], [None, None]
        err = None
        try:
            if r > 0:  # my left band lands in the left neighbour's "from right" buffer and flag
                self.peer[0] = rebuild_cuda_tensor(*allh[r - 1][1])
                self.peer_flag[0] = rebuild_cuda_tensor(*allh[r - 1][2])[1:2]
            if r < n - 1:
                self.peer[1] = rebuild_cuda_tensor(*allh[r + 1][0])
                self.peer_flag[1] = rebuild_cuda_tensor(*allh[r + 1][2])[0:1]
        except Exception as e:  # noqa: BLE001 -- raised after the collective below
            err = e
        self.dist.barrier(group=self.cpu_group)
        if err is not None:
            raise err

    def ensure_capacity(self, max_rows: int):
        """Every rank calls this with the same number (the all-gathered band sizes)."""
        if max_rows > self.cap:
            self._share(int(max_rows * 1.3) + 1024)

    def close(self):
        """Drop the neighbours' mappings before the producers exit (collective)."""
        torch.cuda.synchronize()
        self.peer, self.peer_flag = [None, None], [None, None]
        self.dist.barrier(group=self.cpu_group)

    def next_tag(self) -> int:
        self.tag += 1
        return self.tag

    def recv_view(self, side: int, tag: int):
        return self.recv[side][tag & 1]

    def peer_view(self, side: int, tag: int):
        return self.peer[side][tag & 1] if self.peer[side] is not None else None


# ------------------------------------------------------------------ one rank
class _Arrays:
    def __init__(self, cap, dev):
        self.posp = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.velr = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.prev = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
        self.id = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.key = torch.zeros(cap, dtype=torch.int32, device=dev)  # next sort key (K7 / bands)


class _Sorted:
    """This step's sorted copies and force buffers (read by the interaction and K7)."""

    def __init__(self, cap, dev):
        f4 = lambda: torch.zeros((cap, 4), dtype=torch.float32, device=dev)  # noqa: E731
        self.posp, self.velr, self.prev, self.aux = f4(), f4(), f4(), f4()
        self.id = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.perm = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.cell = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.acc = torch.zeros((cap, 3), dtype=torch.float64, device=dev)
        self.drho = torch.zeros(cap, dtype=torch.float64, device=dev)
        self.visc = torch.zeros(cap, dtype=torch.float64, device=dev)


class DevRank:
    """A slab's arrays, engine scratch and step phases on one device."""

    CAP_FACTOR, CAP_SLACK = 1.25, 4096  # row capacity headroom (tests set it tight: regrowth)

    def __init__(self, rank, nranks, bounds, params, prm, reach, dev, n_hint):
        self.rank, self.nranks = rank, nranks
        self.params, self.prm, self.reach, self.dev = params, prm, int(reach), dev
        self.width = self.reach + 1  # band columns: halo reach + one column of motion
        self.sides = (1 if rank > 0 else 0) | (2 if rank < nranks - 1 else 0)
        _, dims = grid_dims(params)
        self.nx = int(dims[0])
        self.ncells = int(np.prod(dims))
        self.cellbits = cellbits_of(self.ncells)
        self.dead = (2 << self.cellbits) - 1
        self.set_bounds(bounds)
        self.ctrl = new_ctrl(dev)
        self.rec_cap = 4096
        self.rec = torch.zeros(self.rec_cap * _lib.REC_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.totals = torch.zeros(NCAT, dtype=torch.int32, device=dev)
        self.info = torch.zeros(INFO_WORDS, dtype=torch.int64, device=dev)
        self.info_h = torch.zeros(INFO_WORDS, dtype=torch.int64, pin_memory=True)
        self.info_ev = torch.cuda.Event()
        self.pack_ev = torch.cuda.Event()
        self.scratch = torch.zeros(int(_lib.lib().sphb_band_scratch_words(_lib.ref(self.grid))),
                                   dtype=torch.int32, device=dev)
        self.beg = torch.zeros(2 * self.ncells + 1, dtype=torch.int32, device=dev)
        self.end = torch.zeros(2 * self.ncells + 1, dtype=torch.int32, device=dev)
        self.send = [torch.zeros((1, BAND_WORDS), dtype=torch.float32, device=dev) for _ in range(2)]
        self.recv = [torch.zeros((1, BAND_WORDS), dtype=torch.float32, device=dev) for _ in range(2)]
        self.n = self.nb = 0     # rows in the arrays at the start of the step / boundary rows
        self.n_live = self.nb_live = 0
        self.cap = 0
        self.pi_block = None
        self.pi_kernel = None
        self._retired = []       # buffers the running step still reads after a growth
        # (start, end) of the recent interaction phases (since the last rebalance, at most 64)
        self.pi_events = collections.deque(maxlen=64)
        self._grow(n_hint)

    def set_bounds(self, bounds):
        self.bounds = (int(bounds[0]), int(bounds[1]))
        x0, x1 = self.bounds
        self.grid = grid_desc(self.params, self.reach, target_cols=self.bounds)
        w = self.width
        # interaction launches: the edge bands next to each neighbour first, then the interior
        # (a slab narrower than two bands is all edge)
        if self.sides == 0:
            self.edge_cols, self.inner_cols = [(x0, x1)], []
        elif x1 - x0 < 2 * w:
            self.edge_cols, self.inner_cols = [(x0, x1)], []
        else:
            lo = (x0, x0 + w) if self.sides & 1 else None
            hi = (x1 - w, x1) if self.sides & 2 else None
            self.edge_cols = [c for c in (lo, hi) if c]
            a = x0 + w if self.sides & 1 else x0
            b = x1 - w if self.sides & 2 else x1
            self.inner_cols = [(a, b)] if b > a else []
        self.edge_grids = [grid_desc(self.params, self.reach, target_cols=c) for c in self.edge_cols]
        self.inner_grids = [grid_desc(self.params, self.reach, target_cols=c) for c in self.inner_cols]
        # one rank (no neighbour) is the whole-domain path: no band, nothing to hide the host
        # read behind, so the whole interaction is queued before it
        if self.sides == 0:
            self.edge_grids, self.inner_grids = [], self.edge_grids

    # -------------------------------------------------------------- capacity
    def _grow(self, n):
        """Capacity of every per-row array (between steps: nothing to keep but the rows)."""
        if n <= self.cap:
            return
        cap = int(n * self.CAP_FACTOR) + self.CAP_SLACK
        old = getattr(self, "a", None)
        self.a, self.b = _Arrays(cap, self.dev), _Arrays(cap, self.dev)
        if old is not None and self.n:
            for f in ("posp", "velr", "prev", "id", "key"):
                getattr(self.a, f)[: self.n].copy_(getattr(old, f)[: self.n])
        self.s = _Sorted(cap, self.dev)
        self.keys_sorted = torch.zeros(cap, dtype=torch.int32, device=self.dev)
        old_tiles = getattr(self, "tiles", None)
        self.tiles = torch.zeros(NCAT * int(_lib.lib().sphb_slab_tiles(cap)) + NCAT,
                                 dtype=torch.int32, device=self.dev)
        if old_tiles is not None:  # a re-layout grows between its count and its scatter
            self.tiles[: old_tiles.shape[0]].copy_(old_tiles)
        self._new_ws(cap)
        self.cap = cap

    def _new_ws(self, cap):
        self.ws = Workspace(cap, self.ncells)
        if self.pi_kernel:  # a regrown workspace keeps the chosen interaction build
            self.ws.set_pi_kernel(self.pi_kernel)
        if self.pi_block:
            self.ws.set_pi_block(self.pi_block)

    def _grow_mid_step(self, n_next):
        """Capacity for n_next rows at the host read point of a step (its interaction may still
        be running): K7 still reads this step's sorted arrays and writes the new primary arrays,
        the next sort needs the previous order (keys_sorted) and a workspace of the new size
        whose histogram K7 fills.  The old buffers are kept until the next step."""
        cap = int(n_next * self.CAP_FACTOR) + self.CAP_SLACK
        self._retired = [self.s, self.ws, self.a, self.b]
        self.a, self.b = _Arrays(cap, self.dev), _Arrays(cap, self.dev)
        ks = torch.zeros(cap, dtype=torch.int32, device=self.dev)
        ks[: self.n_live].copy_(self.keys_sorted[: self.n_live])
        self.keys_sorted = ks
        self.tiles = torch.zeros(NCAT * int(_lib.lib().sphb_slab_tiles(cap)) + NCAT,
                                 dtype=torch.int32, device=self.dev)
        self._new_ws(cap)
        self._next_sorted = _Sorted(cap, self.dev)
        self.cap = cap

    def _buf(self, lst, side, rows, words):
        if lst[side].shape[0] < rows or lst[side].shape[1] != words:
            lst[side] = torch.zeros((int(rows * 1.3) + 1024, words), dtype=torch.float32,
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
    def _aux(self):
        """The derived rows: only the FP64 kernel reads them (the FP32 gather / paired builds
        recompute a target's own values)."""
        return self.s.aux if int(self.prm.precision) == _lib.SPHB_FP64 else None

    def _interact(self, grids):
        L, s, ws, sa = _lib.lib(), _stream(), self.ws.handle, self.s
        p = _lib.ref(self.prm)
        for g in grids:
            _lib.check(L.sphb_interact(ws, p, _lib.ref(g), self.n, 0, _ptr(sa.posp), _ptr(sa.velr),
                                       _ptr(self._aux()), _ptr(sa.cell), _ptr(self.beg), _ptr(self.end),
                                       _ptr(sa.acc), _ptr(sa.drho), _ptr(sa.visc), _ptr(self.ctrl),
                                       s), "sphb_interact")

    def phase_edges(self):
        """Step begin, NL of the resident rows, band sizes + info read-back, edge targets."""
        self._retired = []
        if getattr(self, "_next_sorted", None) is not None:
            self.s, self._next_sorted = self._next_sorted, None
        if self.sides:
            # every halo row arrives (and leaves) each step: with many arrivals per cell the
            # movers-only sort's per-key chains cost more than the radix passes
            self.ws.set_mover_cap(min(max(4096, self.n // 32), 1 << 20, self.ws.n_max))
        L, s, ws = _lib.lib(), _stream(), self.ws.handle
        g, p, n, a, sa = _lib.ref(self.grid), _lib.ref(self.prm), self.n, self.a, self.s
        _lib.check(L.sphb_step_begin(_ptr(self.ctrl), s), "sphb_step_begin")
        _lib.check(L.sphb_sort_ranges(ws, g, _ptr(a.key), n, _ptr(self.keys_sorted), _ptr(sa.perm),
                                      _ptr(self.beg), _ptr(self.end), _ptr(self.ctrl), s),
                   "sphb_sort_ranges")
        _lib.check(L.sphb_reorder(p, g, n, _ptr(sa.perm), _ptr(self.keys_sorted), _ptr(a.posp),
                                  _ptr(a.velr), _ptr(a.prev), _ptr(a.id), _ptr(sa.posp),
                                  _ptr(sa.velr), _ptr(sa.prev), _ptr(sa.id), _ptr(self._aux()),
                                  _ptr(sa.cell), _ptr(self.ctrl), s), "sphb_reorder")
        _lib.check(L.sphb_band_count(g, self.width, self.sides, _ptr(self.beg), _ptr(self.end),
                                     _ptr(self.scratch), _ptr(self.info), _ptr(self.ctrl), s),
                   "sphb_band_count")
        self.info_h.copy_(self.info, non_blocking=True)
        self.info_ev.record()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        self._pi_ev = ev
        self._interact(self.edge_grids)
        if self.sides == 0:  # one rank: all of it (nothing to send)
            self._interact(self.inner_grids)

    def read_info(self):
        """The host read of the step (the edge interaction is still queued on the GPU)."""
        self.info_ev.synchronize()
        h = self.info_h.numpy()
        self.n_live, self.nb_live = int(h[0]), int(h[1])
        self.band_rows = (int(h[2]), int(h[3]))
        return h.copy()

    def phase_pack(self):
        L, s, sa = _lib.lib(), _stream(), self.s
        sl = self._buf(self.send, 0, self.band_rows[0], BAND_WORDS)
        sr = self._buf(self.send, 1, self.band_rows[1], BAND_WORDS)
        if self.sides:
            _lib.check(L.sphb_band_pack(_lib.ref(self.prm), _lib.ref(self.grid), self.width,
                                        self.sides, _ptr(self.beg), _ptr(self.end),
                                        _ptr(self.scratch), _ptr(sa.posp), _ptr(sa.velr),
                                        _ptr(sa.prev), _ptr(sa.id), _ptr(sa.acc), _ptr(sa.drho),
                                        _ptr(sl), _ptr(sr), s), "sphb_band_pack")
        self.pack_ev.record()

    def phase_put(self, comm, tag):
        """Peer transport: pack the bands straight into the neighbours' buffers (one kernel on
        the comm stream, after the edge interaction) and flag them."""
        L, sa = _lib.lib(), self.s
        comp = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(comp)
        ps = comm.pstream
        ps.wait_event(ev)
        pl, pr = comm.peer_view(0, tag), comm.peer_view(1, tag)
        fl, fr = comm.peer_flag
        _lib.check(L.sphb_band_put(_lib.ref(self.prm), _lib.ref(self.grid), self.width, self.sides,
                                   _ptr(self.beg), _ptr(self.end), _ptr(self.scratch), _ptr(sa.posp),
                                   _ptr(sa.velr), _ptr(sa.prev), _ptr(sa.id), _ptr(sa.acc),
                                   _ptr(sa.drho), _ptr(pl), _ptr(pr), _ptr(fl), _ptr(fr), tag,
                                   _ptr(comm.done), ps.cuda_stream), "sphb_band_put")
        comm.put_ev.record(ps)

    def phase_interior(self):
        if self.sides:
            self._interact(self.inner_grids)
        self._pi_ev[1].record()
        self.pi_events.append(self._pi_ev)

    def dt_words(self):
        return self.ctrl.view(torch.int64)[5:7]

    def phase_update(self, recv_rows, recv_event, peer=None):
        """K7 on the live rows, the received bands integrated and appended, step end.
        ``peer``: (comm, tag) of the peer-memory transport (wait for the flags, read its
        buffers), else the bands are in self.recv."""
        comp = torch.cuda.current_stream()
        if recv_event is not None:
            comp.wait_event(recv_event)
        L, s, ws = _lib.lib(), _stream(), self.ws.handle
        bufs = self.recv
        if peer is not None:
            comm, tag = peer
            comp.wait_event(comm.put_ev)  # the sorted arrays are read by our own put
            fl = comm.flags[0:1] if self.sides & 1 else None
            fr = comm.flags[1:2] if self.sides & 2 else None
            _lib.check(L.sphb_band_wait(_ptr(fl), _ptr(fr), tag, _ptr(self.ctrl), s), "sphb_band_wait")
            bufs = [comm.recv_view(0, tag), comm.recv_view(1, tag)]
        g, p, a, sa = _lib.ref(self.grid), _lib.ref(self.prm), self.a, self.s
        old = self._retired[0] if self._retired else None  # sorted arrays of a regrown rank
        src = old if old is not None else sa
        _lib.check(L.sphb_integrate(ws, p, g, self.n_live, self.nb_live, _ptr(src.posp),
                                    _ptr(src.velr), _ptr(src.prev), _ptr(src.id), _ptr(src.acc),
                                    _ptr(src.drho), _ptr(a.posp), _ptr(a.velr), _ptr(a.prev),
                                    _ptr(a.id), _ptr(a.key), _ptr(self.ctrl), s), "sphb_integrate")
        dst = self.n_live
        for side in (0, 1):
            cnt = int(recv_rows[side])
            if cnt:
                _lib.check(L.sphb_band_integrate(ws, p, g, _ptr(bufs[side]), cnt, dst,
                                                 _ptr(a.posp), _ptr(a.velr), _ptr(a.prev),
                                                 _ptr(a.id), _ptr(a.key), _ptr(self.keys_sorted),
                                                 _ptr(self.ctrl), s), "sphb_band_integrate")
                dst += cnt
        if self.sides:
            _lib.check(L.sphb_slab_tail(g, _ptr(self.end), dst, s), "sphb_slab_tail")
        _lib.check(L.sphb_step_end(_ptr(self.ctrl), p, _ptr(self.rec), self.rec_cap, s), "sphb_step_end")
        self.n = dst

    # -------------------------------------------------------------- re-layout (settle)
    def count_resident(self, fresh_keys: bool):
        """Category counts of the resident rows for the re-layout exchange; ``fresh_keys``: K1
        on an uploaded state (else the keys K7 / the bands wrote, dead keys dropped)."""
        L, s = _lib.lib(), _stream()
        g = _lib.ref(self.grid)
        if fresh_keys:
            self.ws.reset()
            _lib.check(L.sphb_cell_keys(self.ws.handle, g, _ptr(self.a.posp), self.n, self.nb,
                                        _ptr(self.a.key), None, _ptr(self.ctrl), s), "sphb_cell_keys")
        x0, x1 = self.bounds
        nb = self.nb if fresh_keys else 0  # after steps the list comes from the key
        _lib.check(L.sphb_slab_count(g, self.n, nb, _ptr(self.a.key), _ptr(self.a.id), x0, x1,
                                     _ptr(self.tiles), _ptr(self.totals), s), "sphb_slab_count")

    def status_words(self):
        """10 totals + the error word, int64, for the re-layout exchange's all-gather."""
        return torch.cat([self.totals.to(torch.int64), self.ctrl.view(torch.int64)[7:8]])

    def scatter(self, layout):
        L, s = _lib.lib(), _stream()
        g, n, nb, a, b = _lib.ref(self.grid), self.n, min(self.nb, self.n), self.a, self.b
        x0, x1 = self.bounds
        kb = (ctypes.c_int64 * 2)(*layout["keep_bases"])
        sec = (ctypes.c_int64 * 6)(*layout["sections"])
        sl = self._buf(self.send, 0, layout["send_rows"][0], ROW_WORDS)
        sr = self._buf(self.send, 1, layout["send_rows"][1], ROW_WORDS)
        _lib.check(L.sphb_slab_scatter(g, n, nb, _ptr(a.key), _ptr(a.id), x0, x1, _ptr(self.tiles),
                                       _ptr(a.posp), _ptr(a.velr), _ptr(a.prev), kb, _ptr(b.posp),
                                       _ptr(b.velr), _ptr(b.prev), _ptr(b.id), _ptr(b.key), _ptr(sl),
                                       _ptr(sr), sec, s), "sphb_slab_scatter")

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

    def settled(self):
        """After a re-layout: histogram of the carried keys, no previous sort order."""
        self.ws.reset()
        _lib.check(_lib.lib().sphb_cell_hist(self.ws.handle, _lib.ref(self.grid), _ptr(self.a.key),
                                             self.n, _ptr(self.ctrl), _stream()), "sphb_cell_hist")

    # -------------------------------------------------------------- views
    def live_mask(self):
        """Rows of the primary arrays that are this rank's own particles (not halo, not dead)."""
        k = self.a.key[: self.n].to(torch.int64) & 0xFFFFFFFF
        return (self.a.id[: self.n] >= 0) & (k != self.dead)

    def is_fluid(self):
        k = self.a.key[: self.n].to(torch.int64) & 0xFFFFFFFF
        return ((k >> self.cellbits) & 1) == 1


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


def band_recv_rows(tab, r, nranks):
    """Band rows rank r receives (left, right) from the all-gathered per-rank
    (band rows to the left, band rows to the right) table."""
    return (int(tab[r - 1][1]) if r > 0 else 0, int(tab[r + 1][0]) if r < nranks - 1 else 0)


# ------------------------------------------------------------------ the stepper
class DeviceSlabSim:
    """X-slab stepper of the local ranks of ``comm`` (all on this process's current device)."""

    def __init__(self, system, params, comm, reach: int | None = None, precision: int = 0,
                 bounds=None, order: int = 0, rebalance_every: int = 0):
        if getattr(params, "integrator", "verlet") != "verlet":
            raise ValueError("DeviceSlabSim integrates with the Verlet scheme only")
        bf = getattr(params, "boundary_force", None)
        if bf is not None and float(getattr(bf, "d", 0.0)) > 0.0:
            raise ValueError("DeviceSlabSim does not apply the repulsive boundary force extension")
        self.params = params
        self.rebalance_every = int(rebalance_every)
        self.comm = comm
        self.reach = int(params.n_subdiv if reach is None else reach)
        cs, dims = grid_dims(params)
        nx = int(dims[0])
        # slabs at least one band wide (reach + 1 columns): a band row can only reach the
        # neighbouring slab
        self.min_width = self.reach + 1
        pos = torch.as_tensor(np.ascontiguousarray(system.pos, np.float32))
        col = columns_of(pos[:, 0], float(np.asarray(params.domain_min, np.float64)[0]), cs, nx).numpy()
        if bounds is None:
            bounds = balanced_bounds(np.bincount(col, minlength=nx), comm.nranks, self.min_width)
        self.bounds = np.asarray(bounds, np.int64)
        if comm.nranks > 1 and np.any(np.diff(self.bounds) < self.min_width):
            raise ValueError(f"slabs must be at least reach + 1 = {self.min_width} columns wide")
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
            r = DevRank(k, comm.nranks, (x0, x1), params, self.prm, self.reach, dev,
                        int(idx.size * 1.2) + 1024)
            t = lambda v: torch.as_tensor(np.ascontiguousarray(v)).to(dev)  # noqa: E731
            r.upload(t(system.pos[idx]), t(system.vel[idx]), t(system.rho[idx]),
                     t(np.asarray(system.id)[idx].astype(np.int64)), ib.size)
            self.ranks.append(r)
        self.step_index = 0
        self._settled = False

    # -------------------------------------------------------------- re-layout
    def _relayout(self):
        """One re-layout exchange round (counts already computed); returns the totals table."""
        gathered = self.comm.allgather([r.status_words() for r in self.ranks])
        tab = gathered[0].cpu().numpy()
        self._raise_errors(tab[:, NCAT])
        tots = tab[:, :NCAT]
        items, layouts = [], []
        for r in self.ranks:
            lay = rank_layout(tots, r.rank, self.comm.nranks)
            r._grow(max(lay["n_next"], r.n))
            r.scatter(lay)
            rl = r._buf(r.recv, 0, lay["recv_rows"][0], ROW_WORDS)
            rr = r._buf(r.recv, 1, lay["recv_rows"][1], ROW_WORDS)
            items.append(dict(send_l=(r.send[0], lay["send_rows"][0]), send_r=(r.send[1], lay["send_rows"][1]),
                              recv_l=(rl, lay["recv_rows"][0]), recv_r=(rr, lay["recv_rows"][1])))
            layouts.append(lay)
        self.comm.sendrecv(items)
        for r, lay in zip(self.ranks, layouts):
            r.unpack(lay)
        return tots

    def _settle(self, fresh_keys: bool):
        """Re-layout rounds until no particle sits outside its slab (a bound can move several
        slabs' worth of columns; each round is one neighbour hop); the last round rebuilds the
        halos.  The next step sorts from scratch."""
        for k in range(self.comm.nranks + 1):
            for r in self.ranks:
                r.count_resident(fresh_keys and k == 0)
            tots = self._relayout()
            if not np.any(tots[:, MIGL_B:MIGR_F + 1]):
                break
        for r in self.ranks:
            r.settled()
        self._settled = True

    def _raise_errors(self, errs):
        errs = np.asarray(errs).astype(np.uint64)
        if np.any(errs != np.uint64(_lib.ERR_NONE)):
            k = int(np.argmax(errs != np.uint64(_lib.ERR_NONE)))
            raise RuntimeError(f"slab rank {k} diverged: {decode_err(errs[k])}")

    def prime(self):
        """Initial halos: the re-layout exchange of the uploaded owned rows (keys from K1)."""
        self._settle(fresh_keys=True)

    def set_bounds(self, bounds):
        """Move the slab bounds and re-settle the rows (multi-hop re-layout)."""
        bounds = np.asarray(bounds, np.int64)
        if self.comm.nranks > 1 and np.any(np.diff(bounds) < self.min_width):
            raise ValueError(f"slabs must be at least reach + 1 = {self.min_width} columns wide")
        self.bounds = bounds
        for r in self.ranks:
            r.set_bounds((int(bounds[r.rank]), int(bounds[r.rank + 1])))
        self._settle(fresh_keys=False)

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

    def rebalance(self, times=None):
        """Equal-time slab bounds (slab.rebalance_slices, the reference's balance.py:53-88
        restated) from the measured (or given) per-rank interaction times."""
        t = self.measured_pi_ms() if times is None else np.asarray(times, np.float64)
        new = enforce_min_width(rebalance_slices(self.bounds, t), self.min_width)
        if not np.array_equal(new, self.bounds):
            self.set_bounds(new)
        return new

    # -------------------------------------------------------------- the step
    def step(self):
        if not self._settled:
            self.prime()
        if self.rebalance_every and self.step_index and self.step_index % self.rebalance_every == 0:
            self.rebalance()
        ranks, n = self.ranks, self.comm.nranks
        for r in ranks:
            r.phase_edges()
        # the step's host read, while the GPU runs the edge interaction: live / boundary rows,
        # band sizes and the error word of every rank
        mine = [np.concatenate([r.read_info()[[2, 3, 4]]]) for r in ranks]
        tab = self.comm.host_allgather(mine)
        self._raise_errors(tab[:, 2])
        items, recv_rows = [], []
        peer = getattr(self.comm, "transport", None) == "peer" and n > 1
        tag = None
        if peer:  # every rank sees the same table: the same capacity decision
            self.comm.ensure_capacity(int(tab[:, :2].max()))
            tag = self.comm.next_tag()
        for r in ranks:
            rows = band_recv_rows(tab, r.rank, n)
            recv_rows.append(rows)
            n_next = r.n_live + rows[0] + rows[1]
            if n_next > r.cap:
                r._grow_mid_step(n_next)
            if peer:
                r.phase_put(self.comm, tag)
                continue
            r.phase_pack()
            rl = r._buf(r.recv, 0, rows[0], BAND_WORDS)
            rr = r._buf(r.recv, 1, rows[1], BAND_WORDS)
            items.append(dict(send_l=(r.send[0], r.band_rows[0]), send_r=(r.send[1], r.band_rows[1]),
                              recv_l=(rl, rows[0]), recv_r=(rr, rows[1])))
        if peer:
            done = [None] * len(ranks)
        else:
            done = self.comm.band_sendrecv(items, [r.pack_ev for r in ranks]) if n > 1 else [None] * len(ranks)
        for r in ranks:
            r.phase_interior()
        # the step's dt is global (min over ranks); the counters stay per rank in each rank's
        # record ring and are summed over ranks only when read (records())
        self.comm.allreduce([r.dt_words() for r in ranks], "min")
        for r, rows, ev in zip(ranks, recv_rows, done):
            r.phase_update(rows, ev, (self.comm, tag) if peer else None)
        self.step_index += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()
        self.check()

    def check(self):
        """Raise if any local rank recorded an error (the steps read it one step late)."""
        self._raise_errors([int(read_ctrl(r.ctrl)["err"]) for r in self.ranks])

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
            n = r.n
            own = r.live_mask().cpu().numpy()
            pos.append(r.a.posp[:n, :3].cpu().numpy()[own])
            vel.append(r.a.velr[:n, :3].cpu().numpy()[own])
            rho.append(r.a.velr[:n, 3].cpu().numpy()[own])
            ids.append(r.a.id[:n].cpu().numpy()[own])
            fl.append(r.is_fluid().cpu().numpy()[own])
        pos, vel, rho, ids, fl = (np.concatenate(v) for v in (pos, vel, rho, ids, fl))
        o = np.argsort(ids)
        return pos[o], vel[o], rho[o], ids[o], fl[o]

    @property
    def n_owned_max(self) -> int:
        return max(int(r.live_mask().sum().item()) for r in self.ranks)

    def choose_pi_block(self, large_min) -> list[int]:
        """Per rank, run_simulation's rule: 384-target blocks when the rank owns at least
        ``large_min`` targets, else 256; 128 when ``large_min`` is None (h/2 cells); returns
        each local rank's blocking."""
        out = []
        for r in self.ranks:
            owned = int(r.live_mask().sum().item())
            blk = 128 if large_min is None else 384 if owned >= large_min else 256
            r.pi_block = blk
            r.ws.set_pi_block(blk)
            out.append(blk)
        return out

    def select_pi(self, kernel: str, block: int):
        """One FP32 interaction build on every local rank (DeviceSim.select_pi's choices)."""
        if kernel not in ("gather", "paired"):
            raise ValueError("X slabs run the gather kernels (gather, paired): the symmetric "
                             "kernel scatters reactions into halo rows")
        code = {"gather": _lib.SPHB_PI_GATHER, "paired": _lib.SPHB_PI_PAIRED}[kernel]
        blk = {"paired": 512}.get(kernel, block)
        for r in self.ranks:
            r.pi_kernel, r.pi_block = code, blk
            r.ws.set_pi_kernel(code)
            r.ws.set_pi_block(blk)

    def tune_pi(self, candidates) -> list[dict]:
        """DeviceSim.tune_pi per rank: one ordinary step with each candidate build ((kernel,
        block) pairs; the state advances as usual), the fastest interaction phase per local
        rank kept (ranks may differ: a slab at rest and one holding the collapsing column).
        Returns each local rank's {"kernel/block": PI ms}."""
        times = []
        for kern, blk in candidates:
            self.select_pi(kern, blk)
            self.step()
            torch.cuda.synchronize()
            times.append([r.pi_events[-1][0].elapsed_time(r.pi_events[-1][1]) for r in self.ranks])
        out = []
        for k, r in enumerate(self.ranks):
            ms = [t[k] for t in times]
            kern, blk = candidates[int(np.argmin(ms))]
            code = {"gather": _lib.SPHB_PI_GATHER, "paired": _lib.SPHB_PI_PAIRED}[kern]
            r.pi_kernel, r.pi_block = code, (512 if kern == "paired" else blk)
            r.ws.set_pi_kernel(r.pi_kernel)
            r.ws.set_pi_block(r.pi_block)
            out.append({f"{c[0]}/{c[1]}": round(t, 4) for c, t in zip(candidates, ms)})
        return out

    def launches_per_step(self) -> int:
        """This library's kernel launches per step on rank 0 (NL, band count, interaction
        launches, pack, K7, band updates, tail, step begin / end)."""
        r = self.ranks[0]
        base = int(_lib.lib().sphb_step_launch_count(_lib.ref(r.grid), r.n))
        npi = len(r.edge_grids) + len(r.inner_grids)
        # + band count (2); each further interaction launch: k_blocks x 3 + the kernel (+
        # k_cand_cells per launch at reach >= 2); pack, two band updates and the tail on a rank
        # with neighbours
        cand = npi if int(r.grid.reach) >= 2 else 0
        # (the slab stepper plans in line: no k_cand_take, which base counts from 2^19 rows)
        take = 1 if r.n >= 1 << 19 else 0
        return base - take + 2 + cand + 4 * (npi - 1) + (4 if r.sides else 0)


def estimate_steps_per_sync() -> int:
    """Host reads per step of DeviceSlabSim (the info words, read while the edge targets'
    interaction runs)."""
    return 1


def make_dist_comm(transport: str | None = None):
    """The production communicator: edge bands by peer-memory stores (DevPeerComm) unless
    ``transport`` (or $SPHB_SLAB_TRANSPORT) is "nccl"; falls back to NCCL send/recv when the
    peer mappings cannot be set up on every rank (decided collectively)."""
    import os
    import torch.distributed as dist
    want = transport or os.environ.get("SPHB_SLAB_TRANSPORT", "peer")
    if want == "peer" and dist.get_world_size() > 1:
        ok, err = True, None
        try:
            comm = DevPeerComm()
        except Exception as e:  # noqa: BLE001 -- IPC / P2P unavailable on this box
            ok, err, comm = False, e, None
        flags = [None] * dist.get_world_size()
        dist.all_gather_object(flags, ok)
        if all(flags):
            return comm
        print(f"[dslab] peer-memory band transport unavailable ({err}); using NCCL send/recv",
              flush=True)
    return DevDistComm()


__all__ = ["DeviceSlabSim", "DevLoopbackComm", "DevDistComm", "DevPeerComm", "make_dist_comm",
           "rank_layout", "band_recv_rows"]
