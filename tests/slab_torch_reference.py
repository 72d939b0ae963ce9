"""Torch restatement (test infrastructure) of the X-slab domain decomposition of the SPH step over several GPUs.

The global cell grid is cut along x into slabs of whole cell columns [x0_k, x1_k), one per
rank (the reference's Slices geometry, engines/kernels.py:230-323, balance.py:46-88, but with
counts/time-balanced bounds).  Per step every rank:

  1. classifies its owned particles by cell column (the exact f64 formula of assign_cells)
     and sends the ones that left its slab to the neighbour ranks (migration: full state
     incl. Verlet history and id);
  2. sends the particles of its ``reach`` edge columns to the neighbours as read-only halo
     (x, y, z, v, rho; derived quantities are recomputed by the receiver's K3);
  3. runs NL on owned + halo particles and the interaction for OWNED targets only (the
     kernels' target-column window [tx0, tx1)), so every pair a target needs is present;
  4. reduces the dt minima over ranks (allreduce MIN on the ordered-bit words of the device
     control block: no host round trip) before the Verlet update;
  5. drops the halo copies.

The exchange is plumbing in torch: `DistComm` uses torch.distributed send/recv (NCCL over
NVLink between GPUs, gloo on CPU for tests), `LoopbackComm` runs k virtual slabs in one
process (device-local copies), which is how the decomposition is validated on one GPU.
Compute runs in a `LocalEngine`: `DeviceLocalEngine` drives libsphb200; the CPU tests plug
in an oracle-based engine.

State per rank, per list (0 = boundary, 1 = fluid): float32 rows
[x, y, z, vx, vy, vz, rho, vx_prev, vy_prev, vz_prev, rho_prev, 0] and int64 ids.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_1110_3711_b200.slab import balanced_bounds, columns_of, enforce_min_width, rebalance_slices  # noqa: F401

NCOL = 12  # state columns
X, Y, Z, VX, VY, VZ, RHO, PVX, PVY, PVZ, PRHO = range(11)


# ------------------------------------------------------------------ communicators
class LoopbackComm:
    """k virtual slab ranks inside one process (exchanges are local copies)."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.local_ranks = list(range(nranks))

    def exchange(self, payloads):
        """payloads[r] = {'left': [t...], 'right': [t...]} -> received[r] = {'left', 'right'}."""
        n = self.nranks
        recv = [{"left": None, "right": None} for _ in range(n)]
        for r in range(n):
            if r > 0:
                recv[r]["left"] = [t.clone() for t in payloads[r - 1]["right"]]
            if r < n - 1:
                recv[r]["right"] = [t.clone() for t in payloads[r + 1]["left"]]
        return recv

    def allreduce(self, tensors, op: str):
        stacked = torch.stack(tensors)
        red = {"min": lambda t: t.min(0).values, "max": lambda t: t.max(0).values,
               "sum": lambda t: t.sum(0)}[op](stacked)
        for t in tensors:
            t.copy_(red)


class DistComm:
    """One rank per process over torch.distributed (NCCL between GPUs, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self.local_ranks = [self.rank]

    def exchange(self, payloads):
        dist = self.dist
        pay = payloads[0]
        r, n = self.rank, self.nranks
        out = {"left": None, "right": None}
        peers = [("left", r - 1), ("right", r + 1)]
        peers = [(side, p) for side, p in peers if 0 <= p < n]
        dev = pay["left"][0].device if pay["left"] else pay["right"][0].device
        # 1) shapes (leading dims) of every tensor, 2) payload
        meta_send, meta_recv = {}, {}
        for side, _ in peers:
            meta_send[side] = torch.tensor([t.shape[0] for t in pay[side]], dtype=torch.int64,
                                           device=dev)
            meta_recv[side] = torch.empty_like(meta_send[side])
        ops = []
        for side, p in peers:
            ops.append(dist.P2POp(dist.isend, meta_send[side], p))
            ops.append(dist.P2POp(dist.irecv, meta_recv[side], p))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        ops, bufs = [], {}
        for side, p in peers:
            shapes = meta_recv[side].tolist()
            tmpl = pay[side]
            bufs[side] = [torch.empty((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
                          for m, t in zip(shapes, tmpl)]
            for t in pay[side]:
                if t.shape[0]:
                    ops.append(dist.P2POp(dist.isend, t.contiguous(), p))
            for b in bufs[side]:
                if b.shape[0]:
                    ops.append(dist.P2POp(dist.irecv, b, p))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for side, _ in peers:
            out[side] = bufs[side]
        return [out]

    def allreduce(self, tensors, op: str):
        dist = self.dist
        rop = {"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op]
        dist.all_reduce(tensors[0], op=rop)


# ------------------------------------------------------------------ per-rank state
@dataclass
class RankState:
    rank: int
    bounds: tuple            # owned cell columns [x0, x1)
    st: list                 # [boundary (n_b, 12) f32, fluid (n_f, 12) f32]
    ids: list                # [boundary (n_b,) i64, fluid (n_f,) i64]
    engine: object = None
    stats: list = field(default_factory=list)

    @property
    def n_owned(self):
        return int(self.st[0].shape[0] + self.st[1].shape[0])


def split_system(system, layout_bounds, params, device_of):
    """Distribute a host ParticleSystem over slabs by cell column (initial state)."""
    from paper_1110_3711_b200.physics import grid_dims
    cs, dims = grid_dims(params)
    nb = system.count_boundary
    pos = torch.as_tensor(np.ascontiguousarray(system.pos, np.float32))
    col = columns_of(pos[:, 0], float(params.domain_min[0]), cs, int(dims[0])).numpy()
    full = np.zeros((system.n, NCOL), np.float32)
    full[:, 0:3] = system.pos
    full[:, 3:6] = system.vel
    full[:, 6] = system.rho
    full[:, 7:10] = system.vel
    full[:, 10] = system.rho
    ranks = []
    for k in range(len(layout_bounds) - 1):
        x0, x1 = int(layout_bounds[k]), int(layout_bounds[k + 1])
        sel = (col >= x0) & (col < x1)
        lists, ids = [], []
        for lo, hi in ((0, nb), (nb, system.n)):
            m = np.nonzero(sel[lo:hi])[0] + lo
            lists.append(torch.as_tensor(full[m]).to(device_of(k)))
            ids.append(torch.as_tensor(np.asarray(system.id)[m].astype(np.int64)).to(device_of(k)))
        ranks.append(RankState(rank=k, bounds=(x0, x1), st=lists, ids=ids))
    return ranks


# ------------------------------------------------------------------ the decomposed stepper
class SlabSimulation:
    """Drives the slabs of ``comm.local_ranks``; every rank object must share the same
    global grid (params) and slab bounds."""

    def __init__(self, ranks, params, comm, reach: int, make_engine):
        from paper_1110_3711_b200.physics import grid_dims
        self.ranks = ranks
        self.params = params
        self.comm = comm
        self.reach = int(reach)
        self.cs, dims = grid_dims(params)
        self.nx = int(dims[0])
        self.ox = float(np.asarray(params.domain_min, np.float64)[0])
        for r in ranks:
            r.engine = make_engine(r)
        self.step_index = 0
        self.t_sim = 0.0

    # -------------------------------------------------------------- exchange phases
    def _cols(self, st):
        return columns_of(st[:, X], self.ox, self.cs, self.nx)

    def migrate(self):
        """Move particles whose column left the slab to the neighbour rank (repeats until no
        rank holds a foreign particle, so large rebalancing moves also settle)."""
        for _ in range(self.comm.nranks):
            payloads, keep_masks, moved = [], [], torch.zeros(1, dtype=torch.int64)
            total = []
            for r in self.ranks:
                x0, x1 = r.bounds
                pl = {"left": [], "right": []}
                keeps = []
                cnt = 0
                for li in (0, 1):
                    c = self._cols(r.st[li])
                    left, right = c < x0, c >= x1
                    keeps.append(~(left | right))
                    pl["left"] += [r.st[li][left], r.ids[li][left]]
                    pl["right"] += [r.st[li][right], r.ids[li][right]]
                    cnt += int(left.sum()) + int(right.sum())
                payloads.append(pl)
                keep_masks.append(keeps)
                total.append(torch.tensor([cnt], dtype=torch.int64,
                                          device=r.st[0].device))
            self.comm.allreduce(total, "sum")
            if int(total[0].item()) == 0:
                return
            recv = self.comm.exchange(payloads)
            for r, keeps, rc in zip(self.ranks, keep_masks, recv):
                for li in (0, 1):
                    parts = [r.st[li][keeps[li]]]
                    idparts = [r.ids[li][keeps[li]]]
                    for side in ("left", "right"):
                        if rc[side] is not None:
                            parts.append(rc[side][2 * li])
                            idparts.append(rc[side][2 * li + 1])
                    r.st[li] = torch.cat(parts)
                    r.ids[li] = torch.cat(idparts)

    def halos(self):
        """Per rank: [boundary, fluid] halo rows received from the neighbours (read-only)."""
        R = self.reach
        payloads = []
        for r in self.ranks:
            x0, x1 = r.bounds
            pl = {"left": [], "right": []}
            for li in (0, 1):
                c = self._cols(r.st[li])
                pl["left"] += [r.st[li][c < x0 + R], r.ids[li][c < x0 + R]]
                pl["right"] += [r.st[li][c >= x1 - R], r.ids[li][c >= x1 - R]]
            payloads.append(pl)
        recv = self.comm.exchange(payloads)
        out = []
        for r, rc in zip(self.ranks, recv):
            lists, ids = [], []
            for li in (0, 1):
                parts, idp = [], []
                for side in ("left", "right"):
                    if rc[side] is not None:
                        parts.append(rc[side][2 * li])
                        idp.append(rc[side][2 * li + 1])
                dev = r.st[li].device
                lists.append(torch.cat(parts) if parts else torch.zeros((0, NCOL), device=dev))
                ids.append(torch.cat(idp) if idp else torch.zeros(0, dtype=torch.int64, device=dev))
            out.append((lists, ids))
        return out

    # -------------------------------------------------------------- one step
    def step(self):
        self.migrate()
        hal = self.halos()
        for r, (hst, hid) in zip(self.ranks, hal):
            nbo = r.st[0].shape[0]
            st = torch.cat([r.st[0], hst[0], r.st[1], hst[1]])
            # halo rows carry id = -1 - id so they can be dropped after the step
            ids = torch.cat([r.ids[0], -1 - hid[0], r.ids[1], -1 - hid[1]])
            nb_local = nbo + hst[0].shape[0]
            r.engine.nl_pi(st, ids, nb_local, r.bounds, self.step_index)
        parts = [r.engine.dt_words() for r in self.ranks]
        self.comm.allreduce(parts, "min")
        cnt = [r.engine.counter_words() for r in self.ranks]
        self.comm.allreduce(cnt, "sum")
        dts = []
        for r in self.ranks:
            st, ids, nb_local, rec = r.engine.su()
            keep = ids >= 0
            r.st = [st[:nb_local][keep[:nb_local]], st[nb_local:][keep[nb_local:]]]
            r.ids = [ids[:nb_local][keep[:nb_local]], ids[nb_local:][keep[nb_local:]]]
            r.stats.append(rec)
            dts.append(rec["dt"])
        self.step_index += 1
        self.t_sim += dts[0]
        return dts[0]

    def run(self, steps: int):
        for _ in range(steps):
            self.step()

    def gather_host(self):
        """All owned particles of the local ranks as host arrays (pos, vel, rho, id, ptype)."""
        pos, vel, rho, ids, ptype = [], [], [], [], []
        for r in self.ranks:
            for li in (0, 1):
                s = r.st[li].detach().cpu().numpy()
                pos.append(s[:, 0:3])
                vel.append(s[:, 3:6])
                rho.append(s[:, 6])
                ids.append(r.ids[li].detach().cpu().numpy())
                ptype.append(np.full(s.shape[0], li, np.uint8))
        return (np.concatenate(pos), np.concatenate(vel), np.concatenate(rho),
                np.concatenate(ids), np.concatenate(ptype))


# ------------------------------------------------------------------ device engine
class DeviceLocalEngine:
    """Runs one rank's local step with libsphb200 (NL over owned + halo, interaction for the
    owned columns only, Verlet after the cross-rank dt reduction)."""

    def __init__(self, params, mass_fluid, mass_boundary, reach=1, precision=0, order=0,
                 device=None):
        from paper_1110_3711_b200 import _lib
        from paper_1110_3711_b200.physics import grid_dims, params_desc
        self._lib = _lib
        self.device = torch.device(device or "cuda")
        self.params = params
        self.reach = reach
        self.prm = params_desc(params, mass_fluid, mass_boundary, order, precision)
        _, dims = grid_dims(params)
        self.dims = dims
        self.ncells = int(np.prod(dims))
        self.cap = 0
        self.ws = None
        self.ctrl = None
        self.rec = torch.zeros(64 * 40, dtype=torch.uint8, device=self.device)

    def _ensure(self, n):
        from paper_1110_3711_b200.device import Workspace, new_ctrl
        if n <= self.cap:
            return
        cap = int(n * 1.25) + 1024
        dev = self.device
        f4 = lambda: torch.zeros((cap, 4), dtype=torch.float32, device=dev)  # noqa: E731
        self.posp, self.velr, self.prev = f4(), f4(), f4()
        self.posp_s, self.velr_s, self.prev_s, self.aux = f4(), f4(), f4(), f4()
        self.id = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.id_s = torch.zeros_like(self.id)
        i32 = lambda m: torch.zeros(m, dtype=torch.int32, device=dev)  # noqa: E731
        self.keys, self.keys_sorted, self.perm, self.cell_s = i32(cap), i32(cap), i32(cap), i32(cap)
        # slab grids sort with a dead bin after the two lists (include/sphb200.h)
        self.beg, self.end = i32(2 * self.ncells + 1), i32(2 * self.ncells + 1)
        self.acc = torch.zeros((cap, 3), dtype=torch.float64, device=dev)
        self.drho = torch.zeros(cap, dtype=torch.float64, device=dev)
        self.visc = torch.zeros(cap, dtype=torch.float64, device=dev)
        self.ws = Workspace(cap, self.ncells)
        if self.ctrl is None:
            self.ctrl = new_ctrl(dev)
        self.cap = cap

    def nl_pi(self, st, ids, nb, cols, step_index):
        from paper_1110_3711_b200.device import _ptr, _stream
        from paper_1110_3711_b200.physics import grid_desc
        L, _lib = self._lib.lib(), self._lib
        n = int(st.shape[0])
        self._ensure(max(n, 1))
        self.n, self.nb = n, int(nb)
        self.posp[:n, :3] = st[:, 0:3]
        self.posp[:n, 3] = 0
        self.velr[:n, :3] = st[:, 3:6]
        self.velr[:n, 3] = st[:, 6]
        self.prev[:n, :3] = st[:, 7:10]
        self.prev[:n, 3] = st[:, 10]
        self.id[:n] = ids
        self.acc[:n].zero_()
        self.drho[:n].zero_()
        g = grid_desc(self.params, self.reach, target_cols=cols)
        self.grid = g
        s = _stream()
        c = self.ctrl.view(torch.int64)
        c[0] = step_index  # the control block's step counter (sphb_ctrl_t.step)
        ws = self.ws.handle
        self.ws.reset()
        rg, rp = _lib.ref(g), _lib.ref(self.prm)
        _lib.check(L.sphb_cell_keys(ws, rg, _ptr(self.posp), n, nb, _ptr(self.keys), None,
                                    _ptr(self.ctrl), s), "cell_keys")
        _lib.check(L.sphb_step_begin(_ptr(self.ctrl), s), "step_begin")
        _lib.check(L.sphb_sort(ws, rg, _ptr(self.keys), n, _ptr(self.keys_sorted), _ptr(self.perm),
                               _ptr(self.ctrl), s), "sort")
        _lib.check(L.sphb_reorder(rp, rg, n, _ptr(self.perm), _ptr(self.keys_sorted),
                                  _ptr(self.posp), _ptr(self.velr), _ptr(self.prev), _ptr(self.id),
                                  _ptr(self.posp_s), _ptr(self.velr_s), _ptr(self.prev_s),
                                  _ptr(self.id_s), _ptr(self.aux), _ptr(self.cell_s),
                                  _ptr(self.ctrl), s), "reorder")
        _lib.check(L.sphb_cell_ranges(ws, rg, _ptr(self.beg), _ptr(self.end), _ptr(self.ctrl), s),
                   "ranges")
        _lib.check(L.sphb_interact(ws, rp, rg, n, nb, _ptr(self.posp_s), _ptr(self.velr_s),
                                   _ptr(self.aux), _ptr(self.cell_s), _ptr(self.beg),
                                   _ptr(self.end), _ptr(self.acc), _ptr(self.drho),
                                   _ptr(self.visc), _ptr(self.ctrl), s), "interact")

    def dt_words(self):
        return self.ctrl.view(torch.int64)[5:7]   # dtmin_f, dtmin_cv (ordered bits)

    def counter_words(self):
        return self.ctrl.view(torch.int64)[8:12]

    def su(self):
        from paper_1110_3711_b200.device import _ptr, _stream, read_ctrl, decode_err
        L, _lib = self._lib.lib(), self._lib
        s = _stream()
        n, nb = self.n, self.nb
        _lib.check(L.sphb_integrate(self.ws.handle, _lib.ref(self.prm), _lib.ref(self.grid), n, nb,
                                    _ptr(self.posp_s), _ptr(self.velr_s), _ptr(self.prev_s),
                                    _ptr(self.id_s), _ptr(self.acc), _ptr(self.drho),
                                    _ptr(self.posp), _ptr(self.velr), _ptr(self.prev), _ptr(self.id),
                                    _ptr(self.keys), _ptr(self.ctrl), s), "integrate")
        _lib.check(L.sphb_step_end(_ptr(self.ctrl), _lib.ref(self.prm), _ptr(self.rec), 64, s),
                   "step_end")
        c = read_ctrl(self.ctrl)
        err = decode_err(c["err"])
        if err is not None:
            raise RuntimeError(f"slab rank divergence {err}")
        st = torch.empty((n, NCOL), dtype=torch.float32, device=self.device)
        st[:, 0:3] = self.posp[:n, :3]
        st[:, 3:6] = self.velr[:n, :3]
        st[:, 6] = self.velr[:n, 3]
        st[:, 7:10] = self.prev[:n, :3]
        st[:, 10] = self.prev[:n, 3]
        st[:, 11] = 0
        cnt = [int(v) for v in c["counters"]]
        rec = dict(dt=float(c["dt"]), candidate_pairs=cnt[0], true_pairs=cnt[1] // 2,
                   force_evals=cnt[2], ff_force_evals=cnt[3])
        return st, self.id[:n].clone(), nb, rec


def device_slab_simulation(system, params, nslabs: int, comm=None, reach: int | None = None,
                           precision=0, bounds=None):
    """Build a SlabSimulation on the GPU(s): ``comm`` None -> LoopbackComm (k virtual slabs on
    the current device); a DistComm -> one slab per process/GPU."""
    from paper_1110_3711_b200.physics import grid_dims
    reach = int(params.n_subdiv if reach is None else reach)
    cs, dims = grid_dims(params)
    if bounds is None:
        pos = torch.as_tensor(np.ascontiguousarray(system.pos, np.float32))
        col = columns_of(pos[:, 0], float(params.domain_min[0]), cs, int(dims[0])).numpy()
        counts = np.bincount(col, minlength=int(dims[0]))
        bounds = balanced_bounds(counts, nslabs, max(reach, 1))
    comm = comm or LoopbackComm(nslabs)
    dev = lambda k: torch.device("cuda", torch.cuda.current_device())  # noqa: E731
    ranks = split_system(system, bounds, params, dev)
    ranks = [ranks[k] for k in comm.local_ranks]
    mf, mb = float(system.mass_fluid), float(system.mass_boundary)
    sim = SlabSimulation(ranks, params, comm, reach,
                         lambda r: DeviceLocalEngine(params, mf, mb, reach, precision))
    sim.bounds = bounds
    return sim
