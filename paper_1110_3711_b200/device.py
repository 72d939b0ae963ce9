"""Device-resident SPH state and the step driver over libsphb200's C ABI.

PyTorch provides device memory, streams and CUDA graphs (plumbing); every FLOP of the
NL -> PI -> SU step runs in this package's own sm_100a kernels (csrc/).  Layout in HBM:
structure of float4 arrays (see include/sphb200.h); primary arrays hold the state in the
previous step's sorted order, *_s arrays the current step's sorted copies.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .physics import grid_desc, grid_dims, params_desc

F4 = 4


def _ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def cellbits_of(ncells: int) -> int:
    """Sort-key cell bits (sphb_common.cuh cellbits_of)."""
    b = 1
    while (1 << b) <= ncells:
        b += 1
    return b


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def require_cuda():
    if not torch.cuda.is_available():
        raise _lib.SphbError("paper_1110_3711_b200 needs a CUDA device (B200); no CPU fallback")
    _lib.lib()


class Workspace:
    """RAII wrapper of sphb_workspace_t (the only allocating C call)."""

    def __init__(self, n_max: int, ncells_max: int):
        self._h = ctypes.c_void_p()
        _lib.check(_lib.lib().sphb_workspace_create(int(n_max), int(ncells_max), ctypes.byref(self._h)),
                   "sphb_workspace_create")
        self.n_max, self.ncells_max = int(n_max), int(ncells_max)

    @property
    def handle(self):
        return self._h

    def bytes(self) -> int:
        return int(_lib.lib().sphb_workspace_bytes(self._h))

    def reset(self):
        _lib.check(_lib.lib().sphb_workspace_reset(self._h, _stream()), "sphb_workspace_reset")

    def set_mover_cap(self, cap: int):
        """Movers-only sort threshold of sphb_step (-1: always the radix sort)."""
        _lib.check(_lib.lib().sphb_workspace_set_mover_cap(self._h, int(cap)),
                   "sphb_workspace_set_mover_cap")

    def set_pi_block(self, targets: int):
        _lib.check(_lib.lib().sphb_workspace_set_pi_block(self._h, int(targets)),
                   "sphb_workspace_set_pi_block")

    def set_pi_kernel(self, kernel: int):
        _lib.check(_lib.lib().sphb_workspace_set_pi_kernel(self._h, int(kernel)),
                   "sphb_workspace_set_pi_kernel")

    def sort_info(self) -> tuple[int, int]:
        """(movers, mode) of the last sphb_step sort; mode 0 movers-only, 1 radix."""
        m, mode = ctypes.c_int64(), ctypes.c_int32()
        _lib.check(_lib.lib().sphb_workspace_sort_info(self._h, ctypes.byref(m), ctypes.byref(mode)),
                   "sphb_workspace_sort_info")
        return int(m.value), int(mode.value)

    def __del__(self):
        try:
            if self._h:
                _lib.lib().sphb_workspace_destroy(self._h)
        except Exception:
            pass


def new_ctrl(device, max_steps: int = -1, t_end: float = math.inf) -> torch.Tensor:
    ctrl = torch.zeros(_lib.CTRL_BYTES, dtype=torch.uint8, device=device)  # pad bytes defined
    _lib.check(_lib.lib().sphb_ctrl_init(_ptr(ctrl), int(max_steps), float(t_end), _stream()),
               "sphb_ctrl_init")
    return ctrl


def read_ctrl(ctrl: torch.Tensor) -> np.void:
    host = ctrl.cpu().numpy()
    return host[: _lib.CTRL_DTYPE.itemsize].view(_lib.CTRL_DTYPE)[0]


def decode_err(err) -> tuple | None:
    err = int(err)
    if err == int(_lib.ERR_NONE):
        return None
    return (err >> 40, (err >> 32) & 0xFF, err & 0xFFFFFFFF)


class DeviceSim:
    """One particle system resident on the GPU, stepped by libsphb200.

    ``system`` may be this package's ParticleSystem or the reference's (duck typing).
    ``vel_prev``/``rho_prev`` seed the Verlet history (default: current state, as
    VerletState.from_system does, sim.py:40-43).
    """

    def __init__(self, system, params, reach: int, order: int = 0, precision: int = _lib.SPHB_FP32,
                 max_steps: int = -1, t_end: float = math.inf, record_capacity: int = 4096,
                 vel_prev=None, rho_prev=None, device=None, workspace: Workspace | None = None,
                 counters: int = 0):
        require_cuda()
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.params = params
        self.n = int(system.n)
        self.nb = int(system.count_boundary)
        self.mass_fluid = float(system.mass_fluid)
        self.mass_boundary = float(system.mass_boundary)
        self.grid = grid_desc(params, reach)
        self.prm = params_desc(params, self.mass_fluid, self.mass_boundary, order, precision,
                               counters)
        _, dims = grid_dims(params)
        self.ncells = int(np.prod(dims))
        n, dev = self.n, self.device
        f4 = lambda: torch.empty((max(n, 1), F4), dtype=torch.float32, device=dev)  # noqa: E731
        i32 = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=dev)  # noqa: E731
        self.posp, self.velr, self.prev = f4(), f4(), f4()
        self.posp_s, self.velr_s, self.prev_s, self.aux = f4(), f4(), f4(), f4()
        self.id = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.id_s = torch.empty_like(self.id)
        self.keys, self.keys_sorted, self.perm, self.cell_s = i32(n), i32(n), i32(n), i32(n)
        self.beg, self.end = i32(2 * self.ncells), i32(2 * self.ncells)
        self.acc = torch.zeros((max(n, 1), 3), dtype=torch.float64, device=dev)
        self.drho = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self.visc = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self.rec_cap = int(record_capacity)
        self.rec = torch.zeros(self.rec_cap * _lib.REC_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.ws = workspace if workspace is not None else Workspace(n, self.ncells)
        self.ws.reset()
        self.upload(system, vel_prev, rho_prev)
        self.ctrl = new_ctrl(dev, max_steps, t_end)
        self._make_state()
        self.first_keys()
        self._graph = None
        self._graph_steps = 0
        self.pi_block = 128
        self.pi_kernel = "gather"
        self.tuning = None  # the last tune_pi result

    def _make_state(self):
        """The sphb_step descriptor of the current buffers (rebuilt when the id buffers swap)."""
        self._state = _lib.StateDesc(*[_ptr(t) for t in (
            self.posp, self.velr, self.prev, self.id, self.posp_s, self.velr_s, self.prev_s,
            self.aux, self.id_s, self.keys, self.keys_sorted, self.perm, self.cell_s, self.beg,
            self.end, self.acc, self.drho, self.visc)])

    def set_pi_kernel(self, kernel: str):
        """FP32 interaction kernel: "gather" (one-sided, K6 dt in its epilogue) or "symmetric"
        (each unordered pair once, reactions scattered: sphb_workspace_set_pi_kernel).  Drops a
        captured graph."""
        code = {"gather": _lib.SPHB_PI_GATHER, "symmetric": _lib.SPHB_PI_SYMMETRIC,
                "paired": _lib.SPHB_PI_PAIRED}[kernel]
        self.ws.set_pi_kernel(code)
        self.pi_kernel = kernel
        if kernel == "symmetric":  # the symmetric build's blocking (pi384s)
            self.ws.set_pi_block(384)
            self.pi_block = 384
        elif kernel == "paired":  # two targets per lane: 512-target bricks (pi512p)
            self.ws.set_pi_block(512)
            self.pi_block = 512
        self._graph = None

    def select_pi(self, kernel: str, block: int):
        """One FP32 interaction build: ``kernel`` ("gather", "symmetric", "paired") with the
        gather kernel's ``block`` (the other two carry their own blocking)."""
        self.set_pi_kernel(kernel)
        if kernel == "gather":
            self.set_pi_block(block)

    def pi_candidates(self, n_subdiv: int = 1) -> list[tuple[str, int]]:
        """The builds the "tuned" policy times against each other: the gather kernel with the
        size rule's blocking (sim.initial_pi_block; small systems also 384), and the paired kernel
        (two targets per lane, 512-target bricks).  At rest the paired build is the faster one; once cells fill unevenly
        (a collapsed column) its bricks leave more lanes idle and the row blocks win."""
        from .sim import initial_pi_block
        first = initial_pi_block(self.n, n_subdiv)
        # small systems (a few blocks per SM: per-block latency, not lane use, decides) also
        # try the 384-target blocks (C1: 0.10 vs 0.12 ms PI with 256)
        extra = [("gather", 384)] if first != 384 else []
        return [("gather", first)] + extra + [("paired", 512)]

    def tune_pi(self, candidates, events=None, repeats: int | None = None) -> dict:
        """Run ordinary steps with each candidate build (the state advances as usual), time
        each step's PI stage with CUDA events and keep the fastest build.  The first tuning of
        a simulation runs every candidate twice and decides on the second round: a kernel's
        first launch in a process carries its one-time module load (lazy loading), which must
        not decide the choice.  ``events``: the per-step event lists of the deciding round
        (launch_step's layout), else fresh ones.  Returns {"kernel/block": PI ms};
        ``self.tuning_steps`` is the number of steps it ran."""
        reps = (2 if self.tuning is None else 1) if repeats is None else int(repeats)
        for _ in range(reps - 1):  # untimed warm round
            for kern, blk in candidates:
                self.select_pi(kern, blk)
                self.launch_step()
        evs = events if events is not None else [
            [torch.cuda.Event(enable_timing=True) for _ in range(self.n_stage_events())]
            for _ in candidates]
        for (kern, blk), ev in zip(candidates, evs):
            self.select_pi(kern, blk)
            self.launch_step(events=ev)
        torch.cuda.synchronize()
        self.tuning_steps = reps * len(candidates)
        return self.tune_choose(candidates, evs)

    def tune_choose(self, candidates, events) -> dict:
        """The selection half of tune_pi, for steps already launched with ``events`` (one per
        candidate, in order) and completed."""
        ms = [DeviceSim.stage_seconds(ev)[1] * 1e3 for ev in events]
        best = int(np.argmin(ms))
        self.select_pi(*candidates[best])
        self.tuning = {f"{k}/{b}": round(t, 4) for (k, b), t in zip(candidates, ms)}
        return self.tuning

    def set_pi_block(self, targets: int):
        """Targets per FP32 interaction block: 128 (4-warp CTAs, the default), 256 (8-warp CTAs)
        or 384 (12-warp CTAs, one per SM: more resident warps, fewer idle lanes when cells hold
        uneven counts); sim.initial_pi_block is the run policy.  Drops a captured graph."""
        self.ws.set_pi_block(targets)
        self.pi_block = int(targets)
        self._graph = None

    def pi_lane_use(self, ctrl=None) -> float:
        """Targets / (blocks x block size) of the last interaction launch."""
        c = self.ctrl_host() if ctrl is None else ctrl
        nblk = int(c["nblk"][0])
        return self.n / (self.pi_block * nblk) if nblk else 1.0

    # ------------------------------------------------------------------ host <-> device
    def upload(self, system, vel_prev=None, rho_prev=None, stream_copy=True):
        n = self.n
        if n == 0:
            return
        pos = torch.as_tensor(np.ascontiguousarray(system.pos, np.float32))
        vel = torch.as_tensor(np.ascontiguousarray(system.vel, np.float32))
        rho = torch.as_tensor(np.ascontiguousarray(system.rho, np.float32))
        vp = vel if vel_prev is None else torch.as_tensor(np.ascontiguousarray(vel_prev, np.float32))
        rp = rho if rho_prev is None else torch.as_tensor(np.ascontiguousarray(rho_prev, np.float32))
        host = torch.empty((3, n, 4), dtype=torch.float32, pin_memory=True)
        host[0, :, :3] = pos
        host[0, :, 3] = 0.0
        host[1, :, :3] = vel
        host[1, :, 3] = rho
        host[2, :, :3] = vp
        host[2, :, 3] = rp
        self.posp[:n].copy_(host[0], non_blocking=True)
        self.velr[:n].copy_(host[1], non_blocking=True)
        self.prev[:n].copy_(host[2], non_blocking=True)
        self.id[:n].copy_(torch.as_tensor(np.ascontiguousarray(system.id, np.int64)), non_blocking=False)

    def download(self):
        """(pos, vel, rho, id, vel_prev, rho_prev) of the primary arrays as numpy."""
        n = self.n
        p = self.posp[:n].cpu().numpy()
        v = self.velr[:n].cpu().numpy()
        pv = self.prev[:n].cpu().numpy()
        ids = self.id[:n].cpu().numpy()
        return (np.ascontiguousarray(p[:, :3]), np.ascontiguousarray(v[:, :3]),
                np.ascontiguousarray(v[:, 3]), ids, np.ascontiguousarray(pv[:, :3]),
                np.ascontiguousarray(pv[:, 3]))

    # ------------------------------------------------------------------ kernels
    def first_keys(self):
        """K1 on the uploaded state (later steps get their keys from K7)."""
        L = _lib.lib()
        _lib.check(L.sphb_cell_keys(self.ws.handle, _lib.ref(self.grid), _ptr(self.posp), self.n,
                                    self.nb, _ptr(self.keys), None, _ptr(self.ctrl), _stream()),
                   "sphb_cell_keys")

    def first_keys_resync(self, keep_order: bool = False):
        """K1 for a state written from outside (host upload): histogram reset + keys.
        keep_order: the upload replaced the same n rows (e.g. the reference-layout round trip
        of sphb_state_from_soa) -- the next sort may still take the movers-only path, which is
        the stable sort of the rows in any order (sphb_workspace_trust_order)."""
        if keep_order:
            _lib.check(_lib.lib().sphb_workspace_clear_hist(self.ws.handle, _stream()), "clear_hist")
            self.first_keys()
            _lib.check(_lib.lib().sphb_workspace_trust_order(self.ws.handle, _stream()), "trust_order")
        else:
            self.ws.reset()
            self.first_keys()

    @property
    def symplectic(self) -> bool:
        return int(self.prm.integrator) == _lib.SPHB_INT_SYMPLECTIC

    def n_stage_events(self) -> int:
        """Events launch_step records per step: 4 (verlet) or 7 (symplectic)."""
        return 7 if self.symplectic else 4

    def _stage(self, mode: int, ev):
        """NL -> PI -> system update ``mode`` (0 verlet, 1/2 symplectic stages); records
        ev[0] after NL, ev[1] after PI, ev[2] after the update."""
        L, s, ws = _lib.lib(), _stream(), self.ws.handle
        g, p, n, nb = _lib.ref(self.grid), _lib.ref(self.prm), self.n, self.nb
        # the FP32 gather / paired kernels recompute a target's derived row: no aux pass
        aux = self.aux if (int(self.prm.precision) == _lib.SPHB_FP64 or self.pi_kernel == "symmetric") \
            else None
        nvtx = torch.cuda.nvtx
        nvtx.range_push("sphb NL")
        _lib.check(L.sphb_sort_ranges(ws, g, _ptr(self.keys), n, _ptr(self.keys_sorted),
                                      _ptr(self.perm), _ptr(self.beg), _ptr(self.end),
                                      _ptr(self.ctrl), s), "sphb_sort_ranges")
        # the interaction's block list on the workspace's side stream while K3 runs
        _lib.check(L.sphb_interact_plan(ws, p, g, _ptr(self.beg), _ptr(self.end), _ptr(self.ctrl), s),
                   "sphb_interact_plan")
        _lib.check(L.sphb_reorder(p, g, n, _ptr(self.perm), _ptr(self.keys_sorted), _ptr(self.posp),
                                  _ptr(self.velr), _ptr(self.prev), _ptr(self.id), _ptr(self.posp_s),
                                  _ptr(self.velr_s), _ptr(self.prev_s), _ptr(self.id_s),
                                  _ptr(aux), _ptr(self.cell_s), _ptr(self.ctrl), s),
                   "sphb_reorder")
        ev[0].record()
        nvtx.range_pop()
        nvtx.range_push("sphb PI")
        _lib.check(L.sphb_interact(ws, p, g, n, nb, _ptr(self.posp_s), _ptr(self.velr_s),
                                   _ptr(aux), _ptr(self.cell_s), _ptr(self.beg),
                                   _ptr(self.end), _ptr(self.acc), _ptr(self.drho),
                                   _ptr(self.visc), _ptr(self.ctrl), s), "sphb_interact")
        ev[1].record()
        nvtx.range_pop()
        nvtx.range_push("sphb SU")
        args = (_ptr(self.posp_s), _ptr(self.velr_s), _ptr(self.prev_s), _ptr(self.id_s),
                _ptr(self.acc), _ptr(self.drho), _ptr(self.posp), _ptr(self.velr), _ptr(self.prev),
                _ptr(self.id), _ptr(self.keys), _ptr(self.ctrl), s)
        if mode == 0:
            _lib.check(L.sphb_integrate(ws, p, g, n, nb, *args), "sphb_integrate")
        else:
            _lib.check(L.sphb_integrate_stage(ws, p, g, n, nb, mode - 1, *args), "sphb_integrate_stage")
        ev[2].record()
        nvtx.range_pop()

    def launch_step(self, events=None):
        """Enqueue one step (no host sync).  ``events``: n_stage_events() CUDA events recorded
        at the stage boundaries (verlet: start | NL | PI | SU; symplectic: start, then
        NL | PI | SU of each of the two stages)."""
        L, s = _lib.lib(), _stream()
        p = _lib.ref(self.prm)
        if events is None:
            _lib.check(L.sphb_step(self.ws.handle, p, _lib.ref(self.grid), self.n, self.nb,
                                   _lib.ref(self._state), _ptr(self.ctrl), _ptr(self.rec),
                                   self.rec_cap, s), "sphb_step")
            return
        events[0].record()
        _lib.check(L.sphb_step_begin(_ptr(self.ctrl), s), "sphb_step_begin")
        if self.symplectic:
            self._stage(1, events[1:4])
            self._stage(2, events[4:7])
        else:
            self._stage(0, events[1:4])
        _lib.check(L.sphb_step_end(_ptr(self.ctrl), p, _ptr(self.rec), self.rec_cap, s),
                   "sphb_step_end")
        events[-1].record()

    @staticmethod
    def stage_seconds(events) -> tuple[float, float, float, float]:
        """(nl, pi, su, wall) seconds of one step's events (launch_step order)."""
        ms = lambda a, b: a.elapsed_time(b)  # noqa: E731
        if len(events) == 4:
            e0, e1, e2, e3 = events
            return ms(e0, e1) * 1e-3, ms(e1, e2) * 1e-3, ms(e2, e3) * 1e-3, ms(e0, e3) * 1e-3
        e0, n1, p1, s1, n2, p2, s2 = events
        return ((ms(e0, n1) + ms(s1, n2)) * 1e-3, (ms(n1, p1) + ms(n2, p2)) * 1e-3,
                (ms(p1, s1) + ms(p2, s2)) * 1e-3, ms(e0, s2) * 1e-3)

    def capture(self, steps: int):
        """Capture ``steps`` whole steps into one CUDA graph (replayed by run_graph)."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(steps):
                self.launch_step()
        self._graph, self._graph_steps = g, steps
        return g

    def run_graph(self):
        self._graph.replay()

    def launches_per_step(self) -> int:
        k = int(_lib.lib().sphb_step_launch_count(_lib.ref(self.grid), self.n))
        if int(self.prm.precision) == _lib.SPHB_FP32:
            if self.pi_kernel == "symmetric":
                k += 1  # k_dt_f32 after the scatter
            elif int(self.grid.reach) >= 2:
                k += 1  # k_cand_cells (reach 1: the counter rides on k_blocks)
        if int(self.prm.counters) == _lib.SPHB_COUNTERS_SYMMETRIC:
            k += 2  # k_sym_cand, k_sym_final
        return k

    # ------------------------------------------------------------------ diagnostics
    def energy(self) -> dict:
        """sphb_energy on the primary state: KE, PE, IE (Tait), mean fluid rho, mean rho."""
        out = torch.zeros(5, dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().sphb_energy(self.ws.handle, _lib.ref(self.prm), self.n, self.nb,
                                          _ptr(self.posp), _ptr(self.velr), _ptr(out), _stream()),
                   "sphb_energy")
        v = out.cpu().numpy()
        return dict(ke=float(v[0]), pe=float(v[1]), ie=float(v[2]), rho_fluid=float(v[3]),
                    rho_mean=float(v[4]))

    # ------------------------------------------------------------------ checkpoints
    def save_checkpoint(self, path) -> None:
        from .snapshots import save_checkpoint
        torch.cuda.current_stream().synchronize()
        save_checkpoint(path, self)

    @classmethod
    def from_checkpoint(cls, path, params, reach: int, max_steps: int | None = None,
                        t_end: float | None = None, **kw) -> "DeviceSim":
        """Resume: state, Verlet history, step and simulated time from ``path``; the stop
        rules are the caller's (None keeps the checkpointed ones)."""
        from types import SimpleNamespace

        from .snapshots import load_checkpoint
        z = load_checkpoint(path)
        n, nb = int(z["n"]), int(z["nb"])
        posp, velr, prev = z["posp"], z["velr"], z["prev"]
        system = SimpleNamespace(n=n, count_boundary=nb, mass_fluid=float(z["mass_fluid"]),
                                 mass_boundary=float(z["mass_boundary"]), pos=posp[:, :3],
                                 vel=velr[:, :3], rho=velr[:, 3], id=z["id"])
        sim = cls(system, params, reach, vel_prev=prev[:, :3], rho_prev=prev[:, 3], **kw)
        c = z["ctrl"].copy()
        view = c[: _lib.CTRL_DTYPE.itemsize].view(_lib.CTRL_DTYPE)
        if max_steps is not None:
            view["max_steps"] = -1 if max_steps < 0 else int(max_steps)
        if t_end is not None:
            view["t_end"] = float(t_end)
        sim.ctrl.copy_(torch.as_tensor(c).to(sim.device))
        if "pi_block" in z:  # the interaction blocking in use when the checkpoint was written
            sim.set_pi_block(int(z["pi_block"]))
        if "pi_kernel" in z and str(z["pi_kernel"]) in ("symmetric", "paired"):
            sim.set_pi_kernel(str(z["pi_kernel"]))
        return sim

    # ------------------------------------------------------------------ readback
    def ctrl_host(self):
        return read_ctrl(self.ctrl)

    def records(self, first: int, last: int) -> np.ndarray:
        """Step records [first, last) (ring buffer of rec_cap entries)."""
        if last <= first:
            return np.zeros(0, _lib.REC_DTYPE)
        if last - first > self.rec_cap:
            raise ValueError("more steps than the record ring holds; read records more often")
        host = self.rec.cpu().numpy().view(_lib.REC_DTYPE)
        idx = np.arange(first, last) % self.rec_cap
        return host[idx]

    def forces(self, n: int | None = None):
        """The last interaction's ForceOutput arrays as f64 device tensors (acc (n, 3), drho,
        visc) in the current sorted order; FP32 layout widened by sphb_forces_f64."""
        n = self.n if n is None else int(n)
        dev = self.acc.device
        acc = torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev)
        drho = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        visc = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().sphb_forces_f64(_lib.ref(self.prm), n, _ptr(self.acc), _ptr(self.drho),
                                              _ptr(self.visc), _ptr(acc), _ptr(drho), _ptr(visc),
                                              _stream()), "sphb_forces_f64")
        return acc[:n], drho[:n], visc[:n]

    def error(self):
        """None or (step, code, index, particle_id)."""
        c = self.ctrl_host()
        d = decode_err(c["err"])
        if d is None:
            return None
        step, code, index = d
        stop = (int(c["max_steps"]) >= 0 and int(c["step"]) >= int(c["max_steps"])) or \
            float(c["t_sim"]) >= float(c["t_end"])
        if code == _lib.SPHB_DIV_LEFT_DOMAIN and step == int(c["step"]) and stop:
            # escaped during the final step: the stop rule ended the run before that step's
            # assign_cells would have seen it (sim.py:302-315), so the reference returns normally
            return None
        pid = int(self.id[index].item()) if code == _lib.SPHB_DIV_LEFT_DOMAIN else None
        return step, code, index, pid


def compute_derived_device(rho: np.ndarray, params):
    """press/csound/prrho/tensil of ``rho`` with the device EOS (the K3 code path)."""
    require_cuda()
    n = int(np.asarray(rho).shape[0])
    dev = torch.device("cuda")
    velr = torch.zeros((max(n, 1), 4), dtype=torch.float32, device=dev)
    if n:
        velr[:n, 3] = torch.as_tensor(np.ascontiguousarray(rho, np.float32)).to(dev)
    posp = torch.zeros_like(velr)
    posp_o, velr_o, aux = torch.empty_like(velr), torch.empty_like(velr), torch.empty_like(velr)
    prm = params_desc(params, 1.0, 1.0, precision=_lib.SPHB_FP64)  # the exact (pow) EOS
    g = grid_desc(params)
    ctrl = new_ctrl(dev)
    _lib.check(_lib.lib().sphb_reorder(_lib.ref(prm), _lib.ref(g), n, None, None, _ptr(posp),
                                       _ptr(velr), None, None, _ptr(posp_o), _ptr(velr_o), None,
                                       None, _ptr(aux), None, _ptr(ctrl), _stream()),
               "sphb_reorder")
    a = aux[:n].cpu().numpy()
    prrho = posp_o[:n, 3].cpu().numpy()
    return np.ascontiguousarray(a[:, 0]), np.ascontiguousarray(a[:, 1]), prrho, np.ascontiguousarray(a[:, 2])


def nl_frame(pos: np.ndarray, nb: int, params, reach: int | None = None):
    """Device NL on one frame: K1 -> K2 -> K4 (and K3's cell output).  Returns numpy
    (cell_of_unsorted int64, sort_perm int64, cell_of_sorted int64, fbeg, fend, bbeg, bend
    int64) -- the reference's assign_cells / reorder / build_cell_index outputs."""
    require_cuda()
    n = int(pos.shape[0])
    dev = torch.device("cuda")
    g = grid_desc(params, reach)
    _, dims = grid_dims(params)
    ncells = int(np.prod(dims))
    ws = Workspace(n, ncells)
    ws.reset()
    posp = torch.zeros((max(n, 1), 4), dtype=torch.float32, device=dev)
    if n:
        posp[:n, :3] = torch.as_tensor(np.ascontiguousarray(pos, np.float32)).to(dev)
    keys = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ksort = torch.empty_like(keys)
    perm = torch.empty_like(keys)
    cell = torch.empty_like(keys)
    beg = torch.empty(2 * ncells, dtype=torch.int32, device=dev)
    end = torch.empty_like(beg)
    ctrl = new_ctrl(dev)
    L, s = _lib.lib(), _stream()
    _lib.check(L.sphb_cell_keys(ws.handle, _lib.ref(g), _ptr(posp), n, nb, _ptr(keys), _ptr(cell),
                                _ptr(ctrl), s), "sphb_cell_keys")
    c = read_ctrl(ctrl)
    cell_unsorted = cell[:n].cpu().numpy().astype(np.int64)
    if decode_err(c["err"]) is not None:
        return dict(cell_of_unsorted=cell_unsorted, error=decode_err(c["err"]))
    _lib.check(L.sphb_sort(ws.handle, _lib.ref(g), _ptr(keys), n, _ptr(ksort), _ptr(perm),
                           _ptr(ctrl), s), "sphb_sort")
    _lib.check(L.sphb_cell_ranges(ws.handle, _lib.ref(g), _ptr(beg), _ptr(end), _ptr(ctrl), s),
               "sphb_cell_ranges")
    mask = (1 << cellbits_of(ncells)) - 1
    ks = ksort[:n].cpu().numpy().view(np.uint32).astype(np.int64) & mask
    b = beg.cpu().numpy().astype(np.int64)
    e = end.cpu().numpy().astype(np.int64)
    return dict(cell_of_unsorted=cell_unsorted, sort_perm=perm[:n].cpu().numpy().astype(np.int64),
                cell_of=ks, bbeg=b[:ncells], bend=e[:ncells], fbeg=b[ncells:], fend=e[ncells:],
                dims=dims, error=None)
