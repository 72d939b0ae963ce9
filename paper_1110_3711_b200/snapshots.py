"""Snapshot CSV files, the stats JSON-lines stream, snapshot comparison and binary checkpoints.

The text formats are the reference's (sphbench/bench/snapshots.py:1-62, 125-142): a
``id,type,x,y,z,vx,vy,vz,rho,press`` header and one ``%.9g`` row per particle (round-trips
float32 exactly), and one JSON object per step with the ``STATS_KEYS`` fields.  The writers
here are vectorised (a 10M-particle snapshot is formatted by numpy, not a Python loop) and
``DirSink`` formats on a background thread so the device keeps stepping while the CSV is
written (the reference's ``_DirSink``, bench/cli.py:174-181, writes synchronously).

Checkpoints (no reference counterpart) hold the device state in its
current sorted order *with* the Verlet history and the step / simulated time, so a resumed run
is bit-identical to an uninterrupted one (the reference restarts its history from the current
state, sim.py:40-43).
"""
from __future__ import annotations

import json
import os
import queue
import threading
from dataclasses import dataclass

import numpy as np

SNAPSHOT_HEADER = "id,type,x,y,z,vx,vy,vz,rho,press"
STATS_KEYS = ("step", "dt", "wall_s", "candidate_pairs", "true_pairs",
              "force_evals", "stage_nl_s", "stage_pi_s", "stage_su_s")
DEFAULT_TOLERANCES = {"pos": 1e-5, "vel": 1e-5, "rho": 1e-5, "press": 1e-4}
CHECKPOINT_MAGIC = "sphb200-checkpoint-v1"


@dataclass
class Snapshot:
    id: np.ndarray      # (n,) int64
    ptype: np.ndarray   # (n,) uint8
    pos: np.ndarray     # (n, 3) float32
    vel: np.ndarray     # (n, 3) float32
    rho: np.ndarray     # (n,) float32
    press: np.ndarray   # (n,) float32

    FIELDS = ("pos", "vel", "rho", "press")


def snapshot_of(system, derived) -> Snapshot:
    """snapshots.py:33-36."""
    return Snapshot(id=np.array(system.id, copy=True), ptype=np.array(system.ptype, copy=True),
                    pos=np.array(system.pos, copy=True), vel=np.array(system.vel, copy=True),
                    rho=np.array(system.rho, copy=True), press=np.array(derived.press, copy=True))


def format_snapshot(snap: Snapshot) -> str:
    """The CSV text write_snapshot produces (snapshots.py:39-48), built column-wise."""
    n = int(snap.id.shape[0])
    if n == 0:
        return SNAPSHOT_HEADER + "\n"
    cols = [snap.id.astype(np.int64).astype(str), snap.ptype.astype(np.int64).astype(str)]
    vals = np.column_stack([snap.pos.astype(np.float32), snap.vel.astype(np.float32),
                            snap.rho.astype(np.float32), snap.press.astype(np.float32)])
    # '%.9g' of the float32 value promoted to double, exactly as the reference's "%.9g" % v
    fmt = np.char.mod("%.9g", vals.astype(np.float64))
    cols += [fmt[:, k] for k in range(8)]
    rows = cols[0]
    for c in cols[1:]:
        rows = np.char.add(np.char.add(rows, ","), c)
    return SNAPSHOT_HEADER + "\n" + "\n".join(rows.tolist()) + "\n"


def write_snapshot(path, snap: Snapshot) -> None:
    with open(path, "w") as fh:
        fh.write(format_snapshot(snap))


def read_snapshot(path) -> Snapshot:
    """snapshots.py:51-62 (raises on a foreign header)."""
    with open(path) as fh:
        header = fh.readline().strip()
        if header != SNAPSHOT_HEADER:
            raise ValueError(f"unexpected snapshot header {header!r}")
        body = fh.read()
    if not body.strip():
        z = np.zeros(0, np.float32)
        return Snapshot(id=np.zeros(0, np.int64), ptype=np.zeros(0, np.uint8), pos=z.reshape(0, 3),
                        vel=z.reshape(0, 3), rho=z, press=z)
    rows = np.array([line.split(",") for line in body.splitlines() if line.strip()])
    data = rows[:, 2:].astype(np.float64).astype(np.float32)
    return Snapshot(id=rows[:, 0].astype(np.int64), ptype=rows[:, 1].astype(np.int64).astype(np.uint8),
                    pos=data[:, 0:3], vel=data[:, 3:6], rho=data[:, 6], press=data[:, 7])


@dataclass
class FieldDiff:
    field: str
    max_abs: float
    max_rel: float
    worst_id: int
    passed: bool


@dataclass
class CompareReport:
    fields: list
    passed: bool

    def worst(self) -> FieldDiff:
        return max(self.fields, key=lambda f: f.max_rel)

    def __str__(self) -> str:
        return "\n".join(f"{f.field:6s} max_abs={f.max_abs:.3e} max_rel={f.max_rel:.3e} "
                         f"worst_id={f.worst_id} {'ok' if f.passed else 'FAIL'}" for f in self.fields)


def compare_snapshots(a: Snapshot, b: Snapshot, tolerances: dict | None = None) -> CompareReport:
    """Per-field L-inf differences after aligning by id, scaled by the field's max magnitude
    (snapshots.py:89-122; same errors on count / id-set mismatch)."""
    tol = dict(DEFAULT_TOLERANCES)
    if tolerances:
        tol.update(tolerances)
    if a.id.shape[0] != b.id.shape[0]:
        raise ValueError("snapshot particle counts differ")
    oa, ob = np.argsort(a.id, kind="stable"), np.argsort(b.id, kind="stable")
    if not np.array_equal(a.id[oa], b.id[ob]):
        raise ValueError("snapshot id sets differ")
    ids = a.id[oa]
    fields = []
    for name in Snapshot.FIELDS:
        va = getattr(a, name)[oa].astype(np.float64)
        vb = getattr(b, name)[ob].astype(np.float64)
        diff = np.abs(va - vb)
        if diff.ndim > 1:
            diff = diff.max(axis=1)
        scale = max(np.abs(va).max(initial=0.0), np.abs(vb).max(initial=0.0), 1e-30)
        worst = int(np.argmax(diff)) if diff.size else 0
        max_abs = float(diff[worst]) if diff.size else 0.0
        fields.append(FieldDiff(field=name, max_abs=max_abs, max_rel=max_abs / scale,
                                worst_id=int(ids[worst]) if ids.size else -1,
                                passed=max_abs / scale <= tol[name]))
    return CompareReport(fields=fields, passed=all(f.passed for f in fields))


def stats_line(stats) -> str:
    """snapshots.py:125-137."""
    return json.dumps({"step": stats.step, "dt": stats.dt, "wall_s": stats.wall_seconds,
                       "candidate_pairs": stats.candidate_pairs, "true_pairs": stats.true_pairs,
                       "force_evals": stats.force_evals, "stage_nl_s": stats.stage_nl_s,
                       "stage_pi_s": stats.stage_pi_s, "stage_su_s": stats.stage_su_s})


def read_stats(path) -> list[dict]:
    with open(path) as fh:
        return [json.loads(line) for line in fh if line.strip()]


class DirSink:
    """run_simulation snapshot sink writing ``snapshot_{step:06d}.csv`` into ``out_dir``
    (bench/cli.py:174-181), formatted on a background thread.  ``close()`` (or leaving the
    ``with`` block) waits for the queued files; writer errors re-raise there."""

    def __init__(self, out_dir, background: bool = True):
        self.out_dir = out_dir
        os.makedirs(out_dir, exist_ok=True)
        self._q: queue.Queue | None = queue.Queue(maxsize=4) if background else None
        self._err: BaseException | None = None
        self.paths: list[str] = []
        if self._q is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def _run(self):
        while True:
            item = self._q.get()
            if item is None:
                return
            try:
                write_snapshot(*item)
            except BaseException as e:  # surfaced by close()
                self._err = e

    def emit(self, step, system, derived):
        path = os.path.join(self.out_dir, f"snapshot_{step:06d}.csv")
        self.paths.append(path)
        snap = snapshot_of(system, derived)
        if self._q is None:
            write_snapshot(path, snap)
        else:
            self._q.put((path, snap))

    def close(self):
        if self._q is not None:
            self._q.put(None)
            self._t.join()
            self._q = None
        if self._err is not None:
            raise self._err

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class StatsWriter:
    """stats_sink writing one ``stats_line`` per step (bench/cli.py:192-193)."""

    def __init__(self, path):
        self.fh = open(path, "w")

    def __call__(self, stats):
        self.fh.write(stats_line(stats) + "\n")

    def close(self):
        self.fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------------- checkpoints
def save_checkpoint(path, sim) -> None:
    """Binary checkpoint of a DeviceSim: primary state arrays (the order the next step's
    stable sort starts from), Verlet history, ids, and the control block (step, t_sim, dt,
    stop rules).  ``np.savez`` container; floats stored bit-exactly."""
    import torch  # noqa: F401  (device tensors)
    n = sim.n
    ctrl = sim.ctrl.cpu().numpy()
    np.savez(path, magic=np.array(CHECKPOINT_MAGIC), n=np.int64(n), nb=np.int64(sim.nb),
             mass_fluid=np.float64(sim.mass_fluid), mass_boundary=np.float64(sim.mass_boundary),
             posp=sim.posp[:n].cpu().numpy(), velr=sim.velr[:n].cpu().numpy(),
             prev=sim.prev[:n].cpu().numpy(), id=sim.id[:n].cpu().numpy(), ctrl=ctrl,
             pi_block=np.int32(getattr(sim, "pi_block", 128)),
             pi_kernel=np.array(getattr(sim, "pi_kernel", "gather")))


def load_checkpoint(path) -> dict:
    z = np.load(path if str(path).endswith(".npz") else str(path) + ".npz", allow_pickle=False)
    if str(z["magic"]) != CHECKPOINT_MAGIC:
        raise ValueError(f"{path}: not a {CHECKPOINT_MAGIC} file")
    return {k: z[k] for k in z.files}
