"""CPU local-step engine for the X-slab driver, built on the oracle (test infrastructure).

Lets tests/test_slab.py run paper_1110_3711_b200.slab.SlabSimulation on CPU ranks (gloo,
world_size 2) with the same exchange code the GPU path uses."""
import math

import numpy as np
import torch

import oracle


def _bits(x: float) -> int:
    return int(np.array([x], np.float64).view(np.int64)[0])


def _from_bits(b: int) -> float:
    return float(np.array([b], np.int64).view(np.float64)[0])


class OracleLocalEngine:
    def __init__(self, params, mass_fluid, mass_boundary, reach=1):
        self.params = params
        self.mf, self.mb = mass_fluid, mass_boundary
        self.reach = reach
        self.variant = {1: "slowcellsh", 2: "slowcellshalf"}[reach]

    def nl_pi(self, st, ids, nb, cols, step_index):
        prm = self.params
        a = st.detach().cpu().numpy()
        cell, dims, _ = oracle.assign_cells(a[:, 0:3], prm)
        perm = oracle.sort_perm(cell, nb)
        a, ids = a[perm], ids.detach().cpu().numpy()[perm]
        cs_ = cell[perm]
        cidx = oracle.cell_index(cs_, nb, int(np.prod(dims)))
        colx = cs_ % int(dims[0])
        mask = (colx >= cols[0]) & (colx < cols[1])
        pos = np.ascontiguousarray(a[:, 0:3])
        vel = np.ascontiguousarray(a[:, 3:6])
        rho = np.ascontiguousarray(a[:, 6])
        out = oracle.gather(pos, vel, rho, nb, self.mf, self.mb, cs_, dims, cidx, prm,
                            variant=self.variant, target_mask=mask)
        idx = np.arange(a.shape[0])
        fl = mask & (idx >= nb)
        dtf = math.inf
        if fl.any():
            f = out["accel"][fl] + prm.g[None, :]
            fmag = np.maximum(np.sqrt((f * f).sum(axis=1)), oracle.TINY_FORCE)
            dtf = float(np.min(np.sqrt(prm.h / fmag)))
        dtcv = math.inf
        if mask.any():
            csound = out["derived"][1]
            dtcv = float(np.min(prm.h / (csound[mask].astype(np.float64) + out["visc_dt"][mask])))
        self.words = torch.tensor([_bits(dtf), _bits(dtcv)], dtype=torch.int64)
        c = out["counters"]
        self.cnt = torch.tensor([int(c[0]), int(c[2]), int(c[2]), int(c[3])], dtype=torch.int64)
        self.state = (a, ids, nb, out, step_index)

    def dt_words(self):
        return self.words

    def counter_words(self):
        return self.cnt

    def su(self):
        prm = self.params
        a, ids, nb, out, step = self.state
        dt = prm.cfl * min(_from_bits(int(self.words[0])), _from_bits(int(self.words[1])))
        dt = float(min(max(dt, prm.dt_min), prm.dt_max))
        pos, vel, rho, vp, rp = oracle.verlet_update(
            step, a[:, 0:3], a[:, 3:6], a[:, 6], a[:, 7:10], a[:, 10], out["accel"],
            out["drho_dt"], nb, prm, dt)
        st = np.zeros_like(a)
        st[:, 0:3], st[:, 3:6], st[:, 6], st[:, 7:10], st[:, 10] = pos, vel, rho, vp, rp
        c = [int(v) for v in self.cnt]
        rec = dict(dt=dt, candidate_pairs=c[0], true_pairs=c[1] // 2, force_evals=c[2],
                   ff_force_evals=c[3])
        return torch.as_tensor(st), torch.as_tensor(ids), nb, rec
