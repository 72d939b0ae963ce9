"""X-slab decomposition: host logic and the exchange path on CPU ranks.

* bounds / rebalancing known answers (the reference's test_engines.py:328-365 cases);
* the decomposed step (migration + halos + owned-target interaction + dt reduction) with an
  oracle engine: in-process virtual slabs and a real 2-process gloo run, both compared with
  the oracle's single-domain run_simulation (step-0 counters/dt exact, trajectories close).
The same SlabSimulation drives libsphb200 on GPUs (tests/test_gpu_parity.py, NCCL in
bench.py --gpus N)."""
import os

import numpy as np
import pytest
import torch

import oracle
from slab_oracle_engine import OracleLocalEngine
from paper_1110_3711_b200 import Scenario, build_dam_break, make_params
from paper_1110_3711_b200 import slab
import slab_torch_reference as tslab


def test_rebalance_known_answers():
    b = np.array([0, 8, 16, 24, 32])
    assert list(slab.rebalance_slices(b, [1.0, 1.0, 1.0, 1.0])) == list(b)
    assert list(slab.rebalance_slices(b, [3.0, 1.0, 1.0, 1.0])) == [0, 4, 8, 20, 32]
    new = slab.rebalance_slices(np.arange(9), [5.0, 1, 1, 1, 1, 1, 1, 1])
    assert np.all(np.diff(new) >= 1) and new[0] == 0 and new[-1] == 8
    with pytest.raises(ValueError, match="positive"):
        slab.rebalance_slices(np.array([0, 4, 8]), [1.0, 0.0])


def test_balanced_bounds_counts_and_width():
    counts = np.array([0, 0, 10, 10, 10, 10, 0, 0, 1, 1], np.int64)
    b = slab.balanced_bounds(counts, 2, 1)
    assert b[0] == 0 and b[-1] == 10
    left = counts[b[0]:b[1]].sum()
    assert abs(left - counts.sum() / 2) <= 10
    b3 = slab.balanced_bounds(np.ones(6, np.int64), 3, 2)
    assert list(np.diff(b3)) == [2, 2, 2]
    with pytest.raises(ValueError):
        slab.balanced_bounds(np.ones(3, np.int64), 2, 2)


def test_columns_match_assign_cells():
    sc = Scenario(dp=0.02)
    prm = make_params(sc)
    s = build_dam_break(sc, prm)
    cell, dims, cs = oracle.assign_cells(s.pos, prm)
    col = slab.columns_of(torch.as_tensor(s.pos[:, 0]), float(prm.domain_min[0]), cs, int(dims[0]))
    assert np.array_equal(col.numpy(), cell % dims[0])


def _single_domain(system, prm, steps):
    p, v, r, i, stats = oracle.run_simulation(system.pos, system.vel, system.rho, system.id,
                                              system.count_boundary, system.mass_fluid,
                                              system.mass_boundary, prm, steps)
    return p, v, r, i, stats


def _compare(host, ref, tol):
    pos, vel, rho, ids, _ = host
    p, v, r, i, _ = ref
    assert np.array_equal(np.sort(ids), np.sort(i))
    a, b = np.argsort(ids), np.argsort(i)
    assert oracle.rel_linf(pos[a], p[b]) <= tol
    assert oracle.rel_linf(vel[a], v[b]) <= tol
    assert oracle.rel_linf(rho[a], r[b]) <= tol


@pytest.mark.parametrize("nslabs", [2, 3])
def test_virtual_slabs_match_single_domain(nslabs):
    sc = Scenario(dp=0.02)
    prm = make_params(sc)
    system = build_dam_break(sc, prm)
    cs, dims = oracle.grid_dims(prm)
    col = oracle.assign_cells(system.pos, prm)[0] % dims[0]
    bounds = slab.balanced_bounds(np.bincount(col, minlength=int(dims[0])), nslabs, 1)
    comm = tslab.LoopbackComm(nslabs)
    ranks = tslab.split_system(system, bounds, prm, lambda k: torch.device("cpu"))
    sim = tslab.SlabSimulation(ranks, prm, comm, 1, lambda r: OracleLocalEngine(
        prm, system.mass_fluid, system.mass_boundary, 1))
    steps = 12
    sim.run(steps)
    ref = _single_domain(system, prm, steps)
    st0 = ranks[0].stats[0]
    assert st0["dt"] == ref[4][0]["dt"]                       # step 0: identical inputs
    assert [st0["candidate_pairs"], st0["true_pairs"], st0["force_evals"], st0["ff_force_evals"]] \
        == list(ref[4][0]["counters"])
    assert all(r.stats[0]["true_pairs"] == st0["true_pairs"] for r in ranks)
    _compare(sim.gather_host(), ref, 1e-9)


def _gloo_worker(rank, world, port, steps, result_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scenario(dp=0.02)
    prm = make_params(sc)
    system = build_dam_break(sc, prm)
    cs, dims = oracle.grid_dims(prm)
    col = oracle.assign_cells(system.pos, prm)[0] % dims[0]
    bounds = slab.balanced_bounds(np.bincount(col, minlength=int(dims[0])), world, 1)
    comm = tslab.DistComm()
    ranks = tslab.split_system(system, bounds, prm, lambda k: torch.device("cpu"))
    sim = tslab.SlabSimulation([ranks[rank]], prm, comm, 1, lambda r: OracleLocalEngine(
        prm, system.mass_fluid, system.mass_boundary, 1))
    sim.run(steps)
    host = sim.gather_host()
    gathered = [None] * world
    dist.all_gather_object(gathered, (host, ranks[rank].stats))
    if rank == 0:
        np.save(result_path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_domain(tmp_path):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    steps = 8
    out = str(tmp_path / "res.npy")
    mp.spawn(_gloo_worker, args=(2, port, steps, out), nprocs=2, join=True)
    gathered = np.load(out, allow_pickle=True)
    host = tuple(np.concatenate([g[0][k] for g in gathered]) for k in range(5))
    stats = gathered[0][1]
    sc = Scenario(dp=0.02)
    prm = make_params(sc)
    system = build_dam_break(sc, prm)
    ref = _single_domain(system, prm, steps)
    assert stats[0]["dt"] == ref[4][0]["dt"]
    assert stats[0]["true_pairs"] == int(ref[4][0]["counters"][1])
    assert [s["dt"] for s in stats] == pytest.approx([s["dt"] for s in ref[4]], rel=1e-9)
    _compare(host, ref, 1e-9)


def test_device_slab_layout_host_logic():
    """dslab.rank_layout (the host half of the device-resident exchange): next-step layout,
    send sections and unpack destinations from every rank's 10 category totals."""
    from paper_1110_3711_b200 import dslab
    # rank totals: keepB keepF migLB migLF migRB migRF haloLB haloLF haloRB haloRF
    tab = np.array([[5, 50, 0, 0, 1, 2, 0, 0, 3, 7],
                    [6, 60, 2, 1, 0, 3, 4, 9, 1, 8],
                    [4, 40, 1, 4, 0, 0, 2, 6, 0, 0]], np.int64)
    lay = dslab.rank_layout(tab, 1, 3)
    in_l = [1, 2, 3, 7]   # rank 0's right sends: migB, migF, haloB, haloF
    in_r = [1, 4, 2, 6]   # rank 2's left sends
    assert lay["nb_next"] == 6 + in_l[0] + in_r[0] + in_l[2] + in_r[2]
    assert lay["n_next"] == lay["nb_next"] + 60 + in_l[1] + in_r[1] + in_l[3] + in_r[3]
    assert lay["keep_bases"] == (0, lay["nb_next"])
    assert lay["send_rows"] == (2 + 1 + 4 + 9, 0 + 3 + 1 + 8)
    assert lay["recv_rows"] == (sum(in_l), sum(in_r))
    assert lay["sections"] == [2, 3, 7, 0, 3, 4]
    # unpack destinations tile [0, n_next) exactly once with the kept blocks
    cover = np.zeros(lay["n_next"], int)
    cover[0:6] += 1
    cover[lay["nb_next"]:lay["nb_next"] + 60] += 1
    for side in lay["unpack"]:
        for r0, cnt, dst in side:
            cover[dst:dst + cnt] += 1
    assert np.all(cover == 1)
    # edge ranks have no outside neighbours
    lay0 = dslab.rank_layout(tab, 0, 3)
    assert lay0["recv_rows"][0] == 0 and lay0["unpack"][0] == [(0, 0, d) for _, _, d in lay0["unpack"][0]]


def test_band_recv_rows_from_neighbours():
    """dslab.band_recv_rows: a rank receives its left neighbour's right band and its right
    neighbour's left band; the end ranks have one neighbour."""
    from paper_1110_3711_b200 import dslab
    tab = np.array([[0, 7, -1], [5, 9, -1], [4, 0, -1]], np.int64)  # (to left, to right, err)
    assert dslab.band_recv_rows(tab, 0, 3) == (0, 5)
    assert dslab.band_recv_rows(tab, 1, 3) == (7, 4)
    assert dslab.band_recv_rows(tab, 2, 3) == (9, 0)
    assert dslab.band_recv_rows(tab[:1], 0, 1) == (0, 0)
