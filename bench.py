#!/usr/bin/env python
"""SPH step benchmark (BASELINE.json metric): particle-steps/s and interactions/s of the full
NL -> PI -> SU step on B200, with the reference CPU path timed beside it.

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config c3]

One JSON line on rank 0.  A "step" is one whole NL -> PI -> SU pass over the resident
synthetic dam break (state already in HBM; the state (~2 GB at C3) is far larger than the
126 MB L2, so no flush is needed between steps).  Timing: CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks.  See DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0's stdout carries exactly one JSON line: NCCL's own messages go to stderr.  The
# image's NCCL_DEBUG=VERSION prints a banner on stdout; instead NCCL logs at INFO for the INIT
# subsystem only (communicator set-up: nRanks, NVLS / P2P transport, channels), to stderr, so the
# rank count and transport of a multi-GPU run can be checked.  An explicit setting is respected.
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

METRIC = "particle-steps/sec and interactions/sec at 1/2/4/8 B200 vs host-CPU ref; % HBM roofline"
UNIT = "particle-steps/s"
FLOP_PER_CAND, FLOP_PER_EVAL = 9, 70  # SURVEY.md §8(d) algorithmic units
BYTES_NL_SU = 324 - 52                # compulsory NL+SU bytes per particle-step
GRAPH_BELOW = 2_000_000               # systems this small are launch-bound: graph replay


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None,
                    help="c1|c2|c3|c4_1..c4_8|c5 (default c3 at N=1, c3w_N above)")
    ap.add_argument("--n-subdiv", type=int, default=1)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the timed steps as one CUDA graph (auto: below 2M particles)")
    ap.add_argument("--pi-block", default="auto", choices=["auto", "128", "256", "384", "512"],
                    help="targets per interaction block (auto: sim.initial_pi_block)")
    ap.add_argument("--pi-kernel", default="tuned", choices=["tuned", "gather", "symmetric", "paired"],
                    help="FP32 interaction kernel: tuned (the faster of gather / paired, timed in the "
                         "warm-up like run_simulation(pi_kernel='tuned')), one-sided gather, "
                         "symmetric pair evaluation, or the gather with two targets per lane (paired)")
    ap.add_argument("--e2e-chunks", type=int, default=16,
                    help="byte-range chunks of the pipelined H2D/D2H state round trip (1 = serial)")
    ap.add_argument("--collapsed-step", type=int, default=6000,
                    help="N=1: also time the step after advancing the run to this step (the "
                         "column has collapsed: cells hold uneven counts); 0 = skip")
    ap.add_argument("--fp64-steps", type=int, default=5,
                    help="N=1: also time this many FP64 steps (bit-exact to the reference); 0 = skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--slab-path", action="store_true",
                    help="run the X-slab (NCCL) stepper even at one rank (exercises the multi-GPU path)")
    ap.add_argument("--rebalance-every", type=int, default=0,
                    help="N>1: re-place the X-slab bounds from measured per-rank PI time every k steps")
    return ap.parse_args()


def peaks():
    hbm = None
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json"
    except Exception:
        hbm, hbm_src = 6650.0, "fallback B200_PROFILING.md"
    fp32, fp32_src = 69.41, "profiles/peaks_r01.json (FFMA microbenchmark, tools/peaks.cu)"
    try:
        fp32 = json.load(open(os.path.join(ROOT, "profiles", "peaks_r01.json")))["fp32_tflops"]
    except Exception:
        pass
    return hbm, hbm_src, fp32, fp32_src


def traffic_for(cfg_name, n_subdiv, pi_block, pi_kernel):
    """DRAM bytes (read + write) per launch of the interaction kernel from a committed ncu
    capture of exactly this workload and build (profiles/ncu_traffic.json), else None."""
    try:
        key = f"{cfg_name}/n{n_subdiv}/pi{pi_block}/{pi_kernel}"
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[key]
        return float(t["dram_bytes_read"] + t["dram_bytes_write"]), t["source"]
    except Exception:
        return None, None


def composite_roofline(n, cand, evals, hbm_gbs, fp32_tflops, ms_step):
    """the step's floor = sum over kernels of max(bytes/BW, flop/P_fp32,
    mufu/P_mufu): NL+SU bytes at the measured HBM bandwidth, PI at max(FP32, MUFU) with
    4 MUFU per evaluated pair (measured MUFU.RSQ peak, profiles/peaks_r01.json)."""
    try:
        mufu = json.load(open(os.path.join(ROOT, "profiles", "peaks_r01.json")))["mufu_rsqrt_tops"]
    except Exception:
        mufu = 4.55
    t_mem = BYTES_NL_SU * n / (hbm_gbs * 1e9) * 1e3
    t_fp32 = (FLOP_PER_CAND * cand + FLOP_PER_EVAL * evals) / (fp32_tflops * 1e12) * 1e3
    t_mufu = 4.0 * evals / (mufu * 1e12) * 1e3
    floor = t_mem + max(t_fp32, t_mufu)
    return {"floor_ms": floor, "nl_su_hbm_ms": t_mem, "pi_fp32_ms": t_fp32, "pi_mufu_ms": t_mufu,
            "frac": floor / ms_step}


def scenario_kind(sc) -> str:
    import paper_1110_3711_b200 as sph
    return "3-D piston wave tank" if isinstance(sc, sph.WaveTank) else "3-D dam break"


def workload(name, n_subdiv):
    import paper_1110_3711_b200 as sph
    sc = sph.named_scenario(name)
    if isinstance(sc, sph.WaveTank):  # C5: piston wavemaker flume
        prm = sph.make_wave_tank_params(sc, n_subdiv=n_subdiv)
        return sc, prm, sph.build_wave_tank(sc, prm)
    prm = sph.make_params(sc, n_subdiv=n_subdiv)
    return sc, prm, sph.build_dam_break(sc, prm)


# ---------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU reference (oracle port)
_NL_CACHE = {}
FULL_NL_SU_MAX = 12_000_000  # above this, one CPU step is a bounded sample (see cpu_reference)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(cfg_name, sc, system, n_subdiv, world):
    """The ``config`` object of both arms (identical for the same workload)."""
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    n = system.n
    if world > 1:
        wl = f"{cfg_name}: {scenario_kind(sc)}, {n:,} particles over {world} GPUs (~{n // world:,} per GPU)"
        par = f"{world} X-slabs (edge bands with their forces written into the neighbours' memory -- CUDA IPC peer stores, NCCL send/recv fallback -- while the interior interacts)"
    else:
        wl = (f"{cfg_name}: {scenario_kind(sc)}, {n:,} particles per GPU "
              f"({system.count_fluid:,} fluid + {system.count_boundary:,} boundary)")
        par = "1 GPU"
    return {"workload": wl, "particles": n, "particles_per_gpu": n // max(world, 1),
            "n_subdiv": n_subdiv, "variant": variant,
            "l2": ("inputs larger than L2 (resident state ~%.2f GB per GPU, no flush needed)"
                   if n / max(world, 1) * 184 > 126e6 else
                   "inputs smaller than L2 (resident state ~%.3f GB; parity-size configuration, no flush)")
            % (n / max(world, 1) * 184 / 1e9),
            "parallelism": par}


class CpuStepper:
    """The reference step loop (sim.py:300-351 with GatherEngine, gather.py:42-110) on the
    oracle's bit-exact CPU restatement: numpy NL and SU as the reference runs them, the
    gather kernels in C on all host threads (the reference's numba kernels, nogil, one
    ThreadPoolExecutor worker per core).  Each ``step()`` advances the state, so timed steps
    see the evolving system, as harness.py:123-128 times them."""

    def __init__(self, system, prm, n_subdiv, cores):
        import oracle
        self.o, self.prm, self.cores = oracle, prm, cores
        self.variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
        self.pos, self.vel, self.rho = system.pos.copy(), system.vel.copy(), system.rho.copy()
        self.ids = np.asarray(system.id).copy()
        self.vel_prev, self.rho_prev = self.vel.copy(), self.rho.copy()
        self.nb, self.mf, self.mb = system.count_boundary, system.mass_fluid, system.mass_boundary
        self.step_no = 0

    def step(self):
        o, prm, nb = self.o, self.prm, self.nb
        t0 = time.perf_counter()
        cell, dims, _ = o.assign_cells(self.pos, prm)
        if np.any(cell == o.OUT_OF_DOMAIN):
            raise RuntimeError("reference arm: particle left the domain")
        perm = o.sort_perm(cell, nb)
        self.pos, self.vel, self.rho, self.ids = (a[perm] for a in (self.pos, self.vel, self.rho, self.ids))
        self.vel_prev, self.rho_prev = self.vel_prev[perm], self.rho_prev[perm]
        cs = cell[perm]
        cidx = o.cell_index(cs, nb, int(np.prod(dims)))
        t1 = time.perf_counter()
        out = o.gather(self.pos, self.vel, self.rho, nb, self.mf, self.mb, cs, dims, cidx, prm,
                       variant=self.variant, nthreads=self.cores)
        t2 = time.perf_counter()
        dt = o.compute_dt(out["accel"], out["visc_dt"], out["derived"][1], nb, prm)
        self.pos, self.vel, self.rho, self.vel_prev, self.rho_prev = o.verlet_update(
            self.step_no, self.pos, self.vel, self.rho, self.vel_prev, self.rho_prev, out["accel"],
            out["drho_dt"], nb, prm, dt)
        t3 = time.perf_counter()
        self.step_no += 1
        self.last = dict(cidx=cidx, dims=dims)
        return dict(nl=t1 - t0, pi=t2 - t1, su=t3 - t2, step_s=t3 - t0, counters=out["counters"])


def cpu_reference(system, prm, n_subdiv, budget_s, repeats=1):
    """Bounded sample of one reference step for workloads above FULL_NL_SU_MAX particles (the
    multi-GPU weak-scaling and wave-tank workloads, timed on rank 0 alone): NL and SU on the
    first FULL_NL_SU_MAX rows scaled by n / m (n log n for the sort); PI on every
    ``stride``-th target (a spatially uniform sample sized to about ``budget_s``) scaled by the
    stride.  The state is not advanced (one step of the initial frame)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    variant = "slowcellsh" if n_subdiv == 1 else "slowcellshalf"
    n, nb = system.n, system.count_boundary
    m = min(n, FULL_NL_SU_MAX)
    scale_lin = n / m
    scale_sort = scale_lin * (math.log(max(n, 2)) / math.log(max(m, 2)))
    key = id(system)
    if key not in _NL_CACHE:  # the full NL the PI sample needs (setup, not timed)
        cell, dims, _ = oracle.assign_cells(system.pos, prm)
        perm = oracle.sort_perm(cell, nb)
        cs = cell[perm]
        _NL_CACHE.clear()
        _NL_CACHE[key] = (perm, cs, dims, oracle.cell_index(cs, nb, int(np.prod(dims))))
    perm, cs, dims, cidx = _NL_CACHE[key]
    pos, vel, rho = system.pos[perm], system.vel[perm], system.rho[perm]
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        sub = system.pos[:m]
        cell, dims_t, _ = oracle.assign_cells(sub, prm)
        p_t = oracle.sort_perm(cell, min(nb, m))
        oracle.cell_index(cell[p_t], min(nb, m), int(np.prod(dims_t)))
        t_nl = (time.perf_counter() - t0) * scale_sort
        args = (pos, vel, rho, nb, system.mass_fluid, system.mass_boundary, cs, dims, cidx, prm)
        idx = np.arange(n)
        if ("pi", key) not in _NL_CACHE:
            # fixed cost of a pass (EOS of all particles, thread start-up) vs per-item cost,
            # measured once per workload; it sizes the sample stride
            t1 = time.perf_counter()
            oracle.gather(*args, variant=variant, nthreads=cores, target_mask=np.zeros(n, bool))
            t_fixed = time.perf_counter() - t1
            probe = 256
            t1 = time.perf_counter()
            oracle.gather(*args, variant=variant, nthreads=cores, target_mask=(idx % probe) == 0)
            est_full = t_fixed + max(time.perf_counter() - t1 - t_fixed, 0.0) * probe
            _NL_CACHE[("pi", key)] = (t_fixed, max(1, int(math.ceil(est_full / budget_s))))
        t_fixed, stride = _NL_CACHE[("pi", key)]
        t2 = time.perf_counter()
        out = oracle.gather(*args, variant=variant, nthreads=cores,
                            target_mask=(idx % stride) == 0 if stride > 1 else None)
        t_pi = t_fixed + max(time.perf_counter() - t2 - t_fixed, 0.0) * stride
        t3 = time.perf_counter()
        mm = slice(0, m)
        press, csound, _, _ = oracle.derived(rho[mm], prm)
        dt = oracle.compute_dt(out["accel"][mm], out["visc_dt"][mm], csound, min(nb, m), prm)
        oracle.verlet_update(0, pos[mm], vel[mm], rho[mm], vel[mm], rho[mm], out["accel"][mm],
                             out["drho_dt"][mm], min(nb, m), prm, max(dt, prm.dt_min))
        t_su = (time.perf_counter() - t3) * scale_lin
        times.append((t_nl, t_pi, t_su, stride))
    t_nl, t_pi, t_su, stride = min(times, key=lambda t: t[0] + t[1] + t[2])
    step_s = t_nl + t_pi + t_su
    what = "every item" if stride == 1 else f"every {stride}th item (uniform sample, scaled x{stride})"
    return dict(value=n / step_s, unit=UNIT, cores=cores, kind="port",
                sample=f"one {variant} step of the initial frame on {cores} threads ({cpu_model()}): "
                       f"NL+SU (numpy, as the reference) on the first {m} rows, scaled to {n}; "
                       f"PI (oracle C, OpenMP) on {what}; "
                       f"stage s NL {t_nl:.2f} PI {t_pi:.2f} SU {t_su:.2f}",
                step_s=step_s, exact=False)


def cpu_steps(system, prm, n_subdiv, warmup, steps):
    """``warmup`` + ``steps`` whole reference steps (CpuStepper) on all host cores; returns the
    mean of the timed ones."""
    cores = len(os.sched_getaffinity(0))
    st = CpuStepper(system, prm, n_subdiv, cores)
    for _ in range(warmup):
        st.step()
    t = [st.step() for _ in range(steps)]
    mean = lambda k: float(np.mean([x[k] for x in t]))  # noqa: E731
    step_s = mean("step_s")
    return dict(value=system.n / step_s, unit=UNIT, cores=cores, kind="port",
                sample=f"{steps} whole {st.variant} steps (after {warmup} warm-up), state advanced "
                       f"each step, on {cores} threads ({cpu_model()}): NL and SU numpy as the "
                       f"reference, PI the reference's gather kernels in C (OpenMP); mean stage s "
                       f"NL {mean('nl'):.2f} PI {mean('pi'):.2f} SU {mean('su'):.2f}",
                step_s=step_s, exact=True, stages_s={k: mean(k) for k in ("nl", "pi", "su")},
                stepper=st)


def cpu_engine_extras(stepper, prm, cores, budget_s=6.0):
    """The reference's other CPU strategies on the stepper's current frame (cellpairs.py):
    symmetric pair evaluation with private accumulators on all cores (the paper's best CPU
    strategy, cellpairs.py:132-164) and single-threaded symmetric (cellpairs.py:59-69).  Their
    PI pass runs on a uniform sample of cells (every k-th cell) and is scaled; the per-pass fixed
    cost (private buffers, merge) is measured with an empty sample.  NL + SU are the gather
    steps' (same code in the reference)."""
    o = stepper.o
    st, last = stepper, stepper.last
    args = (st.pos, st.vel, st.rho, st.nb, st.mf, st.mb, last["dims"], last["cidx"], prm)
    ncells = int(np.prod(last["dims"]))
    out = {}
    for name, threads in (("symmetric_x%d" % cores, cores), ("symmetric_1core", 1)):
        t0 = time.perf_counter()
        o.cellpairs(*args, symmetric=True, threads=threads, cells_mask=np.zeros(ncells, np.uint8))
        t_fixed = time.perf_counter() - t0
        probe = 64
        t0 = time.perf_counter()
        o.cellpairs(*args, symmetric=True, threads=threads,
                    cells_mask=(np.arange(ncells) % probe == 0).astype(np.uint8))
        est = t_fixed + max(time.perf_counter() - t0 - t_fixed, 0.0) * probe
        stride = max(1, int(math.ceil(est / budget_s)))
        t0 = time.perf_counter()
        o.cellpairs(*args, symmetric=True, threads=threads,
                    cells_mask=(np.arange(ncells) % stride == 0).astype(np.uint8) if stride > 1 else None)
        t_pi = t_fixed + max(time.perf_counter() - t0 - t_fixed, 0.0) * stride
        out[name] = {"pi_s": t_pi, "cells_sample": f"every {stride}th cell, scaled x{stride}",
                     "threads": threads}
    return out


def run_reference(args, cfg_name):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    sc, prm, system = workload(cfg_name, args.n_subdiv)
    extras = None
    if system.n <= FULL_NL_SU_MAX:
        r = cpu_steps(system, prm, args.n_subdiv, args.warmup, args.steps)
        if world == 1:
            ex = cpu_engine_extras(r["stepper"], prm, r["cores"])
            nl_su = r["stages_s"]["nl"] + r["stages_s"]["su"]
            extras = {k: dict(v, value=system.n / (nl_su + v["pi_s"]), unit=UNIT) for k, v in ex.items()}
        step_s = r["step_s"]
    else:
        for _ in range(args.warmup):
            cpu_reference(system, prm, args.n_subdiv, budget_s=1.5)
        t = [cpu_reference(system, prm, args.n_subdiv, budget_s=1.5) for _ in range(args.steps)]
        step_s = float(np.mean([x["step_s"] for x in t]))
        r = dict(t[-1])
    value = system.n / step_s
    cb = {k: r[k] for k in ("unit", "cores", "kind", "sample")}
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference dam-break lattice (Scenario/build_dam_break), hydrostatic rho",
            "config": workload_config(cfg_name, sc, system, args.n_subdiv, args.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if extras:
        line["cpu_engines"] = extras
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- multi-GPU (X slabs)
def run_slabs(args, cfg_name, sc, system, prm, prec, world, rank, local):
    """One X-slab per GPU (dslab.DeviceSlabSim): rows stay in place; the edge-band targets are
    interacted first and their rows + forces travel to the neighbours (NCCL send/recv on a comm
    stream) while the interior targets run; the receivers integrate them into migrants and next
    halos; device all-reduce of the dt minima; counters summed when read."""
    import torch
    import torch.distributed as dist
    from paper_1110_3711_b200 import _lib, dslab

    sim = dslab.DeviceSlabSim(system, prm, dslab.make_dist_comm(), precision=prec,
                              rebalance_every=args.rebalance_every)
    me = sim.ranks[0]
    Ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    pi_blocks = [128]
    tuning = None
    first = args.warmup
    if args.pi_block == "auto" and prec == _lib.SPHB_FP32:  # as the single-GPU path
        from paper_1110_3711_b200.sim import PI_LARGE_MIN_TARGETS, initial_pi_block
        pi_blocks = sim.choose_pi_block(PI_LARGE_MIN_TARGETS if args.n_subdiv == 1 else None)
        if args.pi_kernel == "tuned":  # per rank: the gather blocking vs the paired build
            cands = [("gather", initial_pi_block(sim.n_owned_max, args.n_subdiv)), ("paired", 512)]
            tuning = sim.tune_pi(cands)
            first += len(cands)
            pi_blocks = [r.pi_block for r in sim.ranks]
        else:
            sim.step()
            first += 1
        torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(local)
    t0, t1 = Ev(), Ev()
    t0.record()
    for _ in range(args.steps):
        sim.step()
    t1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    tt = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms = float(tt.item())
    # e2e: the same decomposed step with each rank's resident rows round-tripped through pinned
    # host buffers every step, in the reference's state layout (pos, vel, rho, vel_prev,
    # rho_prev, id: 52 B/row; sphb_state_to_soa / sphb_state_from_soa) and pipelined in
    # byte-range chunks of one buffer per side over the full-duplex PCIe link (as the
    # single-GPU path)
    h2d = d2h = 0
    e2e_value = None
    if args.e2e_steps > 0:
        L = _lib.lib()
        cap = int(me.n * 1.5) + 1024
        names = ("pos", "vel", "rho", "vel_prev", "rho_prev")
        width = {"pos": 3, "vel": 3, "rho": 1, "vel_prev": 3, "rho_prev": 1}
        # the six arrays of this step's n rows as views of one buffer per side (id first, the
        # f32 arrays at 16-B aligned offsets): byte-range chunks, one copy each way per chunk
        hbuf = torch.empty(56 * cap + 128, dtype=torch.uint8, pin_memory=True)
        dbuf = torch.empty(56 * cap + 128, dtype=torch.uint8, device="cuda")

        def layout(n):
            offs, off = {"id": 0}, 8 * n
            for k in names:
                off = (off + 15) // 16 * 16
                offs[k] = off
                off += 4 * width[k] * n
            return offs, off

        def views(buf, n, offs):
            v = {"id": buf[:8 * n].view(torch.int64)}
            for k in names:
                x = buf[offs[k]:offs[k] + 4 * width[k] * n].view(torch.float32)
                v[k] = x.view(n, width[k]) if width[k] > 1 else x
            return v

        nchunk = max(1, args.e2e_chunks)
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_out = [torch.cuda.Event() for _ in range(nchunk)]
        ev_in, ev_packed = torch.cuda.Event(), torch.cuda.Event()
        torch.cuda.synchronize()
        a, b = Ev(), Ev()
        a.record()
        for _ in range(args.e2e_steps):
            comp = torch.cuda.current_stream()
            n = me.n
            if n > cap:
                raise RuntimeError("e2e staging too small for this rank's rows")
            offs, nb_ = layout(n)
            dsoa = views(dbuf, n, offs)
            _lib.check(L.sphb_state_to_soa(0, n, me.a.posp.data_ptr(), me.a.velr.data_ptr(),
                                           me.a.prev.data_ptr(), *[dsoa[k].data_ptr() for k in names],
                                           comp.cuda_stream), "to_soa")
            dsoa["id"].copy_(me.a.id[:n])
            ev_packed.record(comp)
            bounds = [(nb_ * c // nchunk, nb_ * (c + 1) // nchunk) for c in range(nchunk)]
            s_out.wait_event(ev_packed)
            for c, (lo, hi) in enumerate(bounds):
                with torch.cuda.stream(s_out):
                    hbuf[lo:hi].copy_(dbuf[lo:hi], non_blocking=True)
                    ev_out[c].record(s_out)
                with torch.cuda.stream(s_in):
                    s_in.wait_event(ev_out[c])
                    dbuf[lo:hi].copy_(hbuf[lo:hi], non_blocking=True)
            ev_in.record(s_in)
            comp.wait_event(ev_in)
            _lib.check(L.sphb_state_from_soa(0, n, *[dsoa[k].data_ptr() for k in names],
                                             me.a.posp.data_ptr(), me.a.velr.data_ptr(),
                                             me.a.prev.data_ptr(), comp.cuda_stream), "from_soa")
            me.a.id[:n].copy_(dsoa["id"])
            h2d = d2h = n * 52
            sim.step()
        b.record()
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b)], device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = system.n * args.e2e_steps / (float(te.item()) * 1e-3)
    recs = sim.records(first, first + args.steps)
    true_pairs = float(np.mean(recs["hits_ordered"].astype(np.float64))) / 2
    evals = float(np.mean(recs["force_evals"].astype(np.float64)))
    cand = float(np.mean(recs["candidate_pairs"].astype(np.float64)))
    value = system.n * args.steps / (total_ms * 1e-3)
    # roofline of the interaction kernel per GPU: the all-reduced counters over the ranks'
    # mean interaction time (CUDA events around each rank's launch, the last <= 64 steps)
    pi_rank_ms = sim.measured_pi_ms()
    hbm, hbm_src, fp32, fp32_src = peaks()
    achieved = (FLOP_PER_CAND * cand + FLOP_PER_EVAL * evals) / world / \
        (float(np.mean(pi_rank_ms)) * 1e-3) / 1e12
    owned = torch.tensor([sim.n_owned_max], device="cuda", dtype=torch.int64)
    dist.all_reduce(owned, op=dist.ReduceOp.MAX)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic: reference dam-break lattice (Scenario/build_dam_break), hydrostatic rho",
        "config": workload_config(cfg_name, sc, system, args.n_subdiv, world),
        "build": {"slab_bounds": [int(v) for v in sim.bounds], "pi_block_rank0": int(pi_blocks[0]),
                  "pi_kernel_rank0": {_lib.SPHB_PI_PAIRED: "paired"}.get(me.pi_kernel, "gather"),
                  "pi_tuning_ms_rank0": tuning[0] if tuning else None,
                  "max_owned_per_gpu": int(owned.item()),
                  "exchange": ("edge bands (reach + 1 columns per neighbour) interacted first; "
                               + ("one kernel packs them with their forces straight into the "
                                  "neighbours' memory (CUDA IPC, NVLink P2P stores) and flags them, "
                                  "on a comm stream next to the interior targets"
                                  if getattr(sim.comm, "transport", "") == "peer" else
                                  "packed with their forces and sent over NCCL send/recv on a "
                                  "high-priority comm stream while the interior targets run")
                               + "; the receiver integrates them (migrants + next halo); device "
                                 "all-reduce of dt; one host read per step hidden behind the edge "
                                 "interaction"),
                  "band_transport": getattr(sim.comm, "transport", "nccl")},
        "interactions_per_s": true_pairs * args.steps / (total_ms * 1e-3),
        "pair_evals_per_s": evals * args.steps / (total_ms * 1e-3),
        "gpu_launches": args.steps * sim.launches_per_step(),
        "roofline": {"bound": "fp32", "kernel": "the interaction kernel (per GPU, owned targets)",
                     "achieved": achieved, "peak": fp32, "unit": "TFLOP/s", "frac": achieved / fp32,
                     "traffic": None,
                     "work": f"{FLOP_PER_CAND}*candidates + {FLOP_PER_EVAL}*evals per step / GPUs",
                     "pi_ms_per_rank": [float(v) for v in pi_rank_ms], "peak_source": fp32_src},
        "clocks": clk,
    }
    if e2e_value is not None:
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                       "path": "per step: each rank's resident rows through pinned host buffers in the "
                               "reference's layout (52 B/row), chunk-pipelined D2H/H2D, then the "
                               "decomposed step"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if hasattr(sim.comm, "close"):
        sim.comm.close()
    dist.destroy_process_group()


# ---------------------------------------------------------------- B200 arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # N=1: C3 (10.2M, the single-GPU roofline configuration); N>1: the weak-scaling family in
    # C3's tank (~10M particles per GPU), X-slab decomposed with NCCL halo/migration exchange
    cfg_name = args.config or ("c3" if args.gpus == 1 else f"c3w_{args.gpus}")
    if args.impl == "reference":
        run_reference(args, cfg_name)
        return
    import torch
    import torch.distributed as dist
    # SPHB_DIST_BACKEND=gloo runs the N-rank path with ranks sharing the visible GPUs (a code-
    # path check on a single-GPU box; the numbers are not scaling numbers)
    backend = os.environ.get("SPHB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1 or args.slab_path:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_1110_3711_b200 as sph
    from paper_1110_3711_b200 import _lib
    from paper_1110_3711_b200.device import DeviceSim

    sc, prm, system = workload(cfg_name, args.n_subdiv)
    variant = "slowcellsh" if args.n_subdiv == 1 else "slowcellshalf"
    prec = _lib.SPHB_FP64 if args.precision == "fp64" else _lib.SPHB_FP32
    if world > 1 or args.slab_path:
        run_slabs(args, cfg_name, sc, system, prm, prec, world, rank, local)
        return
    sim = DeviceSim(system, prm, reach=args.n_subdiv, precision=prec,
                    record_capacity=max(64, args.warmup + 2 * args.steps + 16))
    Ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # interaction blocking before the warm-up (run_simulation's policy, sim.py)
    if args.pi_block == "auto" and prec == _lib.SPHB_FP32:
        from paper_1110_3711_b200.sim import initial_pi_block
        sim.set_pi_block(initial_pi_block(sim.n, args.n_subdiv))
    elif args.pi_block != "auto":
        sim.set_pi_block(int(args.pi_block))
    tuned = args.pi_kernel == "tuned" and prec == _lib.SPHB_FP32 and args.pi_block == "auto"
    cands = sim.pi_candidates(args.n_subdiv) if tuned else []
    if args.pi_kernel not in ("gather", "tuned") and prec == _lib.SPHB_FP32:
        sim.set_pi_kernel(args.pi_kernel)
    warm = args.warmup
    warm_run = 0
    if tuned and warm >= len(cands):  # the first warm-up steps time the candidate builds
        sim.tune_pi(cands)
        warm -= sim.tuning_steps  # (a first tuning runs each build twice: >= W warm-up steps)
        warm_run = sim.tuning_steps
    warm_run += max(warm, 0)
    for _ in range(warm):
        sim.launch_step()
    torch.cuda.synchronize()
    first = int(sim.ctrl_host()["step"])
    if world > 1:
        dist.barrier()
    # launch-bound small systems replay the timed steps as one CUDA graph; their NL / PI / SU
    # stage times then come from an eager pass of the same length right before (untimed)
    use_graph = args.graph == "on" or (args.graph == "auto" and sim.n < GRAPH_BELOW)
    ev = [[Ev() for _ in range(4)] for _ in range(args.steps)]
    if use_graph:
        for k in range(args.steps):
            sim.launch_step(events=ev[k])
        torch.cuda.synchronize()
        sim.capture(args.steps)
        first = int(sim.ctrl_host()["step"])
    clocks = Clocks(local)
    t0, t1 = Ev(), Ev()
    torch.cuda.synchronize()
    t0.record()
    if use_graph:
        sim.run_graph()
    else:
        for k in range(args.steps):
            sim.launch_step(events=ev[k])
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    err = sim.error()
    if err is not None:
        raise RuntimeError(f"divergence during bench: {err}")
    build_info = {"warmup_steps_run": warm_run, "pi_block": sim.pi_block, "pi_kernel": sim.pi_kernel,
                  "pi_lane_use": round(sim.pi_lane_use(), 4), "cuda_graph": use_graph,
                  "pi_policy": "tuned" if tuned else args.pi_kernel, "pi_tuning_ms": sim.tuning}
    recs = sim.records(first, first + args.steps)
    nl_ms = [e[0].elapsed_time(e[1]) for e in ev]
    pi_ms = [e[1].elapsed_time(e[2]) for e in ev]
    su_ms = [e[2].elapsed_time(e[3]) for e in ev]
    cand = float(np.mean(recs["candidate_pairs"].astype(np.float64)))
    evals = float(np.mean(recs["force_evals"].astype(np.float64)))
    true_pairs = float(np.mean(recs["hits_ordered"].astype(np.float64))) / 2
    ms_step = total_ms / args.steps
    n_all = system.n * world
    value = n_all * args.steps / (total_ms * 1e-3)
    hbm, hbm_src, fp32, fp32_src = peaks()
    pi_mean = float(np.mean(pi_ms))
    flops = FLOP_PER_CAND * cand + FLOP_PER_EVAL * evals
    achieved = flops / (pi_mean * 1e-3) / 1e12
    nl_su_ms = float(np.mean(nl_ms) + np.mean(su_ms))
    traffic, traffic_src = traffic_for(cfg_name, args.n_subdiv, build_info["pi_block"],
                                       build_info["pi_kernel"])
    nlsu_gbs = BYTES_NL_SU * system.n / (nl_su_ms * 1e-3) / 1e9

    # ---- e2e: the same step through the C ABI with HOST buffers (H2D state in, D2H state out)
    # Every step copies its input state H2D from pinned host memory in the reference's own
    # layout (ParticleSystem id/pos/vel/rho + VerletState vel_prev/rho_prev, 52 B/particle),
    # converts it to the step's rows (sphb_state_from_soa), steps, converts back
    # (sphb_state_to_soa) and copies the result state D2H.  The six host arrays are views of
    # one pinned allocation (and their device images of one device buffer), so the round trip
    # moves byte-range chunks of a single buffer -- one copy per chunk and direction, which
    # keeps the full-duplex PCIe link busy (six copies per row chunk measured 13.7 vs 12.4 ms
    # per round trip, profiles/r02br_pcie_chunks.txt): the H2D of chunk c for step k+1 starts
    # as soon as the D2H of chunk c of step k has landed.
    h2d = d2h = 0
    e2e_value = None
    if args.e2e_steps > 0:
        L = _lib.lib()
        n = sim.n
        names = ("pos", "vel", "rho", "vel_prev", "rho_prev")
        width = {"pos": 3, "vel": 3, "rho": 1, "vel_prev": 3, "rho_prev": 1}
        ptr = lambda t: t.data_ptr()  # noqa: E731
        stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        # layout: id (int64) first, then the f32 arrays, each at a 16-B aligned offset
        offs, off = {"id": 0}, 8 * n
        for k in names:
            off = (off + 15) // 16 * 16
            offs[k] = off
            off += 4 * width[k] * n
        nbytes = off
        hbuf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        dbuf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

        def views(buf):
            v = {"id": buf[:8 * n].view(torch.int64)}
            for k in names:
                a = buf[offs[k]:offs[k] + 4 * width[k] * n].view(torch.float32)
                v[k] = a.view(n, width[k]) if width[k] > 1 else a
            return v

        hsoa, dsoa = views(hbuf), views(dbuf)

        def to_soa():
            _lib.check(L.sphb_state_to_soa(0, n, ptr(sim.posp), ptr(sim.velr), ptr(sim.prev),
                                           *[ptr(dsoa[k]) for k in names], stream()), "to_soa")
            dsoa["id"].copy_(sim.id[:n])

        def from_soa():
            _lib.check(L.sphb_state_from_soa(0, n, *[ptr(dsoa[k]) for k in names],
                                             ptr(sim.posp), ptr(sim.velr), ptr(sim.prev), stream()),
                       "from_soa")
            sim.id[:n].copy_(dsoa["id"])

        to_soa()  # the host arrays start as the current state
        hbuf.copy_(dbuf)
        h2d = d2h = 8 * n + sum(4 * width[k] * n for k in names)  # the arrays' bytes (no padding)
        nchunk = max(1, min(args.e2e_chunks, nbytes // (1 << 20)))
        bounds = [(nbytes * c // nchunk, nbytes * (c + 1) // nchunk) for c in range(nchunk)]
        comp = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_out = [torch.cuda.Event() for _ in bounds]
        ev_in, ev_packed = torch.cuda.Event(), torch.cuda.Event()

        def h2d_all(after_out):
            with torch.cuda.stream(s_in):
                for c, (lo, hi) in enumerate(bounds):
                    if after_out:
                        s_in.wait_event(ev_out[c])
                    dbuf[lo:hi].copy_(hbuf[lo:hi], non_blocking=True)
                ev_in.record(s_in)

        torch.cuda.synchronize()
        a, b = Ev(), Ev()
        a.record()
        s_in.wait_stream(comp)
        h2d_all(False)
        for k in range(args.e2e_steps):
            comp.wait_event(ev_in)
            from_soa()
            sim.first_keys_resync(keep_order=True)  # the same n rows: movers-only sort stays valid
            sim.launch_step()
            to_soa()
            ev_packed.record(comp)
            s_out.wait_event(ev_packed)
            with torch.cuda.stream(s_out):
                for c, (lo, hi) in enumerate(bounds):
                    hbuf[lo:hi].copy_(dbuf[lo:hi], non_blocking=True)
                    ev_out[c].record(s_out)
            if k + 1 < args.e2e_steps:
                h2d_all(True)
        comp.wait_stream(s_out)
        b.record()
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b)
        if world > 1:
            tt = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e_value = n_all * args.e2e_steps / (e2e_ms * 1e-3)

    launches = sim.launches_per_step() * args.steps

    def timed_steps(dsim, k, use_graph_k):
        """k steps of ``dsim`` timed with CUDA events (graph replay when asked); mean stage
        times from an eager pass of the same length right before when replaying."""
        evs = [[Ev() for _ in range(4)] for _ in range(k)]
        for j in range(k):
            dsim.launch_step(events=evs[j])
        torch.cuda.synchronize()
        stage = {"nl": float(np.mean([e[0].elapsed_time(e[1]) for e in evs])),
                 "pi": float(np.mean([e[1].elapsed_time(e[2]) for e in evs])),
                 "su": float(np.mean([e[2].elapsed_time(e[3]) for e in evs]))}
        f0 = int(dsim.ctrl_host()["step"])
        if use_graph_k:
            dsim.capture(k)
        a0, a1 = Ev(), Ev()
        torch.cuda.synchronize()
        a0.record()
        if use_graph_k:
            dsim.run_graph()
        else:
            for _ in range(k):
                dsim.launch_step()
        a1.record()
        torch.cuda.synchronize()
        recs_k = dsim.records(f0, f0 + k)
        return a0.elapsed_time(a1) / k, stage, recs_k

    # ---- the collapsed state: the same run advanced to --collapsed-step (cells hold 30-100
    # particles instead of the lattice's 64), then timed again
    collapsed = None
    if world == 1 and args.collapsed_step > 0:
        now = int(sim.ctrl_host()["step"])
        chunk = 500
        while now < args.collapsed_step:
            for _ in range(min(chunk, args.collapsed_step - now)):
                sim.launch_step()
            torch.cuda.synchronize()
            now = int(sim.ctrl_host()["step"])
            if sim.error() is not None:
                raise RuntimeError(f"divergence while advancing: {sim.error()}")
        if tuned:  # the measured selection again, in this state
            sim.tune_pi(cands)
        ms_c, stage_c, recs_c = timed_steps(sim, args.steps, False)
        e_c = float(np.mean(recs_c["force_evals"].astype(np.float64)))
        c_c = float(np.mean(recs_c["candidate_pairs"].astype(np.float64)))
        collapsed = {"step": now, "value": system.n / (ms_c * 1e-3), "unit": UNIT, "ms_per_step": ms_c,
                     "stage_ms": stage_c, "pi_lane_use": round(sim.pi_lane_use(), 4),
                     "pi_kernel": sim.pi_kernel, "pi_block": sim.pi_block, "pi_tuning_ms": sim.tuning,
                     "t_sim_s": float(sim.ctrl_host()["t_sim"]),
                     "interactions_per_s": e_c / 2 / (ms_c * 1e-3),
                     "pi_fp32_frac": (FLOP_PER_CAND * c_c + FLOP_PER_EVAL * e_c) / (stage_c["pi"] * 1e-3) / 1e12 / fp32,
                     "steps": args.steps}
    # ---- FP64: the instantiation that is bit-identical to the reference (its arithmetic)
    fp64 = None
    if world == 1 and args.fp64_steps > 0 and prec == _lib.SPHB_FP32:
        del sim  # room for the second system
        torch.cuda.empty_cache()
        sim64 = DeviceSim(system, prm, reach=args.n_subdiv, precision=_lib.SPHB_FP64,
                          record_capacity=max(64, 3 * args.fp64_steps + 8))
        for _ in range(2):
            sim64.launch_step()
        ms64, stage64, _ = timed_steps(sim64, args.fp64_steps, False)
        fp64 = {"value": system.n / (ms64 * 1e-3), "unit": UNIT, "ms_per_step": ms64,
                "stage_ms": stage64, "steps": args.fp64_steps,
                "note": "FP64 kernels: forces, dt and trajectories bit-identical to the reference"}
        del sim64
        torch.cuda.empty_cache()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if world > 1 else "weak", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic: reference dam-break lattice (Scenario/build_dam_break), hydrostatic rho",
        "config": workload_config(cfg_name, sc, system, args.n_subdiv, world),
        "build": build_info,
        "interactions_per_s": true_pairs * world * args.steps / (total_ms * 1e-3),
        "pair_evals_per_s": evals * world * args.steps / (total_ms * 1e-3),
        "stage_ms": {"nl": float(np.mean(nl_ms)), "pi": pi_mean, "su": float(np.mean(su_ms))},
        "counters_per_step": {"candidates": cand, "force_evals": evals, "true_pairs": true_pairs},
        "roofline": {"bound": "fp32", "kernel": ("k_interact_v12 (paired)" if build_info["pi_kernel"] == "paired" else
                                                     "k_interact_v8 (" + str(build_info["pi_kernel"]) + ")") +
                     " -- one launch: fluid + boundary targets",
                     "achieved": achieved, "peak": fp32, "unit": "TFLOP/s",
                     "frac": achieved / fp32, "traffic": traffic,
                     "traffic_note": ("dram read+write bytes of one launch, " + traffic_src)
                     if traffic else None,
                     "algorithmic_bytes": 52 * system.n,
                     "work": f"{FLOP_PER_CAND}*candidates + {FLOP_PER_EVAL}*evals per launch",
                     "peak_source": fp32_src},
        "roofline_hbm_nl_su": {"bound": "hbm", "achieved": nlsu_gbs, "peak": hbm, "unit": "GB/s",
                               "frac": nlsu_gbs / hbm, "traffic": None,
                               "work": f"{BYTES_NL_SU} B/particle-step over NL+SU stages",
                               "note": "the NL stage also hosts the interaction's block planning "
                                       "(k_blocks with the candidate counter) on a side stream, concurrent "
                                       "with K3 (sphb_interact_plan)",
                               "peak_source": hbm_src},
        "roofline_composite": composite_roofline(system.n, cand, evals, hbm, fp32, ms_step),
        "gpu_launches": launches,
        "clocks": clk,
    }
    if e2e_value is not None:
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                       "path": "per step: pinned host state in the reference's layout (pos, vel, "
                               "rho, vel_prev, rho_prev, id: 52 B/particle) -> H2D -> "
                               "sphb_state_from_soa -> sphb_* step -> sphb_state_to_soa -> D2H, "
                               f"round trip pipelined in {args.e2e_chunks} byte-range chunks of "
                               "one buffer per side (the six arrays are views of one pinned "
                               "allocation) over full-duplex PCIe (H2D of step k+1 chunk c after "
                               "D2H of step k chunk c)"}
    if collapsed is not None:
        line["collapsed"] = collapsed
    if fp64 is not None:
        line["fp64"] = fp64
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if system.n <= FULL_NL_SU_MAX:  # ~3 whole reference steps (C3: ~15-20 s of CPU work)
            cb = cpu_steps(system, prm, args.n_subdiv, 1, 2)
        else:
            cb = cpu_reference(system, prm, args.n_subdiv, args.cpu_budget_s)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
