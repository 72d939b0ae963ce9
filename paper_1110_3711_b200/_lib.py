"""ctypes binding of libsphb200.so (include/sphb200.h).

The CUDA library is mandatory: there is no CPU fallback anywhere in this package.  If
the shared object is missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsphb200.so")
CSRC = os.path.join(HERE, "csrc")

SPHB_OK, SPHB_E_INVALID, SPHB_E_CUDA, SPHB_E_CAPACITY = 0, -1, -2, -3
SPHB_DIV_LEFT_DOMAIN, SPHB_DIV_NONFINITE_FORCES, SPHB_DIV_NONFINITE_STATE = 1, 2, 3
SPHB_DIV_SLAB_MARGIN = 4  # X slabs: a particle moved more than one cell column in one step
SPHB_DIV_EXCHANGE_TIMEOUT = 5  # X slabs, peer-memory transport: a band never arrived
SPHB_COUNTERS_GATHER, SPHB_COUNTERS_SYMMETRIC = 0, 1
SPHB_PI_GATHER, SPHB_PI_SYMMETRIC, SPHB_PI_PAIRED = 0, 1, 2
SPHB_FP32, SPHB_FP64 = 0, 1
SPHB_KERNEL_CUBIC, SPHB_KERNEL_WENDLAND = 0, 1
SPHB_INT_VERLET, SPHB_INT_SYMPLECTIC = 0, 1

c_i32, c_i64, c_f64, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class GridDesc(ctypes.Structure):
    _fields_ = [("origin", c_f64 * 3), ("domain_max", c_f64 * 3), ("cell_size", c_f64),
                ("dims", c_i32 * 3), ("reach", c_i32), ("tx0", c_i32), ("tx1", c_i32)]


class ParamsDesc(ctypes.Structure):
    _fields_ = [(k, c_f64) for k in ("sup2", "h", "invh", "kc", "eta2", "alpha", "invwdp", "c0",
                                     "rho0", "gamma", "mass_fluid", "mass_boundary", "tait_b")] + \
               [("g", c_f64 * 3), ("cfl", c_f64), ("dt_min", c_f64), ("dt_max", c_f64),
                ("verlet_stride", c_i32), ("order", c_i32), ("precision", c_i32),
                ("kernel", c_i32), ("integrator", c_i32), ("counters", c_i32),
                ("piston_id0", c_i64), ("piston_id1", c_i64), ("piston_x0", c_f64),
                ("piston_stroke", c_f64), ("piston_period", c_f64),
                ("wall_d", c_f64), ("wall_r0", c_f64), ("wall_p1", c_i32), ("wall_p2", c_i32)]


class StateDesc(ctypes.Structure):
    _fields_ = [(k, c_p) for k in ("posp", "velr", "prev", "id", "posp_s", "velr_s", "prev_s",
                                   "aux", "id_s", "keys", "keys_sorted", "perm", "cell_s", "beg",
                                   "end", "acc", "drho", "visc")]


# numpy views of the device structs (sphb200.h)
CTRL_DTYPE = np.dtype([("step", "<i8"), ("max_steps", "<i8"), ("t_sim", "<f8"), ("t_end", "<f8"),
                       ("dt", "<f8"), ("dtmin_f", "<u8"), ("dtmin_cv", "<u8"), ("err", "<u8"),
                       ("counters", "<u8", (4,)), ("active", "<i4"), ("tile_next", "<u4", (2,)),
                       ("nblk", "<u4", (2,)), ("pad_", "<i4"), ("dt_stage", "<f8"),
                       ("counters_stage", "<u8", (4,))])
CTRL_BYTES = 256
assert CTRL_DTYPE.itemsize <= CTRL_BYTES
REC_DTYPE = np.dtype([("dt", "<f8"), ("candidate_pairs", "<u8"), ("hits_ordered", "<u8"),
                      ("force_evals", "<u8"), ("ff_force_evals", "<u8")])
ERR_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


class SphbError(RuntimeError):
    pass


_L = None


def build(verbose: bool = False) -> str:
    """Compile libsphb200.so in place for sm_100a (make -C csrc)."""
    out = subprocess.run(["make", "-C", CSRC, "-j4"], capture_output=True, text=True)
    if verbose or out.returncode != 0:
        print(out.stdout[-4000:], out.stderr[-4000:])
    if out.returncode != 0:
        raise SphbError("libsphb200 build failed")
    return LIB_PATH


def lib():
    """The loaded library; raises when the CUDA extension is absent (no fallback)."""
    global _L
    if _L is not None:
        return _L
    if not os.path.exists(LIB_PATH):
        raise SphbError(f"{LIB_PATH} not built: run paper_1110_3711_b200._lib.build() "
                        "(the B200 path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = c_p
    sig = {
        "sphb_last_error": ([], ctypes.c_char_p),
        "sphb_version": ([], ctypes.c_char_p),
        "sphb_workspace_create": ([c_i64, c_i64, ctypes.POINTER(c_p)], c_i32),
        "sphb_workspace_destroy": ([P], c_i32),
        "sphb_workspace_reset": ([P, P], c_i32),
        "sphb_workspace_clear_hist": ([P, P], c_i32),
        "sphb_interact_plan": ([P, P, P, P, P, P, P], c_i32),
        "sphb_workspace_trust_order": ([P, P], c_i32),
        "sphb_workspace_bytes": ([P], c_i64),
        "sphb_workspace_set_mover_cap": ([P, c_i64], c_i32),
        "sphb_workspace_sort_info": ([P, P, P], c_i32),
        "sphb_workspace_set_pi_block": ([P, c_i32], c_i32),
        "sphb_workspace_set_pi_kernel": ([P, c_i32], c_i32),
        "sphb_ctrl_init": ([P, c_i64, c_f64, P], c_i32),
        "sphb_cell_keys": ([P, P, P, c_i64, c_i64, P, P, P, P], c_i32),
        "sphb_sort": ([P, P, P, c_i64, P, P, P, P], c_i32),
        "sphb_sort_ranges": ([P, P, P, c_i64, P, P, P, P, P, P], c_i32),
        "sphb_nl_build": ([P, P, P, c_i64, c_i64, P, P, P, P, P, P, P], c_i32),
        "sphb_reorder": ([P, P, c_i64, P, P, P, P, P, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_cell_ranges": ([P, P, P, P, P, P], c_i32),
        "sphb_cell_ranges_from_sorted": ([P, P, P, c_i64, c_i64, P, P, P], c_i32),
        "sphb_interact": ([P, P, P, c_i64, c_i64, P, P, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_step_begin": ([P, P], c_i32),
        "sphb_integrate": ([P, P, P, c_i64, c_i64, P, P, P, P, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_step_end": ([P, P, P, c_i64, P], c_i32),
        "sphb_integrate_stage": ([P, P, P, c_i64, c_i64, c_i32, P, P, P, P, P, P, P, P, P, P, P, P,
                                  P], c_i32),
        "sphb_energy": ([P, P, c_i64, c_i64, P, P, P, P], c_i32),
        "sphb_slab_tiles": ([c_i64], c_i64),
        "sphb_slab_count": ([P, c_i64, c_i64, P, P, c_i32, c_i32, P, P, P], c_i32),
        "sphb_slab_scatter": ([P, c_i64, c_i64, P, P, c_i32, c_i32, P, P, P, P, P, P, P, P, P, P,
                               P, P, P, P], c_i32),
        "sphb_slab_unpack": ([P, c_i64, c_i64, c_i64, P, P, P, P, P, P], c_i32),
        "sphb_band_scratch_words": ([P], c_i64),
        "sphb_band_count": ([P, c_i32, c_i32, P, P, P, P, P, P], c_i32),
        "sphb_band_pack": ([P, P, c_i32, c_i32, P, P, P, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_band_integrate": ([P, P, P, P, c_i64, c_i64, P, P, P, P, P, P, P, P], c_i32),
        "sphb_slab_tail": ([P, P, c_i64, P], c_i32),
        "sphb_band_put": ([P, P, c_i32, c_i32, P, P, P, P, P, P, P, P, P, P, P, P, P,
                           ctypes.c_uint64, P, P], c_i32),
        "sphb_band_wait": ([P, P, ctypes.c_uint64, P, P], c_i32),
        "sphb_cell_hist": ([P, P, P, c_i64, P, P], c_i32),
        "sphb_step": ([P, P, P, c_i64, c_i64, P, P, P, c_i64, P], c_i32),
        "sphb_state_from_soa": ([c_i64, c_i64, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_state_to_soa": ([c_i64, c_i64, P, P, P, P, P, P, P, P, P], c_i32),
        "sphb_build_ranges": ([P, P, c_i32, c_i32, c_i32, c_i32, P, P, P], c_i32),
        "sphb_dt_terms": ([P, c_i64, c_i64, P, P, P, P, P], c_i32),
        "sphb_verlet_soa": ([P, c_i64, c_i64, c_i32, c_f64, P, P, P, P, P, P, P, P], c_i32),
        "sphb_step_launch_count": ([P, c_i64], c_i64),
        "sphb_forces_f64": ([P, c_i64, P, P, P, P, P, P, P], c_i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _L = L
    return L


EXPORTED = ("sphb_last_error", "sphb_version", "sphb_workspace_create", "sphb_workspace_destroy",
            "sphb_workspace_reset", "sphb_workspace_clear_hist", "sphb_workspace_trust_order",
            "sphb_workspace_bytes",
            "sphb_workspace_set_mover_cap", "sphb_workspace_sort_info", "sphb_workspace_set_pi_block", "sphb_workspace_set_pi_kernel", "sphb_ctrl_init", "sphb_cell_keys",
            "sphb_sort", "sphb_sort_ranges", "sphb_nl_build", "sphb_reorder", "sphb_cell_ranges",
            "sphb_cell_ranges_from_sorted", "sphb_cell_hist",
            "sphb_interact", "sphb_interact_plan", "sphb_step_begin", "sphb_integrate", "sphb_step_end", "sphb_step",
            "sphb_step_launch_count", "sphb_integrate_stage", "sphb_energy", "sphb_slab_tiles",
            "sphb_slab_count", "sphb_slab_scatter", "sphb_slab_unpack", "sphb_band_scratch_words",
            "sphb_band_count", "sphb_band_pack", "sphb_band_integrate", "sphb_slab_tail",
            "sphb_band_put", "sphb_band_wait",
            "sphb_state_from_soa",
            "sphb_state_to_soa", "sphb_build_ranges", "sphb_dt_terms", "sphb_verlet_soa",
            "sphb_forces_f64")


def check(rc: int, what: str = "") -> None:
    if rc != SPHB_OK:
        msg = lib().sphb_last_error().decode()
        if rc in (SPHB_E_INVALID, SPHB_E_CAPACITY):
            raise ValueError(f"{what}: {msg}")
        raise SphbError(f"{what}: rc={rc} {msg}")


def ref(obj):
    return ctypes.byref(obj)
