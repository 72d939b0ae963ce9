// sphb_common.cuh -- shared device helpers for libsphb200 (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sphb200.h"

#define SPHB_FULL 0xffffffffu

namespace sphb {

// ---------------------------------------------------------------- exact f64
// The reference's numba/numpy arithmetic is IEEE binary64 without FMA contraction
// (SURVEY.md §2.1).  Every f64 expression that must match it bit for bit goes through
// these round-to-nearest intrinsics, which nvcc never contracts into DFMA.
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------- EOS (physics.py:119-134)
struct Derived {
  float prrho, csound, tensil;
};

// eos_press_scalar: f32(tait_b * ((rho/rho0)**gamma - 1.0))
__device__ __forceinline__ float eos_press(double rho, double tait_b, double rho0, double gamma) {
  return __double2float_rn(xmul(tait_b, xsub(pow(xdiv(rho, rho0), gamma), 1.0)));
}

// derive_scalar(press, rho, c0, rho0, gamma)
__device__ __forceinline__ Derived derive(double press, double rho, double c0, double rho0,
                                          double gamma) {
  Derived d;
  double inv_rho2 = xdiv(1.0, xmul(rho, rho));
  d.prrho = __double2float_rn(xmul(press, inv_rho2));
  d.csound = __double2float_rn(xmul(c0, pow(xdiv(rho, rho0), xmul(xsub(gamma, 1.0), 0.5))));
  if (press > 0.0)
    d.tensil = __double2float_rn(xmul(xmul(0.01, press), inv_rho2));
  else
    d.tensil = __double2float_rn(xmul(xmul(-0.2, press), inv_rho2));
  return d;
}

// The step's derived quantities of one particle from its density (physics.py:119-134).
// FAST (FP32 precision, gamma = 7): x^7 and x^3 by multiplication, every operation explicitly
// rounded, so K3 and the FP32 interaction kernels (which recompute a target's values instead of
// reading the aux row) get the same bits; else the exact f64 pow path (bit-identical to the
// reference, FP64 precision and the public compute_derived).
struct Deriv4 {
  float press, prrho, csound, tensil;
};
template <bool FAST>
__device__ __forceinline__ Deriv4 derived_of(double rho, const sphb_params_t& p) {
  Deriv4 r;
  if (FAST) {
    const double x = xmul(rho, xdiv(1.0, p.rho0)), x3 = xmul(xmul(x, x), x);
    r.press = __double2float_rn(xmul(p.tait_b, xsub(xmul(xmul(x3, x3), x), 1.0)));
    const double inv_rho2 = xdiv(1.0, xmul(rho, rho));
    r.prrho = __double2float_rn(xmul((double)r.press, inv_rho2));
    r.csound = __double2float_rn(xmul(p.c0, x3));
    r.tensil = __double2float_rn(xmul(xmul(r.press > 0.0f ? 0.01 : -0.2, (double)r.press), inv_rho2));
  } else {
    r.press = eos_press(rho, p.tait_b, p.rho0, p.gamma);
    const Derived d = derive((double)r.press, rho, p.c0, p.rho0, p.gamma);
    r.prrho = d.prrho;
    r.csound = d.csound;
    r.tensil = d.tensil;
  }
  return r;
}

// A target's (csound, tensil) in the FP32 interaction kernels when no aux rows were written:
// csound with K3's arithmetic (inv_rho0 = 1 / rho0 from the host: no division here), tensil
// from the staged prrho (within 1 f32 ulp of K3's; it only scales the tensile correction)
template <bool G7>
__device__ __forceinline__ float2 target_cs_tensil(double rho, float prrho, double inv_rho0,
                                                   const sphb_params_t& p) {
  const double x = xmul(rho, inv_rho0);
  const double cs = G7 ? xmul(p.c0, xmul(xmul(x, x), x))
                       : xmul(p.c0, pow(x, xmul(xsub(p.gamma, 1.0), 0.5)));
  const float ten = __double2float_rn(xmul(prrho > 0.0f ? 0.01 : -0.2, (double)prrho));
  return make_float2(__double2float_rn(cs), ten);
}

// ---------------------------------------------------------------- cells (grid.py:77-93)
// Returns the linear cell (x fastest) or -1 when outside [origin, domain_max] (NaN -> -1).
__device__ __forceinline__ int32_t cell_of(float x, float y, float z, const sphb_grid_t& g) {
  double p[3] = {(double)x, (double)y, (double)z};
  int64_t idx[3];
  bool inside = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    inside = inside && (p[k] >= g.origin[k]) && (p[k] <= g.domain_max[k]);
  }
  if (!inside) return -1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double f = floor(xdiv(xsub(p[k], g.origin[k]), g.cell_size));
    int64_t v = (int64_t)f;
    idx[k] = v < (int64_t)g.dims[k] - 1 ? v : (int64_t)g.dims[k] - 1;
  }
  return (int32_t)(idx[0] + (int64_t)g.dims[0] * (idx[1] + (int64_t)g.dims[1] * idx[2]));
}

__host__ __device__ __forceinline__ int64_t ncells_of(const sphb_grid_t& g) {
  return (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
}

// bits of the cell field of a sort key (list << cellbits | cell): 2^b > ncells, so the all-ones
// cell field of list 1 is never a real cell (the X-slab dead key below)
__host__ __device__ __forceinline__ int cellbits_of(const sphb_grid_t& g) {
  int64_t nc = ncells_of(g);
  int b = 1;
  while ((int64_t(1) << b) <= nc) ++b;
  return b;
}

// ---------------------------------------------------------------- X-slab grids (dslab)
// A grid whose interaction targets are a proper sub-range of columns is one rank's X slab.
// Its sort has one extra bin after the two lists: rows that left the slab during the last
// update and last step's halo copies carry the dead key, sort to the tail and drop out of
// the next step (n_live = begin of the dead bin).  Single-domain grids have no dead bin.
__host__ __device__ __forceinline__ bool slab_grid(const sphb_grid_t& g) {
  return g.tx0 > 0 || g.tx1 < g.dims[0];
}
__host__ __device__ __forceinline__ uint32_t dead_key(int cellbits) { return (2u << cellbits) - 1u; }
// per-key bins of the histogram / begin-end tables: both lists (+ the dead bin of a slab)
__host__ __device__ __forceinline__ int64_t nbins_of(const sphb_grid_t& g) {
  return 2 * ncells_of(g) + (slab_grid(g) ? 1 : 0);
}
// histogram / table index of a sort key; the dead key -> 2 ncells
__host__ __device__ __forceinline__ uint32_t key_bin(uint32_t key, int cellbits, uint32_t ncells) {
  return key == dead_key(cellbits) ? 2u * ncells
                                   : (key >> cellbits) * ncells + (key & ((1u << cellbits) - 1u));
}

// ---------------------------------------------------------------- errors / ctrl
__device__ __forceinline__ uint64_t err_key(int64_t step, int code, uint64_t index) {
  return ((uint64_t)step << 40) | ((uint64_t)code << 32) | (index & 0xffffffffull);
}

__device__ __forceinline__ void raise_div(sphb_ctrl_t* ctrl, int64_t step, int code,
                                          uint64_t index) {
  atomicMin((unsigned long long*)&ctrl->err, (unsigned long long)err_key(step, code, index));
}

// positive doubles (and +inf) order like their bit patterns
__device__ __forceinline__ void atomic_min_pos(uint64_t* addr, double v) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  unsigned long long cur = *(volatile unsigned long long*)addr;
  if (bits < cur) atomicMin((unsigned long long*)addr, bits);
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(SPHB_FULL, v, o));
  return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SPHB_FULL, v, o);
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace sphb

// host-side error helpers (capi.cu)
int sphb_set_error(int code, const char* fmt, ...);
int sphb_check_launch(const char* what);
