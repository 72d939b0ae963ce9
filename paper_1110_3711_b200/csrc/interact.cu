// interact.cu -- particle interaction (PI) of the SPH step on sm_100a.
//
// Replaces GatherEngine.compute (engines/gather.py:42-110): the fused fluid pass
// (gather_fluid_cells / gather_fluid_ranges, engines/kernels.py:326-497) and the
// boundary pass (gather_boundary_cells / _ranges, kernels.py:500-596), with the
// compute_dt reductions (sim.py:215-232) fused into the epilogue (K6).
//
// Decomposition (FP32 CUDA cores: the pair math is a data-dependent gather-reduce, not a
// dense contraction, so tensor cores do not apply):
//   * k_blocks cuts every (y, z) cell row of a particle list into blocks of whole cells
//     holding <= 128 consecutive cell-sorted targets.  Because cells are x-fastest (grid.py:1-8), a
//     block's candidate set is, per stencil row, ONE contiguous particle range
//     [beg(cx_first - r), end(cx_last + r)).
//   * k_interact is persistent: two 4-warp CTAs per SM pull blocks dynamically.  The CTA
//     stages the block's whole candidate set into shared memory once (32 B/candidate:
//     x, y, z, prrho | vx, vy, vz, +-rho; the sign of rho marks the boundary list, cs and
//     the tensile factor are recomputed in-loop), so every pair reads SMEM, not L2 -- each
//     particle is fetched from L2 by ~13 blocks per step instead of by its ~250 neighbours.
//   * Each warp owns 32 targets (one per lane) and screens the sub-range of every staged
//     row that its lanes' stencils cover: LDS.128 broadcast + 6 FP32 ops + one compare per
//     candidate, giving a 32-bit "maybe" mask per lane per 32 candidates
//     (r2 < sup2 (1 + 1e-5)).
//   * Each lane queues its non-empty mask words (a block's worth) and the warp drains them
//     in lock-step, two candidates per lane per iteration with straight-line, masked pair
//     math: each lane pops its next candidates (FIFO == candidate order == the reference's
//     accumulation order), so the ~15-25% hit rate costs no divergence in the pair math --
//     the device analogue of the reference's pack-of-4 lane batching (kernels.py:97-118).
//   * Maybes that are not sure hits (inside the 1e-5 guard band around the cutoff, or
//     r2 ~ 0 such as the particle itself) are re-decided in the drain with the
//     reference's exact f64 predicate and stencil bounds, so hit sets -- hence
//     true_pairs / force_evals / ff counters -- are bit-exact (SURVEY.md §8(a')).
//   * The FP64 instantiation screens with the exact predicate and evaluates in the
//     reference's exact operation order: bit-identical forces.
#include <cuda_fp16.h>

#include <climits>

#include <cstdlib>

#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

#ifndef SPHB_NW
#define SPHB_NW 4
#endif
constexpr int NW = SPHB_NW;      // warps per CTA (pi128: 4, two CTAs per SM; pi384: 12, one)
#ifndef SPHB_PAIR
#define SPHB_PAIR 0              // 1: two targets per lane (k_interact_v12, interact_pair.cuh)
#endif
constexpr int BT = NW * 32 * (SPHB_PAIR ? 2 : 1);  // targets per block
#ifndef SPHB_H16
#define SPHB_H16 1
#endif
#ifndef SPHB_V8
#define SPHB_V8 1  // FP32 path: packed FFMA2 kernel (k_interact_v8); 0 = the generic template
#endif
constexpr int RING = SPHB_H16 ? 32 : 48;  // per-lane FIFO entries (non-empty 32-candidate words)
constexpr int MAXSEG = 128;      // stencil row segments per block (2 lists x (2r+1)^2, r <= 3)
#ifndef HYBRID_T
#define HYBRID_T 32  // n = 1, 384-target build: quads below this mean cell count become bricks
#endif

template <typename R>
struct Cfg;
template <>
struct Cfg<float> {
#ifndef V8_SCAP
#define V8_SCAP 2304
#endif
  static constexpr int SCAP = V8_SCAP;  // staged candidates (A, B float4 [+ x/y/z FP16 copies])
  static constexpr int NARR = 2;
  static constexpr int H16 = SPHB_H16;
};
template <>
struct Cfg<double> {
  static constexpr int SCAP = 1024;  // staged candidates (A, B, C float4)
  static constexpr int NARR = 3;
  static constexpr int H16 = 0;
};
// FP16 screen: block-centred coordinates in units of the support radius 2h; maybe = r^2 <
// 1.025.  Valid while |x| <= 4 (the block's x extent <= 8 support radii): coordinate
// quantisation <= 2^-9, |d(r^2)| <= 1.6e-2 at the cutoff, so no true hit is screened out.
constexpr float H16_THR = 1.025f;
constexpr float H16_MAXABS = 4.0f;

struct KArgs {
  sphb_params_t p;
  sphb_grid_t g;
  int64_t n, nb, ncells;
  const float4* __restrict__ posp;
  const float4* __restrict__ velr;
  const float4* __restrict__ aux;
  const int32_t* __restrict__ cell;
  const int32_t* __restrict__ beg;
  const int32_t* __restrict__ end;
  const int4* __restrict__ blocks;  // (fluid i0, i1, boundary i0, i1) per block
  // force outputs: FP64 = the ForceOutput layout (acc (n,3), drho (n), visc (n) f64);
  // FP32 = acc4 (ax, ay, az, drho) float4 per particle + visc32 float (include/sphb200.h)
  double* __restrict__ acc;
  double* __restrict__ drho;
  double* __restrict__ visc;
  float4* __restrict__ acc4;
  float* __restrict__ visc32;
  sphb_ctrl_t* ctrl;
  // FP32 constants
  float sup2_lo, sup2_hi, tiny, h, invh, k_gc, k_tw, eta2, alpha, massf, massb, k_cs, cs_exp;
  int gamma7;
  double inv_rho0;  // 1 / rho0 (host): a target's csound without a division
};

// FP32 constants of the pair loop, pinned in registers (an opaque move stops the compiler
// from re-loading them from the parameter bank inside the hot loop).
struct C32 {
  float sup2_lo, sup2_hi, tiny, h, invh, k_gc, k_tw, eta2, nalpha, massf, massb, k_cs, cs_exp;
};
__device__ __forceinline__ float pin(float v) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ C32 pin_constants(const KArgs& a) {
  C32 c;
  c.sup2_lo = pin(a.sup2_lo); c.sup2_hi = pin(a.sup2_hi); c.tiny = pin(a.tiny);
  c.h = pin(a.h); c.invh = pin(a.invh); c.k_gc = pin(a.k_gc); c.k_tw = pin(a.k_tw);
  c.eta2 = pin(a.eta2); c.nalpha = pin(-a.alpha); c.massf = pin(a.massf);
  c.massb = pin(a.massb); c.k_cs = pin(a.k_cs); c.cs_exp = pin(a.cs_exp);
  return c;
}

struct Seg {
  int g0, g1;   // global particle range of the block's union for this stencil row
  int pos;      // start in the concatenated candidate sequence
  int rowoff;   // offset of the row's first cell in beg/end (list offset included)
  int dyz;      // row offset from the block's origin row: (dy + 16) | (dz + 16) << 8
};

// Staging of a batch [q0, q1) of the block's candidate sequence, issued by the 32 lanes of one
// warp in parallel (h/2 cells: 2 x 36 stencil rows per brick, so one thread issuing every copy
// serialised the batch start): one TMA bulk copy per (stencil row, array) into the A (posp:
// x, y, z, prrho) and B (velr) rows, completion counted in bytes on the mbarrier.
__device__ __forceinline__ void stage_batch(const float4* posp, const float4* velr,
                                            const Seg* sSeg, int nseg, int q0, int q1,
                                            uint32_t smA, uint32_t offB, uint32_t mbar, int lane) {
  uint32_t bytes = 0;
  for (int k = lane; k < nseg; k += 32) {
    const Seg sg = sSeg[k];
    const int lo_p = max(sg.pos, q0), hi_p = min(sg.pos + (sg.g1 - sg.g0), q1);
    if (hi_p > lo_p) bytes += 32u * (uint32_t)(hi_p - lo_p);
  }
  bytes = __reduce_add_sync(SPHB_FULL, bytes);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (lane == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                 : "memory");
  __syncwarp();
  for (int k = lane; k < nseg; k += 32) {
    const Seg sg = sSeg[k];
    const int lo_p = max(sg.pos, q0), hi_p = min(sg.pos + (sg.g1 - sg.g0), q1);
    if (hi_p <= lo_p) continue;
    const int j0 = sg.g0 + (lo_p - sg.pos);
    const uint32_t nbytes = 16u * (uint32_t)(hi_p - lo_p);
    const uint32_t dA = smA + 16u * (uint32_t)(lo_p - q0), dB = dA + offB;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dA), "l"(posp + j0), "r"(nbytes), "r"(mbar) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dB), "l"(velr + j0), "r"(nbytes), "r"(mbar) : "memory");
  }
}

__device__ __forceinline__ double ipow(double q, int k) {
  double r = 1.0;
  for (int e = 0; e < k; ++e) r = xmul(r, q);
  return r;
}

__device__ __forceinline__ bool step_live(const sphb_ctrl_t* c) {
  return c->active && c->err >= ((uint64_t)(c->step + 1) << 40);
}

// exact reference predicate 0 < r2 < sup2 with r2 = (dx*dx + dy*dy) + dz*dz in f64
// (kernels.py:372-376), dx = f64(x_i) - f64(x_j)
__device__ __forceinline__ bool exact_hit(double xi, double yi, double zi, double xj, double yj,
                                          double zj, double sup2) {
  double dx = xsub(xi, xj), dy = xsub(yi, yj), dz = xsub(zi, zj);
  double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
  return r2 < sup2 && r2 > 0.0;
}

// x cell of a coordinate, exactly as assign_cells computes it (grid.py:87-89)
__device__ __forceinline__ int xcell_of(float x, const sphb_grid_t& g) {
  double f = floor(xdiv(xsub((double)x, g.origin[0]), g.cell_size));
  int v = (int)f;
  return v < g.dims[0] - 1 ? v : g.dims[0] - 1;
}

// Explicit 32-bit shared-window addressing: keeps the address arithmetic to one IMAD per
// access (the compiler otherwise rematerialises the window base for every dynamic index).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return h;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((uint16_t)v));
}

template <typename R>
struct Own {
  R x, y, z, vx, vy, vz, rho, prrho, cs, ten;
};

template <typename R>
struct Accum {
  R ax, ay, az, dr, vd;
};

// ------------------------------------------------------------------ fused boundary repulsion
// Extension (off by default): the Lennard-Jones wall force of one fluid
// target, a += D ((r0/r)^p1 - (r0/r)^p2) r_ij / r^2 over boundary particles closer than r0
// (<= 2h: all in the stencil), evaluated in the FP32 interaction kernels' epilogue of each
// staging batch from the staged boundary rows -- in the order of the separate k_wall_force pass
// (stencil rows z-major, then y, then candidate index), f64, so the result is the same bits.
// Returns whether any boundary particle was within r0.
__device__ __forceinline__ bool wall_batch(const KArgs& a, const Seg* sSeg, int nseg, int q0,
                                           int q1, uint32_t smA, float ox, float oy, float oz,
                                           int xlo, int xhi, int rsy, int rsz, double& fx,
                                           double& fy, double& fz) {
  const double r02 = xmul(a.p.wall_r0, a.p.wall_r0);
  const int reach = a.g.reach;
  bool hit = false;
  for (int k = 0; k < nseg; ++k) {
    const Seg sg = sSeg[k];
    if (sg.rowoff >= a.ncells || sg.g1 <= sg.g0) continue;  // boundary-list rows
    const int dy = (sg.dyz & 255) - 16, dz = (sg.dyz >> 8) - 16;
    if (abs(dy - rsy) > reach || abs(dz - rsz) > reach) continue;  // not this target's stencil
    const int j0 = a.beg[sg.rowoff + xlo], j1 = a.end[sg.rowoff + xhi];
    const int p0 = max(sg.pos + (j0 - sg.g0), q0), p1 = min(sg.pos + (j1 - sg.g0), q1);
    for (int p = p0; p < p1; ++p) {
      const float4 A = lds4(smA + 16u * (uint32_t)(p - q0));
      const double dx = xsub((double)ox, (double)A.x);
      const double dy2 = xsub((double)oy, (double)A.y);
      const double dz2 = xsub((double)oz, (double)A.z);
      const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy2, dy2)), xmul(dz2, dz2));
      if (!(r2 > 0.0 && r2 < r02)) continue;
      const double q = xdiv(a.p.wall_r0, __dsqrt_rn(r2));
      const double f = xdiv(xmul(a.p.wall_d, xsub(ipow(q, a.p.wall_p1), ipow(q, a.p.wall_p2))), r2);
      fx = xadd(fx, xmul(f, dx));
      fy = xadd(fy, xmul(f, dy2));
      fz = xadd(fz, xmul(f, dz2));
      hit = true;
    }
  }
  return hit;
}

// the wall term joins the FP32 acceleration as the separate pass adds it (f64 sum, rounded),
// and the target's force dt term with it joins the minimum (the SPH-only one is already in)
__device__ __forceinline__ void wall_finish(const KArgs& a, int64_t i, int64_t step, float ax,
                                            float ay, float az, float dr, double fx, double fy,
                                            double fz, double& dtf_min) {
  const float wx = (float)xadd((double)ax, fx), wy = (float)xadd((double)ay, fy),
              wz = (float)xadd((double)az, fz);
  a.acc4[i] = make_float4(wx, wy, wz, dr);
  const double gx = xadd((double)wx, a.p.g[0]), gy = xadd((double)wy, a.p.g[1]),
               gz = xadd((double)wz, a.p.g[2]);
  double fmag = __dsqrt_rn(xadd(xadd(xmul(gx, gx), xmul(gy, gy)), xmul(gz, gz)));
  fmag = fmag > 1e-30 ? fmag : 1e-30;
  dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(a.p.h, fmag)));
  if (!(isfinite(wx) && isfinite(wy) && isfinite(wz)))
    raise_div(a.ctrl, step, SPHB_DIV_NONFINITE_FORCES, 0);
}

// ------------------------------------------------------------------ pair math
// FP32 (physics.py:183-220 restated for FP32 CUDA cores).  Branch-free cubic spline:
// W ~ t^3/4 - u^3, dW/dq ~ -3/4 t^2 + 3 u^2 with t = 2 - q, u = max(1 - q, 0).
// Folded constants: k_gc = kc/h, k_tw = kc/W(dp); the viscous 0.5 factors cancel.
template <bool G7, bool EQM>
__device__ __forceinline__ void pair_eval32(const C32& a, const Own<float>& o, float dx,
                                            float dy, float dz, float r2in, const float4& A,
                                            const float4& B, bool ok, Accum<float>& s) {
  const float r2 = ok ? r2in : a.sup2_lo;  // masked slots stay finite; their terms are zeroed
  const float rinv = rsqrtf(r2);
  const float q = r2 * rinv * a.invh;
  const float t = 2.0f - q;
  const float u = fmaxf(1.0f - q, 0.0f);
  const float t2 = t * t, u2 = u * u;
  const float w = fmaf(0.25f * t2, t, -u2 * u);
  const float dw = fmaf(3.0f, u2, -0.75f * t2);
  const float gc = dw * a.k_gc * rinv;
  const float rho_j = fabsf(B.w);
  const float mj = EQM ? 1.0f : (B.w < 0.0f ? a.massb : a.massf);  // EQM: mass applied once
  const float prrho_j = A.w;
  float cs_j;
  if (G7) {  // gamma = 7: cs = c0 (rho/rho0)^3
    const float rr = rho_j * a.k_cs;  // (rho/rho0) * c0^(1/3)
    cs_j = rr * rr * rr;
  } else {
    cs_j = a.k_cs * exp2f(a.cs_exp * __log2f(rho_j));
  }
  const float ten_j = prrho_j * (prrho_j > 0.0f ? 0.01f : -0.2f);
  const float dvx = o.vx - B.x, dvy = o.vy - B.y, dvz = o.vz - B.z;
  const float dot = fmaf(dvz, dz, fmaf(dvy, dy, dvx * dx));
  const float mu = __fdividef(a.h * dot, r2 + a.eta2);
  const float vterm = __fdividef(a.nalpha * (o.cs + cs_j) * mu, o.rho + rho_j);
  const float visc = dot < 0.0f ? vterm : 0.0f;
  const float tw = w * a.k_tw;
  const float tw2 = tw * tw;
  const float pterm = fmaf((o.ten + ten_j) * tw2, tw2, o.prrho + prrho_j + visc);
  const float fm = ok ? (EQM ? pterm * gc : mj * pterm * gc) : 0.0f;
  const float gd = ok ? (EQM ? gc : mj * gc) : 0.0f;
  s.ax = fmaf(-fm, dx, s.ax);
  s.ay = fmaf(-fm, dy, s.ay);
  s.az = fmaf(-fm, dz, s.az);
  s.dr = fmaf(gd, dot, s.dr);
  s.vd = fmaxf(s.vd, ok ? fabsf(mu) : 0.0f);
}

// FP64: the reference's exact operation order (physics.py:196-220, kernels.py:382-390),
// no contraction; cs and tensil are the exact f32 values of K3 (C.x, C.y).
__device__ __forceinline__ void pair_eval64(const KArgs& a, const Own<double>& o, double dx,
                                            double dy, double dz, double r2, const float4& A,
                                            const float4& B, const float4& C,
                                            Accum<double>& s) {
  const sphb_params_t& p = a.p;
  const double r = __dsqrt_rn(r2);
  const double q = xmul(r, p.invh);
  const double kc = p.kc;
  double wab, dwdq;
  if (p.kernel == SPHB_KERNEL_WENDLAND) {  // W = kc t^4 (2q + 1), dW/dq = -5 kc q t^3
    const double t = xsub(1.0, xmul(0.5, q));
    const double t2 = xmul(t, t);
    wab = xmul(xmul(kc, xmul(t2, t2)), xadd(xmul(2.0, q), 1.0));
    dwdq = xmul(xmul(xmul(-5.0, kc), q), xmul(t2, t));
  } else if (q < 1.0) {
    wab = xmul(kc, xadd(xsub(1.0, xmul(xmul(1.5, q), q)), xmul(xmul(xmul(0.75, q), q), q)));
    dwdq = xmul(xmul(kc, xsub(xmul(2.25, q), 3.0)), q);
  } else {
    const double t = xsub(2.0, q);
    wab = xmul(xmul(xmul(xmul(0.25, kc), t), t), t);
    dwdq = xmul(xmul(xmul(-0.75, kc), t), t);
  }
  const double gc = xdiv(xmul(dwdq, p.invh), r);
  const double dvx = xsub(o.vx, (double)B.x), dvy = xsub(o.vy, (double)B.y),
               dvz = xsub(o.vz, (double)B.z);
  const double dot = xadd(xadd(xmul(dvx, dx), xmul(dvy, dy)), xmul(dvz, dz));
  const double mu = xdiv(xmul(p.h, dot), xadd(r2, p.eta2));
  double visc = 0.0;
  if (dot < 0.0) {
    const double rho_j = (double)fabsf(B.w), cs_j = (double)C.x;
    visc = xdiv(xmul(xmul(-p.alpha, xmul(0.5, xadd(o.cs, cs_j))), mu),
                xmul(0.5, xadd(o.rho, rho_j)));
  }
  const double tw = xmul(wab, p.invwdp);
  const double tw2 = xmul(tw, tw);
  const double pterm = xadd(xadd(xadd(o.prrho, (double)A.w), visc),
                            xmul(xmul(xadd(o.ten, (double)C.y), tw2), tw2));
  const double mj = B.w < 0.0f ? p.mass_boundary : p.mass_fluid;
  const double pg = xmul(pterm, gc);
  s.ax = xsub(s.ax, xmul(mj, xmul(pg, dx)));
  s.ay = xsub(s.ay, xmul(mj, xmul(pg, dy)));
  s.az = xsub(s.az, xmul(mj, xmul(pg, dz)));
  s.dr = xadd(s.dr, xmul(mj, xmul(gc, dot)));
  const double ma = fabs(mu);
  if (ma > s.vd) s.vd = ma;
}

// Evaluate staged candidate (A, B[, C]); false if a guard-band maybe is rejected.
// Stencil x-bound of a candidate (y/z rows are the lane's own); out of line, it only runs
// for exact hits within 1e-12 of the cutoff.
__device__ __noinline__ bool in_stencil_x(float x, int xlo, int xhi, sphb_grid_t g) {
  const int cxj = xcell_of(x, g);
  return cxj >= xlo && cxj <= xhi;
}

// Cold path of the FP32 screen: exact f64 predicate; a hit outside the lane's own stencil
// x-range needs |dx| > 2h (1 - 1e-15), so the cell test only runs within 1e-12 of sup2.
__device__ __forceinline__ bool cold_accept(const KArgs& a, float ox, float oy, float oz,
                                            const float4 A, int xlo, int xhi) {
  const double dx = xsub((double)ox, (double)A.x), dy = xsub((double)oy, (double)A.y),
               dz = xsub((double)oz, (double)A.z);
  const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
  if (!(r2 < a.p.sup2 && r2 > 0.0)) return false;
  if (r2 > a.p.sup2 * (1.0 - 1e-12)) return in_stencil_x(A.x, xlo, xhi, a.g);
  return true;
}

template <bool G7, bool EQM>
__device__ __forceinline__ bool eval_one(const KArgs& a, const C32&, const Own<double>& o,
                                         const float4& A,
                                         const float4& B, const float4& C, int, int,
                                         Accum<double>& s) {
  const double dx = xsub(o.x, (double)A.x), dy = xsub(o.y, (double)A.y),
               dz = xsub(o.z, (double)A.z);
  const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
  pair_eval64(a, o, dx, dy, dz, r2, A, B, C, s);
  return true;
}

// Two queued candidates (staged indices k1, k2; < 0 = empty slot) for one lane.  The exact
// re-decision of non-sure maybes is a rare divergent pre-pass; the pair math itself is
// straight-line for both candidates (independent chains interleave) with masked terms.
// Returns the number of rejected maybes; *rej_f counts the fluid-list ones.
template <bool G7, bool EQM>
__device__ __forceinline__ uint32_t eval_two(const KArgs& a, const C32& c, const Own<float>& o,
                                             uint32_t smA, uint32_t smB, uint32_t, int k1, int k2,
                                             int xlo, int xhi, Accum<float>& s, uint32_t* rej_f) {
  const bool v1 = k1 >= 0, v2 = k2 >= 0;
  const uint32_t i1 = v1 ? (uint32_t)k1 : 0u, i2 = v2 ? (uint32_t)k2 : 0u;
  const float4 A1 = lds4(smA + 16u * i1), B1 = lds4(smB + 16u * i1);
  const float4 A2 = lds4(smA + 16u * i2), B2 = lds4(smB + 16u * i2);
  const float dx1 = o.x - A1.x, dy1 = o.y - A1.y, dz1 = o.z - A1.z;
  const float dx2 = o.x - A2.x, dy2 = o.y - A2.y, dz2 = o.z - A2.z;
  const float r21 = fmaf(dz1, dz1, fmaf(dy1, dy1, dx1 * dx1));
  const float r22 = fmaf(dz2, dz2, fmaf(dy2, dy2, dx2 * dx2));
  const bool f1 = r21 < c.sup2_lo && r21 > c.tiny, f2 = r22 < c.sup2_lo && r22 > c.tiny;
  bool ok1 = v1 && f1, ok2 = v2 && f2;
  // FP32 r2 >= sup2 (1 + 1e-5) is a certain miss (the FP16 screen's shell); only the guard
  // band and r2 ~ 0 need the exact f64 decision
  if (v1 && !f1 && r21 < c.sup2_hi) ok1 = cold_accept(a, o.x, o.y, o.z, A1, xlo, xhi);
  if (v2 && !f2 && r22 < c.sup2_hi) ok2 = cold_accept(a, o.x, o.y, o.z, A2, xlo, xhi);
  pair_eval32<G7, EQM>(c, o, dx1, dy1, dz1, r21, A1, B1, ok1, s);
  pair_eval32<G7, EQM>(c, o, dx2, dy2, dz2, r22, A2, B2, ok2, s);
  const uint32_t r1 = (v1 && !ok1) ? 1u : 0u, r2 = (v2 && !ok2) ? 1u : 0u;
  *rej_f += (r1 && B1.w > 0.0f ? 1u : 0u) + (r2 && B2.w > 0.0f ? 1u : 0u);
  return r1 + r2;
}
template <bool G7, bool EQM>
__device__ __forceinline__ uint32_t eval_two(const KArgs& a, const C32& c, const Own<double>& o,
                                             uint32_t smA, uint32_t smB, uint32_t smC, int k1,
                                             int k2, int xlo, int xhi, Accum<double>& s,
                                             uint32_t* rej_f) {
  (void)rej_f;
  if (k1 >= 0)
    eval_one<G7, EQM>(a, c, o, lds4(smA + 16u * k1), lds4(smB + 16u * k1), lds4(smC + 16u * k1),
                      xlo, xhi, s);
  if (k2 >= 0)
    eval_one<G7, EQM>(a, c, o, lds4(smA + 16u * k2), lds4(smB + 16u * k2), lds4(smC + 16u * k2),
                      xlo, xhi, s);
  return 0u;
}

// candidate screen: FP32 "maybe" (r2 < sup2 (1 + 1e-5)); FP64 exact predicate
__device__ __forceinline__ bool screen(const KArgs&, const C32& c, const Own<float>& o,
                                       const float4& A) {
  const float dx = o.x - A.x, dy = o.y - A.y, dz = o.z - A.z;
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx)) < c.sup2_hi;
}
__device__ __forceinline__ bool screen(const KArgs& a, const C32&, const Own<double>& o,
                                       const float4& A) {
  return exact_hit(o.x, o.y, o.z, (double)A.x, (double)A.y, (double)A.z, a.p.sup2);
}

// ------------------------------------------------------------------ block builder
// Cuts each (y, z) cell row into blocks of whole cells holding <= BT targets of BOTH lists
// (fluid targets and boundary targets of the same cells share one staged candidate set).
// Only cell columns [tx0, tx1) hold targets (the owned slab of an X-slab decomposition;
// halo columns outside it are candidates only).  A cell with more than BT targets is split
// into single-list chunks.
// Block record (2 x int4): (fluid i0, i1, boundary i0, i1), (row, first cell x, last cell x, 0)
//
// Two passes over the rows (COUNT: records per row; then, after an exclusive scan over the
// rows, WRITE: records at the row's offset), so the block list is in row order (z-major, then
// y): the persistent interaction CTAs pulling consecutive blocks work on neighbouring rows
// whose stencil rows overlap, and the staged rows come from L2 instead of DRAM.
//
// Bricks (h/2 cells, reach 2, cell order): the unit is a pair of rows in y times a pair in z,
// cut along x into blocks of whole cell columns (4 cells) holding <= BT targets.  A brick
// stages the union of its rows' stencils, (2r + 2)^2 rows instead of (2r + 1)^2 per row, so
// per target ~12 staged candidates at rest (2 x 2 rows x 12 cells of 8 particles over
// 6 x 6 rows x 16 cells) where 1-row blocks need ~31.  Record: (0, 0, 0, 0),
// (row of (y0, z0), first cell x, last cell x, 1).  A column with more than BT targets falls
// back to 1-row single-list chunks.
// Hybrid (brick = T > 1: the 384-target build at n = 1): the unit is the quad, but a quad
// whose non-empty cells hold >= T targets on average is cut into row blocks, row by row --
// the FP16 screen's column cap (6 lattice cells) leaves sparse 1-row blocks mostly empty,
// while dense rows fill them and stage fewer rows per target than a brick.
// Paired build (two targets per lane): a lane's two targets must come from the same list, so
// the fluid targets of a block take an even number of slots (padded) -- a block fits when
// pad2(fluid) + boundary <= BT.
__device__ __forceinline__ int block_slots(int nf, int ntot) {
  return SPHB_PAIR ? ntot + (nf & 1) : ntot;
}
// candidate_pairs of the gather traversal (kernels.py:355-371, counted before the distance
// test) depends on the cell tables alone: a fluid target of cell c visits every particle of
// both lists in its stencil rows' x ranges [max(x - r, 0), min(x + r, nx - 1)] except itself, a
// boundary target the fluid ones, so  cand = sum_c nf_c (F_c + B_c - 1) + nb_c F_c.  k_blocks'
// count pass sums it per cell (its lanes walk the cells anyway); the FP32 gather kernels then
// carry no per-target counting (its global loads sat on every block's setup path).
__device__ __forceinline__ unsigned long long cell_cand(const sphb_grid_t& g, int64_t ncells,
                                                        const int32_t* __restrict__ beg,
                                                        const int32_t* __restrict__ end, int x,
                                                        int y, int z, int nf, int nb) {
  if (nf <= 0 && nb <= 0) return 0ull;
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2], R = g.reach;
  const int xlo = max(x - R, 0), xhi = min(x + R, nx - 1);
  long long F = 0, B = 0;
  for (int zz = max(z - R, 0); zz <= min(z + R, nz - 1); ++zz)
    for (int yy = max(y - R, 0); yy <= min(y + R, ny - 1); ++yy) {
      const int64_t rb = (int64_t)nx * (yy + (int64_t)ny * zz), rf = ncells + rb;
      F += end[rf + xhi] - beg[rf + xlo];
      B += end[rb + xhi] - beg[rb + xlo];
    }
  return (unsigned long long)((long long)max(nf, 0) * (F + B - 1) + (long long)max(nb, 0) * F);
}
__device__ __forceinline__ void add_cand(unsigned long long* acc, unsigned long long c) {
  c = warp_sum_u64(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(acc, c);
}

// Reach >= 2 (h/2 cells: 25 stencil rows per cell) the count pass's lanes would walk too many
// rows each: one thread per target cell of the window instead (x fastest: coalesced table
// loads, empty cells leave after two loads), on the same side stream.
constexpr int KC_THREADS = 256;
__global__ void __launch_bounds__(KC_THREADS) k_cand_cells(sphb_grid_t g, int64_t ncells,
                                                          const int32_t* __restrict__ beg,
                                                          const int32_t* __restrict__ end,
                                                          const sphb_ctrl_t* ctrl,
                                                          unsigned long long* cand_acc) {
  if (!step_live(ctrl)) return;
  const int ny = g.dims[1], nx = g.dims[0];
  const int span = g.tx1 - g.tx0;
  const int64_t total = (int64_t)span * ny * g.dims[2];
  unsigned long long acc = 0;
  for (int64_t t = (int64_t)blockIdx.x * KC_THREADS + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * KC_THREADS) {
    const int64_t row = t / span;
    const int x = g.tx0 + (int)(t - row * span);
    const int64_t cb = (int64_t)nx * row + x, cf = ncells + cb;
    acc += cell_cand(g, ncells, beg, end, x, (int)(row % ny), (int)(row / ny), end[cf] - beg[cf],
                     end[cb] - beg[cb]);
  }
  __shared__ unsigned long long s_acc[KC_THREADS / 32];
  acc = warp_sum_u64(acc);
  if ((threadIdx.x & 31) == 0) s_acc[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < KC_THREADS / 32 ? s_acc[threadIdx.x] : 0ull;
    acc = warp_sum_u64(acc);
    if (threadIdx.x == 0 && acc) atomicAdd(cand_acc, acc);
  }
}

// the side-stream plan's candidate count into the step counters (one thread)
__global__ void k_cand_take(unsigned long long* cand_acc, sphb_ctrl_t* ctrl) {
  const unsigned long long c = *cand_acc;
  *cand_acc = 0ull;
  if (c) atomicAdd((unsigned long long*)&ctrl->counters[0], c);
}

// Row blocks of one cell row r (records written at out when !COUNT); the record count, on
// every lane.  s_ends: [span] fluid ends, then [span] boundary ends of the row.
template <bool COUNT>
__device__ int row_records(const sphb_grid_t& g, int64_t ncells, const int32_t* __restrict__ beg,
                           const int32_t* __restrict__ end, int64_t r, int4* out, int maxc,
                           int32_t* s_ends, int lane, unsigned long long* cand_ctrl) {
  const int nx = g.dims[0], span = g.tx1 - g.tx0;
  const int64_t cb = r * nx, cf = ncells + r * nx;  // row offsets in the B / F tables
  if (span <= 0 ||
      (end[cf + g.tx1 - 1] <= beg[cf + g.tx0] && end[cb + g.tx1 - 1] <= beg[cb + g.tx0]))
    return 0;
  unsigned long long cand = 0;
  for (int k = lane; k < span; k += 32) {
    const int32_t fe = end[cf + g.tx0 + k], be = end[cb + g.tx0 + k];
    s_ends[k] = fe;
    s_ends[span + k] = be;
    if (COUNT && cand_ctrl)
      cand += cell_cand(g, ncells, beg, end, g.tx0 + k, (int)(r % g.dims[1]), (int)(r / g.dims[1]),
                        fe - beg[cf + g.tx0 + k], be - beg[cb + g.tx0 + k]);
  }
  if (COUNT && cand_ctrl) add_cand(cand_ctrl, cand);
  __syncwarp();
  int nrec = 0;
  if (lane == 0) {
    auto emit = [&](int4 b, int x0, int x1) {
      if (!COUNT) {
        out[2 * nrec] = b;
        out[2 * nrec + 1] = make_int4((int)r, x0, x1, 0);
      }
      ++nrec;
    };
    int32_t f0 = beg[cf + g.tx0], b0 = beg[cb + g.tx0];  // open block
    int32_t fcur = f0, bcur = b0;
    int xa = -1, xl = -1;  // first / last non-empty cell of the open block
    for (int k = 0; k < span; ++k) {
      const int x = g.tx0 + k;
      const int32_t fe = s_ends[k], be = s_ends[span + k];
      if (fe == fcur && be == bcur) continue;  // empty cell
      if ((block_slots(fe - f0, (fe - f0) + (be - b0)) > BT ||
           (xa >= 0 && x - xa + 1 > maxc && 4 * ((fcur - f0) + (bcur - b0)) >= BT)) &&
          (fcur > f0 || bcur > b0)) {  // close before this cell
        emit(make_int4(f0, fcur, b0, bcur), xa, xl);
        f0 = fcur;
        b0 = bcur;
        xa = -1;
      }
      if (block_slots(fe - f0, (fe - f0) + (be - b0)) > BT) {  // one oversized cell: single-list chunks of <= BT
        for (int32_t p = f0; p < fe; p += BT) emit(make_int4(p, min(p + BT, fe), be, be), x, x);
        for (int32_t p = b0; p < be; p += BT) emit(make_int4(fe, fe, p, min(p + BT, be)), x, x);
        f0 = fe;
        b0 = be;
      } else {
        if (xa < 0) xa = x;
        xl = x;
      }
      fcur = fe;
      bcur = be;
    }
    if (fcur > f0 || bcur > b0) emit(make_int4(f0, fcur, b0, bcur), xa, xl);
  }
  __syncwarp();
  return __shfl_sync(SPHB_FULL, nrec, 0);
}

template <bool COUNT>
__global__ void __launch_bounds__(32) k_blocks(sphb_grid_t g, int64_t ncells,
                                               const int32_t* __restrict__ beg,
                                               const int32_t* __restrict__ end,
                                               int32_t* __restrict__ row_off,
                                               int4* __restrict__ blk, sphb_ctrl_t* ctrl,
                                               int brick, int maxc,
                                               unsigned long long* cand_acc) {
  // count pass of the FP32 gather builds (reach 1): also the candidate counter (cell_cand),
  // into the plan's accumulator (the interaction kernel moves it into the step counters)
  unsigned long long* const cand_ctrl = COUNT ? cand_acc : nullptr;
  // one warp per cell row: the lanes stage the row's cumulative ends (both lists) in shared
  // memory, lane 0 makes the greedy cut
  extern __shared__ int32_t s_ends[];  // [span] fluid ends, then [span] boundary ends
  if (!step_live(ctrl)) return;
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  const int nyb = brick ? (ny + 1) / 2 : ny, nzb = brick ? (nz + 1) / 2 : nz;
  const int64_t nrows = (int64_t)nyb * nzb;
  const int span = g.tx1 - g.tx0, lane = threadIdx.x;
  if (brick) {
    for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
      const int y0 = 2 * (int)(r % nyb), z0 = 2 * (int)(r / nyb);
      int tot_all = 0;
      int ne = 0;  // non-empty cells of the four rows (hybrid blocking)
      unsigned long long cand = 0;
      for (int k = lane; k < span; k += 32) {  // targets of the brick's cell column x
        const int x = g.tx0 + k;
        int c = 0, cf = 0;
        for (int sub = 0; sub < 4; ++sub) {
          const int yy = y0 + (sub & 1), zz = z0 + (sub >> 1);
          if (yy >= ny || zz >= nz) continue;
          const int64_t rb = (int64_t)nx * (yy + (int64_t)ny * zz) + x, rf = ncells + rb;
          const int nfc = end[rf] - beg[rf], nbc = end[rb] - beg[rb], call = nfc + nbc;
          cf += nfc;
          c += call;
          ne += call > 0 ? 1 : 0;
          if (cand_ctrl) cand += cell_cand(g, ncells, beg, end, x, yy, zz, nfc, nbc);
        }
        s_ends[k] = c;
        s_ends[span + k] = cf;  // fluid part (the paired build's slot padding)
        tot_all += c;
      }
      tot_all = __reduce_add_sync(SPHB_FULL, tot_all);
      ne = __reduce_add_sync(SPHB_FULL, ne);
      if (cand_ctrl) add_cand(cand_ctrl, cand);
      __syncwarp();
      if (tot_all == 0) {
        if (COUNT && lane == 0) row_off[r] = 0;
        continue;
      }
      if (brick > 1 && tot_all >= brick * ne) {
        // hybrid blocking (n = 1 gather builds): a quad whose cells hold >= `brick` targets on
        // average is cut into row blocks, row by row (dense rows fill 1-row blocks; bricks pay
        // for sparse ones, where the column cap leaves 1-row blocks mostly empty)
        int nrec = 0;
        for (int sub = 0; sub < 4; ++sub) {
          const int yy = y0 + (sub & 1), zz = z0 + (sub >> 1);
          if (yy >= ny || zz >= nz) continue;
          nrec += row_records<COUNT>(g, ncells, beg, end, (int64_t)yy + (int64_t)ny * zz,
                                     COUNT ? nullptr : blk + 2 * ((int64_t)row_off[r] + nrec), maxc,
                                     s_ends, lane, nullptr);
        }
        if (COUNT && lane == 0) row_off[r] = nrec;
        continue;
      }
      if (lane == 0) {
        int nrec = 0;
        int4* out = COUNT ? nullptr : blk + 2 * (int64_t)row_off[r];
        auto emit = [&](int4 b, int4 m) {
          if (!COUNT) {
            out[2 * nrec] = b;
            out[2 * nrec + 1] = m;
          }
          ++nrec;
        };
        const int key0 = y0 + ny * z0;
        int tot = 0, totf = 0, xa = -1, xl = -1;
        for (int k = 0; k < span; ++k) {
          const int x = g.tx0 + k, c = s_ends[k], cf = s_ends[span + k];
          if (c == 0) continue;
          // close before x when the targets would not fit, or when the block's columns would
          // exceed maxc (the FP16 tensor-core screen's coordinate range, else the kernel falls
          // back to the CUDA-core screen) and the block is at least a quarter full (sparse rows,
          // e.g. a small system's mostly empty tank: fuller blocks on the fallback screen win)
          if ((block_slots(totf + cf, tot + c) > BT || (xa >= 0 && x - xa + 1 > maxc && 4 * tot >= BT)) &&
              tot > 0) {
            emit(make_int4(0, 0, 0, 0), make_int4(key0, xa, xl, 1));
            tot = totf = 0;
            xa = -1;
          }
          if (block_slots(cf, c) > BT) {  // oversized column: 1-row single-list chunks
            for (int sub = 0; sub < 4; ++sub) {
              const int yy = y0 + (sub & 1), zz = z0 + (sub >> 1);
              if (yy >= ny || zz >= nz) continue;
              const int key = yy + ny * zz;
              const int64_t rb = (int64_t)nx * key + x, rf = ncells + rb;
              const int32_t fb = beg[rf], fe = end[rf], bb0 = beg[rb], be = end[rb];
              for (int32_t p = fb; p < fe; p += BT)
                emit(make_int4(p, min(p + BT, fe), be, be), make_int4(key, x, x, 0));
              for (int32_t p = bb0; p < be; p += BT)
                emit(make_int4(fe, fe, p, min(p + BT, be)), make_int4(key, x, x, 0));
            }
            continue;
          }
          if (xa < 0) xa = x;
          xl = x;
          tot += c;
          totf += cf;
        }
        if (tot > 0) emit(make_int4(0, 0, 0, 0), make_int4(key0, xa, xl, 1));
        if (COUNT) row_off[r] = nrec;
      }
      __syncwarp();
    }
    return;
  }
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int nrec = row_records<COUNT>(g, ncells, beg, end, r,
                                        COUNT ? nullptr : blk + 2 * (int64_t)row_off[r], maxc,
                                        s_ends, lane, cand_ctrl);
    if (COUNT && lane == 0) row_off[r] = nrec;
  }
}

// exclusive scan of the per-row record counts (one CTA: rows ~10^4); the total is the launch's
// block count (ctrl->nblk[0], read by the interaction CTAs)
constexpr int KB_SCAN = 1024;
__global__ void __launch_bounds__(KB_SCAN) k_blocks_scan(int32_t* row_off, int64_t nrows,
                                                         sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  __shared__ int32_t s_w[KB_SCAN / 32];
  __shared__ int32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nrows; base += KB_SCAN) {
    const int64_t r = base + tid;
    const int32_t v = r < nrows ? row_off[r] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(SPHB_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(SPHB_FULL, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;  // inclusive per-warp totals
    }
    __syncthreads();
    const int32_t carry = s_carry;
    const int32_t excl = carry + (warp ? s_w[warp - 1] : 0) + x - v;
    if (r < nrows) row_off[r] = excl;
    __syncthreads();
    if (tid == KB_SCAN - 1) s_carry = carry + s_w[KB_SCAN / 32 - 1];
    __syncthreads();
  }
  if (tid == 0) {
    ctrl->nblk[0] = (uint32_t)s_carry;
    ctrl->tile_next[0] = 0u;  // this launch's block queue (several launches per step: X slabs)
  }
}

// ------------------------------------------------------------------ the interaction kernel
extern __shared__ float4 g_sm4[];  // staged candidates: A | B | (C)
extern __shared__ uint32_t g_sm32[];

template <typename R, bool G7, bool EQM>
__global__ void __launch_bounds__(NW * 32, 2) k_interact(KArgs a) {
  if (!step_live(a.ctrl)) return;
  const C32 c32 = pin_constants(a);
  constexpr int SCAP = Cfg<R>::SCAP;
  constexpr int SB = SCAP, SC = 2 * SCAP;                  // float4 offsets of B and C
  constexpr int HBYTES = Cfg<R>::H16 ? 6 * SCAP : 0;        // FP16 x | y | z screen copies
  constexpr int MASK0 = (16 * Cfg<R>::NARR * SCAP + HBYTES) / 4;  // uint32 offset of the rings
  uint32_t* sMask = g_sm32 + MASK0;                          // [NW][RING][32] mask words
  uint16_t* sBase = reinterpret_cast<uint16_t*>(sMask + NW * RING * 32);  // [NW][RING][32]
  __shared__ Seg sSeg[MAXSEG];
  __shared__ int s_blk, s_nseg_tot, s_scan[MAXSEG];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = a.g.dims[0], ny = a.g.dims[1], nz = a.g.dims[2];
  const int reach = a.g.reach, side = 2 * reach + 1;
  const uint32_t nblocks = a.ctrl->nblk[0];
  const int64_t step = a.ctrl->step;
  const int4* blocks = a.blocks;
  uint32_t* myMask = sMask + warp * RING * 32;
  uint16_t* myBase = sBase + warp * RING * 32;

  unsigned long long c_cand = 0, c_hits = 0, c_ff = 0;
  double dtf_min = INFINITY, dtcv_min = INFINITY;

  for (;;) {
    if (tid == 0) s_blk = (int)atomicAdd(&a.ctrl->tile_next[0], 1u);
    __syncthreads();
    const uint32_t blk = (uint32_t)s_blk;
    if (blk >= nblocks) break;
    const int4 bb = blocks[2 * blk];
    const int f0 = bb.x, nf = bb.y - bb.x, b0 = bb.z, nbt = bb.w - bb.z;
    // the block's cells: one row, columns [cxa, cxb] (sorted lists: first/last targets)
    const int cfirst = min(nf ? a.cell[f0] : INT_MAX, nbt ? a.cell[b0] : INT_MAX);
    const int clast = max(nf ? a.cell[f0 + nf - 1] : -1, nbt ? a.cell[b0 + nbt - 1] : -1);
    const int rowkey = cfirst / nx;
    const int cxa = cfirst - rowkey * nx, cxb = clast - rowkey * nx;
    // fluid targets need both lists' rows; a pure-boundary block only the fluid rows
    const int nlist = nf ? 2 : 1;
    const int nseg = nlist * side * side;
    const int gcz = rowkey / ny, gcy = rowkey - gcz * ny;
    const int bxlo = max(cxa - reach, 0), bxhi = min(cxb + reach, nx - 1);
    // FP16 screen frame: block centre, unit = 2h (Cfg<float> only)
    const double cs = a.g.cell_size;
    const float h16_s = (float)(0.5 * a.p.invh);
    const float h16_xc = (float)(a.g.origin[0] + 0.5 * (bxlo + bxhi + 1) * cs);
    const float h16_yc = (float)(a.g.origin[1] + (gcy + 0.5) * cs);
    const float h16_zc = (float)(a.g.origin[2] + (gcz + 0.5) * cs);
    const bool use16 = Cfg<R>::H16 && (0.5 * (bxhi - bxlo + 1) * cs * (0.5 * a.p.invh) <= H16_MAXABS) &&
                       ((reach + 0.5) * cs * (0.5 * a.p.invh) <= H16_MAXABS);

    // ---- stencil row segments in the reference's traversal order + their prefix
    if (tid < MAXSEG) {
      int len = 0;
      Seg sg = {0, 0, 0, 0};
      if (tid < nseg) {
        int li, rr;
        if (nlist == 2 && a.p.order == 1) {  // gather_fluid_ranges: all F rows, then all B rows
          li = tid / (side * side);
          rr = tid - li * side * side;
        } else {                              // gather_*_cells: per row F then B
          li = tid % nlist;
          rr = tid / nlist;
        }
        const int dz = rr / side - reach, dy = rr % side - reach;
        const int zz = gcz + dz, yy = gcy + dy;
        if (zz >= 0 && zz < nz && yy >= 0 && yy < ny) {
          const int64_t rowoff = (li == 0 ? a.ncells : 0) + (int64_t)nx * (yy + (int64_t)ny * zz);
          sg.g0 = a.beg[rowoff + bxlo];
          sg.g1 = a.end[rowoff + bxhi];
          sg.rowoff = (int)rowoff;  // < 2^31 (ncells < 2^30)
          len = max(sg.g1 - sg.g0, 0);
          if (len == 0) sg.g1 = sg.g0;
        }
      }
      s_scan[tid] = len;
      sSeg[tid] = sg;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of MAXSEG (=128) lengths, 4 per lane
      int v[4], run = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = s_scan[lane * 4 + k];
        run += v[k];
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(SPHB_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      int ex = incl - run;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        sSeg[lane * 4 + k].pos = ex;
        ex += v[k];
      }
      if (lane == 31) s_nseg_tot = incl;
    }
    __syncthreads();
    const int total = s_nseg_tot;

    // ---- this warp's targets
    const int t = warp * 32 + lane;                 // fluid targets first, then boundary
    const bool isf = t < nf;
    const int i = isf ? f0 + t : b0 + (t - nf);
    const bool valid = t < nf + nbt;
    const bool wactive = warp * 32 < nf + nbt;
    Own<R> o;
    int xlo = 0, xhi = -1;
    if (valid) {
      const float4 pi = a.posp[i], vi = a.velr[i], xi = a.aux[i];
      o.x = (R)pi.x; o.y = (R)pi.y; o.z = (R)pi.z;
      o.vx = (R)vi.x; o.vy = (R)vi.y; o.vz = (R)vi.z; o.rho = (R)vi.w;
      o.prrho = (R)pi.w; o.cs = (R)xi.y; o.ten = (R)xi.z;
      const int cxi = a.cell[i] - rowkey * nx;
      xlo = max(cxi - reach, 0);
      xhi = min(cxi + reach, nx - 1);
    } else {
      o.x = o.y = o.z = o.vx = o.vy = o.vz = o.prrho = o.cs = o.ten = (R)0;
      o.rho = (R)1;
    }
    const int wxlo = __reduce_min_sync(SPHB_FULL, valid ? xlo : INT_MAX);
    const int wxhi = __reduce_max_sync(SPHB_FULL, valid ? xhi : INT_MIN);
    Accum<R> s = {(R)0, (R)0, (R)0, (R)0, (R)0};
    uint32_t tail = 0, pend = 0, pushed = 0, pushed_b = 0, rej = 0, rej_f = 0;
    unsigned long long cand = 0;
    if (valid) {  // candidate count = sum of this lane's row-range lengths
      for (int k = 0; k < nseg; ++k) {
        const Seg sg = sSeg[k];
        if (sg.g1 <= sg.g0) continue;
        if (!isf && sg.rowoff < a.ncells) continue;  // boundary targets: fluid rows only
        cand += (unsigned long long)(a.end[sg.rowoff + xhi] - a.beg[sg.rowoff + xlo]);
      }
      if (isf) cand -= 1;  // the reference skips j == i before counting (kernels.py:369-371)
    }

    // Lock-step FIFO drain.  Each lane queued only its non-empty mask words (with the staged
    // index of the word's first candidate), so a pop refills at most once and never loops.
    const uint32_t smA = pin_u32(smem_addr(g_sm4)), smB = pin_u32(smA + 16u * SB);
    const uint32_t smC = pin_u32(smA + 16u * SC);
    const uint32_t smMask = pin_u32(smem_addr(myMask) + 4u * lane);
    const uint32_t smBase = pin_u32(smem_addr(myBase) + 2u * lane);
    const uint32_t smH = pin_u32(smA + 16u * Cfg<R>::NARR * SCAP);
    const __half2 thr16 = __float2half2_rn(H16_THR);
    const __half2 ohx = __float2half2_rn(((float)o.x - h16_xc) * h16_s);
    const __half2 ohy = __float2half2_rn(((float)o.y - h16_yc) * h16_s);
    const __half2 ohz = __float2half2_rn(((float)o.z - h16_zc) * h16_s);
    auto drain = [&]() {
      __syncwarp();
      const uint32_t mx = __reduce_max_sync(SPHB_FULL, pend);
      uint32_t head = 0, cur = 0;
      int cbase = 0;
      auto pop = [&]() -> int {
        if (cur == 0u && head < tail) {
          cur = lds32(smMask + 128u * head);
          cbase = (int)lds16(smBase + 64u * head);
          ++head;
        }
        const int t = __ffs(cur) - 1;  // -1 when empty
        cur &= cur - 1u;
        return t < 0 ? -1 : cbase + t;
      };
      for (uint32_t it = 0; it < mx; it += 2) {
        const int k1 = pop();
        const int k2 = pop();
        rej += eval_two<G7, EQM>(a, c32, o, smA, smB, smC, k1, k2, xlo, xhi, s, &rej_f);
      }
      tail = 0;
      pend = 0;
      __syncwarp();
    };

    // ---- batches of <= SCAP staged candidates (normally one)
    for (int q0 = 0; q0 < total; q0 += SCAP) {
      const int q1 = min(q0 + SCAP, total);
      // stage [q0, q1): thread-strided, monotone segment cursor
      {
        int sk = 0;
        for (int p = q0 + tid; p < q1; p += NW * 32) {
          while (sSeg[sk].pos + (sSeg[sk].g1 - sSeg[sk].g0) <= p) ++sk;
          const Seg sg = sSeg[sk];
          const int j = sg.g0 + (p - sg.pos);
          const float4 pp = __ldg(&a.posp[j]);
          const float4 vr = __ldg(&a.velr[j]);
          const float4 xa = __ldg(&a.aux[j]);
          const bool boundary_list = sg.rowoff < a.ncells;
          g_sm4[p - q0] = pp;  // (x, y, z, prrho)
          g_sm4[SB + p - q0] = make_float4(vr.x, vr.y, vr.z, boundary_list ? -vr.w : vr.w);
          if (sizeof(R) == 8) g_sm4[SC + p - q0] = make_float4(xa.y, xa.z, 0.f, 0.f);
          if (Cfg<R>::H16) {
            __half* h = reinterpret_cast<__half*>(g_sm4 + Cfg<R>::NARR * SCAP);
            h[p - q0] = __float2half_rn((pp.x - h16_xc) * h16_s);
            h[SCAP + p - q0] = __float2half_rn((pp.y - h16_yc) * h16_s);
            h[2 * SCAP + p - q0] = __float2half_rn((pp.z - h16_zc) * h16_s);
          }
        }
      }
      __syncthreads();
      if (wactive) {
        for (int k = 0; k < nseg; ++k) {
          const Seg sg = sSeg[k];
          const int len = sg.g1 - sg.g0;
          if (len <= 0 || sg.pos >= q1 || sg.pos + len <= q0) continue;
          // this warp's part of the row: cells [wxlo, wxhi]
          const int wg0 = a.beg[sg.rowoff + wxlo], wg1 = a.end[sg.rowoff + wxhi];
          const int lo = max(sg.pos + (wg0 - sg.g0), q0) - q0;
          const int hi = min(sg.pos + (wg1 - sg.g0), q1) - q0;
          if (hi <= lo) continue;
          const bool boundary_list = sg.rowoff < a.ncells;
          int la = 0, lb = 0;  // FP64: this lane's own stencil range, staged coordinates
          if (sizeof(R) == 8 && valid) {
            la = sg.pos + (a.beg[sg.rowoff + xlo] - sg.g0) - q0;
            lb = sg.pos + (a.end[sg.rowoff + xhi] - sg.g0) - q0;
          }
          const int lo8 = use16 ? (lo & ~7) : lo;  // FP16 loads are 8-candidate aligned
          for (int k0 = lo8; k0 < hi; k0 += 32) {
            uint32_t bits = 0;
            if (use16) {
              const uint32_t hx = smH + 2u * k0, hy = hx + 2u * SCAP, hz = hy + 2u * SCAP;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint4 vx = lds128u(hx + 16u * q), vy = lds128u(hy + 16u * q),
                            vz = lds128u(hz + 16u * q);
                const uint32_t ux[4] = {vx.x, vx.y, vx.z, vx.w}, uy[4] = {vy.x, vy.y, vy.z, vy.w},
                               uz[4] = {vz.x, vz.y, vz.z, vz.w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                  const __half2 dx = __hsub2(ohx, u32_as_h2(ux[w]));
                  const __half2 dy = __hsub2(ohy, u32_as_h2(uy[w]));
                  const __half2 dz = __hsub2(ohz, u32_as_h2(uz[w]));
                  const __half2 r2 = __hfma2(dz, dz, __hfma2(dy, dy, __hmul2(dx, dx)));
                  const uint32_t m = __hlt2_mask(r2, thr16);
                  const int t = q * 8 + w * 2;
                  bits |= ((m & 1u) << t) | (((m >> 16) & 1u) << (t + 1));
                }
              }
              if (k0 < lo) bits &= 0xffffffffu << (lo - k0);
            } else {
              const uint32_t sk = smA + 16u * k0;
#pragma unroll
              for (int t = 0; t < 32; ++t) {
                const float4 A = lds4(sk + 16u * t);  // reads past hi stay inside shared memory
                if (screen(a, c32, o, A)) bits |= 1u << t;
              }
            }
            const int nvalid = hi - k0;
            if (nvalid < 32) bits &= (1u << nvalid) - 1u;
            if (sizeof(R) == 8) {  // exact stencil bounds for the FP64 (no guard band) path
              const int d0 = la - k0, d1 = lb - k0;
              const uint32_t m0 = d0 <= 0 ? 0xffffffffu : (d0 >= 32 ? 0u : (0xffffffffu << d0));
              const uint32_t m1 = d1 >= 32 ? 0xffffffffu : (d1 <= 0 ? 0u : ((1u << d1) - 1u));
              bits &= m0 & m1;
            }
            bits = (valid && (isf || !boundary_list)) ? bits : 0u;  // B-B pairs are never visited
            if (__any_sync(SPHB_FULL, bits != 0u && tail == (uint32_t)RING)) drain();
            if (bits) {
              sts32(smMask + 128u * tail, bits);
              sts16(smBase + 64u * tail, (uint32_t)k0);
              ++tail;
              const uint32_t pc = __popc(bits);
              pend += pc;
              pushed += pc;
              if (boundary_list) pushed_b += pc;
            }
          }
        }
        drain();
      }
      __syncthreads();  // staging buffer reuse
    }

    if (valid) {
      c_cand += cand;
      c_hits += pushed - rej;
      if (isf) c_ff += (pushed - pushed_b) - rej_f;
      if (sizeof(R) == 4 && EQM) {  // the pair loop left the (equal) neighbour mass out
        s.ax *= (R)a.massf;
        s.ay *= (R)a.massf;
        s.az *= (R)a.massf;
        s.dr *= (R)a.massf;
      }
      const double ax = (double)s.ax, ay = (double)s.ay, az = (double)s.az;
      const double dr = (double)s.dr, vd = (double)s.vd;
      if (isf) {
        a.acc[3 * (int64_t)i + 0] = ax;
        a.acc[3 * (int64_t)i + 1] = ay;
        a.acc[3 * (int64_t)i + 2] = az;
      } else {
        a.acc[3 * (int64_t)i + 0] = 0.0;
        a.acc[3 * (int64_t)i + 1] = 0.0;
        a.acc[3 * (int64_t)i + 2] = 0.0;
      }
      a.drho[i] = dr;
      a.visc[i] = vd;
      if (!(isfinite(ax) && isfinite(ay) && isfinite(az) && isfinite(dr)))
        raise_div(a.ctrl, step, SPHB_DIV_NONFINITE_FORCES, 0);
      // compute_dt terms (sim.py:222-229); min is order-free so this is exact
      if (isf) {
        const double fx = xadd(ax, a.p.g[0]), fy = xadd(ay, a.p.g[1]), fz = xadd(az, a.p.g[2]);
        double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
        fmag = fmag > 1e-30 ? fmag : 1e-30;
        dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(a.p.h, fmag)));
      }
      dtcv_min = fmin(dtcv_min, xdiv(a.p.h, xadd((double)o.cs, vd)));
    }
  }

  dtf_min = warp_min(dtf_min);
  dtcv_min = warp_min(dtcv_min);
  c_cand = warp_sum_u64(c_cand);
  c_hits = warp_sum_u64(c_hits);
  c_ff = warp_sum_u64(c_ff);
  if (lane == 0) {
    if (dtf_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_f, dtf_min);
    if (dtcv_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_cv, dtcv_min);
    if (c_cand) atomicAdd((unsigned long long*)&a.ctrl->counters[0], c_cand);
    if (c_hits) {
      atomicAdd((unsigned long long*)&a.ctrl->counters[1], c_hits);
      atomicAdd((unsigned long long*)&a.ctrl->counters[2], c_hits);
    }
    if (c_ff) atomicAdd((unsigned long long*)&a.ctrl->counters[3], c_ff);
  }
}

// ====================================================================== FP32 kernel (v8)
// Same block decomposition and FIFO discipline as k_interact, retuned for sm_100a
// (DESIGN.md §4):
//   * staging: one TMA bulk copy (cp.async.bulk + mbarrier) per stencil row and array of the
//     K3-sorted rows (x, y, z, prrho | vx, vy, vz, rho), then 8-B FP16 screen records
//     (x, y, z, |x|^2 in block-centred units of 2h) built from shared memory;
//   * screen on the tensor cores: r^2 - thr = |x_j|^2 - 2 x_i.x_j + |x_i|^2 - thr for 32 targets
//     x 32 candidates per warp as 8 HMMA.1688 (FP32 accumulation); the sign bits are packed
//     (F2FP + sign-replicating PRMT) and routed to the target lanes by a quad byte transpose,
//     bit b <-> candidate k0 + b; the target itself is cleared from its own row's mask;
//   * FIFO entries are (mask, staged row address) pairs in a circular 20-entry ring per lane; a
//     full ring triggers a partial drain sized to the lightest busy lane;
//   * pair math: 3 independent groups of 2 popped candidates per lane per iteration, each one
//     packed FP32x2 chain (FFMA2/FADD2/FMUL2), constants folded (-alpha h into cs, W(dp)^-4
//     into the tensile factors, kc/h and the neighbour mass into the mask factor), viscosity as
//     max(., 0) (the term is positive iff v.r < 0); masked slots read a far dummy row and are
//     zeroed through the mask factor;
//   * exactness: FP32 r^2 within 5e-7 of sup2 (or coincident) is re-decided with the
//     reference's f64 predicate, one slot per lane per round;
//   * counters: hits per lane accumulate in a packed float; ff = sum over fluid targets minus
//     sum over boundary targets (F-B and B-F hit sets are mirror images).
// Accumulation order differs from the reference inside each 32-candidate word only; the
// FP32 path's contract is rel 1e-5 (the FP64 path above stays bit-exact).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2_t bc(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ void lds_2x64(uint32_t addr, f2_t& a, f2_t& b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}
__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, no slow path
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint2 lds64u(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts64u(uint32_t addr, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(x), "r"(y));
}
// sign-replicating byte permute: result byte n = 0xff if the msb of the selected byte is set
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// D = A B + C, m16n8k8, FP16 operands, FP32 accumulation (warp-wide)
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0,
                                          const float (&c)[4]) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
      "{%7, %8, %9, %10};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}
__device__ __forceinline__ uint32_t h2u(__half2 h) {
  uint32_t u;
  memcpy(&u, &h, 4);
  return u;
}
__device__ __forceinline__ int flo32(uint32_t v) {  // index of the highest set bit, -1 if none
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t clear_bit(uint32_t v, int t) {  // bit t is set; t = -1: v
  uint32_t m;
  asm("shl.b32 %0, 1, %1;" : "=r"(m) : "r"(t));
  return v ^ m;
}

struct K32 {  // folded FP32 constants of the v8 pair loop
  float sup2_lo, sup2_hi, tiny, invh, eta2, kcs, tpos, tneg, nkgc, nkgc_b, cs_exp, ktw4;
};

struct Own32 {
  f2_t xy, vxy;
  float x, y, z, vz, rho, prrho, csn, tenk;  // csn = -alpha h cs_i, tenk = tensil_i / W(dp)^4
};

struct Acc32 {
  f2_t axy, az, dr, hits, hitsf;  // hitsf: hits on fluid candidates (symmetric build only)
  float vd;
};

constexpr int V8_ROWS = V8_SCAP + 8;  // staged rows: SCAP candidates + the dummy (row SCAP)
// dynamic shared memory of k_interact_v8: A rows | B rows | screen records (8 B) | 64 B of
// zeros (B fragments of the K = 4..7 lanes) | FIFO
#ifndef V8_RING
#define V8_RING 20
#endif
constexpr int V8_REC_OFF = 32 * V8_ROWS;
constexpr int V8_ZERO_OFF = V8_REC_OFF + 8 * V8_SCAP;
constexpr int V8_FIFO_OFF = V8_ZERO_OFF + 64;
// symmetric build (K5s, SPHB_SYM): per staged row the reactions it receives from this block's
// targets, float4 (ax, ay, az, drho) + u32 (visc bits), flushed to global memory per batch
#ifndef SPHB_SYM
#define SPHB_SYM 0
#endif
constexpr bool V8_SYM = SPHB_SYM != 0;
constexpr int V8_ACC_OFF = V8_FIFO_OFF + 8 * NW * V8_RING * 32;
constexpr int V8_VD_OFF = V8_ACC_OFF + (V8_SYM ? 16 * V8_ROWS : 0);
constexpr int V8_SMEM = V8_VD_OFF + (V8_SYM ? 4 * V8_ROWS : 0);
// tensor-core screen: D = |x_j|^2 - 2 x_i.x_j + (|x_i|^2 - thr) in units of (2h)^2 from FP16
// block-centred coordinates (|x| <= 4, |x|^2 < 32): coordinate rounding moves r^2 by <= 6.8e-3
// at the cutoff and the FP16 |x_j|^2 by <= 7.8e-3, so thr = 1.02 never drops a true hit
constexpr float MMA_THR = 1.02f;
#ifndef V8_NG
#define V8_NG 2    // candidate pairs per lane per drain iteration (independent FP32x2 chains;
                   // 2 beat 3 by ~1% at C3: 185 vs 217 registers)
#endif
#ifndef V8_KMIN
#define V8_KMIN 8  // minimum iterations of a partial drain
#endif
// a partial drain pops >= 2 NG KMIN maybes per busy lane, i.e. frees at least its oldest word
static_assert(2 * V8_NG * V8_KMIN >= 32, "partial drains must free a FIFO entry");

// NG groups of two popped candidates (staged byte addresses of their A rows) of one lane.
// Each group is one packed FP32x2 chain; the groups are independent (ILP), and the rare
// exact re-decision is one warp-uniform branch for all of them.
// r2 inside the FP32 guard band [sup2_lo, sup2_hi) or coincident (r2 <= tiny)
__device__ __forceinline__ bool in_cold(float r2, const K32& c) {
  const uint32_t b = __float_as_uint(r2);
  return (b - __float_as_uint(c.sup2_lo) < __float_as_uint(c.sup2_hi) - __float_as_uint(c.sup2_lo)) |
         (b <= __float_as_uint(c.tiny));
}

// sure hit: tiny < r2 < sup2_lo, one unsigned compare of the (non-negative) float bits
__device__ __forceinline__ bool is_sure(float r2, const K32& c) {
  const uint32_t t = __float_as_uint(c.tiny);
  return __float_as_uint(r2) - (t + 1u) < __float_as_uint(c.sup2_lo) - (t + 1u);
}

struct Geo2 {
  f2_t a1xy, a1zw, b1zw, a2xy, a2zw, b2zw, dxy1, dxy2, dz, r2, dot;
};

// Symmetric build: where a pair's reaction goes.  The staged row's accumulators (float4 +
// u32) receive -ratio * (i-side force term), ratio * (i-side drho term) and |mu|, ratio =
// m_i / m_j (1 with equal masses: the masses are applied once, at the flush).
struct SymCtx {
  uint32_t smA, acc, vd;   // shared addresses: staged A rows, reaction rows, visc rows
  float ratio_f, ratio_b;  // m_i / m_j for a fluid / boundary candidate
};

__device__ __forceinline__ void sym_react(const SymCtx& y, uint32_t ad, float fx, float fy,
                                          float fz, float dr, float mu) {
  const bool jb = ad & 1u;  // boundary candidate: drho and visc only (accel stays 0)
  const uint32_t row = ((ad & ~1u) - y.smA) >> 4;
  const float r = jb ? y.ratio_b : y.ratio_f;
  float* acc = reinterpret_cast<float*>(__cvta_shared_to_generic(y.acc + 16u * row));
  if (!jb) {
    atomicAdd(acc + 0, -r * fx);
    atomicAdd(acc + 1, -r * fy);
    atomicAdd(acc + 2, -r * fz);
  }
  atomicAdd(acc + 3, r * dr);
  atomicMax(reinterpret_cast<unsigned*>(__cvta_shared_to_generic(y.vd + 4u * row)),
            __float_as_uint(mu));
}

template <bool G7, bool EQM, bool WEND, int NG>
__device__ __forceinline__ void eval_v8(const KArgs& a, const K32& c, const Own32& o,
                                        const uint32_t (&ad)[2 * NG], int xlo, int xhi,
                                        Acc32 (&s)[NG], const SymCtx& sy) {
  constexpr uint32_t OFFB = 16u * V8_ROWS;  // A -> B rows
  Geo2 g[NG];
  // the sure-hit mask and the clamped r2 live in float registers across the (rare) exact
  // branch, so the hot path carries no predicate / byte juggling
  float okf[2 * NG], r2m[2 * NG];
  bool anycold = false;
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    f2_t b1xy, b2xy;
    // non-EQM: bit 0 of a popped address flags a boundary-list candidate (its mass)
    const uint32_t p1 = (EQM && !V8_SYM) ? ad[2 * k] : (ad[2 * k] & ~1u),
                   p2 = (EQM && !V8_SYM) ? ad[2 * k + 1] : (ad[2 * k + 1] & ~1u);
    lds_2x64(p1, g[k].a1xy, g[k].a1zw);
    lds_2x64(p2, g[k].a2xy, g[k].a2zw);
    lds_2x64(p1 + OFFB, b1xy, g[k].b1zw);
    lds_2x64(p2 + OFFB, b2xy, g[k].b2zw);
    g[k].dxy1 = sub2(o.xy, g[k].a1xy);
    g[k].dxy2 = sub2(o.xy, g[k].a2xy);
    const f2_t dvxy1 = sub2(o.vxy, b1xy), dvxy2 = sub2(o.vxy, b2xy);
    const f2_t sq1 = mul2(g[k].dxy1, g[k].dxy1), sq2 = mul2(g[k].dxy2, g[k].dxy2);
    const f2_t dd1 = mul2(dvxy1, g[k].dxy1), dd2 = mul2(dvxy2, g[k].dxy2);
    g[k].dz = pk(o.z - lo(g[k].a1zw), o.z - lo(g[k].a2zw));
    const f2_t dvz = pk(o.vz - lo(g[k].b1zw), o.vz - lo(g[k].b2zw));
    g[k].r2 = fma2(g[k].dz, g[k].dz, pk(lo(sq1) + hi(sq1), lo(sq2) + hi(sq2)));
    g[k].dot = fma2(dvz, g[k].dz, pk(lo(dd1) + hi(dd1), lo(dd2) + hi(dd2)));
    // sure hit: r2 < sup2_lo (an empty slot reads the dummy row, r2 ~ 1e8 sup2: never a hit);
    // cold (exact f64 re-decision): r2 in [sup2_lo, sup2_hi) or r2 <= tiny, tested as
    // unsigned ranges of the (non-negative) float bits; a cold slot is not a sure hit
    const float r21 = lo(g[k].r2), r22 = hi(g[k].r2);
    const bool s1 = is_sure(r21, c), s2 = is_sure(r22, c);
    const bool c1 = !s1 & (r21 < c.sup2_hi), c2 = !s2 & (r22 < c.sup2_hi);
    okf[2 * k] = s1 ? 1.0f : 0.0f;
    okf[2 * k + 1] = s2 ? 1.0f : 0.0f;
    r2m[2 * k] = s1 ? r21 : c.sup2_lo;
    r2m[2 * k + 1] = s2 ? r22 : c.sup2_lo;
    anycold |= c1 | c2;
  }
  if (__any_sync(SPHB_FULL, anycold)) {
    // guard band / coincident (lattice ties sit on the cutoff): exact f64 decision, one
    // candidate per lane per round so the f64 path is issued once, not once per slot
    uint32_t cm = 0;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      cm |= (in_cold(lo(g[k].r2), c) ? 1u : 0u) << (2 * k);
      cm |= (in_cold(hi(g[k].r2), c) ? 1u : 0u) << (2 * k + 1);
    }
    // (in_cold == !is_sure && r2 < sup2_hi: r2 in [sup2_lo, sup2_hi) or r2 <= tiny)
    uint32_t accm = 0;  // accepted cold slots
    do {
      const int k = __ffs(cm) - 1;
      // the popped address by explicit selects (an indexed pick keeps the pops in local memory)
      uint32_t adk = ad[0];
#pragma unroll
      for (int kk = 1; kk < 2 * NG; ++kk) {
        const uint32_t hit = (uint32_t)(k == kk);
        asm("{ .reg .pred q; setp.ne.u32 q, %2, 0; selp.b32 %0, %1, %0, q; }"
            : "+r"(adk) : "r"(ad[kk]), "r"(hit));
      }
      bool acc = false;
      if (cm) {
        const float4 A = lds4(adk & ~1u);
        acc = cold_accept(a, o.x, o.y, o.z, A, xlo, xhi);
        cm &= cm - 1u;
      }
      accm |= acc ? 1u << k : 0u;
    } while (__any_sync(SPHB_FULL, cm != 0u));
#pragma unroll
    for (int kk = 0; kk < NG; ++kk) {  // once after the rounds, not once per round
      if ((accm >> (2 * kk)) & 1u) {
        okf[2 * kk] = 1.0f;
        r2m[2 * kk] = lo(g[kk].r2);
      }
      if ((accm >> (2 * kk + 1)) & 1u) {
        okf[2 * kk + 1] = 1.0f;
        r2m[2 * kk + 1] = hi(g[kk].r2);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const f2_t OK = pk(okf[2 * k], okf[2 * k + 1]);
    const f2_t R2M = pk(r2m[2 * k], r2m[2 * k + 1]);
    const f2_t RINV = pk(rsqrtf(lo(R2M)), rsqrtf(hi(R2M)));
    const f2_t Q = mul2(mul2(R2M, RINV), bc(c.invh));
    f2_t W, DWR;  // kernel shape W/kc and the gradient shape (-gc / mask factor)
    if (WEND) {   // Wendland C2: W = kc t^4 (2q + 1), gc = -5 kc t^3 / h^2, t = 1 - q/2
      const f2_t T = fma2(Q, bc(-0.5f), bc(1.0f));
      const f2_t T2 = mul2(T, T);
      W = mul2(mul2(T2, T2), fma2(Q, bc(2.0f), bc(1.0f)));
      DWR = mul2(T2, T);
    } else {      // cubic spline (physics.py:196-205)
      const f2_t T = sub2(bc(2.0f), Q);
      const f2_t UM = sub2(Q, bc(1.0f));
      const f2_t UN = pk(fminf(lo(UM), 0.0f), fminf(hi(UM), 0.0f));  // -max(1 - q, 0)
      const f2_t T2Q = mul2(mul2(T, T), bc(0.25f));
      const f2_t U2 = mul2(UN, UN);
      W = fma2(T2Q, T, mul2(U2, UN));      // t^3/4 - u^3
      DWR = mul2(sub2(U2, T2Q), RINV);     // (3 u^2 - 3/4 t^2) / (3 r)
    }
    const float sr1 = hi(g[k].b1zw), sr2 = hi(g[k].b2zw);
    const float rj1 = fabsf(sr1), rj2 = fabsf(sr2);
    const f2_t RHOJ = pk(rj1, rj2);
    f2_t MJ;  // mask factor: ok * (-3 kc/h) [* m_j]
    if (EQM) {
      MJ = mul2(OK, bc(c.nkgc));
    } else {
      MJ = mul2(OK, pk((ad[2 * k] & 1u) ? c.nkgc_b : c.nkgc, (ad[2 * k + 1] & 1u) ? c.nkgc_b : c.nkgc));
    }
    const f2_t GCN = mul2(DWR, MJ);  // -gc [m_j], zero when masked
    f2_t CSJ;                                    // -alpha h cs_j
    if (G7) {
      const f2_t RR = mul2(RHOJ, bc(c.kcs));
      CSJ = mul2(mul2(RR, RR), RR);
    } else {
      CSJ = mul2(pk(exp2f(c.cs_exp * __log2f(rj1)), exp2f(c.cs_exp * __log2f(rj2))), bc(c.kcs));
    }
    const float pr1 = hi(g[k].a1zw), pr2 = hi(g[k].a2zw);
    const f2_t TENJ = pk(pr1 * (pr1 > 0.0f ? c.tpos : c.tneg), pr2 * (pr2 > 0.0f ? c.tpos : c.tneg));
    const f2_t PSUM = pk(o.prrho + pr1, o.prrho + pr2);
    const f2_t E = add2(R2M, bc(c.eta2));
    const f2_t MU = mul2(mul2(g[k].dot, pk(rcp_approx(lo(E)), rcp_approx(hi(E)))), OK);  // mu / h
    const f2_t RS = add2(RHOJ, bc(o.rho));
    const f2_t VT = mul2(mul2(add2(CSJ, bc(o.csn)), MU), pk(rcp_approx(lo(RS)), rcp_approx(hi(RS))));
    const f2_t VISC = pk(fmaxf(lo(VT), 0.0f), fmaxf(hi(VT), 0.0f));
    const f2_t W2 = mul2(W, W);
    const f2_t PT = fma2(mul2(add2(TENJ, bc(o.tenk)), W2), W2, add2(PSUM, VISC));
    const f2_t FM = mul2(PT, GCN);
    s[k].axy = fma2(g[k].dxy1, bc(lo(FM)), s[k].axy);
    s[k].axy = fma2(g[k].dxy2, bc(hi(FM)), s[k].axy);
    s[k].az = fma2(g[k].dz, FM, s[k].az);
    s[k].dr = fma2(GCN, g[k].dot, s[k].dr);
    s[k].vd = fmaxf(s[k].vd, fmaxf(fabsf(lo(MU)), fabsf(hi(MU))));
    s[k].hits = add2(s[k].hits, OK);
    if (V8_SYM) {
      // ff hits: fluid candidates (the target side is applied at the epilogue)
      s[k].hitsf = add2(s[k].hitsf, mul2(OK, pk((ad[2 * k] & 1u) ? 0.0f : 1.0f,
                                                  (ad[2 * k + 1] & 1u) ? 0.0f : 1.0f)));
      const f2_t DR = mul2(GCN, g[k].dot);
      if (okf[2 * k] != 0.0f)
        sym_react(sy, ad[2 * k], lo(g[k].dxy1) * lo(FM), hi(g[k].dxy1) * lo(FM), lo(g[k].dz) * lo(FM),
                  lo(DR), fabsf(lo(MU)));
      if (okf[2 * k + 1] != 0.0f)
        sym_react(sy, ad[2 * k + 1], lo(g[k].dxy2) * hi(FM), hi(g[k].dxy2) * hi(FM),
                  hi(g[k].dz) * hi(FM), hi(DR), fabsf(hi(MU)));
    }
  }
}

template <bool G7, bool EQM, bool WEND, bool WALL>
#ifndef V8_MINB
#define V8_MINB 2  // CTAs per SM: shared memory (V8_SMEM) and registers allow 2
#endif
__global__ void __launch_bounds__(NW * 32, V8_MINB) k_interact_v8(KArgs a, K32 k32) {
  if (!step_live(a.ctrl)) return;
  constexpr int SCAP = Cfg<float>::SCAP;
  constexpr int RINGC = V8_RING;                          // FIFO entries per lane (8 B)
  constexpr int MASK0 = V8_FIFO_OFF / 4;                 // uint32 offset of the FIFO
  __shared__ Seg sSeg[MAXSEG];
  __shared__ int s_blk, s_nseg_tot, s_scan[MAXSEG];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = a.g.dims[0], ny = a.g.dims[1], nz = a.g.dims[2];
  const int reach = a.g.reach, side = 2 * reach + 1;
  const uint32_t nblocks = a.ctrl->nblk[0];
  const int64_t step = a.ctrl->step;
  // the dummy row popped by empty FIFO slots: far away (r2 ~ 1e8 sup2), at rest, finite
  __shared__ __align__(8) unsigned long long s_mbar;
  const uint32_t mbar = smem_addr(&s_mbar);
  uint32_t mphase = 0;
  if (tid == 0) {
    const float far = (float)(1e4 * 2.0 * a.p.h);
    g_sm4[SCAP] = make_float4(far, far, far, 0.f);
    g_sm4[V8_ROWS + SCAP] = make_float4(0.f, 0.f, 0.f, 1.f);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  const uint32_t smA = pin_u32(smem_addr(g_sm4));
  const uint32_t smR = smA + V8_REC_OFF;  // screen records: half2 (x, y), half2 (z, |x|^2)
  const uint32_t dummy = smA + 16u * SCAP;
  if (tid < 16) g_sm32[V8_ZERO_OFF / 4 + tid] = 0u;
  if (V8_SYM)  // reaction rows start at zero; every flush re-zeroes the rows it drained
    for (int r = tid; r < 5 * V8_ROWS; r += NW * 32) g_sm32[V8_ACC_OFF / 4 + r] = 0u;
  // tensor-core screen lane roles: g = lane / 4 (fragment row / column), t = lane % 4
  const int fg = lane >> 2, ft = lane & 3;
  // B fragment (K rows 2t, 2t+1; column g of N-tile n <-> candidate 8 (g/2) + 2n + g%2):
  // t = 0 reads (x, y), t = 1 reads (z, |x|^2) of the record, t >= 2 reads zeros
  const uint32_t bl_off = ft < 2 ? 64u * (fg >> 1) + 8u * (fg & 1) + 4u * ft : 0u;
  const uint32_t bl_kmul = ft < 2 ? 8u : 0u;
  const uint32_t bl_base = ft < 2 ? smR : smA + V8_ZERO_OFF;
  // quad byte transpose selectors and the final route (lane r <- lane 4 (r % 8) + r / 8)
  const uint32_t tsel1 = (ft & 1) ? 0x3715u : 0x6240u;
  const uint32_t tsel2 = (ft & 2) ? 0x3276u : 0x5410u;
  const int troute = 4 * (lane & 7) + (lane >> 3);
  // FIFO: [NW][RINGC][32 lanes] of (mask u32, staged row address u32)
  const uint32_t ring = pin_u32(smem_addr(g_sm32 + MASK0) + 8u * (warp * RINGC * 32 + lane));
  const uint32_t rend = ring + 256u * RINGC;

  unsigned long long c_cand = 0, c_hits = 0;
  long long c_ff = 0;
  double dtf_min = INFINITY, dtcv_min = INFINITY;

  // block records are fetched one block ahead by thread 0 (the next record's L2 latency
  // overlaps the current block)
  __shared__ int4 s_bb[2];
  int4 nxt_b = make_int4(0, 0, 0, 0), nxt_m = make_int4(0, 0, 0, 0);
  uint32_t nxt = 0;
  if (tid == 0) {
    nxt = atomicAdd(&a.ctrl->tile_next[0], 1u);
    if (nxt < nblocks) {
      nxt_b = a.blocks[2 * nxt];
      nxt_m = a.blocks[2 * nxt + 1];
    }
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_blk = (int)nxt;
      s_bb[0] = nxt_b;
      s_bb[1] = nxt_m;
    }
    __syncthreads();
    if (tid == 0) {  // the next record: its atomic and loads overlap this block (not the barrier)
      nxt = atomicAdd(&a.ctrl->tile_next[0], 1u);
      if (nxt < nblocks) {
        nxt_b = a.blocks[2 * nxt];
        nxt_m = a.blocks[2 * nxt + 1];
      }
    }
    const uint32_t blk = (uint32_t)s_blk;
    if (blk >= nblocks) break;
    const int4 bb = s_bb[0], bm = s_bb[1];
    // brick block (h/2 cells, reach >= 2: bm.w = 1): rows (y0 + sy, z0 + sz), sy, sz in {0, 1},
    // over cells [cxa, cxb]; its targets are the four rows' fluid ranges, then their boundary
    // ranges (derived from beg / end below).  Row block (bm.w = 0): one row, ranges in bb.
    const bool brick = bm.w != 0;
    const int bsd = brick ? 2 : 1;  // rows per side of the block
    const int rowkey = bm.x;
    const int cxa = bm.y, cxb = bm.z;
    const int nlist = (brick || bb.y > bb.x) ? 2 : 1;
    // symmetric build: the own row (forward cells only, j > i per target) and the forward rows
    // (dz = 0, dy = 1..r; dz = 1..r, dy = -r..r): every unordered pair once, as
    // run_cells_symmetric / forward_offsets (kernels.py:121-175, grid.py:147-156)
    const int bside = side + bsd - 1;  // staged rows per side: 2r + 1 (row) / 2r + 2 (brick)
    const int nrow = V8_SYM ? 1 + reach + reach * side : bside * bside;
    const int nseg = nlist * nrow;
    const int gcz = rowkey / ny, gcy = rowkey - gcz * ny;
    const int bxlo = max(cxa - reach, 0), bxhi = min(cxb + reach, nx - 1);
    const double cs = a.g.cell_size;
    const float h16_s = (float)(0.5 * a.p.invh);
    const float h16_xc = (float)(a.g.origin[0] + 0.5 * (bxlo + bxhi + 1) * cs);
    const float h16_yc = (float)(a.g.origin[1] + (gcy + 0.5 * bsd) * cs);
    const float h16_zc = (float)(a.g.origin[2] + (gcz + 0.5 * bsd) * cs);
    const double xext = 0.5 * (bxhi - bxlo + 1) * cs * (0.5 * a.p.invh);
    const double yzext = (reach + 0.5 * bsd) * cs * (0.5 * a.p.invh);
    const bool use16 = xext <= H16_MAXABS && yzext <= H16_MAXABS &&
                       xext * xext + 2.0 * yzext * yzext < 30.0;
    // the fluid targets' own row (fluid list, dy = dz = 0)
    const int rr_c = reach * side + reach;
    const int selfseg = (bb.y > bb.x && !V8_SYM) ? ((nlist == 2 && a.p.order == 1) ? rr_c : rr_c * nlist) : -1;

    __shared__ int s_tlo[8], s_tlen[8];  // brick targets: F rows 0..3, then B rows 0..3
    if (brick && tid < 8) {
      const int li = tid >> 2, sub = tid & 3, yy = gcy + (sub & 1), zz = gcz + (sub >> 1);
      int lo = 0, len = 0;
      if (yy < ny && zz < nz) {
        const int64_t ro = (li == 0 ? a.ncells : 0) + (int64_t)nx * (yy + (int64_t)ny * zz);
        lo = a.beg[ro + cxa];
        len = max(a.end[ro + cxb] - lo, 0);
      }
      s_tlo[tid] = lo;
      s_tlen[tid] = len;
    }
    if (tid < MAXSEG) {
      int len = 0;
      Seg sg = {0, 0, 0, 0, 0};
      if (tid < nseg) {
        int li, rr;
        if (nlist == 2 && a.p.order == 1) {
          li = tid / (side * side);
          rr = tid - li * side * side;
        } else {
          li = tid % nlist;
          rr = tid / nlist;
        }
        int dz = rr / bside - reach, dy = rr % bside - reach, sxlo = bxlo;
        if (V8_SYM) {
          const int q = rr - 1 - reach;
          dz = rr == 0 ? 0 : (q < 0 ? 0 : 1 + q / side);
          dy = rr == 0 ? 0 : (q < 0 ? rr : q % side - reach);
          sxlo = rr == 0 ? cxa : bxlo;
        }
        const int zz = gcz + dz, yy = gcy + dy;
        if (zz >= 0 && zz < nz && yy >= 0 && yy < ny) {
          const int64_t rowoff = (li == 0 ? a.ncells : 0) + (int64_t)nx * (yy + (int64_t)ny * zz);
          sg.g0 = a.beg[rowoff + sxlo];
          sg.g1 = a.end[rowoff + bxhi];
          sg.rowoff = (int)rowoff;
          sg.dyz = (dy + 16) | ((dz + 16) << 8);
          len = max(sg.g1 - sg.g0, 0);
          if (len == 0) sg.g1 = sg.g0;
        }
      }
      s_scan[tid] = len;
      sSeg[tid] = sg;
    }
    __syncthreads();
    if (warp == 0) {
      int v[4], run = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = s_scan[lane * 4 + k];
        run += v[k];
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(SPHB_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      int ex = incl - run;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        sSeg[lane * 4 + k].pos = ex;
        ex += v[k];
      }
      if (lane == 31) s_nseg_tot = incl;
    }
    __syncthreads();
    const int total = s_nseg_tot;
    // the first staging batch goes out now: its bulk copies land while the lanes set up their
    // targets, windows and candidate counts (global loads)
    if (warp == 0 && total > 0)  // (no batch, no mbarrier phase: an empty block stages nothing)
      stage_batch(a.posp, a.velr, sSeg, nseg, 0, min(SCAP, total), smA, 16u * V8_ROWS, mbar, lane);

    const int t = warp * 32 + lane;
    int nf = bb.y - bb.x, nbt = bb.w - bb.z, i, rsy = 0, rsz = 0;
    if (brick) {  // lane t -> (sub-range, offset): fluid ranges first, then boundary ranges
      int pre = 0, kk = 0, lo = s_tlo[0];
      nf = s_tlen[0] + s_tlen[1] + s_tlen[2] + s_tlen[3];
      nbt = s_tlen[4] + s_tlen[5] + s_tlen[6] + s_tlen[7];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int len = s_tlen[k];
        if (t >= pre && t < pre + len) {
          kk = k;
          lo = s_tlo[k] + (t - pre);
        }
        pre += len;
      }
      i = lo;
      rsy = kk & 1;
      rsz = (kk >> 1) & 1;
    } else {
      i = t < nf ? bb.x + t : bb.z + (t - nf);
    }
    const bool isf = t < nf;
    const bool valid = t < nf + nbt;
    const bool wactive = warp * 32 < nf + nbt;
    // the lane's stencil rows among the staged ones (a brick stages the union of its rows')
    auto in_rows = [&](int dyz) {
      return abs((dyz & 255) - 16 - rsy) <= reach && abs((dyz >> 8) - 16 - rsz) <= reach;
    };
    // the fluid target's own row among the segments (brick: per lane)
    const int selfseg_l =
        !brick ? selfseg : ((rsz + reach) * bside + (rsy + reach)) * nlist;
    Own32 o;
    float ocs = 0.f;
    int xlo = 0, xhi = -1, cxi = INT_MAX;
    {
      float4 pi = make_float4(0.f, 0.f, 0.f, 0.f), vi = make_float4(0.f, 0.f, 0.f, 1.f),
             xi = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) {
        pi = a.posp[i];
        vi = a.velr[i];
        if (a.aux) {
          xi = a.aux[i];
        } else {  // no aux rows this step: the target's own csound / tensil
          const float2 ct = target_cs_tensil<G7>((double)vi.w, pi.w, a.inv_rho0, a.p);
          xi = make_float4(0.f, ct.x, ct.y, 0.f);
        }
        cxi = a.cell[i] - (rowkey + rsy + ny * rsz) * nx;
        xlo = max(cxi - reach, 0);
        xhi = min(cxi + reach, nx - 1);
      }
      o.x = pi.x; o.y = pi.y; o.z = pi.z; o.vz = vi.z; o.rho = vi.w;
      o.xy = pk(pi.x, pi.y);
      o.vxy = pk(vi.x, vi.y);
      o.prrho = pi.w;
      ocs = xi.y;
      o.csn = (float)(-a.p.alpha * a.p.h) * xi.y;
      o.tenk = xi.z * k32.ktw4;
    }
    const int wxlo = __reduce_min_sync(SPHB_FULL, valid ? xlo : INT_MAX);
    const int wxhi = __reduce_max_sync(SPHB_FULL, valid ? xhi : INT_MIN);
    // symmetric build: own-row lower bounds (global indices) -- fluid targets take fluid
    // candidates j > i and boundary candidates from their own cell on, boundary targets fluid
    // candidates from the next cell on (kernels.py:144-175); the warp's own-row window starts
    // at its lowest target cell
    int lbF = INT_MAX, lbB = INT_MAX;
    const int wcxlo = V8_SYM ? __reduce_min_sync(SPHB_FULL, valid ? cxi : INT_MAX) : 0;
    SymCtx sy = {0u, 0u, 0u, 1.0f, 1.0f};
    if (V8_SYM) {
      if (valid) {
        const int64_t rB = (int64_t)rowkey * nx, rF = a.ncells + rB;
        lbF = isf ? i + 1 : a.end[rF + cxi];
        lbB = isf ? a.beg[rB + cxi] : INT_MAX;
      }
      const float mi = isf ? (float)a.p.mass_fluid : (float)a.p.mass_boundary;
      sy.smA = smA;
      sy.acc = smA + V8_ACC_OFF;
      sy.vd = smA + V8_VD_OFF;
      sy.ratio_f = EQM ? 1.0f : mi / (float)a.p.mass_fluid;
      sy.ratio_b = EQM ? 1.0f : mi / (float)a.p.mass_boundary;
    }
    Acc32 s[V8_NG];
#pragma unroll
    for (int k = 0; k < V8_NG; ++k) {
      s[k].axy = s[k].az = s[k].dr = s[k].hits = s[k].hitsf = bc(0.0f);
      s[k].vd = 0.0f;
    }
    unsigned long long cand = 0;
    if (valid && V8_SYM) {  // the gather traversal's candidate count (full stencil rows)
      for (int dz = -reach; dz <= reach; ++dz) {
        const int zz = gcz + dz;
        if (zz < 0 || zz >= nz) continue;
        for (int dy = -reach; dy <= reach; ++dy) {
          const int yy = gcy + dy;
          if (yy < 0 || yy >= ny) continue;
          const int64_t rb = (int64_t)nx * (yy + (int64_t)ny * zz), rf = a.ncells + rb;
          cand += (unsigned long long)(a.end[rf + xhi] - a.beg[rf + xlo]);
          if (isf) cand += (unsigned long long)(a.end[rb + xhi] - a.beg[rb + xlo]);
        }
      }
      if (isf) cand -= 1;
    }  // (gather builds: counted from the cell tables, k_blocks' count pass)

    // A / C fragments of the tensor-core screen: target row r = 16 m + g (+ 8) holds
    // K = (-2x, -2y, -2z, 1, 0, 0, 0, 0) and C = |x|^2 - thr of its FP16 block-centred position
    uint32_t fa[2][2];
    float fc[2][4];
    {
      const __half hx = __float2half_rn((o.x - h16_xc) * h16_s);
      const __half hy = __float2half_rn((o.y - h16_yc) * h16_s);
      const __half hz = __float2half_rn((o.z - h16_zc) * h16_s);
      const float fx = __half2float(hx), fy = __half2float(hy), fz = __half2float(hz);
      const uint32_t alo = h2u(__floats2half2_rn(-2.0f * fx, -2.0f * fy));
      const uint32_t ahi = h2u(__floats2half2_rn(-2.0f * fz, 1.0f));
      const float cv = fmaf(fz, fz, fmaf(fy, fy, fx * fx)) - MMA_THR;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 16 * m + 8 * h + fg;
          const uint32_t vlo = __shfl_sync(SPHB_FULL, alo, r), vhi = __shfl_sync(SPHB_FULL, ahi, r);
          fa[m][h] = ft == 0 ? vlo : (ft == 1 ? vhi : 0u);
          const float c = __shfl_sync(SPHB_FULL, cv, r);
          fc[m][2 * h] = c;
          fc[m][2 * h + 1] = c;
        }
      }
    }

    // Per-lane circular FIFO of non-empty screen words: (mask, staged row address).  A
    // partial drain runs K lock-step iterations of 2*V8_NG pops per lane; pend counts the
    // lane's queued maybes (every pop yields one while pend > 0).
    // Entries are (mask, row address) pairs, 8 B, RINGC per lane; hp / tp are the lane's read
    // and write entry addresses (stride 256 B: 32 lanes), cnt the entries queued.  An
    // exhausted FIFO points cb one row past the dummy: the empty pop (bfind = -1) lands on it.
    // Symmetric build: masks are queued rotated left by the lane index, so lanes holding the
    // same word (neighbouring targets share most candidates) pop different candidates in the
    // same iteration -- their reactions then hit different shared-memory rows (no CAS
    // contention).  rot = 0 in the gather builds (pop order = staged order).
    const uint32_t rot = V8_SYM ? (uint32_t)lane : 0u;
    // an empty pop (bfind = -1) must land on the dummy row: b = 31 - rot rotated, -1 plain
    const uint32_t dummy_cb = V8_SYM ? dummy - 16u * (31u - rot) : dummy + 16u;
    uint32_t hp = ring, tp = ring, cnt = 0, pend = 0, cur = 0u, cb = dummy_cb;
    // the head entry is held in registers (nx_mask, nx_cb): a refill is a register move plus
    // the load of the following entry, which has several pops to land
    uint32_t nx_mask = 0u, nx_cb = 0u;
    auto pop = [&]() -> uint32_t {
      const bool need = cur == 0u, have = cnt != 0u;
      if (need & have) {
        cur = nx_mask;
        cb = nx_cb;
        hp = hp + 256u == rend ? ring : hp + 256u;
        --cnt;
        const uint2 e = lds64u(hp);  // stale when the ring just emptied: never used then
        nx_mask = e.x;
        nx_cb = e.y;
      }
      cb = (need & !have) ? dummy_cb : cb;
      const int tb = flo32(cur);
      cur = clear_bit(cur, tb);
      // bit b <-> candidate k0 + b (rotated: b = tb - rot); empty (tb = -1) -> the dummy
      if (V8_SYM) return cb + 16u * (((uint32_t)tb - rot) & 31u);
      return cb + 16u * (uint32_t)tb;
    };
    auto drain = [&](bool full) {
      __syncwarp();
      {
        const uint2 e = lds64u(hp);  // (re)load the head entry: pushes may have refilled the ring
        nx_mask = e.x;
        nx_cb = e.y;
      }
      constexpr uint32_t P = 2 * V8_NG;  // pops per lane per iteration
      const uint32_t mx = __reduce_max_sync(SPHB_FULL, pend);
      uint32_t K = (mx + P - 1) / P;
      if (!full) {  // enough to free ring space without idling the lightest busy lane
        const uint32_t mn = __reduce_min_sync(SPHB_FULL, pend ? pend : 0xffffffffu);
        K = min(K, max((mn + P - 1) / P, (uint32_t)V8_KMIN));
      }
      for (uint32_t it = 0; it < K; ++it) {
        uint32_t ad[2 * V8_NG];
#pragma unroll
        for (int k = 0; k < 2 * V8_NG; ++k) ad[k] = pop();
        eval_v8<G7, EQM, WEND, V8_NG>(a, k32, o, ad, xlo, xhi, s, sy);
      }
      pend = pend > P * K ? pend - P * K : 0u;
      __syncwarp();
    };

    // The warp's part of every staged row: cells [wxlo, wxhi] (symmetric own row: from its
    // lowest target cell), as staged positions [wpos0, wpos1) -- computed once per block, the
    // lanes' global loads in parallel (lane l: rows l, l + 32, ...) -- and which rows some lane
    // of the warp needs (a brick's lanes sit in up to four rows: the warp's set wrows)
    int wpos0[MAXSEG / 32], wpos1[MAXSEG / 32];
    uint32_t wlive = 0;
    {
      const uint32_t mine = valid ? 1u << (rsy + 2 * rsz) : 0u;
      const uint32_t wrows_all = __reduce_or_sync(SPHB_FULL, mine);
      const uint32_t wrows_f = __reduce_or_sync(SPHB_FULL, isf ? mine : 0u);
#pragma unroll
      for (int g = 0; g < MAXSEG / 32; ++g) {
        const int k = g * 32 + lane;
        wpos0[g] = wpos1[g] = 0;
        if (wactive && k < nseg) {
          const Seg sg = sSeg[k];
          if (sg.g1 > sg.g0) {
            const int lo = (V8_SYM && k < nlist) ? max(wcxlo, 0) : wxlo;
            const int w0 = a.beg[sg.rowoff + lo], w1 = a.end[sg.rowoff + wxhi];
            wpos0[g] = sg.pos + (w0 - sg.g0);
            wpos1[g] = sg.pos + (w1 - sg.g0);
            // boundary-list rows serve the fluid targets only
            const uint32_t wr = sg.rowoff < a.ncells ? wrows_f : wrows_all;
            const int dy = (sg.dyz & 255) - 16, dz = (sg.dyz >> 8) - 16;
            bool need = false;
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4)
              need |= ((wr >> r4) & 1u) && abs(dy - (r4 & 1)) <= reach && abs(dz - (r4 >> 1)) <= reach;
            if (w1 > w0 && need) wlive |= 1u << g;
          }
        }
      }
    }

    // fused wall force (extension; the FP32 gather builds): f64 sums over the batches
    constexpr bool wall = WALL && !V8_SYM;  // (its own instantiation: none of it otherwise)
    double wfx = 0.0, wfy = 0.0, wfz = 0.0;
    bool whit = false;

    for (int q0 = 0; q0 < total; q0 += SCAP) {
      const int q1 = min(q0 + SCAP, total);
      // ---- stage rows [q0, q1): one TMA bulk copy per (stencil row, array) -- the sorted
      // posp rows are (x, y, z, prrho), velr rows (vx, vy, vz, rho) -- then the 8-B screen
      // records from shared memory
      if (warp == 0 && q0 > 0) stage_batch(a.posp, a.velr, sSeg, nseg, q0, q1, smA, 16u * V8_ROWS, mbar, lane);
      {  // wait for the bytes (phase parity flips per batch)
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done) : "r"(mbar), "r"(mphase) : "memory");
        mphase ^= 1u;
      }
      {
        uint2* rec = reinterpret_cast<uint2*>(reinterpret_cast<char*>(g_sm4) + V8_REC_OFF);
        for (int r = tid; r < q1 - q0; r += NW * 32) {
          const float4 pp = lds4(smA + 16u * r);
          const __half hx = __float2half_rn((pp.x - h16_xc) * h16_s);
          const __half hy = __float2half_rn((pp.y - h16_yc) * h16_s);
          const __half hz = __float2half_rn((pp.z - h16_zc) * h16_s);
          const float fx = __half2float(hx), fy = __half2float(hy), fz = __half2float(hz);
          rec[r] = make_uint2(h2u(__halves2half2(hx, hy)),
                              h2u(__halves2half2(hz, __float2half_rn(fmaf(fz, fz, fmaf(fy, fy, fx * fx))))));
        }
      }
      __syncthreads();
      if (wactive) {
        // the warp's windows (precomputed per block, wpos0/wpos1) of the live rows, in row order
#pragma unroll
        for (int g = 0; g < MAXSEG / 32; ++g) {
          uint32_t mlive = __ballot_sync(SPHB_FULL, (wlive >> g) & 1u);
          while (mlive) {
          const int l = __ffs(mlive) - 1;
          mlive &= mlive - 1u;
          const int k = g * 32 + l;
          const int lo_ = max(__shfl_sync(SPHB_FULL, wpos0[g], l), q0) - q0;
          const int hi_ = min(__shfl_sync(SPHB_FULL, wpos1[g], l), q1) - q0;
          if (hi_ <= lo_) continue;
          const Seg sg = sSeg[k];
          const bool boundary_list = sg.rowoff < a.ncells;
          const bool inr = in_rows(sg.dyz);
          const uint32_t lanemask = (valid && inr && (isf || !boundary_list)) ? 0xffffffffu : 0u;
          const bool selfrow = k == selfseg_l;
          // own staged position in the self row (fluid targets), else out of range
          const int selfpos = (selfrow && isf) ? sg.pos + (i - sg.g0) - q0 : INT_MIN / 2;
          // symmetric own row: staged position of the lane's lower bound (batch-relative)
          int lbpos = INT_MIN / 2;
          if (V8_SYM && k < nlist) {
            const int lb = boundary_list ? lbB : lbF;
            lbpos = lb == INT_MAX ? INT_MAX / 2 : sg.pos + (lb - sg.g0) - q0;
          }
          for (int k0 = lo_; k0 < hi_; k0 += 32) {
            uint32_t hit;
            if (use16) {
              // 32 targets x 32 candidates on the tensor cores: 2 M-tiles x 4 N-tiles
              const uint32_t wb = bl_base + bl_kmul * (uint32_t)k0 + bl_off;
              uint32_t fb[4];
#pragma unroll
              for (int n = 0; n < 4; ++n) fb[n] = lds32(wb + 16u * n);
              float d[2][4][4];
#pragma unroll
              for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 4; ++n) mma_16816(d[m][n], fa[m][0], fa[m][1], fb[n], fc[m]);
              // sign (D < 0: r^2 < thr) of target slot s = 2m + h, candidate 8t + 2n + e ->
              // byte s, bit 2n + e
              uint32_t w = 0;
#pragma unroll
              for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const uint32_t pa = h2u(__floats2half2_rn(d[0][n][e], d[0][n][2 + e]));
                  const uint32_t pb = h2u(__floats2half2_rn(d[1][n][e], d[1][n][2 + e]));
                  w |= prmt_sign(pa, pb) & (0x01010101u << (2 * n + e));
                }
              // quad byte transpose: lane (g, t) <- target g + 8t, byte j from lane (g, j)
              w = prmt(w, __shfl_xor_sync(SPHB_FULL, w, 1), tsel1);
              w = prmt(w, __shfl_xor_sync(SPHB_FULL, w, 2), tsel2);
              hit = __shfl_sync(SPHB_FULL, w, troute);  // bit b <-> candidate k0 + b
            } else {
              const uint32_t sk = smA + 16u * k0;
              hit = 0;
#pragma unroll
              for (int tt = 0; tt < 32; ++tt) {
                const float4 A = lds4(sk + 16u * tt);
                const float dx = o.x - A.x, dy = o.y - A.y, dz = o.z - A.z;
                if (fmaf(dz, dz, fmaf(dy, dy, dx * dx)) < k32.sup2_hi) hit |= 1u << tt;
              }
            }
            uint32_t bits = hit & lanemask;  // k0 >= lo_: only the row's last word is partial
            if (hi_ - k0 < 32) bits &= (1u << (hi_ - k0)) - 1u;
            if (selfrow) {
              const int d = selfpos - k0;
              if ((unsigned)d < 32u) bits &= ~(1u << d);
            }
            if (V8_SYM) {  // own row: candidates at or above the lane's lower bound only
              const int d = lbpos - k0;
              bits = d >= 32 ? 0u : (d > 0 ? bits & ~((1u << d) - 1u) : bits);
            }
            if (__any_sync(SPHB_FULL, bits != 0u && cnt == (uint32_t)RINGC)) drain(false);
            if (bits) {
              const uint32_t qb = V8_SYM ? __funnelshift_l(bits, bits, rot) : bits;
              sts64u(tp, qb, smA + 16u * (uint32_t)k0 + (((!EQM || V8_SYM) && boundary_list) ? 1u : 0u));
              tp = tp + 256u == rend ? ring : tp + 256u;
              ++cnt;
              pend += __popc(bits);
            }
          }
          }
        }
        drain(true);
        if constexpr (wall) if (valid && isf)
          whit |= wall_batch(a, sSeg, nseg, q0, q1, smA, o.x, o.y, o.z, xlo, xhi, rsy, rsz, wfx, wfy, wfz);
      }
      __syncthreads();
      if (V8_SYM) {
        // the batch's reactions -> global memory (one REDG.F32x4 + RED.MAX per touched row, rows
        // contiguous per stencil row: coalesced), scaled as the targets' own sums below
        const float mfac = EQM ? (float)a.p.mass_fluid : 1.0f, hq = (float)a.p.h;
        for (int k = 0; k < nseg; ++k) {
          const Seg sg = sSeg[k];
          const int lo_p = max(sg.pos, q0), hi_p = min(sg.pos + (sg.g1 - sg.g0), q1);
          for (int p = lo_p + tid; p < hi_p; p += NW * 32) {
            const uint32_t r = (uint32_t)(p - q0);
            const float4 v = lds4(smA + V8_ACC_OFF + 16u * r);
            const uint32_t m = lds32(smA + V8_VD_OFF + 4u * r);
            if (m != 0u || v.w != 0.0f || v.x != 0.0f || v.y != 0.0f || v.z != 0.0f) {
              const int64_t j = (int64_t)sg.g0 + (p - sg.pos);
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a.acc4 + j),
                           "f"(v.x * mfac), "f"(v.y * mfac), "f"(v.z * mfac), "f"(-v.w * mfac)
                           : "memory");
              asm volatile("red.global.max.u32 [%0], %1;" ::"l"(a.visc32 + j),
                           "r"(__float_as_uint(__uint_as_float(m) * hq)) : "memory");
              asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(smA + V8_ACC_OFF + 16u * r),
                           "r"(0u) : "memory");
              sts32(smA + V8_VD_OFF + 4u * r, 0u);
            }
          }
        }
        __syncthreads();
      }
    }

    if (valid) {
#pragma unroll
      for (int k = 1; k < V8_NG; ++k) {
        s[0].axy = add2(s[0].axy, s[k].axy);
        s[0].az = add2(s[0].az, s[k].az);
        s[0].dr = add2(s[0].dr, s[k].dr);
        s[0].hits = add2(s[0].hits, s[k].hits);
        s[0].vd = fmaxf(s[0].vd, s[k].vd);
      }
      const int hits = (int)(lo(s[0].hits) + hi(s[0].hits));
      c_cand += cand;
      c_hits += (unsigned long long)hits;
      if (V8_SYM) {
#pragma unroll
        for (int k = 1; k < V8_NG; ++k) s[0].hitsf = add2(s[0].hitsf, s[k].hitsf);
        c_ff += isf ? (int)(lo(s[0].hitsf) + hi(s[0].hitsf)) : 0;
      } else {
        c_ff += isf ? hits : -hits;  // ff = F targets' hits - B targets' hits (F-B == B-F)
      }
      const float mfac = EQM ? (float)a.p.mass_fluid : 1.0f;
      const double ax = (double)(lo(s[0].axy) * mfac), ay = (double)(hi(s[0].axy) * mfac);
      const double az = (double)((lo(s[0].az) + hi(s[0].az)) * mfac);
      const double dr = (double)(-(lo(s[0].dr) + hi(s[0].dr)) * mfac);
      const float vd32 = s[0].vd * (float)a.p.h;
      const double vd = (double)vd32;
      if (V8_SYM) {  // other blocks add this particle's reactions too: atomics, dt after PI
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a.acc4 + i),
                     "f"(isf ? (float)ax : 0.f), "f"(isf ? (float)ay : 0.f), "f"(isf ? (float)az : 0.f),
                     "f"((float)dr) : "memory");
        asm volatile("red.global.max.u32 [%0], %1;" ::"l"(a.visc32 + i), "r"(__float_as_uint(vd32))
                     : "memory");
        continue;
      }
      // FP32 layout: 20 B per particle (the values are f32 already; K7 widens them exactly)
      a.acc4[i] = isf ? make_float4((float)ax, (float)ay, (float)az, (float)dr)
                      : make_float4(0.f, 0.f, 0.f, (float)dr);
      a.visc32[i] = vd32;
      if (!(isfinite(ax) && isfinite(ay) && isfinite(az) && isfinite(dr)))
        raise_div(a.ctrl, step, SPHB_DIV_NONFINITE_FORCES, 0);
      if (isf) {
        const double fx = xadd(ax, a.p.g[0]), fy = xadd(ay, a.p.g[1]), fz = xadd(az, a.p.g[2]);
        double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
        fmag = fmag > 1e-30 ? fmag : 1e-30;
        dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(a.p.h, fmag)));
      }
      if (whit)
        wall_finish(a, i, step, (float)ax, (float)ay, (float)az, (float)dr, wfx, wfy, wfz, dtf_min);
      dtcv_min = fmin(dtcv_min, xdiv(a.p.h, xadd((double)ocs, vd)));
    }
  }

  dtf_min = warp_min(dtf_min);
  dtcv_min = warp_min(dtcv_min);
  c_cand = warp_sum_u64(c_cand);
  c_hits = warp_sum_u64(c_hits);
  unsigned long long ffu = warp_sum_u64((unsigned long long)c_ff);
  if (V8_SYM) {  // unordered hits -> the gather traversal's ordered counts (each pair twice)
    c_hits *= 2;
    ffu *= 2;
  }
  if (lane == 0) {
    if (dtf_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_f, dtf_min);
    if (dtcv_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_cv, dtcv_min);
    if (c_cand) atomicAdd((unsigned long long*)&a.ctrl->counters[0], c_cand);
    if (c_hits) {
      atomicAdd((unsigned long long*)&a.ctrl->counters[1], c_hits);
      atomicAdd((unsigned long long*)&a.ctrl->counters[2], c_hits);
    }
    if (ffu) atomicAdd((unsigned long long*)&a.ctrl->counters[3], ffu);
  }
}

#include "interact_pair.cuh"

template <typename R>
constexpr size_t smem_bytes() {
  return sizeof(float4) * Cfg<R>::NARR * Cfg<R>::SCAP + (Cfg<R>::H16 ? 6 * Cfg<R>::SCAP : 0) +
         sizeof(uint32_t) * NW * RING * 32 + sizeof(uint16_t) * NW * RING * 32;
}

template <typename R, bool G7, bool EQM>
int launch_kernel(const KArgs& a, int nsm, cudaStream_t s) {
  static int grid = 0;
  const size_t bytes = smem_bytes<R>();
  if (grid == 0) {
    cudaError_t e = cudaFuncSetAttribute(k_interact<R, G7, EQM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess)
      return sphb_set_error(SPHB_E_CUDA, "smem attribute: %s", cudaGetErrorString(e));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_interact<R, G7, EQM>, NW * 32, bytes);
    grid = nsm * (per_sm > 0 ? per_sm : 1);
  }
  k_interact<R, G7, EQM><<<grid, NW * 32, bytes, s>>>(a);
  return sphb_check_launch("k_interact");
}

template <bool G7, bool EQM, bool WEND, bool WALL>
int launch_v8(const KArgs& a, const K32& k, int nsm, cudaStream_t s) {
  static int grid = 0;
  const size_t bytes = V8_SMEM;
  if (grid == 0) {
    cudaError_t e = cudaFuncSetAttribute(k_interact_v8<G7, EQM, WEND, WALL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess)
      return sphb_set_error(SPHB_E_CUDA, "smem attribute: %s", cudaGetErrorString(e));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_interact_v8<G7, EQM, WEND, WALL>, NW * 32, bytes);
    grid = nsm * (per_sm > 0 ? per_sm : 1);
  }
  k_interact_v8<G7, EQM, WEND, WALL><<<grid, NW * 32, bytes, s>>>(a, k);
  return sphb_check_launch("k_interact_v8");
}

#if SPHB_PAIR
template <bool G7, bool EQM, bool WEND, bool WALL>
int launch_v12(const KArgs& a, const K32& k, int nsm, cudaStream_t s) {
  static bool init = false;
  const size_t bytes = V8_SMEM;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(k_interact_v12<G7, EQM, WEND, WALL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess)
      return sphb_set_error(SPHB_E_CUDA, "smem attribute: %s", cudaGetErrorString(e));
    init = true;
  }
  k_interact_v12<G7, EQM, WEND, WALL><<<nsm, NW * 32, bytes, s>>>(a, k);
  return sphb_check_launch("k_interact_v12");
}
#endif

template <bool WEND>
int launch_v8_kernel(const KArgs& a, const K32& k, bool eqm, int nsm, cudaStream_t s) {
  // the fused wall force (extension) has its own instantiations, gamma = 7 only (the other
  // EOS exponents take the separate k_wall_force pass, launch_interact)
  const bool wall = a.p.wall_d > 0.0 && a.gamma7;
#if SPHB_PAIR
  if (wall)
    return eqm ? launch_v12<true, true, WEND, true>(a, k, nsm, s) : launch_v12<true, false, WEND, true>(a, k, nsm, s);
  if (a.gamma7)
    return eqm ? launch_v12<true, true, WEND, false>(a, k, nsm, s) : launch_v12<true, false, WEND, false>(a, k, nsm, s);
  return eqm ? launch_v12<false, true, WEND, false>(a, k, nsm, s) : launch_v12<false, false, WEND, false>(a, k, nsm, s);
#endif
  if (wall)
    return eqm ? launch_v8<true, true, WEND, true>(a, k, nsm, s) : launch_v8<true, false, WEND, true>(a, k, nsm, s);
  if (a.gamma7)
    return eqm ? launch_v8<true, true, WEND, false>(a, k, nsm, s) : launch_v8<true, false, WEND, false>(a, k, nsm, s);
  return eqm ? launch_v8<false, true, WEND, false>(a, k, nsm, s) : launch_v8<false, false, WEND, false>(a, k, nsm, s);
}

template <typename R>
int launch_one(const KArgs& a, int nsm, cudaStream_t s) {
  if constexpr (sizeof(R) == 8) {
    return launch_kernel<R, true, false>(a, nsm, s);
  } else if constexpr (SPHB_V8) {
    const sphb_params_t& p = a.p;
    K32 k;
    // sure-hit / sure-miss band of the FP32 r^2: |r2_32 / r2_64 - 1| <= 5.1 u (u = 2^-24: the
    // rounded difference, product, sum and FMA), so +-5e-7 (8.4 u, threshold rounding
    // included) decides every pair the f64 predicate would, except the ones inside it
    k.sup2_lo = (float)(p.sup2 * (1.0 - 5e-7));
    k.sup2_hi = (float)(p.sup2 * (1.0 + 5e-7));
    k.tiny = a.tiny;
    k.invh = a.invh;
    k.eta2 = a.eta2;
    const double ktw = p.kc * p.invwdp;
    k.ktw4 = (float)(ktw * ktw * ktw * ktw);
    k.tpos = (float)(0.01 * ktw * ktw * ktw * ktw);
    k.tneg = (float)(-0.2 * ktw * ktw * ktw * ktw);
    const double nalh = -p.alpha * p.h;  // -alpha h folded into cs
    k.cs_exp = a.cs_exp;
    k.kcs = a.gamma7 ? (float)(cbrt(p.c0) / p.rho0 * cbrt(nalh))
                     : (float)(p.c0 * pow(p.rho0, -(p.gamma - 1.0) * 0.5) * nalh);
    const bool eqm = p.mass_fluid == p.mass_boundary;
    const bool wend = p.kernel == SPHB_KERNEL_WENDLAND;
    // -gc / (gradient shape): cubic -3 kc/h (shape (u^2 - t^2/4)/r), Wendland 5 kc/h^2 (t^3)
    const double gk = wend ? 5.0 * p.kc * p.invh * p.invh : -3.0 * p.kc * p.invh;
    k.nkgc = (float)(gk * (eqm ? 1.0 : p.mass_fluid));
    k.nkgc_b = (float)(gk * (eqm ? 1.0 : p.mass_boundary));
    return wend ? launch_v8_kernel<true>(a, k, eqm, nsm, s) : launch_v8_kernel<false>(a, k, eqm, nsm, s);
  } else {
    const bool eqm = a.p.mass_fluid == a.p.mass_boundary;
    if (a.gamma7)
      return eqm ? launch_kernel<R, true, true>(a, nsm, s) : launch_kernel<R, true, false>(a, nsm, s);
    return eqm ? launch_kernel<R, false, true>(a, nsm, s) : launch_kernel<R, false, false>(a, nsm, s);
  }
}

// ------------------------------------------------------------------ boundary repulsion
// Extension (off by default): Monaghan's (1994) Lennard-Jones wall
// force per unit mass on fluid targets from boundary particles closer than r0 (<= 2h, so the
// interaction stencil holds them all):  a_i += D ((r0/r)^p1 - (r0/r)^p2) r_ij / r^2.  f64,
// added to the PI accelerations; the fluid dt term sqrt(h / |a + g|) of every target it
// touches joins the minimum (the SPH-only term is already in it: dt stays conservative).
template <bool F32>
__global__ void __launch_bounds__(256) k_wall_force(sphb_params_t p, sphb_grid_t g, int64_t n,
                                                    int64_t nb, int64_t ncells,
                                                    const float4* __restrict__ posp,
                                                    const int32_t* __restrict__ cell,
                                                    const int32_t* __restrict__ beg,
                                                    const int32_t* __restrict__ end,
                                                    void* __restrict__ accv, sphb_ctrl_t* ctrl) {
  double* acc = (double*)accv;
  float4* acc4 = (float4*)accv;
  if (!step_live(ctrl)) return;
  (void)ncells;
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2], R = g.reach;
  const double r02 = xmul(p.wall_r0, p.wall_r0);
  double dtf_min = INFINITY;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int c = cell[i];
    const int cx = c % nx, cy = (c / nx) % ny, cz = c / (nx * ny);
    if (cx < g.tx0 || cx >= g.tx1) continue;
    const float4 pi = posp[i];
    const int x0 = max(cx - R, 0), x1 = min(cx + R, nx - 1);
    double fx = 0.0, fy = 0.0, fz = 0.0;
    bool hit = false;
    for (int z = max(cz - R, 0); z <= min(cz + R, nz - 1); ++z) {
      for (int y = max(cy - R, 0); y <= min(cy + R, ny - 1); ++y) {
        const int64_t row = ((int64_t)z * ny + y) * nx;
        const int32_t j1 = end[row + x1];  // boundary list: the first ncells entries
        for (int32_t j = beg[row + x0]; j < j1; ++j) {
          const float4 pj = posp[j];
          const double dx = xsub((double)pi.x, (double)pj.x);
          const double dy = xsub((double)pi.y, (double)pj.y);
          const double dz = xsub((double)pi.z, (double)pj.z);
          const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
          if (!(r2 > 0.0 && r2 < r02)) continue;
          const double q = xdiv(p.wall_r0, __dsqrt_rn(r2));
          const double f = xdiv(xmul(p.wall_d, xsub(ipow(q, p.wall_p1), ipow(q, p.wall_p2))), r2);
          fx = xadd(fx, xmul(f, dx));
          fy = xadd(fy, xmul(f, dy));
          fz = xadd(fz, xmul(f, dz));
          hit = true;
        }
      }
    }
    if (!hit) continue;
    double ax, ay, az;
    if (F32) {
      float4 v = acc4[i];
      v.x = (float)xadd((double)v.x, fx);
      v.y = (float)xadd((double)v.y, fy);
      v.z = (float)xadd((double)v.z, fz);
      acc4[i] = v;
      ax = v.x;
      ay = v.y;
      az = v.z;
    } else {
      ax = xadd(acc[3 * i + 0], fx);
      ay = xadd(acc[3 * i + 1], fy);
      az = xadd(acc[3 * i + 2], fz);
      acc[3 * i + 0] = ax;
      acc[3 * i + 1] = ay;
      acc[3 * i + 2] = az;
    }
    const double gx = xadd(ax, p.g[0]), gy = xadd(ay, p.g[1]), gz = xadd(az, p.g[2]);
    double fmag = __dsqrt_rn(xadd(xadd(xmul(gx, gx), xmul(gy, gy)), xmul(gz, gz)));
    fmag = fmag > 1e-30 ? fmag : 1e-30;
    dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(p.h, fmag)));
    if (!(isfinite(ax) && isfinite(ay) && isfinite(az)))
      raise_div(ctrl, ctrl->step, SPHB_DIV_NONFINITE_FORCES, 0);
  }
  dtf_min = warp_min(dtf_min);
  if ((threadIdx.x & 31) == 0 && dtf_min < INFINITY) atomic_min_pos(&ctrl->dtmin_f, dtf_min);
}

// Symmetric build: the compute_dt reductions (sim.py:215-232) once every reaction has landed
// (the gather build does this in its epilogue, K6), on the FP32 force layout: min over fluid of
// sqrt(h / max(|a + g|, 1e-30)), min over all of h / (csound + visc_dt); non-finite forces
// flagged as the gather epilogue does (sim.py:328-329).
__global__ void __launch_bounds__(256) k_dt_f32(sphb_params_t p, int64_t n, int64_t nb,
                                                const float4* __restrict__ acc4,
                                                const float* __restrict__ visc32,
                                                const float4* __restrict__ aux, sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  double dtf = INFINITY, dtcv = INFINITY;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float4 a = acc4[i];
    const double vd = (double)visc32[i], cs = (double)aux[i].y;
    if (!(isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w)))
      raise_div(ctrl, ctrl->step, SPHB_DIV_NONFINITE_FORCES, 0);
    if (i >= nb) {
      const double fx = xadd((double)a.x, p.g[0]), fy = xadd((double)a.y, p.g[1]),
                   fz = xadd((double)a.z, p.g[2]);
      double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
      fmag = fmag > 1e-30 ? fmag : 1e-30;
      dtf = fmin(dtf, __dsqrt_rn(xdiv(p.h, fmag)));
    }
    dtcv = fmin(dtcv, xdiv(p.h, xadd(cs, vd)));
  }
  dtf = warp_min(dtf);
  dtcv = warp_min(dtcv);
  if ((threadIdx.x & 31) == 0) {
    if (dtf < INFINITY) atomic_min_pos(&ctrl->dtmin_f, dtf);
    if (dtcv < INFINITY) atomic_min_pos(&ctrl->dtmin_cv, dtcv);
  }
}

}  // namespace

#ifndef SPHB_PI_NS
#define SPHB_PI_NS pi128  // this build's blocking (see sphb_internal.h: pi128 / pi256 / pi384)
#endif
#ifdef SPHB_PI_LARGE
static_assert(BT == PI_LARGE_BLOCK, "the large build's block size is sphb_internal.h's");
#endif
namespace SPHB_PI_NS {

int64_t interact_launch_count(int64_t n) {
  (void)n;
  // k_blocks (count, scan, write), the interaction kernel (the symmetric build adds k_dt_f32,
  // the gather builds at reach >= 2 k_cand_cells: counted by the callers, device.py)
  return 4;
}

static int launch_wall(const sphb_params_t& p, const sphb_grid_t& g, int64_t n, int64_t nb,
                       int64_t ncells, const float4* posp, const int32_t* cell_sorted,
                       const int32_t* beg, const int32_t* end, void* acc, sphb_ctrl_t* ctrl,
                       cudaStream_t s) {
  const unsigned wb = (unsigned)std::min<int64_t>((n - nb + 255) / 256, 148 * 16);
  if (p.precision == SPHB_FP64)
    k_wall_force<false><<<wb, 256, 0, s>>>(p, g, n, nb, ncells, posp, cell_sorted, beg, end, acc, ctrl);
  else
    k_wall_force<true><<<wb, 256, 0, s>>>(p, g, n, nb, ncells, posp, cell_sorted, beg, end, acc, ctrl);
  return sphb_check_launch("k_wall_force");
}

// The interaction's block list: k_blocks (count -- with the FP32 gather builds' candidate
// counter --, scan, write), on stream s (sphb_step / sphb_interact_plan run it on the workspace's
// side stream, concurrently with K3).
int plan_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                  const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s,
                  unsigned long long* cand_acc) {
  if (g.reach < 1 || g.reach > 3) return sphb_set_error(SPHB_E_INVALID, "reach must be 1..3");
  const int64_t ncells = ncells_of(g);
  const int64_t nrows = (int64_t)g.dims[1] * g.dims[2];
  // one warp per cell row (rows ~10^4): every SM busy, the row's ends staged in shared memory
  int gb = (int)(nrows < 148 * 32 ? nrows : 148 * 32);
  if (gb < 1) gb = 1;
  const size_t sm_blocks = sizeof(int32_t) * 2 * (size_t)(g.tx1 - g.tx0);
  if (sm_blocks > 48 * 1024) return sphb_set_error(SPHB_E_INVALID, "more than 6144 cell columns per slab");
  // bricks for h/2 cells (reach 2) in the FP32 gather kernel's cell order
  // (the 512-target build cuts bricks at every reach: 2 x 2 rows x 2 lattice cells at n = 1)
  // hybrid at n = 1 (the row-block gather builds): 2 x 2-row quads whose cells hold fewer than
  // HYBRID_T targets on average become bricks, the others row blocks (k_blocks)
  const bool brickable = p.order == 0 && p.precision == SPHB_FP32 && !V8_SYM;
  static const char* hyb_env = getenv("SPHB_HYBRID_T");  // A/B experiments only (0 = rows)
  // (measured, profiles/r02bu_hybrid_blocking_ab.txt: 384-target blocks collapsed 16.01 ->
  // 15.79 ms at T = 32, at rest neutral; the 256-target build loses at rest, so rows only)
  // Small systems (fewer than ~8 blocks per SM) keep row blocks: fuller bricks mean fewer
  // blocks than SMs there (C1: gather 384 PI 0.103 -> 0.117 ms with bricks)
  const int hyb_t = hyb_env ? atoi(hyb_env)
                            : ((BT == PI_LARGE_BLOCK && ws->n_max >= (int64_t)148 * 8 * BT) ? HYBRID_T : 0);
  const int brick = !brickable ? 0
                    : (g.reach == 2 || BT == 512 || SPHB_PAIR) ? 1
                    : (hyb_t > 1 ? hyb_t : 0);
  const int64_t nunits = brick ? (int64_t)((g.dims[1] + 1) / 2) * ((g.dims[2] + 1) / 2) : nrows;
  // block x extent: columns [cxa - r, cxb + r] must stay within the FP16 screen's +-4 (2h)
  // around the block centre (use16 in the kernels), span <= 16 / (cell_size / h) columns
  int maxc = INT_MAX;
  if (p.precision == SPHB_FP32) {
    const int span = (int)floor(16.0 / (g.cell_size * p.invh) + 1e-9);
    maxc = span - 2 * g.reach > 1 ? span - 2 * g.reach : 1;
  }
  static const char* maxc_env = getenv("SPHB_BLOCK_MAXC");  // A/B experiments only
  if (maxc_env && atoi(maxc_env) > 0) maxc = atoi(maxc_env);
  // the FP32 gather builds' candidate counter rides on the count pass (reach 1), or takes its
  // own kernel (reach >= 2)
  const bool cand = p.precision == SPHB_FP32 && !V8_SYM;
  const bool count_cand = cand && g.reach == 1;
  k_blocks<true><<<gb, 32, sm_blocks, s>>>(g, ncells, beg, end, ws->row_off, ws->blocks, ctrl, brick,
                                           maxc, count_cand ? cand_acc : nullptr);
  if (int rc = sphb_check_launch("k_blocks count")) return rc;
  k_blocks_scan<<<1, KB_SCAN, 0, s>>>(ws->row_off, nunits, ctrl);
  if (int rc = sphb_check_launch("k_blocks_scan")) return rc;
  k_blocks<false><<<gb, 32, sm_blocks, s>>>(g, ncells, beg, end, ws->row_off, ws->blocks, ctrl, brick,
                                            maxc, nullptr);
  if (int rc = sphb_check_launch("k_blocks")) return rc;
  if (cand && !count_cand) {
    const int64_t ncand = (int64_t)(g.tx1 - g.tx0) * g.dims[1] * g.dims[2];
    const unsigned kc = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ncand + KC_THREADS - 1) / KC_THREADS, 148 * 8));
    k_cand_cells<<<kc, KC_THREADS, 0, s>>>(g, ncells, beg, end, ctrl, cand_acc);
    if (int rc = sphb_check_launch("k_cand_cells")) return rc;
  }
  return SPHB_OK;
}

int launch_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g, int64_t n,
                    int64_t nb, const float4* posp, const float4* velr, const float4* aux,
                    const int32_t* cell_sorted, const int32_t* beg, const int32_t* end,
                    void* acc, void* drho, void* visc, sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (g.reach < 1 || g.reach > 3) return sphb_set_error(SPHB_E_INVALID, "reach must be 1..3");
  // the block list: built on the side stream during K3 when this call's tables, window and
  // build match the pending plan, else here
  // (a pending plan that does not match is still waited for: it writes the same buffers)
  const sphb_workspace::Plan& pl = ws->plan;
  const bool pending = pl.valid;
  const bool match = pending && pl.beg == beg && pl.end == end && pl.dims[0] == g.dims[0] &&
                     pl.dims[1] == g.dims[1] && pl.dims[2] == g.dims[2] && pl.tx0 == g.tx0 &&
                     pl.tx1 == g.tx1 && pl.reach == g.reach && pl.precision == p.precision &&
                     pl.order == p.order && pl.pi_block == ws->pi_block &&
                     pl.pi_kernel == ws->pi_kernel;
  ws->plan.valid = false;
  if (pending)
    if (cudaError_t e = cudaStreamWaitEvent(s, ws->ev_plan, 0))
      return sphb_set_error(SPHB_E_CUDA, "plan wait: %s", cudaGetErrorString(e));
  if (match) {  // the side-stream plan counted candidates into the workspace: take them
    k_cand_take<<<1, 1, 0, s>>>(ws->cand_acc, ctrl);
    if (int rc = sphb_check_launch("k_cand_take")) return rc;
  } else {
    if (pending)  // the discarded plan's candidate count
      if (cudaError_t e = cudaMemsetAsync(ws->cand_acc, 0, sizeof(unsigned long long), s))
        return sphb_set_error(SPHB_E_CUDA, "plan reset: %s", cudaGetErrorString(e));
    // in line: straight into the step counters
    if (int rc = plan_interact(ws, p, g, beg, end, ctrl, s,
                               (unsigned long long*)&ctrl->counters[0]))
      return rc;
  }
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  KArgs a;
  a.p = p;
  a.g = g;
  a.n = n;
  a.nb = nb;
  a.ncells = ncells_of(g);
  a.posp = posp;
  a.velr = velr;
  a.aux = aux;
  a.cell = cell_sorted;
  a.beg = beg;
  a.end = end;
  a.acc = (double*)acc;
  a.drho = (double*)drho;
  a.visc = (double*)visc;
  a.acc4 = (float4*)acc;
  a.visc32 = (float*)visc;
  a.ctrl = ctrl;
  a.sup2_lo = (float)(p.sup2 * (1.0 - 1e-5));
  a.sup2_hi = (float)(p.sup2 * (1.0 + 1e-5));
  a.tiny = 1e-30f;
  a.h = (float)p.h;
  a.invh = (float)p.invh;
  a.k_gc = (float)(p.kc * p.invh);
  a.k_tw = (float)(p.kc * p.invwdp);
  a.eta2 = (float)p.eta2;
  a.alpha = (float)p.alpha;
  a.massf = (float)p.mass_fluid;
  a.massb = (float)p.mass_boundary;
  a.gamma7 = p.gamma == 7.0;
  a.inv_rho0 = 1.0 / p.rho0;
  a.cs_exp = (float)((p.gamma - 1.0) * 0.5);
  a.k_cs = a.gamma7 ? (float)(cbrt(p.c0) / p.rho0)
                    : (float)(p.c0 * pow(p.rho0, -(p.gamma - 1.0) * 0.5));
  // one launch for both item classes: fluid targets (F-F + F-B) and boundary targets (B-F,
  // drho + visc only) of the same cells share the staged candidates
  a.blocks = ws->blocks;
  const bool sym = V8_SYM && p.precision == SPHB_FP32;
  if (sym) {  // every block adds into these (targets' own sums and their partners' reactions)
    cudaMemsetAsync(acc, 0, sizeof(float4) * (size_t)n, s);
    cudaMemsetAsync(visc, 0, sizeof(float) * (size_t)n, s);
  }
  int rc = p.precision == SPHB_FP64 ? launch_one<double>(a, nsm, s) : launch_one<float>(a, nsm, s);
  // the wall force is fused into the FP32 gather kernels' epilogue (gamma = 7); the FP64 and
  // symmetric kernels take the separate pass
  if (!rc && p.wall_d > 0.0 && n > nb && (p.precision == SPHB_FP64 || sym || p.gamma != 7.0))
    rc = launch_wall(p, g, n, nb, a.ncells, posp, cell_sorted, beg, end, acc, ctrl, s);
  if (rc || !sym) return rc;
  k_dt_f32<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
      p, n, nb, a.acc4, a.visc32, aux, ctrl);
  return sphb_check_launch("k_dt_f32");
}

}  // namespace SPHB_PI_NS
