// interact.cu -- particle interaction (PI) of the SPH step on sm_100a.
//
// Replaces GatherEngine.compute (engines/gather.py:42-110): the fused fluid pass
// (gather_fluid_cells / gather_fluid_ranges, engines/kernels.py:326-497) and the
// boundary pass (gather_boundary_cells / _ranges, kernels.py:500-596), with the
// compute_dt reductions (sim.py:215-232) fused into the epilogue (K6).
//
// Work decomposition (FP32 CUDA cores; the pair math is a data-dependent gather-reduce,
// not a dense contraction, so no tensor cores):
//   * one warp owns 32 consecutive cell-sorted target particles (one per lane);
//   * lanes are grouped by their cell's (y, z) row; for each of the (2r+1)^2 stencil rows a
//     group walks the UNION of its lanes' x-ranges, which is one contiguous particle range
//     because cells are x-fastest (grid.py:1-8);
//   * candidates are staged 32 at a time into shared memory with one coalesced float4 load
//     and broadcast to every lane (LDS.128 broadcast);
//   * the distance test runs in FP32 with a relative guard band of 1e-5 around the cutoff;
//     anything inside the band (or with r2 ~ 0) is re-decided with the reference's exact f64
//     expression, so hit sets -- hence true_pairs / force_evals / ff counters -- are
//     bit-exact (SURVEY.md §8(a') "Neighbour predicate");
//   * hits go to a per-lane FIFO in shared memory and are evaluated in lock-step drains
//     (the device analogue of the reference's pack-of-4 lane batching, kernels.py:97-118):
//     a warp only evaluates when a lane's FIFO is about to overflow, and then drains at
//     least the warp-minimum backlog, so divergence on the ~15-25% hit rate costs little;
//   * FIFO order == candidate order == the reference's accumulation order, so the f64
//     instantiation reproduces the reference's forces bit for bit.
#include <climits>

#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

constexpr int IW = 4;   // warps per block
constexpr int QD = 64;  // per-lane hit FIFO depth (power of two)
constexpr int QM = QD - 1;

struct KArgs {
  sphb_params_t p;
  sphb_grid_t g;
  int64_t n, nb, item_lo, item_hi, ncells;
  const float4* __restrict__ posp;
  const float4* __restrict__ velr;
  const float4* __restrict__ aux;
  const int32_t* __restrict__ cell;
  const int32_t* __restrict__ beg;
  const int32_t* __restrict__ end;
  double* __restrict__ acc;
  double* __restrict__ drho;
  double* __restrict__ visc;
  sphb_ctrl_t* ctrl;
  // FP32 constants
  float sup2_lo, sup2_hi, tiny, h, invh, k_gc, k_tw, eta2, alpha, massf, massb;
};

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

// ------------------------------------------------------------------ per-precision traits
template <typename R>
struct Own {
  R x, y, z, vx, vy, vz, rho, prrho, cs, ten;
};

template <typename R>
struct Accum {
  R ax, ay, az, dr, vd;
};

// FP32 pair evaluation (physics.py:183-220 restated for FP32 CUDA cores).
// Folded constants: k_gc = kc/h, k_tw = kc/W(dp); the 0.5 factors of the viscous term cancel.
__device__ __forceinline__ void pair_eval(const KArgs& a, const Own<float>& o, float xj, float yj,
                                          float zj, const float4& vj, const float4& xa, float mj,
                                          Accum<float>& s) {
  const float dx = o.x - xj, dy = o.y - yj, dz = o.z - zj;
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float rinv = rsqrtf(r2);
  const float r = r2 * rinv;
  const float q = r * a.invh;
  float w, dw;
  if (q < 1.0f) {
    const float q2 = q * q;
    w = fmaf(0.75f * q, q2, fmaf(-1.5f, q2, 1.0f));
    dw = fmaf(2.25f, q, -3.0f) * q;
  } else {
    const float t = 2.0f - q;
    const float t2 = t * t;
    w = 0.25f * t2 * t;
    dw = -0.75f * t2;
  }
  const float gc = dw * a.k_gc * rinv;
  const float dvx = o.vx - vj.x, dvy = o.vy - vj.y, dvz = o.vz - vj.z;
  const float dot = fmaf(dvz, dz, fmaf(dvy, dy, dvx * dx));
  const float mu = __fdividef(a.h * dot, r2 + a.eta2);
  const float visc = dot < 0.0f ? __fdividef(-a.alpha * (o.cs + xa.y) * mu, o.rho + vj.w) : 0.0f;
  const float tw = w * a.k_tw;
  const float tw2 = tw * tw;
  const float pterm = fmaf((o.ten + xa.z) * tw2, tw2, o.prrho + xa.x + visc);
  const float fm = mj * pterm * gc;
  s.ax = fmaf(-fm, dx, s.ax);
  s.ay = fmaf(-fm, dy, s.ay);
  s.az = fmaf(-fm, dz, s.az);
  s.dr = fmaf(mj * gc, dot, s.dr);
  s.vd = fmaxf(s.vd, fabsf(mu));
}

// FP64 pair evaluation: the reference's exact operation order (physics.py:196-220,
// kernels.py:382-390), no contraction.  Bit-identical to numba.
__device__ __forceinline__ void pair_eval(const KArgs& a, const Own<double>& o, double xj,
                                          double yj, double zj, const float4& vj, const float4& xa,
                                          double mj, Accum<double>& s) {
  const sphb_params_t& p = a.p;
  const double dx = xsub(o.x, xj), dy = xsub(o.y, yj), dz = xsub(o.z, zj);
  const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
  const double r = __dsqrt_rn(r2);
  const double q = xmul(r, p.invh);
  const double kc = p.kc;
  double wab, dwdq;
  if (q < 1.0) {
    wab = xmul(kc, xadd(xsub(1.0, xmul(xmul(1.5, q), q)), xmul(xmul(xmul(0.75, q), q), q)));
    dwdq = xmul(xmul(kc, xsub(xmul(2.25, q), 3.0)), q);
  } else {
    const double t = xsub(2.0, q);
    wab = xmul(xmul(xmul(xmul(0.25, kc), t), t), t);
    dwdq = xmul(xmul(xmul(-0.75, kc), t), t);
  }
  const double gc = xdiv(xmul(dwdq, p.invh), r);
  const double dvx = xsub(o.vx, (double)vj.x), dvy = xsub(o.vy, (double)vj.y),
               dvz = xsub(o.vz, (double)vj.z);
  const double dot = xadd(xadd(xmul(dvx, dx), xmul(dvy, dy)), xmul(dvz, dz));
  const double mu = xdiv(xmul(p.h, dot), xadd(r2, p.eta2));
  double visc = 0.0;
  if (dot < 0.0) {
    const double rho_j = (double)vj.w, cs_j = (double)xa.y;
    visc = xdiv(xmul(xmul(-p.alpha, xmul(0.5, xadd(o.cs, cs_j))), mu),
                xmul(0.5, xadd(o.rho, rho_j)));
  }
  const double tw = xmul(wab, p.invwdp);
  const double tw2 = xmul(tw, tw);
  const double pterm = xadd(xadd(xadd(o.prrho, (double)xa.x), visc),
                            xmul(xmul(xadd(o.ten, (double)xa.z), tw2), tw2));
  const double pg = xmul(pterm, gc);
  s.ax = xsub(s.ax, xmul(mj, xmul(pg, dx)));
  s.ay = xsub(s.ay, xmul(mj, xmul(pg, dy)));
  s.az = xsub(s.az, xmul(mj, xmul(pg, dz)));
  s.dr = xadd(s.dr, xmul(mj, xmul(gc, dot)));
  const double ma = fabs(mu);
  if (ma > s.vd) s.vd = ma;
}

template <typename R>
struct Stage;
template <>
struct Stage<float> {
  float4 v;
};
template <>
struct Stage<double> {
  double x, y, z, pad;
};

__device__ __forceinline__ void stage_store(Stage<float>* s, const float4& p) { s->v = p; }
__device__ __forceinline__ void stage_store(Stage<double>* s, const float4& p) {
  s->x = (double)p.x;
  s->y = (double)p.y;
  s->z = (double)p.z;
}

// candidate test: FP32 fast path with exact f64 re-decision in the guard band
__device__ __forceinline__ bool cand_hit(const KArgs& a, const Own<float>& o, const Stage<float>& c) {
  const float dx = o.x - c.v.x, dy = o.y - c.v.y, dz = o.z - c.v.z;
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  if (r2 >= a.sup2_hi) return false;
  if (r2 < a.sup2_lo && r2 > a.tiny) return true;
  return exact_hit((double)o.x, (double)o.y, (double)o.z, (double)c.v.x, (double)c.v.y,
                   (double)c.v.z, a.p.sup2);
}
__device__ __forceinline__ bool cand_hit(const KArgs& a, const Own<double>& o,
                                         const Stage<double>& c) {
  return exact_hit(o.x, o.y, o.z, c.x, c.y, c.z, a.p.sup2);
}

template <typename R>
__device__ __forceinline__ R load_coord(const float4& p, int k) {
  return (R)(k == 0 ? p.x : (k == 1 ? p.y : p.z));
}

// ------------------------------------------------------------------ the kernel
template <typename R, bool FLUID_ITEMS>
__global__ void __launch_bounds__(IW * 32) k_interact(KArgs a) {
  if (!step_live(a.ctrl)) return;
  __shared__ Stage<R> s_stage[IW][32];
  __shared__ int32_t s_q[IW][QD][32];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nitems = a.item_hi - a.item_lo;
  const int64_t ntiles = (nitems + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * IW + warp;
  const int64_t nwarps = (int64_t)gridDim.x * IW;
  const int64_t step = a.ctrl->step;
  const int nx = a.g.dims[0], ny = a.g.dims[1], nz = a.g.dims[2];
  const int reach = a.g.reach;
  const int64_t nb = a.nb;

  unsigned long long c_cand = 0, c_hits = 0, c_ff = 0;
  double dtf_min = INFINITY, dtcv_min = INFINITY;

  for (int64_t tile = gwarp; tile < ntiles; tile += nwarps) {
    const int64_t i = a.item_lo + tile * 32 + lane;
    const bool valid = i < a.item_hi;
    Own<R> o;
    int cx = 0, rowkey = -1;
    if (valid) {
      const float4 pi = a.posp[i], vi = a.velr[i], xi = a.aux[i];
      o.x = (R)pi.x; o.y = (R)pi.y; o.z = (R)pi.z;
      o.vx = (R)vi.x; o.vy = (R)vi.y; o.vz = (R)vi.z; o.rho = (R)vi.w;
      o.prrho = (R)xi.x; o.cs = (R)xi.y; o.ten = (R)xi.z;
      const int c = a.cell[i];
      const int cyz = c / nx;
      cx = c - cyz * nx;
      rowkey = cyz;
    } else {
      o.x = o.y = o.z = o.vx = o.vy = o.vz = o.prrho = o.cs = o.ten = (R)0;
      o.rho = (R)1;
    }
    const int xlo = max(cx - reach, 0), xhi = min(cx + reach, nx - 1);
    Accum<R> s = {(R)0, (R)0, (R)0, (R)0, (R)0};
    uint32_t head = 0, tail = 0;
    unsigned long long cand = 0;

    // lock-step drain of up to k queued hits per lane
    auto drain = [&](uint32_t k) {
      for (uint32_t it = 0; it < k; ++it) {
        if (tail != head) {
          const int32_t j = s_q[warp][head & QM][lane];
          ++head;
          const float4 pj = __ldg(&a.posp[j]);
          const float4 vj = __ldg(&a.velr[j]);
          const float4 xa = __ldg(&a.aux[j]);
          const bool jb = j < nb;
          const R mj = jb ? (R)a.p.mass_boundary : (R)a.p.mass_fluid;
          pair_eval(a, o, (R)pj.x, (R)pj.y, (R)pj.z, vj, xa, mj, s);
          c_hits += 1;
          if (FLUID_ITEMS && !jb) c_ff += 1;
        }
      }
    };

    uint32_t todo = __ballot_sync(SPHB_FULL, valid);
    while (todo) {
      const int leader = __ffs(todo) - 1;
      const int key = __shfl_sync(SPHB_FULL, rowkey, leader);
      const uint32_t grp = __ballot_sync(SPHB_FULL, valid && rowkey == key);
      todo &= ~grp;
      const bool ing = (grp >> lane) & 1u;
      const int gxlo = __reduce_min_sync(SPHB_FULL, ing ? xlo : INT_MAX);
      const int gxhi = __reduce_max_sync(SPHB_FULL, ing ? xhi : INT_MIN);
      const int gcz = key / ny, gcy = key - gcz * ny;
      const int npass = (FLUID_ITEMS && a.p.order == 1) ? 2 : 1;
      for (int pass = 0; pass < npass; ++pass) {
        for (int dz = -reach; dz <= reach; ++dz) {
          const int zz = gcz + dz;
          if (zz < 0 || zz >= nz) continue;
          for (int dy = -reach; dy <= reach; ++dy) {
            const int yy = gcy + dy;
            if (yy < 0 || yy >= ny) continue;
            const int64_t base = (int64_t)nx * (yy + (int64_t)ny * zz);
#pragma unroll 1
            for (int li = 0; li < 2; ++li) {
              // li 0: fluid list (offset ncells in beg/end), li 1: boundary list
              const bool fluid_list = li == 0;
              if (!fluid_list && !FLUID_ITEMS) continue;
              if (npass == 2 && (pass == 0) != fluid_list) continue;
              const int64_t off = fluid_list ? a.ncells : 0;
              const int32_t u0 = a.beg[off + base + gxlo];
              const int32_t u1 = a.end[off + base + gxhi];
              if (u1 <= u0) continue;
              int32_t al = 0, bl = 0;
              if (ing) {
                al = a.beg[off + base + xlo];
                bl = a.end[off + base + xhi];
                cand += (unsigned long long)(bl - al);
              }
              const uint32_t span = (uint32_t)(bl - al);
              for (int32_t j0 = u0; j0 < u1; j0 += 32) {
                const int32_t jj = j0 + lane;
                if (jj < u1) stage_store(&s_stage[warp][lane], __ldg(&a.posp[jj]));
                __syncwarp();
                const int cnt = min(32, u1 - j0);
                for (int t = 0; t < cnt; ++t) {
                  const int32_t j = j0 + t;
                  const bool inr = (uint32_t)(j - al) < span;
                  if (inr && cand_hit(a, o, s_stage[warp][t])) {
                    s_q[warp][tail & QM][lane] = j;
                    ++tail;
                  }
                }
                __syncwarp();
                const uint32_t pend = tail - head;
                const uint32_t mx = __reduce_max_sync(SPHB_FULL, ing ? pend : 0u);
                if (mx > (uint32_t)(QD - 32)) {
                  const uint32_t mn = __reduce_min_sync(SPHB_FULL, ing ? pend : 0xffffffffu);
                  drain(max(mn, mx - (uint32_t)(QD - 32)));
                }
              }
            }
          }
        }
      }
    }
    drain(__reduce_max_sync(SPHB_FULL, tail - head));

    if (valid) {
      if (FLUID_ITEMS) cand -= 1;  // the reference skips j == i before counting (kernels.py:369-371)
      c_cand += cand;
      const double ax = (double)s.ax, ay = (double)s.ay, az = (double)s.az;
      const double dr = (double)s.dr, vd = (double)s.vd;
      if (FLUID_ITEMS) {
        a.acc[3 * i + 0] = ax;
        a.acc[3 * i + 1] = ay;
        a.acc[3 * i + 2] = az;
      } else {
        a.acc[3 * i + 0] = 0.0;
        a.acc[3 * i + 1] = 0.0;
        a.acc[3 * i + 2] = 0.0;
      }
      a.drho[i] = dr;
      a.visc[i] = vd;
      if (!(isfinite(ax) && isfinite(ay) && isfinite(az) && isfinite(dr)))
        raise_div(a.ctrl, step, SPHB_DIV_NONFINITE_FORCES, 0);
      // compute_dt terms (sim.py:222-229); min is order-free so this is exact
      if (FLUID_ITEMS) {
        const double fx = xadd(ax, a.p.g[0]), fy = xadd(ay, a.p.g[1]), fz = xadd(az, a.p.g[2]);
        double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
        fmag = fmag > 1e-30 ? fmag : 1e-30;
        dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(a.p.h, fmag)));
      }
      dtcv_min = fmin(dtcv_min, xdiv(a.p.h, xadd((double)o.cs, vd)));
    }
  }

  // epilogue: one reduction + a few atomics per warp (persistent grid)
  dtf_min = warp_min(dtf_min);
  dtcv_min = warp_min(dtcv_min);
  c_cand = warp_sum_u64(c_cand);
  c_hits = warp_sum_u64(c_hits);
  c_ff = warp_sum_u64(c_ff);
  if (lane == 0) {
    if (FLUID_ITEMS && dtf_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_f, dtf_min);
    if (dtcv_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_cv, dtcv_min);
    if (c_cand) atomicAdd((unsigned long long*)&a.ctrl->counters[0], c_cand);
    if (c_hits) {
      atomicAdd((unsigned long long*)&a.ctrl->counters[1], c_hits);
      atomicAdd((unsigned long long*)&a.ctrl->counters[2], c_hits);
    }
    if (c_ff) atomicAdd((unsigned long long*)&a.ctrl->counters[3], c_ff);
  }
}

template <typename R, bool F>
int launch_one(const KArgs& a, cudaStream_t s) {
  const int64_t ntiles = (a.item_hi - a.item_lo + 31) / 32;
  if (ntiles <= 0) return SPHB_OK;
  static int blocks_per_sm = 0, nsm = 0;
  if (blocks_per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_interact<R, F>, IW * 32, 0);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int64_t want = (ntiles + IW - 1) / IW;
  int64_t cap = (int64_t)nsm * blocks_per_sm;
  int grid = (int)(want < cap ? want : cap);
  k_interact<R, F><<<grid, IW * 32, 0, s>>>(a);
  return sphb_check_launch("k_interact");
}

}  // namespace

int64_t interact_launch_count(int64_t n) {
  (void)n;
  return 2;
}

int launch_interact(const sphb_params_t& p, const sphb_grid_t& g, int64_t n, int64_t nb,
                    const float4* posp, const float4* velr, const float4* aux,
                    const int32_t* cell_sorted, const int32_t* beg, const int32_t* end,
                    double* acc, double* drho, double* visc, sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (g.reach < 1 || g.reach > 4) return sphb_set_error(SPHB_E_INVALID, "reach must be 1..4");
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
  a.acc = acc;
  a.drho = drho;
  a.visc = visc;
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
  int rc;
  // fluid items [nb, n): F-F + F-B
  a.item_lo = nb;
  a.item_hi = n;
  rc = p.precision == SPHB_FP64 ? launch_one<double, true>(a, s) : launch_one<float, true>(a, s);
  if (rc) return rc;
  // boundary items [0, nb): B-F only, drho + visc
  a.item_lo = 0;
  a.item_hi = nb;
  rc = p.precision == SPHB_FP64 ? launch_one<double, false>(a, s) : launch_one<float, false>(a, s);
  return rc;
}
