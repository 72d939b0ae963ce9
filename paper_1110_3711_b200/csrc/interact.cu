// interact.cu -- particle interaction (PI) of the SPH step on sm_100a.
//
// Replaces GatherEngine.compute (engines/gather.py:42-110): the fused fluid pass
// (gather_fluid_cells / gather_fluid_ranges, engines/kernels.py:326-497) and the
// boundary pass (gather_boundary_cells / _ranges, kernels.py:500-596), with the
// compute_dt reductions (sim.py:215-232) fused into the epilogue (K6).
//
// Work decomposition (FP32 CUDA cores; the pair math is a data-dependent gather-reduce,
// not a dense contraction, so no tensor cores):
//   * one warp owns 32 consecutive cell-sorted target particles (one per lane); warps pull
//     32-target tiles dynamically (atomic tile counter) until the list is exhausted;
//   * lanes are grouped by their cell's (y, z) row; for each of the (2r+1)^2 stencil rows a
//     group walks the UNION of its lanes' x-ranges, which is one contiguous particle range
//     because cells are x-fastest (grid.py:1-8).  No per-candidate range test is needed:
//     a sure FP32 hit lies strictly inside 2h, hence inside the lane's own stencil;
//   * candidates are staged 32 at a time into shared memory with one coalesced float4 load
//     and broadcast to every lane (LDS.128 broadcast); the screen is branch-free
//     (r2 < sup2*(1+1e-5)) and produces one 32-bit "maybe" mask per lane per chunk;
//   * mask words are queued per lane in shared memory (a whole tile's worth), then drained
//     once in lock-step: every lane pops its next candidate (FIFO == candidate order ==
//     the reference's accumulation order) and evaluates it -- the device analogue of the
//     reference's pack-of-4 lane batching (kernels.py:97-118), so the ~15-25% hit rate
//     costs no divergence in the pair math;
//   * maybes that are not sure hits (inside the 1e-5 guard band around the cutoff, or
//     r2 ~ 0 -- e.g. the particle itself) are re-decided in the drain with the reference's
//     exact f64 predicate, so hit sets -- hence true_pairs / force_evals / ff counters --
//     are bit-exact (SURVEY.md §8(a') "Neighbour predicate");
//   * the FP64 instantiation uses the exact predicate in the screen and the reference's
//     exact operation order in the pair math: bit-identical forces.
#include <climits>

#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

constexpr int IW = 4;     // warps per block
constexpr int RING = 64;  // queued 32-candidate chunks per warp (covers a whole tile)

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

// FP32 pair evaluation (physics.py:183-220 restated for FP32 CUDA cores).  dx, r2 come
// from the caller.  Folded constants: k_gc = kc/h, k_tw = kc/W(dp); the 0.5 factors of the
// viscous term cancel; the neighbour's list mass travels in aux.w.
__device__ __forceinline__ void pair_eval(const KArgs& a, const Own<float>& o, float dx, float dy,
                                          float dz, float r2, const float4& vj, const float4& xa,
                                          Accum<float>& s) {
  const float rinv = rsqrtf(r2);
  const float r = r2 * rinv;
  const float q = r * a.invh;
  const float t = 2.0f - q;
  const float t2 = t * t;
  const float q2 = q * q;
  const bool inner = q < 1.0f;
  const float w = inner ? fmaf(0.75f * q, q2, fmaf(-1.5f, q2, 1.0f)) : 0.25f * t2 * t;
  const float dw = inner ? fmaf(2.25f, q, -3.0f) * q : -0.75f * t2;
  const float gc = dw * a.k_gc * rinv;
  const float dvx = o.vx - vj.x, dvy = o.vy - vj.y, dvz = o.vz - vj.z;
  const float dot = fmaf(dvz, dz, fmaf(dvy, dy, dvx * dx));
  const float mu = __fdividef(a.h * dot, r2 + a.eta2);
  const float vterm = __fdividef(-a.alpha * (o.cs + xa.y) * mu, o.rho + vj.w);
  const float visc = dot < 0.0f ? vterm : 0.0f;
  const float tw = w * a.k_tw;
  const float tw2 = tw * tw;
  const float pterm = fmaf((o.ten + xa.z) * tw2, tw2, o.prrho + xa.x + visc);
  const float mj = xa.w;
  const float fm = mj * pterm * gc;
  s.ax = fmaf(-fm, dx, s.ax);
  s.ay = fmaf(-fm, dy, s.ay);
  s.az = fmaf(-fm, dz, s.az);
  s.dr = fmaf(mj * gc, dot, s.dr);
  s.vd = fmaxf(s.vd, fabsf(mu));
}

// FP64 pair evaluation: the reference's exact operation order (physics.py:196-220,
// kernels.py:382-390), no contraction.  Bit-identical to numba.
__device__ __forceinline__ void pair_eval(const KArgs& a, const Own<double>& o, double dx,
                                          double dy, double dz, double r2, const float4& vj,
                                          const float4& xa, double mj, Accum<double>& s) {
  const sphb_params_t& p = a.p;
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

// Candidate screen.  FP32: "maybe" = r2 < sup2*(1+1e-5); the drain re-decides the rare
// maybes that are not sure hits (guard band, r2 ~ 0) exactly.  FP64: the exact predicate.
__device__ __forceinline__ bool cand_maybe(const KArgs& a, const Own<float>& o,
                                           const Stage<float>& c) {
  const float dx = o.x - c.v.x, dy = o.y - c.v.y, dz = o.z - c.v.z;
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  return r2 < a.sup2_hi;
}
__device__ __forceinline__ bool cand_maybe(const KArgs& a, const Own<double>& o,
                                           const Stage<double>& c) {
  return exact_hit(o.x, o.y, o.z, c.x, c.y, c.z, a.p.sup2);
}

// Evaluate one queued candidate j; returns false if it was a maybe that the exact
// predicate (or the stencil range) rejects.
__device__ __forceinline__ bool eval_one(const KArgs& a, const Own<float>& o, int32_t j, int xlo,
                                         int xhi, Accum<float>& s) {
  const float4 pj = __ldg(&a.posp[j]);
  const float4 vj = __ldg(&a.velr[j]);
  const float4 xa = __ldg(&a.aux[j]);
  const float dx = o.x - pj.x, dy = o.y - pj.y, dz = o.z - pj.z;
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  if (!(r2 < a.sup2_lo && r2 > a.tiny)) {
    // cold path: exact f64 predicate + stencil x-range (the y/z rows are the lane's own)
    const int cj = __ldg(&a.cell[j]);
    const int cxj = cj % a.g.dims[0];
    const bool ok = exact_hit((double)o.x, (double)o.y, (double)o.z, (double)pj.x, (double)pj.y,
                              (double)pj.z, a.p.sup2) && cxj >= xlo && cxj <= xhi;
    if (!ok) return false;
  }
  pair_eval(a, o, dx, dy, dz, r2, vj, xa, s);
  return true;
}
__device__ __forceinline__ bool eval_one(const KArgs& a, const Own<double>& o, int32_t j, int,
                                         int, Accum<double>& s) {
  const float4 pj = __ldg(&a.posp[j]);
  const float4 vj = __ldg(&a.velr[j]);
  const float4 xa = __ldg(&a.aux[j]);
  const double dx = xsub(o.x, (double)pj.x), dy = xsub(o.y, (double)pj.y),
               dz = xsub(o.z, (double)pj.z);
  const double r2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
  const double mj = j < a.nb ? a.p.mass_boundary : a.p.mass_fluid;
  pair_eval(a, o, dx, dy, dz, r2, vj, xa, mj, s);
  return true;
}

// ------------------------------------------------------------------ the kernel
template <typename R, bool FLUID_ITEMS>
__global__ void __launch_bounds__(IW * 32, sizeof(R) == 4 ? 6 : 3) k_interact(KArgs a) {
  if (!step_live(a.ctrl)) return;
  __shared__ Stage<R> s_stage[IW][32];
  __shared__ uint32_t s_mask[IW][RING][32];  // per-lane hit bitmask of each queued chunk
  __shared__ int32_t s_cbase[IW][RING];      // first candidate index of each queued chunk

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nitems = a.item_hi - a.item_lo;
  const uint32_t ntiles = (uint32_t)((nitems + 31) / 32);
  const int64_t step = a.ctrl->step;
  const int nx = a.g.dims[0], ny = a.g.dims[1], nz = a.g.dims[2];
  const int reach = a.g.reach;
  const int64_t nb = a.nb;

  unsigned long long c_cand = 0, c_hits = 0, c_ff = 0;
  double dtf_min = INFINITY, dtcv_min = INFINITY;

  for (;;) {
    uint32_t tile = 0;
    if (lane == 0) tile = atomicAdd(&a.ctrl->tile_next[FLUID_ITEMS ? 0 : 1], 1u);
    tile = __shfl_sync(SPHB_FULL, tile, 0);
    if (tile >= ntiles) break;
    const int64_t i = a.item_lo + (int64_t)tile * 32 + lane;
    const bool valid = i < a.item_hi;
    Own<R> o;
    int cx = 0, rowkey = -1;
    if (valid) {
      const float4 pi = a.posp[i], vi = a.velr[i], xi = a.aux[i];
      o.x = (R)pi.x; o.y = (R)pi.y; o.z = (R)pi.z;
      o.vx = (R)vi.x; o.vy = (R)vi.y; o.vz = (R)vi.z; o.rho = (R)vi.w;
      o.prrho = (R)xi.x; o.cs = (R)xi.y; o.ten = (R)xi.z;
      const int c = a.cell[i];
      rowkey = c / nx;
      cx = c - rowkey * nx;
    } else {
      o.x = o.y = o.z = o.vx = o.vy = o.vz = o.prrho = o.cs = o.ten = (R)0;
      o.rho = (R)1;
    }
    const int xlo = max(cx - reach, 0), xhi = min(cx + reach, nx - 1);
    Accum<R> s = {(R)0, (R)0, (R)0, (R)0, (R)0};
    uint32_t nslot = 0;        // queued chunks (warp-uniform)
    uint32_t pend = 0;         // queued candidate bits of this lane
    uint32_t pushed = 0, pushed_b = 0, rej = 0, rej_f = 0;
    unsigned long long cand = 0;

    // Evaluate every queued candidate, FIFO per lane, lock-step across the warp.
    auto drain = [&]() {
      __syncwarp();
      const uint32_t mx = __reduce_max_sync(SPHB_FULL, pend);
      uint32_t sl = 0;
      uint32_t cur = nslot ? s_mask[warp][0][lane] : 0u;
      for (uint32_t it = 0; it < mx; ++it) {
        while (cur == 0u && sl + 1 < nslot) cur = s_mask[warp][++sl][lane];
        if (cur) {
          const int t = __ffs(cur) - 1;
          cur &= cur - 1u;
          const int32_t j = s_cbase[warp][sl] + t;
          if (!eval_one(a, o, j, xlo, xhi, s)) {
            ++rej;
            if (j >= nb) ++rej_f;
          }
        }
      }
      nslot = 0;
      pend = 0;
      __syncwarp();
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
              const bool fluid_list = li == 0;  // li 1: boundary list
              if (!fluid_list && !FLUID_ITEMS) continue;
              if (npass == 2 && (pass == 0) != fluid_list) continue;
              const int64_t off = fluid_list ? a.ncells : 0;
              const int32_t u0 = a.beg[off + base + gxlo];
              const int32_t u1 = a.end[off + base + gxhi];
              if (u1 <= u0) continue;
              if (ing) cand += (unsigned long long)(a.end[off + base + xhi] - a.beg[off + base + xlo]);
              for (int32_t j0 = u0; j0 < u1; j0 += 32) {
                const int32_t jj = j0 + lane;
                const float4 pc = jj < u1 ? __ldg(&a.posp[jj])
                                          : make_float4(INFINITY, INFINITY, INFINITY, 0.f);
                stage_store(&s_stage[warp][lane], pc);
                __syncwarp();
                uint32_t bits = 0;
#pragma unroll
                for (int t = 0; t < 32; ++t)
                  if (cand_maybe(a, o, s_stage[warp][t])) bits |= 1u << t;
                bits = ing ? bits : 0u;
                __syncwarp();
                if (__any_sync(SPHB_FULL, bits != 0u)) {
                  if (nslot == RING) drain();
                  s_mask[warp][nslot][lane] = bits;
                  if (lane == 0) s_cbase[warp][nslot] = j0;
                  ++nslot;
                  const uint32_t pc2 = __popc(bits);
                  pend += pc2;
                  pushed += pc2;
                  if (!fluid_list) pushed_b += pc2;
                }
              }
            }
          }
        }
      }
    }
    drain();

    if (valid) {
      if (FLUID_ITEMS) cand -= 1;  // the reference skips j == i before counting (kernels.py:369-371)
      c_cand += cand;
      c_hits += pushed - rej;
      if (FLUID_ITEMS) c_ff += (pushed - pushed_b) - rej_f;
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
