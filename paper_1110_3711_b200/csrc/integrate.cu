// integrate.cu -- system update (SU) of the SPH step on sm_100a.
//
//   k_step_begin   stop rules of run_simulation (sim.py:302-305), per-step accumulators reset
//   K7 k_integrate compute_dt finalize (sim.py:231-232) + verlet_update (sim.py:235-259),
//                  fused with the NEXT step's assign_cells (grid.py:77-93, K1) and its
//                  per-list histogram; non-finite state / out-of-domain detection
//                  (sim.py:309-314, 332-333) recorded on the device
//   k_step_end     StepStats record (dt, counters), t_sim += dt, step += 1 (sim.py:336-351)
//
// All f64 arithmetic uses round-to-nearest intrinsics in the reference's numpy evaluation
// order, so the update is bit-identical to the reference for identical forces.
#include "sphb_common.cuh"
#include "sphb_internal.h"
#include "su_row.cuh"

using namespace sphb;

namespace {

__device__ __forceinline__ bool step_live(const sphb_ctrl_t* c) { return su_step_live(c); }

__global__ void k_ctrl_init(sphb_ctrl_t* c, int64_t max_steps, double t_end) {
  c->step = 0;
  c->max_steps = max_steps;
  c->t_sim = 0.0;
  c->t_end = t_end;
  c->dt = 0.0;
  c->dtmin_f = (uint64_t)__double_as_longlong(INFINITY);
  c->dtmin_cv = (uint64_t)__double_as_longlong(INFINITY);
  c->err = ~0ull;
  for (int k = 0; k < 4; ++k) c->counters[k] = 0;
  c->active = 1;
  c->tile_next[0] = c->tile_next[1] = 0;
  c->nblk[0] = c->nblk[1] = 0;
}

__global__ void k_step_begin(sphb_ctrl_t* c) {
  if (!c->active) return;
  // the stop rule first (sim.py:302-305 runs before assign_cells at 309-314): a particle that
  // left the domain during the final step (K7 records it against step + 1) ends the run
  // normally, as in the reference; the host ignores that record (DeviceSim.error)
  if ((c->max_steps >= 0 && c->step >= c->max_steps) || (c->t_sim >= c->t_end)) {
    c->active = 0;
    return;
  }
  if (!step_live(c)) return;
  c->dtmin_f = (uint64_t)__double_as_longlong(INFINITY);
  c->dtmin_cv = (uint64_t)__double_as_longlong(INFINITY);
  for (int k = 0; k < 4; ++k) c->counters[k] = 0;
  c->tile_next[0] = c->tile_next[1] = 0;
  c->nblk[0] = c->nblk[1] = 0;
}

// MODE 0: verlet_update (sim.py:235-259), the reference.  MODE 1 / 2: symplectic predictor /
// corrector (extension).  All fused with the next stage's assign_cells (K1) + histogram.
// F32: the FP32 force layout (float4 (ax, ay, az, drho) per particle in `acc`, include/
// sphb200.h), widened exactly to f64 -- the same arithmetic as the FP64 layout's values.
template <int MODE, bool F32, bool SLAB>
#ifndef SU_MINB
#define SU_MINB 4  // 64 registers: 2x the resident warps of the default (memory-bound kernel)
#endif
__global__ void __launch_bounds__(256, SU_MINB) k_integrate(
    sphb_params_t p, sphb_grid_t g, int cellbits, int64_t ncells, int64_t n, int64_t nb,
    const float4* __restrict__ posp_s, const float4* __restrict__ velr_s,
    const float4* __restrict__ prev_s, const int64_t* __restrict__ id_s,
    const void* __restrict__ accv, const double* __restrict__ drho, float4* __restrict__ posp,
    float4* __restrict__ velr, float4* __restrict__ prev, int64_t* __restrict__ id,
    uint32_t* __restrict__ keys_next, uint32_t* __restrict__ cnt, sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  const int64_t step = ctrl->step;
  const SuStep st = su_step<MODE>(p, ctrl);
  // X slab (dslab): last step's halo copies and rows that left the slab get the dead key (they
  // sort to the tail and drop out); a row moving more than one column in one step would escape
  // the neighbours' edge bands (slab.cu), which is flagged
  constexpr bool slab = MODE == 0 && SLAB;  // the single-domain build carries none of it
  const uint32_t dead = dead_key(cellbits);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int64_t slot = -1;
    if (i < n) {
      const int64_t pid = id_s[i];
      if (slab && pid < 0) {  // a halo copy (its owner integrates the particle)
        id[i] = pid;
        keys_next[i] = dead;
        slot = 2 * ncells;
      } else {
        const float4 ps = posp_s[i], vs = velr_s[i], pv = prev_s[i];
        double fa[3] = {0.0, 0.0, 0.0}, dr;
        if (F32) {
          const float4 a4 = ((const float4*)accv)[i];
          fa[0] = a4.x;
          fa[1] = a4.y;
          fa[2] = a4.z;
          dr = a4.w;
        } else {
          const double* acc = (const double*)accv;
          dr = drho[i];
          if (i >= nb) {
            fa[0] = acc[3 * i + 0];
            fa[1] = acc[3 * i + 1];
            fa[2] = acc[3 * i + 2];
          }
        }
        float4 np, nv, nprev;
        su_row<MODE>(p, st, i >= nb, pid, ps, vs, pv, fa, dr, np, nv, nprev);
        posp[i] = np;
        velr[i] = nv;
        prev[i] = nprev;
        id[i] = pid;
        if (!(isfinite(nv.x) && isfinite(nv.y) && isfinite(nv.z) && isfinite(nv.w)))
          raise_div(ctrl, step, SPHB_DIV_NONFINITE_STATE, 0);
        // next step's assign_cells (K1), fused
        const int32_t c = cell_of(np.x, np.y, np.z, g);
        if (c < 0) {
          raise_div(ctrl, MODE == 1 ? step : step + 1, SPHB_DIV_LEFT_DOMAIN, (uint64_t)i);
          keys_next[i] = 0xffffffffu;
        } else {
          const uint32_t list = i >= nb ? 1u : 0u;
          keys_next[i] = (list << cellbits) | (uint32_t)c;
          slot = (int64_t)list * ncells + c;
          if (slab) {
            const int col = c % g.dims[0], ocol = column_of(ps.x, g);
            if (col - ocol > 1 || ocol - col > 1)
              raise_div(ctrl, step + 1, SPHB_DIV_SLAB_MARGIN, (uint64_t)i);
            if (col < g.tx0 || col >= g.tx1) {  // migrated: the neighbour integrated it too
              keys_next[i] = dead;
              slot = 2 * ncells;
            }
          }
        }
      }
    }
    const uint32_t peers = __match_any_sync(SPHB_FULL, (unsigned long long)slot);
    if (slot >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[slot], (uint32_t)__popc(peers));
  }
}

// symplectic: fix the step's dt and counters after the first stage, reset the per-stage
// accumulators for the second interaction
__global__ void k_stage_mid(sphb_ctrl_t* c, sphb_params_t p) {
  if (!step_live(c)) return;
  c->dt_stage = step_dt(c, p);
  for (int k = 0; k < 4; ++k) {
    c->counters_stage[k] = c->counters[k];
    c->counters[k] = 0;
  }
  c->dtmin_f = (uint64_t)__double_as_longlong(INFINITY);
  c->dtmin_cv = (uint64_t)__double_as_longlong(INFINITY);
  c->tile_next[0] = c->tile_next[1] = 0;
  c->nblk[0] = c->nblk[1] = 0;
}

// ---------------------------------------------------------------- energy diagnostics
constexpr int EN_BLOCKS = 592, EN_THREADS = 256;

__device__ __forceinline__ double tait_u(double r, const sphb_params_t& p) {
  const double B = p.tait_b, gm = p.gamma;
  return xadd(xdiv(xmul(xdiv(B, xsub(gm, 1.0)), pow(r, xsub(gm, 1.0))), pow(p.rho0, gm)), xdiv(B, r));
}

__global__ void __launch_bounds__(EN_THREADS) k_energy_part(sphb_params_t p, int64_t n, int64_t nb,
                                                            const float4* __restrict__ posp,
                                                            const float4* __restrict__ velr,
                                                            double* __restrict__ part) {
  __shared__ double sm[5][EN_THREADS];
  double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double gmag = sqrt(p.g[0] * p.g[0] + p.g[1] * p.g[1] + p.g[2] * p.g[2]);
  const double u0 = tait_u(p.rho0, p);
  for (int64_t i = (int64_t)blockIdx.x * EN_THREADS + threadIdx.x; i < n;
       i += (int64_t)EN_BLOCKS * EN_THREADS) {
    const float4 v = velr[i];
    const bool fl = i >= nb;
    const double m = fl ? p.mass_fluid : p.mass_boundary;
    const double r = (double)v.w;
    if (fl) {
      const double vx = v.x, vy = v.y, vz = v.z;
      a[0] += m * (vx * vx + vy * vy + vz * vz);
      a[1] += m * gmag * (double)posp[i].z;
      a[3] += r;
    }
    a[2] += m * (tait_u(r, p) - u0);
    a[4] += r;
  }
  for (int k = 0; k < 5; ++k) sm[k][threadIdx.x] = a[k];
  __syncthreads();
  for (int w = EN_THREADS / 2; w > 0; w >>= 1) {  // fixed-shape tree: deterministic
    if (threadIdx.x < w)
      for (int k = 0; k < 5; ++k) sm[k][threadIdx.x] += sm[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 5) part[blockIdx.x * 5 + threadIdx.x] = sm[threadIdx.x][0];
}

__global__ void k_energy_final(int64_t n, int64_t nb, const double* __restrict__ part,
                               double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < EN_BLOCKS; ++b)
    for (int k = 0; k < 5; ++k) a[k] += part[b * 5 + k];
  out[0] = 0.5 * a[0];
  out[1] = a[1];
  out[2] = a[2];
  out[3] = n > nb ? a[3] / (double)(n - nb) : 0.0;
  out[4] = n > 0 ? a[4] / (double)n : 0.0;
}

__global__ void k_step_end(sphb_ctrl_t* c, sphb_params_t p, sphb_step_record_t* rec, int64_t cap) {
  if (!step_live(c)) return;
  const bool symp = p.integrator == SPHB_INT_SYMPLECTIC;
  const double dt = symp ? c->dt_stage : step_dt(c, p);
  const uint64_t* cnt = symp ? c->counters_stage : c->counters;
  if (rec && cap > 0) {
    sphb_step_record_t r;
    r.dt = dt;
    r.candidate_pairs = cnt[0];
    r.hits_ordered = cnt[1];
    r.force_evals = cnt[2];
    r.ff_force_evals = cnt[3];
    rec[c->step % cap] = r;
  }
  c->dt = dt;
  c->t_sim = xadd(c->t_sim, dt);
  c->step = c->step + 1;
}

}  // namespace

int launch_ctrl_init(sphb_ctrl_t* ctrl, int64_t max_steps, double t_end, cudaStream_t s) {
  k_ctrl_init<<<1, 1, 0, s>>>(ctrl, max_steps, t_end);
  return sphb_check_launch("k_ctrl_init");
}

int launch_step_begin(sphb_ctrl_t* ctrl, cudaStream_t s) {
  k_step_begin<<<1, 1, 0, s>>>(ctrl);
  return sphb_check_launch("k_step_begin");
}

int launch_integrate_mode(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                          int64_t n, int64_t nb, int mode, const float4* posp_s,
                          const float4* velr_s, const float4* prev_s, const int64_t* id_s,
                          const void* acc, const void* drho, float4* posp, float4* velr,
                          float4* prev, int64_t* id, uint32_t* keys_next, sphb_ctrl_t* ctrl,
                          cudaStream_t s) {
  if (p.verlet_stride < 1) return sphb_set_error(SPHB_E_INVALID, "verlet_corrector_stride must be >= 1");
  if (p.piston_id1 > p.piston_id0 && !(p.piston_period > 0.0))
    return sphb_set_error(SPHB_E_INVALID, "piston period must be positive");
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    const int cb = cellbits_of(g);
    const int64_t nc = ncells_of(g);
    const double* dr = (const double*)drho;
    const bool f32 = p.precision == SPHB_FP32;
#define SPHB_K7(M, F, S)                                                                        \
  k_integrate<M, F, S><<<(unsigned)blocks, 256, 0, s>>>(p, g, cb, nc, n, nb, posp_s, velr_s,    \
                                                        prev_s, id_s, acc, dr, posp, velr, prev, \
                                                        id, keys_next, ws->cnt, ctrl)
    const bool slab = slab_grid(g);  // an X slab's dead-key rules (verlet only)
    if (mode == 0) {
      if (slab) {
        if (f32) SPHB_K7(0, true, true); else SPHB_K7(0, false, true);
      } else {
        if (f32) SPHB_K7(0, true, false); else SPHB_K7(0, false, false);
      }
    } else if (mode == 1) {
      if (f32) SPHB_K7(1, true, false); else SPHB_K7(1, false, false);
    } else {
      if (f32) SPHB_K7(2, true, false); else SPHB_K7(2, false, false);
    }
#undef SPHB_K7
    if (int rc = sphb_check_launch("k_integrate")) return rc;
  }
  if (mode == 1) {
    k_stage_mid<<<1, 1, 0, s>>>(ctrl, p);
    return sphb_check_launch("k_stage_mid");
  }
  return SPHB_OK;
}

int launch_integrate(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g, int64_t n,
                     int64_t nb, const float4* posp_s, const float4* velr_s, const float4* prev_s,
                     const int64_t* id_s, const void* acc, const void* drho, float4* posp,
                     float4* velr, float4* prev, int64_t* id, uint32_t* keys_next,
                     sphb_ctrl_t* ctrl, cudaStream_t s) {
  return launch_integrate_mode(ws, p, g, n, nb, 0, posp_s, velr_s, prev_s, id_s, acc, drho, posp,
                               velr, prev, id, keys_next, ctrl, s);
}

int launch_energy(sphb_workspace* ws, const sphb_params_t& p, int64_t n, int64_t nb,
                  const float4* posp, const float4* velr, double* out, cudaStream_t s) {
  k_energy_part<<<EN_BLOCKS, EN_THREADS, 0, s>>>(p, n, nb, posp, velr, ws->energy_part);
  if (int rc = sphb_check_launch("k_energy_part")) return rc;
  k_energy_final<<<1, 32, 0, s>>>(n, nb, ws->energy_part, out);
  return sphb_check_launch("k_energy_final");
}

int launch_step_end(sphb_ctrl_t* ctrl, const sphb_params_t& p, sphb_step_record_t* rec,
                    int64_t cap, cudaStream_t s) {
  k_step_end<<<1, 1, 0, s>>>(ctrl, p, rec, cap);
  return sphb_check_launch("k_step_end");
}
