// su_row.cuh -- the per-particle system update (verlet_update, sim.py:235-259; the symplectic
// stages of the extension), shared by K7 (integrate.cu) and the X-slab band update (slab.cu,
// which integrates a neighbour's edge rows with exactly K7's arithmetic).
#pragma once
#include "sphb_common.cuh"

namespace sphb {

__device__ __forceinline__ bool su_step_live(const sphb_ctrl_t* c) {
  return c->active && c->err >= ((uint64_t)(c->step + 1) << 40);
}

// compute_dt finalize (sim.py:231-232): clamp(cfl min(dt_f, dt_cv), dt_min, dt_max)
__device__ __forceinline__ double step_dt(const sphb_ctrl_t* c, const sphb_params_t& p) {
  const double dt_f = __longlong_as_double((long long)c->dtmin_f);
  const double dt_cv = __longlong_as_double((long long)c->dtmin_cv);
  double dt = xmul(p.cfl, fmin(dt_f, dt_cv));
  dt = fmax(dt, p.dt_min);
  return fmin(dt, p.dt_max);
}

// Piston law of the wave tank (extension): x(t) = x0 + S/2 (1 - cos wt),
// v(t) = S/2 w sin wt, w = 2 pi / T, for boundary ids in [piston_id0, piston_id1).
__device__ __forceinline__ void piston_at(const sphb_params_t& p, double t, float& x, float& vx) {
  const double w = xdiv(2.0 * 3.141592653589793, p.piston_period);
  const double hs = xmul(0.5, p.piston_stroke);
  x = __double2float_rn(xadd(p.piston_x0, xmul(hs, xsub(1.0, cos(xmul(w, t))))));
  vx = __double2float_rn(xmul(xmul(hs, w), sin(xmul(w, t))));
}

// Step constants of the update (one per launch).
struct SuStep {
  double dt, c2, dt2, hdt, t_new;
  bool corrector, piston;
  float px, pvx;  // the piston's x and vx at t_new (one law for every piston particle)
};

template <int MODE>
__device__ __forceinline__ SuStep su_step(const sphb_params_t& p, const sphb_ctrl_t* ctrl) {
  SuStep s;
  s.dt = MODE == 2 ? ctrl->dt_stage : step_dt(ctrl, p);
  s.corrector = (ctrl->step % p.verlet_stride) == 0;
  s.c2 = xmul(xmul(0.5, s.dt), s.dt);
  s.dt2 = xmul(2.0, s.dt);
  s.hdt = xmul(0.5, s.dt);
  s.piston = p.piston_id1 > p.piston_id0;
  // time the updated state belongs to (the piston law is evaluated there)
  s.t_new = MODE == 1 ? xadd(ctrl->t_sim, s.hdt) : xadd(ctrl->t_sim, s.dt);
  s.px = s.pvx = 0.f;
  if (s.piston) piston_at(p, s.t_new, s.px, s.pvx);
  return s;
}

// One particle: MODE 0 verlet_update (the reference), MODE 1 / 2 symplectic predictor /
// corrector.  f64 in numpy's evaluation order; the forces fa (fluid only) and drho widened
// exactly from either force layout.  np.w = 0 (press is recomputed by the next K3).
template <int MODE>
__device__ __forceinline__ void su_row(const sphb_params_t& p, const SuStep& s, bool fluid,
                                       int64_t pid, const float4 ps, const float4 vs,
                                       const float4 pv, const double fa[3], double dr, float4& np,
                                       float4& nv, float4& nprev) {
  double nrho;
  if (MODE == 0)
    nrho = s.corrector ? xadd((double)vs.w, xmul(s.dt, dr)) : xadd((double)pv.w, xmul(s.dt2, dr));
  else if (MODE == 1)
    nrho = xadd((double)vs.w, xmul(s.hdt, dr));
  else
    nrho = xadd((double)pv.w, xmul(s.dt, dr));
  if (fluid) {
    const double ax = xadd(fa[0], p.g[0]);
    const double ay = xadd(fa[1], p.g[1]);
    const double az = xadd(fa[2], p.g[2]);
    const double vx = (double)vs.x, vy = (double)vs.y, vz = (double)vs.z;
    if (MODE == 0) {
      np.x = __double2float_rn(xadd(xadd((double)ps.x, xmul(s.dt, vx)), xmul(s.c2, ax)));
      np.y = __double2float_rn(xadd(xadd((double)ps.y, xmul(s.dt, vy)), xmul(s.c2, ay)));
      np.z = __double2float_rn(xadd(xadd((double)ps.z, xmul(s.dt, vz)), xmul(s.c2, az)));
      if (s.corrector) {
        nv.x = __double2float_rn(xadd(vx, xmul(s.dt, ax)));
        nv.y = __double2float_rn(xadd(vy, xmul(s.dt, ay)));
        nv.z = __double2float_rn(xadd(vz, xmul(s.dt, az)));
      } else {
        nv.x = __double2float_rn(xadd((double)pv.x, xmul(s.dt2, ax)));
        nv.y = __double2float_rn(xadd((double)pv.y, xmul(s.dt2, ay)));
        nv.z = __double2float_rn(xadd((double)pv.z, xmul(s.dt2, az)));
      }
    } else if (MODE == 1) {  // r* = r + dt/2 v, v* = v + dt/2 (a + g)
      np.x = __double2float_rn(xadd((double)ps.x, xmul(s.hdt, vx)));
      np.y = __double2float_rn(xadd((double)ps.y, xmul(s.hdt, vy)));
      np.z = __double2float_rn(xadd((double)ps.z, xmul(s.hdt, vz)));
      nv.x = __double2float_rn(xadd(vx, xmul(s.hdt, ax)));
      nv.y = __double2float_rn(xadd(vy, xmul(s.hdt, ay)));
      nv.z = __double2float_rn(xadd(vz, xmul(s.hdt, az)));
    } else {  // v' = v + dt (a* + g), r' = r* + dt/2 v'
      const double ux = xadd((double)pv.x, xmul(s.dt, ax));
      const double uy = xadd((double)pv.y, xmul(s.dt, ay));
      const double uz = xadd((double)pv.z, xmul(s.dt, az));
      nv.x = __double2float_rn(ux);
      nv.y = __double2float_rn(uy);
      nv.z = __double2float_rn(uz);
      np.x = __double2float_rn(xadd((double)ps.x, xmul(s.hdt, (double)nv.x)));
      np.y = __double2float_rn(xadd((double)ps.y, xmul(s.hdt, (double)nv.y)));
      np.z = __double2float_rn(xadd((double)ps.z, xmul(s.hdt, (double)nv.z)));
    }
  } else {
    np.x = ps.x; np.y = ps.y; np.z = ps.z;  // boundary frozen (sim.py:256-258)
    nv.x = vs.x; nv.y = vs.y; nv.z = vs.z;
    if (s.piston && pid >= p.piston_id0 && pid < p.piston_id1) {
      np.x = s.px;
      nv.x = s.pvx;
    }
  }
  np.w = 0.f;  // press is recomputed by the next step's reorder (K3)
  nv.w = __double2float_rn(nrho);
  if (MODE == 2)
    nprev = nv;
  else
    nprev = vs;  // history <- current (sim.py:254-255); symplectic: (v, rho) at t
}

// x column of an in-domain position (grid.py:87-89, the x component of cell_of)
__device__ __forceinline__ int column_of(float x, const sphb_grid_t& g) {
  const int64_t v = (int64_t)floor(xdiv(xsub((double)x, g.origin[0]), g.cell_size));
  return (int)(v < 0 ? 0 : v < (int64_t)g.dims[0] - 1 ? v : (int64_t)g.dims[0] - 1);
}

}  // namespace sphb
