// stepfn.cu -- the reference's module-level step functions on the device, for callers that run
// their own loop around them (the whole-step surface, and the monkeypatch
// parity trick on sphbench.sim).  sphb_step fuses all of this; these kernels take the
// reference's own array layouts instead.
//
//   k_build_ranges  build_ranges (grid.py:170-200): per cell, the (2n+1)^2 row ranges of its
//                   candidate block from one list's begin/end, clipped to the grid
//   k_dt_terms      compute_dt (sim.py:215-232): min over fluid of sqrt(h / max(|a + g|, TINY))
//                   and min over all of h / (csound + visc_dt), f64 in the reference's order
//   k_verlet_soa    verlet_update (sim.py:235-259) on (n, 3) / (n,) f32 arrays, f64 arithmetic
//                   in numpy's evaluation order (bit-identical)
//   k_sym_cand      StepStats of the symmetric traversal (SPHB_COUNTERS_SYMMETRIC): the
//   k_sym_final     half-stencil candidate count of run_cells_symmetric (kernels.py:121-175)
//                   per cell from begin/end, force_evals = unordered pairs, ff unordered
//                   (cellpairs.py:92-99 reports the symmetric counts as they are)
//   k_forces_f64    the FP32 force layout (float4 acc + drho, float visc) widened to the
//                   ForceOutput f64 arrays (config.py:94-103)
#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

__global__ void __launch_bounds__(256) k_build_ranges(const int32_t* __restrict__ beg,
                                                      const int32_t* __restrict__ end, int nx,
                                                      int ny, int nz, int n_sub,
                                                      long long* __restrict__ rb,
                                                      long long* __restrict__ re) {
  const int side = 2 * n_sub + 1, nr = side * side;
  const int64_t ncells = (int64_t)nx * ny * nz;
  const int64_t total = ncells * nr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t c = t / nr;
    const int k = (int)(t - c * nr);
    const int dz = k / side - n_sub, dy = k % side - n_sub;
    const int cx = (int)(c % nx), cy = (int)((c / nx) % ny), cz = (int)(c / ((int64_t)nx * ny));
    const int yy = cy + dy, zz = cz + dz;
    const bool ok = zz >= 0 && zz < nz && yy >= 0 && yy < ny;
    const int xlo = max(cx - n_sub, 0), xhi = min(cx + n_sub, nx - 1);
    const int64_t row = ((int64_t)zz * ny + yy) * nx;
    rb[t] = ok ? beg[row + xlo] : 0;
    re[t] = ok ? end[row + xhi] : 0;
  }
}

__global__ void __launch_bounds__(256) k_dt_terms(int64_t n, int64_t nb, const double* __restrict__ acc,
                                                  const double* __restrict__ visc,
                                                  const float* __restrict__ csound,
                                                  sphb_params_t p, uint64_t* __restrict__ out) {
  double dtf = INFINITY, dtcv = INFINITY;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (i >= nb) {
      const double fx = xadd(acc[3 * i], p.g[0]), fy = xadd(acc[3 * i + 1], p.g[1]),
                   fz = xadd(acc[3 * i + 2], p.g[2]);
      double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
      fmag = fmag > 1e-30 ? fmag : 1e-30;  // TINY_FORCE (sim.py:19)
      dtf = fmin(dtf, __dsqrt_rn(xdiv(p.h, fmag)));
    }
    dtcv = fmin(dtcv, xdiv(p.h, xadd((double)csound[i], visc[i])));
  }
  dtf = warp_min(dtf);
  dtcv = warp_min(dtcv);
  if ((threadIdx.x & 31) == 0) {
    if (dtf < INFINITY) atomic_min_pos(&out[0], dtf);
    if (dtcv < INFINITY) atomic_min_pos(&out[1], dtcv);
  }
}

__global__ void __launch_bounds__(256) k_verlet_soa(int64_t n, int64_t nb, int corrector, double dt,
                                                    sphb_params_t p, float* __restrict__ pos,
                                                    float* __restrict__ vel, float* __restrict__ rho,
                                                    float* __restrict__ vel_prev,
                                                    float* __restrict__ rho_prev,
                                                    const double* __restrict__ acc,
                                                    const double* __restrict__ drho) {
  const double c2 = xmul(xmul(0.5, dt), dt), dt2 = xmul(2.0, dt);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float r0 = rho[i], rp = rho_prev[i];
    const double nr = corrector ? xadd((double)r0, xmul(dt, drho[i]))
                                : xadd((double)rp, xmul(dt2, drho[i]));
    float v[3], vp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = vel[3 * i + k];
      vp[k] = vel_prev[3 * i + k];
    }
    if (i >= nb) {  // fluid moves; boundary keeps pos / vel (sim.py:256-258)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double a = xadd(acc[3 * i + k], p.g[k]);
        const double vk = (double)v[k];
        pos[3 * i + k] = __double2float_rn(xadd(xadd((double)pos[3 * i + k], xmul(dt, vk)), xmul(c2, a)));
        vel[3 * i + k] = __double2float_rn(corrector ? xadd(vk, xmul(dt, a))
                                                     : xadd((double)vp[k], xmul(dt2, a)));
      }
    }
    // history <- the state before this update (sim.py:254-255)
#pragma unroll
    for (int k = 0; k < 3; ++k) vel_prev[3 * i + k] = v[k];
    rho_prev[i] = r0;
    rho[i] = __double2float_rn(nr);
  }
}

__global__ void __launch_bounds__(256) k_forces_f64(int64_t n, const float4* __restrict__ acc4,
                                                    const float* __restrict__ visc32,
                                                    double* __restrict__ acc, double* __restrict__ drho,
                                                    double* __restrict__ visc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float4 a = acc4[i];
    acc[3 * i + 0] = a.x;
    acc[3 * i + 1] = a.y;
    acc[3 * i + 2] = a.z;
    drho[i] = a.w;
    visc[i] = visc32[i];
  }
}

__device__ __forceinline__ bool live(const sphb_ctrl_t* c) {
  return c->active && c->err >= ((uint64_t)(c->step + 1) << 40);
}

// per cell c: nf(nf-1)/2 + nf nb + sum over forward cells d of (nf nf_d + nf nb_d + nb nf_d)
// (scan_block calls of run_cells_symmetric, kernels.py:144-175; forward_offsets grid.py:147-156)
__global__ void __launch_bounds__(256) k_sym_cand(sphb_grid_t g, const int32_t* __restrict__ beg,
                                                  const int32_t* __restrict__ end,
                                                  unsigned long long* out, const sphb_ctrl_t* ctrl) {
  if (!live(ctrl)) return;
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2], R = g.reach;
  const int64_t nc = (int64_t)nx * ny * nz;
  unsigned long long acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += stride) {
    const long long nf = end[nc + c] - beg[nc + c], nbc = end[c] - beg[c];
    if (nf == 0 && nbc == 0) continue;
    const int cz = (int)(c / ((int64_t)nx * ny)), rem = (int)(c - (int64_t)cz * nx * ny);
    const int cy = rem / nx, cx = rem - cy * nx;
    long long t = nf * (nf - 1) / 2 + nf * nbc;
    for (int dz = 0; dz <= R; ++dz) {
      const int zz = cz + dz;
      if (zz >= nz) continue;
      for (int dy = dz > 0 ? -R : 0; dy <= R; ++dy) {
        const int yy = cy + dy;
        if (yy < 0 || yy >= ny) continue;
        for (int dx = (dz > 0 || dy > 0) ? -R : 1; dx <= R; ++dx) {
          const int xx = cx + dx;
          if (xx < 0 || xx >= nx) continue;
          const int64_t d = xx + (int64_t)nx * (yy + (int64_t)ny * zz);
          const long long nfd = end[nc + d] - beg[nc + d], nbd = end[d] - beg[d];
          t += nf * nfd + nf * nbd + nbc * nfd;
        }
      }
    }
    acc += (unsigned long long)t;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// gather-type counters (ordered hits, evals = ordered hits, ff ordered) -> symmetric ones
__global__ void k_sym_final(sphb_ctrl_t* ctrl, unsigned long long* cand) {
  if (live(ctrl)) {
    ctrl->counters[0] = *cand;
    ctrl->counters[2] = ctrl->counters[1] / 2;
    ctrl->counters[3] = ctrl->counters[3] / 2;
  }
  *cand = 0;
}

unsigned grid_of(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

int launch_sym_counters(sphb_workspace* ws, const sphb_grid_t& g, const int32_t* beg,
                        const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s) {
  const int64_t nc = (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
  k_sym_cand<<<grid_of(nc), 256, 0, s>>>(g, beg, end, ws->sym_scratch, ctrl);
  if (int rc = sphb_check_launch("k_sym_cand")) return rc;
  k_sym_final<<<1, 1, 0, s>>>(ctrl, ws->sym_scratch);
  return sphb_check_launch("k_sym_final");
}

extern "C" {

int sphb_build_ranges(const int32_t* beg, const int32_t* end, int32_t nx, int32_t ny, int32_t nz,
                      int32_t n_subdiv, int64_t* range_begin, int64_t* range_end,
                      sphb_stream_t s) {
  if (nx < 1 || ny < 1 || nz < 1) return sphb_set_error(SPHB_E_INVALID, "bad dims");
  if (n_subdiv != 1 && n_subdiv != 2)
    return sphb_set_error(SPHB_E_INVALID, "interaction ranges support n_subdiv in {1, 2} only");
  if (!beg || !end || !range_begin || !range_end) return sphb_set_error(SPHB_E_INVALID, "null pointer");
  const int64_t total = (int64_t)nx * ny * nz * (2 * n_subdiv + 1) * (2 * n_subdiv + 1);
  k_build_ranges<<<grid_of(total), 256, 0, (cudaStream_t)s>>>(beg, end, nx, ny, nz, n_subdiv,
                                                              (long long*)range_begin,
                                                              (long long*)range_end);
  return sphb_check_launch("k_build_ranges");
}

int sphb_dt_terms(const sphb_params_t* prm, int64_t n, int64_t nb, const double* accel,
                  const double* visc_dt, const float* csound, uint64_t* out2, sphb_stream_t s) {
  if (!prm || !out2) return sphb_set_error(SPHB_E_INVALID, "null pointer");
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0 && (!accel || !visc_dt || !csound)) return sphb_set_error(SPHB_E_INVALID, "null pointer");
  if (n == 0) return SPHB_OK;
  k_dt_terms<<<grid_of(n), 256, 0, (cudaStream_t)s>>>(n, nb, accel, visc_dt, csound, *prm, out2);
  return sphb_check_launch("k_dt_terms");
}

int sphb_verlet_soa(const sphb_params_t* prm, int64_t n, int64_t nb, int32_t corrector, double dt,
                    float* pos, float* vel, float* rho, float* vel_prev, float* rho_prev,
                    const double* accel, const double* drho_dt, sphb_stream_t s) {
  if (!prm) return sphb_set_error(SPHB_E_INVALID, "null pointer");
  if (!(dt > 0.0)) return sphb_set_error(SPHB_E_INVALID, "dt must be positive");
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n == 0) return SPHB_OK;
  if (!pos || !vel || !rho || !vel_prev || !rho_prev || !accel || !drho_dt)
    return sphb_set_error(SPHB_E_INVALID, "null pointer");
  k_verlet_soa<<<grid_of(n), 256, 0, (cudaStream_t)s>>>(n, nb, corrector, dt, *prm, pos, vel, rho,
                                                        vel_prev, rho_prev, accel, drho_dt);
  return sphb_check_launch("k_verlet_soa");
}

int sphb_forces_f64(const sphb_params_t* prm, int64_t n, const void* acc, const void* drho,
                    const void* visc, double* acc64, double* drho64, double* visc64,
                    sphb_stream_t s) {
  if (!prm) return sphb_set_error(SPHB_E_INVALID, "null pointer");
  if (n < 0) return sphb_set_error(SPHB_E_INVALID, "bad n");
  if (n == 0) return SPHB_OK;
  if (!acc || !visc || !acc64 || !drho64 || !visc64 || (prm->precision == SPHB_FP64 && !drho))
    return sphb_set_error(SPHB_E_INVALID, "null pointer");
  cudaStream_t cs = (cudaStream_t)s;
  if (prm->precision == SPHB_FP64) {
    cudaMemcpyAsync(acc64, acc, 24 * (size_t)n, cudaMemcpyDeviceToDevice, cs);
    cudaMemcpyAsync(drho64, drho, 8 * (size_t)n, cudaMemcpyDeviceToDevice, cs);
    cudaMemcpyAsync(visc64, visc, 8 * (size_t)n, cudaMemcpyDeviceToDevice, cs);
    return sphb_check_launch("forces copy");
  }
  k_forces_f64<<<grid_of(n), 256, 0, cs>>>(n, (const float4*)acc, (const float*)visc, acc64,
                                           drho64, visc64);
  return sphb_check_launch("k_forces_f64");
}

}  // extern "C"
