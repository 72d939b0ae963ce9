// state.cu -- the reference's host state layout <-> the device rows.
//
// The reference keeps a particle system as structure-of-arrays (model.py:25-43: pos (n, 3)
// f32, vel (n, 3) f32, rho (n,) f32, id (n,) i64) plus the Verlet history (sim.py:31-43:
// vel_prev (n, 3) f32, rho_prev (n,) f32).  A caller that round-trips that state through the
// GPU every step copies those arrays as they are (52 B per particle) into device staging
// buffers; these kernels convert them to / from the float4 rows of the step (posp, velr,
// prev; ids are the same int64 array and need no conversion).  Rows [r0, r0 + cnt) only, so
// chunked copies can convert each chunk as it lands.
#include "sphb_common.cuh"
#include "sphb_internal.h"

namespace {

__global__ void __launch_bounds__(256) k_state_unpack(int64_t r0, int64_t cnt,
                                                      const float* __restrict__ pos,
                                                      const float* __restrict__ vel,
                                                      const float* __restrict__ rho,
                                                      const float* __restrict__ vel_prev,
                                                      const float* __restrict__ rho_prev,
                                                      float4* __restrict__ posp,
                                                      float4* __restrict__ velr,
                                                      float4* __restrict__ prev) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += stride) {
    const int64_t i = r0 + k;
    posp[i] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], 0.0f);
    velr[i] = make_float4(vel[3 * i], vel[3 * i + 1], vel[3 * i + 2], rho[i]);
    prev[i] = make_float4(vel_prev[3 * i], vel_prev[3 * i + 1], vel_prev[3 * i + 2], rho_prev[i]);
  }
}

__global__ void __launch_bounds__(256) k_state_pack(int64_t r0, int64_t cnt,
                                                    const float4* __restrict__ posp,
                                                    const float4* __restrict__ velr,
                                                    const float4* __restrict__ prev,
                                                    float* __restrict__ pos, float* __restrict__ vel,
                                                    float* __restrict__ rho,
                                                    float* __restrict__ vel_prev,
                                                    float* __restrict__ rho_prev) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += stride) {
    const int64_t i = r0 + k;
    const float4 p = posp[i], v = velr[i], q = prev[i];
    pos[3 * i] = p.x;
    pos[3 * i + 1] = p.y;
    pos[3 * i + 2] = p.z;
    vel[3 * i] = v.x;
    vel[3 * i + 1] = v.y;
    vel[3 * i + 2] = v.z;
    rho[i] = v.w;
    vel_prev[3 * i] = q.x;
    vel_prev[3 * i + 1] = q.y;
    vel_prev[3 * i + 2] = q.z;
    rho_prev[i] = q.w;
  }
}

unsigned grid_of(int64_t cnt) {
  int64_t b = (cnt + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

int launch_state_unpack(int64_t r0, int64_t cnt, const float* pos, const float* vel,
                        const float* rho, const float* vel_prev, const float* rho_prev,
                        float4* posp, float4* velr, float4* prev, cudaStream_t s) {
  if (cnt <= 0) return SPHB_OK;
  k_state_unpack<<<grid_of(cnt), 256, 0, s>>>(r0, cnt, pos, vel, rho, vel_prev, rho_prev, posp,
                                              velr, prev);
  return sphb_check_launch("k_state_unpack");
}

int launch_state_pack(int64_t r0, int64_t cnt, const float4* posp, const float4* velr,
                      const float4* prev, float* pos, float* vel, float* rho, float* vel_prev,
                      float* rho_prev, cudaStream_t s) {
  if (cnt <= 0) return SPHB_OK;
  k_state_pack<<<grid_of(cnt), 256, 0, s>>>(r0, cnt, posp, velr, prev, pos, vel, rho, vel_prev,
                                            rho_prev);
  return sphb_check_launch("k_state_pack");
}
