// capi.cu -- extern "C" entry points of libsphb200.so (see include/sphb200.h).
//
// Thin: argument checks, workspace management, error strings; the kernels live in
// nl.cu / interact.cu / integrate.cu.  No C++ exception crosses the ABI.
#include <nvtx3/nvToolsExt.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "sphb_common.cuh"
#include "sphb_internal.h"

// NVTX stage ranges (header-only NVTX v3: free unless a tool such as nsys / ncu --nvtx attaches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local char g_err[512] = "";

int sphb_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int sphb_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return sphb_set_error(SPHB_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return SPHB_OK;
}

#define SPHB_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return sphb_set_error(SPHB_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_));        \
  } while (0)

#define SPHB_NONNULL(p)                                                                  \
  do {                                                                                   \
    if (!(p)) return sphb_set_error(SPHB_E_INVALID, "%s: null pointer %s", __func__, #p); \
  } while (0)

static int check_grid(const sphb_grid_t* g) {
  SPHB_NONNULL(g);
  for (int k = 0; k < 3; ++k)
    if (g->dims[k] < 1) return sphb_set_error(SPHB_E_INVALID, "grid dims must be >= 1");
  if (!(g->cell_size > 0)) return sphb_set_error(SPHB_E_INVALID, "cell_size must be positive");
  if (g->tx0 < 0 || g->tx1 > g->dims[0] || g->tx0 > g->tx1)
    return sphb_set_error(SPHB_E_INVALID, "target columns [tx0, tx1) must lie in [0, dims[0]]");
  if (sphb::ncells_of(*g) >= (int64_t(1) << 30))
    return sphb_set_error(SPHB_E_INVALID, "ncells >= 2^30 unsupported (31-bit sort keys)");
  return SPHB_OK;
}

static int check_params(const sphb_params_t* p) {
  SPHB_NONNULL(p);
  if (p->kernel != SPHB_KERNEL_CUBIC && p->kernel != SPHB_KERNEL_WENDLAND)
    return sphb_set_error(SPHB_E_INVALID, "kernel must be SPHB_KERNEL_CUBIC or SPHB_KERNEL_WENDLAND");
  if (p->integrator != SPHB_INT_VERLET && p->integrator != SPHB_INT_SYMPLECTIC)
    return sphb_set_error(SPHB_E_INVALID, "integrator must be SPHB_INT_VERLET or SPHB_INT_SYMPLECTIC");
  if (p->precision != SPHB_FP32 && p->precision != SPHB_FP64)
    return sphb_set_error(SPHB_E_INVALID, "precision must be SPHB_FP32 or SPHB_FP64");
  if (!(p->wall_d >= 0.0)) return sphb_set_error(SPHB_E_INVALID, "wall_d must be >= 0");
  if (p->counters != SPHB_COUNTERS_GATHER && p->counters != SPHB_COUNTERS_SYMMETRIC)
    return sphb_set_error(SPHB_E_INVALID, "counters must be SPHB_COUNTERS_GATHER or SPHB_COUNTERS_SYMMETRIC");
  if (p->wall_d > 0.0) {
    if (!(p->wall_r0 > 0.0 && p->wall_r0 <= 2.0 * p->h))
      return sphb_set_error(SPHB_E_INVALID, "wall_r0 must lie in (0, 2h]");
    if (!(p->wall_p2 >= 1 && p->wall_p1 > p->wall_p2 && p->wall_p1 <= 16))
      return sphb_set_error(SPHB_E_INVALID, "wall exponents need 1 <= p2 < p1 <= 16");
  }
  return SPHB_OK;
}

int launch_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g, int64_t n,
                    int64_t nb, const float4* posp, const float4* velr, const float4* aux,
                    const int32_t* cell_sorted, const int32_t* beg, const int32_t* end,
                    void* acc, void* drho, void* visc, sphb_ctrl_t* ctrl, cudaStream_t s) {
  int rc;
  const bool f32 = p.precision == SPHB_FP32;
  if (ws->pi_kernel == SPHB_PI_PAIRED && f32)
    rc = pi512p::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                 visc, ctrl, s);
  else if (ws->pi_kernel == SPHB_PI_SYMMETRIC && f32 && p.order == 0)
    rc = pi384s::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                 visc, ctrl, s);
  else if (ws->pi_block == 256 && f32)
    rc = pi256::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                visc, ctrl, s);
  else if (ws->pi_block == 512 && f32)
    rc = pi512::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                visc, ctrl, s);
  else if (ws->pi_block == PI_LARGE_BLOCK && f32)
    rc = pi384::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                visc, ctrl, s);
  else
    rc = pi128::launch_interact(ws, p, g, n, nb, posp, velr, aux, cell_sorted, beg, end, acc, drho,
                                visc, ctrl, s);
  if (rc || p.counters != SPHB_COUNTERS_SYMMETRIC) return rc;
  return launch_sym_counters(ws, g, beg, end, ctrl, s);
}

constexpr int64_t PLAN_ASYNC_MIN_ROWS = 1 << 19;
static int plan_dispatch(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                         const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s) {
  const bool f32 = p.precision == SPHB_FP32;  // the same build choice as launch_interact
  if (ws->pi_kernel == SPHB_PI_PAIRED && f32) return pi512p::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
  if (ws->pi_kernel == SPHB_PI_SYMMETRIC && f32 && p.order == 0)
    return pi384s::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
  if (ws->pi_block == 256 && f32) return pi256::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
  if (ws->pi_block == 512 && f32) return pi512::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
  if (ws->pi_block == PI_LARGE_BLOCK && f32) return pi384::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
  return pi128::plan_interact(ws, p, g, beg, end, ctrl, s, ws->cand_acc);
}

int plan_interact_async(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                        const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s) {
  ws->plan.valid = false;
  // small systems (launch-bound, CUDA graphs): K3 takes a few microseconds, the side branch
  // would only add its fork / join -- sphb_interact builds the list in line
  if (ws->n_max < PLAN_ASYNC_MIN_ROWS) return SPHB_OK;
  if (cudaError_t e = cudaEventRecord(ws->ev_fork, s))
    return sphb_set_error(SPHB_E_CUDA, "plan fork: %s", cudaGetErrorString(e));
  if (cudaError_t e = cudaStreamWaitEvent(ws->side, ws->ev_fork, 0))
    return sphb_set_error(SPHB_E_CUDA, "plan fork: %s", cudaGetErrorString(e));
  if (int rc = plan_dispatch(ws, p, g, beg, end, ctrl, ws->side)) return rc;
  if (cudaError_t e = cudaEventRecord(ws->ev_plan, ws->side))
    return sphb_set_error(SPHB_E_CUDA, "plan join: %s", cudaGetErrorString(e));
  sphb_workspace::Plan& pl = ws->plan;
  pl.beg = beg;
  pl.end = end;
  for (int k = 0; k < 3; ++k) pl.dims[k] = g.dims[k];
  pl.tx0 = g.tx0;
  pl.tx1 = g.tx1;
  pl.reach = g.reach;
  pl.precision = p.precision;
  pl.order = p.order;
  pl.pi_block = ws->pi_block;
  pl.pi_kernel = ws->pi_kernel;
  pl.valid = true;
  return SPHB_OK;
}

int64_t interact_launch_count(int64_t n) { return pi128::interact_launch_count(n); }

extern "C" {

const char* sphb_last_error(void) { return g_err; }
const char* sphb_version(void) { return "sphb200 0.1 (sm_100a)"; }

int sphb_workspace_create(int64_t n_max, int64_t ncells_max, sphb_workspace_t** out) {
  SPHB_NONNULL(out);
  if (n_max < 0 || ncells_max < 1) return sphb_set_error(SPHB_E_INVALID, "bad capacities");
  if (n_max >= (int64_t(1) << 31)) return sphb_set_error(SPHB_E_INVALID, "n_max >= 2^31");
  sphb_workspace* ws = new (std::nothrow) sphb_workspace();
  if (!ws) return sphb_set_error(SPHB_E_INVALID, "host allocation failed");
  ws->n_max = n_max;
  ws->ncells_max = ncells_max;
  const int64_t n1 = n_max > 0 ? n_max : 1;
  ws->max_sort_tiles = (n1 + SORT_TILE - 1) / SORT_TILE;
  ws->max_scan_tiles = (2 * ncells_max + 1 + SCAN_TILE - 1) / SCAN_TILE;  // + an X slab's dead bin
  size_t bytes = 0;
  auto alloc = [&](void** p, size_t b) -> cudaError_t {
    bytes += b;
    return cudaMalloc(p, b);
  };
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = alloc((void**)&ws->cnt, sizeof(uint32_t) * (2 * ncells_max + 1));
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = alloc((void**)&ws->keys_tmp[k], sizeof(uint32_t) * n1);
    if (e == cudaSuccess) e = alloc((void**)&ws->vals_tmp[k], sizeof(int32_t) * n1);
  }
  if (e == cudaSuccess)
    e = alloc((void**)&ws->radix_hist, sizeof(uint32_t) * RADIX * ws->max_sort_tiles);
  if (e == cudaSuccess) e = alloc((void**)&ws->digit_total, sizeof(uint32_t) * RADIX);
  if (e == cudaSuccess)
    e = alloc((void**)&ws->scan_partials, sizeof(uint32_t) * (ws->max_scan_tiles + 1));
  // a block never spans two cell rows and holds >= 1 target: #blocks <= n/BT + n
  ws->max_blocks = n1 + n1 / 64 + 16;
  if (e == cudaSuccess) e = alloc((void**)&ws->blocks, 2 * sizeof(int4) * ws->max_blocks);
  if (e == cudaSuccess) e = alloc((void**)&ws->row_off, sizeof(int32_t) * (ncells_max + 1));
  if (e == cudaSuccess) e = alloc((void**)&ws->energy_part, sizeof(double) * 5 * 592);
  if (e == cudaSuccess) e = alloc((void**)&ws->sym_scratch, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(ws->sym_scratch, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = alloc((void**)&ws->cand_acc, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(ws->cand_acc, 0, sizeof(unsigned long long));
  {
    const int64_t words = (n1 + MV_TILE_ROWS - 1) / MV_TILE_ROWS * (MV_TILE_ROWS / 32);
    ws->mover_cap_max = n1 < MOVER_CAP_MAX ? n1 : MOVER_CAP_MAX;
    ws->mover_cap = ws->mover_cap_max;
    const size_t mc = (size_t)ws->mover_cap_max;
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_state, sizeof(uint32_t) * 8);
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_bits, sizeof(uint32_t) * words);
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_wpre, sizeof(uint32_t) * words);
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_tile, sizeof(uint32_t) * (words / 32 + 1));
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_pos, sizeof(int32_t) * mc);
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_next, sizeof(int32_t) * mc);
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_head, sizeof(int32_t) * (2 * ncells_max + 1));
    if (e == cudaSuccess) e = alloc((void**)&ws->mv_kv, sizeof(int4) * (2 * ncells_max + 1));
    if (e == cudaSuccess) e = cudaMemset(ws->mv_state, 0, sizeof(uint32_t) * 8);
    if (e == cudaSuccess) e = cudaMemset(ws->mv_head, 0xff, sizeof(int32_t) * (2 * ncells_max + 1));
  }
  if (e == cudaSuccess) e = cudaMemset(ws->cnt, 0, sizeof(uint32_t) * (2 * ncells_max + 1));
  if (e == cudaSuccess) {  // the interaction plan's side stream (highest priority) and events
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&ws->side, cudaStreamNonBlocking, hi);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_plan, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  ws->bytes = bytes;
  if (e != cudaSuccess) {
    sphb_workspace_destroy(ws);
    return sphb_set_error(SPHB_E_CUDA, "workspace allocation: %s", cudaGetErrorString(e));
  }
  *out = ws;
  return SPHB_OK;
}

int sphb_workspace_destroy(sphb_workspace_t* ws) {
  if (!ws) return SPHB_OK;
  cudaFree(ws->cnt);
  cudaFree(ws->sym_scratch);
  cudaFree(ws->cand_acc);
  cudaFree(ws->row_off);
  for (int k = 0; k < 2; ++k) {
    cudaFree(ws->keys_tmp[k]);
    cudaFree(ws->vals_tmp[k]);
  }
  cudaFree(ws->radix_hist);
  cudaFree(ws->digit_total);
  cudaFree(ws->scan_partials);
  cudaFree(ws->blocks);
  cudaFree(ws->energy_part);
  if (ws->side) cudaStreamDestroy(ws->side);
  if (ws->ev_fork) cudaEventDestroy(ws->ev_fork);
  if (ws->ev_plan) cudaEventDestroy(ws->ev_plan);
  for (void* p : {(void*)ws->mv_state, (void*)ws->mv_bits, (void*)ws->mv_wpre, (void*)ws->mv_tile,
                  (void*)ws->mv_pos, (void*)ws->mv_next, (void*)ws->mv_head, (void*)ws->mv_kv})
    cudaFree(p);
  delete ws;
  return SPHB_OK;
}

int sphb_workspace_reset(sphb_workspace_t* ws, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  ws->plan.valid = false;  // a pending interaction plan is dropped, with its candidate count
  if (ws->side) SPHB_CUDA(cudaStreamSynchronize(ws->side));
  SPHB_CUDA(cudaMemsetAsync(ws->cand_acc, 0, sizeof(unsigned long long), (cudaStream_t)s));
  SPHB_CUDA(cudaMemsetAsync(ws->cnt, 0, sizeof(uint32_t) * (2 * ws->ncells_max + 1), (cudaStream_t)s));
  SPHB_CUDA(cudaMemsetAsync(ws->mv_state, 0, sizeof(uint32_t) * 8, (cudaStream_t)s));
  SPHB_CUDA(cudaMemsetAsync(ws->mv_head, 0xff, sizeof(int32_t) * (2 * ws->ncells_max + 1), (cudaStream_t)s));
  return SPHB_OK;
}

int sphb_workspace_clear_hist(sphb_workspace_t* ws, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_CUDA(cudaMemsetAsync(ws->cnt, 0, sizeof(uint32_t) * (2 * ws->ncells_max + 1), (cudaStream_t)s));
  return SPHB_OK;
}

int sphb_workspace_trust_order(sphb_workspace_t* ws, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  // state words 0 (order established) = 1, 1 (inconsistency seen) = 0 (little endian)
  SPHB_CUDA(cudaMemsetAsync(ws->mv_state, 0, 2 * sizeof(uint32_t), (cudaStream_t)s));
  SPHB_CUDA(cudaMemsetAsync(ws->mv_state, 1, 1, (cudaStream_t)s));
  return SPHB_OK;
}

int sphb_workspace_set_mover_cap(sphb_workspace_t* ws, int64_t cap) {
  SPHB_NONNULL(ws);
  if (cap < -1 || cap > ws->mover_cap_max)
    return sphb_set_error(SPHB_E_INVALID, "mover cap must lie in [-1, %lld]",
                          (long long)ws->mover_cap_max);
  ws->mover_cap = cap;
  return SPHB_OK;
}

int sphb_workspace_set_pi_block(sphb_workspace_t* ws, int32_t targets) {
  SPHB_NONNULL(ws);
  if (targets != 128 && targets != 256 && targets != PI_LARGE_BLOCK && targets != 512)
    return sphb_set_error(SPHB_E_INVALID, "interaction block must be 128, 256, %d or 512 targets",
                          PI_LARGE_BLOCK);
  ws->pi_block = targets;
  return SPHB_OK;
}

int sphb_workspace_set_pi_kernel(sphb_workspace_t* ws, int32_t kernel) {
  SPHB_NONNULL(ws);
  if (kernel != SPHB_PI_GATHER && kernel != SPHB_PI_SYMMETRIC && kernel != SPHB_PI_PAIRED)
    return sphb_set_error(SPHB_E_INVALID,
                          "interaction kernel must be SPHB_PI_GATHER, SPHB_PI_SYMMETRIC or SPHB_PI_PAIRED");
  ws->pi_kernel = kernel;
  return SPHB_OK;
}

int sphb_workspace_sort_info(const sphb_workspace_t* ws, int64_t* movers, int32_t* mode) {
  SPHB_NONNULL(ws);
  uint32_t st[4];
  SPHB_CUDA(cudaMemcpy(st, ws->mv_state, sizeof(st), cudaMemcpyDeviceToHost));
  if (movers) *movers = st[3];
  if (mode) *mode = (int32_t)st[2];
  return SPHB_OK;
}

int64_t sphb_workspace_bytes(const sphb_workspace_t* ws) { return ws ? (int64_t)ws->bytes : 0; }

int sphb_ctrl_init(sphb_ctrl_t* ctrl, int64_t max_steps, double t_end, sphb_stream_t s) {
  SPHB_NONNULL(ctrl);
  return launch_ctrl_init(ctrl, max_steps, t_end, (cudaStream_t)s);
}

int sphb_cell_keys(sphb_workspace_t* ws, const sphb_grid_t* grid, const void* posp, int64_t n,
                   int64_t nb, uint32_t* keys_out, int32_t* cell_out, sphb_ctrl_t* ctrl,
                   sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0) {
    SPHB_NONNULL(posp);
    SPHB_NONNULL(keys_out);
  }
  return launch_cell_keys(ws, *grid, (const float4*)posp, n, nb, keys_out, cell_out, ctrl,
                          (cudaStream_t)s);
}

int sphb_sort(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys, int64_t n,
              uint32_t* keys_sorted_out, int32_t* perm_out, const sphb_ctrl_t* ctrl,
              sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (n > 0) {
    SPHB_NONNULL(keys);
    SPHB_NONNULL(perm_out);
  }
  return launch_sort(ws, *grid, keys, n, keys_sorted_out, perm_out, ctrl, (cudaStream_t)s);
}

int sphb_sort_ranges(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys,
                     int64_t n, uint32_t* keys_sorted, int32_t* perm, int32_t* beg, int32_t* end,
                     const sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(ctrl);
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  if (n < 0) return sphb_set_error(SPHB_E_INVALID, "n < 0");
  if (n > 0) {
    SPHB_NONNULL(keys); SPHB_NONNULL(keys_sorted); SPHB_NONNULL(perm);
  }
  return launch_sort_and_ranges(ws, *grid, keys, n, keys_sorted, perm, beg, end, ctrl,
                                (cudaStream_t)s);
}

int sphb_reorder(const sphb_params_t* prm, const sphb_grid_t* grid, int64_t n,
                 const int32_t* perm, const uint32_t* keys_sorted, const void* posp_in,
                 const void* velr_in, const void* prev_in, const int64_t* id_in, void* posp_out,
                 void* velr_out, void* prev_out, int64_t* id_out, void* aux_out,
                 int32_t* cell_out, const sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(prm);
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (n > 0) {
    SPHB_NONNULL(posp_in);
    SPHB_NONNULL(velr_in);
    SPHB_NONNULL(posp_out);
    SPHB_NONNULL(velr_out);
  }
  return launch_reorder(*prm, *grid, n, perm, keys_sorted, (const float4*)posp_in,
                        (const float4*)velr_in, (const float4*)prev_in, id_in, (float4*)posp_out,
                        (float4*)velr_out, (float4*)prev_out, id_out, (float4*)aux_out, cell_out,
                        ctrl, (cudaStream_t)s);
}

int sphb_nl_build(sphb_workspace_t* ws, const sphb_grid_t* grid, const void* posp, int64_t n,
                  int64_t nb, uint32_t* keys_out, uint32_t* keys_sorted_out, int32_t* perm_out,
                  int32_t* beg, int32_t* end, sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(ctrl);
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0) {
    SPHB_NONNULL(posp); SPHB_NONNULL(keys_out); SPHB_NONNULL(keys_sorted_out);
    SPHB_NONNULL(perm_out);
  }
  cudaStream_t cs = (cudaStream_t)s;
  int rc;
  if ((rc = launch_cell_keys(ws, *grid, (const float4*)posp, n, nb, keys_out, nullptr, ctrl, cs)))
    return rc;
  if ((rc = launch_sort(ws, *grid, keys_out, n, keys_sorted_out, perm_out, ctrl, cs))) return rc;
  return launch_cell_ranges(ws, *grid, beg, end, ctrl, cs);
}

int sphb_cell_hist(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys, int64_t n,
                   const sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0) return sphb_set_error(SPHB_E_INVALID, "n < 0");
  if (n > 0) SPHB_NONNULL(keys);
  return launch_cell_hist(ws, *grid, keys, n, ctrl, (cudaStream_t)s);
}

int sphb_cell_ranges(sphb_workspace_t* ws, const sphb_grid_t* grid, int32_t* beg, int32_t* end,
                     const sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  if (int rc = check_grid(grid)) return rc;
  return launch_cell_ranges(ws, *grid, beg, end, ctrl, (cudaStream_t)s);
}

int sphb_cell_ranges_from_sorted(sphb_workspace_t* ws, const sphb_grid_t* grid,
                                 const int32_t* cell_sorted, int64_t n, int64_t nb, int32_t* beg,
                                 int32_t* end, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (int rc = sphb_workspace_reset(ws, s)) return rc;
  if (n > 0) {
    SPHB_NONNULL(cell_sorted);
    if (int rc = launch_hist_from_sorted(ws, *grid, cell_sorted, n, nb, (cudaStream_t)s)) return rc;
  }
  return launch_cell_ranges(ws, *grid, beg, end, nullptr, (cudaStream_t)s);
}

int sphb_interact_plan(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                       const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  return plan_interact_async(ws, *prm, *grid, beg, end, ctrl, (cudaStream_t)s);
}

int sphb_interact(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                  int64_t n, int64_t nb,
                  const void* posp, const void* velr, const void* aux, const int32_t* cell_sorted,
                  const int32_t* beg, const int32_t* end, void* acc, void* drho, void* visc,
                  sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > ws->n_max) return sphb_set_error(SPHB_E_CAPACITY, "n exceeds workspace");
  if (prm->precision != SPHB_FP32 && prm->precision != SPHB_FP64)
    return sphb_set_error(SPHB_E_INVALID, "precision must be SPHB_FP32 or SPHB_FP64");
  if (n == 0) return SPHB_OK;
  SPHB_NONNULL(posp);
  SPHB_NONNULL(velr);
  // aux (derived rows) may be NULL for the FP32 gather / paired builds: they recompute a
  // target's own values; the FP64 kernel and the symmetric build read them
  if (prm->precision == SPHB_FP64 || ws->pi_kernel == SPHB_PI_SYMMETRIC) SPHB_NONNULL(aux);
  SPHB_NONNULL(cell_sorted);
  SPHB_NONNULL(beg);
  SPHB_NONNULL(end);
  SPHB_NONNULL(acc);
  if (prm->precision == SPHB_FP64) SPHB_NONNULL(drho);  /* FP32: drho travels in acc.w */
  SPHB_NONNULL(visc);
  return launch_interact(ws, *prm, *grid, n, nb, (const float4*)posp, (const float4*)velr,
                         (const float4*)aux, cell_sorted, beg, end, acc, drho, visc, ctrl,
                         (cudaStream_t)s);
}

int sphb_step_begin(sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ctrl);
  return launch_step_begin(ctrl, (cudaStream_t)s);
}

int sphb_integrate(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                   int64_t n, int64_t nb, const void* posp_s, const void* velr_s,
                   const void* prev_s, const int64_t* id_s, const void* acc, const void* drho,
                   void* posp, void* velr, void* prev, int64_t* id, uint32_t* keys_next,
                   sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0) {
    SPHB_NONNULL(posp_s); SPHB_NONNULL(velr_s); SPHB_NONNULL(prev_s); SPHB_NONNULL(id_s);
    SPHB_NONNULL(acc); if (prm->precision == SPHB_FP64) SPHB_NONNULL(drho);
    SPHB_NONNULL(posp); SPHB_NONNULL(velr);
    SPHB_NONNULL(prev); SPHB_NONNULL(id); SPHB_NONNULL(keys_next);
  }
  return launch_integrate(ws, *prm, *grid, n, nb, (const float4*)posp_s, (const float4*)velr_s,
                          (const float4*)prev_s, id_s, acc, drho, (float4*)posp, (float4*)velr,
                          (float4*)prev, id, keys_next, ctrl, (cudaStream_t)s);
}

int sphb_step_end(sphb_ctrl_t* ctrl, const sphb_params_t* prm, sphb_step_record_t* rec,
                  int64_t rec_capacity, sphb_stream_t s) {
  SPHB_NONNULL(ctrl);
  SPHB_NONNULL(prm);
  return launch_step_end(ctrl, *prm, rec, rec_capacity, (cudaStream_t)s);
}

int sphb_integrate_stage(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                         int64_t n, int64_t nb, int32_t stage, const void* posp_s,
                         const void* velr_s, const void* prev_s, const int64_t* id_s,
                         const void* acc, const void* drho, void* posp, void* velr,
                         void* prev, int64_t* id, uint32_t* keys_next, sphb_ctrl_t* ctrl,
                         sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  if (stage != 0 && stage != 1) return sphb_set_error(SPHB_E_INVALID, "stage must be 0 or 1");
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0) {
    SPHB_NONNULL(posp_s); SPHB_NONNULL(velr_s); SPHB_NONNULL(prev_s); SPHB_NONNULL(id_s);
    SPHB_NONNULL(acc); if (prm->precision == SPHB_FP64) SPHB_NONNULL(drho);
    SPHB_NONNULL(posp); SPHB_NONNULL(velr);
    SPHB_NONNULL(prev); SPHB_NONNULL(id); SPHB_NONNULL(keys_next);
  }
  return launch_integrate_mode(ws, *prm, *grid, n, nb, 1 + stage, (const float4*)posp_s,
                               (const float4*)velr_s, (const float4*)prev_s, id_s, acc, drho,
                               (float4*)posp, (float4*)velr, (float4*)prev, id, keys_next, ctrl,
                               (cudaStream_t)s);
}

int sphb_energy(sphb_workspace_t* ws, const sphb_params_t* prm, int64_t n, int64_t nb,
                const void* posp, const void* velr, double* out, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  SPHB_NONNULL(prm);
  SPHB_NONNULL(out);
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (n > 0) {
    SPHB_NONNULL(posp);
    SPHB_NONNULL(velr);
  }
  return launch_energy(ws, *prm, n, nb, (const float4*)posp, (const float4*)velr, out,
                       (cudaStream_t)s);
}

// NL -> PI on the primary state, then the system update of `mode` (0 verlet, 1/2 symplectic
// predictor/corrector)
static int stage_pass(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                      int64_t n, int64_t nb, const sphb_state_t* st, sphb_ctrl_t* ctrl, int mode,
                      cudaStream_t cs) {
  int rc;
  // the FP32 gather / paired kernels need no aux rows (16 B per particle less to write)
  float4* aux = (prm->precision == SPHB_FP32 && ws->pi_kernel != SPHB_PI_SYMMETRIC)
                    ? nullptr : (float4*)st->aux;
  {
    NvtxRange r("sphb NL");  // stage ranges (the reference's perf_counter stages, sim.py:306-348)
    if ((rc = launch_sort_and_ranges(ws, *grid, st->keys, n, st->keys_sorted, st->perm, st->beg,
                                     st->end, ctrl, cs)))
      return rc;
    // the interaction's block list on the side stream, concurrently with K3
    if ((rc = plan_interact_async(ws, *prm, *grid, st->beg, st->end, ctrl, cs))) return rc;
    if ((rc = launch_reorder(*prm, *grid, n, st->perm, st->keys_sorted, (const float4*)st->posp,
                             (const float4*)st->velr, (const float4*)st->prev, st->id,
                             (float4*)st->posp_s, (float4*)st->velr_s, (float4*)st->prev_s, st->id_s,
                             aux, st->cell_s, ctrl, cs)))
      return rc;
  }
  {
    NvtxRange r("sphb PI");
    if ((rc = launch_interact(ws, *prm, *grid, n, nb, (const float4*)st->posp_s,
                              (const float4*)st->velr_s, aux, st->cell_s, st->beg,
                              st->end, st->acc, st->drho, st->visc, ctrl, cs)))
      return rc;
  }
  NvtxRange r("sphb SU");
  return launch_integrate_mode(ws, *prm, *grid, n, nb, mode, (const float4*)st->posp_s,
                               (const float4*)st->velr_s, (const float4*)st->prev_s, st->id_s,
                               st->acc, st->drho, (float4*)st->posp, (float4*)st->velr,
                               (float4*)st->prev, st->id, st->keys, ctrl, cs);
}

int sphb_step(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid, int64_t n,
              int64_t nb, const sphb_state_t* st, sphb_ctrl_t* ctrl, sphb_step_record_t* rec,
              int64_t rec_capacity, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  SPHB_NONNULL(st);
  SPHB_NONNULL(ctrl);
  if (int rc = check_grid(grid)) return rc;
  cudaStream_t cs = (cudaStream_t)s;
  int rc;
  if ((rc = launch_step_begin(ctrl, cs))) return rc;
  if (prm->integrator == SPHB_INT_SYMPLECTIC) {
    if ((rc = stage_pass(ws, prm, grid, n, nb, st, ctrl, 1, cs))) return rc;
    if ((rc = stage_pass(ws, prm, grid, n, nb, st, ctrl, 2, cs))) return rc;
  } else {
    if ((rc = stage_pass(ws, prm, grid, n, nb, st, ctrl, 0, cs))) return rc;
  }
  return launch_step_end(ctrl, *prm, rec, rec_capacity, cs);
}

int64_t sphb_slab_tiles(int64_t n) { return n > 0 ? slab_tiles(n) : 0; }

int sphb_slab_count(const sphb_grid_t* grid, int64_t n, int64_t nb, const uint32_t* keys,
                    const int64_t* id, int32_t x0, int32_t x1, uint32_t* tile_counts,
                    uint32_t* totals, sphb_stream_t s) {
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(totals);
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (x0 < 0 || x1 > grid->dims[0] || x0 >= x1)
    return sphb_set_error(SPHB_E_INVALID, "slab columns [x0, x1) must lie in [0, dims[0])");
  if (n > 0) {
    SPHB_NONNULL(keys); SPHB_NONNULL(id); SPHB_NONNULL(tile_counts);
  }
  return launch_slab_count(*grid, n, nb, keys, id, x0, x1, tile_counts, totals, (cudaStream_t)s);
}

int sphb_slab_scatter(const sphb_grid_t* grid, int64_t n, int64_t nb, const uint32_t* keys,
                      const int64_t* id, int32_t x0, int32_t x1, const uint32_t* tile_offsets,
                      const void* posp, const void* velr, const void* prev,
                      const int64_t* keep_bases, void* nposp, void* nvelr, void* nprev,
                      int64_t* nid, uint32_t* nkeys, void* send_l, void* send_r,
                      const int64_t* sections, sphb_stream_t s) {
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(keep_bases);
  SPHB_NONNULL(sections);
  if (n < 0 || nb < 0 || nb > n) return sphb_set_error(SPHB_E_INVALID, "bad n/nb");
  if (x0 < 0 || x1 > grid->dims[0] || x0 >= x1)
    return sphb_set_error(SPHB_E_INVALID, "slab columns [x0, x1) must lie in [0, dims[0])");
  if (n > 0) {
    SPHB_NONNULL(keys); SPHB_NONNULL(id); SPHB_NONNULL(tile_offsets); SPHB_NONNULL(posp);
    SPHB_NONNULL(velr); SPHB_NONNULL(prev); SPHB_NONNULL(nposp); SPHB_NONNULL(nvelr);
    SPHB_NONNULL(nprev); SPHB_NONNULL(nid);
  }
  return launch_slab_scatter(*grid, n, nb, keys, id, x0, x1, tile_offsets, (const float4*)posp,
                             (const float4*)velr, (const float4*)prev, keep_bases, (float4*)nposp,
                             (float4*)nvelr, (float4*)nprev, nid, nkeys, send_l, send_r,
                             sections, (cudaStream_t)s);
}

int sphb_slab_unpack(const void* buf, int64_t r0, int64_t cnt, int64_t dst, void* nposp,
                     void* nvelr, void* nprev, int64_t* nid, uint32_t* nkeys, sphb_stream_t s) {
  if (cnt < 0 || r0 < 0 || dst < 0) return sphb_set_error(SPHB_E_INVALID, "bad unpack range");
  if (cnt > 0) {
    SPHB_NONNULL(buf); SPHB_NONNULL(nposp); SPHB_NONNULL(nvelr); SPHB_NONNULL(nprev);
    SPHB_NONNULL(nid);
  }
  return launch_slab_unpack(buf, r0, cnt, dst, (float4*)nposp, (float4*)nvelr, (float4*)nprev, nid,
                            nkeys, (cudaStream_t)s);
}

int64_t sphb_band_scratch_words(const sphb_grid_t* grid) {
  if (!grid || check_grid(grid)) return 0;
  return band_scratch_words(*grid);
}

static int check_band(const sphb_grid_t* grid, int32_t width, int32_t sides) {
  if (int rc = check_grid(grid)) return rc;
  if (width < 1) return sphb_set_error(SPHB_E_INVALID, "band width must be >= 1");
  if (sides < 0 || sides > 3) return sphb_set_error(SPHB_E_INVALID, "sides must be a 2-bit mask");
  return SPHB_OK;
}

int sphb_band_count(const sphb_grid_t* grid, int32_t width, int32_t sides, const int32_t* beg,
                    const int32_t* end, int32_t* scratch, int64_t* info, const sphb_ctrl_t* ctrl,
                    sphb_stream_t s) {
  if (int rc = check_band(grid, width, sides)) return rc;
  SPHB_NONNULL(beg); SPHB_NONNULL(end); SPHB_NONNULL(scratch); SPHB_NONNULL(info);
  SPHB_NONNULL(ctrl);
  return launch_band_count(*grid, width, sides, beg, end, scratch, info, ctrl, (cudaStream_t)s);
}

int sphb_band_pack(const sphb_params_t* prm, const sphb_grid_t* grid, int32_t width,
                   int32_t sides, const int32_t* beg, const int32_t* end, const int32_t* scratch,
                   const void* posp_s, const void* velr_s, const void* prev_s,
                   const int64_t* id_s, const void* acc, const void* drho, void* send_l,
                   void* send_r, sphb_stream_t s) {
  if (int rc = check_params(prm)) return rc;
  if (int rc = check_band(grid, width, sides)) return rc;
  SPHB_NONNULL(beg); SPHB_NONNULL(end); SPHB_NONNULL(scratch);
  SPHB_NONNULL(posp_s); SPHB_NONNULL(velr_s); SPHB_NONNULL(prev_s); SPHB_NONNULL(id_s);
  SPHB_NONNULL(acc);
  if (prm->precision == SPHB_FP64) SPHB_NONNULL(drho);
  if (sides & 1) SPHB_NONNULL(send_l);
  if (sides & 2) SPHB_NONNULL(send_r);
  return launch_band_pack(*prm, *grid, width, sides, beg, end, scratch, (const float4*)posp_s,
                          (const float4*)velr_s, (const float4*)prev_s, id_s, acc, drho, send_l,
                          send_r, (cudaStream_t)s);
}

int sphb_band_integrate(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                        const void* buf, int64_t cnt, int64_t dst, void* posp, void* velr,
                        void* prev, int64_t* id, uint32_t* keys_next, uint32_t* keys_sorted,
                        sphb_ctrl_t* ctrl, sphb_stream_t s) {
  SPHB_NONNULL(ws);
  if (int rc = check_params(prm)) return rc;
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(ctrl);
  if (cnt < 0 || dst < 0) return sphb_set_error(SPHB_E_INVALID, "bad cnt/dst");
  if (dst + cnt > ws->n_max) return sphb_set_error(SPHB_E_CAPACITY, "band rows exceed the workspace");
  if (prm->integrator != SPHB_INT_VERLET)
    return sphb_set_error(SPHB_E_INVALID, "X-slab bands integrate with the Verlet scheme only");
  if (cnt == 0) return SPHB_OK;
  SPHB_NONNULL(buf); SPHB_NONNULL(posp); SPHB_NONNULL(velr); SPHB_NONNULL(prev);
  SPHB_NONNULL(id); SPHB_NONNULL(keys_next); SPHB_NONNULL(keys_sorted);
  return launch_band_integrate(ws, *prm, *grid, buf, cnt, dst, (float4*)posp, (float4*)velr,
                               (float4*)prev, id, keys_next, keys_sorted, ctrl, (cudaStream_t)s);
}

int sphb_band_put(const sphb_params_t* prm, const sphb_grid_t* grid, int32_t width, int32_t sides,
                  const int32_t* beg, const int32_t* end, const int32_t* scratch,
                  const void* posp_s, const void* velr_s, const void* prev_s, const int64_t* id_s,
                  const void* acc, const void* drho, void* peer_l, void* peer_r,
                  uint64_t* peer_flag_l, uint64_t* peer_flag_r, uint64_t tag, uint32_t* done,
                  sphb_stream_t s) {
  if (int rc = check_params(prm)) return rc;
  if (int rc = check_band(grid, width, sides)) return rc;
  SPHB_NONNULL(beg); SPHB_NONNULL(end); SPHB_NONNULL(scratch); SPHB_NONNULL(done);
  SPHB_NONNULL(posp_s); SPHB_NONNULL(velr_s); SPHB_NONNULL(prev_s); SPHB_NONNULL(id_s);
  SPHB_NONNULL(acc);
  if (prm->precision == SPHB_FP64) SPHB_NONNULL(drho);
  if (sides & 1) { SPHB_NONNULL(peer_l); SPHB_NONNULL(peer_flag_l); }
  if (sides & 2) { SPHB_NONNULL(peer_r); SPHB_NONNULL(peer_flag_r); }
  return launch_band_put(*prm, *grid, width, sides, beg, end, scratch, (const float4*)posp_s,
                         (const float4*)velr_s, (const float4*)prev_s, id_s, acc, drho, peer_l,
                         peer_r, (sides & 1) ? peer_flag_l : nullptr, (sides & 2) ? peer_flag_r : nullptr,
                         tag, done, (cudaStream_t)s);
}

int sphb_band_wait(const uint64_t* flag_l, const uint64_t* flag_r, uint64_t tag, sphb_ctrl_t* ctrl,
                   sphb_stream_t s) {
  SPHB_NONNULL(ctrl);
  return launch_band_wait(flag_l, flag_r, tag, ctrl, (cudaStream_t)s);
}

int sphb_slab_tail(const sphb_grid_t* grid, int32_t* end, int64_t n_next, sphb_stream_t s) {
  if (int rc = check_grid(grid)) return rc;
  SPHB_NONNULL(end);
  if (n_next < 0 || n_next >= (int64_t(1) << 31)) return sphb_set_error(SPHB_E_INVALID, "bad n_next");
  return launch_slab_tail(*grid, end, n_next, (cudaStream_t)s);
}

int sphb_state_from_soa(int64_t r0, int64_t cnt, const float* pos, const float* vel,
                        const float* rho, const float* vel_prev, const float* rho_prev,
                        void* posp, void* velr, void* prev, sphb_stream_t s) {
  if (r0 < 0 || cnt < 0) return sphb_set_error(SPHB_E_INVALID, "bad row range");
  if (cnt > 0) {
    SPHB_NONNULL(pos); SPHB_NONNULL(vel); SPHB_NONNULL(rho); SPHB_NONNULL(vel_prev);
    SPHB_NONNULL(rho_prev); SPHB_NONNULL(posp); SPHB_NONNULL(velr); SPHB_NONNULL(prev);
  }
  return launch_state_unpack(r0, cnt, pos, vel, rho, vel_prev, rho_prev, (float4*)posp,
                             (float4*)velr, (float4*)prev, (cudaStream_t)s);
}

int sphb_state_to_soa(int64_t r0, int64_t cnt, const void* posp, const void* velr,
                      const void* prev, float* pos, float* vel, float* rho, float* vel_prev,
                      float* rho_prev, sphb_stream_t s) {
  if (r0 < 0 || cnt < 0) return sphb_set_error(SPHB_E_INVALID, "bad row range");
  if (cnt > 0) {
    SPHB_NONNULL(pos); SPHB_NONNULL(vel); SPHB_NONNULL(rho); SPHB_NONNULL(vel_prev);
    SPHB_NONNULL(rho_prev); SPHB_NONNULL(posp); SPHB_NONNULL(velr); SPHB_NONNULL(prev);
  }
  return launch_state_pack(r0, cnt, (const float4*)posp, (const float4*)velr,
                           (const float4*)prev, pos, vel, rho, vel_prev, rho_prev,
                           (cudaStream_t)s);
}

int64_t sphb_step_launch_count(const sphb_grid_t* grid, int64_t n) {
  if (!grid) return 0;
  return 1 /*begin*/ + nl_launch_count(*grid, n) + interact_launch_count(n) + 1 /*integrate*/ +
         1 /*end*/ + (n >= PLAN_ASYNC_MIN_ROWS ? 1 : 0) /*k_cand_take after a side-stream plan*/;  // (a symplectic step runs the middle three twice, plus k_stage_mid)
}

}  // extern "C"
