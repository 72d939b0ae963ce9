// nl.cu -- neighbour-list stage (NL) of the SPH step on sm_100a.
//
//   K1 k_cell_keys        assign_cells (grid.py:77-93) + per-list per-cell histogram
//   K2 k_radix_*          the stable per-list argsort of reorder (grid.py:96-109), LSD radix
//   K3 k_reorder          reorder gathers (grid.py:111-114) fused with compute_derived
//                         (physics.py:96-110): press into posp.w, (prrho, cs, tensil) into aux
//   K4 k_scan_*           build_cell_begin_end / build_cell_index (grid.py:123-144) as a
//                         warp-shuffle exclusive scan of the K1 histogram
//
// All kernels are HBM-bound integer/byte work: coalesced float4 SoA accesses, warp-
// aggregated shared/global atomics (sorted input means long runs of equal keys),
// no tensor cores.
#include <climits>

#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

__device__ __forceinline__ bool step_live(const sphb_ctrl_t* c) {
  // abort once an error is recorded for this or an earlier step (see sphb_ctrl_t.err)
  return c->active && c->err >= ((uint64_t)(c->step + 1) << 40);
}

inline int grid_for(int64_t work, int block, int cap = 148 * 32) {
  int64_t b = (work + block - 1) / block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// ------------------------------------------------------------------ K1
__global__ void __launch_bounds__(256) k_cell_keys(sphb_grid_t g, const float4* __restrict__ posp,
                                                   int64_t n, int64_t nb, int cellbits,
                                                   uint32_t* __restrict__ keys,
                                                   int32_t* __restrict__ cell_out,
                                                   uint32_t* __restrict__ cnt, int64_t ncells,
                                                   sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  const int64_t step = ctrl->step;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    int64_t i = base + threadIdx.x;
    bool valid = i < n;
    int32_t c = -2;
    if (valid) {
      float4 p = posp[i];
      c = cell_of(p.x, p.y, p.z, g);
      if (c < 0) raise_div(ctrl, step, SPHB_DIV_LEFT_DOMAIN, (uint64_t)i);
      uint32_t list = i >= nb ? 1u : 0u;
      keys[i] = c >= 0 ? ((list << cellbits) | (uint32_t)c) : 0xffffffffu;
      if (cell_out) cell_out[i] = c;
    }
    int64_t slot = (valid && c >= 0) ? (i >= nb ? ncells : 0) + c : -1;
    uint32_t peers = __match_any_sync(SPHB_FULL, (unsigned long long)slot);
    if (slot >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[slot], (uint32_t)__popc(peers));
  }
}

__global__ void __launch_bounds__(256) k_hist_sorted(const int32_t* __restrict__ cell, int64_t n,
                                                     int64_t nb, uint32_t* __restrict__ cnt,
                                                     int64_t ncells) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    int64_t i = base + threadIdx.x;
    int64_t slot = -1;
    if (i < n && cell[i] >= 0) slot = (i >= nb ? ncells : 0) + cell[i];
    uint32_t peers = __match_any_sync(SPHB_FULL, (unsigned long long)slot);
    if (slot >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[slot], (uint32_t)__popc(peers));
  }
}

// ------------------------------------------------------------------ block scan helper
template <int BLOCK>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total,
                                                         uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(SPHB_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NW ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(SPHB_FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  uint32_t warp_excl = warp > 0 ? s_warp[warp - 1] : 0;
  *total = s_warp[NW - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// ------------------------------------------------------------------ K2 radix sort
__global__ void __launch_bounds__(SORT_BLOCK) k_radix_hist(const uint32_t* __restrict__ keys,
                                                           int64_t n, int shift,
                                                           uint32_t* __restrict__ hist,
                                                           int64_t ntiles,
                                                           const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  __shared__ uint32_t s[RADIX];
  for (int d = threadIdx.x; d < RADIX; d += SORT_BLOCK) s[d] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t tile0 = (int64_t)blockIdx.x * SORT_TILE;
#pragma unroll 4
  for (int r = 0; r < SORT_ITEMS; ++r) {
    int64_t idx = tile0 + r * SORT_BLOCK + threadIdx.x;
    uint32_t d = idx < n ? (keys[idx] >> shift) & (RADIX - 1) : RADIX;
    uint32_t peers = __match_any_sync(SPHB_FULL, d);
    if (d < RADIX && lane == __ffs(peers) - 1) atomicAdd(&s[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RADIX; d += SORT_BLOCK) hist[(int64_t)d * ntiles + blockIdx.x] = s[d];
}

__global__ void __launch_bounds__(1024) k_radix_rowscan(uint32_t* __restrict__ hist, int64_t ntiles,
                                                        uint32_t* __restrict__ digit_total,
                                                        const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  __shared__ uint32_t s_warp[32];
  uint32_t* row = hist + (int64_t)blockIdx.x * ntiles;
  uint32_t running = 0;
  for (int64_t base = 0; base < ntiles; base += 1024) {
    int64_t k = base + threadIdx.x;
    uint32_t v = k < ntiles ? row[k] : 0;
    uint32_t total;
    uint32_t ex = block_exclusive_scan<1024>(v, &total, s_warp);
    if (k < ntiles) row[k] = running + ex;
    running += total;
  }
  if (threadIdx.x == 0) digit_total[blockIdx.x] = running;
}

// Stable scatter: items are ranked in their original order (round-major, then thread),
// warps rank with __match_any_sync, the block combines warp counts per digit.
__global__ void __launch_bounds__(SORT_BLOCK) k_radix_scatter(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, int64_t n, int shift,
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ digit_total, int64_t ntiles,
    uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out, const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  constexpr int NW = SORT_BLOCK / 32;
  __shared__ uint32_t s_base[RADIX];
  __shared__ uint32_t s_run[RADIX];
  __shared__ uint32_t s_wc[2][NW][RADIX];
  __shared__ uint32_t s_warp[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x;
  // digit base = exclusive scan of digit totals (RADIX == SORT_BLOCK)
  {
    uint32_t v = digit_total[threadIdx.x], total;
    uint32_t ex = block_exclusive_scan<SORT_BLOCK>(v, &total, s_warp);
    s_base[threadIdx.x] = ex + hist[(int64_t)threadIdx.x * ntiles + tile];
    s_run[threadIdx.x] = 0;
    for (int w = 0; w < NW; ++w) s_wc[0][w][threadIdx.x] = 0;
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  const int64_t tile0 = tile * SORT_TILE;
  for (int r = 0; r < SORT_ITEMS; ++r) {
    const int p = r & 1;
    int64_t idx = tile0 + r * SORT_BLOCK + threadIdx.x;
    bool valid = idx < n;
    uint32_t key = valid ? keys_in[idx] : 0u;
    uint32_t d = valid ? (key >> shift) & (RADIX - 1) : RADIX;
    uint32_t peers = __match_any_sync(SPHB_FULL, d);
    uint32_t lrank = __popc(peers & lt);
    if (valid && lane == __ffs(peers) - 1) s_wc[p][warp][d] = __popc(peers);
    __syncthreads();
    {
      uint32_t run = s_run[threadIdx.x];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        uint32_t c = s_wc[p][w][threadIdx.x];
        s_wc[p][w][threadIdx.x] = run;
        run += c;
        s_wc[p ^ 1][w][threadIdx.x] = 0;
      }
      s_run[threadIdx.x] = run;
    }
    __syncthreads();
    if (valid) {
      uint32_t pos = s_base[d] + s_wc[p][warp][d] + lrank;
      keys_out[pos] = key;
      vals_out[pos] = vals_in ? vals_in[idx] : (int32_t)idx;
    }
  }
}

// ------------------------------------------------------------------ K3 reorder + EOS
#ifndef NL_MINB
#define NL_MINB 4  // 64 registers: 2x the resident warps of the default (memory-bound kernel)
#endif
__global__ void __launch_bounds__(256, NL_MINB) k_reorder(
    sphb_params_t p, uint32_t cellmask, int cellbits, int64_t n, const int32_t* __restrict__ perm,
    const uint32_t* __restrict__ keys_sorted, const float4* __restrict__ posp_in,
    const float4* __restrict__ velr_in, const float4* __restrict__ prev_in,
    const int64_t* __restrict__ id_in, float4* __restrict__ posp_out, float4* __restrict__ velr_out,
    float4* __restrict__ prev_out, int64_t* __restrict__ id_out, float4* __restrict__ aux_out,
    int32_t* __restrict__ cell_out, const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int32_t o = perm ? perm[i] : (int32_t)i;
    float4 pp = posp_in[o];
    float4 vr = velr_in[o];
    double rho = (double)vr.w;
    float press = eos_press(rho, p.tait_b, p.rho0, p.gamma);
    Derived d = derive((double)press, rho, p.c0, p.rho0, p.gamma);
    // posp.w = prrho: the interaction stages (x, y, z, prrho) rows with one bulk copy
    pp.w = d.prrho;
    posp_out[i] = pp;
    velr_out[i] = vr;
    const bool boundary = keys_sorted ? ((keys_sorted[i] >> cellbits) & 1u) == 0u : false;
    aux_out[i] = make_float4(press, d.csound, d.tensil,
                             (float)(boundary ? p.mass_boundary : p.mass_fluid));
    if (prev_in && prev_out) prev_out[i] = prev_in[o];
    if (id_in && id_out) id_out[i] = id_in[o];
    if (cell_out && keys_sorted) cell_out[i] = (int32_t)(keys_sorted[i] & cellmask);
  }
}

// ------------------------------------------------------------------ K4 begin/end scan
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_reduce(const uint32_t* __restrict__ cnt,
                                                            int64_t len,
                                                            uint32_t* __restrict__ partials,
                                                            const sphb_ctrl_t* ctrl) {
  if (ctrl && !step_live(ctrl)) return;
  __shared__ uint32_t s_warp[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t v = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k)
    if (base + k < len) v += cnt[base + k];
  uint32_t total;
  block_exclusive_scan<SCAN_BLOCK>(v, &total, s_warp);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_partials(uint32_t* __restrict__ partials,
                                                        int64_t ntiles, const sphb_ctrl_t* ctrl) {
  if (ctrl && !step_live(ctrl)) return;
  __shared__ uint32_t s_warp[32];
  uint32_t running = 0;
  for (int64_t base = 0; base < ntiles; base += 1024) {
    int64_t k = base + threadIdx.x;
    uint32_t v = k < ntiles ? partials[k] : 0;
    uint32_t total;
    uint32_t ex = block_exclusive_scan<1024>(v, &total, s_warp);
    if (k < ntiles) partials[k] = running + ex;
    running += total;
  }
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_apply(uint32_t* __restrict__ cnt, int64_t len,
                                                           const uint32_t* __restrict__ partials,
                                                           int32_t* __restrict__ beg,
                                                           int32_t* __restrict__ end,
                                                           const sphb_ctrl_t* ctrl) {
  if (ctrl && !step_live(ctrl)) return;
  __shared__ uint32_t s_warp[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t c[SCAN_ITEMS];
  uint32_t v = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    c[k] = base + k < len ? cnt[base + k] : 0;
    v += c[k];
  }
  uint32_t total;
  uint32_t ex = block_exclusive_scan<SCAN_BLOCK>(v, &total, s_warp) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < len) {
      beg[base + k] = (int32_t)ex;
      ex += c[k];
      end[base + k] = (int32_t)ex;
      cnt[base + k] = 0;  // self-cleaning for the next step's histogram
    }
  }
}

}  // namespace

// ====================================================================== launchers
int sort_pass_count(const sphb_grid_t& g) {
  int bits = cellbits_of(g) + 1;  // + list bit
  return (bits + RADIX_BITS - 1) / RADIX_BITS;
}

int64_t nl_launch_count(const sphb_grid_t& g, int64_t n) {
  (void)n;
  return 3 * sort_pass_count(g) + 1 /*reorder*/ + 3 /*scan*/;
}

int launch_cell_keys(sphb_workspace* ws, const sphb_grid_t& g, const float4* posp, int64_t n,
                     int64_t nb, uint32_t* keys, int32_t* cell_out, sphb_ctrl_t* ctrl,
                     cudaStream_t s) {
  int64_t nc = ncells_of(g);
  if (n > ws->n_max || nc > ws->ncells_max)
    return sphb_set_error(SPHB_E_CAPACITY, "n=%lld ncells=%lld exceed workspace (%lld, %lld)",
                          (long long)n, (long long)nc, (long long)ws->n_max,
                          (long long)ws->ncells_max);
  if (n == 0) return SPHB_OK;
  k_cell_keys<<<grid_for(n, 256), 256, 0, s>>>(g, posp, n, nb, cellbits_of(g), keys, cell_out,
                                                ws->cnt, nc, ctrl);
  return sphb_check_launch("k_cell_keys");
}

int launch_hist_from_sorted(sphb_workspace* ws, const sphb_grid_t& g, const int32_t* cell_sorted,
                            int64_t n, int64_t nb, cudaStream_t s) {
  int64_t nc = ncells_of(g);
  if (n > ws->n_max || nc > ws->ncells_max)
    return sphb_set_error(SPHB_E_CAPACITY, "n/ncells exceed workspace");
  if (n == 0) return SPHB_OK;
  k_hist_sorted<<<grid_for(n, 256), 256, 0, s>>>(cell_sorted, n, nb, ws->cnt, nc);
  return sphb_check_launch("k_hist_sorted");
}

int launch_sort(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys, int64_t n,
                uint32_t* keys_sorted, int32_t* perm, const sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (n > ws->n_max) return sphb_set_error(SPHB_E_CAPACITY, "n exceeds workspace");
  if (n == 0) return SPHB_OK;
  const int passes = sort_pass_count(g);
  const int64_t ntiles = (n + SORT_TILE - 1) / SORT_TILE;
  const uint32_t* kin = keys;
  const int32_t* vin = nullptr;
  for (int pass = 0; pass < passes; ++pass) {
    const bool last = pass == passes - 1;
    uint32_t* kout = last ? (keys_sorted ? keys_sorted : ws->keys_tmp[pass & 1]) : ws->keys_tmp[pass & 1];
    int32_t* vout = last ? perm : ws->vals_tmp[pass & 1];
    const int shift = pass * RADIX_BITS;
    k_radix_hist<<<(unsigned)ntiles, SORT_BLOCK, 0, s>>>(kin, n, shift, ws->radix_hist, ntiles, ctrl);
    k_radix_rowscan<<<RADIX, 1024, 0, s>>>(ws->radix_hist, ntiles, ws->digit_total, ctrl);
    k_radix_scatter<<<(unsigned)ntiles, SORT_BLOCK, 0, s>>>(kin, vin, n, shift, ws->radix_hist,
                                                            ws->digit_total, ntiles, kout, vout,
                                                            ctrl);
    kin = kout;
    vin = vout;
  }
  return sphb_check_launch("radix sort");
}

int launch_reorder(const sphb_params_t& p, const sphb_grid_t& g, int64_t n, const int32_t* perm,
                   const uint32_t* keys_sorted, const float4* posp_in, const float4* velr_in,
                   const float4* prev_in, const int64_t* id_in, float4* posp_out,
                   float4* velr_out, float4* prev_out, int64_t* id_out, float4* aux_out,
                   int32_t* cell_out, const sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (n == 0) return SPHB_OK;
  uint32_t cellmask = (1u << cellbits_of(g)) - 1u;
  k_reorder<<<grid_for(n, 256), 256, 0, s>>>(p, cellmask, cellbits_of(g), n, perm, keys_sorted, posp_in, velr_in,
                                             prev_in, id_in, posp_out, velr_out, prev_out, id_out,
                                             aux_out, cell_out, ctrl);
  return sphb_check_launch("k_reorder");
}

int launch_cell_ranges(sphb_workspace* ws, const sphb_grid_t& g, int32_t* beg, int32_t* end,
                       const sphb_ctrl_t* ctrl, cudaStream_t s) {
  const int64_t len = 2 * ncells_of(g);
  const int64_t ntiles = (len + SCAN_TILE - 1) / SCAN_TILE;
  if (ntiles > ws->max_scan_tiles) return sphb_set_error(SPHB_E_CAPACITY, "ncells exceeds workspace");
  k_scan_reduce<<<(unsigned)ntiles, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, ctrl);
  k_scan_partials<<<1, 1024, 0, s>>>(ws->scan_partials, ntiles, ctrl);
  k_scan_apply<<<(unsigned)ntiles, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, beg, end,
                                                       ctrl);
  return sphb_check_launch("cell ranges scan");
}
