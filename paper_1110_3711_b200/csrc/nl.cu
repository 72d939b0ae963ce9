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

// per-list per-cell histogram of known sort keys (key = list << cellbits | cell)
__global__ void __launch_bounds__(256) k_hist_keys(const uint32_t* __restrict__ keys, int64_t n,
                                                   int cellbits, int64_t ncells, bool slab,
                                                   uint32_t* __restrict__ cnt,
                                                   const sphb_ctrl_t* ctrl) {
  if (ctrl && !step_live(ctrl)) return;
  const int lane = threadIdx.x & 31;
  const uint32_t cm = (1u << cellbits) - 1u, dead = dead_key(cellbits);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int64_t slot = -1;
    if (i < n) {
      const uint32_t k = keys[i];
      if ((k >> cellbits) <= 1u && (k & cm) < (uint32_t)ncells) slot = (k >> cellbits) * ncells + (k & cm);
      else if (slab && k == dead) slot = 2 * ncells;  // X slab: the dead bin
    }
    const uint32_t peers = __match_any_sync(SPHB_FULL, (unsigned long long)slot);
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
                                                           const sphb_ctrl_t* ctrl,
                                                           const uint32_t* skip) {
  if (!step_live(ctrl) || (skip && *skip == 0u)) return;
  __shared__ uint32_t s[RADIX];
  const int lane = threadIdx.x & 31;
  // persistent over tiles: a skipped pass (movers-only sort ran) costs one small launch
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int d = threadIdx.x; d < RADIX; d += SORT_BLOCK) s[d] = 0;
    __syncthreads();
    const int64_t tile0 = tile * SORT_TILE;
#pragma unroll 4
    for (int r = 0; r < SORT_ITEMS; ++r) {
      int64_t idx = tile0 + r * SORT_BLOCK + threadIdx.x;
      uint32_t d = idx < n ? (keys[idx] >> shift) & (RADIX - 1) : RADIX;
      uint32_t peers = __match_any_sync(SPHB_FULL, d);
      if (d < RADIX && lane == __ffs(peers) - 1) atomicAdd(&s[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += SORT_BLOCK) hist[(int64_t)d * ntiles + tile] = s[d];
    __syncthreads();
  }
}

constexpr int RS_BLOCK = 256;  // k_radix_rowscan threads (a skipped pass dispatches 256 x 256 threads)
__global__ void __launch_bounds__(RS_BLOCK) k_radix_rowscan(uint32_t* __restrict__ hist, int64_t ntiles,
                                                        uint32_t* __restrict__ digit_total,
                                                        const sphb_ctrl_t* ctrl,
                                                        const uint32_t* skip) {
  if (!step_live(ctrl) || (skip && *skip == 0u)) return;
  __shared__ uint32_t s_warp[32];
  uint32_t* row = hist + (int64_t)blockIdx.x * ntiles;
  uint32_t running = 0;
  for (int64_t base = 0; base < ntiles; base += RS_BLOCK) {
    int64_t k = base + threadIdx.x;
    uint32_t v = k < ntiles ? row[k] : 0;
    uint32_t total;
    uint32_t ex = block_exclusive_scan<RS_BLOCK>(v, &total, s_warp);
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
    uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out, const sphb_ctrl_t* ctrl,
    const uint32_t* skip) {
  if (!step_live(ctrl) || (skip && *skip == 0u)) return;
  constexpr int NW = SORT_BLOCK / 32;
  __shared__ uint32_t s_base[RADIX];
  __shared__ uint32_t s_run[RADIX];
  __shared__ uint32_t s_wc[2][NW][RADIX];
  __shared__ uint32_t s_warp[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // persistent (see hist)
    // digit base = exclusive scan of digit totals (RADIX == SORT_BLOCK)
    {
      uint32_t v = digit_total[threadIdx.x], total;
      uint32_t ex = block_exclusive_scan<SORT_BLOCK>(v, &total, s_warp);
      s_base[threadIdx.x] = ex + hist[(int64_t)threadIdx.x * ntiles + tile];
      s_run[threadIdx.x] = 0;
      for (int w = 0; w < NW; ++w) s_wc[0][w][threadIdx.x] = 0;
    }
    __syncthreads();
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
    __syncthreads();
  }
}

// ------------------------------------------------------------------ K3 reorder + EOS
#ifndef NL_MINB
#define NL_MINB 4  // 64 registers: 2x the resident warps of the default (memory-bound kernel)
#endif
// FAST (FP32 precision with gamma = 7, the reference default): x^7 and x^3 by multiplication
// instead of two f64 pow calls -- press/csound then differ from the reference's pow in the
// last f32 bit at most, far inside the FP32 tolerance, and the kernel keeps all loads in
// flight (no calls).  The FP64 precision keeps pow: its results are bit-identical.
template <bool FAST>
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
    const int32_t o = perm ? perm[i] : (int32_t)i;
    const uint32_t ks = keys_sorted ? keys_sorted[i] : 0u;
    float4 pp = posp_in[o];
    const float4 vr = velr_in[o];
    const bool has_prev = prev_in && prev_out, has_id = id_in && id_out;
    float4 pv;
    long long id = 0;
    if (has_prev) pv = prev_in[o];
    if (has_id) id = id_in[o];
    const Deriv4 d = derived_of<FAST>((double)vr.w, p);
    // posp.w = prrho: the interaction stages (x, y, z, prrho) rows with one bulk copy
    pp.w = d.prrho;
    posp_out[i] = pp;
    velr_out[i] = vr;
    const bool boundary = keys_sorted ? ((ks >> cellbits) & 1u) == 0u : false;
    // aux may be absent: the FP32 gather / paired interaction recomputes a target's row
    if (aux_out)
      aux_out[i] = make_float4(d.press, d.csound, d.tensil,
                               (float)(boundary ? p.mass_boundary : p.mass_fluid));
    if (has_prev) prev_out[i] = pv;
    if (has_id) id_out[i] = id;
    if (cell_out && keys_sorted) cell_out[i] = (int32_t)(ks & cellmask);
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

// Per-key constants of the movers-only sort (k_mv_scatter), written while the previous ranges
// are still in beg/end: kv = (SB, MB, ob, head) with ob/oe the old range, nb the new begin,
// M(p) the movers before p:  SB = nb - ob + M(ob) (stayers: position = SB + i - M(i) + chain),
// MB = nb + (oe - ob) - (M(oe) - M(ob)) (movers after the old range), head = the key's mover
// chain (reset here for the next step).
struct MvApply {
  int4* kv;
  int32_t* head;
  const uint32_t* bits;
  const uint32_t* wpre;
  const uint32_t* state;
  int64_t n;
};

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_apply(uint32_t* __restrict__ cnt, int64_t len,
                                                           const uint32_t* __restrict__ partials,
                                                           int32_t* __restrict__ beg,
                                                           int32_t* __restrict__ end, MvApply mv,
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
  const bool movers = mv.kv && mv.state[2] == 0u;
  const uint32_t m = movers ? mv.state[3] : 0u;
  auto M = [&](int64_t p) -> int32_t {
    if (p >= mv.n) return (int32_t)m;
    const int64_t wi = p >> 5;
    return (int32_t)(mv.wpre[wi] + __popc(mv.bits[wi] & ((1u << (p & 31)) - 1u)));
  };
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const int64_t x = base + k;
    if (x < len) {
      if (mv.kv) {
        // chains are reset whatever the mode (k_mv_compact may have switched to the radix)
        const int32_t ob = beg[x], oe = end[x], h = mv.head[x];
        if (h >= 0) mv.head[x] = -1;
        if (movers && c[k] != 0u) {
          const int32_t mob = M(ob);
          mv.kv[x] = make_int4((int32_t)ex - ob + mob,
                               (int32_t)ex + (oe - ob) - (M(oe) - mob), ob, h);
        }
      }
      beg[x] = (int32_t)ex;
      ex += c[k];
      end[x] = (int32_t)ex;
      cnt[x] = 0;  // self-cleaning for the next step's histogram
    }
  }
}

// ------------------------------------------------------------------ K2' movers-only sort
// Inside sphb_step the rows arrive in the previous step's sorted order with K7's new keys, and
// the previous sort's keys (keys_sorted) and per-cell ranges (beg/end) are still in the state.
// A row whose key did not change ("stayer") keeps its place inside its old cell range; only
// the few rows that changed cell ("movers", 0.04% per step on average)
// need placing.  The stable order (grid.py:107-109: key, then current index) follows by
// counting, without a radix pass.  With M(p) = movers before position p (bitmap + prefix),
// [ob, oe) the key's old range and nb its new begin (this step's K4):
//   stayer i of key k:  position = nb + (i - ob) - (M(i) - M(ob)) + #{movers into k at < i}
//   mover  i into  k:   position = nb + (i < ob ? 0 : stayers of k) + #{movers into k at < i}
// Movers into a key are chained in a per-key list (only counts are read, so the chain order
// does not matter): the result is deterministic and identical to the radix sort.
//   k_mv_flag     mover bitmap + tile counts; checks the previous order (sorted keys_sorted,
//                 runs == [beg, end))
//   k_mv_scan     tile prefix, mover count, path decision
//   k_mv_compact  mover positions + per-key chains, per-word mover prefix
//   k_scan_apply  (K4) per-key constants (SB, MB, ob, chain) from the old ranges, then the new
//   k_mv_scatter  perm / keys_sorted
// The radix passes run instead (mode 1) unless the previous order is established (set by a
// sort, cleared by K1 and the standalone sphb_sort), consistent, and movers <= cap.
// state words: [0] order established, [1] inconsistency seen, [2] mode (0 movers, 1 radix), [3] m,
// [4] the dead-bin placement counter (X slabs)
constexpr int MV_BLOCK = 256, MV_ITEMS = 16, MV_TILE = MV_BLOCK * MV_ITEMS;  // 128 words per tile
static_assert(MV_TILE == MV_TILE_ROWS, "workspace sizing");

__device__ __forceinline__ uint32_t mv_index(uint32_t key, int cellbits, uint32_t ncells) {
  return key_bin(key, cellbits, ncells);  // X slabs: the dead key -> the dead bin (2 ncells)
}

// Each thread checks 4 consecutive rows per round (one 16-B load of keys and of keys_sorted
// when both are 16-B aligned), MV_ITEMS / 4 rounds per tile; the 4-row nibbles of 8 lanes
// make one bitmap word.
__global__ void __launch_bounds__(MV_BLOCK) k_mv_flag(const uint32_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ prev, int64_t n,
                                                      int cellbits, uint32_t ncells,
                                                      const int32_t* __restrict__ obeg,
                                                      const int32_t* __restrict__ oend,
                                                      uint32_t* __restrict__ bits,
                                                      uint32_t* __restrict__ tile_cnt, bool vec,
                                                      bool slab, uint32_t* state,
                                                      const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl) || state[0] == 0u) return;
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * MV_TILE;
  const uint32_t cm = (1u << cellbits) - 1u;
  const uint32_t dead = dead_key(cellbits);
  auto bad_key = [&](uint32_t k) {
    return k == dead ? !slab : ((k >> cellbits) > 1u || (k & cm) >= ncells);
  };
  bool bad = false;
  uint32_t c = 0;
  constexpr int RROWS = 4 * MV_BLOCK;  // rows per round
  for (int r = 0; r < MV_TILE / RROWS; ++r) {
    const int64_t e0 = t0 + (int64_t)r * RROWS + 4 * threadIdx.x;
    uint32_t k[4], kp[4];
    if (vec && e0 + 3 < n) {
      const uint4 a = reinterpret_cast<const uint4*>(keys)[e0 >> 2];
      const uint4 b = reinterpret_cast<const uint4*>(prev)[e0 >> 2];
      k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
      kp[0] = b.x; kp[1] = b.y; kp[2] = b.z; kp[3] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool in = e0 + j < n;
        k[j] = in ? keys[e0 + j] : 0u;
        kp[j] = in ? prev[e0 + j] : 0u;
      }
    }
    // consistency of the previous order (keys_sorted, beg, end of the last sort): keys_sorted
    // ascending and every run of equal keys exactly its [beg, end) -- checked at run ends
    uint32_t kl = __shfl_up_sync(SPHB_FULL, kp[3], 1), kr = __shfl_down_sync(SPHB_FULL, kp[0], 1);
    if (lane == 0 && e0 > 0 && e0 < n) kl = prev[e0 - 1];
    if (lane == 31 && e0 + 4 < n) kr = prev[e0 + 4];
    uint32_t nib = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t e = e0 + j;
      if (e >= n) break;
      nib |= (k[j] != kp[j] ? 1u : 0u) << j;
      if (bad_key(k[j]) || bad_key(kp[j])) {
        bad = true;  // out-of-domain key (the step is aborting) or no previous order
        continue;
      }
      const uint32_t left = j ? kp[j - 1] : kl, right = j < 3 ? kp[j + 1] : kr;
      const uint32_t x = key_bin(kp[j], cellbits, ncells);
      if (e == 0 || left != kp[j]) bad |= (e > 0 && left > kp[j]) || obeg[x] != (int32_t)e;
      if (e + 1 == n || right != kp[j]) bad |= oend[x] != (int32_t)(e + 1);
    }
    c += __popc(nib);
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(SPHB_FULL, w, 1);
    w |= __shfl_xor_sync(SPHB_FULL, w, 2);
    w |= __shfl_xor_sync(SPHB_FULL, w, 4);
    if ((lane & 7) == 0) bits[((t0 + (int64_t)r * RROWS + warp * 128) >> 5) + (lane >> 3)] = w;
  }
  c = __reduce_add_sync(SPHB_FULL, c);
  if (lane == 0 && c) atomicAdd(&s_cnt, c);
  if (__any_sync(SPHB_FULL, bad) && lane == 0) atomicOr(&state[1], 1u);
  __syncthreads();
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = s_cnt;
}

// one block: exclusive scan of the tile counts, mover total, path decision
__global__ void __launch_bounds__(1024) k_mv_scan(uint32_t* __restrict__ tile_cnt, int64_t ntiles,
                                                  int64_t cap, uint32_t* state,
                                                  const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl)) return;
  __shared__ uint32_t s_warp[32];
  const bool ordered = state[0] != 0u && state[1] == 0u && cap >= 0;
  uint32_t running = 0;
  if (ordered) {
    for (int64_t base = 0; base < ntiles; base += 1024) {
      const int64_t k = base + threadIdx.x;
      const uint32_t v = k < ntiles ? tile_cnt[k] : 0u;
      uint32_t total;
      const uint32_t ex = block_exclusive_scan<1024>(v, &total, s_warp);
      if (k < ntiles) tile_cnt[k] = running + ex;
      running += total;
    }
  }
  if (threadIdx.x == 0) {
    state[2] = (ordered && (int64_t)running <= cap) ? 0u : 1u;
    state[4] = 0u;  // dead-bin placement counter of k_mv_scatter
    state[3] = ordered ? running : 0u;
    state[1] = 0u;
    state[0] = 1u;  // this step's sort (either path) establishes the order for the next one
  }
}

// movers -> (position, key) list in index order + per-key chains; per-word mover prefix
__global__ void __launch_bounds__(MV_BLOCK) k_mv_compact(
    const uint32_t* __restrict__ keys, int cellbits, uint32_t ncells,
    const uint32_t* __restrict__ bits, const uint32_t* __restrict__ tile_pre,
    uint32_t* __restrict__ wpre, int32_t* __restrict__ mv_pos,
    int32_t* __restrict__ mv_next, int32_t* __restrict__ mv_head, const uint32_t* __restrict__ prev,
    const int32_t* __restrict__ obeg, const int32_t* __restrict__ oend, uint32_t* state,
    const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl) || state[2] != 0u) return;
  constexpr int NWORD = MV_TILE / 32;  // bitmap words per tile
  static_assert(NWORD <= MV_BLOCK, "one word per thread");
  __shared__ uint32_t s_w[NWORD], s_pre[NWORD], s_wsum[MV_BLOCK / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * NWORD;
  {  // exclusive prefix of the tile's word popcounts (one word per thread)
    const uint32_t w = threadIdx.x < NWORD ? bits[w0 + threadIdx.x] : 0u;
    const uint32_t c = __popc(w);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(SPHB_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t before = tile_pre[blockIdx.x];
    for (int k = 0; k < warp; ++k) before += s_wsum[k];
    if (threadIdx.x < NWORD) {
      const uint32_t pre = before + x - c;
      wpre[w0 + threadIdx.x] = pre;
      s_w[threadIdx.x] = w;
      s_pre[threadIdx.x] = pre;
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < MV_ITEMS; ++r) {
    const int wi = r * (MV_BLOCK / 32) + warp;
    const uint32_t w = s_w[wi];
    if ((w >> lane) & 1u) {
      const int64_t i = (int64_t)blockIdx.x * MV_TILE + r * MV_BLOCK + threadIdx.x;
      const int32_t j = (int32_t)(s_pre[wi] + __popc(w & lt));
      const uint32_t k = keys[i];
      const uint32_t x = mv_index(k, cellbits, ncells);
      mv_pos[j] = (int32_t)i;
      // an X slab's dead bin is placed by a counter (k_mv_scatter), not by chains: its rows
      // are dropped, their order is irrelevant, and the bin can take many movers per step
      mv_next[j] = x == 2u * ncells ? -1 : atomicExch(&mv_head[x], j);
      // a key absent from the previous order must have an empty old range (the run check of
      // k_mv_flag covers the keys present); otherwise fall back to the radix passes
      const int32_t ob = obeg[x];
      if (ob < oend[x] && prev[ob] != k) state[2] = 1u;
    }
  }
}

// 4 rows per thread, 32 apart (loads and stores stay coalesced; the 4 dependent load chains
// keys -> kv -> chains overlap)
__global__ void __launch_bounds__(256) k_mv_scatter(
    const uint32_t* __restrict__ keys, int64_t n, int cellbits, uint32_t ncells,
    const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wpre,
    const int4* __restrict__ kv, const int32_t* __restrict__ nbeg,
    const int32_t* __restrict__ mv_pos, const int32_t* __restrict__ mv_next,
    uint32_t* state, uint32_t* __restrict__ keys_sorted, int32_t* __restrict__ perm,
    const sphb_ctrl_t* ctrl) {
  if (!step_live(ctrl) || state[2] != 0u) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (n + 127) >> 7;  // 128-row warp chunks
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t cw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); cw < nw;
       cw += wstride) {
    uint32_t k[4], x[4], w[4], wp[4];
    int4 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = (cw << 7) + 32 * u + lane;
      k[u] = i < n ? keys[i] : 0u;
      w[u] = bits[(cw << 2) + u];
      wp[u] = wpre[(cw << 2) + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = mv_index(k[u], cellbits, ncells);
      if ((cw << 7) + 32 * u + lane < n) c[u] = kv[x[u]];  // (SB, MB, ob, head)
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = (cw << 7) + 32 * u + lane;
      if (i >= n) break;
      int64_t pos;
      if (x[u] == 2u * ncells)  // an X slab's dead rows (stayers and movers): any order
        pos = nbeg[x[u]] + (int64_t)atomicAdd(&state[4], 1u);
      else if (!((w[u] >> lane) & 1u))
        pos = (int64_t)c[u].x + i - (int64_t)(wp[u] + __popc(w[u] & ((1u << lane) - 1u)));
      else
        pos = i < c[u].z ? nbeg[x[u]] : c[u].y;
      if (x[u] != 2u * ncells)
        for (int32_t m = c[u].w; m >= 0; m = mv_next[m]) pos += mv_pos[m] < i;
      perm[pos] = (int32_t)i;
      keys_sorted[pos] = k[u];
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
  // movers-only path (4) + the radix passes (no-ops when the movers path ran) + K3 + K4
  return 4 + 3 * sort_pass_count(g) + 1 /*reorder*/ + 3 /*scan*/;
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
  // rows written from outside: the next sphb_step sort cannot trust the previous order
  if (cudaError_t e = cudaMemsetAsync(ws->mv_state, 0, sizeof(uint32_t), s))
    return sphb_set_error(SPHB_E_CUDA, "mv_state reset: %s", cudaGetErrorString(e));
  k_cell_keys<<<grid_for(n, 256), 256, 0, s>>>(g, posp, n, nb, cellbits_of(g), keys, cell_out,
                                                ws->cnt, nc, ctrl);
  return sphb_check_launch("k_cell_keys");
}

int launch_cell_hist(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys, int64_t n,
                     const sphb_ctrl_t* ctrl, cudaStream_t s) {
  const int64_t nc = ncells_of(g);
  if (n > ws->n_max || nc > ws->ncells_max) return sphb_set_error(SPHB_E_CAPACITY, "n/ncells exceed workspace");
  if (n == 0) return SPHB_OK;
  k_hist_keys<<<grid_for(n, 256), 256, 0, s>>>(keys, n, cellbits_of(g), nc, slab_grid(g), ws->cnt, ctrl);
  return sphb_check_launch("k_hist_keys");
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

static void radix_passes(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys,
                         int64_t n, uint32_t* keys_sorted, int32_t* perm,
                         const sphb_ctrl_t* ctrl, const uint32_t* skip, cudaStream_t s) {
  const int passes = sort_pass_count(g);
  const int64_t ntiles = (n + SORT_TILE - 1) / SORT_TILE;
  const uint32_t* kin = keys;
  const int32_t* vin = nullptr;
  for (int pass = 0; pass < passes; ++pass) {
    const bool last = pass == passes - 1;
    uint32_t* kout = last ? (keys_sorted ? keys_sorted : ws->keys_tmp[pass & 1]) : ws->keys_tmp[pass & 1];
    int32_t* vout = last ? perm : ws->vals_tmp[pass & 1];
    const int shift = pass * RADIX_BITS;
    // persistent over tiles; 2 CTAs per SM keep a skipped pass (the movers-only sort ran) cheap
    const unsigned grid = (unsigned)(ntiles < 148 * 2 ? ntiles : 148 * 2);
    k_radix_hist<<<grid, SORT_BLOCK, 0, s>>>(kin, n, shift, ws->radix_hist, ntiles, ctrl, skip);
    k_radix_rowscan<<<RADIX, RS_BLOCK, 0, s>>>(ws->radix_hist, ntiles, ws->digit_total, ctrl, skip);
    k_radix_scatter<<<grid, SORT_BLOCK, 0, s>>>(kin, vin, n, shift, ws->radix_hist,
                                                            ws->digit_total, ntiles, kout, vout,
                                                            ctrl, skip);
    kin = kout;
    vin = vout;
  }
}

int launch_sort(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys, int64_t n,
                uint32_t* keys_sorted, int32_t* perm, const sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (n > ws->n_max) return sphb_set_error(SPHB_E_CAPACITY, "n exceeds workspace");
  if (n == 0) return SPHB_OK;
  // arbitrary buffers: the movers-only path of the next sphb_step must not trust them
  if (cudaError_t e = cudaMemsetAsync(ws->mv_state, 0, sizeof(uint32_t), s))
    return sphb_set_error(SPHB_E_CUDA, "mv_state reset: %s", cudaGetErrorString(e));
  radix_passes(ws, g, keys, n, keys_sorted, perm, ctrl, nullptr, s);
  return sphb_check_launch("radix sort");
}

int launch_sort_and_ranges(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys,
                           int64_t n, uint32_t* keys_sorted, int32_t* perm, int32_t* beg,
                           int32_t* end, const sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (n > ws->n_max) return sphb_set_error(SPHB_E_CAPACITY, "n exceeds workspace");
  const int64_t nc = ncells_of(g);
  const int64_t len = nbins_of(g);  // both lists (+ an X slab's dead bin)
  const int64_t nscan = (len + SCAN_TILE - 1) / SCAN_TILE;
  if (nscan > ws->max_scan_tiles) return sphb_set_error(SPHB_E_CAPACITY, "ncells exceeds workspace");
  if (n == 0) return launch_cell_ranges(ws, g, beg, end, ctrl, s);
  const int cb = cellbits_of(g);
  const int64_t tiles = (n + MV_TILE - 1) / MV_TILE;
  uint32_t* st = ws->mv_state;
  const bool vec = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(keys_sorted)) & 15u) == 0;
  k_mv_flag<<<(unsigned)tiles, MV_BLOCK, 0, s>>>(keys, keys_sorted, n, cb, (uint32_t)nc, beg, end,
                                                 ws->mv_bits, ws->mv_tile, vec, slab_grid(g), st, ctrl);
  k_mv_scan<<<1, 1024, 0, s>>>(ws->mv_tile, tiles, ws->mover_cap, st, ctrl);
  k_mv_compact<<<(unsigned)tiles, MV_BLOCK, 0, s>>>(keys, cb, (uint32_t)nc, ws->mv_bits, ws->mv_tile,
                                                    ws->mv_wpre, ws->mv_pos,
                                                    ws->mv_next, ws->mv_head, keys_sorted, beg,
                                                    end, st, ctrl);
  // K4 for this step, keeping the previous ranges for the scatter
  k_scan_reduce<<<(unsigned)nscan, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, ctrl);
  k_scan_partials<<<1, 1024, 0, s>>>(ws->scan_partials, nscan, ctrl);
  const MvApply mva{ws->mv_kv, ws->mv_head, ws->mv_bits, ws->mv_wpre, st, n};
  k_scan_apply<<<(unsigned)nscan, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, beg, end,
                                                      mva, ctrl);
  k_mv_scatter<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(keys, n, cb, (uint32_t)nc, ws->mv_bits,
                                                         ws->mv_wpre, ws->mv_kv, beg, ws->mv_pos,
                                                         ws->mv_next, st, keys_sorted, perm, ctrl);
  radix_passes(ws, g, keys, n, keys_sorted, perm, ctrl, st + 2, s);  // mode 1 only
  return sphb_check_launch("sort + cell ranges");
}

int launch_reorder(const sphb_params_t& p, const sphb_grid_t& g, int64_t n, const int32_t* perm,
                   const uint32_t* keys_sorted, const float4* posp_in, const float4* velr_in,
                   const float4* prev_in, const int64_t* id_in, float4* posp_out,
                   float4* velr_out, float4* prev_out, int64_t* id_out, float4* aux_out,
                   int32_t* cell_out, const sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (n == 0) return SPHB_OK;
  uint32_t cellmask = (1u << cellbits_of(g)) - 1u;
  auto kern = (p.precision == SPHB_FP32 && p.gamma == 7.0) ? k_reorder<true> : k_reorder<false>;
  kern<<<grid_for(n, 256), 256, 0, s>>>(p, cellmask, cellbits_of(g), n, perm, keys_sorted, posp_in,
                                        velr_in, prev_in, id_in, posp_out, velr_out, prev_out,
                                        id_out, aux_out, cell_out, ctrl);
  return sphb_check_launch("k_reorder");
}

int launch_cell_ranges(sphb_workspace* ws, const sphb_grid_t& g, int32_t* beg, int32_t* end,
                       const sphb_ctrl_t* ctrl, cudaStream_t s) {
  const int64_t len = nbins_of(g);
  const int64_t ntiles = (len + SCAN_TILE - 1) / SCAN_TILE;
  if (ntiles > ws->max_scan_tiles) return sphb_set_error(SPHB_E_CAPACITY, "ncells exceeds workspace");
  k_scan_reduce<<<(unsigned)ntiles, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, ctrl);
  k_scan_partials<<<1, 1024, 0, s>>>(ws->scan_partials, ntiles, ctrl);
  k_scan_apply<<<(unsigned)ntiles, SCAN_BLOCK, 0, s>>>(ws->cnt, len, ws->scan_partials, beg, end,
                                                       MvApply{}, ctrl);
  return sphb_check_launch("cell ranges scan");
}
