// slab.cu -- device-resident X-slab exchange.
//
// After a rank's system update (K7) its primary arrays hold owned rows and last step's halo
// rows (negative ids), in the step's sorted order, with K7's next-step sort keys.  Three
// kernels rebuild the next step's arrays without host-side compaction:
//
//   k_slab_count    per 256-row tile, how many rows fall in each of the 10 categories
//                   {keep, migrate left, migrate right, halo left, halo right} x {boundary,
//                   fluid}; halo rows of the last step are dropped.  Column = (key & cellmask)
//                   mod nx, i.e. exactly assign_cells' x index (grid.py:87-89) from K7.
//   k_slab_scan     exclusive scan of the tile counts per category (deterministic offsets)
//                   + the 10 totals (the only numbers the host needs: one D2H per step).
//   k_slab_scatter  kept rows -> the next arrays (boundary block then fluid block, at bases
//                   the host derives from all ranks' totals); migrants / halo copies -> one
//                   packed 64-B-row send buffer per side, sections [mig B | mig F | halo B |
//                   halo F]; halo copies carry id' = -1 - id.
//   k_slab_unpack   a neighbour's packed rows -> their slots in the next arrays.
//
// Row order inside every category follows the input order (tile order, then thread order),
// so the exchange is deterministic.  The next step re-sorts everything by cell anyway.
#include "sphb_common.cuh"
#include "sphb_internal.h"

using namespace sphb;

namespace {

constexpr int ST = 256;   // rows per tile (= threads per block)
constexpr int NCAT = 10;  // category c = 2 * kind + list, kind in {keep, migL, migR, haloL, haloR}

struct SlabRow {  // 64 B packed exchange row
  float4 posp, velr, prev;
  long long id;
  uint32_t key;  // the sender's K7 sort key (global grid): the receiver needs no K1
  uint32_t pad;
};

__device__ __forceinline__ int col_of_key(uint32_t key, uint32_t cellmask, int nx) {
  return (int)((key & cellmask) % (uint32_t)nx);
}

// membership bits of row i: bit (2 kind + list)
__device__ __forceinline__ uint32_t row_cats(int64_t i, int64_t n, int64_t nb, const uint32_t* keys,
                                             const int64_t* id, uint32_t cellmask, int nx, int x0,
                                             int x1, int R) {
  if (i >= n) return 0u;
  if (id[i] < 0) return 0u;  // last step's halo copy: dropped
  const uint32_t list = i >= nb ? 1u : 0u;
  const uint32_t key = keys[i];
  if (key == 0xffffffffu) return 1u << list;  // out of domain: the error word already holds it
  const int c = col_of_key(key, cellmask, nx);
  if (c < x0) return 1u << (2 + list);
  if (c >= x1) return 1u << (4 + list);
  uint32_t m = 1u << list;
  if (c < x0 + R) m |= 1u << (6 + list);
  if (c >= x1 - R) m |= 1u << (8 + list);
  return m;
}

__global__ void __launch_bounds__(ST) k_slab_count(int64_t n, int64_t nb, const uint32_t* keys,
                                                   const int64_t* id, uint32_t cellmask, int nx,
                                                   int x0, int x1, int R, uint32_t* tile_counts) {
  __shared__ uint32_t sc[NCAT];
  if (threadIdx.x < NCAT) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * ST + threadIdx.x;
  const uint32_t m = row_cats(i, n, nb, keys, id, cellmask, nx, x0, x1, R);
#pragma unroll
  for (int c = 0; c < NCAT; ++c) {
    const uint32_t b = __ballot_sync(SPHB_FULL, (m >> c) & 1u);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(&sc[c], (uint32_t)__popc(b));
  }
  __syncthreads();
  if (threadIdx.x < NCAT) tile_counts[(int64_t)blockIdx.x * NCAT + threadIdx.x] = sc[threadIdx.x];
}

// one warp per category: exclusive scan over tiles, totals[c] at the end
__global__ void k_slab_scan(int64_t ntiles, uint32_t* tile_counts, uint32_t* totals) {
  const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (c >= NCAT) return;
  uint32_t run = 0;
  for (int64_t t0 = 0; t0 < ntiles; t0 += 32) {
    const int64_t t = t0 + lane;
    const uint32_t v = t < ntiles ? tile_counts[t * NCAT + c] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(SPHB_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (t < ntiles) tile_counts[t * NCAT + c] = run + incl - v;
    run += __shfl_sync(SPHB_FULL, incl, 31);
  }
  if (lane == 0) totals[c] = run;
}

__global__ void __launch_bounds__(ST) k_slab_scatter(
    int64_t n, int64_t nb, const uint32_t* keys, uint32_t cellmask, int nx, int x0, int x1, int R,
    const uint32_t* tile_offsets, const float4* __restrict__ posp, const float4* __restrict__ velr,
    const float4* __restrict__ prev, const int64_t* __restrict__ id, int64_t keep_base_b,
    int64_t keep_base_f, float4* __restrict__ nposp, float4* __restrict__ nvelr,
    float4* __restrict__ nprev, int64_t* __restrict__ nid, uint32_t* __restrict__ nkeys,
    SlabRow* __restrict__ send_l,
    SlabRow* __restrict__ send_r, int64_t sec_l_migf, int64_t sec_l_halob, int64_t sec_l_halof,
    int64_t sec_r_migf, int64_t sec_r_halob, int64_t sec_r_halof) {
  __shared__ uint32_t swarp[ST / 32][NCAT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * ST + threadIdx.x;
  const uint32_t m = row_cats(i, n, nb, keys, id, cellmask, nx, x0, x1, R);
  uint32_t rank_in_warp[NCAT];
#pragma unroll
  for (int c = 0; c < NCAT; ++c) {
    const uint32_t b = __ballot_sync(SPHB_FULL, (m >> c) & 1u);
    rank_in_warp[c] = __popc(b & lanemask_lt());
    if (lane == 0) swarp[warp][c] = __popc(b);
  }
  __syncthreads();
  if (!m) return;
  SlabRow row;
  row.posp = posp[i];
  row.velr = velr[i];
  row.prev = prev[i];
  row.id = id[i];
  row.key = keys[i];
  row.pad = 0;
#pragma unroll
  for (int c = 0; c < NCAT; ++c) {
    if (!((m >> c) & 1u)) continue;
    uint32_t r = tile_offsets[(int64_t)blockIdx.x * NCAT + c] + rank_in_warp[c];
    for (int w = 0; w < warp; ++w) r += swarp[w][c];
    const int kind = c >> 1, list = c & 1;
    if (kind == 0) {  // keep
      const int64_t o = (list ? keep_base_f : keep_base_b) + r;
      nposp[o] = row.posp;
      nvelr[o] = row.velr;
      nprev[o] = row.prev;
      nid[o] = row.id;
      if (nkeys) nkeys[o] = row.key;
    } else if (kind == 1 || kind == 3) {  // to the left neighbour
      const int64_t o = kind == 1 ? (list ? sec_l_migf : 0) + r : (list ? sec_l_halof : sec_l_halob) + r;
      SlabRow q = row;
      if (kind == 3) q.id = -1 - q.id;
      send_l[o] = q;
    } else {  // to the right neighbour
      const int64_t o = kind == 2 ? (list ? sec_r_migf : 0) + r : (list ? sec_r_halof : sec_r_halob) + r;
      SlabRow q = row;
      if (kind == 4) q.id = -1 - q.id;
      send_r[o] = q;
    }
  }
}

// rows [r0, r0 + cnt) of a received buffer -> next arrays at dst
__global__ void __launch_bounds__(ST) k_slab_unpack(const SlabRow* __restrict__ buf, int64_t r0,
                                                    int64_t cnt, int64_t dst, float4* nposp,
                                                    float4* nvelr, float4* nprev, int64_t* nid,
                                                    uint32_t* nkeys) {
  for (int64_t k = (int64_t)blockIdx.x * ST + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * ST) {
    const SlabRow q = buf[r0 + k];
    nposp[dst + k] = q.posp;
    nvelr[dst + k] = q.velr;
    nprev[dst + k] = q.prev;
    nid[dst + k] = q.id;
    if (nkeys) nkeys[dst + k] = q.key;
  }
}

}  // namespace

int64_t slab_tiles(int64_t n) { return (n + ST - 1) / ST; }

int launch_slab_count(const sphb_grid_t& g, int64_t n, int64_t nb, const uint32_t* keys,
                      const int64_t* id, int x0, int x1, uint32_t* tile_counts, uint32_t* totals,
                      cudaStream_t s) {
  const int64_t nt = slab_tiles(n);
  const uint32_t cellmask = (1u << cellbits_of(g)) - 1u;
  if (nt > 0) {
    k_slab_count<<<(unsigned)nt, ST, 0, s>>>(n, nb, keys, id, cellmask, g.dims[0], x0, x1, g.reach,
                                             tile_counts);
    if (int rc = sphb_check_launch("k_slab_count")) return rc;
  }
  k_slab_scan<<<1, 32 * NCAT, 0, s>>>(nt, tile_counts, totals);
  return sphb_check_launch("k_slab_scan");
}

int launch_slab_scatter(const sphb_grid_t& g, int64_t n, int64_t nb, const uint32_t* keys,
                        const int64_t* id, int x0, int x1, const uint32_t* tile_offsets,
                        const float4* posp, const float4* velr, const float4* prev,
                        const int64_t* keep_bases, float4* nposp, float4* nvelr, float4* nprev,
                        int64_t* nid, uint32_t* nkeys, void* send_l, void* send_r,
                        const int64_t* sections, cudaStream_t s) {
  const int64_t nt = slab_tiles(n);
  if (nt == 0) return SPHB_OK;
  const uint32_t cellmask = (1u << cellbits_of(g)) - 1u;
  k_slab_scatter<<<(unsigned)nt, ST, 0, s>>>(
      n, nb, keys, cellmask, g.dims[0], x0, x1, g.reach, tile_offsets, posp, velr, prev, id,
      keep_bases[0], keep_bases[1], nposp, nvelr, nprev, nid, nkeys, (SlabRow*)send_l, (SlabRow*)send_r,
      sections[0], sections[1], sections[2], sections[3], sections[4], sections[5]);
  return sphb_check_launch("k_slab_scatter");
}

int launch_slab_unpack(const void* buf, int64_t r0, int64_t cnt, int64_t dst, float4* nposp,
                       float4* nvelr, float4* nprev, int64_t* nid, uint32_t* nkeys,
                       cudaStream_t s) {
  if (cnt <= 0) return SPHB_OK;
  int64_t blocks = (cnt + ST - 1) / ST;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_slab_unpack<<<(unsigned)blocks, ST, 0, s>>>((const SlabRow*)buf, r0, cnt, dst, nposp, nvelr,
                                                nprev, nid, nkeys);
  return sphb_check_launch("k_slab_unpack");
}
