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
// These rebuild a slab's arrays from scratch: the initial halos and re-settling after the
// bounds move (DeviceSlabSim.prime / set_bounds).
//
// The per-step exchange keeps the rows in place instead (edge bands):
//
//   k_band_seg / k_band_info  right after NL: per (list, cell row) segment of the W = reach + 1
//                   edge columns on each side with a neighbour, the contiguous sorted range and
//                   its offset in that side's send buffer; the host-read info words (live rows,
//                   boundary rows, band rows per side, error word)
//   k_band_pack     after the edge targets' interaction: each band row's sorted state + its
//                   forces (96-B BandRow) into the send buffer of its side -- the neighbour's
//                   halo and migrants of the NEXT step are exactly these rows once integrated,
//                   so they travel while the interior targets' interaction runs
//   k_band_integrate  the receiver integrates a neighbour's band rows with K7's arithmetic
//                   (su_row.cuh, same dt) and keeps those that land in its slab (owned:
//                   migrants) or its halo columns (id' = -1 - id), the rest get the dead key;
//                   appended after the live rows, sort keys + histogram for the next NL
//   k_slab_tail     the dead bin's end = the next step's row count (previous-order
//                   bookkeeping of the movers-only sort)
#include "sphb_common.cuh"
#include "sphb_internal.h"
#include "su_row.cuh"

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
  const uint32_t key = keys[i];
  if (key == 0xffffffffu) return 1u << (i >= nb ? 1u : 0u);  // out of domain: the error word holds it
  if (key == (cellmask << 1 | 1u)) return 0u;  // dead key (left the slab / stale): dropped
  // the list from the key: after steps of the edge-band exchange the rows are no longer
  // [boundary | fluid] by index (arrivals are appended)
  const uint32_t list = key > cellmask ? 1u : 0u;
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


// ====================================================================== edge bands
constexpr int BS = 1024;  // segments per k_band_seg CTA

struct BandRow {  // 96 B: one sorted row of the sender and its interaction result
  float4 posp, velr, prev;
  double acc[3];
  double drho;
  long long id;
  uint32_t list;
  uint32_t pad;
};
static_assert(sizeof(BandRow) == SPHB_BAND_ROW_BYTES, "band row layout (include/sphb200.h)");

struct BandGeom {
  int64_t nrows, nseg, cps, ncells;
  int nx, xa[2], xb[2];  // columns [xa, xb) of the left / right band
  int sides;
};

__host__ __device__ inline BandGeom band_geom(const sphb_grid_t& g, int width, int sides) {
  BandGeom b;
  b.nx = g.dims[0];
  b.nrows = (int64_t)g.dims[1] * g.dims[2];
  b.nseg = 2 * b.nrows;
  b.cps = (b.nseg + BS - 1) / BS;
  b.ncells = ncells_of(g);
  b.xa[0] = g.tx0;
  b.xb[0] = g.tx0 + width < g.tx1 ? g.tx0 + width : g.tx1;
  b.xa[1] = g.tx1 - width > g.tx0 ? g.tx1 - width : g.tx0;
  b.xb[1] = g.tx1;
  b.sides = sides;
  return b;
}

// sorted rows of segment s (list = s / nrows, cell row r = s % nrows) of a side
__device__ __forceinline__ int2 band_rows(const BandGeom& b, int side, int64_t s,
                                          const int32_t* beg, const int32_t* end) {
  const int64_t list = s / b.nrows, r = s - list * b.nrows;
  const int64_t c0 = list * b.ncells + r * b.nx;
  return make_int2(beg[c0 + b.xa[side]], end[c0 + b.xb[side] - 1]);
}

// scratch (int32): seg_off[2][nseg] | chunk_sum[2][cps] | chunk_pre[2][cps]
__global__ void __launch_bounds__(BS) k_band_seg(BandGeom b, const int32_t* __restrict__ beg,
                                                 const int32_t* __restrict__ end,
                                                 int32_t* __restrict__ scratch) {
  __shared__ int32_t s_w[BS / 32];
  const int side = (int)(blockIdx.x / b.cps);
  const int64_t chunk = blockIdx.x - (int64_t)side * b.cps;
  const int64_t s = chunk * BS + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t v = 0;
  if (((b.sides >> side) & 1) && s < b.nseg) {
    const int2 r = band_rows(b, side, s, beg, end);
    v = r.y - r.x;
  }
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(SPHB_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(SPHB_FULL, w, o);
      if (lane >= o) w += y;
    }
    s_w[lane] = w;
  }
  __syncthreads();
  if (s < b.nseg) scratch[side * b.nseg + s] = (warp ? s_w[warp - 1] : 0) + x - v;
  if (threadIdx.x == 0) scratch[2 * b.nseg + side * b.cps + chunk] = s_w[BS / 32 - 1];
}

// one CTA: chunk prefixes per side, band totals, the host-read info words
__global__ void __launch_bounds__(1024) k_band_info(BandGeom b, const int32_t* __restrict__ beg,
                                                    const int32_t* __restrict__ end,
                                                    int32_t* __restrict__ scratch,
                                                    int64_t* __restrict__ info,
                                                    const sphb_ctrl_t* ctrl) {
  __shared__ int64_t s_tot[2];
  if (threadIdx.x < 2) s_tot[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x < 64) {  // warp 0: left side, warp 1: right side
    const int side = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t* sum = scratch + 2 * b.nseg + side * b.cps;
    int32_t* pre = scratch + 2 * b.nseg + 2 * b.cps + side * b.cps;
    int64_t run = 0;
    for (int64_t c0 = 0; c0 < b.cps; c0 += 32) {
      const int64_t c = c0 + lane;
      const int32_t v = c < b.cps ? sum[c] : 0;
      int32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(SPHB_FULL, x, o);
        if (lane >= o) x += y;
      }
      if (c < b.cps) pre[c] = (int32_t)run + x - v;
      run += __shfl_sync(SPHB_FULL, x, 31);
    }
    if (lane == 0) s_tot[side] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = end[2 * b.ncells - 1];  // live rows (= the dead bin's begin)
    info[1] = beg[b.ncells];          // boundary rows: the fluid list starts at nb
    info[2] = s_tot[0];
    info[3] = s_tot[1];
    info[4] = (int64_t)ctrl->err;
    info[5] = ctrl->active;
    info[6] = ctrl->step;
    info[7] = 0;
  }
}

// one warp per segment: rows [sb, se) -> the side's send buffer at the segment's offset.  The
// peer-memory transport passes the neighbours' receive buffers (NVLink stores) and their flag
// words: every block fences its stores at system scope, the last one (elected on `done`)
// releases `tag` into the flags.
__global__ void __launch_bounds__(256) k_band_pack(
    BandGeom b, const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
    const int32_t* __restrict__ scratch, const float4* __restrict__ posp_s,
    const float4* __restrict__ velr_s, const float4* __restrict__ prev_s,
    const int64_t* __restrict__ id_s, const void* __restrict__ accv,
    const double* __restrict__ drho, bool f32, BandRow* __restrict__ send_l,
    BandRow* __restrict__ send_r, unsigned long long* flag_l, unsigned long long* flag_r,
    unsigned long long tag, uint32_t* done) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < 2 * b.nseg;
       w += nw) {
    const int side = (int)(w / b.nseg);
    if (!((b.sides >> side) & 1)) continue;
    const int64_t s = w - side * b.nseg;
    const int2 r = band_rows(b, side, s, beg, end);
    if (r.y <= r.x) continue;
    const int64_t off = (int64_t)scratch[2 * b.nseg + 2 * b.cps + side * b.cps + s / BS] +
                        scratch[side * b.nseg + s];
    BandRow* out = (side ? send_r : send_l) + off;
    const uint32_t list = s >= b.nrows ? 1u : 0u;
    for (int k = lane; k < r.y - r.x; k += 32) {
      const int64_t i = r.x + k;
      BandRow q;
      q.posp = posp_s[i];
      q.velr = velr_s[i];
      q.prev = prev_s[i];
      if (f32) {
        const float4 a4 = ((const float4*)accv)[i];
        q.acc[0] = a4.x;
        q.acc[1] = a4.y;
        q.acc[2] = a4.z;
        q.drho = a4.w;
      } else {
        const double* a = (const double*)accv;
        q.acc[0] = a[3 * i];
        q.acc[1] = a[3 * i + 1];
        q.acc[2] = a[3 * i + 2];
        q.drho = drho[i];
      }
      q.id = id_s[i];
      q.list = list;
      q.pad = 0;
      out[k] = q;
    }
  }
  if (done) {  // peer-memory transport: signal the neighbours once every block's rows are out
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0u;
      __threadfence_system();
      if (flag_l) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag_l), "l"(tag) : "memory");
      if (flag_r) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag_r), "l"(tag) : "memory");
    }
  }
}

// the receiving side: wait for this rank's flag words (written by the neighbours' k_band_pack)
__global__ void k_band_wait(const unsigned long long* flag_l, const unsigned long long* flag_r,
                            unsigned long long tag, sphb_ctrl_t* ctrl) {
  const unsigned long long* f = threadIdx.x == 0 ? flag_l : flag_r;
  if (threadIdx.x > 1 || !f) return;
  const long long t0 = clock64();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
    if (v >= tag) return;
    if (clock64() - t0 > 20000000000ll) {  // ~10 s at 2 GHz: the neighbour is gone
      raise_div(ctrl, ctrl->step, SPHB_DIV_EXCHANGE_TIMEOUT, 0);
      return;
    }
    __nanosleep(200);
  }
}

// a neighbour's band rows, integrated here (K7's arithmetic and dt) and classified by the new
// column: this slab -> owned (a migrant when it came from the neighbour's side of the bound),
// this slab's halo columns -> halo copy (id' = -1 - id), elsewhere -> dead key
__global__ void __launch_bounds__(256) k_band_integrate(
    sphb_params_t p, sphb_grid_t g, int cellbits, int64_t ncells, const BandRow* __restrict__ buf,
    int64_t cnt, int64_t dst, float4* __restrict__ posp, float4* __restrict__ velr,
    float4* __restrict__ prev, int64_t* __restrict__ id, uint32_t* __restrict__ keys_next,
    uint32_t* __restrict__ keys_sorted, uint32_t* __restrict__ hist, sphb_ctrl_t* ctrl) {
  if (!su_step_live(ctrl)) return;
  const SuStep st = su_step<0>(p, ctrl);
  const uint32_t dead = dead_key(cellbits);
  const int nx = g.dims[0], R = g.reach, lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < cnt; base += stride) {
    const int64_t k = base + threadIdx.x;
    int64_t slot = -1;
    if (k < cnt) {
      const BandRow q = buf[k];
      const bool fluid = q.list != 0u;
      float4 np, nv, nprev;
      su_row<0>(p, st, fluid, q.id, q.posp, q.velr, q.prev, q.acc, q.drho, np, nv, nprev);
      const int32_t c = cell_of(np.x, np.y, np.z, g);  // out of domain: the owner flags it
      uint32_t key = dead;
      long long pid = q.id;
      if (c >= 0) {
        const int col = c % nx;
        const bool owned = col >= g.tx0 && col < g.tx1;
        const bool halo = (col >= g.tx0 - R && col < g.tx0) || (col >= g.tx1 && col < g.tx1 + R);
        if (owned || halo) {
          key = (q.list << cellbits) | (uint32_t)c;
          slot = (int64_t)q.list * ncells + c;
          if (halo) pid = -1 - pid;
        }
      }
      if (slot < 0) slot = 2 * ncells;
      const int64_t o = dst + k;
      posp[o] = np;
      velr[o] = nv;
      prev[o] = nprev;
      id[o] = pid;
      keys_next[o] = key;
      keys_sorted[o] = dead;  // previous order: the appended rows sit in the dead bin
    }
    const uint32_t peers = __match_any_sync(SPHB_FULL, (unsigned long long)slot);
    if (slot >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[slot], (uint32_t)__popc(peers));
  }
}

__global__ void k_slab_tail(int32_t* end, int64_t dead_bin, int64_t n_next) {
  end[dead_bin] = (int32_t)n_next;
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

// ---------------------------------------------------------------- edge-band launchers
int64_t band_scratch_words(const sphb_grid_t& g) {
  const BandGeom b = band_geom(g, 1, 3);
  return 2 * b.nseg + 4 * b.cps + 8;
}

int launch_band_count(const sphb_grid_t& g, int width, int sides, const int32_t* beg,
                      const int32_t* end, int32_t* scratch, int64_t* info,
                      const sphb_ctrl_t* ctrl, cudaStream_t s) {
  const BandGeom b = band_geom(g, width, sides);
  k_band_seg<<<(unsigned)(2 * b.cps), BS, 0, s>>>(b, beg, end, scratch);
  if (int rc = sphb_check_launch("k_band_seg")) return rc;
  k_band_info<<<1, 1024, 0, s>>>(b, beg, end, scratch, info, ctrl);
  return sphb_check_launch("k_band_info");
}

int launch_band_pack(const sphb_params_t& p, const sphb_grid_t& g, int width, int sides,
                     const int32_t* beg, const int32_t* end, const int32_t* scratch,
                     const float4* posp_s, const float4* velr_s, const float4* prev_s,
                     const int64_t* id_s, const void* acc, const void* drho, void* send_l,
                     void* send_r, cudaStream_t s) {
  const BandGeom b = band_geom(g, width, sides);
  if (!sides) return SPHB_OK;
  int64_t blocks = (2 * b.nseg + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_band_pack<<<(unsigned)blocks, 256, 0, s>>>(b, beg, end, scratch, posp_s, velr_s, prev_s, id_s,
                                               acc, (const double*)drho, p.precision == SPHB_FP32,
                                               (BandRow*)send_l, (BandRow*)send_r, nullptr, nullptr,
                                               0ull, nullptr);
  return sphb_check_launch("k_band_pack");
}

int launch_band_put(const sphb_params_t& p, const sphb_grid_t& g, int width, int sides,
                    const int32_t* beg, const int32_t* end, const int32_t* scratch,
                    const float4* posp_s, const float4* velr_s, const float4* prev_s,
                    const int64_t* id_s, const void* acc, const void* drho, void* peer_l,
                    void* peer_r, uint64_t* flag_l, uint64_t* flag_r, uint64_t tag, uint32_t* done,
                    cudaStream_t s) {
  const BandGeom b = band_geom(g, width, sides);
  if (!sides) return SPHB_OK;
  // a few CTAs: the put runs on a comm stream next to the interior interaction, whose
  // persistent CTAs take the other SMs; 32 x 8 warps keep enough NVLink stores in flight
  int64_t blocks = (2 * b.nseg + 7) / 8;
  if (blocks > 32) blocks = 32;
  k_band_pack<<<(unsigned)blocks, 256, 0, s>>>(b, beg, end, scratch, posp_s, velr_s, prev_s, id_s,
                                               acc, (const double*)drho, p.precision == SPHB_FP32,
                                               (BandRow*)peer_l, (BandRow*)peer_r,
                                               (unsigned long long*)flag_l, (unsigned long long*)flag_r,
                                               (unsigned long long)tag, done);
  return sphb_check_launch("k_band_pack (peer)");
}

int launch_band_wait(const uint64_t* flag_l, const uint64_t* flag_r, uint64_t tag, sphb_ctrl_t* ctrl,
                     cudaStream_t s) {
  if (!flag_l && !flag_r) return SPHB_OK;
  k_band_wait<<<1, 32, 0, s>>>((const unsigned long long*)flag_l, (const unsigned long long*)flag_r,
                                (unsigned long long)tag, ctrl);
  return sphb_check_launch("k_band_wait");
}

int launch_band_integrate(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                          const void* buf, int64_t cnt, int64_t dst, float4* posp, float4* velr,
                          float4* prev, int64_t* id, uint32_t* keys_next, uint32_t* keys_sorted,
                          sphb_ctrl_t* ctrl, cudaStream_t s) {
  if (cnt <= 0) return SPHB_OK;
  int64_t blocks = (cnt + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_band_integrate<<<(unsigned)blocks, 256, 0, s>>>(p, g, cellbits_of(g), ncells_of(g),
                                                    (const BandRow*)buf, cnt, dst, posp, velr, prev,
                                                    id, keys_next, keys_sorted, ws->cnt, ctrl);
  return sphb_check_launch("k_band_integrate");
}

int launch_slab_tail(const sphb_grid_t& g, int32_t* end, int64_t n_next, cudaStream_t s) {
  k_slab_tail<<<1, 1, 0, s>>>(end, 2 * ncells_of(g), n_next);
  return sphb_check_launch("k_slab_tail");
}
