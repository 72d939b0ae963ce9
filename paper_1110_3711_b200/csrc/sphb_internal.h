// sphb_internal.h -- workspace layout and kernel launchers shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sphb200.h"

constexpr int SORT_BLOCK = 256;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_BLOCK * SORT_ITEMS;  // keys per radix tile
constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;
constexpr int MV_TILE_ROWS = 4096;          // rows per movers-only sort tile (128 bitmap words)
constexpr int64_t MOVER_CAP_MAX = 1 << 20;  // movers per step the movers-only sort accepts

struct sphb_workspace {
  int64_t n_max = 0, ncells_max = 0;
  uint32_t* cnt = nullptr;          // 2*ncells_max (+1: a slab's dead bin) per-key histogram, kept zero between steps
  uint32_t* keys_tmp[2] = {nullptr, nullptr};
  int32_t* vals_tmp[2] = {nullptr, nullptr};
  uint32_t* radix_hist = nullptr;   // RADIX * max tiles
  uint32_t* digit_total = nullptr;  // RADIX
  uint32_t* scan_partials = nullptr;
  int4* blocks = nullptr;  // interaction target blocks (fluid i0,i1, boundary i0,i1)
  int64_t max_blocks = 0;
  int32_t* row_off = nullptr;  // per cell row: block records (k_blocks count pass), then offsets
  int64_t max_sort_tiles = 0, max_scan_tiles = 0;
  double* energy_part = nullptr;  // 592 x 5 partial sums of sphb_energy
  // movers-only sort (nl.cu, k_mv_*): state words, per-32-row mover bitmap and prefix, tile
  // counts, the mover list and per-key chains, per-key placement constants
  uint32_t* mv_state = nullptr;  // [order established, inconsistency, mode, movers]
  uint32_t* mv_bits = nullptr;
  uint32_t* mv_wpre = nullptr;
  uint32_t* mv_tile = nullptr;
  int32_t* mv_pos = nullptr;
  int32_t* mv_next = nullptr;
  int32_t* mv_head = nullptr;  // 2*ncells_max + 1, -1 between steps
  int4* mv_kv = nullptr;       // 2*ncells_max + 1 per-key (SB, MB, old begin, chain head)
  int64_t mover_cap_max = 0, mover_cap = 0;
  int32_t pi_block = 128;  // targets per interaction block: 128, 256 or 384 (pi128/256/384)
  int32_t pi_kernel = 0;   // SPHB_PI_GATHER | SPHB_PI_SYMMETRIC (pi384s) | SPHB_PI_PAIRED (pi512p)
  unsigned long long* sym_scratch = nullptr;  // half-stencil candidate count (SPHB_COUNTERS_SYMMETRIC)
  size_t bytes = 0;
  // the interaction's block list built on a side stream while K3 reorders (sphb_interact_plan,
  // sphb_step): the next sphb_interact with the same tables and window waits on ev_plan
  // instead of building it again
  unsigned long long* cand_acc = nullptr;  // the plan's candidate count until the kernel takes it
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_plan = nullptr;
  struct Plan {
    bool valid = false;
    const int32_t* beg = nullptr;
    const int32_t* end = nullptr;
    int32_t dims[3] = {0, 0, 0}, tx0 = 0, tx1 = 0, reach = 0, precision = 0, order = 0;
    int32_t pi_block = 0, pi_kernel = 0;
  } plan;
};

// nl.cu
int launch_cell_keys(sphb_workspace* ws, const sphb_grid_t& g, const float4* posp, int64_t n,
                     int64_t nb, uint32_t* keys, int32_t* cell_out, sphb_ctrl_t* ctrl,
                     cudaStream_t s);
int launch_sort(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys, int64_t n,
                uint32_t* keys_sorted, int32_t* perm, const sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_reorder(const sphb_params_t& p, const sphb_grid_t& g, int64_t n, const int32_t* perm,
                   const uint32_t* keys_sorted, const float4* posp_in, const float4* velr_in,
                   const float4* prev_in, const int64_t* id_in, float4* posp_out,
                   float4* velr_out, float4* prev_out, int64_t* id_out, float4* aux_out,
                   int32_t* cell_out, const sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_cell_ranges(sphb_workspace* ws, const sphb_grid_t& g, int32_t* beg, int32_t* end,
                       const sphb_ctrl_t* ctrl, cudaStream_t s);
// sphb_step's NL: movers-only stable sort (radix fallback on the device) + K4
int launch_sort_and_ranges(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys,
                           int64_t n, uint32_t* keys_sorted, int32_t* perm, int32_t* beg,
                           int32_t* end, const sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_hist_from_sorted(sphb_workspace* ws, const sphb_grid_t& g, const int32_t* cell_sorted,
                            int64_t n, int64_t nb, cudaStream_t s);
int sort_pass_count(const sphb_grid_t& g);
int64_t nl_launch_count(const sphb_grid_t& g, int64_t n);

// interact.cu, compiled three times: pi128 (4-warp CTAs, 128-target blocks over <= 2,304 staged
// candidates, 2 CTAs/SM), pi256 (8-warp CTAs, 256 targets over <= 4,224, 1 CTA/SM: small
// systems, where 384-target blocks leave SMs idle) and pi384 (12-warp CTAs, 384-target blocks over <= 4,608 staged
// candidates, 1 CTA/SM: more resident warps, 25% less screen work per target, fewer idle
// lanes once cells fill unevenly)
constexpr int PI_LARGE_BLOCK = 384;
#define SPHB_DECLARE_PI(NS)                                                                     \
  namespace NS {                                                                                \
  int plan_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,         \
                    const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s,  \
                    unsigned long long* cand_acc);                                            \
  int launch_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,       \
                      int64_t n, int64_t nb, const float4* posp, const float4* velr,           \
                      const float4* aux, const int32_t* cell_sorted, const int32_t* beg,       \
                      const int32_t* end, void* acc, void* drho, void* visc,             \
                      sphb_ctrl_t* ctrl, cudaStream_t s);                                      \
  int64_t interact_launch_count(int64_t n);                                                    \
  }
SPHB_DECLARE_PI(pi128)
SPHB_DECLARE_PI(pi256)
SPHB_DECLARE_PI(pi384)
SPHB_DECLARE_PI(pi384s)
SPHB_DECLARE_PI(pi512)   // 16-warp CTAs on 2 x 2-row bricks
SPHB_DECLARE_PI(pi512p)  // 8-warp CTAs, two targets per lane, 512-target bricks (SPHB_PI_PAIRED)
// the workspace's blocking (FP64 always pi128)
int launch_interact(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g, int64_t n, int64_t nb,
                    const float4* posp, const float4* velr, const float4* aux,
                    const int32_t* cell_sorted, const int32_t* beg, const int32_t* end,
                    void* acc, void* drho, void* visc, sphb_ctrl_t* ctrl, cudaStream_t s);
int64_t interact_launch_count(int64_t n);

// the block list of the next interaction (k_blocks with the candidate counter, its scan; k_cand_cells at reach 2) on the workspace's
// side stream, forked from s after the cell ranges (capi.cu)
int plan_interact_async(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                        const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s);
// stepfn.cu: StepStats of the symmetric traversal (SPHB_COUNTERS_SYMMETRIC) from the gather-type
// counters of either kernel
int launch_sym_counters(sphb_workspace* ws, const sphb_grid_t& g, const int32_t* beg,
                        const int32_t* end, sphb_ctrl_t* ctrl, cudaStream_t s);

// integrate.cu
int launch_step_begin(sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_integrate(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g, int64_t n,
                     int64_t nb, const float4* posp_s, const float4* velr_s, const float4* prev_s,
                     const int64_t* id_s, const void* acc, const void* drho, float4* posp,
                     float4* velr, float4* prev, int64_t* id, uint32_t* keys_next,
                     sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_integrate_mode(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                          int64_t n, int64_t nb, int mode, const float4* posp_s,
                          const float4* velr_s, const float4* prev_s, const int64_t* id_s,
                          const void* acc, const void* drho, float4* posp, float4* velr,
                          float4* prev, int64_t* id, uint32_t* keys_next, sphb_ctrl_t* ctrl,
                          cudaStream_t s);
int launch_energy(sphb_workspace* ws, const sphb_params_t& p, int64_t n, int64_t nb,
                  const float4* posp, const float4* velr, double* out, cudaStream_t s);
// slab.cu
int64_t slab_tiles(int64_t n);
int launch_slab_count(const sphb_grid_t& g, int64_t n, int64_t nb, const uint32_t* keys,
                      const int64_t* id, int x0, int x1, uint32_t* tile_counts, uint32_t* totals,
                      cudaStream_t s);
int launch_slab_scatter(const sphb_grid_t& g, int64_t n, int64_t nb, const uint32_t* keys,
                        const int64_t* id, int x0, int x1, const uint32_t* tile_offsets,
                        const float4* posp, const float4* velr, const float4* prev,
                        const int64_t* keep_bases, float4* nposp, float4* nvelr, float4* nprev,
                        int64_t* nid, uint32_t* nkeys, void* send_l, void* send_r,
                        const int64_t* sections, cudaStream_t s);
int launch_slab_unpack(const void* buf, int64_t r0, int64_t cnt, int64_t dst, float4* nposp,
                       float4* nvelr, float4* nprev, int64_t* nid, uint32_t* nkeys,
                       cudaStream_t s);
int64_t band_scratch_words(const sphb_grid_t& g);
int launch_band_count(const sphb_grid_t& g, int width, int sides, const int32_t* beg,
                      const int32_t* end, int32_t* scratch, int64_t* info,
                      const sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_band_pack(const sphb_params_t& p, const sphb_grid_t& g, int width, int sides,
                     const int32_t* beg, const int32_t* end, const int32_t* scratch,
                     const float4* posp_s, const float4* velr_s, const float4* prev_s,
                     const int64_t* id_s, const void* acc, const void* drho, void* send_l,
                     void* send_r, cudaStream_t s);
int launch_band_integrate(sphb_workspace* ws, const sphb_params_t& p, const sphb_grid_t& g,
                          const void* buf, int64_t cnt, int64_t dst, float4* posp, float4* velr,
                          float4* prev, int64_t* id, uint32_t* keys_next, uint32_t* keys_sorted,
                          sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_slab_tail(const sphb_grid_t& g, int32_t* end, int64_t n_next, cudaStream_t s);
int launch_band_put(const sphb_params_t& p, const sphb_grid_t& g, int width, int sides,
                    const int32_t* beg, const int32_t* end, const int32_t* scratch,
                    const float4* posp_s, const float4* velr_s, const float4* prev_s,
                    const int64_t* id_s, const void* acc, const void* drho, void* peer_l,
                    void* peer_r, uint64_t* flag_l, uint64_t* flag_r, uint64_t tag, uint32_t* done,
                    cudaStream_t s);
int launch_band_wait(const uint64_t* flag_l, const uint64_t* flag_r, uint64_t tag, sphb_ctrl_t* ctrl,
                     cudaStream_t s);
int launch_cell_hist(sphb_workspace* ws, const sphb_grid_t& g, const uint32_t* keys, int64_t n,
                     const sphb_ctrl_t* ctrl, cudaStream_t s);
int launch_step_end(sphb_ctrl_t* ctrl, const sphb_params_t& p, sphb_step_record_t* rec, int64_t cap,
                    cudaStream_t s);
int launch_ctrl_init(sphb_ctrl_t* ctrl, int64_t max_steps, double t_end, cudaStream_t s);

int sphb_set_error(int code, const char* fmt, ...);
int sphb_check_launch(const char* what);

// state.cu
int launch_state_unpack(int64_t r0, int64_t cnt, const float* pos, const float* vel,
                        const float* rho, const float* vel_prev, const float* rho_prev,
                        float4* posp, float4* velr, float4* prev, cudaStream_t s);
int launch_state_pack(int64_t r0, int64_t cnt, const float4* posp, const float4* velr,
                      const float4* prev, float* pos, float* vel, float* rho, float* vel_prev,
                      float* rho_prev, cudaStream_t s);
