/*
 * sphb200.h -- C ABI of libsphb200.so, the B200 (sm_100a) SPH step hot path.
 *
 * Drop-in boundary for the reference's step loop (arXiv 1110.3711 re-implementation
 * "sphbench", /root/reference/pkg/src/sphbench).  The reference's plug-in interface is
 * a Python protocol (make_engine(cfg).compute(...), run_simulation(...)); the Python
 * package paper_1110_3711_b200 mirrors that protocol and calls the entry points below
 * through ctypes.  Each entry point names the reference function(s) it replaces.
 *
 * Conventions
 *   - every array argument is a DEVICE pointer owned by the caller (torch tensors);
 *   - every call is stream-ordered on the caller's cudaStream_t, never synchronises,
 *     never allocates after sphb_workspace_create (CUDA-graph capturable);
 *   - return value 0 = SPHB_OK, negative = SPHB_E_*; sphb_last_error() gives a
 *     thread-local message; no C++ exception crosses the ABI;
 *   - physics failures (the reference's DivergenceError, sim.py:22-29, 310-333) are
 *     recorded on the device in sphb_ctrl_t.err (see SPHB_DIV_*) and read by the host
 *     when it chooses to (no per-step host sync).
 *
 * Particle state layout in HBM (structure of float4 arrays, one 16-B load per field):
 *   posp  float4 (x, y, z, w)            w = 0 in the primary arrays; the sorted copy (K3) carries
 *                                        prrho = press / rho^2 (physics.py:124-134)
 *   velr  float4 (vx, vy, vz, rho)
 *   prev  float4 (vx_prev, vy_prev, vz_prev, rho_prev)   Verlet history (sim.py:31-43)
 *   aux   float4 (press, csound, tensil, mass)            derived (physics.py:119-134) + list mass
 *   id    int64
 * Boundary particles occupy [0, nb), fluid [nb, n) (model.py:24-32).
 */
#ifndef SPHB200_H
#define SPHB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sphb_stream_t; /* == cudaStream_t */

enum {
  SPHB_OK = 0,
  SPHB_E_INVALID = -1,  /* contract violation -> ValueError in the shim */
  SPHB_E_CUDA = -2,     /* CUDA runtime error */
  SPHB_E_CAPACITY = -3, /* n / ncells above the workspace capacity */
};

/* Device-side divergence codes; ordered as the reference checks them inside one step:
 * out-of-domain at step start (sim.py:309-314), non-finite forces (328-329), non-finite
 * state (332-333). */
enum {
  SPHB_DIV_LEFT_DOMAIN = 1,
  SPHB_DIV_NONFINITE_FORCES = 2,
  SPHB_DIV_NONFINITE_STATE = 3,
  SPHB_DIV_SLAB_MARGIN = 4, /* X slabs only: a particle moved more than one cell column in one
                               step, beyond the edge bands the neighbours exchange */
  SPHB_DIV_EXCHANGE_TIMEOUT = 5, /* X slabs, peer-memory transport: a neighbour's band did not
                                    arrive within the wait limit */
};

enum { SPHB_FP32 = 0, SPHB_FP64 = 1 };

/* Grid descriptor; cell_size and dims are computed on the host in f64 exactly as
 * grid.py:81-84 / model.py:131-135 do. */
typedef struct {
  double origin[3];     /* params.domain_min */
  double domain_max[3]; /* params.domain_max */
  double cell_size;     /* 2h / n_subdiv */
  int32_t dims[3];      /* max(ceil(extent/cs - 1e-12), 1) */
  int32_t reach;        /* candidate rows per side: gather slowcellsh 1, *half 2 */
  int32_t tx0, tx1;     /* interaction targets restricted to cell columns [tx0, tx1) (X-slab
                           decomposition; the whole grid is [0, dims[0])) */
} sphb_grid_t;

/* Physics constants.  The first twelve are physics.pack_params (physics.py:149-180). */
typedef struct {
  double sup2, h, invh, kc, eta2, alpha, invwdp, c0, rho0, gamma, mass_fluid, mass_boundary;
  double tait_b;                 /* c0^2 rho0 / gamma (model.py:141-143) */
  double g[3];                   /* gravity, applied once per particle (sim.py:223, 245) */
  double cfl, dt_min, dt_max;    /* compute_dt (sim.py:215-232) */
  int32_t verlet_stride;         /* corrector every k steps (sim.py:242) */
  int32_t order;                 /* 0: per row F then B (gather_*_cells, kernels.py:326-418)
                                    1: all F rows then all B rows (gather_fluid_ranges 421-497) */
  int32_t precision;             /* SPHB_FP32 (production) | SPHB_FP64 (bit-exact to reference) */
  /* ---- extensions beyond the reference; the zero values are the
   * reference's behaviour */
  int32_t kernel;                /* SPHB_KERNEL_CUBIC (reference, physics.py:25-33) |
                                    SPHB_KERNEL_WENDLAND (C2, support 2h); kc / invwdp above
                                    are that kernel's normalisation and 1/W(dp) */
  int32_t integrator;            /* SPHB_INT_VERLET (reference, sim.py:235-259) |
                                    SPHB_INT_SYMPLECTIC (two-stage position-Verlet) */
  int32_t counters;              /* SPHB_COUNTERS_GATHER: the gather traversal's StepStats
                                    (gather.py:103-109, cellpairs asymmetric);
                                    SPHB_COUNTERS_SYMMETRIC: run_cells_symmetric's (kernels.py:
                                    121-175, cellpairs.py:92-99): half-stencil candidates,
                                    force_evals = unordered pairs, ff unordered */
  int64_t piston_id0, piston_id1; /* boundary particles with id in [id0, id1) follow the
                                     piston x(t) = x0 + S/2 (1 - cos 2 pi t/T); id0 == id1: none */
  double piston_x0, piston_stroke, piston_period;
  /* repulsive boundary force (Monaghan 1994 Lennard-Jones form), per unit mass, on fluid
   * particles from boundary particles closer than wall_r0 (<= 2h):
   *   a_i += wall_d ((r0/r)^p1 - (r0/r)^p2) r_ij / r^2;  wall_d == 0: none (the reference) */
  double wall_d, wall_r0;
  int32_t wall_p1, wall_p2;
} sphb_params_t;

enum { SPHB_KERNEL_CUBIC = 0, SPHB_KERNEL_WENDLAND = 1 };
enum { SPHB_INT_VERLET = 0, SPHB_INT_SYMPLECTIC = 1 };
enum { SPHB_COUNTERS_GATHER = 0, SPHB_COUNTERS_SYMMETRIC = 1 };
enum { SPHB_PI_GATHER = 0, SPHB_PI_SYMMETRIC = 1, SPHB_PI_PAIRED = 2 };

/* Device-resident control block (one per simulation, caller allocates 256 B). */
typedef struct {
  int64_t step;          /* index of the step about to run / running */
  int64_t max_steps;     /* run_simulation stop rule (sim.py:302-303); <0 = none */
  double t_sim;          /* simulated time so far */
  double t_end;          /* sim.py:304-305; +inf = none */
  double dt;             /* dt of the last completed step */
  uint64_t dtmin_f;      /* ordered bits of min_fluid sqrt(h/|a+g|) of the running step */
  uint64_t dtmin_cv;     /* ordered bits of min_all h/(cs+visc_dt) */
  uint64_t err;          /* (step << 40) | (code << 32) | first offending index; ~0 = none */
  uint64_t counters[4];  /* running step: candidates, ordered hits, evals, ff evals */
  int32_t active;        /* 1 while no error and no stop rule fired */
  uint32_t tile_next[2]; /* dynamic work counters of the interaction launches (reset per step) */
  uint32_t nblk[2];      /* target blocks built for the fluid / boundary interaction passes */
  int32_t pad_;
  double dt_stage;              /* symplectic: the step's dt, fixed by the first stage */
  uint64_t counters_stage[4];   /* symplectic: the first stage's counters (the step's stats) */
} sphb_ctrl_t;

/* Per-step record written at the end of every step (StepStats, model.py:176-212). */
typedef struct {
  double dt;
  uint64_t candidate_pairs, hits_ordered, force_evals, ff_force_evals;
} sphb_step_record_t;

typedef struct sphb_workspace sphb_workspace_t;

const char* sphb_last_error(void);
const char* sphb_version(void);

/* Allocates every internal scratch buffer (radix ping-pong, histograms, scan partials)
 * for up to n_max particles and ncells_max cells.  The only allocating call. */
int sphb_workspace_create(int64_t n_max, int64_t ncells_max, sphb_workspace_t** ws);
int sphb_workspace_destroy(sphb_workspace_t* ws);
/* Zeroes the workspace histogram (needed only after an aborted step). */
int sphb_workspace_reset(sphb_workspace_t* ws, sphb_stream_t s);
/* Rows rewritten from outside (a host upload of the same n rows, e.g. the reference-layout
 * round trip of sphb_state_from_soa): sphb_workspace_clear_hist zeroes the per-cell
 * histogram that sphb_cell_keys then recounts (K7 already counted the device's own keys).
 * sphb_cell_keys marks the previous sort's order as unknown (the next sphb_sort_ranges /
 * sphb_step sorts by radix); sphb_workspace_trust_order, called after it, lets that sort
 * take the movers-only path again.  Valid whenever keys_sorted, beg and end are still those
 * of the previous sort of n rows: the movers-only sort is the stable sort of the current rows
 * in ANY order (a row whose key differs from keys_sorted at its index is a mover; a permuted
 * upload exceeds the mover cap and takes the radix path), and the device re-checks the
 * previous order's consistency before using it (nl.cu, K2' movers-only sort). */
int sphb_workspace_clear_hist(sphb_workspace_t* ws, sphb_stream_t s);
int sphb_workspace_trust_order(sphb_workspace_t* ws, sphb_stream_t s);
/* Movers-only sort threshold of sphb_step (default and maximum min(n_max, 2^20)): a
 * step whose rows changed cell for at most `cap` rows is sorted by counting from the previous
 * order; otherwise (or cap = -1) by the LSD radix sort.  Both give the identical permutation
 * (grid.py:107-109 stable order); the choice is made on the device. */
int sphb_workspace_set_mover_cap(sphb_workspace_t* ws, int64_t cap);
/* Targets per interaction block of the FP32 kernel: 128 (default: 4-warp CTAs, two per SM,
 * <= 2,304 staged candidates), 256 (8-warp CTAs, one per SM, <= 4,224: small systems) or 384 (12-warp CTAs, one per SM, <= 4,608 staged candidates:
 * more resident warps, less screen work per target, fewer idle lanes when cells hold uneven
 * particle counts, e.g. after a dam collapses).
 * Results agree within the FP32 tolerance (accumulation order); FP64 always uses 128. */
int sphb_workspace_set_pi_block(sphb_workspace_t* ws, int32_t targets);
/* The FP32 interaction kernel (FP64 always runs the gather kernel):
 *   SPHB_PI_GATHER     one-sided gather (each ordered pair evaluated by its target, the
 *                      reference's GPU strategy, gather.py:1-10; K6 dt in its epilogue);
 *   SPHB_PI_SYMMETRIC  symmetric pair evaluation (K5s): each unordered pair once over the
 *                      forward half stencil (run_cells_symmetric, kernels.py:121-175), the
 *                      reaction scattered to the partner (eval_scatter, kernels.py:29-68) through
 *                      shared-memory rows flushed with vector reductions; 384-target blocks,
 *                      cell order (order 0) only; dt after the scatter (one extra pass);
 *   SPHB_PI_PAIRED     the gather with two targets per lane (k_interact_v12): 8-warp CTAs on
 *                      512-target bricks, one FIFO of the two targets' union of maybes, pair
 *                      math packed across the two targets; gather semantics and K6 epilogue.
 * Hit sets and counters are identical; forces agree within the FP32 tolerance (summation
 * order).  Counters follow prm->counters either way. */
int sphb_workspace_set_pi_kernel(sphb_workspace_t* ws, int32_t kernel);
/* The last sphb_step sort's path (0 movers-only, 1 radix) and mover count (synchronising
 * read, diagnostics only). */
int sphb_workspace_sort_info(const sphb_workspace_t* ws, int64_t* movers, int32_t* mode);
/* Bytes of device memory the workspace holds. */
int64_t sphb_workspace_bytes(const sphb_workspace_t* ws);

/* Control block reset: step=0, t_sim=0, err=none, active=1, stop rules as given. */
int sphb_ctrl_init(sphb_ctrl_t* ctrl, int64_t max_steps, double t_end, sphb_stream_t s);

/* K1 -- assign_cells (grid.py:77-93): f64-exact cell id per particle, -1 outside.
 * keys_out[i] = (is_fluid << cellbits) | cell (sort key); cell_out[i] = cell or -1;
 * first out-of-domain index recorded in ctrl->err as SPHB_DIV_LEFT_DOMAIN at ctrl->step;
 * per-list per-cell histogram accumulated into the workspace for sphb_cell_ranges. */
int sphb_cell_keys(sphb_workspace_t* ws, const sphb_grid_t* grid, const void* posp, int64_t n,
                   int64_t nb, uint32_t* keys_out, int32_t* cell_out, sphb_ctrl_t* ctrl,
                   sphb_stream_t s);

/* K2 -- the stable per-list argsort of reorder (grid.py:96-109): LSD radix sort of keys.
 * perm_out[new] = old (grid.sort_perm, grid.py:116); keys_sorted_out optional (may be NULL). */
int sphb_sort(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys, int64_t n,
              uint32_t* keys_sorted_out, int32_t* perm_out, const sphb_ctrl_t* ctrl,
              sphb_stream_t s);

/* K2 + K4 of a step (what sphb_step runs): the stable per-list argsort of the keys K7 wrote
 * (grid.py:96-109) and this step's cell ranges (grid.py:123-144).  When the rows are still
 * in the order of the previous sort of this state (keys_sorted, beg, end as that call left
 * them), only the rows whose key changed are placed (counting, no radix pass); otherwise, or
 * beyond the workspace's mover cap, the radix sort runs.  The choice is made and checked on
 * the device; both paths give the identical permutation.  sphb_cell_keys and sphb_sort mark
 * the previous order as unknown. */
int sphb_sort_ranges(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys,
                     int64_t n, uint32_t* keys_sorted, int32_t* perm, int32_t* beg, int32_t* end,
                     const sphb_ctrl_t* ctrl, sphb_stream_t s);

/* K1 + K2 + K4 in one call (SURVEY.md §8(b)'s sphb_nl_build): cell keys of the rows as they
 * are, the stable per-list permutation (radix) and both lists' per-cell [beg, end).  The
 * first out-of-domain row is recorded in ctrl->err (SPHB_DIV_LEFT_DOMAIN) and the step's
 * later kernels skip.  Equivalent to sphb_cell_keys, sphb_sort, sphb_cell_ranges. */
int sphb_nl_build(sphb_workspace_t* ws, const sphb_grid_t* grid, const void* posp, int64_t n,
                  int64_t nb, uint32_t* keys_out, uint32_t* keys_sorted_out, int32_t* perm_out,
                  int32_t* beg, int32_t* end, sphb_ctrl_t* ctrl, sphb_stream_t s);

/* K3 -- reorder gathers (grid.py:111-114) fused with compute_derived (physics.py:96-110):
 * *_out[i] = *_in[perm[i]] for posp, velr, prev, id; posp_out.w = prrho; aux_out = (press,
 * csound, tensil, list mass);
 * cell_out[i] = cell of the sorted key.  prev_in/prev_out/id may be NULL; aux_out may be NULL
 * when the interaction that follows is an FP32 gather / paired build (they recompute a
 * target's row with this kernel's arithmetic: sphb_step skips the aux pass then).
 * The derived values are the reference's (f64 pow, f32-rounded, bit-identical) for
 * prm->precision == SPHB_FP64; SPHB_FP32 with gamma = 7 evaluates (rho/rho0)^7 and ^3 by
 * multiplication (press / csound within 1 f32 ulp; the FP32 force tolerance is 1e-5). */
int sphb_reorder(const sphb_params_t* prm, const sphb_grid_t* grid, int64_t n,
                 const int32_t* perm, const uint32_t* keys_sorted, const void* posp_in,
                 const void* velr_in, const void* prev_in, const int64_t* id_in, void* posp_out,
                 void* velr_out, void* prev_out, int64_t* id_out, void* aux_out,
                 int32_t* cell_out, const sphb_ctrl_t* ctrl, sphb_stream_t s);

/* The per-list per-cell histogram of sort keys that are already known (e.g. carried through a
 * slab exchange), accumulated into the workspace for sphb_cell_ranges / sphb_sort_ranges. */
int sphb_cell_hist(sphb_workspace_t* ws, const sphb_grid_t* grid, const uint32_t* keys, int64_t n,
                   const sphb_ctrl_t* ctrl, sphb_stream_t s);

/* K4 -- build_cell_index (grid.py:123-144): warp-level exclusive scan of the per-list
 * histogram from sphb_cell_keys.  beg/end hold 2*ncells int32: [0,ncells) boundary list,
 * [ncells, 2*ncells) fluid list already offset by nb; empty cells carry the running prefix.
 * Re-zeroes the histogram for the next step. */
int sphb_cell_ranges(sphb_workspace_t* ws, const sphb_grid_t* grid, int32_t* beg, int32_t* end,
                     const sphb_ctrl_t* ctrl, sphb_stream_t s);

/* Same table from an already sorted cell array (no histogram needed), for frames whose NL
 * ran elsewhere (engine.compute parity mode). cell_sorted[i] in [0, ncells). */
int sphb_cell_ranges_from_sorted(sphb_workspace_t* ws, const sphb_grid_t* grid,
                                 const int32_t* cell_sorted, int64_t n, int64_t nb, int32_t* beg,
                                 int32_t* end, sphb_stream_t s);

/* Force buffers (acc, drho, visc) of sphb_interact / sphb_integrate* / sphb_step.  Callers
 * size them for the FP64 layout (24 + 8 + 8 B per particle); what is stored depends on
 * prm->precision:
 *   SPHB_FP64  the ForceOutput layout (config.py:94-103): acc (n,3) f64 (boundary rows 0),
 *              drho (n) f64, visc (n) f64 -- bit-identical to the reference;
 *   SPHB_FP32  acc holds one float4 (ax, ay, az, drho) per particle, visc one float per
 *              particle; drho is unused (may be NULL).  20 B per particle written by PI and
 *              16 B read by K7; sphb_forces_f64 widens it (exactly) to the FP64 layout. */

/* The block list of the next sphb_interact (the interaction's work decomposition: k_blocks and
 * the FP32 gather builds' candidate counter) built from the cell ranges on the workspace's own
 * high-priority stream, forked from s -- call it after the ranges (sphb_sort_ranges) and
 * before K3 (sphb_reorder), so it runs while K3 moves the rows.  The next sphb_interact with
 * the same beg / end, grid window and build waits for it instead of building it (sphb_step
 * does this internally).  Optional: without it sphb_interact builds the list itself.  A plan
 * belongs to the step's own sphb_interact (call them in pairs); sphb_workspace_reset drops a
 * pending one. */
int sphb_interact_plan(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                       const int32_t* beg, const int32_t* end, sphb_ctrl_t* ctrl, sphb_stream_t s);

/* K5/K5b/K6 -- GatherEngine.compute (engines/gather.py:42-110): fused fluid pass
 * (gather_fluid_cells / _ranges, kernels.py:326-497) and boundary pass (gather_boundary_*,
 * kernels.py:500-596), plus the compute_dt reductions (sim.py:215-232) in the epilogue.
 * Raw counters and the two dt minima accumulate into ctrl.  aux may be NULL for the FP32
 * gather / paired builds (not for SPHB_FP64 or the symmetric build). */
int sphb_interact(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                  int64_t n, int64_t nb,
                  const void* posp, const void* velr, const void* aux, const int32_t* cell_sorted,
                  const int32_t* beg, const int32_t* end, void* acc, void* drho, void* visc,
                  sphb_ctrl_t* ctrl, sphb_stream_t s);

/* The force buffers of prm->precision widened to the ForceOutput layout (f64 acc (n,3), drho,
 * visc), rows [0, n); the FP32 -> f64 conversion is exact.  (gather.py:103-110 returns f64.) */
int sphb_forces_f64(const sphb_params_t* prm, int64_t n, const void* acc, const void* drho,
                    const void* visc, double* acc64, double* drho64, double* visc64,
                    sphb_stream_t s);

/* Resets the per-step accumulators (dt minima, counters) and evaluates the stop rules. */
int sphb_step_begin(sphb_ctrl_t* ctrl, sphb_stream_t s);

/* K7 -- compute_dt finalize + verlet_update (sim.py:215-259) fused with the next step's
 * assign_cells (K1) and its histogram; writes the integrated state back into the primary
 * (unsorted-for-next-step) arrays.  Flags non-finite state / out-of-domain in ctrl. */
int sphb_integrate(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                   int64_t n, int64_t nb, const void* posp_s, const void* velr_s,
                   const void* prev_s, const int64_t* id_s, const void* acc, const void* drho,
                   void* posp, void* velr, void* prev, int64_t* id, uint32_t* keys_next,
                   sphb_ctrl_t* ctrl, sphb_stream_t s);

/* Symplectic integrator (params.integrator == SPHB_INT_SYMPLECTIC), replacing
 * sphb_integrate: stage 0 (predictor, after the step's first interaction) fixes the step's
 * dt and counters in ctrl and writes the half-step state r* = r + dt/2 v, v* = v + dt/2 (a+g),
 * rho* = rho + dt/2 drho with (v, rho) kept in prev; stage 1 (corrector, after the second
 * interaction on the half-step state) writes v' = v + dt (a*+g), r' = r* + dt/2 v',
 * rho' = rho + dt drho*.  Both fuse the next assign_cells like sphb_integrate; piston
 * particles follow their law at t + dt/2 and t + dt. */
int sphb_integrate_stage(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                         int64_t n, int64_t nb, int32_t stage, const void* posp_s,
                         const void* velr_s, const void* prev_s, const int64_t* id_s,
                         const void* acc, const void* drho, void* posp, void* velr,
                         void* prev, int64_t* id, uint32_t* keys_next, sphb_ctrl_t* ctrl,
                         sphb_stream_t s);

/* The reference's state layout <-> the step's rows (rows [r0, r0 + cnt)).  pos / vel /
 * vel_prev are (n, 3) f32 row-major, rho / rho_prev (n,) f32: ParticleSystem.pos/vel/rho
 * (model.py:25-43) and VerletState.vel_prev/rho_prev (sim.py:31-43), as device copies of the
 * caller's host arrays (52 B per particle with the int64 ids, which the step uses as they
 * are).  posp.w is written 0 (the step derives prrho itself). */
int sphb_state_from_soa(int64_t r0, int64_t cnt, const float* pos, const float* vel,
                        const float* rho, const float* vel_prev, const float* rho_prev,
                        void* posp, void* velr, void* prev, sphb_stream_t s);
int sphb_state_to_soa(int64_t r0, int64_t cnt, const void* posp, const void* velr,
                      const void* prev, float* pos, float* vel, float* rho, float* vel_prev,
                      float* rho_prev, sphb_stream_t s);

/* The reference's module-level step functions on the caller's own arrays (device pointers),
 * for loops that keep the reference's structure:
 *   sphb_build_ranges  build_ranges (grid.py:170-200) from one list's begin/end (int32, ncells
 *                      = nx ny nz): range_begin/range_end (ncells, (2n+1)^2) int64 row-major;
 *   sphb_dt_terms      the two minima of compute_dt (sim.py:215-232) as f64 bit patterns in
 *                      out2[0] (fluid force term) / out2[1] (sound + viscosity term); out2 must
 *                      hold +inf bits on entry; the cfl product and clamp stay with the caller;
 *   sphb_verlet_soa    verlet_update (sim.py:235-259) in place on pos/vel (n, 3), rho (n,)
 *                      and the history vel_prev (n, 3) / rho_prev (n,), bit-identical. */
int sphb_build_ranges(const int32_t* beg, const int32_t* end, int32_t nx, int32_t ny, int32_t nz,
                      int32_t n_subdiv, int64_t* range_begin, int64_t* range_end,
                      sphb_stream_t s);
int sphb_dt_terms(const sphb_params_t* prm, int64_t n, int64_t nb, const double* accel,
                  const double* visc_dt, const float* csound, uint64_t* out2, sphb_stream_t s);
int sphb_verlet_soa(const sphb_params_t* prm, int64_t n, int64_t nb, int32_t corrector, double dt,
                    float* pos, float* vel, float* rho, float* vel_prev, float* rho_prev,
                    const double* accel, const double* drho_dt, sphb_stream_t s);

/* Energy diagnostics (SURVEY.md §8(d) functional, no reference counterpart): out[0..4] =
 * KE (fluid), PE = sum m |g| z (fluid), IE = sum m (u(rho) - u(rho0)) with the Tait internal
 * energy u(rho) = B/(gamma-1) rho^(gamma-1)/rho0^gamma + B/rho (all particles), mean fluid rho,
 * mean rho.  f64, deterministic (fixed-order two-pass reduction).  velr rows (vx,vy,vz,rho),
 * posp rows (x,y,z,*); boundary rows first.  out is a device pointer to 5 doubles. */
int sphb_energy(sphb_workspace_t* ws, const sphb_params_t* prm, int64_t n, int64_t nb,
                const void* posp, const void* velr, double* out, sphb_stream_t s);

/* ---- X-slab exchange: device-resident migration + halo packing.
 * Replaces the exchange phases of a slab decomposition of run_simulation's loop (the reference
 * has no multi-device path; its Slices geometry is engines/kernels.py:230-323).  After the
 * system update, a rank's primary arrays (owned rows + last step's halo rows with id < 0, sort
 * keys from sphb_integrate) are classified by cell column against its slab [x0, x1) into 10
 * categories c = 2 kind + list (kind 0 keep, 1 migrate left, 2 migrate right, 3 halo left,
 * 4 halo right; list 0 boundary, 1 fluid); halo = kept rows within grid->reach columns of an
 * edge.  Last step's halo rows are dropped. */
int64_t sphb_slab_tiles(int64_t n); /* tile_counts holds 10 * sphb_slab_tiles(n) uint32 */
/* per-tile category counts, their exclusive scan (in place) and the 10 totals (device). */
int sphb_slab_count(const sphb_grid_t* grid, int64_t n, int64_t nb, const uint32_t* keys,
                    const int64_t* id, int32_t x0, int32_t x1, uint32_t* tile_counts,
                    uint32_t* totals, sphb_stream_t s);
/* kept rows -> next arrays at keep_bases[list] + rank; migrants / halo copies (id' = -1 - id)
 * -> packed 64-B rows (float4 posp, velr, prev, int64 id, pad) in send_l / send_r with sections
 * [mig B | mig F | halo B | halo F]; sections = {l_migF, l_haloB, l_haloF, r_migF, r_haloB,
 * r_haloF} start rows.  keep_bases and sections are host arrays. */
int sphb_slab_scatter(const sphb_grid_t* grid, int64_t n, int64_t nb, const uint32_t* keys,
                      const int64_t* id, int32_t x0, int32_t x1, const uint32_t* tile_offsets,
                      const void* posp, const void* velr, const void* prev,
                      const int64_t* keep_bases, void* nposp, void* nvelr, void* nprev,
                      int64_t* nid, uint32_t* nkeys, void* send_l, void* send_r,
                      const int64_t* sections, sphb_stream_t s);
/* rows [r0, r0 + cnt) of a received packed buffer -> next arrays rows [dst, dst + cnt).
 * The packed rows carry the sender's sort keys: with nkeys (and nkeys of the scatter) the next
 * step needs no K1, only sphb_cell_hist on those keys. */
int sphb_slab_unpack(const void* buf, int64_t r0, int64_t cnt, int64_t dst, void* nposp,
                     void* nvelr, void* nprev, int64_t* nid, uint32_t* nkeys, sphb_stream_t s);

/* ---- X-slab edge bands: the per-step exchange with rows kept in place (dslab.DeviceSlabSim).
 * A slab grid (tx0 > 0 or tx1 < dims[0]) sorts with one extra bin after the two lists, so its
 * begin/end tables hold 2 ncells + 1 entries: rows that left the slab and last step's halo
 * copies get the dead key from sphb_integrate and sort to the tail; the live rows are the
 * first end[2 ncells - 1].  Per step, after NL: sphb_band_count sizes the edge bands (the
 * `width` = reach + 1 edge columns on each side with a neighbour, `sides` bit 0 left, bit 1
 * right) and writes info[8] = {live rows, boundary rows, band rows left, band rows right,
 * error word, active, step, 0} (device; the host reads it while the interaction runs).
 * After the edge targets' interaction, sphb_band_pack writes each band row's sorted state and
 * forces (SPHB_BAND_ROW_BYTES each) into the side's send buffer; they travel while the
 * interior targets run.  The receiver's sphb_band_integrate applies the step's update with
 * sphb_integrate's arithmetic and dt to a received buffer, appends the rows at [dst, dst +
 * cnt) and classifies them by their new column: inside the slab -> owned (migrants), within
 * reach columns outside -> halo copies (id' = -1 - id), else dead.  sphb_slab_tail then sets
 * the dead bin's end to the next step's row count.  scratch holds
 * sphb_band_scratch_words(grid) int32 (device). */
#define SPHB_BAND_ROW_BYTES 96
int64_t sphb_band_scratch_words(const sphb_grid_t* grid);
int sphb_band_count(const sphb_grid_t* grid, int32_t width, int32_t sides, const int32_t* beg,
                    const int32_t* end, int32_t* scratch, int64_t* info, const sphb_ctrl_t* ctrl,
                    sphb_stream_t s);
int sphb_band_pack(const sphb_params_t* prm, const sphb_grid_t* grid, int32_t width,
                   int32_t sides, const int32_t* beg, const int32_t* end, const int32_t* scratch,
                   const void* posp_s, const void* velr_s, const void* prev_s,
                   const int64_t* id_s, const void* acc, const void* drho, void* send_l,
                   void* send_r, sphb_stream_t s);
int sphb_band_integrate(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid,
                        const void* buf, int64_t cnt, int64_t dst, void* posp, void* velr,
                        void* prev, int64_t* id, uint32_t* keys_next, uint32_t* keys_sorted,
                        sphb_ctrl_t* ctrl, sphb_stream_t s);
int sphb_slab_tail(const sphb_grid_t* grid, int32_t* end, int64_t n_next, sphb_stream_t s);
/* Peer-memory transport of the edge bands (NVLink P2P stores; one kernel packs AND sends):
 * sphb_band_put is sphb_band_pack writing each side's rows straight into the neighbour's
 * receive buffer (peer_l / peer_r: device pointers of the neighbours' memory, CUDA IPC), then --
 * every block's stores fenced at system scope, the last block elected through `done` (a
 * device uint32, zero between launches) -- stores `tag` into the neighbours' flag words
 * (peer_flag_l / _r, release, system scope).  sphb_band_wait makes the stream wait until this
 * rank's own flag words (flag_l / flag_r, NULL = no neighbour) reach `tag` (acquire, system
 * scope); after ~10 s it records SPHB_DIV_EXCHANGE_TIMEOUT in ctrl and returns. */
int sphb_band_put(const sphb_params_t* prm, const sphb_grid_t* grid, int32_t width, int32_t sides,
                  const int32_t* beg, const int32_t* end, const int32_t* scratch,
                  const void* posp_s, const void* velr_s, const void* prev_s, const int64_t* id_s,
                  const void* acc, const void* drho, void* peer_l, void* peer_r,
                  uint64_t* peer_flag_l, uint64_t* peer_flag_r, uint64_t tag, uint32_t* done,
                  sphb_stream_t s);
int sphb_band_wait(const uint64_t* flag_l, const uint64_t* flag_r, uint64_t tag, sphb_ctrl_t* ctrl,
                   sphb_stream_t s);

/* Closes the step: dt/counters into rec[step % rec_capacity], t_sim += dt, step += 1. */
int sphb_step_end(sphb_ctrl_t* ctrl, const sphb_params_t* prm, sphb_step_record_t* rec,
                  int64_t rec_capacity, sphb_stream_t s);

/* One whole NL -> PI -> SU step on resident state (the run_simulation loop body,
 * sim.py:306-351).  Composes the calls above; graph-capturable. */
typedef struct {
  void *posp, *velr, *prev;      /* primary state (this step's pre-sort order) */
  int64_t* id;
  void *posp_s, *velr_s, *prev_s, *aux; /* sorted copies */
  int64_t* id_s;
  uint32_t *keys, *keys_sorted;
  int32_t *perm, *cell_s, *beg, *end;
  void *acc, *drho, *visc;       /* force buffers, layout of prm->precision (above) */
} sphb_state_t;

int sphb_step(sphb_workspace_t* ws, const sphb_params_t* prm, const sphb_grid_t* grid, int64_t n,
              int64_t nb, const sphb_state_t* st, sphb_ctrl_t* ctrl, sphb_step_record_t* rec,
              int64_t rec_capacity, sphb_stream_t s);

/* Number of this library's kernel launches one sphb_step issues (for the bench's
 * gpu_launches claim). */
int64_t sphb_step_launch_count(const sphb_grid_t* grid, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* SPHB200_H */
