/*
 * sph_oracle.c -- CPU ORACLE (test infrastructure only; never on the product path).
 *
 * Plain-C restatement of the reference's particle-interaction hot loop so the
 * CUDA path can be checked (and the reference CPU path timed) on a box where
 * /root/reference does not exist.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load this library.
 *
 * Pinned against golden vectors produced by running the unmodified reference
 * (tests/golden/make_golden.py); tests/test_oracle.py asserts bit equality.
 *
 * Arithmetic contract (why bit-exactness with numba holds):
 *   - the reference kernels are numba @njit without fastmath: IEEE binary64,
 *     no FMA contraction.  This file is compiled with
 *     -O2 -ffp-contract=off -fno-fast-math so gcc emits the same operations;
 *   - every expression below keeps the reference's left-to-right evaluation
 *     order (Python operator associativity);
 *   - pow() comes from the same libm numba links against.
 *
 * Reference functions restated (file:line under /root/reference/pkg/src/sphbench):
 *   eos_press_scalar   physics.py:119-121
 *   derive_scalar      physics.py:124-134
 *   _derived_pass      physics.py:137-146
 *   pair_eval          physics.py:183-220
 *   load_side          physics.py:223-244
 *   gather_fluid_cells     engines/kernels.py:326-418
 *   gather_fluid_ranges    engines/kernels.py:421-497  (order=1: all fluid rows, then boundary rows)
 *   gather_boundary_cells  engines/kernels.py:500-555
 *   counter normalisation  engines/gather.py:103-109 (done by the Python caller)
 *   eval_scatter           engines/kernels.py:29-68
 *   scan_block (lanes=1)   engines/kernels.py:71-118 (lanes=4 evaluates the same pairs in the
 *                          same order, only delayed within the block: identical sums)
 *   run_cells_symmetric    engines/kernels.py:121-175
 *   run_cells_asymmetric   engines/kernels.py:178-223
 *   symmetric threading    engines/cellpairs.py:132-164 + balance.py:12-43 (private buffers,
 *                          cyclic blocks of cells, merged in thread order)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* packed constants, physics.py:149-162 */
enum { PP_SUP2 = 0, PP_H, PP_INVH, PP_KC, PP_ETA2, PP_ALPHA, PP_INVWDP, PP_C0,
       PP_RHO0, PP_GAMMA, PP_MASSF, PP_MASSB, PP_LEN };

static inline float eos_press_scalar(double rho, double tait_b, double rho0, double gamma) {
  return (float)(tait_b * (pow(rho / rho0, gamma) - 1.0));
}

static inline void derive_scalar(double press, double rho, double c0, double rho0, double gamma,
                                 float* prrho, float* csound, float* tensil) {
  double inv_rho2 = 1.0 / (rho * rho);
  *prrho = (float)(press * inv_rho2);
  *csound = (float)(c0 * pow(rho / rho0, (gamma - 1.0) * 0.5));
  if (press > 0.0)
    *tensil = (float)(0.01 * press * inv_rho2);
  else
    *tensil = (float)(-0.2 * press * inv_rho2);
}

void oracle_derived(int64_t n, const float* rho32, double tait_b, double rho0, double c0,
                    double gamma, float* press, float* csound, float* prrho, float* tensil) {
  for (int64_t i = 0; i < n; ++i) {
    double r = (double)rho32[i];
    float p32 = eos_press_scalar(r, tait_b, rho0, gamma);
    press[i] = p32;
    derive_scalar((double)p32, r, c0, rho0, gamma, &prrho[i], &csound[i], &tensil[i]);
  }
}

typedef struct {
  double x, y, z, vx, vy, vz, rh, pr, cs, te;
} side_t;

typedef struct {
  const float *pos, *vel, *rho, *press, *prrho, *csound, *tensil;
  const double* pp;
  int dmode;
} state_t;

static inline void load_side(const state_t* s, int64_t j, side_t* o) {
  o->x = (double)s->pos[3 * j + 0];
  o->y = (double)s->pos[3 * j + 1];
  o->z = (double)s->pos[3 * j + 2];
  o->vx = (double)s->vel[3 * j + 0];
  o->vy = (double)s->vel[3 * j + 1];
  o->vz = (double)s->vel[3 * j + 2];
  o->rh = (double)s->rho[j];
  if (s->dmode == 0) {
    o->pr = (double)s->prrho[j];
    o->cs = (double)s->csound[j];
    o->te = (double)s->tensil[j];
  } else {
    float pr32, cs32, te32;
    derive_scalar((double)s->press[j], o->rh, s->pp[PP_C0], s->pp[PP_RHO0], s->pp[PP_GAMMA],
                  &pr32, &cs32, &te32);
    o->pr = (double)pr32;
    o->cs = (double)cs32;
    o->te = (double)te32;
  }
}

/* physics.py:183-220 -- operation order kept exactly */
static inline void pair_eval(double dx, double dy, double dz, double r2, double dvx, double dvy,
                             double dvz, double rho_i, double rho_j, double prrho_i, double prrho_j,
                             double cs_i, double cs_j, double ten_i, double ten_j, const double* pp,
                             double* fx, double* fy, double* fz, double* drc, double* mu_abs) {
  double r = sqrt(r2);
  double q = r * pp[PP_INVH];
  double kc = pp[PP_KC];
  double wab, dwdq;
  if (q < 1.0) {
    wab = kc * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
    dwdq = kc * (2.25 * q - 3.0) * q;
  } else {
    double t = 2.0 - q;
    wab = 0.25 * kc * t * t * t;
    dwdq = -0.75 * kc * t * t;
  }
  double gc = dwdq * pp[PP_INVH] / r;
  double dot_vr = dvx * dx + dvy * dy + dvz * dz;
  double mu = pp[PP_H] * dot_vr / (r2 + pp[PP_ETA2]);
  double visc = 0.0;
  if (dot_vr < 0.0) visc = -pp[PP_ALPHA] * (0.5 * (cs_i + cs_j)) * mu / (0.5 * (rho_i + rho_j));
  double tw = wab * pp[PP_INVWDP];
  double tw2 = tw * tw;
  double pterm = prrho_i + prrho_j + visc + (ten_i + ten_j) * tw2 * tw2;
  *fx = pterm * gc * dx;
  *fy = pterm * gc * dy;
  *fz = pterm * gc * dz;
  *drc = gc * dot_vr;
  *mu_abs = fabs(mu);
}

typedef struct {
  double ax, ay, az, dr, vd;
  int64_t cand, tru, evals, ff;
} acc_t;

/* inner j-loop over one contiguous candidate range; `fluid_list` selects the
 * skip-self rule and the ff counter (kernels.py:368-412) */
static inline void scan_range(const state_t* s, const side_t* si, int64_t i, int64_t j0, int64_t j1,
                              int fluid_list, double mass_j, double sup2, acc_t* a) {
  const double* pp = s->pp;
  for (int64_t j = j0; j < j1; ++j) {
    if (fluid_list && j == i) continue;
    a->cand += 1;
    double dx = si->x - (double)s->pos[3 * j + 0];
    double dy = si->y - (double)s->pos[3 * j + 1];
    double dz = si->z - (double)s->pos[3 * j + 2];
    double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 < sup2 && r2 > 0.0) {
      a->tru += 1;
      a->evals += 1;
      if (fluid_list) a->ff += 1;
      side_t sj;
      load_side(s, j, &sj);
      double fx, fy, fz, drc, mu;
      pair_eval(dx, dy, dz, r2, si->vx - sj.vx, si->vy - sj.vy, si->vz - sj.vz, si->rh, sj.rh,
                si->pr, sj.pr, si->cs, sj.cs, si->te, sj.te, pp, &fx, &fy, &fz, &drc, &mu);
      a->ax -= mass_j * fx;
      a->ay -= mass_j * fy;
      a->az -= mass_j * fz;
      a->dr += mass_j * drc;
      if (mu > a->vd) a->vd = mu;
    }
  }
}

/*
 * One gather pass.  Items [i_lo, i_hi) are fluid items when fluid_items != 0
 * (F-F then F-B per row), boundary items otherwise (fluid rows only, drho and
 * visc only).  order: 0 = per-row interleaving (gather_*_cells),
 * 1 = all fluid rows then all boundary rows (gather_fluid_ranges).
 * counters_out[4] = raw (cand, true, evals, ff) summed over items.  target_mask (may be
 * NULL) restricts the items (X-slab decomposition tests: owned targets only).
 */
void oracle_gather_pass(int fluid_items, int order, int64_t i_lo, int64_t i_hi, int reach,
                        const int64_t* cell_of, int64_t nx, int64_t ny, int64_t nz,
                        const int64_t* fbeg, const int64_t* fend, const int64_t* bbeg,
                        const int64_t* bend, int dmode, const float* pos, const float* vel,
                        const float* rho, const float* press, const float* prrho,
                        const float* csound, const float* tensil, const double* pp, double* acc,
                        double* drho, double* viscdt, int64_t* counters_out, int nthreads,
                        const uint8_t* target_mask) {
  state_t s = {pos, vel, rho, press, prrho, csound, tensil, pp, dmode};
  const double sup2 = pp[PP_SUP2], massf = pp[PP_MASSF], massb = pp[PP_MASSB];
  const int64_t nxy = nx * ny;
  int64_t c_cand = 0, c_true = 0, c_eval = 0, c_ff = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : c_cand, c_true, c_eval, c_ff)
#endif
  for (int64_t i = i_lo; i < i_hi; ++i) {
    if (target_mask && !target_mask[i]) continue; /* not a target of this slab */
    side_t si;
    load_side(&s, i, &si);
    acc_t a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0, 0};
    int64_t c = cell_of[i];
    int64_t cz = c / nxy;
    int64_t rem = c - cz * nxy;
    int64_t cy = rem / nx;
    int64_t cx = rem - cy * nx;
    int64_t xlo = cx - reach > 0 ? cx - reach : 0;
    int64_t xhi = cx + reach < nx - 1 ? cx + reach : nx - 1;
    int passes = (fluid_items && order == 1) ? 2 : 1;
    for (int pass = 0; pass < passes; ++pass) {
      for (int64_t dz = -reach; dz <= reach; ++dz) {
        int64_t zz = cz + dz;
        if (zz < 0 || zz >= nz) continue;
        for (int64_t dy = -reach; dy <= reach; ++dy) {
          int64_t yy = cy + dy;
          if (yy < 0 || yy >= ny) continue;
          int64_t base = nx * (yy + ny * zz);
          int do_fluid = (order == 0) || (pass == 0);
          int do_bound = fluid_items && ((order == 0) || (pass == 1));
          if (do_fluid)
            scan_range(&s, &si, fluid_items ? i : -1, fbeg[xlo + base], fend[xhi + base], 1, massf,
                       sup2, &a);
          if (do_bound)
            scan_range(&s, &si, -1, bbeg[xlo + base], bend[xhi + base], 0, massb, sup2, &a);
        }
      }
    }
    if (!fluid_items) a.ff = 0; /* boundary items never count ff (kernels.py:555) */
    if (fluid_items) {
      acc[3 * i + 0] = a.ax;
      acc[3 * i + 1] = a.ay;
      acc[3 * i + 2] = a.az;
    }
    drho[i] = a.dr;
    viscdt[i] = a.vd;
    c_cand += a.cand;
    c_true += a.tru;
    c_eval += a.evals;
    c_ff += a.ff;
  }
  counters_out[0] = c_cand;
  counters_out[1] = c_true;
  counters_out[2] = c_eval;
  counters_out[3] = c_ff;
}

/* ---------------------------------------------------------------- cell-pair engines */
typedef struct {
  int64_t cand, tru, evals, ff;
} cnt_t;

/* kernels.py:29-68: pair (i, j) evaluated once, scattered to i and (both) to j */
static inline void eval_scatter(const state_t* s, int64_t i, int64_t j, int both, int64_t nb,
                                double* acc, double* drho, double* viscdt, cnt_t* c) {
  const double* pp = s->pp;
  side_t si, sj;
  load_side(s, i, &si);
  load_side(s, j, &sj);
  double dx = si.x - sj.x;
  double dy = si.y - sj.y;
  double dz = si.z - sj.z;
  double r2 = dx * dx + dy * dy + dz * dz;
  double fx, fy, fz, drc, mu;
  pair_eval(dx, dy, dz, r2, si.vx - sj.vx, si.vy - sj.vy, si.vz - sj.vz, si.rh, sj.rh, si.pr,
            sj.pr, si.cs, sj.cs, si.te, sj.te, pp, &fx, &fy, &fz, &drc, &mu);
  double mi = i < nb ? pp[PP_MASSB] : pp[PP_MASSF];
  double mj = j < nb ? pp[PP_MASSB] : pp[PP_MASSF];
  if (i >= nb) {
    acc[3 * i + 0] -= mj * fx;
    acc[3 * i + 1] -= mj * fy;
    acc[3 * i + 2] -= mj * fz;
  }
  drho[i] += mj * drc;
  if (mu > viscdt[i]) viscdt[i] = mu;
  c->evals += 1;
  if (i >= nb && j >= nb) c->ff += 1;
  if (both) {
    if (j >= nb) {
      acc[3 * j + 0] += mi * fx;
      acc[3 * j + 1] += mi * fy;
      acc[3 * j + 2] += mi * fz;
    }
    drho[j] += mi * drc;
    if (mu > viscdt[j]) viscdt[j] = mu;
  }
}

/* kernels.py:71-118 with lanes == 1 */
static inline void scan_block(const state_t* s, int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                              int ordered, int skip_self, int both, int64_t nb, double* acc,
                              double* drho, double* viscdt, cnt_t* c) {
  const double sup2 = s->pp[PP_SUP2];
  for (int64_t i = i0; i < i1; ++i) {
    double xi = (double)s->pos[3 * i + 0], yi = (double)s->pos[3 * i + 1],
           zi = (double)s->pos[3 * i + 2];
    int64_t js = ordered ? i + 1 : j0;
    for (int64_t j = js; j < j1; ++j) {
      if (skip_self && j == i) continue;
      c->cand += 1;
      double dx = xi - (double)s->pos[3 * j + 0];
      double dy = yi - (double)s->pos[3 * j + 1];
      double dz = zi - (double)s->pos[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 < sup2 && r2 > 0.0) {
        c->tru += 1;
        eval_scatter(s, i, j, both, nb, acc, drho, viscdt, c);
      }
    }
  }
}

/* kernels.py:121-175 (symmetric) / 178-223 (asymmetric) over cells[0..ncl) */
static void run_cells(const state_t* s, int symmetric, const int64_t* cells, int64_t ncl,
                      int64_t nx, int64_t ny, int64_t nz, int reach, const int64_t* fbeg,
                      const int64_t* fend, const int64_t* bbeg, const int64_t* bend, int64_t nb,
                      double* acc, double* drho, double* viscdt, cnt_t* c) {
  const int64_t nxy = nx * ny;
  for (int64_t t = 0; t < ncl; ++t) {
    int64_t cc = cells[t];
    int64_t cz = cc / nxy, rem = cc - cz * (nx * ny), cy = rem / nx, cx = rem - cy * nx;
    int64_t cf0 = fbeg[cc], cf1 = fend[cc], cb0 = bbeg[cc], cb1 = bend[cc];
    if (cf1 == cf0 && cb1 == cb0) continue;
    if (symmetric) {
      scan_block(s, cf0, cf1, cf0, cf1, 1, 0, 1, nb, acc, drho, viscdt, c);
      scan_block(s, cf0, cf1, cb0, cb1, 0, 0, 1, nb, acc, drho, viscdt, c);
      for (int64_t dz = 0; dz <= reach; ++dz) {
        int64_t zz = cz + dz;
        if (zz >= nz) continue;
        for (int64_t dy = dz > 0 ? -reach : 0; dy <= reach; ++dy) {
          int64_t yy = cy + dy;
          if (yy < 0 || yy >= ny) continue;
          for (int64_t dxo = (dz > 0 || dy > 0) ? -reach : 1; dxo <= reach; ++dxo) {
            int64_t xx = cx + dxo;
            if (xx < 0 || xx >= nx) continue;
            int64_t d = xx + nx * (yy + ny * zz);
            scan_block(s, cf0, cf1, fbeg[d], fend[d], 0, 0, 1, nb, acc, drho, viscdt, c);
            scan_block(s, cf0, cf1, bbeg[d], bend[d], 0, 0, 1, nb, acc, drho, viscdt, c);
            scan_block(s, cb0, cb1, fbeg[d], fend[d], 0, 0, 1, nb, acc, drho, viscdt, c);
          }
        }
      }
    } else {
      int64_t xlo = cx - reach > 0 ? cx - reach : 0;
      int64_t xhi = cx + reach < nx - 1 ? cx + reach : nx - 1;
      for (int64_t dz = -reach; dz <= reach; ++dz) {
        int64_t zz = cz + dz;
        if (zz < 0 || zz >= nz) continue;
        for (int64_t dy = -reach; dy <= reach; ++dy) {
          int64_t yy = cy + dy;
          if (yy < 0 || yy >= ny) continue;
          int64_t base = nx * (yy + ny * zz);
          int64_t jf0 = fbeg[xlo + base], jf1 = fend[xhi + base];
          int64_t jb0 = bbeg[xlo + base], jb1 = bend[xhi + base];
          scan_block(s, cf0, cf1, jf0, jf1, 0, 1, 0, nb, acc, drho, viscdt, c);
          scan_block(s, cf0, cf1, jb0, jb1, 0, 0, 0, nb, acc, drho, viscdt, c);
          scan_block(s, cb0, cb1, jf0, jf1, 0, 0, 0, nb, acc, drho, viscdt, c);
        }
      }
    }
  }
}

/*
 * CellPairsEngine.compute (cellpairs.py:41-90) for threading "single" (nthreads_logical <= 1:
 * all cells in order into the outputs) and "symmetric" (nthreads_logical = T: blocks of
 * block_of_cells cells dealt cyclically to T private accumulators, merged in thread order --
 * bit-identical to the reference at the same T).  cells_mask (may be NULL) restricts the
 * traversal to a subset of cells (bounded CPU-baseline samples).  counters_out = raw counters
 * (symmetric: unordered; asymmetric: ordered, the caller halves `true`).
 */
void oracle_cellpairs(int symmetric, int nthreads_logical, int64_t block_of_cells, int reach,
                      int64_t nx, int64_t ny, int64_t nz, const int64_t* fbeg, const int64_t* fend,
                      const int64_t* bbeg, const int64_t* bend, int64_t n, int64_t nb, int dmode,
                      const float* pos, const float* vel, const float* rho, const float* press,
                      const float* prrho, const float* csound, const float* tensil,
                      const double* pp, const uint8_t* cells_mask, double* acc, double* drho,
                      double* viscdt, int64_t* counters_out) {
  state_t s = {pos, vel, rho, press, prrho, csound, tensil, pp, dmode};
  const int64_t ncells = nx * ny * nz;
  int T = nthreads_logical > 1 ? nthreads_logical : 1;
  int64_t* cells = (int64_t*)malloc(sizeof(int64_t) * (ncells > 0 ? ncells : 1));
  cnt_t total = {0, 0, 0, 0};
  if (T == 1) {
    int64_t m = 0;
    for (int64_t c = 0; c < ncells; ++c)
      if (!cells_mask || cells_mask[c]) cells[m++] = c;
    run_cells(&s, symmetric, cells, m, nx, ny, nz, reach, fbeg, fend, bbeg, bend, nb, acc, drho,
              viscdt, &total);
  } else {
    /* thread t's cell list = blocks t, t + T, t + 2T, ... in order (cellpairs.py:141-146) */
    int64_t nblocks = (ncells + block_of_cells - 1) / block_of_cells;
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (T + 1));
    int64_t m = 0;
    for (int t = 0; t < T; ++t) {
      start[t] = m;
      for (int64_t b = t; b < nblocks; b += T)
        for (int64_t c = b * block_of_cells; c < (b + 1) * block_of_cells && c < ncells; ++c)
          if (!cells_mask || cells_mask[c]) cells[m++] = c;
    }
    start[T] = m;
    double** pa = (double**)malloc(sizeof(double*) * T);
    double** pd = (double**)malloc(sizeof(double*) * T);
    double** pv = (double**)malloc(sizeof(double*) * T);
    cnt_t* pc = (cnt_t*)calloc(T, sizeof(cnt_t));
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 1)
#endif
    for (int t = 0; t < T; ++t) {
      pa[t] = t == 0 ? acc : (double*)calloc(3 * n, sizeof(double));
      pd[t] = t == 0 ? drho : (double*)calloc(n, sizeof(double));
      pv[t] = t == 0 ? viscdt : (double*)calloc(n, sizeof(double));
      run_cells(&s, symmetric, cells + start[t], start[t + 1] - start[t], nx, ny, nz, reach, fbeg,
                fend, bbeg, bend, nb, pa[t], pd[t], pv[t], &pc[t]);
    }
    /* merge_accumulators: out = acc[0]; out += acc[1]; ... elementwise, thread order */
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
      for (int t = 1; t < T; ++t) {
        acc[3 * i + 0] += pa[t][3 * i + 0];
        acc[3 * i + 1] += pa[t][3 * i + 1];
        acc[3 * i + 2] += pa[t][3 * i + 2];
        drho[i] += pd[t][i];
        if (pv[t][i] > viscdt[i]) viscdt[i] = pv[t][i];
      }
    }
    for (int t = 0; t < T; ++t) {
      total.cand += pc[t].cand;
      total.tru += pc[t].tru;
      total.evals += pc[t].evals;
      total.ff += pc[t].ff;
      if (t) {
        free(pa[t]);
        free(pd[t]);
        free(pv[t]);
      }
    }
    free(pa);
    free(pd);
    free(pv);
    free(pc);
    free(start);
  }
  free(cells);
  counters_out[0] = total.cand;
  counters_out[1] = total.tru;
  counters_out[2] = total.evals;
  counters_out[3] = total.ff;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
