// interact_pair.cuh -- the FP32 gather interaction with TWO targets per lane (k_interact_v12).
// Included by interact.cu inside its anonymous namespace when built with SPHB_PAIR (the pi512p
// object): it reuses the v8 helpers (staging, tensor-core screen, FIFO ring, guard band).
//
// Same contract as k_interact_v8 (gather_fluid_* / gather_boundary_*, kernels.py:326-596; pair
// math physics.py:183-220; compute_dt epilogue sim.py:215-232), different lane mapping:
//   * lane r of warp w owns targets 64 w + 2 r and 64 w + 2 r + 1 -- consecutive cell-sorted
//     particles, usually lattice neighbours, whose neighbour sets overlap ~80%;
//   * the tensor-core screen runs 64 targets x 32 candidates per word (4 M-tiles); the two
//     targets' sign words are OR-ed before the quad transpose, so a lane queues the UNION of its
//     targets' maybes -- one FIFO, one pop per candidate for both targets;
//   * the pair math is packed vertically: every FFMA2/FADD2/FMUL2 evaluates (target 0,
//     target 1) x (the popped candidate), the candidate's fields enter as a broadcast scalar
//     operand, so the x/y/z horizontal sums of v8 disappear and the candidate-only terms (cs_j,
//     tensile_j, mass_j) are computed once for both pairs;
//   * a pair whose candidate is the target itself (r2 = 0) is recognised by its staged address
//     and skipped without the exact f64 branch; every other guard-band / coincident pair is
//     re-decided exactly as in v8, so hit sets and counters stay bit-exact.
// Work per popped candidate is two pair evaluations of which ~85% are hits of the union at rest
// (DESIGN.md §4): the pop, the two staged loads and the candidate terms are shared.

#if SPHB_PAIR
constexpr int P12_PAIRS = V8_NG;  // pops (one candidate, two targets) per lane per drain iteration
#ifndef V12_KMIN
#define V12_KMIN 16               // minimum iterations of a partial drain
#endif
#ifndef V12_SORT
#define V12_SORT 0                // 1: pair the lane's targets by position (warp bitonic sort)
#endif
static_assert(P12_PAIRS * V12_KMIN >= 32, "partial drains must free a FIFO entry");
static_assert(BT == 64 * NW, "two targets per lane");

struct Own2 {  // (slot 0, slot 1) of the lane's two targets
  f2_t x, y, z, vx, vy, vz, rho, prrho, csn, tenk;
};
struct Acc2 {
  f2_t ax, ay, az, dr, hits;
  float vd0, vd1;
};
// an opaque 64-bit move: keeps a packed pair in one aligned register pair (otherwise ptxas may
// hold the halves apart and re-pack them with two MOVs at every use)
__device__ __forceinline__ f2_t pin2(f2_t v) {
  f2_t r;  // v + (-0, -0) == v exactly; a real FADD2, so its result is one 64-bit register
  asm volatile("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(0x8000000080000000ull));
  return r;
}

// NG popped candidates (staged A-row byte addresses; bit 0 = boundary list when masses differ)
// against both targets of the lane
template <bool G7, bool EQM, bool WEND, int NG>
__device__ __forceinline__ void eval_v12(const KArgs& a, const K32& c, const Own2& o,
                                         const uint32_t (&ad)[NG], uint32_t own0, uint32_t own1,
                                         const int (&ti)[2], const int (&xlo)[2],
                                         const int (&xhi)[2], Acc2 (&s)[NG]) {
  constexpr uint32_t OFFB = 16u * V8_ROWS;  // A -> B rows
  f2_t DX[NG], DY[NG], DZ[NG], R2[NG], DOT[NG];
  float bw[NG], aw[NG];
  float okf[2 * NG], r2m[2 * NG];
  bool anycold = false;
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const uint32_t p = EQM ? ad[k] : (ad[k] & ~1u);
    const float4 A = lds4(p);
    const float4 B = lds4(p + OFFB);
    aw[k] = A.w;
    bw[k] = B.w;
    DX[k] = sub2(o.x, bc(A.x));
    DY[k] = sub2(o.y, bc(A.y));
    DZ[k] = sub2(o.z, bc(A.z));
    R2[k] = fma2(DZ[k], DZ[k], fma2(DY[k], DY[k], mul2(DX[k], DX[k])));
    const f2_t DVX = sub2(o.vx, bc(B.x)), DVY = sub2(o.vy, bc(B.y)), DVZ = sub2(o.vz, bc(B.z));
    DOT[k] = fma2(DVZ, DZ[k], fma2(DVY, DY[k], mul2(DVX, DX[k])));
    const float r20 = lo(R2[k]), r21 = hi(R2[k]);
    const bool s0 = is_sure(r20, c), s1 = is_sure(r21, c);
    // the target itself (r2 = 0) is no pair: skipped by address, not re-decided
    const bool c0 = !s0 & (r20 < c.sup2_hi) & (ad[k] != own0);
    const bool c1 = !s1 & (r21 < c.sup2_hi) & (ad[k] != own1);
    okf[2 * k] = s0 ? 1.0f : 0.0f;
    okf[2 * k + 1] = s1 ? 1.0f : 0.0f;
    r2m[2 * k] = s0 ? r20 : c.sup2_lo;
    r2m[2 * k + 1] = s1 ? r21 : c.sup2_lo;
    anycold |= c0 | c1;
  }
  if (__any_sync(SPHB_FULL, anycold)) {
    // guard band / coincident: the exact f64 decision, one (candidate, target) per lane per round
    uint32_t cm = 0;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      cm |= ((in_cold(lo(R2[k]), c) && ad[k] != own0) ? 1u : 0u) << (2 * k);
      cm |= ((in_cold(hi(R2[k]), c) && ad[k] != own1) ? 1u : 0u) << (2 * k + 1);
    }
    uint32_t accm = 0;  // accepted cold slots
    do {
      const int b = __ffs(cm) - 1;  // slot 2 k + t: candidate k, target t
      // the popped address of candidate b / 2 by explicit selects (an indexed pick made ptxas
      // keep the pops in local memory: three stores per drain iteration)
      uint32_t adk = ad[0];
#pragma unroll
      for (int kk = 1; kk < NG; ++kk) {
        const uint32_t hit = (uint32_t)((b >> 1) == kk);
        asm("{ .reg .pred q; setp.ne.u32 q, %2, 0; selp.b32 %0, %1, %0, q; }"
            : "+r"(adk) : "r"(ad[kk]), "r"(hit));
      }
      const bool t1 = b & 1;
      bool acc = false;
      if (cm) {  // the target's coordinates: a half of the packed registers
        const float4 A = lds4(adk & ~1u);
        const float px = t1 ? hi(o.x) : lo(o.x), py = t1 ? hi(o.y) : lo(o.y),
                    pz = t1 ? hi(o.z) : lo(o.z);
        acc = cold_accept(a, px, py, pz, A, t1 ? xlo[1] : xlo[0], t1 ? xhi[1] : xhi[0]);
        cm &= cm - 1u;
      }
      accm |= acc ? 1u << b : 0u;
    } while (__any_sync(SPHB_FULL, cm != 0u));
#pragma unroll
    for (int kk = 0; kk < 2 * NG; ++kk) {  // once after the rounds, not once per round
      if ((accm >> kk) & 1u) {
        okf[kk] = 1.0f;
        r2m[kk] = (kk & 1) ? hi(R2[kk >> 1]) : lo(R2[kk >> 1]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const f2_t OK = pk(okf[2 * k], okf[2 * k + 1]);
    const f2_t R2M = pk(r2m[2 * k], r2m[2 * k + 1]);
    const f2_t RINV = pk(rsqrtf(lo(R2M)), rsqrtf(hi(R2M)));
    const f2_t Q = mul2(mul2(R2M, RINV), bc(c.invh));
    f2_t W, DWR;  // kernel shape W/kc and the gradient shape (-gc / mask factor)
    if (WEND) {   // Wendland C2: W = kc t^4 (2q + 1), gc = -5 kc t^3 / h^2, t = 1 - q/2
      const f2_t T = fma2(Q, bc(-0.5f), bc(1.0f));
      const f2_t T2 = mul2(T, T);
      W = mul2(mul2(T2, T2), fma2(Q, bc(2.0f), bc(1.0f)));
      DWR = mul2(T2, T);
    } else {      // cubic spline (physics.py:196-205)
      const f2_t T = sub2(bc(2.0f), Q);
      const f2_t UM = sub2(Q, bc(1.0f));
      const f2_t UN = pk(fminf(lo(UM), 0.0f), fminf(hi(UM), 0.0f));  // -max(1 - q, 0)
      const f2_t T2Q = mul2(mul2(T, T), bc(0.25f));
      const f2_t U2 = mul2(UN, UN);
      W = fma2(T2Q, T, mul2(U2, UN));   // t^3/4 - u^3
      DWR = mul2(sub2(U2, T2Q), RINV);  // (3 u^2 - 3/4 t^2) / (3 r)
    }
    // candidate-only terms, once for both pairs
    const float rj = fabsf(bw[k]);
    const float mj = (EQM || !(ad[k] & 1u)) ? c.nkgc : c.nkgc_b;  // -3 kc/h [m_j]
    float csj;                                                  // -alpha h cs_j
    if (G7) {
      const float rr = rj * c.kcs;
      csj = rr * rr * rr;
    } else {
      csj = exp2f(c.cs_exp * __log2f(rj)) * c.kcs;
    }
    const float pr = aw[k];
    const float tenj = pr * (pr > 0.0f ? c.tpos : c.tneg);
    const f2_t GCN = mul2(DWR, mul2(OK, bc(mj)));  // -gc [m_j], zero when masked
    const f2_t E = add2(R2M, bc(c.eta2));
    const f2_t MU = mul2(mul2(DOT[k], pk(rcp_approx(lo(E)), rcp_approx(hi(E)))), OK);  // mu / h
    const f2_t RS = add2(o.rho, bc(rj));
    const f2_t VT = mul2(mul2(add2(o.csn, bc(csj)), MU), pk(rcp_approx(lo(RS)), rcp_approx(hi(RS))));
    const f2_t VISC = pk(fmaxf(lo(VT), 0.0f), fmaxf(hi(VT), 0.0f));
    const f2_t W2 = mul2(W, W);
    const f2_t PT = fma2(mul2(add2(o.tenk, bc(tenj)), W2), W2, add2(add2(o.prrho, bc(pr)), VISC));
    const f2_t FM = mul2(PT, GCN);
    s[k].ax = fma2(DX[k], FM, s[k].ax);
    s[k].ay = fma2(DY[k], FM, s[k].ay);
    s[k].az = fma2(DZ[k], FM, s[k].az);
    s[k].dr = fma2(GCN, DOT[k], s[k].dr);
    s[k].vd0 = fmaxf(s[k].vd0, fabsf(lo(MU)));
    s[k].vd1 = fmaxf(s[k].vd1, fabsf(hi(MU)));
    s[k].hits = add2(s[k].hits, OK);
  }
}

template <bool G7, bool EQM, bool WEND, bool WALL>
__global__ void __launch_bounds__(NW * 32, 1) k_interact_v12(KArgs a, K32 k32) {
  if (!step_live(a.ctrl)) return;
  constexpr int SCAP = Cfg<float>::SCAP;
  constexpr int RINGC = V8_RING;       // FIFO entries per lane (8 B)
  constexpr int MASK0 = V8_FIFO_OFF / 4;
  constexpr float NOHIT = 1e30f;       // C of a target row that must not screen in
  __shared__ Seg sSeg[MAXSEG];
  __shared__ int s_blk, s_nseg_tot, s_scan[MAXSEG];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = a.g.dims[0], ny = a.g.dims[1], nz = a.g.dims[2];
  const int reach = a.g.reach, side = 2 * reach + 1;
  const uint32_t nblocks = a.ctrl->nblk[0];
  const int64_t step = a.ctrl->step;
  __shared__ __align__(8) unsigned long long s_mbar;
  const uint32_t mbar = smem_addr(&s_mbar);
  uint32_t mphase = 0;
  if (tid == 0) {  // the dummy row popped by empty FIFO slots: far away, at rest, finite
    const float far = (float)(1e4 * 2.0 * a.p.h);
    g_sm4[SCAP] = make_float4(far, far, far, 0.f);
    g_sm4[V8_ROWS + SCAP] = make_float4(0.f, 0.f, 0.f, 1.f);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t smA = pin_u32(smem_addr(g_sm4));
  const uint32_t smR = smA + V8_REC_OFF;
  const uint32_t dummy = smA + 16u * SCAP;
  if (tid < 16) g_sm32[V8_ZERO_OFF / 4 + tid] = 0u;
  const int fg = lane >> 2, ft = lane & 3;
  const uint32_t bl_off = ft < 2 ? 64u * (fg >> 1) + 8u * (fg & 1) + 4u * ft : 0u;
  const uint32_t bl_kmul = ft < 2 ? 8u : 0u;
  const uint32_t bl_base = ft < 2 ? smR : smA + V8_ZERO_OFF;
  const uint32_t tsel1 = (ft & 1) ? 0x3715u : 0x6240u;
  const uint32_t tsel2 = (ft & 2) ? 0x3276u : 0x5410u;
  const int troute = 4 * (lane & 7) + (lane >> 3);
  const uint32_t ring = pin_u32(smem_addr(g_sm32 + MASK0) + 8u * (warp * RINGC * 32 + lane));
  const uint32_t rend = ring + 256u * RINGC;

  unsigned long long c_hits = 0;
  long long c_ff = 0;
  double dtf_min = INFINITY, dtcv_min = INFINITY;

  __shared__ int4 s_bb[2];
  int4 nxt_b = make_int4(0, 0, 0, 0), nxt_m = make_int4(0, 0, 0, 0);
  uint32_t nxt = 0;
  if (tid == 0) {
    nxt = atomicAdd(&a.ctrl->tile_next[0], 1u);
    if (nxt < nblocks) {
      nxt_b = a.blocks[2 * nxt];
      nxt_m = a.blocks[2 * nxt + 1];
    }
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_blk = (int)nxt;
      s_bb[0] = nxt_b;
      s_bb[1] = nxt_m;
    }
    __syncthreads();
    if (tid == 0) {  // the next record: its atomic and loads overlap this block (not the barrier)
      nxt = atomicAdd(&a.ctrl->tile_next[0], 1u);
      if (nxt < nblocks) {
        nxt_b = a.blocks[2 * nxt];
        nxt_m = a.blocks[2 * nxt + 1];
      }
    }
    const uint32_t blk = (uint32_t)s_blk;
    if (blk >= nblocks) break;
    const int4 bb = s_bb[0], bm = s_bb[1];
    const bool brick = bm.w != 0;
    const int bsd = brick ? 2 : 1;
    const int rowkey = bm.x;
    const int cxa = bm.y, cxb = bm.z;
    const int nlist = (brick || bb.y > bb.x) ? 2 : 1;
    const int bside = side + bsd - 1;
    const int nrow = bside * bside;
    const int nseg = nlist * nrow;
    const int gcz = rowkey / ny, gcy = rowkey - gcz * ny;
    const int bxlo = max(cxa - reach, 0), bxhi = min(cxb + reach, nx - 1);
    const double cs = a.g.cell_size;
    const float h16_s = (float)(0.5 * a.p.invh);
    const float h16_xc = (float)(a.g.origin[0] + 0.5 * (bxlo + bxhi + 1) * cs);
    const float h16_yc = (float)(a.g.origin[1] + (gcy + 0.5 * bsd) * cs);
    const float h16_zc = (float)(a.g.origin[2] + (gcz + 0.5 * bsd) * cs);
    const double xext = 0.5 * (bxhi - bxlo + 1) * cs * (0.5 * a.p.invh);
    const double yzext = (reach + 0.5 * bsd) * cs * (0.5 * a.p.invh);
    const bool use16 = xext <= H16_MAXABS && yzext <= H16_MAXABS &&
                       xext * xext + 2.0 * yzext * yzext < 30.0;
    const int rr_c = reach * side + reach;
    const int selfseg = (bb.y > bb.x) ? ((nlist == 2 && a.p.order == 1) ? rr_c : rr_c * nlist) : -1;

    __shared__ int s_tlo[8], s_tlen[8];  // brick targets: F rows 0..3, then B rows 0..3
    if (brick && tid < 8) {
      const int li = tid >> 2, sub = tid & 3, yy = gcy + (sub & 1), zz = gcz + (sub >> 1);
      int lo_ = 0, len = 0;
      if (yy < ny && zz < nz) {
        const int64_t ro = (li == 0 ? a.ncells : 0) + (int64_t)nx * (yy + (int64_t)ny * zz);
        lo_ = a.beg[ro + cxa];
        len = max(a.end[ro + cxb] - lo_, 0);
      }
      s_tlo[tid] = lo_;
      s_tlen[tid] = len;
    }
    if (tid < MAXSEG) {
      int len = 0;
      Seg sg = {0, 0, 0, 0, 0};
      if (tid < nseg) {
        int li, rr;
        if (nlist == 2 && a.p.order == 1) {
          li = tid / (side * side);
          rr = tid - li * side * side;
        } else {
          li = tid % nlist;
          rr = tid / nlist;
        }
        const int dz = rr / bside - reach, dy = rr % bside - reach;
        const int zz = gcz + dz, yy = gcy + dy;
        if (zz >= 0 && zz < nz && yy >= 0 && yy < ny) {
          const int64_t rowoff = (li == 0 ? a.ncells : 0) + (int64_t)nx * (yy + (int64_t)ny * zz);
          sg.g0 = a.beg[rowoff + bxlo];
          sg.g1 = a.end[rowoff + bxhi];
          sg.rowoff = (int)rowoff;
          sg.dyz = (dy + 16) | ((dz + 16) << 8);
          len = max(sg.g1 - sg.g0, 0);
          if (len == 0) sg.g1 = sg.g0;
        }
      }
      s_scan[tid] = len;
      sSeg[tid] = sg;
    }
    __syncthreads();
    if (warp == 0) {
      int v[4], run = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = s_scan[lane * 4 + k];
        run += v[k];
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(SPHB_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      int ex = incl - run;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        sSeg[lane * 4 + k].pos = ex;
        ex += v[k];
      }
      if (lane == 31) s_nseg_tot = incl;
    }
    __syncthreads();
    const int total = s_nseg_tot;
    // the first staging batch goes out now: its bulk copies land during the targets' setup
    if (warp == 0 && total > 0)  // (no batch, no mbarrier phase: an empty block stages nothing)
      stage_batch(a.posp, a.velr, sSeg, nseg, 0, min(SCAP, total), smA, 16u * V8_ROWS, mbar, lane);

    // ---- the lane's two targets: block slots 64 w + 2 lane + t
    // slots: fluid targets [0, nf), boundary targets from the even slot nfp = pad2(nf) on, so
    // a lane's two targets are of one list (k_blocks reserves the padding slot)
    int nf = bb.y - bb.x, nbt = bb.w - bb.z;
    int ti[2], rsy[2] = {0, 0}, rsz[2] = {0, 0};
    bool isf[2], valid[2];
    if (brick) {
      nf = s_tlen[0] + s_tlen[1] + s_tlen[2] + s_tlen[3];
      nbt = s_tlen[4] + s_tlen[5] + s_tlen[6] + s_tlen[7];
    }
    const int nfp = (nf + 1) & ~1;
    {
      const int t0 = warp * 64 + 2 * lane;
      int u[2];  // index in the block's target order (fluid ranges, then boundary ranges)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        isf[t] = t0 + t < nf;
        valid[t] = isf[t] || (t0 + t >= nfp && t0 + t < nfp + nbt);
        u[t] = isf[t] ? t0 + t : nf + (t0 + t - nfp);
      }
      if (brick) {
        int pre = 0, k0 = 0, k1 = 0, lo0 = s_tlo[0], lo1 = s_tlo[0];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int len = s_tlen[k];
          if (u[0] >= pre && u[0] < pre + len) {
            k0 = k;
            lo0 = s_tlo[k] + (u[0] - pre);
          }
          if (u[1] >= pre && u[1] < pre + len) {
            k1 = k;
            lo1 = s_tlo[k] + (u[1] - pre);
          }
          pre += len;
        }
        ti[0] = lo0;
        ti[1] = lo1;
        rsy[0] = k0 & 1;
        rsz[0] = (k0 >> 1) & 1;
        rsy[1] = k1 & 1;
        rsz[1] = (k1 >> 1) & 1;
      } else {
#pragma unroll
        for (int t = 0; t < 2; ++t) ti[t] = isf[t] ? bb.x + u[t] : bb.z + (u[t] - nf);
      }
    }
    const bool wactive = warp * 64 < nfp + nbt;
#if V12_SORT
    // Pairing by position: the warp's 64 slots are re-ordered by (list, padding, Morton code of
    // the position at cell/16 resolution) with a warp bitonic sort, and lane r takes sorted
    // slots 2r, 2r + 1 -- near neighbours, whose neighbour sets overlap most, even once the
    // order inside a cell has mixed (a collapsed column).  The padding slot sorts between the
    // lists, so a lane's two targets stay of one list.
    if (wactive) {
      uint32_t key[2];
      const double q = 16.0 / a.g.cell_size;
      const double ox = a.g.origin[0] + (double)cxa * a.g.cell_size;
      const double oy = a.g.origin[1] + (double)gcy * a.g.cell_size;
      const double oz = a.g.origin[2] + (double)gcz * a.g.cell_size;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int slot = warp * 64 + 2 * lane + t;
        uint32_t rank = valid[t] ? (isf[t] ? 0u : 2u) : (slot < nfp ? 1u : 3u);
        uint32_t m = 0;
        if (valid[t]) {
          const float4 p = a.posp[ti[t]];
          const int qx = min(max((int)((p.x - ox) * q), 0), 127);
          const int qy = min(max((int)((p.y - oy) * q), 0), 127);
          const int qz = min(max((int)((p.z - oz) * q), 0), 127);
#pragma unroll
          for (int b = 0; b < 7; ++b)
            m |= (((qx >> b) & 1u) << (3 * b)) | (((qy >> b) & 1u) << (3 * b + 1)) |
                 (((qz >> b) & 1u) << (3 * b + 2));
        }
        key[t] = (rank << 30) | (m << 6) | (uint32_t)(2 * lane + t);  // unique keys
      }
#pragma unroll
      for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          if (j == 1) {
            const bool asc = ((2 * lane) & k) == 0;
            if ((key[0] > key[1]) == asc) {
              const uint32_t tmp = key[0];
              key[0] = key[1];
              key[1] = tmp;
            }
          } else {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const uint32_t ok = __shfl_xor_sync(SPHB_FULL, key[t], j >> 1);
              const int e = 2 * lane + t;
              const bool asc = (e & k) == 0, lower = (e & j) == 0;
              key[t] = (lower == asc) ? min(key[t], ok) : max(key[t], ok);
            }
          }
        }
      }
      const uint32_t fl0 = (isf[0] ? 1u : 0u) | (valid[0] ? 2u : 0u) | (uint32_t)rsy[0] << 2 | (uint32_t)rsz[0] << 3;
      const uint32_t fl1 = (isf[1] ? 1u : 0u) | (valid[1] ? 2u : 0u) | (uint32_t)rsy[1] << 2 | (uint32_t)rsz[1] << 3;
      int nti[2];
      uint32_t nfl[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int src = (int)((key[t] & 63u) >> 1);
        const bool hi1 = key[t] & 1u;
        const int a0 = __shfl_sync(SPHB_FULL, ti[0], src), a1 = __shfl_sync(SPHB_FULL, ti[1], src);
        const uint32_t f0 = __shfl_sync(SPHB_FULL, fl0, src), f1 = __shfl_sync(SPHB_FULL, fl1, src);
        nti[t] = hi1 ? a1 : a0;
        nfl[t] = hi1 ? f1 : f0;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        ti[t] = nti[t];
        isf[t] = nfl[t] & 1u;
        valid[t] = (nfl[t] >> 1) & 1u;
        rsy[t] = (nfl[t] >> 2) & 1u;
        rsz[t] = (nfl[t] >> 3) & 1u;
      }
    }
#endif
    auto in_rows = [&](int dyz, int t) {
      return abs((dyz & 255) - 16 - rsy[t]) <= reach && abs((dyz >> 8) - 16 - rsz[t]) <= reach;
    };
    int selfseg_t[2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
      selfseg_t[t] = !brick ? selfseg : ((rsz[t] + reach) * bside + (rsy[t] + reach)) * nlist;
    Own2 o;
    float ocs[2] = {0.f, 0.f};
    float ox2[2], oy2[2], oz2[2];  // scalar copies for the screen's A fragments (block setup)
    int xlo[2] = {0, 0}, xhi[2] = {-1, -1};
    {
      float4 pi[2], vi[2], xi[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        pi[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        vi[t] = make_float4(0.f, 0.f, 0.f, 1.f);
        xi[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid[t]) {
          pi[t] = a.posp[ti[t]];
          vi[t] = a.velr[ti[t]];
          if (a.aux) {
            xi[t] = a.aux[ti[t]];
          } else {  // no aux rows this step: the target's own csound / tensil
            const float2 ct = target_cs_tensil<G7>((double)vi[t].w, pi[t].w, a.inv_rho0, a.p);
            xi[t] = make_float4(0.f, ct.x, ct.y, 0.f);
          }
          const int cxi = a.cell[ti[t]] - (rowkey + rsy[t] + ny * rsz[t]) * nx;
          xlo[t] = max(cxi - reach, 0);
          xhi[t] = min(cxi + reach, nx - 1);
        }
        ocs[t] = xi[t].y;
      }
      o.x = pin2(pk(pi[0].x, pi[1].x));
      o.y = pin2(pk(pi[0].y, pi[1].y));
      o.z = pin2(pk(pi[0].z, pi[1].z));
      o.prrho = pin2(pk(pi[0].w, pi[1].w));
      o.vx = pin2(pk(vi[0].x, vi[1].x));
      o.vy = pin2(pk(vi[0].y, vi[1].y));
      o.vz = pin2(pk(vi[0].z, vi[1].z));
      o.rho = pin2(pk(vi[0].w, vi[1].w));
      const float nah = (float)(-a.p.alpha * a.p.h);
      o.csn = pin2(pk(nah * xi[0].y, nah * xi[1].y));
      o.tenk = pin2(pk(xi[0].z * k32.ktw4, xi[1].z * k32.ktw4));
      ox2[0] = pi[0].x; ox2[1] = pi[1].x; oy2[0] = pi[0].y; oy2[1] = pi[1].y;
      oz2[0] = pi[0].z; oz2[1] = pi[1].z;
    }
    const int wxlo = __reduce_min_sync(SPHB_FULL, min(valid[0] ? xlo[0] : INT_MAX, valid[1] ? xlo[1] : INT_MAX));
    const int wxhi = __reduce_max_sync(SPHB_FULL, max(valid[0] ? xhi[0] : INT_MIN, valid[1] ? xhi[1] : INT_MIN));
    Acc2 s[P12_PAIRS];
#pragma unroll
    for (int k = 0; k < P12_PAIRS; ++k) {
      s[k].ax = s[k].ay = s[k].az = s[k].dr = s[k].hits = bc(0.0f);
      s[k].vd0 = s[k].vd1 = 0.0f;
    }
    // A fragments of the screen: M-tile m holds target slot m / 2 of lanes 16 (m % 2) + row
    // (rows g, g + 8 of the tile); C = |x|^2 - thr, or NOHIT for a target the row must skip
    uint32_t fa[4][2];
    float cv[2];
    {
      uint32_t alo[2], ahi[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float ox = ox2[t], oy = oy2[t], oz = oz2[t];
        const __half hx = __float2half_rn((ox - h16_xc) * h16_s);
        const __half hy = __float2half_rn((oy - h16_yc) * h16_s);
        const __half hz = __float2half_rn((oz - h16_zc) * h16_s);
        const float fx = __half2float(hx), fy = __half2float(hy), fz = __half2float(hz);
        alo[t] = h2u(__floats2half2_rn(-2.0f * fx, -2.0f * fy));
        ahi[t] = h2u(__floats2half2_rn(-2.0f * fz, 1.0f));
        cv[t] = fmaf(fz, fz, fmaf(fy, fy, fx * fx)) - MMA_THR;
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 16 * (m & 1) + 8 * h + fg;
          const uint32_t vlo = __shfl_sync(SPHB_FULL, alo[m >> 1], r);
          const uint32_t vhi = __shfl_sync(SPHB_FULL, ahi[m >> 1], r);
          fa[m][h] = ft == 0 ? vlo : (ft == 1 ? vhi : 0u);
        }
      }
    }

    const uint32_t dummy_cb = dummy + 16u;  // an empty pop (bfind = -1) lands on the dummy row
    uint32_t hp = ring, tp = ring, cnt = 0, pend = 0, cur = 0u, cb = dummy_cb;
    uint32_t nx_mask = 0u, nx_cb = 0u;
    uint32_t own[2] = {0xffffffffu, 0xffffffffu};
    auto pop = [&]() -> uint32_t {
      const bool need = cur == 0u, have = cnt != 0u;
      if (need & have) {
        cur = nx_mask;
        cb = nx_cb;
        hp = hp + 256u == rend ? ring : hp + 256u;
        --cnt;
        const uint2 e = lds64u(hp);
        nx_mask = e.x;
        nx_cb = e.y;
      }
      cb = (need & !have) ? dummy_cb : cb;
      const int tb = flo32(cur);
      cur = clear_bit(cur, tb);
      return cb + 16u * (uint32_t)tb;
    };
    auto drain = [&](bool full) {
      __syncwarp();
      {
        const uint2 e = lds64u(hp);
        nx_mask = e.x;
        nx_cb = e.y;
      }
      constexpr uint32_t P = P12_PAIRS;
      const uint32_t mx = __reduce_max_sync(SPHB_FULL, pend);
      uint32_t K = (mx + P - 1) / P;
      if (!full) {
        const uint32_t mn = __reduce_min_sync(SPHB_FULL, pend ? pend : 0xffffffffu);
        K = min(K, max((mn + P - 1) / P, (uint32_t)V12_KMIN));
      }
      for (uint32_t it = 0; it < K; ++it) {
        uint32_t ad[P12_PAIRS];
#pragma unroll
        for (int k = 0; k < P12_PAIRS; ++k) ad[k] = pop();
        eval_v12<G7, EQM, WEND, P12_PAIRS>(a, k32, o, ad, own[0], own[1], ti, xlo, xhi, s);
      }
      pend = pend > P * K ? pend - P * K : 0u;
      __syncwarp();
    };

    // The warp's part of every staged row (cells [wxlo, wxhi]) as staged positions [wpos0,
    // wpos1), computed once per block by the lanes in parallel (lane l: rows l, l + 32, ...), and
    // whether a target of the warp uses the row (its rows: wrows_all; boundary-list rows only
    // the fluid targets': wrows_f)
    int wpos0[MAXSEG / 32], wpos1[MAXSEG / 32];
    uint32_t wlive = 0;
    {
      uint32_t mine_all = 0, mine_f = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t b = valid[t] ? 1u << (rsy[t] + 2 * rsz[t]) : 0u;
        mine_all |= b;
        mine_f |= isf[t] ? b : 0u;
      }
      const uint32_t wrows_all = __reduce_or_sync(SPHB_FULL, mine_all);
      const uint32_t wrows_f = __reduce_or_sync(SPHB_FULL, mine_f);
#pragma unroll
      for (int g = 0; g < MAXSEG / 32; ++g) {
        const int k = g * 32 + lane;
        wpos0[g] = wpos1[g] = 0;
        if (wactive && k < nseg) {
          const Seg sg = sSeg[k];
          if (sg.g1 > sg.g0) {
            const int w0 = a.beg[sg.rowoff + wxlo], w1 = a.end[sg.rowoff + wxhi];
            wpos0[g] = sg.pos + (w0 - sg.g0);
            wpos1[g] = sg.pos + (w1 - sg.g0);
            const uint32_t wr = sg.rowoff < a.ncells ? wrows_f : wrows_all;
            const int dy = (sg.dyz & 255) - 16, dz = (sg.dyz >> 8) - 16;
            bool need = false;
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4)
              need |= ((wr >> r4) & 1u) && abs(dy - (r4 & 1)) <= reach && abs(dz - (r4 >> 1)) <= reach;
            if (w1 > w0 && need) wlive |= 1u << g;
          }
        }
      }
    }

    // fused wall force (extension): f64 sums per target over the batches
    constexpr bool wall = WALL;  // (its own instantiation: none of it otherwise)
    double wf[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    bool whit[2] = {false, false};

    for (int q0 = 0; q0 < total; q0 += SCAP) {
      const int q1 = min(q0 + SCAP, total);
      if (warp == 0 && q0 > 0) stage_batch(a.posp, a.velr, sSeg, nseg, q0, q1, smA, 16u * V8_ROWS, mbar, lane);
      {
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done) : "r"(mbar), "r"(mphase) : "memory");
        mphase ^= 1u;
      }
      {
        uint2* rec = reinterpret_cast<uint2*>(reinterpret_cast<char*>(g_sm4) + V8_REC_OFF);
        for (int r = tid; r < q1 - q0; r += NW * 32) {
          const float4 pp = lds4(smA + 16u * r);
          const __half hx = __float2half_rn((pp.x - h16_xc) * h16_s);
          const __half hy = __float2half_rn((pp.y - h16_yc) * h16_s);
          const __half hz = __float2half_rn((pp.z - h16_zc) * h16_s);
          const float fx = __half2float(hx), fy = __half2float(hy), fz = __half2float(hz);
          rec[r] = make_uint2(h2u(__halves2half2(hx, hy)),
                              h2u(__halves2half2(hz, __float2half_rn(fmaf(fz, fz, fmaf(fy, fy, fx * fx))))));
        }
      }
      // the targets' own staged rows in this batch (fluid targets, own row of the fluid list)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        own[t] = 0xffffffffu;
        if (valid[t] && isf[t] && selfseg_t[t] >= 0) {
          const Seg sg = sSeg[selfseg_t[t]];
          const int p = sg.pos + (ti[t] - sg.g0) - q0;
          if (p >= 0 && p < q1 - q0) own[t] = smA + 16u * (uint32_t)p;
        }
      }
      __syncthreads();
      if (wactive) {
        // the warp's windows (precomputed per block, wpos0/wpos1) of the live rows, in row order
#pragma unroll
        for (int g = 0; g < MAXSEG / 32; ++g) {
          uint32_t mlive = __ballot_sync(SPHB_FULL, (wlive >> g) & 1u);
          while (mlive) {
          const int l = __ffs(mlive) - 1;
          mlive &= mlive - 1u;
          const int k = g * 32 + l;
          const int lo_ = max(__shfl_sync(SPHB_FULL, wpos0[g], l), q0) - q0;
          const int hi_ = min(__shfl_sync(SPHB_FULL, wpos1[g], l), q1) - q0;
          if (hi_ <= lo_) continue;
          const Seg sg = sSeg[k];
          const bool boundary_list = sg.rowoff < a.ncells;
          bool use[2];
#pragma unroll
          for (int t = 0; t < 2; ++t)
            use[t] = valid[t] && in_rows(sg.dyz, t) && (isf[t] || !boundary_list);
          // C per M-tile row for this staged row: targets that skip it never screen in
          float fcv[4][2];
          {
            const float c0 = use[0] ? cv[0] : NOHIT, c1 = use[1] ? cv[1] : NOHIT;
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                fcv[m][h] = __shfl_sync(SPHB_FULL, (m >> 1) ? c1 : c0, 16 * (m & 1) + 8 * h + fg);
          }
          for (int k0 = lo_; k0 < hi_; k0 += 32) {
            uint32_t hit;
            if (use16) {
              const uint32_t wb = bl_base + bl_kmul * (uint32_t)k0 + bl_off;
              uint32_t fb[4];
#pragma unroll
              for (int n = 0; n < 4; ++n) fb[n] = lds32(wb + 16u * n);
              uint32_t w = 0;
#pragma unroll
              for (int mp = 0; mp < 2; ++mp) {  // M-tile pairs: target slot 0, then slot 1
                float d[2][4][4];
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                  const float cc[4] = {fcv[2 * mp + m][0], fcv[2 * mp + m][0], fcv[2 * mp + m][1],
                                       fcv[2 * mp + m][1]};
#pragma unroll
                  for (int n = 0; n < 4; ++n)
                    mma_16816(d[m][n], fa[2 * mp + m][0], fa[2 * mp + m][1], fb[n], cc);
                }
#pragma unroll
                for (int n = 0; n < 4; ++n)
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const uint32_t pa = h2u(__floats2half2_rn(d[0][n][e], d[0][n][2 + e]));
                    const uint32_t pb = h2u(__floats2half2_rn(d[1][n][e], d[1][n][2 + e]));
                    w |= prmt_sign(pa, pb) & (0x01010101u << (2 * n + e));
                  }
              }
              // quad byte transpose: lane r <- the union of its targets' words
              w = prmt(w, __shfl_xor_sync(SPHB_FULL, w, 1), tsel1);
              w = prmt(w, __shfl_xor_sync(SPHB_FULL, w, 2), tsel2);
              hit = __shfl_sync(SPHB_FULL, w, troute);
            } else {
              const uint32_t sk = smA + 16u * k0;
              hit = 0;
#pragma unroll 8
              for (int tt = 0; tt < 32; ++tt) {
                const float4 A = lds4(sk + 16u * tt);
                const f2_t DX = sub2(o.x, bc(A.x)), DY = sub2(o.y, bc(A.y)), DZ = sub2(o.z, bc(A.z));
                const f2_t R2 = fma2(DZ, DZ, fma2(DY, DY, mul2(DX, DX)));
                const bool h0 = use[0] && lo(R2) < k32.sup2_hi, h1 = use[1] && hi(R2) < k32.sup2_hi;
                if (h0 || h1) hit |= 1u << tt;
              }
            }
            uint32_t bits = hit;  // k0 >= lo_: only the row's last word is partial
            if (hi_ - k0 < 32) bits &= (1u << (hi_ - k0)) - 1u;
            if (__any_sync(SPHB_FULL, bits != 0u && cnt == (uint32_t)RINGC)) drain(false);
            if (bits) {
              sts64u(tp, bits, smA + 16u * (uint32_t)k0 + ((!EQM && boundary_list) ? 1u : 0u));
              tp = tp + 256u == rend ? ring : tp + 256u;
              ++cnt;
              pend += __popc(bits);
            }
          }
          }
        }
        drain(true);
        if constexpr (wall) {
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (valid[t] && isf[t])
              whit[t] |= wall_batch(a, sSeg, nseg, q0, q1, smA, ox2[t], oy2[t], oz2[t], xlo[t], xhi[t],
                                    rsy[t], rsz[t], wf[t][0], wf[t][1], wf[t][2]);
        }
      }
      __syncthreads();
    }

#pragma unroll
    for (int k = 1; k < P12_PAIRS; ++k) {
      s[0].ax = add2(s[0].ax, s[k].ax);
      s[0].ay = add2(s[0].ay, s[k].ay);
      s[0].az = add2(s[0].az, s[k].az);
      s[0].dr = add2(s[0].dr, s[k].dr);
      s[0].hits = add2(s[0].hits, s[k].hits);
      s[0].vd0 = fmaxf(s[0].vd0, s[k].vd0);
      s[0].vd1 = fmaxf(s[0].vd1, s[k].vd1);
    }
    const float mfac = EQM ? (float)a.p.mass_fluid : 1.0f;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (!valid[t]) continue;
      const int hits = (int)(t ? hi(s[0].hits) : lo(s[0].hits));
      c_hits += (unsigned long long)hits;
      c_ff += isf[t] ? hits : -hits;  // ff = F targets' hits - B targets' hits (F-B == B-F)
      const double ax = (double)((t ? hi(s[0].ax) : lo(s[0].ax)) * mfac);
      const double ay = (double)((t ? hi(s[0].ay) : lo(s[0].ay)) * mfac);
      const double az = (double)((t ? hi(s[0].az) : lo(s[0].az)) * mfac);
      const double dr = (double)(-(t ? hi(s[0].dr) : lo(s[0].dr)) * mfac);
      const float vd32 = (t ? s[0].vd1 : s[0].vd0) * (float)a.p.h;
      const double vd = (double)vd32;
      const int i = ti[t];
      a.acc4[i] = isf[t] ? make_float4((float)ax, (float)ay, (float)az, (float)dr)
                         : make_float4(0.f, 0.f, 0.f, (float)dr);
      a.visc32[i] = vd32;
      if (!(isfinite(ax) && isfinite(ay) && isfinite(az) && isfinite(dr)))
        raise_div(a.ctrl, step, SPHB_DIV_NONFINITE_FORCES, 0);
      if (isf[t]) {
        const double fx = xadd(ax, a.p.g[0]), fy = xadd(ay, a.p.g[1]), fz = xadd(az, a.p.g[2]);
        double fmag = __dsqrt_rn(xadd(xadd(xmul(fx, fx), xmul(fy, fy)), xmul(fz, fz)));
        fmag = fmag > 1e-30 ? fmag : 1e-30;
        dtf_min = fmin(dtf_min, __dsqrt_rn(xdiv(a.p.h, fmag)));
      }
      if (whit[t])
        wall_finish(a, i, step, (float)ax, (float)ay, (float)az, (float)dr, wf[t][0], wf[t][1],
                    wf[t][2], dtf_min);
      dtcv_min = fmin(dtcv_min, xdiv(a.p.h, xadd((double)ocs[t], vd)));
    }
  }

  dtf_min = warp_min(dtf_min);
  dtcv_min = warp_min(dtcv_min);
  c_hits = warp_sum_u64(c_hits);
  const unsigned long long ffu = warp_sum_u64((unsigned long long)c_ff);
  if (lane == 0) {
    if (dtf_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_f, dtf_min);
    if (dtcv_min < INFINITY) atomic_min_pos(&a.ctrl->dtmin_cv, dtcv_min);
    if (c_hits) {
      atomicAdd((unsigned long long*)&a.ctrl->counters[1], c_hits);
      atomicAdd((unsigned long long*)&a.ctrl->counters[2], c_hits);
    }
    if (ffu) atomicAdd((unsigned long long*)&a.ctrl->counters[3], ffu);
  }
}
#endif  // SPHB_PAIR
