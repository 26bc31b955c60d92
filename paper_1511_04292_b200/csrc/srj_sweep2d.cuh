// srj_sweep2d.cuh -- temporally blocked 2D 5-point weighted-Jacobi sweep.
//
// One warp streams a column band of the grid down axis 0 and applies T
// consecutive SRJ steps (each with its own omega_k) in a single pass over HBM:
// stage t (t = 1..T) turns stage t-1 rows into step k+t rows entirely in
// registers.  The pipeline is skewed by two rows per stage -- at tick tau stage
// t relaxes row tau-2t from stage t-1 rows produced in EARLIER ticks -- so the
// T stages of a tick carry no dependency on each other and their DP chains
// overlap (instruction-level parallelism T x V per lane).  Horizontal neighbours move with warp
// shuffles; bands overlap by TP >= T columns per side so every owned column is
// exact at stage T (the overlap cells are recomputed, never stored).
//
// Rows arrive in groups of G = 3 (the window period): one 2D TMA tensor copy
// (cp.async.bulk.tensor.2d, box BAND x 3) for u^k and one for the source per
// group, completing on one mbarrier per ring slot.  A slot is recycled once
// the last stage has read its source rows (ceil(2T/3) groups later), so loads
// run NS - ceil(2T/3) - 1 groups ahead.
//
// Instruction economy (the kernel is issue-bound, not HBM-bound, at T>=2):
//  * the row window of each stage rotates by register renaming -- the tick
//    loop is unrolled by 3, the window period;
//  * one warp vote per tick for the rare IEEE-division fixups;
//  * interior ticks of interior bands take a predicate-free path;
//  * with a constant stencil only max|r| is tracked per step: |d| =
//    |RN(RN(omega*r)/c)| is a monotone function of |r|, so
//    max|d| = |RN(RN(omega*max|r|)/c)| exactly (evaluated once per warp);
//  * with a constant stencil the division uses a precomputed y = RN(1/c) and
//    two Markstein corrections, branch-free (correctly rounded, div_recip);
//    one warp vote per stage sends the rare subnormal/huge/inf/NaN
//    numerators to the IEEE division.
//
// Bitwise contract: the arithmetic per cell and step is exactly the reference
// _wj2 (grids.py:351-376); ghost rows/columns and inactive (masked) cells pass
// their value through unchanged (grids.py:374-375, FIXED ghosts :225-247).
#pragma once
#include <cuda.h>

#include "srj_device.cuh"

namespace srj {

struct Sweep2DParams {
  const double *src;   // interior origin (cell (0,0)) of u^k
  double *dst;         // interior origin of the output buffer
  const double *f;     // source s, or kappa for the nonlinear source
  const uint8_t *act;  // mask (padded byte layout) or nullptr
  const double *c, *am0, *ap0, *am1, *ap1;  // per-cell coefficients (VAR)
  double kc, kam0, kap0, kam1, kap1;        // constant stencil (!VAR)
  double kinv;         // RN(1/kc) when the reciprocal division is safe, else 0
  double kinv_lo;      // RN(1/c - kinv): low word of the reciprocal
  int64_t pitch;       // elements per row
  int n0, n1;          // interior extents
  int lo_c, hi_c;      // rows that relax (others pass through): [lo_c, hi_c)
  int ld_lo, ld_hi;    // rows present in memory: [ld_lo, ld_hi]
  int own_b, own_e;    // rows stored + counted in the norms
  int H, nbands, nstrips;
  int tma_col0;        // tensor-map column of interior column 0
  int tma_row0;        // tensor-map row of interior row 0
  double omega[kMaxFuse];
  double *norms;       // [T][2]: (dmax, rmax) per fused step
  // MIRROR / FACE_DIRICHLET faces under fusion (kernel flag BCF): stages 2..T
  // see the ghost the reference refreshes after every sweep, a pure function
  // of the adjacent cell -- substituted for column faces (stage2d, SUB),
  // written into the stage windows for row faces (SRJ_BCFIX)
  int bc_kind[2][2];           // SRJ_BC_* per (axis, side)
  const double *bc_ptr[2][2];  // face_dirichlet value at face position q: bc_ptr[q * bc_step]
  int bc_step[2][2];           // 1: per-position array; 0: the face's scalar
  PeerSend send;               // slab ranks: rows also stored into the neighbours' halos
};

template <int T, int V_ = 2>
struct Band2D {
  static constexpr int V = V_;                   // columns per lane
  static constexpr int BAND = 32 * V;            // columns per warp
  static constexpr int TP = (T + V - 1) / V * V; // overlap: whole lanes
  static constexpr int OWN = BAND - 2 * TP;      // columns a band owns
  static constexpr int G = 3;                    // rows per TMA group
  static constexpr int LAG = (2 * T + G - 1) / G;  // groups a source row stays live
  static constexpr int NU = 4;                      // u-box slots: prefetch NU-1 groups
  static constexpr int NF = (NU + LAG <= 8) ? 8 : 16;  // source slots >= NU + LAG
  static constexpr int LOG_NF = (NF == 8) ? 3 : 4;
  static constexpr int WARPS = 2;
  static constexpr int BOX_BYTES = G * BAND * 8;      // one array, one group
  static constexpr int WARP_BYTES = ((NU + NF) * BOX_BYTES + NF * 8 + 127) / 128 * 128;
  static constexpr size_t smem_bytes() { return size_t(WARPS) * WARP_BYTES; }
};


// One stage of the skewed pipeline for the lane's V cells.  (up, mid, down)
// hold stage t-1 rows r-1, r, r+1, all produced in earlier ticks, so the T
// stages of a tick are mutually independent.  Writes the stage-t value of row
// r to y and the numerators to num; bad collects div_recip range failures.
template <bool FAST, bool EDGE, bool VAR, bool NL, bool RECIP, int SUB, int V, bool EXACT = false>
__device__ __forceinline__ void stage2d(const Sweep2DParams &p, const double (&up)[V],
                                        const double (&mid)[V], const double (&down)[V],
                                        const double *frow, int r, double om, int lane_col,
                                        int i0, int i1, int own_c0, int own_c1, int f_lo,
                                        int f_hi, unsigned colact, bool cnt, unsigned bcm,
                                        double (&y)[V],
                                        double (&num)[V], double &rmx, double &dmx, bool &bad) {
  double fv[V];
#pragma unroll
  for (int v = 0; v < V; v += 2) {
    const double2 q = *reinterpret_cast<const double2 *>(frow + v);
    fv[v] = q.x;
    fv[v + 1] = q.y;
  }
  const double west0 = __shfl_up_sync(kFull, mid[V - 1], 1);
  const double eastV = __shfl_down_sync(kFull, mid[0], 1);
  // SUB (fused MIRROR / FACE_DIRICHLET column faces; bcm = 0 for stage 1,
  // which reads the refreshed ghosts from memory): column 0's
  // west and column n1-1's east neighbours are the ghosts the per-sweep
  // refresh would hold, computed here from the cell itself.  Branch-free and
  // off the critical path: resid5 consumes them last.
  double gw = 0.0, ge = 0.0;
  if (SUB) {
    static_assert(V == 2, "east-face cell select assumes two cells per lane");
    if (r < 0 || r >= p.n0) bcm = 0;  // ghost rows (slow ticks): corners untouched
    const double ae = (bcm & 4u) ? mid[1] : mid[0];
    if (SUB == 2) {  // column faces MIRROR (or FIXED): the cell itself
      gw = mid[0];
      ge = ae;
    } else {
      const int rq = min(max(r, 0), p.n0 - 1);
      const double vw = __ldg(p.bc_ptr[1][0] + int64_t(rq) * p.bc_step[1][0]);
      const double ve = __ldg(p.bc_ptr[1][1] + int64_t(rq) * p.bc_step[1][1]);
      const double fw = __dsub_rn(__dmul_rn(2.0, vw), mid[0]);
      const double fe = __dsub_rn(__dmul_rn(2.0, ve), ae);
      gw = p.bc_kind[1][0] == 1 ? mid[0] : fw;
      ge = p.bc_kind[1][1] == 1 ? ae : fe;
    }
  }
  bool row_act = true, row_own = true;
  int rc = 0;
  if (!FAST) {
    row_act = (r >= p.lo_c) && (r < p.hi_c);
    row_own = (r >= i0) && (r < i1);
    rc = min(max(r, f_lo), f_hi);
  }
  double cv[V];
  bool actv[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double uc = mid[v];
    double uw = (v == 0) ? west0 : mid[v - 1];
    double ue = (v == V - 1) ? eastV : mid[v + 1];
    if (SUB) {
      if (v == 0 && (bcm & 1u)) uw = gw;
      if ((bcm >> (1 + v)) & 1u) ue = ge;
    }
    double c = p.kc, a0 = p.kam0, b0 = p.kap0, a1 = p.kam1, b1 = p.kap1;
    bool act = true;
    const int col = lane_col + v;
    if (!FAST) {
      act = row_act && (col >= 0) && (col < p.n1);
      if (VAR) {
        const int64_t q = int64_t(rc) * p.pitch + col;
        c = __ldg(p.c + q);
        a0 = __ldg(p.am0 + q);
        b0 = __ldg(p.ap0 + q);
        a1 = __ldg(p.am1 + q);
        b1 = __ldg(p.ap1 + q);
        if (p.act) act = act && (__ldg(p.act + q) != 0);
      }
    }
    if (FAST && EDGE) act = (colact >> v) & 1u;
    const double s = NL ? nl_source(fv[v], uc) : fv[v];
    const double rr = resid5(s, c, uc, a0, up[v], b0, down[v], a1, uw, b1, ue);
    double nm = __dmul_rn(om, rr);
    if ((!FAST || EDGE) && !act) nm = 1.0;  // passthrough cell: keep garbage off the slow path
    num[v] = nm;
    cv[v] = c;
    actv[v] = act;
    if (FAST && !EDGE) {
      if (cnt) acc_absmax(rmx, rr);  // garbage lanes are excluded at the warp vote
    } else if (FAST) {
      if (cnt && ((colact >> (V + v)) & 1u)) acc_absmax(rmx, rr);  // owned-column bit
    } else if (act && row_own && col >= own_c0 && col < own_c1) {
      acc_absmax(rmx, rr);
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double uc = mid[v];
    double d;
    if (RECIP) {
      d = div_recip(num[v], p.kc, p.kinv, p.kinv_lo);
      // superset test (also flags zero numerators) in fewer integer ops; the
      // fix-up pass (fix_stage) applies the exact one.  EXACT (face-Dirichlet
      // kernels): zero numerators are frequent there, so the exact test is
      // cheaper overall (measured: 269 vs 319 GLUPS at 4096^2)
      bad |= EXACT ? recip_unsafe(num[v]) : recip_maybe_unsafe(num[v]);
    } else {
      d = __ddiv_rn(num[v], cv[v]);
    }
    if (FAST && !EDGE) {
      y[v] = __dadd_rn(uc, d);
    } else {
      y[v] = actv[v] ? __dadd_rn(uc, d) : uc;
      if (!FAST && VAR && actv[v] && row_own && lane_col + v >= own_c0 && lane_col + v < own_c1)
        acc_absmax(dmx, d);
    }
  }
}

// Redo the cells whose numerator fell outside div_recip's range with the IEEE
// division (rare: zero/subnormal/huge/inf/NaN numerators).
template <bool FAST, bool EDGE, int V>
__device__ __forceinline__ void fix_stage(const Sweep2DParams &p, const double (&mid)[V],
                                          const double (&num)[V], int r, int lane_col,
                                          unsigned colact, double (&y)[V]) {
  const bool row_act = FAST || ((r >= p.lo_c) && (r < p.hi_c));
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int col = lane_col + v;
    bool act = FAST || (row_act && col >= 0 && col < p.n1);
    if (FAST && EDGE) act = (colact >> v) & 1u;
    if (act && recip_unsafe(num[v])) y[v] = __dadd_rn(mid[v], div_ieee(num[v], p.kc));
  }
}

// The refreshed ghost next to boundary cell value adj at face position q
// (ghost_refresh's arithmetic, srj_reduce.cuh).
__device__ __forceinline__ double bc_ghost(const Sweep2DParams &p, int ax, int side, double adj,
                                           int q) {
  if (p.bc_kind[ax][side] == 1) return adj;
  const double v = __ldg(p.bc_ptr[ax][side] + int64_t(q) * p.bc_step[ax][side]);
  return __dsub_rn(__dmul_rn(2.0, v), adj);
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// SEND: slab ranks' copy of the kernel that also stores the edge rows into
// the neighbours' halo rows (PeerSend); every other instantiation carries no
// trace of it.
template <int T, int V, bool VAR, bool NL, bool RECIP, int BCF, bool SEND = false>
__global__ void __launch_bounds__(Band2D<T, V>::WARPS * 32)
    sweep2d_tb(const __grid_constant__ Sweep2DParams p, const __grid_constant__ CUtensorMap tm_u,
               const __grid_constant__ CUtensorMap tm_f) {
  using B = Band2D<T, V>;
  constexpr int BAND = B::BAND, TP = B::TP, OWN = B::OWN, NU = B::NU, NF = B::NF, G = B::G;
  constexpr int BOXD = B::BOX_BYTES / 8;  // doubles per box
  // dynamic shared memory starts the CTA's shared window (no static smem), so
  // it is 1024-byte aligned; indexing the symbol directly keeps every ring
  // access an LDS (pointer arithmetic through integers would turn them into
  // generic loads)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char *wbase = smem_raw + size_t(warp) * B::WARP_BYTES;
  double *ring_u = reinterpret_cast<double *>(wbase);  // NU u boxes
  double *ring_f = ring_u + NU * BOXD;                   // NF source boxes
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring_f + NF * BOXD);  // one per group mod NF

  // Piece order: the SM's warp scheduler favours older warps, so the CTAs of
  // a one-wave launch finish in tiers by block index.  The edge-band pieces
  // (column-masked fast path, ~16% more work per row) go first, onto the
  // oldest warps, then the interior pieces strip-major.
  const int gw = blockIdx.x * B::WARPS + warp;
  const int ne = (p.nbands >= 3) ? 2 * p.nstrips : 0;
  int band, strip;
  if (gw < ne) {
    band = (gw & 1) ? p.nbands - 1 : 0;
    strip = gw >> 1;
  } else {
    const int j = gw - ne, nb = ne ? p.nbands - 2 : p.nbands;
    band = (ne ? 1 : 0) + j % nb;
    strip = j / nb;
  }
  if (strip >= p.nstrips) return;  // warp-independent kernel: no block barriers

  const int i0 = p.own_b + strip * p.H;
  const int i1 = min(i0 + p.H, p.own_e);
  const int rho_b = max(i0 - T, p.ld_lo);
  const int nreal = i1 + 2 * T - rho_b;        // last real tick emits stage-T row i1-1
  const int ngroups = (nreal + G - 1) / G;     // extra ticks emit unowned rows only
  const int col_band = band * OWN - TP;
  const int own_c0 = band * OWN;
  const int own_c1 = min(own_c0 + OWN, p.n1);
  const int f_lo = p.lo_c, f_hi = p.hi_c - 1;
  const bool band_interior = (col_band >= 0) && (col_band + BAND <= p.n1) && !VAR;
  const bool band_edge = !band_interior && !VAR;  // fast rows, masked columns
  // fast ticks: every stage row rho-2t (t=1..T) relaxes (rows outside the
  // strip -- its dependency halo and the pipeline fill/drain -- are computed
  // the same way; only the owned ones count in the norms, flag cnt)
  const int fast_lo = p.lo_c + 2 * T;
  const int fast_hi = p.hi_c + 1;
  const int lane_col = col_band + V * lane;
  const bool lane_owned = (lane_col >= own_c0) && (lane_col + V <= own_c1);
  // bit v: column lane_col+v is interior (relaxes); bit V+v: it is owned
  unsigned colact = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (lane_col + v >= 0 && lane_col + v < p.n1) colact |= 1u << v;
    if (lane_col + v >= own_c0 && lane_col + v < own_c1) colact |= 1u << (V + v);
  }
  // fused non-FIXED column faces at this lane's cells: bit 0 = column 0 (at
  // v = 0, since TP is a multiple of V), bit 1+v = column n1-1 at v
  unsigned bcm = 0;
  if (BCF) {
    if (lane_col == 0 && p.bc_kind[1][0]) bcm |= 1u;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (lane_col + v == p.n1 - 1 && p.bc_kind[1][1]) bcm |= 2u << v;
  }
  // every edge band takes the substituting path once any column face is
  // non-FIXED (bcm = 0 lanes just select their own neighbours): two edge
  // code paths live at once on an SM cost more (i-cache) than the selects
  const bool warp_sub = BCF && (p.bc_kind[1][0] || p.bc_kind[1][1]);
  const int tma_col = p.tma_col0 + col_band;
  const int tma_row = p.tma_row0 + rho_b;

  // group g: u box -> ring_u[g mod NU], source box -> ring_f[g mod NF], both
  // completing on bars[g mod NF].  Issued at the end of group g-NU, when the
  // u slot is free; the source slot is free too because NF >= NU + LAG.
  auto issue = [&](int g) {
    uint64_t *bar = &bars[g & (NF - 1)];
    mbar_expect_tx(bar, 2 * B::BOX_BYTES);
    tma_load_2d(ring_u + (g & (NU - 1)) * BOXD, &tm_u, tma_col, tma_row + G * g, bar);
    tma_load_2d(ring_f + (g & (NF - 1)) * BOXD, &tm_f, tma_col, tma_row + G * g, bar);
  };

  if (lane == 0) {
    tma_prefetch_desc(&tm_u);
    tma_prefetch_desc(&tm_f);
#pragma unroll 1
    for (int s = 0; s < NF; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll 1
    for (int g = 0; g < NU && g < ngroups; ++g) issue(g);
  }
  __syncwarp();

  double w[T + 2][3][V];  // w[t]: window of stage t (rows of stage t-1); w[T+1] unused
  double rmx[T], dmx[T];
#pragma unroll
  for (int t = 0; t <= T + 1; ++t)
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) w[t][k][v] = 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t) rmx[t] = dmx[t] = 0.0;

  double *out = p.dst + int64_t(rho_b - 2 * T) * p.pitch + lane_col;  // row of tick 0's output

#pragma unroll 1
  for (int g = 0; g < ngroups; ++g) {
    mbar_wait(&bars[g & (NF - 1)], (g >> B::LOG_NF) & 1);
#pragma unroll
    for (int ph = 0; ph < G; ++ph) {
      const int it = G * g + ph;
      const int rho = rho_b + it;
      double num[T + 1][V], yT[V];
      bool bad = false;
      const bool fast_rows = rho >= fast_lo && rho <= fast_hi;
      // stages in descending order: stage t reads its window, then stage t-1
      // writes its output into stage t's free window row (no register copies)
// BCF row-face fix-up after the stages of a slow tick: stage t's output row
// r = rho-2t (w[t+1][ph%3]; row r-1 in w[t+1][(ph+2)%3]) feeds stage t+1, so
// the ghost rows -1 / n0 in that window get the values the per-sweep refresh
// would give them (stage T's row is stored; the ghost kernel refreshes memory
// after the launch).  Rows 0 and n0-1 meet stages >= 2 in slow ticks only.
#define SRJ_BCFIX                                                                             \
  _Pragma("unroll") for (int t = 1; t < T; ++t) {                                             \
    const int r = rho - 2 * t;                                                                \
    double(&cur)[V] = w[t + 1][ph % 3];                                                       \
    double(&prv)[V] = w[t + 1][(ph + 2) % 3];                                                 \
    if (r == 0 && p.bc_kind[0][0]) { /* row -1, already in the window */                      \
      _Pragma("unroll") for (int v = 0; v < V; ++v) if ((colact >> v) & 1u) prv[v] =          \
          bc_ghost(p, 0, 0, cur[v], lane_col + v);                                            \
    }                                                                                         \
    if (r == p.n0 && p.bc_kind[0][1]) { /* row n0, just passed through */                     \
      _Pragma("unroll") for (int v = 0; v < V; ++v) if ((colact >> v) & 1u) cur[v] =          \
          bc_ghost(p, 0, 1, prv[v], lane_col + v);                                            \
    }                                                                                         \
  }
#define SRJ_STAGE(FASTV, EDGEV, SUBV, CNTV)                                                           \
  _Pragma("unroll") for (int t = T; t >= 1; --t) {                                            \
    const int fg = g + ((ph - 2 * t) >= 0 ? 0 : -((2 * t - ph + G - 1) / G));                 \
    const int fr = ph - 2 * t + G * (g - fg);                                                 \
    const double *frow = ring_f + (fg & (NF - 1)) * BOXD + fr * BAND + V * lane;              \
    double(&dst)[V] = (t == T) ? yT : w[t + 1][ph % 3];                                       \
    stage2d<FASTV, EDGEV, VAR, NL, RECIP, SUBV, V, BCF == 1>(p, w[t][ph % 3],                \
                                      w[t][(ph + 1) % 3],                                     \
                                      w[t][(ph + 2) % 3], frow, rho - 2 * t, p.omega[t - 1],  \
                                      lane_col, i0, i1, own_c0, own_c1, f_lo, f_hi, colact,   \
                                      CNTV || (rho - 2 * t >= i0 && rho - 2 * t < i1),           \
                                      t >= 2 ? bcm : 0u,                                         \
                                      dst, num[t],                                            \
                                      rmx[t - 1], dmx[t - 1], bad);                           \
  }                                                                                           \
  if (RECIP && __any_sync(kFull, bad)) {                                                      \
    _Pragma("unroll") for (int t = T; t >= 1; --t) {                                          \
      double(&dst)[V] = (t == T) ? yT : w[t + 1][ph % 3];                                     \
      fix_stage<FASTV, EDGEV, V>(p, w[t][(ph + 1) % 3], num[t], rho - 2 * t, lane_col, colact, \
                                 dst);                                                        \
    }                                                                                         \
  }
      // every stage row of the tick inside the strip: no per-cell count gate
      const bool all_cnt = rho - 2 * T >= i0 && rho - 2 < i1;
      if (band_interior && fast_rows && all_cnt) {
        SRJ_STAGE(true, false, 0, true)
      } else if (band_interior && fast_rows) {
        SRJ_STAGE(true, false, 0, false)
      } else if (band_edge && fast_rows) {
        if (BCF && warp_sub) {
          SRJ_STAGE(true, true, BCF, false)
        } else {
          SRJ_STAGE(true, true, 0, false)
        }
      } else {
        SRJ_STAGE(false, false, BCF, false)
        if (BCF) SRJ_BCFIX
      }
#undef SRJ_BCFIX
#undef SRJ_STAGE
      {  // stage 0: the freshly loaded row enters stage 1's window
        const double *urow = ring_u + (g & (NU - 1)) * BOXD + ph * BAND + V * lane;
#pragma unroll
        for (int v = 0; v < V; v += 2) {
          const double2 q = *reinterpret_cast<const double2 *>(urow + v);
          w[1][ph % 3][v] = q.x;
          w[1][ph % 3][v + 1] = q.y;
        }
      }
      const int rs = rho - 2 * T;  // yT holds stage-T row rs
      if (rs >= i0 && rs < i1) {
        auto store_row = [&](double *o) {
          if (lane_owned) {
#pragma unroll
            for (int v = 0; v < V; v += 2)
              *reinterpret_cast<double2 *>(o + v) = make_double2(yT[v], yT[v + 1]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const int col = lane_col + v;
              if (col >= own_c0 && col < own_c1) o[v] = yT[v];
            }
          }
        };
        store_row(out);
      }
      out += p.pitch;
    }
    __syncwarp();
    if (lane == 0 && g + NU < ngroups) {
      fence_proxy_async();
      issue(g + NU);
    }
  }

  // Slab edge rows (SEND): each lane copies the cells it stored in rows next
  // to a neighbour rank into that neighbour's halo rows -- after the tick
  // loop, so the loop is the plain kernel's (a send test inside it cost 6%).
  if constexpr (SEND) {
    auto send_rows = [&](double *peer, int shift, int rb, int re) {
#pragma unroll 1
      for (int r = max(rb, i0); r < min(re, i1); ++r) {
        const double *srow = p.dst + int64_t(r) * p.pitch + lane_col;
        double *drow = peer + int64_t(r + shift) * p.pitch + lane_col;
        if (lane_owned) {
#pragma unroll
          for (int v = 0; v < V; v += 2)
            *reinterpret_cast<double2 *>(drow + v) = *reinterpret_cast<const double2 *>(srow + v);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int col = lane_col + v;
            if (col >= own_c0 && col < own_c1) drow[v] = srow[v];
          }
        }
      }
    };
    send_rows(p.send.lo, p.send.lo_shift, p.own_b, p.send.lo_end);
    send_rows(p.send.hi, p.send.hi_shift, p.send.hi_beg, p.own_e);
  }

  // per-step norms: in interior bands the fast ticks accumulate every lane
  // (non-owned lanes hold garbage) so only owned lanes vote; edge bands and
  // predicated ticks accumulate owned cells only
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double rl = (!band_interior || lane_owned) ? fabs(rmx[t]) : 0.0;
    const double rm = warp_max(rl);
    double dm;
    if (VAR) {
      dm = warp_max(fabs(dmx[t]));
    } else {
      dm = fabs(__ddiv_rn(__dmul_rn(p.omega[t], rm), p.kc));
    }
    if (lane == 0) {
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm);
    }
  }
}

}  // namespace srj
