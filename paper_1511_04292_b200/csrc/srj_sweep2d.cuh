// srj_sweep2d.cuh -- temporally blocked 2D 5-point weighted-Jacobi sweep.
//
// One warp streams a column band of the grid down axis 0 and applies T
// consecutive SRJ steps (each with its own omega_k) in a single pass over HBM:
// stage t (t = 1..T) turns stage t-1 rows into step k+t rows, with a one-row
// lag per stage, entirely in registers.  Horizontal neighbours move with warp
// shuffles; bands overlap by TP >= T columns per side so every owned column is
// exact at stage T (the overlap cells are recomputed, never stored).
//
// Stage-0 rows (u^k) and the source rows arrive through a per-warp ring of S
// shared-memory slots filled by the TMA engine (cp.async.bulk, completion on
// one mbarrier per slot).  The slot of tick tau is recycled after stage T
// consumed its source row at tick tau+T, so loads run S-T-1 rows ahead.
//
// Instruction economy (the kernel is issue-bound, not HBM-bound, at T>=2):
//  * the row window of each stage rotates by register renaming -- the tick
//    loop is unrolled by 3, the window period;
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
  int64_t pitch;       // elements per row
  int n0, n1;          // interior extents
  int lo_c, hi_c;      // rows that relax (others pass through): [lo_c, hi_c)
  int ld_lo, ld_hi;    // rows present in memory: [ld_lo, ld_hi]
  int own_b, own_e;    // rows stored + counted in the norms
  int H, nbands, nstrips;
  double omega[kMaxFuse];
  double *norms;       // [T][2]: (dmax, rmax) per fused step
};

template <int T>
struct Band2D {
  static constexpr int V = 4;                    // columns per lane
  static constexpr int BAND = 32 * V;            // columns per warp
  static constexpr int TP = (T + V - 1) / V * V; // overlap: whole lanes
  static constexpr int OWN = BAND - 2 * TP;      // columns a band owns
  static constexpr int S = (T + 4 <= 8) ? 8 : 16;  // ring slots (power of 2)
  static constexpr int LOG_S = (S == 8) ? 3 : 4;
  static constexpr int WARPS = 4;
  static constexpr int ROW_BYTES = BAND * 8;
  static constexpr int SLOT_BYTES = 2 * ROW_BYTES;  // u row + source row
  static constexpr size_t smem_bytes() {
    return size_t(WARPS) * S * SLOT_BYTES + size_t(WARPS) * S * 8;
  }
};

// RN(a/c) for a fixed divisor c > 0 with y = RN(1/c), branch-free:
// q0 = RN(a*y) is within 1.5 ulp of a/c; one Markstein correction
// q1 = RN(q0 + RN(a - c*q0)*y) brings it within 1 ulp; with q1 faithful and y
// within 1/2 ulp of 1/c, Markstein's theorem makes r1 = a - c*q1 exact and
// RN(q1 + r1*y) = RN(a/c).  The sign is copied from a, which is exact for
// c > 0 and restores IEEE's -0/c = -0.  Valid for a = +-0 and for normal a
// with exponent in [-899, 899] (no overflow/underflow in q, r); other inputs
// (subnormal, huge, inf, NaN) are flagged by recip_unsafe() and redone with
// the IEEE division after a warp vote (see stage2d).
__device__ __forceinline__ double div_recip(double a, double c, double y) {
  double q = __dmul_rn(a, y);
  double r = __fma_rn(-q, c, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-q, c, a);
  q = __fma_rn(r, y, q);
  const int hi = (__double2hiint(q) & 0x7fffffff) | (__double2hiint(a) & int(0x80000000));
  return __hiloint2double(hi, __double2loint(q));
}

__device__ __forceinline__ bool recip_unsafe(double a) {
  const unsigned hi = unsigned(__double2hiint(a)) & 0x7fffffffu;
  const unsigned e = hi >> 20;
  const bool zero = (hi | unsigned(__double2loint(a))) == 0u;
  return (e - 124u > 1798u) && !zero;  // exponent outside [-899, 899], nonzero
}

// out of line: the IEEE division is the rare path and its inline expansion
// would triple the size of the unrolled fast loop
__device__ __noinline__ double div_ieee(double a, double c) { return __ddiv_rn(a, c); }

// keep the entry of larger magnitude (signed); NaN never replaces m
__device__ __forceinline__ void acc_absmax(double &m, double x) {
  m = (fabs(x) > fabs(m)) ? x : m;
}

// One stage of the fused pipeline for the lane's V cells: the window rows
// (up, mid) hold stage t-1 rows r-1, r; x arrives holding row r+1 and leaves
// holding the stage-t value of row r.
template <bool FAST, bool VAR, bool NL, bool RECIP, int V, int S, int BAND>
__device__ __forceinline__ void stage2d(const Sweep2DParams &p, double (&up)[V], double (&mid)[V],
                                        double (&down)[V], double (&x)[V],
                                        const double *ring_f, int fslot, int lane, int r,
                                        double om, int lane_col, int i0, int i1,
                                        int own_c0, int own_c1, int f_lo, int f_hi, double &rmx,
                                        double &dmx) {
#pragma unroll
  for (int v = 0; v < V; ++v) down[v] = x[v];
  const double *frow = ring_f + (fslot & (S - 1)) * BAND + V * lane;
  double fv[V];
#pragma unroll
  for (int v = 0; v < V; v += 2) {
    const double2 q = *reinterpret_cast<const double2 *>(frow + v);
    fv[v] = q.x;
    fv[v + 1] = q.y;
  }
  const double west0 = __shfl_up_sync(kFull, mid[V - 1], 1);
  const double eastV = __shfl_down_sync(kFull, mid[0], 1);
  bool row_act = true, row_own = true;
  int rc = 0;
  if (!FAST) {
    row_act = (r >= p.lo_c) && (r < p.hi_c);
    row_own = (r >= i0) && (r < i1);
    rc = min(max(r, f_lo), f_hi);
  }
  double num[V], cv[V];
  bool actv[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double uc = mid[v];
    const double uw = (v == 0) ? west0 : mid[v - 1];
    const double ue = (v == V - 1) ? eastV : mid[v + 1];
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
    const double s = NL ? nl_source(fv[v], uc) : fv[v];
    const double rr = resid5(s, c, uc, a0, up[v], b0, down[v], a1, uw, b1, ue);
    num[v] = __dmul_rn(om, rr);
    if (!FAST && !act) num[v] = 0.0;  // passthrough cell: keep garbage off the slow path
    cv[v] = c;
    actv[v] = act;
    if (FAST) {
      acc_absmax(rmx, rr);
    } else if (act && (r >= i0) && (r < i1) && col >= own_c0 && col < own_c1) {
      acc_absmax(rmx, rr);
    }
  }
  double d[V];
  if (RECIP) {
    bool bad = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      d[v] = div_recip(num[v], p.kc, p.kinv);
      bad |= recip_unsafe(num[v]);
    }
    if (__any_sync(kFull, bad)) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (recip_unsafe(num[v])) d[v] = div_ieee(num[v], p.kc);
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) d[v] = __ddiv_rn(num[v], cv[v]);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double uc = mid[v];
    if (FAST) {
      x[v] = __dadd_rn(uc, d[v]);
    } else {
      x[v] = actv[v] ? __dadd_rn(uc, d[v]) : uc;
      if (VAR && actv[v] && row_own && lane_col + v >= own_c0 && lane_col + v < own_c1)
        acc_absmax(dmx, d[v]);
    }
  }
}

template <int T, bool VAR, bool NL, bool RECIP>
__global__ void __launch_bounds__(Band2D<T>::WARPS * 32)
    sweep2d_tb(const __grid_constant__ Sweep2DParams p) {
  using B = Band2D<T>;
  constexpr int V = B::V, BAND = B::BAND, TP = B::TP, OWN = B::OWN, S = B::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double *ring_u = reinterpret_cast<double *>(smem_raw) + size_t(warp) * S * 2 * BAND;
  double *ring_f = ring_u + S * BAND;
  uint64_t *bars =
      reinterpret_cast<uint64_t *>(smem_raw + size_t(B::WARPS) * S * B::SLOT_BYTES) + warp * S;

  const int gw = blockIdx.x * B::WARPS + warp;
  const int band = gw % p.nbands;
  const int strip = gw / p.nbands;
  if (strip >= p.nstrips) return;  // warp-independent kernel: no block barriers

  const int i0 = p.own_b + strip * p.H;
  const int i1 = min(i0 + p.H, p.own_e);
  const int rho_b = max(i0 - T, p.ld_lo);
  const int nreal = i1 + T - rho_b;            // last real tick emits stage-T row i1-1
  const int nticks = (nreal + 2) / 3 * 3;      // extra ticks emit unowned rows only
  const int col_band = band * OWN - TP;
  const int own_c0 = band * OWN;
  const int own_c1 = min(own_c0 + OWN, p.n1);
  const int f_lo = p.lo_c, f_hi = p.hi_c - 1;
  const bool band_interior = (col_band >= 0) && (col_band + BAND <= p.n1) && !VAR;
  // fast ticks: all T stage rows owned and relaxing
  const int fast_lo = max(i0, p.lo_c) + T;     // rho >= fast_lo  <=> rho - T >= ...
  const int fast_hi = min(i1, p.hi_c);         // rho - 1 < fast_hi
  const int lane_col = col_band + V * lane;
  const bool lane_owned = (lane_col >= own_c0) && (lane_col + V <= own_c1);

  auto issue = [&](int slot, int tick) {
    const int r = rho_b + tick;
    const int ru = min(max(r, p.ld_lo), p.ld_hi);
    const int rf = min(max(r, f_lo), f_hi);
    mbar_expect_tx(&bars[slot], B::SLOT_BYTES);
    bulk_g2s(ring_u + slot * BAND, p.src + int64_t(ru) * p.pitch + col_band, B::ROW_BYTES,
             &bars[slot]);
    bulk_g2s(ring_f + slot * BAND, p.f + int64_t(rf) * p.pitch + col_band, B::ROW_BYTES,
             &bars[slot]);
  };

  if (lane == 0) {
#pragma unroll 1
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll 1
    for (int s = 0; s < S && s < nticks; ++s) issue(s, s);
  }
  __syncwarp();

  double w[T + 1][3][V];  // w[t]: 3-row window of stage t's input (stage t-1 rows)
  double rmx[T], dmx[T];
#pragma unroll
  for (int t = 0; t <= T; ++t)
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) w[t][k][v] = 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t) rmx[t] = dmx[t] = 0.0;

#pragma unroll 1
  for (int it0 = 0; it0 < nticks; it0 += 3) {
#pragma unroll
    for (int ph = 0; ph < 3; ++ph) {
      const int it = it0 + ph;
      const int rho = rho_b + it;
      const int slot = it & (S - 1);
      mbar_wait(&bars[slot], (it >> B::LOG_S) & 1);
      double x[V];
      {
        const double *urow = ring_u + slot * BAND + V * lane;
#pragma unroll
        for (int v = 0; v < V; v += 2) {
          const double2 q = *reinterpret_cast<const double2 *>(urow + v);
          x[v] = q.x;
          x[v + 1] = q.y;
        }
      }
      if (band_interior && rho >= fast_lo && rho <= fast_hi) {
#pragma unroll
        for (int t = 1; t <= T; ++t)
          stage2d<true, VAR, NL, RECIP, V, S, BAND>(p, w[t][ph % 3], w[t][(ph + 1) % 3],
                                             w[t][(ph + 2) % 3], x, ring_f, slot - t, lane,
                                             rho - t, p.omega[t - 1], lane_col, i0,
                                             i1, own_c0, own_c1, f_lo, f_hi, rmx[t - 1],
                                             dmx[t - 1]);
      } else {
#pragma unroll
        for (int t = 1; t <= T; ++t)
          stage2d<false, VAR, NL, RECIP, V, S, BAND>(p, w[t][ph % 3], w[t][(ph + 1) % 3],
                                              w[t][(ph + 2) % 3], x, ring_f, slot - t, lane,
                                              rho - t, p.omega[t - 1], lane_col, i0,
                                              i1, own_c0, own_c1, f_lo, f_hi, rmx[t - 1],
                                              dmx[t - 1]);
      }
      const int rs = rho - T;  // x holds stage-T row rs
      if (rs >= i0 && rs < i1) {
        double *o = p.dst + int64_t(rs) * p.pitch + lane_col;
        if (lane_owned) {
#pragma unroll
          for (int v = 0; v < V; v += 2)
            *reinterpret_cast<double2 *>(o + v) = make_double2(x[v], x[v + 1]);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int col = lane_col + v;
            if (col >= own_c0 && col < own_c1) o[v] = x[v];
          }
        }
      }
      __syncwarp();
      if (lane == 0 && it >= T && it - T + S < nticks) {
        fence_proxy_async();
        issue((it - T) & (S - 1), it - T + S);
      }
    }
  }

  // per-step norms: lanes outside the owned columns may hold garbage from
  // fast ticks; they do not vote
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double rl = lane_owned || !band_interior ? fabs(rmx[t]) : 0.0;
    const double rm = warp_max(rl);
    double dm;
    if constexpr (VAR) {
      dm = warp_max(fabs(dmx[t]));
    } else {
      const double num = __dmul_rn(p.omega[t], rm);
      dm = fabs(__ddiv_rn(num, p.kc));
    }
    if (lane == 0) {
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm);
    }
  }
}

}  // namespace srj
