// srj_sweep2d.cuh -- temporally blocked 2D 5-point weighted-Jacobi sweep.
//
// One warp streams a column band of the grid down axis 0 and applies T
// consecutive SRJ steps (each with its own omega_k) in a single pass over HBM:
// stage t (t = 1..T) turns stage t-1 rows into step k+t rows, with a one-row
// lag per stage, entirely in registers.  Horizontal neighbours move with warp
// shuffles; bands overlap by TP >= T columns per side so every owned column is
// exact at stage T (the overlap cells are recomputed, never stored).
//
// Stage-0 rows (u^k) and the source rows arrive through a per-warp ring of
// shared-memory slots filled by the TMA engine (cp.async.bulk, completion on an
// mbarrier per slot); slot of tick tau is recycled after stage T consumed its
// source row at tick tau+T, so the prefetch distance is S-T-1 rows.
//
// Bitwise contract: the arithmetic per cell and step is exactly the reference
// _wj2 (grids.py:351-376); the per-step (dmax, rmax) are max-reductions over
// owned active cells (exact, order-free).  Ghost rows/columns and inactive
// (masked) cells pass their value through unchanged, as the reference does for
// inactive cells (grids.py:374-375) and FIXED ghosts (grids.py:225-247).
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
  static constexpr int V = 2;                    // columns per lane (double2)
  static constexpr int BAND = 32 * V;            // columns per warp
  static constexpr int TP = (T + 1) & ~1;        // overlap, even => 16 B aligned
  static constexpr int OWN = BAND - 2 * TP;      // columns a band owns
  static constexpr int S = (T + 9 > 16) ? 16 : T + 9;  // ring slots
  static constexpr int WARPS = 4;
  static constexpr int SLOT_BYTES = 2 * BAND * 8;      // u row + source row
  static constexpr size_t smem_bytes() {
    return size_t(WARPS) * S * SLOT_BYTES + size_t(WARPS) * S * 8;
  }
};

template <int T, bool VAR, bool NL>
__global__ void __launch_bounds__(Band2D<T>::WARPS * 32)
    sweep2d_tb(const __grid_constant__ Sweep2DParams p) {
  using B = Band2D<T>;
  constexpr int V = B::V, BAND = B::BAND, TP = B::TP, OWN = B::OWN, S = B::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double *ring_u = reinterpret_cast<double *>(smem_raw) + size_t(warp) * S * 2 * BAND;
  double *ring_f = ring_u + S * BAND;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + size_t(B::WARPS) * S * B::SLOT_BYTES) +
                   warp * S;

  const int gw = blockIdx.x * B::WARPS + warp;
  const int band = gw % p.nbands;
  const int strip = gw / p.nbands;
  if (strip >= p.nstrips) return;  // warp-independent kernel: no block barriers

  const int i0 = p.own_b + strip * p.H;
  const int i1 = min(i0 + p.H, p.own_e);
  const int rho_b = max(i0 - T, p.ld_lo);
  const int nticks = i1 + T - rho_b;  // last tick emits stage-T row i1-1
  const int col_band = band * OWN - TP;
  const int own_c0 = band * OWN;
  const int own_c1 = min(own_c0 + OWN, p.n1);
  const int f_lo = p.lo_c, f_hi = p.hi_c - 1;

  auto u_row = [&](int r) {
    r = min(max(r, p.ld_lo), p.ld_hi);
    return p.src + int64_t(r) * p.pitch + col_band;
  };
  auto f_row = [&](int r) {
    r = min(max(r, f_lo), f_hi);
    return p.f + int64_t(r) * p.pitch + col_band;
  };
  auto issue = [&](int slot, int tick) {
    mbar_expect_tx(&bars[slot], B::SLOT_BYTES);
    bulk_g2s(ring_u + slot * BAND, u_row(rho_b + tick), BAND * 8, &bars[slot]);
    bulk_g2s(ring_f + slot * BAND, f_row(rho_b + tick), BAND * 8, &bars[slot]);
  };

  if (lane == 0) {
#pragma unroll 1
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll 1
    for (int s = 0; s < S && s < nticks; ++s) issue(s, s);
  }
  __syncwarp();

  double up[T + 1][V], mid[T + 1][V];
  double dmx[T], rmx[T];
#pragma unroll
  for (int t = 0; t <= T; ++t)
#pragma unroll
    for (int v = 0; v < V; ++v) up[t][v] = mid[t][v] = 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t) dmx[t] = rmx[t] = 0.0;

  const int lane_col = col_band + V * lane;

#pragma unroll 1
  for (int it = 0; it < nticks; ++it) {
    const int rho = rho_b + it;
    const int slot = it % S;
    mbar_wait(&bars[slot], (it / S) & 1);
    double x[V];
    {
      const double2 w = *reinterpret_cast<const double2 *>(ring_u + slot * BAND + V * lane);
      x[0] = w.x;
      x[1] = w.y;
    }
#pragma unroll
    for (int t = 1; t <= T; ++t) {
      const int r = rho - t;
      const int fslot = (it - t + S) % S;
      const double2 fw = *reinterpret_cast<const double2 *>(ring_f + fslot * BAND + V * lane);
      const double fv[V] = {fw.x, fw.y};
      const double west0 = __shfl_up_sync(kFull, mid[t][V - 1], 1);
      const double eastV = __shfl_down_sync(kFull, mid[t][0], 1);
      const bool row_act = (r >= p.lo_c) && (r < p.hi_c);
      const bool row_own = (r >= i0) && (r < i1);
      const int rc = min(max(r, f_lo), f_hi);
      double y[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int col = lane_col + v;
        const double uc = mid[t][v];
        const double uw = (v == 0) ? west0 : mid[t][v - 1];
        const double ue = (v == V - 1) ? eastV : mid[t][v + 1];
        bool act = row_act && (col >= 0) && (col < p.n1);
        double c, a0, b0, a1, b1;
        if constexpr (VAR) {
          const int64_t q = int64_t(rc) * p.pitch + col;
          c = __ldg(p.c + q);
          a0 = __ldg(p.am0 + q);
          b0 = __ldg(p.ap0 + q);
          a1 = __ldg(p.am1 + q);
          b1 = __ldg(p.ap1 + q);
          if (p.act) act = act && (__ldg(p.act + q) != 0);
        } else {
          c = p.kc; a0 = p.kam0; b0 = p.kap0; a1 = p.kam1; b1 = p.kap1;
        }
        const double s = NL ? nl_source(fv[v], uc) : fv[v];
        const double rr = resid5(s, c, uc, a0, up[t][v], b0, x[v], a1, uw, b1, ue);
        const double d = relax(p.omega[t - 1], rr, c);
        y[v] = act ? __dadd_rn(uc, d) : uc;
        if (act && row_own && col >= own_c0 && col < own_c1) {
          acc_max(dmx[t - 1], d);
          acc_max(rmx[t - 1], rr);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        up[t][v] = mid[t][v];
        mid[t][v] = x[v];
        x[v] = y[v];
      }
    }
    // x now holds stage-T row rho-T
    const int rs = rho - T;
    if (rs >= i0 && rs < i1) {
      double *o = p.dst + int64_t(rs) * p.pitch + lane_col;
      const bool ok0 = lane_col >= own_c0 && lane_col < own_c1;
      const bool ok1 = lane_col + 1 >= own_c0 && lane_col + 1 < own_c1;
      if (ok0 && ok1) {
        *reinterpret_cast<double2 *>(o) = make_double2(x[0], x[1]);
      } else {
        if (ok0) o[0] = x[0];
        if (ok1) o[1] = x[1];
      }
    }
    __syncwarp();
    if (lane == 0 && it >= T && it - T + S < nticks) {
      fence_proxy_async();
      issue((it - T) % S, it - T + S);
    }
  }

#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double dm = warp_max(dmx[t]);
    const double rm = warp_max(rmx[t]);
    if (lane == 0) {
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm);
    }
  }
}

}  // namespace srj
