// srj_sweep3d.cuh -- 3D 7-point weighted-Jacobi sweep, the reference _wj3
// (grids.py:379-408) restated for sm_100a.
//
// A warp owns J consecutive axis-1 rows j..j+J-1 and a 64-wide band of the
// contiguous axis 2 (2 cells per lane); it streams down axis 0 keeping planes
// i-1, i, i+1 of its rows in registers (each HBM byte of u read once per
// sweep), takes k-1/k+1 by warp shuffle (edge lanes load the band's outer
// neighbours), and reads only the two rows j-1 and j+J of plane i from L1/L2
// (they are neighbouring warps' streams).  The next plane and its source are
// prefetched one tick ahead.  Constant stencils divide with the branch-free
// reciprocal refinement (div_recip, one warp vote per tick for IEEE fixups)
// and derive dmax from rmax (monotone map), as the 2D kernel does.
#pragma once
#include "srj_device.cuh"

namespace srj {

struct Sweep3DParams {
  const double *src;   // interior origin (cell (0,0,0))
  double *dst;
  const double *f;     // source or kappa (nonlinear)
  const uint8_t *act;
  const double *coef[7];  // c, am0, ap0, am1, ap1, am2, ap2 (VAR)
  int64_t cplane[7];      // CLS: plane stride of each coefficient array, 0 if constant along axis 0
  int ccol[7];            // CLS: 1, or 0 if constant along axis 2 (read at k = 0)
  double kc[7];           // constant stencil
  double kinv;            // RN(1/kc[0]) when the reciprocal path is used
  double kinv_lo;      // RN(1/c - kinv): low word of the reciprocal
  int64_t pitch, plane;
  int n0, n1, n2;
  int lo_c, hi_c, ld_lo, ld_hi, own_b, own_e;
  int H, nbands, nstrips, njg;
  double omega;
  double *norms;          // [2]
  PeerSend send;          // slab ranks: planes also stored into the neighbours' halos
};

constexpr int kWarps3D = 4;
constexpr int kRows3D = 2;  // J: axis-1 rows per warp

// CLS (VAR only): coefficient classes (srj_plan_set_coef_classes) -- arrays
// constant along axis 0 / axis 2 are read at i = 0 / k = 0 (L1 / L2 hits
// instead of HBM); a separate instantiation so the all-per-cell path keeps
// its single offset per cell.
// SEND: slab ranks' copy that also stores the edge planes into the
// neighbours' halo planes (PeerSend).
template <bool VAR, bool NL, bool RECIP, bool CLS = false, bool SEND = false>
__global__ void __launch_bounds__(kWarps3D * 32)
    sweep3d(const __grid_constant__ Sweep3DParams p) {
  constexpr int V = 2, BAND = 64, J = kRows3D;  // cells per lane, cells per band
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long gw = long(blockIdx.x) * kWarps3D + warp;
  const int jg = int(gw % p.njg);
  const long rest = gw / p.njg;
  const int band = int(rest % p.nbands);
  const int strip = int(rest / p.nbands);
  double rmx = 0.0, dmx = 0.0;
  if (strip < p.nstrips) {
    const int i0 = p.own_b + strip * p.H;
    const int i1 = min(i0 + p.H, p.own_e);
    const int j0 = jg * J;
    const int col = band * BAND + V * lane;  // axis-2 index of this lane's first cell
    const bool in0 = col < p.n2, in1 = col + 1 < p.n2;
    const double *base = p.src + int64_t(j0) * p.pitch + col;  // plane 0, row j0
    auto ld2 = [](const double *a) { return __ldg(reinterpret_cast<const double2 *>(a)); };
    auto U = [&](int i, int q) { return base + int64_t(i) * p.plane + int64_t(q) * p.pitch; };
    auto F = [&](int i, int q) {
      return p.f + int64_t(min(max(i, p.lo_c), p.hi_c - 1)) * p.plane +
             int64_t(j0 + q) * p.pitch + col;
    };
    double2 um[J], uc[J], ud[J], fc[J];
#pragma unroll
    for (int q = 0; q < J; ++q) {
      um[q] = ld2(U(max(i0 - 1, p.ld_lo), q));
      uc[q] = ld2(U(i0, q));
      ud[q] = ld2(U(min(i0 + 1, p.ld_hi), q));
      fc[q] = ld2(F(i0, q));
    }
    double *out = p.dst + int64_t(i0) * p.plane + int64_t(j0) * p.pitch + col;
    // the centre plane's rows j0-1 / j0+J and the band-edge cells of lanes
    // 0 / 31 are loaded one tick ahead too (they were same-tick loads whose
    // latency every tick exposed)
    const int eoff = lane == 0 ? -1 : 2;
    const bool elane = lane == 0 || lane == 31;
    double2 nrow = ld2(U(i0, -1)), srow = ld2(U(i0, J));
    double edge[J];
#pragma unroll
    for (int q = 0; q < J; ++q) edge[q] = elane ? __ldg(U(i0, q) + eoff) : 0.0;
    // running pointers of the prefetched planes (row j0): u of plane i+1 and
    // i+2, the source of plane i+1 -- advanced by one plane per tick instead
    // of rebuilt from 64-bit products (clamped at the ends of what exists)
    const double *pu1 = U(min(i0 + 1, p.ld_hi), 0);
    const double *pu2 = U(min(i0 + 2, p.ld_hi), 0);
    const double *pf1 = F(i0 + 1, 0);
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
      // prefetch tick i+1
      double2 udn[J], fcn[J];
      double edgen[J];
      // (the per-cell instantiations keep the rebuilt addresses: with the
      // running pointers they measured 6-15% slower)
      const double *cu1 = VAR ? U(min(i + 1, p.ld_hi), 0) : pu1;
      const double *cu2 = VAR ? U(min(i + 2, p.ld_hi), 0) : pu2;
      const double *cf1 = VAR ? F(i + 1, 0) : pf1;
#pragma unroll
      for (int q = 0; q < J; ++q) {
        udn[q] = ld2(cu2 + q * p.pitch);
        fcn[q] = ld2(cf1 + q * p.pitch);
        edgen[q] = elane ? __ldg(cu1 + q * p.pitch + eoff) : 0.0;
      }
      const double2 nrown = ld2(cu1 - p.pitch);     // row j0-1 of plane i+1
      const double2 srown = ld2(cu1 + J * p.pitch);  // row j0+J of plane i+1
      if (!VAR) {
        if (i + 2 <= p.ld_hi) pu1 += p.plane;
        if (i + 3 <= p.ld_hi) pu2 += p.plane;
        if (i + 1 >= p.lo_c && i + 2 < p.hi_c) pf1 += p.plane;
      }
      double west[J], east[J];
#pragma unroll
      for (int q = 0; q < J; ++q) {
        west[q] = __shfl_up_sync(kFull, uc[q].y, 1);
        east[q] = __shfl_down_sync(kFull, uc[q].x, 1);
        if (lane == 0) west[q] = edge[q];
        if (lane == 31) east[q] = edge[q];
      }
      const bool row_act = (i >= p.lo_c) && (i < p.hi_c);
      double num[J][V], y[J][V];
      bool actv[J][V];
      bool bad = false;
#pragma unroll
      for (int q = 0; q < J; ++q) {
        const double2 nq = (q == 0) ? nrow : uc[q - 1];
        const double2 sq = (q == J - 1) ? srow : uc[q + 1];
        const double ucv[2] = {uc[q].x, uc[q].y}, umv[2] = {um[q].x, um[q].y},
                     udv[2] = {ud[q].x, ud[q].y}, nv[2] = {nq.x, nq.y}, sv[2] = {sq.x, sq.y},
                     fv[2] = {fc[q].x, fc[q].y};
        const double wv[2] = {west[q], uc[q].x}, ev[2] = {uc[q].y, east[q]};
        const bool rowq = row_act && (j0 + q < p.n1);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          bool act = rowq && (v == 0 ? in0 : in1);
          double k[7];
          if (VAR) {
            const int64_t o = int64_t(min(i, p.hi_c - 1)) * p.plane +
                              int64_t(min(j0 + q, p.n1 - 1)) * p.pitch + col + v;
            if (CLS) {
              const int64_t ii = min(i, p.hi_c - 1), oj = int64_t(min(j0 + q, p.n1 - 1)) * p.pitch;
#pragma unroll
              for (int a = 0; a < 7; ++a)
                k[a] = __ldg(p.coef[a] + ii * p.cplane[a] + oj + (col + v) * p.ccol[a]);
            } else {
#pragma unroll
              for (int a = 0; a < 7; ++a) k[a] = __ldg(p.coef[a] + o);
            }
            if (p.act) act = act && (__ldg(p.act + o) != 0);
          } else {
#pragma unroll
            for (int a = 0; a < 7; ++a) k[a] = p.kc[a];
          }
          const double s = NL ? nl_source(fv[v], ucv[v]) : fv[v];
          const double rr = resid7(s, k[0], ucv[v], k[1], umv[v], k[2], udv[v], k[3], nv[v],
                                   k[4], sv[v], k[5], wv[v], k[6], ev[v]);
          double nm = __dmul_rn(p.omega, rr);
          if (!act) nm = 1.0;  // keep garbage off the IEEE fixup path
          double d;
          if (RECIP) {
            d = div_recip(nm, p.kc[0], p.kinv, p.kinv_lo);
            bad |= recip_unsafe(nm);
          } else {
            d = __ddiv_rn(nm, k[0]);
          }
          num[q][v] = nm;
          actv[q][v] = act;
          y[q][v] = act ? __dadd_rn(ucv[v], d) : ucv[v];
          if (act) {
            acc_absmax(rmx, rr);
            if (VAR) acc_absmax(dmx, d);
          }
        }
      }
      if (RECIP && __any_sync(kFull, bad)) {
#pragma unroll
        for (int q = 0; q < J; ++q) {
          const double ucv[2] = {uc[q].x, uc[q].y};
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (actv[q][v] && recip_unsafe(num[q][v]))
              y[q][v] = __dadd_rn(ucv[v], div_ieee(num[q][v], p.kc[0]));
        }
      }
#pragma unroll
      for (int q = 0; q < J; ++q) {
        if (j0 + q < p.n1) {
          auto store_row = [&](double *o) {
            if (in0 && in1) {
              *reinterpret_cast<double2 *>(o) = make_double2(y[q][0], y[q][1]);
            } else if (in0) {
              o[0] = y[q][0];
            }
          };
          store_row(out + int64_t(q) * p.pitch);
          if constexpr (SEND) {  // slab edge planes: the same cells into the neighbour's halo
            const int64_t inplane = int64_t(j0 + q) * p.pitch + col;
            if (i < p.send.lo_end)
              store_row(p.send.lo + int64_t(i + p.send.lo_shift) * p.plane + inplane);
            if (i >= p.send.hi_beg)
              store_row(p.send.hi + int64_t(i + p.send.hi_shift) * p.plane + inplane);
          }
        }
        um[q] = uc[q];
        uc[q] = ud[q];
        ud[q] = udn[q];
        fc[q] = fcn[q];
        edge[q] = edgen[q];
      }
      nrow = nrown;
      srow = srown;
      out += p.plane;
    }
  }
  const double rm = warp_max(fabs(rmx));
  double dm;
  if (VAR) {
    dm = warp_max(fabs(dmx));
  } else {
    dm = fabs(__ddiv_rn(__dmul_rn(p.omega, rm), p.kc[0]));
  }
  if (lane == 0) {
    global_max(p.norms, dm);
    global_max(p.norms + 1, rm);
  }
}

}  // namespace srj
