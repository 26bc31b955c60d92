// srj_sweep3d.cuh -- 3D 7-point weighted-Jacobi sweep, the reference _wj3
// (grids.py:379-408) restated for sm_100a.
//
// A warp owns one axis-1 row j and a 64-wide band of the contiguous axis 2; it
// streams down axis 0 keeping u[i-1], u[i], u[i+1] of its row in registers
// (each HBM byte of u read once per sweep), takes the k-1/k+1 neighbours by
// warp shuffle (edge lanes load the band's outer neighbours) and the j-1/j+1
// rows from L1/L2 (they are the neighbouring warps' streams, resident in the
// same block).  The next row and its source are prefetched one tick ahead.
#pragma once
#include "srj_device.cuh"

namespace srj {

struct Sweep3DParams {
  const double *src;   // interior origin (cell (0,0,0))
  double *dst;
  const double *f;     // source or kappa (nonlinear)
  const uint8_t *act;
  const double *coef[7];  // c, am0, ap0, am1, ap1, am2, ap2 (VAR)
  double kc[7];           // constant stencil
  int64_t pitch, plane;
  int n0, n1, n2;
  int lo_c, hi_c, ld_lo, ld_hi, own_b, own_e;
  int H, nbands, nstrips;
  double omega;
  double *norms;          // [2]
};

constexpr int kWarps3D = 8;

template <bool VAR, bool NL>
__global__ void __launch_bounds__(kWarps3D * 32)
    sweep3d(const __grid_constant__ Sweep3DParams p) {
  constexpr int V = 2, BAND = 64;  // cells per lane, cells per warp band
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long gw = long(blockIdx.x) * kWarps3D + warp;
  const int j = int(gw % p.n1);
  const long rest = gw / p.n1;
  const int band = int(rest % p.nbands);
  const int strip = int(rest / p.nbands);
  double dmx = 0.0, rmx = 0.0;
  if (strip < p.nstrips) {
    const int i0 = p.own_b + strip * p.H;
    const int i1 = min(i0 + p.H, p.own_e);
    const int col = band * BAND + V * lane;  // axis-2 index of this lane's first cell
    const bool in0 = col < p.n2, in1 = col + 1 < p.n2;
    const int64_t jo = int64_t(j) * p.pitch + col;
    auto U = [&](int i) { return p.src + int64_t(i) * p.plane + jo; };
    auto ld2 = [](const double *a) { return __ldg(reinterpret_cast<const double2 *>(a)); };

    double2 um = ld2(U(max(i0 - 1, p.ld_lo)));
    double2 uc = ld2(U(i0));
    double2 ud = ld2(U(min(i0 + 1, p.ld_hi)));
    double2 fc = ld2(p.f + int64_t(i0) * p.plane + jo);
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
      // prefetch tick i+1
      const int inext = min(i + 2, p.ld_hi);
      const double2 ud_n = ld2(U(inext));
      const double2 fc_n = ld2(p.f + int64_t(min(i + 1, p.hi_c - 1)) * p.plane + jo);
      const double *row = U(i);
      const double2 uN = ld2(row - p.pitch);
      const double2 uS = ld2(row + p.pitch);
      double west = __shfl_up_sync(kFull, uc.y, 1);
      double east = __shfl_down_sync(kFull, uc.x, 1);
      if (lane == 0) west = row[-1];
      if (lane == 31) east = row[2];
      const bool row_act = (i >= p.lo_c) && (i < p.hi_c);
      const double ucv[2] = {uc.x, uc.y}, umv[2] = {um.x, um.y},
                   udv[2] = {ud.x, ud.y}, nv[2] = {uN.x, uN.y},
                   sv[2] = {uS.x, uS.y}, fv[2] = {fc.x, fc.y};
      const double wv[2] = {west, uc.x}, ev[2] = {uc.y, east};
      const bool inv[2] = {in0, in1};
      double y[2];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        bool act = row_act && inv[v];
        double k[7];
        if constexpr (VAR) {
          const int64_t q = int64_t(i) * p.plane + jo + v;
#pragma unroll
          for (int a = 0; a < 7; ++a) k[a] = __ldg(p.coef[a] + q);
          if (p.act) act = act && (__ldg(p.act + q) != 0);
        } else {
#pragma unroll
          for (int a = 0; a < 7; ++a) k[a] = p.kc[a];
        }
        const double s = NL ? nl_source(fv[v], ucv[v]) : fv[v];
        const double rr = resid7(s, k[0], ucv[v], k[1], umv[v], k[2], udv[v],
                                 k[3], nv[v], k[4], sv[v], k[5], wv[v], k[6], ev[v]);
        const double d = relax(p.omega, rr, k[0]);
        y[v] = act ? __dadd_rn(ucv[v], d) : ucv[v];
        if (act) {
          acc_max(dmx, d);
          acc_max(rmx, rr);
        }
      }
      double *o = p.dst + int64_t(i) * p.plane + jo;
      if (in0 && in1) {
        *reinterpret_cast<double2 *>(o) = make_double2(y[0], y[1]);
      } else if (in0) {
        o[0] = y[0];
      }
      um = uc;
      uc = ud;
      ud = ud_n;
      fc = fc_n;
    }
  }
  dmx = warp_max(dmx);
  rmx = warp_max(rmx);
  if (lane == 0) {
    global_max(p.norms, dmx);
    global_max(p.norms + 1, rmx);
  }
}

}  // namespace srj
