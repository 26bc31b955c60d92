// srj_sweep2d_var.cuh -- one 2D 5-point weighted-Jacobi step on per-cell
// coefficient arrays (the reference's layout: GridProblem center/lower/upper
// and the mask, grids.py:351-376), HBM-bound at 65 B per update.
//
// A warp owns a 64-column band (2 cells per lane) and a strip of rows and
// streams down the rows keeping rows i-1, i, i+1 of u in registers; the
// horizontal neighbours come by warp shuffle (edge lanes load the band's
// outer columns).  Everything row i+1 needs -- u of row i+2, the source, the
// five coefficients and the mask bytes -- is loaded one tick ahead as double2
// (two cells per load), so the per-row dependency chain never waits on HBM.
// The division is the IEEE one (the centre varies per cell); dmax and rmax
// are tracked per cell.  Inactive cells and rows outside the plan's owned
// range pass through / are not stored, exactly as the reference kernel.
#pragma once
#include "srj_device.cuh"

namespace srj {

struct Var2DParams {
  const double *src;  // interior origin (cell (0,0)) of u^k
  double *dst;        // interior origin of the output buffer
  const double *f;    // source s, or kappa for the nonlinear source
  const uint8_t *act; // mask (padded byte layout) or nullptr
  const double *c, *am0, *ap0, *am1, *ap1;
  int64_t pitch;
  int n0, n1;
  int ld_lo, ld_hi;   // rows present in memory: [ld_lo, ld_hi]
  int own_b, own_e;   // rows relaxed, stored and counted
  int H, nbands, nstrips;
  double omega;
  double *norms;      // [2]: (dmax, rmax)
  PeerSend send;      // slab ranks: rows also stored into the neighbours' halos
};

constexpr int kWarps2DVar = 4;

// SEND: slab ranks' copy that also stores the edge rows into the neighbours'
// halo rows (PeerSend).
template <bool NL, bool SEND = false>
__global__ void __launch_bounds__(kWarps2DVar * 32)
    sweep2d_var(const __grid_constant__ Var2DParams p) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps2DVar + warp;
  const int band = gw % p.nbands;
  const int strip = gw / p.nbands;
  double rmx = 0.0, dmx = 0.0;
  if (strip < p.nstrips) {
    const int i0 = p.own_b + strip * p.H;
    const int i1 = min(i0 + p.H, p.own_e);
    const int col = band * 64 + 2 * lane;
    const bool in0 = col < p.n1, in1 = col + 1 < p.n1;
    const int64_t pitch = p.pitch;
    auto ld2 = [](const double *a) { return __ldg(reinterpret_cast<const double2 *>(a)); };
    auto mask2 = [&](int64_t o) -> unsigned {
      if (!p.act) return 3u;
      const unsigned short m = __ldg(reinterpret_cast<const unsigned short *>(p.act + o));
      return (m & 0xffu ? 1u : 0u) | (m >> 8 ? 2u : 0u);
    };
    const double *u = p.src + col;
    // registers: rows i-1, i, i+1 of u and row i's source/coefficients/mask
    double2 um = ld2(u + int64_t(max(i0 - 1, p.ld_lo)) * pitch);
    double2 uc = ld2(u + int64_t(i0) * pitch);
    double2 ud = ld2(u + int64_t(min(i0 + 1, p.ld_hi)) * pitch);
    int64_t o = int64_t(i0) * pitch + col;
    double2 f = ld2(p.f + o), c = ld2(p.c + o), a0 = ld2(p.am0 + o), b0 = ld2(p.ap0 + o),
            a1 = ld2(p.am1 + o), b1 = ld2(p.ap1 + o);
    unsigned mk = mask2(o);
    double *out = p.dst + o;
    // the band-edge neighbours of lanes 0 / 31 (columns col-1 / col+2 of the
    // centre row) come one tick ahead as well: as same-tick loads their
    // latency stalled the whole warp every row
    const bool elane = lane == 0 || lane == 31;
    const int eoff = lane == 0 ? -1 : 2;
    double edge = elane ? __ldg(u + int64_t(i0) * pitch + eoff) : 0.0;
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
      // prefetch tick i+1 (clamped to rows that exist; unused past i1)
      const int inext = min(i + 1, i1 - 1);
      const int64_t on = int64_t(inext) * pitch + col;
      const double2 udn = ld2(u + int64_t(min(i + 2, p.ld_hi)) * pitch);
      const double2 fn = ld2(p.f + on), cn = ld2(p.c + on), a0n = ld2(p.am0 + on),
                    b0n = ld2(p.ap0 + on), a1n = ld2(p.am1 + on), b1n = ld2(p.ap1 + on);
      const unsigned mkn = mask2(on);
      const double edgen = elane ? __ldg(u + int64_t(min(i + 1, p.ld_hi)) * pitch + eoff) : 0.0;
      double west = __shfl_up_sync(kFull, uc.y, 1);
      double east = __shfl_down_sync(kFull, uc.x, 1);
      if (lane == 0) west = edge;
      if (lane == 31) east = edge;
      const double ucv[2] = {uc.x, uc.y}, umv[2] = {um.x, um.y}, udv[2] = {ud.x, ud.y},
                   fv[2] = {f.x, f.y}, cv[2] = {c.x, c.y}, a0v[2] = {a0.x, a0.y},
                   b0v[2] = {b0.x, b0.y}, a1v[2] = {a1.x, a1.y}, b1v[2] = {b1.x, b1.y},
                   wv[2] = {west, uc.x}, ev[2] = {uc.y, east};
      double y[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const bool act = (v == 0 ? in0 : in1) && ((mk >> v) & 1u);
        const double s = NL ? nl_source(fv[v], ucv[v]) : fv[v];
        const double rr = resid5(s, cv[v], ucv[v], a0v[v], umv[v], b0v[v], udv[v], a1v[v], wv[v],
                                 b1v[v], ev[v]);
        const double d = __ddiv_rn(__dmul_rn(p.omega, act ? rr : 0.0), act ? cv[v] : 1.0);
        y[v] = act ? __dadd_rn(ucv[v], d) : ucv[v];
        if (act) {
          acc_absmax(rmx, rr);
          acc_absmax(dmx, d);
        }
      }
      auto store_row = [&](double *o) {
        if (in0 && in1) {
          *reinterpret_cast<double2 *>(o) = make_double2(y[0], y[1]);
        } else if (in0) {
          o[0] = y[0];
        }
      };
      store_row(out);
      if constexpr (SEND) {  // slab edge rows: the same cells into the neighbour's halo row
        if (i < p.send.lo_end) store_row(p.send.lo + int64_t(i + p.send.lo_shift) * pitch + col);
        if (i >= p.send.hi_beg) store_row(p.send.hi + int64_t(i + p.send.hi_shift) * pitch + col);
      }
      out += pitch;
      um = uc;
      uc = ud;
      ud = udn;
      f = fn;
      c = cn;
      a0 = a0n;
      b0 = b0n;
      a1 = a1n;
      b1 = b1n;
      mk = mkn;
      edge = edgen;
    }
  }
  const double rm = warp_max(fabs(rmx));
  const double dm = warp_max(fabs(dmx));
  if (lane == 0) {
    global_max(p.norms, dm);
    global_max(p.norms + 1, rm);
  }
}

}  // namespace srj
