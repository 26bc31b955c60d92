// srj_sweep2d_vtb.cuh -- two fused 2D 5-point weighted-Jacobi steps (T = 2)
// on per-cell coefficient arrays (the reference's layout: GridProblem
// center/lower/upper and the mask, grids.py:351-376).
//
// The one-sweep kernel (srj_sweep2d_var.cuh) is HBM-bound at 65 B per update
// (u, s, c, four coefficients, the mask byte, u').  Fusing two steps reads the
// seven input arrays once per two updates (32.5 B/update):
//   * a warp streams a 64-column band down a strip of rows (2 cells per lane,
//     double2 loads); bands overlap by 2 columns per side (stage 1 relaxes
//     band columns 1..62, stage 2 the owned columns 2..61; the overlap is
//     recomputed, never stored);
//   * tick rho: stage 1 relaxes row rho-1 from u rows rho-2..rho (registers,
//     west/east by shuffle), stage 2 relaxes row rho-3 from the stage-1 rows
//     rho-4..rho-2 (registers, a 3-row ring); no shared memory, no barrier;
//   * everything the next tick needs -- u of row rho+1, the source,
//     coefficients and mask of row rho (stage 1) and of row rho-2 (stage 2) --
//     is loaded one tick ahead; the stage-2 operands were read two ticks
//     earlier by this warp, so their second read hits L1/L2, not HBM.
// Division is the IEEE one (the centre varies); dmax and rmax per cell.
// Inactive (masked) cells, ghost columns and rows outside [lo_c, hi_c) pass
// their value through; only owned rows and columns are stored and counted.
#pragma once
#include "srj_device.cuh"

namespace srj {

struct VarTB2DParams {
  const double *src;  // interior origin (cell (0,0)) of u^k
  double *dst;        // interior origin of the output buffer
  const double *f;    // source s, or kappa for the nonlinear source
  const uint8_t *act; // mask (padded byte layout) or nullptr
  const double *c, *am0, *ap0, *am1, *ap1;
  int64_t pitch;
  int n0, n1;
  int lo_c, hi_c;     // rows relaxed: [lo_c, hi_c)
  int ld_lo, ld_hi;   // rows present in memory: [ld_lo, ld_hi]
  int own_b, own_e;   // rows stored and counted
  int col_max;        // largest even interior column a double2 load may start at
  int H, nbands, nstrips;
  double omega[2];
  double *norms;      // [2][2]: (dmax, rmax) per step
};

constexpr int kWarps2DVTB = 4;
constexpr int kVTBOwn = 60;  // owned columns per band

template <bool NL>
__global__ void __launch_bounds__(kWarps2DVTB * 32)
    sweep2d_vtb(const __grid_constant__ VarTB2DParams p) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps2DVTB + warp;
  const int band = gw % p.nbands;
  const int strip = gw / p.nbands;
  double rmx[2] = {0.0, 0.0}, dmx[2] = {0.0, 0.0};
  if (strip < p.nstrips) {
    const int i0 = p.own_b + strip * p.H;
    const int i1 = min(i0 + p.H, p.own_e);
    const int col = band * kVTBOwn - 2 + 2 * lane;  // interior column of the lane's first cell
    const int colc = min(col, p.col_max);          // clamped for loads past the row end
    const bool in0 = col >= 0 && col < p.n1, in1 = col + 1 >= 0 && col + 1 < p.n1;
    const bool own_l = lane >= 1 && lane <= 30;  // band columns 2..61
    const int64_t pitch = p.pitch;
    auto ld2 = [](const double *a) { return __ldg(reinterpret_cast<const double2 *>(a)); };
    auto mask2 = [&](int64_t o) -> unsigned {
      if (!p.act) return 3u;
      const unsigned short m = __ldg(reinterpret_cast<const unsigned short *>(p.act + o));
      return (m & 0xffu ? 1u : 0u) | (m >> 8 ? 2u : 0u);
    };
    auto rowc = [&](int r) { return min(max(r, p.ld_lo), p.ld_hi); };
    struct Coef {
      double2 f, c, a0, b0, a1, b1;
      unsigned mk;
    };
    auto load_coef = [&](int r) {
      const int64_t o = int64_t(rowc(r)) * pitch + colc;
      Coef k;
      k.f = ld2(p.f + o);
      k.c = ld2(p.c + o);
      k.a0 = ld2(p.am0 + o);
      k.b0 = ld2(p.ap0 + o);
      k.a1 = ld2(p.am1 + o);
      k.b1 = ld2(p.ap1 + o);
      k.mk = mask2(o);
      return k;
    };
    const double *u = p.src + colc;
    // one relaxation of the lane's two cells of row r: (y, counted r, counted d)
    auto relax_row = [&](int t, int r, const double2 &um, const double2 &uc, const double2 &ud,
                         const Coef &k, double2 &y) {
      double w = __shfl_up_sync(kFull, uc.y, 1);
      double e = __shfl_down_sync(kFull, uc.x, 1);
      const bool row_ok = r >= p.lo_c && r < p.hi_c;
      const bool cnt = own_l && r >= i0 && r < i1;
      const double ucv[2] = {uc.x, uc.y}, umv[2] = {um.x, um.y}, udv[2] = {ud.x, ud.y},
                   fv[2] = {k.f.x, k.f.y}, cv[2] = {k.c.x, k.c.y}, a0v[2] = {k.a0.x, k.a0.y},
                   b0v[2] = {k.b0.x, k.b0.y}, a1v[2] = {k.a1.x, k.a1.y},
                   b1v[2] = {k.b1.x, k.b1.y}, wv[2] = {w, uc.x}, ev[2] = {uc.y, e};
      double yv[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        // lane 0's west / lane 31's east neighbour is outside the band: those
        // two cells are never needed by stage 2 of an owned column
        const bool edge = (v == 0 && lane == 0) || (v == 1 && lane == 31);
        const bool act = row_ok && !edge && (v == 0 ? in0 : in1) && ((k.mk >> v) & 1u);
        const double s = NL ? nl_source(fv[v], ucv[v]) : fv[v];
        const double rr = resid5(s, cv[v], ucv[v], a0v[v], umv[v], b0v[v], udv[v], a1v[v], wv[v],
                                 b1v[v], ev[v]);
        const double d = __ddiv_rn(__dmul_rn(p.omega[t], act ? rr : 0.0), act ? cv[v] : 1.0);
        yv[v] = act ? __dadd_rn(ucv[v], d) : ucv[v];
        if (act && cnt) {
          acc_absmax(rmx[t], rr);
          acc_absmax(dmx[t], d);
        }
      }
      y = make_double2(yv[0], yv[1]);
    };

    // tick rho: stage 1 -> row rho-1, stage 2 -> row rho-3
    const int rb = i0;
    double2 U0 = ld2(u + int64_t(rowc(rb - 2)) * pitch);  // u rows rho-2, rho-1, rho
    double2 U1 = ld2(u + int64_t(rowc(rb - 1)) * pitch);
    double2 U2 = ld2(u + int64_t(rowc(rb)) * pitch);
    Coef K1 = load_coef(rb - 1), K2 = load_coef(rb - 3);  // stage-1 / stage-2 rows
    double2 S0 = make_double2(0.0, 0.0), S1 = S0, S2 = S0;  // stage 1 of rows rho-4..rho-2
    const bool st0 = own_l && in0, st1 = own_l && in1;
#pragma unroll 1
    for (int rho = rb; rho <= i1 + 2; ++rho) {
      // prefetch for tick rho+1
      const double2 Un = ld2(u + int64_t(rowc(rho + 1)) * pitch);
      const Coef K1n = load_coef(rho), K2n = load_coef(rho - 2);
      // stage 2: row rho-3 from stage-1 rows rho-4, rho-3, rho-2
      const int r2 = rho - 3;
      if (r2 >= i0) {
        double2 y;
        relax_row(1, r2, S0, S1, S2, K2, y);
        double *out = p.dst + int64_t(r2) * pitch + col;
        if (st0 && st1) {
          *reinterpret_cast<double2 *>(out) = y;
        } else {
          if (st0) out[0] = y.x;
          if (st1) out[1] = y.y;
        }
      }
      // stage 1: row rho-1 from u rows rho-2, rho-1, rho
      double2 s1;
      relax_row(0, rho - 1, U0, U1, U2, K1, s1);
      U0 = U1;
      U1 = U2;
      U2 = Un;
      S0 = S1;
      S1 = S2;
      S2 = s1;
      K1 = K1n;
      K2 = K2n;
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double rm = warp_max(fabs(rmx[t]));
    const double dm = warp_max(fabs(dmx[t]));
    if (lane == 0) {
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm);
    }
  }
}

}  // namespace srj
