// srj_sweep2d_vtb.cuh -- two fused 2D 5-point weighted-Jacobi steps (T = 2)
// on per-cell coefficient arrays (the reference's layout: GridProblem
// center/lower/upper and the mask, grids.py:351-376).
//
// The one-sweep kernel (srj_sweep2d_var.cuh) is HBM-bound at 65 B per update
// (u, s, c, four coefficients, the mask byte, u').  Fusing two steps reads the
// input arrays once per two updates (32.5 B/update):
//   * a warp streams a 64-column band down a strip of rows (2 cells per lane);
//     bands overlap by 2 columns per side (stage 1 relaxes band columns
//     1..62, stage 2 the owned columns 2..61; the overlap is recomputed,
//     never stored);
//   * tick rho: stage 1 relaxes row rho-1 from u rows rho-2..rho (west/east
//     by shuffle), stage 2 relaxes row rho-3 from the stage-1 rows
//     rho-4..rho-2 (a 3-row register ring); no barrier;
//   * the seven arrays of a row (u, source, c, am0, ap0, am1, ap1) reach
//     shared memory by per-lane asynchronous copies (cp.async, 16 B = the
//     lane's two cells per array) three rows ahead, into a 7-row ring per warp
//     (rows rho-3 .. rho+3); stage 2 re-reads row rho-3's coefficients from
//     the ring, so every input byte crosses HBM once.  A lane only reads what
//     it copied itself, so cp.async.wait_group is the only synchronisation,
//     and no prefetch lives in registers (the first version prefetched one
//     row into registers: 164 registers, 12 warps/SM, latency-bound at 86
//     GLUPS).
// Division: per-cell double-word reciprocals yh = RN(1/c), yl = RN((1 -
// c*yh)/c), precomputed once per plan (vtb_recip below, the host formula of
// the constant-stencil path), feed the 4-op correctly rounded div_recip; cells
// whose centre is outside [2^-100, 2^100] (yh = 0) or whose numerator is
// outside div_recip's range take the IEEE division after a warp vote.  (With
// the IEEE division inline the kernel spent 37% of its instructions in it.)
// dmax and rmax per cell.
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
  const double *yh, *yl;  // per-cell double-word reciprocal of c (padded layout)
  int64_t pitch;
  int n0, n1;
  int lo_c, hi_c;     // rows relaxed: [lo_c, hi_c)
  int ld_lo, ld_hi;   // rows present in memory: [ld_lo, ld_hi]
  int own_b, own_e;   // rows stored and counted
  int col_max;        // largest even interior column a double2 load may start at
  int mcol_max;       // largest 4-aligned interior column a 4-byte mask copy may start at
  int H, nbands, nstrips;
  double omega[2];
  double *norms;      // [2][2]: (dmax, rmax) per step
};

constexpr int kWarps2DVTB = 1;   // one warp per CTA: the ring is per warp
constexpr int kVTBOwn = 60;      // owned columns per band
constexpr int kVTBArrays = 9;    // u, f, c, am0, ap0, am1, ap1, yh, yl
constexpr int kVTBRing = 7;      // rows rho-3 .. rho+3
constexpr int kVTBAhead = 3;     // rows in flight beyond the current one
constexpr int kVTBMaskRow = 80;  // mask bytes per ring row: 17 chunks of 4 (68) + pad
// dynamic shared memory per warp: 32,256 B (7 per SM); with a mask 32,816 B (6)
constexpr size_t kVTBSmem = size_t(kVTBRing) * kVTBArrays * 32 * 16;
constexpr size_t kVTBSmemMask = kVTBSmem + size_t(kVTBRing) * kVTBMaskRow;

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <bool NL>
__global__ void __launch_bounds__(kWarps2DVTB * 32)
    sweep2d_vtb(const __grid_constant__ VarTB2DParams p) {
  extern __shared__ __align__(16) double2 vtb_ring[];  // [slot][array][lane]
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x;
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
    const double *arr[kVTBArrays] = {p.src, p.f, p.c, p.am0, p.ap0, p.am1, p.ap1, p.yh, p.yl};
    auto rowc = [&](int r) { return min(max(r, p.ld_lo), p.ld_hi); };
    // ring slot of row r: (r - i0 + 3) mod 7, advanced incrementally (an
    // integer modulo per access cost ~20 instructions)
    auto wrap = [](int x) { return x >= kVTBRing ? x - kVTBRing : x; };
    auto ring_at = [&](int slot, int k) -> double2 {
      return vtb_ring[(slot * kVTBArrays + k) * 32 + lane];
    };
    // mask bytes of a band row: 17 four-byte chunks from column col0 - 2
    // (4-byte aligned: the padded rows start 16 B past 64-element boundaries
    // and col0 = 60 band - 2), lanes 0..16; lane l's cells are bytes 2l+2, 2l+3
    unsigned char *mring = reinterpret_cast<unsigned char *>(vtb_ring + kVTBRing * kVTBArrays * 32);
    const int col0 = band * kVTBOwn - 2;
    const int mcs = min(col0 - 2 + 4 * lane, p.mcol_max);
    auto issue_slot = [&](int r, int slot) {  // row r -> ring slot (one commit group)
      const int64_t rb = int64_t(rowc(r)) * pitch;
      const int64_t o = rb + colc;
      double2 *dst = vtb_ring + slot * kVTBArrays * 32 + lane;
#pragma unroll
      for (int k = 0; k < kVTBArrays; ++k) cp_async16(dst + k * 32, arr[k] + o);
      if (p.act && lane <= 16) cp_async4(mring + slot * kVTBMaskRow + 4 * lane, p.act + rb + mcs);
      cp_async_commit();
    };
    auto mask_at = [&](int slot) -> unsigned {
      if (!p.act) return 3u;
      const unsigned short m =
          *reinterpret_cast<const unsigned short *>(mring + slot * kVTBMaskRow + 2 * lane + 2);
      return (m & 0xffu ? 1u : 0u) | (m >> 8 ? 2u : 0u);
    };
    // one relaxation of the lane's two cells of row r with the coefficients
    // of ring row r: returns the new pair, counts owned cells
    auto relax_row = [&](int t, int r, int slot, const double2 &um, const double2 &uc,
                         const double2 &ud, unsigned mk) {
      const double2 f = ring_at(slot, 1), c = ring_at(slot, 2), a0 = ring_at(slot, 3),
                    b0 = ring_at(slot, 4), a1 = ring_at(slot, 5), b1 = ring_at(slot, 6),
                    yh = ring_at(slot, 7), yl = ring_at(slot, 8);
      const double w = __shfl_up_sync(kFull, uc.y, 1);
      const double e = __shfl_down_sync(kFull, uc.x, 1);
      const bool row_ok = r >= p.lo_c && r < p.hi_c;
      const bool cnt = own_l && r >= i0 && r < i1;
      const double ucv[2] = {uc.x, uc.y}, umv[2] = {um.x, um.y}, udv[2] = {ud.x, ud.y},
                   fv[2] = {f.x, f.y}, cv[2] = {c.x, c.y}, a0v[2] = {a0.x, a0.y},
                   b0v[2] = {b0.x, b0.y}, a1v[2] = {a1.x, a1.y}, b1v[2] = {b1.x, b1.y},
                   yhv[2] = {yh.x, yh.y}, ylv[2] = {yl.x, yl.y}, wv[2] = {w, uc.x},
                   ev[2] = {uc.y, e};
      double nm[2], d[2], rr[2];
      bool act[2], slow = false;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        // lane 0's west / lane 31's east neighbour is outside the band: those
        // two cells are never needed by stage 2 of an owned column
        const bool edge = (v == 0 && lane == 0) || (v == 1 && lane == 31);
        act[v] = row_ok && !edge && (v == 0 ? in0 : in1) && ((mk >> v) & 1u);
        const double s = NL ? nl_source(fv[v], ucv[v]) : fv[v];
        rr[v] = resid5(s, cv[v], ucv[v], a0v[v], umv[v], b0v[v], udv[v], a1v[v], wv[v], b1v[v],
                       ev[v]);
        nm[v] = __dmul_rn(p.omega[t], rr[v]);
        d[v] = div_recip(nm[v], cv[v], yhv[v], ylv[v]);
        slow |= act[v] && (yhv[v] == 0.0 || recip_unsafe(nm[v]));
      }
      if (__any_sync(kFull, slow)) {  // rare: IEEE division for the flagged cells
#pragma unroll
        for (int v = 0; v < 2; ++v)
          if (act[v] && (yhv[v] == 0.0 || recip_unsafe(nm[v]))) d[v] = div_ieee(nm[v], cv[v]);
      }
      double yv[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        yv[v] = act[v] ? __dadd_rn(ucv[v], d[v]) : ucv[v];
        if (act[v] && cnt) {
          acc_absmax(rmx[t], rr[v]);
          acc_absmax(dmx[t], d[v]);
        }
      }
      return make_double2(yv[0], yv[1]);
    };

    // prologue: rows i0-3 .. i0+2 in flight (the ring holds i0-3 .. i0+3);
    // row i0-3+x lives in slot x
#pragma unroll 1
    for (int x = 0; x < kVTBAhead + 3; ++x) issue_slot(i0 - 3 + x, x);
    int s3 = 0;  // slot of row rho-3 (rho-2: s3+1, rho-1: s3+2, rho: s3+3, rho+3: s3+6, mod 7)
    double2 S0 = make_double2(0.0, 0.0), S1 = S0, S2 = S0;  // stage 1 of rows rho-4..rho-2
    const bool st0 = own_l && in0, st1 = own_l && in1;
#pragma unroll 1
    for (int rho = i0; rho <= i1 + 2; ++rho) {
      const int s2 = wrap(s3 + 1), s1 = wrap(s3 + 2), s0 = wrap(s3 + 3), sn = wrap(s3 + 6);
      issue_slot(rho + kVTBAhead, sn);  // row rho+3 into the slot row rho-4 left
      cp_async_wait<kVTBAhead>();       // rows <= rho have landed
      // stage 2: row rho-3 from stage-1 rows rho-4, rho-3, rho-2
      const int r2 = rho - 3;
      if (r2 >= i0) {
        const double2 y = relax_row(1, r2, s3, S0, S1, S2, mask_at(s3));
        double *out = p.dst + int64_t(r2) * pitch + col;
        if (st0 && st1) {
          *reinterpret_cast<double2 *>(out) = y;
        } else {
          if (st0) out[0] = y.x;
          if (st1) out[1] = y.y;
        }
      }
      // stage 1: row rho-1 from u rows rho-2, rho-1, rho
      const double2 y1 = relax_row(0, rho - 1, s1, ring_at(s2, 0), ring_at(s1, 0),
                                   ring_at(s0, 0), mask_at(s1));
      S0 = S1;
      S1 = S2;
      S2 = y1;
      s3 = s2;
    }
    cp_async_wait<0>();
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

// Per-cell double-word reciprocal of the centre over the interior (padded
// layout; the host's recip_or_zero / recip_lo, bit for bit): yh = RN(1/c)
// for c in [2^-100, 2^100] (else 0 = use the IEEE division), yl = RN((1 -
// c*yh)/c).
static __global__ void vtb_recip(const double *c, double *yh, double *yl, int64_t pitch, int n0, int n1) {
  const int64_t n = int64_t(n0) * n1;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = (q / n1) * pitch + q % n1;
    const double cc = c[o];
    const bool ok = cc >= 0x1p-100 && cc <= 0x1p+100;
    const double h = ok ? __ddiv_rn(1.0, cc) : 0.0;
    yh[o] = h;
    yl[o] = ok ? __ddiv_rn(__fma_rn(-cc, h, 1.0), cc) : 0.0;
  }
}

}  // namespace srj
