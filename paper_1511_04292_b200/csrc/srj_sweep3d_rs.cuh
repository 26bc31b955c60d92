// srj_sweep3d_rs.cuh -- temporally blocked 3D 7-point sweep, T = 2, with
// REGISTER STREAMING along axis 0 (constant stencil, FIXED faces).
//
// Same tick schedule as sweep3d_tb<2> (stage 1 relaxes plane rho-1, stage 2
// plane rho-3, rho = the plane loaded at this tick; one CTA barrier per
// tick), but every thread owns fixed (j, k) columns of the tile for the whole
// strip, so the i-1 / i / i+1 values of a column never touch shared memory:
//   * u of the column: the new plane is one LDS from the TMA ring, the two
//     older planes are registers (U ring, period 3);
//   * stage-1 results of the column for the last three planes: registers
//     (S ring); only the j+-1 / k+-1 neighbours of stage 2 come from the
//     shared stage-1 window (one STS per stage-1 cell, four LDS per stage-2
//     cell);
//   * the source of the column: one LDS per plane, carried two ticks in
//     registers (F ring) for stage 2.
// The tick loop is unrolled by the ring period 3, so the rings rotate by
// renaming and every shared-memory address is a per-tick base plus an
// immediate.  Per stage-1 cell: 6 LDS + 1 STS; per stage-2 cell: 4 LDS + 1 STG
// (sweep3d_tb: 8 LDS per cell and stage, all addresses recomputed per tick).
//
// Work: persistent CTAs over (tile, plane) segments (see the kernel head).
// Tile (8 warps): stage 2 owns 14 (j) x 64 (k) cells; stage 1 covers the
// 16 x 66 cone around it.  Warp w holds rows a = 2w, 2w+1 of the 16 stage-1
// rows, lanes hold k = lane and lane + 32 (4 columns per thread); the 32
// k-halo cells of stage 1 (k = -1 and 64 of every row) are a fifth column
// slot of warp 0, which has no stage-2 work in row a = 0 (warp 7 neither in
// row 15), so the 8 warps carry 7-8 column slots each.  A 64-wide owned tile
// divides the BASELINE sizes (512, 256) exactly.
//
// Per-cell arithmetic is the reference _wj3 (grids.py:379-408) in the exact
// association order (resid7), with the double-word reciprocal division and
// IEEE fix-ups after a warp vote, as in every constant-stencil kernel.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "srj_device.cuh"
#include "srj_sweep3d_tb.cuh"  // Sweep3DTBParams

namespace srj {

struct RS3D {
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  static constexpr int TJ = 14, TK = 64;  // owned cells per tile (stage 2)
  static constexpr int AJ = 16;           // stage-1 rows (TJ + 2)
  static constexpr int UC = 68, UR = 18;  // u box: k = kb-2 .. kb+65, j = jb-2 .. jb+15
  static constexpr int FC = 68, FR = 16;  // source box: same columns, j = jb-1 .. jb+14
  static constexpr int WC = 68;           // window row stride (stage-1 column b at b+1)
  static constexpr int NS = 4;            // TMA ring slots (u + source per slot)
  static constexpr int U_BYTES = UR * UC * 8, F_BYTES = FR * FC * 8;
  static constexpr int U_TILE = (U_BYTES + 127) / 128 * 16;  // doubles, 128-B aligned
  static constexpr int F_TILE = (F_BYTES + 127) / 128 * 16;
  static constexpr int W_TILE = (AJ * WC * 8 + 127) / 128 * 16;
  static constexpr size_t smem_bytes() {
    // + one window row of slack: rows a = 0 / 15 of stage 2 read a row
    // beyond their window slot (values discarded)
    return size_t(NS * (U_TILE + F_TILE) + 3 * W_TILE + WC) * 8 + NS * 8;
  }
};

// act ? a : b without letting the compiler turn the select into a branch
// around the computation of a (the FP64 chains of the columns must interleave)
__device__ __forceinline__ double sel(bool act, double a, double b) {
  double r;
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\nselp.f64 %0, %1, %2, q;\n}\n"
      : "=d"(r)
      : "d"(a), "d"(b), "r"(int(act)));
  return r;
}

// predicated global store (no branch around the address arithmetic)
__device__ __forceinline__ void st_global_if(double *ptr, double v, bool pred) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}\n" ::"l"(ptr),
      "d"(v), "r"(int(pred))
      : "memory");
}

__device__ __forceinline__ void tma_box_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                           uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

// SEND: slab ranks' copy that also stores the edge planes into the
// neighbours' halo planes (PeerSend).
template <bool NL, bool RECIP, bool SEND = false>
__global__ void __launch_bounds__(RS3D::THREADS, 2)
    sweep3d_rs(const __grid_constant__ Sweep3DTBParams p, const __grid_constant__ CUtensorMap tm_u,
               const __grid_constant__ CUtensorMap tm_f) {
  using B = RS3D;
  constexpr int NS = B::NS, UC = B::UC, FC = B::FC, WC = B::WC;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double *ring_u = reinterpret_cast<double *>(smem_raw);
  double *ring_f = ring_u + NS * B::U_TILE;
  double *win = ring_f + NS * B::F_TILE;
  uint64_t *bar = reinterpret_cast<uint64_t *>(win + 3 * B::W_TILE + WC);

  // Persistent CTAs: the (tile, plane) units of the launch, tile-major, are
  // split into gridDim.x equal contiguous shares; a share is one or two
  // segments (a tile's planes [i0, i1)), each streamed like a strip.  Equal
  // shares instead of whole strips keep every SM busy when the tile count
  // does not fill whole waves (256^3: 76 tiles on 296 slots).
  const int ntiles = p.ntj * p.ntk;
  const int rows = p.own_e - p.own_b;
  const int64_t total = int64_t(ntiles) * rows;
  const int64_t share = (total + gridDim.x - 1) / gridDim.x;
  int64_t u_beg = int64_t(blockIdx.x) * share;
  const int64_t u_end = min(u_beg + share, total);
  if (u_beg >= u_end) return;  // whole CTA exits together
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr int NC = 4;
  const double kc0 = p.kc[0], kc1 = p.kc[1], kc2 = p.kc[2], kc3 = p.kc[3], kc4 = p.kc[4],
               kc5 = p.kc[5], kc6 = p.kc[6];
  const double om1 = p.omega[0], om2 = p.omega[1];
  double rmx1 = 0.0, rmx2 = 0.0;
  int gt0 = 0;  // ticks of earlier segments: ring slot / mbarrier phase of tick it = gt0 + it

#pragma unroll 1
  while (u_beg < u_end) {
  const int tile = int(u_beg / rows);
  const int i0 = p.own_b + int(u_beg - int64_t(tile) * rows);
  const int i1 = p.own_b + int(min(u_end, int64_t(tile + 1) * rows) - int64_t(tile) * rows);
  u_beg = int64_t(tile) * rows + (i1 - p.own_b);
  const int tj = tile / p.ntk, tk = tile % p.ntk;
  const int jb = tj * B::TJ, kb = tk * B::TK;  // first owned (j, k)
  const int rho_b = max(i0 - 2, p.ld_lo);
  const int nticks = i1 + 3 - rho_b;  // last tick: stage 2 emits plane i1 - 1

  auto issue = [&](int q) {  // planes of tick q into ring slot (gt0 + q) % NS
    const int s = (gt0 + q) % NS;
    const int plane = min(max(rho_b + q, p.ld_lo), p.ld_hi);
    const int row = p.tma_row0 + plane * p.rows_per_plane + jb;
    mbar_expect_tx(&bar[s], B::U_BYTES + B::F_BYTES);
    tma_box_2d(ring_u + s * B::U_TILE, &tm_u, p.tma_col0 + kb - 2, row - 2, &bar[s]);
    tma_box_2d(ring_f + s * B::F_TILE, &tm_f, p.tma_col0 + kb - 2, row - 1, &bar[s]);
  };
  if (tid == 0) {
    // the previous segment's last barrier ended every read of the slots
    fence_proxy_async();
#pragma unroll 1
    for (int q = 0; q < NS && q < nticks; ++q) issue(q);
  }

  // Column c = 0..3: stage-1 row a = 2*warp + (c >> 1), column b = lane +
  // 32*(c & 1); (j, k) = (jb - 1 + a, kb + b).  Column 4 (warp 0 only): the
  // stage-1 k-halo, a = lane & 15, b = lane < 16 ? -1 : 64.
  const int a0 = 2 * warp;
  const bool edge = warp == 0;
  const int ae = lane & 15, be = lane < 16 ? -1 : 64;
  unsigned act1 = 0, act2 = 0;  // bit c: stage-1 / stage-2 cell relaxed (in the domain)
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int a = a0 + (c >> 1), b = lane + 32 * (c & 1);
    const int j = jb - 1 + a, k = kb + b;
    const bool in = j >= 0 && j < p.n1 && k < p.n2;
    act1 |= in ? 1u << c : 0u;
    act2 |= (in && a >= 1 && a <= B::TJ) ? 1u << c : 0u;
  }
  {
    const int j = jb - 1 + ae, k = kb + be;
    act1 |= (edge && j >= 0 && j < p.n1 && k >= 0 && k < p.n2) ? 1u << NC : 0u;
  }
  // per-column shared-memory offsets (doubles): u box (a+1, b+2), source box
  // (a, b+2), window (a, b+1); the second column of a row is +32, the second
  // row +1 row
  const int ou = (a0 + 1) * UC + lane + 2;
  const int of = a0 * FC + lane + 2;
  const int ow = a0 * WC + lane + 1;
  const int oue = (ae + 1) * UC + be + 2, ofe = ae * FC + be + 2, owe = ae * WC + be + 1;
  // global offset of column 0's owned cell (row j = jb - 1 + a0)
  const int64_t g0 = int64_t(jb - 1 + a0) * p.pitch + kb + lane;

  double U[3][NC], S[3][NC], F[3][NC], UE[3];
#pragma unroll
  for (int x = 0; x < 3; ++x) {
#pragma unroll
    for (int c = 0; c < NC; ++c) U[x][c] = S[x][c] = F[x][c] = 0.0;
    UE[x] = 0.0;
  }

  // d = (om*rr)/c: double-word reciprocal (flagging numerators it cannot
  // take) or, in the fix-up pass, exact per cell
  auto relaxd = [&](double om, double rr, bool &bad, auto fixc) -> double {
    constexpr bool FIX = decltype(fixc)::value;
    const double num = __dmul_rn(om, rr);
    if (!RECIP) return __ddiv_rn(num, kc0);
    if (FIX) return recip_unsafe(num) ? div_ieee(num, kc0) : div_recip(num, kc0, p.kinv, p.kinv_lo);
    bad |= recip_maybe_unsafe(num);
    return div_recip(num, kc0, p.kinv, p.kinv_lo);
  };

  auto tick = [&](auto phc, int it) {
    constexpr int PH = decltype(phc)::value;           // it % 3
    constexpr int P1 = (PH + 2) % 3, P2 = (PH + 1) % 3;  // ticks it-1, it-2 (it-3 = PH)
    const int g = gt0 + it;
    mbar_wait(&bar[g % NS], (g / NS) & 1);
    const double *un = ring_u + (g % NS) * B::U_TILE;             // plane rho
    const double *uo = ring_u + ((g + NS - 1) % NS) * B::U_TILE;  // plane rho - 1
    const double *fo = ring_f + ((g + NS - 1) % NS) * B::F_TILE;  // source of rho - 1
    double *wnew = win + PH * B::W_TILE;                           // stage 1 of this tick
    const double *w2 = win + P2 * B::W_TILE;                       // stage 1 of tick it - 2
    const int pl1 = rho_b + it - 1, pl2 = rho_b + it - 3;
    const bool pa1 = it >= 1 && pl1 >= 0 && pl1 < p.n0;
    const bool pa2 = it >= 3 && pl2 >= 0 && pl2 < p.n0;
    const bool po1 = pl1 >= i0 && pl1 < i1, po2 = pl2 >= i0 && pl2 < i1;
    double *drow = p.dst + int64_t(pl2) * p.plane + g0;

    // ---- stage 2 (plane rho-3): reads S[PH] (tick it-3) before stage 1
    // overwrites it
    auto stage2 = [&](auto fixc) {
      constexpr bool FIX = decltype(fixc)::value;
      bool bad = false;
      // branch-free over the columns (one select per cell) so the four FP64
      // chains interleave; rows a = 0 / 15 compute discarded values (their
      // window reads stay inside the allocation, see smem_bytes)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int o = ow + (c >> 1) * WC + 32 * (c & 1);
        const bool act = pa2 && ((act2 >> c) & 1u);
        const double c0 = S[P2][c];
        const double sv = NL ? nl_source(F[P2][c], c0) : F[P2][c];
        const double rr = resid7(sv, kc0, c0, kc1, S[PH][c], kc2, S[P1][c], kc3, w2[o - WC],
                                 kc4, w2[o + WC], kc5, w2[o - 1], kc6, w2[o + 1]);
        bool b = false;
        const double y = sel(act, __dadd_rn(c0, relaxd(om2, rr, b, fixc)), c0);
        bad |= act && b;
        // signed running max of |r| (no FP64 op for fabs)
        if (!FIX) rmx2 = (act && po2 && fabs(rr) > fabs(rmx2)) ? rr : rmx2;
        st_global_if(drow + (c >> 1) * p.pitch + 32 * (c & 1), y, act && po2);
      }
      return bad;
    };
    // ---- stage 1 (plane rho-1)
    auto stage1 = [&](auto fixc) {
      constexpr bool FIX = decltype(fixc)::value;
      bool bad = false;
      auto cell = [&](double c0, double um, double up, double f, int q, bool act) {
        const double sv = NL ? nl_source(f, c0) : f;
        const double rr = resid7(sv, kc0, c0, kc1, um, kc2, up, kc3, uo[q], kc4, uo[q + 2 * UC],
                                 kc5, uo[q + UC - 1], kc6, uo[q + UC + 1]);
        bool b = false;
        const double y = sel(act, __dadd_rn(c0, relaxd(om1, rr, b, fixc)), c0);
        bad |= act && b;
        if (!FIX) rmx1 = (act && po1 && fabs(rr) > fabs(rmx1)) ? rr : rmx1;
        return y;
      };
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int o = (c >> 1) * UC + 32 * (c & 1);
        if (!FIX) {
          U[PH][c] = un[ou + o];
          F[PH][c] = fo[of + (c >> 1) * FC + 32 * (c & 1)];
        }
        // q: (a, b+2) of the old plane = the j-1 neighbour
        const double y = cell(U[P1][c], U[P2][c], U[PH][c], F[PH][c], ou + o - UC,
                              pa1 && ((act1 >> c) & 1u));
        S[PH][c] = y;
        wnew[ow + (c >> 1) * WC + 32 * (c & 1)] = y;
      }
      if (edge) {
        if (!FIX) UE[PH] = un[oue];
        wnew[owe] = cell(UE[P1], UE[P2], UE[PH], fo[ofe], oue - UC, pa1 && ((act1 >> NC) & 1u));
      }
      return bad;
    };

    const bool bad2 = stage2(std::false_type{});
    if (RECIP && __any_sync(kFull, bad2)) stage2(std::true_type{});
    // slab edge planes (a few per launch): every thread copies the cells it
    // just stored into the neighbour's halo plane -- outside the stage code,
    // so the hot path keeps its registers and instruction count
    if (SEND && po2 && (pl2 < p.send.lo_end || pl2 >= p.send.hi_beg)) {
      auto send_plane = [&](double *peer, int shift) {
        double *rrow = peer + int64_t(pl2 + shift) * p.plane + g0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int64_t o = (c >> 1) * p.pitch + 32 * (c & 1);
          if (pa2 && ((act2 >> c) & 1u)) rrow[o] = drow[o];
        }
      };
      if (pl2 < p.send.lo_end) send_plane(p.send.lo, p.send.lo_shift);
      if (pl2 >= p.send.hi_beg) send_plane(p.send.hi, p.send.hi_shift);
    }
    const bool bad1 = stage1(std::false_type{});
    if (RECIP && __any_sync(kFull, bad1)) stage1(std::true_type{});
    __syncthreads();
    // slot of tick it-1 is free: load tick it-1+NS into it
    if (tid == 0 && it >= 1 && it - 1 + NS < nticks) {
      fence_proxy_async();
      issue(it - 1 + NS);
    }
  };

#pragma unroll 1
  for (int it = 0; it < nticks; it += 3) {
    tick(std::integral_constant<int, 0>{}, it);
    if (it + 1 >= nticks) break;
    tick(std::integral_constant<int, 1>{}, it + 1);
    if (it + 2 >= nticks) break;
    tick(std::integral_constant<int, 2>{}, it + 2);
  }
  gt0 += nticks;
  }  // segments

  // per-step norms: dmax is monotone in rmax (constant centre)
  const double rm[2] = {warp_max(fabs(rmx1)), warp_max(fabs(rmx2))};
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double dm = fabs(__ddiv_rn(__dmul_rn(p.omega[t], rm[t]), kc0));
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm[t]);
    }
  }
}

}  // namespace srj
