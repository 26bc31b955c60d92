// srj_sweep3d_tb.cuh -- temporally blocked 3D 7-point sweep (constant stencil).
//
// A CTA owns a TJ x TK tile of the (j, k) plane and streams axis 0.  Each
// plane's u and source tile, widened by T cells per side, arrives by one 2D
// TMA copy each (the padded 3D field viewed as a 2D tensor of
// (n0+2)(n1+2) rows) into a ring of NS shared slots.  T stages are applied per
// tick with a CTA barrier between them: stage t relaxes plane tau-t from
// stage t-1 planes tau-t-1 .. tau-t+1 over the tile shrunk by t cells per side
// (the dependency cone), intermediate stages keep their last 3 planes in a
// shared window, and stage T writes the owned cells straight to HBM.  So T
// sweeps cost one read of u and f and one write per owned cell (plus the tile
// halo), like the 2D band kernel.  Per-cell arithmetic is the reference _wj3
// (grids.py:379-408); ghost and inactive positions pass their value through.
#pragma once
#include <cuda.h>

#include "srj_device.cuh"

namespace srj {

struct Sweep3DTBParams {
  double *dst;         // interior origin of the output
  double kc[7];        // constant stencil
  double kinv;         // RN(1/kc[0]) or 0 (IEEE division)
  double kinv_lo;      // RN(1/c - kinv): low word of the reciprocal
  int64_t pitch, plane;
  int n0, n1, n2;
  int ld_lo, ld_hi;    // planes present (interior indices)
  int own_b, own_e;    // owned planes
  int ntj, ntk, nstrips, H;
  int tma_col0;        // tensor column of interior k = 0
  int rows_per_plane;  // n1 + 2
  int tma_row0;        // tensor row of interior (i=0, j=0)
  double omega[kMaxFuse];
  double *norms;       // [T][2]
};

template <int T>
struct Tile3D {
  // T=2: two 256-thread CTAs per SM (113 KB of shared memory each) so one
  // CTA computes while the other drains its stage barrier; T=3 needs the
  // whole shared memory for one 512-thread CTA.
  static constexpr int TJ = T == 2 ? 12 : 16, TK = 64;  // owned cells per tile
  static constexpr int HJ = TJ + 2 * T, HK = TK + 2 * T; // loaded tile
  // A TMA box must start on a 16-B aligned column (an fp64 box at an odd
  // column faults): for odd T the box starts one column left of the tile
  // (KOFF) and is widened to an even number of columns (HS, the smem row
  // stride).  Tile cell (jj, kk) lives at jj * HS + kk + KOFF.
  static constexpr int KOFF = T & 1;
  static constexpr int HS = (HK + KOFF + 1) / 2 * 2;
  static constexpr int L = (T > 2 ? T : 2);              // ticks a slot stays live
  static constexpr int NS = L + 3;                       // slots: prefetch 2 planes
  static constexpr int THREADS = T == 2 ? 256 : 512;
  static constexpr int MINB = T == 2 ? 2 : 1;  // resident CTAs per SM
  // cell slots per thread: stage 1 has the largest region
  static constexpr int UM = ((HJ - 2) * (HK - 2) + THREADS - 1) / THREADS;
  static_assert(UM <= 8, "flag bits hold 8 slots");
  static constexpr int BOX_BYTES = HJ * HS * 8;          // one TMA box (u or f)
  // slot stride padded to 128 B: every TMA destination must be 128-B aligned
  static constexpr int TILE = (HJ * HS + 15) / 16 * 16;  // doubles per slot
  static constexpr size_t smem_bytes() {
    // NS x (u + f) tiles, (T-1) stage windows of 3 planes, NS barriers
    return size_t(NS) * 2 * TILE * 8 + size_t(T > 1 ? T - 1 : 0) * 3 * TILE * 8 +
           size_t(NS) * 8;
  }
};

template <int T, bool NL, bool RECIP>
__global__ void __launch_bounds__(Tile3D<T>::THREADS, Tile3D<T>::MINB)
    sweep3d_tb(const __grid_constant__ Sweep3DTBParams p, const __grid_constant__ CUtensorMap tm_u,
               const __grid_constant__ CUtensorMap tm_f) {
  using B = Tile3D<T>;
  constexpr int HJ = B::HJ, HK = B::HK, TJ = B::TJ, TK = B::TK, NS = B::NS, TILE = B::TILE;
  constexpr int HS = B::HS, KOFF = B::KOFF;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double *ring_u = reinterpret_cast<double *>(smem_raw);  // NS tiles
  double *ring_f = ring_u + NS * TILE;                    // NS tiles
  double *win = ring_f + NS * TILE;                       // (T-1) x 3 tiles
  uint64_t *bars = reinterpret_cast<uint64_t *>(win + (T > 1 ? T - 1 : 0) * 3 * TILE);

  const int tile = blockIdx.x % (p.ntj * p.ntk);
  const int strip = blockIdx.x / (p.ntj * p.ntk);
  if (strip >= p.nstrips) return;  // whole CTA exits together
  const int tj = tile / p.ntk, tk = tile % p.ntk;
  const int j0 = tj * TJ - T, k0 = tk * TK - T;  // interior index of tile cell (0,0)
  const int i0 = p.own_b + strip * p.H;
  const int i1 = min(i0 + p.H, p.own_e);
  const int rho_b = max(i0 - T, p.ld_lo);
  const int nticks = i1 + T - rho_b;
  const int tid = threadIdx.x;

  auto issue = [&](int tick) {
    const int s = tick % NS;
    const int plane = min(max(rho_b + tick, p.ld_lo), p.ld_hi);
    const int row = p.tma_row0 + plane * p.rows_per_plane + j0;
    mbar_expect_tx(&bars[s], 2 * B::BOX_BYTES);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(ring_u + s * TILE)),
        "l"(reinterpret_cast<uint64_t>(&tm_u)), "r"(p.tma_col0 + k0 - KOFF), "r"(row),
        "r"(smem_addr(&bars[s]))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(ring_f + s * TILE)),
        "l"(reinterpret_cast<uint64_t>(&tm_f)), "r"(p.tma_col0 + k0 - KOFF), "r"(row),
        "r"(smem_addr(&bars[s]))
        : "memory");
  };

  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll 1
    for (int s = 0; s < NS && s < nticks; ++s) issue(s);
  }
  __syncthreads();

  // Tick-invariant cell slots: stage t's region (the tile shrunk by t per
  // side) is dealt round-robin to the threads, at most UM cells per thread.
  // Offsets, grid-bounds and owned flags are computed once per CTA.
  constexpr int UM = B::UM;
  int off[T][UM];        // smem offset of the cell, -1 for an empty slot
  unsigned flg[T];       // bit u: inside the grid; bit 8+u: owned (tile interior)
  int64_t goff[UM];      // stage T: global offset of the cell within its plane
#pragma unroll
  for (int t = 1; t <= T; ++t) {
    const int RJ = HJ - 2 * t, RK = HK - 2 * t, NC = RJ * RK;
    flg[t - 1] = 0u;
#pragma unroll
    for (int u = 0; u < UM; ++u) {
      const int q = tid + u * B::THREADS;
      off[t - 1][u] = -1;
      if (t == T) goff[u] = 0;
      if (q < NC) {
        const int jj = t + q / RK, kk = t + q % RK;
        const int j = j0 + jj, k = k0 + kk;
        off[t - 1][u] = jj * HS + kk + KOFF;
        const bool inb = j >= 0 && j < p.n1 && k >= 0 && k < p.n2;
        const bool own = inb && jj >= T && jj < T + TJ && kk >= T && kk < T + TK;
        flg[t - 1] |= (inb ? 1u << u : 0u) | (own ? 1u << (8 + u) : 0u);
        if (t == T) goff[u] = int64_t(j) * p.pitch + k;
      }
    }
  }

  double rmx[T];  // dmax follows from rmax (monotone map, constant stencil)
#pragma unroll
  for (int t = 0; t < T; ++t) rmx[t] = 0.0;

#pragma unroll 1
  for (int it = 0; it < nticks; ++it) {
    const int rho = rho_b + it;
    mbar_wait(&bars[it % NS], (it / NS) & 1);
#pragma unroll
    for (int t = 1; t <= T; ++t) {
      const int pl = rho - t;  // plane this stage relaxes
      // stage t-1 planes pl-1, pl, pl+1
      const double *dn, *md, *up;
      if (t == 1) {
        up = ring_u + ((it - 2 + 2 * NS) % NS) * TILE;
        md = ring_u + ((it - 1 + NS) % NS) * TILE;
        dn = ring_u + (it % NS) * TILE;
      } else {
        const double *w = win + (t - 2) * 3 * TILE;
        up = w + (((pl - 1) % 3 + 3) % 3) * TILE;
        md = w + (((pl) % 3 + 3) % 3) * TILE;
        dn = w + (((pl + 1) % 3 + 3) % 3) * TILE;
      }
      const double *fp = ring_f + ((it - t + 2 * NS) % NS) * TILE;
      double *out = (t < T) ? win + (t - 1) * 3 * TILE + ((pl % 3 + 3) % 3) * TILE : nullptr;
      // whole-plane predicates fold into the per-cell flags
      const unsigned pa = (pl >= 0 && pl < p.n0) ? 0xffu : 0u;
      const unsigned po = (pl >= i0 && pl < i1) ? 0xffu : 0u;
      const unsigned act_m = flg[t - 1] & pa;
      const unsigned own_m = (flg[t - 1] >> 8) & pa & po;
      const double om = p.omega[t - 1];
      double y[UM], num[UM], uc[UM];
      bool bad = false;
#pragma unroll
      for (int u = 0; u < UM; ++u) {
        const int o = off[t - 1][u];
        if (o < 0) continue;
        // branch-free: every slot is computed, inactive ones keep their value
        uc[u] = md[o];
        const bool a = (act_m >> u) & 1u;
        const double sv = NL ? nl_source(fp[o], uc[u]) : fp[o];
        const double rr = resid7(sv, p.kc[0], uc[u], p.kc[1], up[o], p.kc[2], dn[o], p.kc[3],
                                 md[o - HS], p.kc[4], md[o + HS], p.kc[5], md[o - 1], p.kc[6],
                                 md[o + 1]);
        num[u] = __dmul_rn(om, rr);
        double d;
        if (RECIP) {
          d = div_recip(num[u], p.kc[0], p.kinv, p.kinv_lo);
          bad |= a && recip_unsafe(num[u]);
        } else {
          d = __ddiv_rn(num[u], p.kc[0]);
        }
        y[u] = a ? __dadd_rn(uc[u], d) : uc[u];
        if ((own_m >> u) & 1u) acc_max(rmx[t - 1], rr);
      }
      if (RECIP && __any_sync(kFull, bad)) {
#pragma unroll
        for (int u = 0; u < UM; ++u)
          if (off[t - 1][u] >= 0 && (act_m & (1u << u)) && recip_unsafe(num[u]))
            y[u] = __dadd_rn(uc[u], div_ieee(num[u], p.kc[0]));
      }
#pragma unroll
      for (int u = 0; u < UM; ++u) {
        const int o = off[t - 1][u];
        if (o < 0) continue;
        if (t < T) {
          out[o] = y[u];
        } else if (own_m & (1u << u)) {
          p.dst[int64_t(pl) * p.plane + goff[u]] = y[u];
        }
      }
      __syncthreads();
    }
    // slot of tick it - L is no longer read (u: up of stage 1, f: stage T)
    if (tid == 0 && it >= B::L && it - B::L + NS < nticks) {
      fence_proxy_async();
      issue(it - B::L + NS);
    }
  }
  // per-step norms: warp max, then one atomic per warp
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double rm = warp_max(fabs(rmx[t]));
    const double dm = fabs(__ddiv_rn(__dmul_rn(p.omega[t], rm), p.kc[0]));  // monotone in |r|
    if ((tid & 31) == 0) {
      global_max(p.norms + 2 * t, dm);
      global_max(p.norms + 2 * t + 1, rm);
    }
  }
}

}  // namespace srj
