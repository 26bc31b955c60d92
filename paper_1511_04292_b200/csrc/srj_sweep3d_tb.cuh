// srj_sweep3d_tb.cuh -- temporally blocked 3D 7-point sweep (constant
// stencil) with skewed stages: one CTA barrier per tick.
//
// A CTA owns a TJ x TK tile of the (j, k) plane and streams axis 0.  Each
// plane's u and source tile, widened by T cells per side, arrives by one 2D
// TMA copy each (the padded 3D field viewed as a 2D tensor of (n0+2)(n1+2)
// rows).  Stage t at tick it relaxes plane rho - 2t + 1 (rho = the plane
// loaded at tick it) over the tile shrunk by t cells per side (the dependency
// cone):
//   stage 1 reads u planes rho-2 .. rho (u ring) and the source of rho-1;
//   stage t >= 2 reads stage t-1 planes rho-2t .. rho-2t+2, which stage t-1
//   wrote in ticks it-3 .. it-1 (a 4-plane shared window per stage: three
//   being read, one being written this tick);
//   stage T writes the owned cells to HBM.
// Every stage of a tick reads only data of earlier ticks, so the T stages of a
// tick run between the same two barriers.  The source ring holds 2T+1 planes
// (stage T reads the source loaded 2T-1 ticks earlier), the u ring 4.  T
// sweeps cost one read of u and f and one write per owned cell plus the tile
// halo.  Per-cell arithmetic is the reference _wj3 (grids.py:379-408); ghost
// and inactive positions pass their value through.
#pragma once
#include <cuda.h>

#include <type_traits>

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
  // MIRROR / FACE_DIRICHLET faces under fusion (kernel flag BCF): stages
  // 2..T relax every boundary cell against the ghost the per-sweep refresh
  // would hold, computed from the cell's own (previous-stage) value
  int bc_kind[3][2];           // SRJ_BC_* per (axis, side)
  const double *bc_ptr[3][2];  // face_dirichlet value at face position q: bc_ptr[q * bc_step]
  int bc_step[3][2];           // 1: per-position array; 0: the face's scalar
  PeerSend send;               // slab ranks (sweep3d_rs): planes also stored into the neighbours' halos
};

// The refreshed ghost next to boundary cell value adj at face position q
// (ghost_refresh's arithmetic, srj_reduce.cuh).
// BCF == 2: every non-FIXED face is MIRROR (the ghost is the cell itself);
// BCF == 1: the general branch-free form.
template <int BCF>
__device__ __forceinline__ double bc_ghost3(const Sweep3DTBParams &p, int ax, int side,
                                            double adj, int64_t q) {
  if (BCF == 2) return adj;
  const double v = __ldg(p.bc_ptr[ax][side] + q * p.bc_step[ax][side]);
  const double fd = __dsub_rn(__dmul_rn(2.0, v), adj);
  return p.bc_kind[ax][side] == 1 ? adj : fd;
}

template <int T>
struct Tile3D {
  static constexpr int TJ = 12, TK = 64;                  // owned cells per tile
  static constexpr int HJ = TJ + 2 * T, HK = TK + 2 * T;  // loaded tile
  static constexpr int KOFF = T & 1;                      // 16-B aligned TMA origin
  static constexpr int HS = (HK + KOFF + 1) / 2 * 2;      // smem row stride
  static constexpr int NSU = 4;                           // u planes: it-2 .. it+1
  static constexpr int NSF = 2 * T + 1;                   // source: it-2T+1 .. it+1
  static constexpr int NW = 4;                            // window planes per stage
  static constexpr int THREADS = 256;
  static constexpr int UM = ((HJ - 2) * (HK - 2) + THREADS - 1) / THREADS;
  static_assert(UM <= 8, "flag bits hold 8 slots");
  static constexpr int BOX_BYTES = HJ * HS * 8;
  static constexpr int TILE = (HJ * HS + 15) / 16 * 16;  // 128-B aligned slots
  static constexpr int NTILES = NSU + NSF + (T - 1) * NW;
  static constexpr size_t smem_bytes() {
    return size_t(NTILES) * TILE * 8 + size_t(NSU + NSF) * 8;
  }
  static constexpr int MINB = (smem_bytes() + 1024) * 2 <= 233472 ? 2 : 1;
};

template <int T, bool NL, bool RECIP, int BCF>
__global__ void __launch_bounds__(Tile3D<T>::THREADS, Tile3D<T>::MINB)
    sweep3d_tb(const __grid_constant__ Sweep3DTBParams p, const __grid_constant__ CUtensorMap tm_u,
                const __grid_constant__ CUtensorMap tm_f) {
  using B = Tile3D<T>;
  constexpr int HJ = B::HJ, HK = B::HK, TJ = B::TJ, TK = B::TK, TILE = B::TILE;
  constexpr int HS = B::HS, KOFF = B::KOFF, NSU = B::NSU, NSF = B::NSF, NW = B::NW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double *ring_u = reinterpret_cast<double *>(smem_raw);  // NSU tiles
  double *ring_f = ring_u + NSU * TILE;                   // NSF tiles
  double *win = ring_f + NSF * TILE;                      // (T-1) x NW tiles
  uint64_t *bar_u = reinterpret_cast<uint64_t *>(win + (T - 1) * NW * TILE);
  uint64_t *bar_f = bar_u + NSU;

  const int tile = blockIdx.x % (p.ntj * p.ntk);
  const int strip = blockIdx.x / (p.ntj * p.ntk);
  if (strip >= p.nstrips) return;  // whole CTA exits together
  const int tj = tile / p.ntk, tk = tile % p.ntk;
  const int j0 = tj * TJ - T, k0 = tk * TK - T;  // interior index of tile cell (0,0)
  const int i0 = p.own_b + strip * p.H;
  const int i1 = min(i0 + p.H, p.own_e);
  const int rho_b = max(i0 - T, p.ld_lo);
  const int nticks = i1 + 2 * T - 1 - rho_b;  // last tick: stage T emits plane i1-1
  const int tid = threadIdx.x;

  auto load = [&](const CUtensorMap *map, double *dst, uint64_t *bar, int tick) {
    const int plane = min(max(rho_b + tick, p.ld_lo), p.ld_hi);
    const int row = p.tma_row0 + plane * p.rows_per_plane + j0;
    mbar_expect_tx(bar, B::BOX_BYTES);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(p.tma_col0 + k0 - KOFF), "r"(row),
        "r"(smem_addr(bar))
        : "memory");
  };
  auto issue_u = [&](int tick) {
    const int s = tick % NSU;
    load(&tm_u, ring_u + s * TILE, &bar_u[s], tick);
  };
  auto issue_f = [&](int tick) {
    const int s = tick % NSF;
    load(&tm_f, ring_f + s * TILE, &bar_f[s], tick);
  };

  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < NSU + NSF; ++s) mbar_init(&bar_u[s], 1);
    fence_mbar_init();
#pragma unroll 1
    for (int s = 0; s < NSU && s < nticks; ++s) issue_u(s);
#pragma unroll 1
    for (int s = 0; s < NSF && s < nticks; ++s) issue_f(s);
  }
  __syncthreads();

  // tick-invariant cell slots of every stage (as in sweep3d_tb)
  constexpr int UM = B::UM;
  int off[T][UM];
  unsigned flg[T];
  int64_t goff[UM];
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

  // BCF, stages 2..T, 4 bits per slot: the cell is next to a non-FIXED j-1 /
  // j+1 / k-1 / k+1 face (interior cells only); jk = packed (j, k) for the
  // face-value index.  cta_faces: some cell of this tile has such a face.
  unsigned fb[T];
  int jk[T][UM];
  bool cta_faces = false;
#pragma unroll
  for (int t = 1; t <= T; ++t) {
    fb[t - 1] = 0;
    if (!BCF || t == 1) continue;
    const int RK = HK - 2 * t, NC = (HJ - 2 * t) * RK;
#pragma unroll
    for (int u = 0; u < UM; ++u) {
      const int q = tid + u * B::THREADS;
      jk[t - 1][u] = 0;
      if (q >= NC) continue;
      const int j = j0 + t + q / RK, k = k0 + t + q % RK;
      if (j < 0 || j >= p.n1 || k < 0 || k >= p.n2) continue;
      jk[t - 1][u] = (j << 16) | k;  // host: n1 < 2^15, n2 < 2^16 under BCF
      unsigned b = 0;
      if (j == 0 && p.bc_kind[1][0]) b |= 1u;
      if (j == p.n1 - 1 && p.bc_kind[1][1]) b |= 2u;
      if (k == 0 && p.bc_kind[2][0]) b |= 4u;
      if (k == p.n2 - 1 && p.bc_kind[2][1]) b |= 8u;
      fb[t - 1] |= b << (4 * u);
    }
    cta_faces |= fb[t - 1] != 0;
  }
  if (BCF) cta_faces = __syncthreads_or(cta_faces);

  double rmx[T];
#pragma unroll
  for (int t = 0; t < T; ++t) rmx[t] = 0.0;

#pragma unroll 1
  for (int it = 0; it < nticks; ++it) {
    const int rho = rho_b + it;
    mbar_wait(&bar_u[it % NSU], (it / NSU) & 1);
    mbar_wait(&bar_f[it % NSF], (it / NSF) & 1);
    bool bad = false;
    double y[T][UM], num[T][UM], uc[T][UM];
    // SUBV: stages >= 2 substitute the ghosts of non-FIXED faces (tiles
    // holding j/k boundary cells, and the ticks where a stage relaxes plane
    // 0 or n0-1); every other tick runs the FIXED kernel's code
    auto stages = [&](auto subc) {
      constexpr bool SUBV = decltype(subc)::value;
#pragma unroll
      for (int t = 1; t <= T; ++t) {
        const int pl = rho - 2 * t + 1;  // plane this stage relaxes
        const double *dn, *md, *up;
        if (t == 1) {
          up = ring_u + ((it + 2 * NSU - 2) % NSU) * TILE;
          md = ring_u + ((it + NSU - 1) % NSU) * TILE;
          dn = ring_u + (it % NSU) * TILE;
        } else {
          const double *w = win + (t - 2) * NW * TILE;
          up = w + ((pl - 1) & (NW - 1)) * TILE;
          md = w + (pl & (NW - 1)) * TILE;
          dn = w + ((pl + 1) & (NW - 1)) * TILE;
        }
        const double *fp = ring_f + ((it - 2 * t + 1 + 2 * NSF) % NSF) * TILE;
        const unsigned pa = (pl >= 0 && pl < p.n0) ? 0xffu : 0u;
        const unsigned po = (pl >= i0 && pl < i1) ? 0xffu : 0u;
        const unsigned act_m = flg[t - 1] & pa;
        const unsigned own_m = (flg[t - 1] >> 8) & pa & po;
        const double om = p.omega[t - 1];
        const bool plo = SUBV && t >= 2 && pl == 0 && p.bc_kind[0][0];
        const bool phi = SUBV && t >= 2 && pl == p.n0 - 1 && p.bc_kind[0][1];
#pragma unroll
        for (int u = 0; u < UM; ++u) {
          const int o = off[t - 1][u];
          if (o < 0) continue;
          const double c0 = md[o];
          uc[t - 1][u] = c0;
          const bool a = (act_m >> u) & 1u;
          double nu = up[o], nd = dn[o], njm = md[o - HS], njp = md[o + HS], nkm = md[o - 1],
                 nkp = md[o + 1];
          if (SUBV && t >= 2) {
            const unsigned b = a ? (fb[t - 1] >> (4 * u)) & 15u : 0u;
            const int j = jk[t - 1][u] >> 16, k = jk[t - 1][u] & 0xffff;
            const int64_t qi = int64_t(j) * p.n2 + k, qj = int64_t(pl) * p.n2 + k,
                          qk = int64_t(pl) * p.n1 + j;
            if (plo && a) nu = bc_ghost3<BCF>(p, 0, 0, c0, qi);
            if (phi && a) nd = bc_ghost3<BCF>(p, 0, 1, c0, qi);
            if (b & 1u) njm = bc_ghost3<BCF>(p, 1, 0, c0, qj);
            if (b & 2u) njp = bc_ghost3<BCF>(p, 1, 1, c0, qj);
            if (b & 4u) nkm = bc_ghost3<BCF>(p, 2, 0, c0, qk);
            if (b & 8u) nkp = bc_ghost3<BCF>(p, 2, 1, c0, qk);
          }
          const double sv = NL ? nl_source(fp[o], c0) : fp[o];
          const double rr = resid7(sv, p.kc[0], c0, p.kc[1], nu, p.kc[2], nd, p.kc[3], njm,
                                   p.kc[4], njp, p.kc[5], nkm, p.kc[6], nkp);
          num[t - 1][u] = __dmul_rn(om, rr);
          double d;
          if (RECIP) {
            d = div_recip(num[t - 1][u], p.kc[0], p.kinv, p.kinv_lo);
            bad |= a && recip_unsafe(num[t - 1][u]);
          } else {
            d = __ddiv_rn(num[t - 1][u], p.kc[0]);
          }
          y[t - 1][u] = a ? __dadd_rn(c0, d) : c0;
          if ((own_m >> u) & 1u) acc_max(rmx[t - 1], rr);
        }
      }
    };
    bool sub = false;
    if (BCF) {
      sub = cta_faces;
#pragma unroll
      for (int t = 2; t <= T; ++t) {
        const int pl = rho - 2 * t + 1;
        sub |= (pl == 0 && p.bc_kind[0][0]) || (pl == p.n0 - 1 && p.bc_kind[0][1]);
      }
    }
    if (BCF && sub)
      stages(std::integral_constant<bool, true>{});
    else
      stages(std::integral_constant<bool, false>{});
    if (RECIP && __any_sync(kFull, bad)) {
#pragma unroll
      for (int t = 1; t <= T; ++t) {
        const int pl = rho - 2 * t + 1;
        const unsigned act_m = flg[t - 1] & ((pl >= 0 && pl < p.n0) ? 0xffu : 0u);
#pragma unroll
        for (int u = 0; u < UM; ++u)
          if (off[t - 1][u] >= 0 && ((act_m >> u) & 1u) && recip_unsafe(num[t - 1][u]))
            y[t - 1][u] = __dadd_rn(uc[t - 1][u], div_ieee(num[t - 1][u], p.kc[0]));
      }
    }
#pragma unroll
    for (int t = 1; t <= T; ++t) {
      const int pl = rho - 2 * t + 1;
      const bool own_plane = pl >= i0 && pl < i1;
      double *out = (t < T) ? win + (t - 1) * NW * TILE + (pl & (NW - 1)) * TILE : nullptr;
#pragma unroll
      for (int u = 0; u < UM; ++u) {
        const int o = off[t - 1][u];
        if (o < 0) continue;
        if (t < T) {
          out[o] = y[t - 1][u];
        } else if (own_plane && ((flg[t - 1] >> (8 + u)) & 1u)) {
          p.dst[int64_t(pl) * p.plane + goff[u]] = y[t - 1][u];
        }
      }
    }
    __syncthreads();
    // u plane of tick it-2 and source plane of tick it-2T+1 are no longer read
    if (tid == 0) {
      const int nx = it + 2;
      if (nx >= NSU && nx < nticks) {
        fence_proxy_async();
        issue_u(nx);
      }
      if (nx >= NSF && nx < nticks) {
        fence_proxy_async();
        issue_f(nx);
      }
    }
  }

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
