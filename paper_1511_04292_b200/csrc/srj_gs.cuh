// srj_gs.cuh -- lexicographic Gauss-Seidel / SOR sweeps (reference _gs2 /
// _gs3, grids.py:426-474), bitwise, as a GPU wavefront.
//
// The reference updates u in place, cell by cell in C order: a cell reads the
// NEW values of its lower neighbours (i-1, j-1[, k-1]) and the OLD values of
// its upper ones.  Flatten the interior rows in C order (R = i in 2D,
// R = i*n1 + j in 3D; the columns are the last axis).  A warp owns 32
// consecutive rows (lane = row) and walks the columns skewed by one per lane:
// at step d lane r relaxes column d - r.  Then
//   left  (j-1): the lane's own previous result (register),
//   up    (row R-1): lane r-1's result of step d-1 (shuffle); lane 0 reads the
//                    previous strip's last row, waiting on its progress;
//                    in 3D the first row of a plane reads its ghost row,
//   right (j+1), down (row R+1), next plane (3D): not yet touched this sweep,
//                    read from memory (lane 31 waits until the next strip has
//                    finished the previous sweep there),
//   previous plane (3D): finished this sweep by an earlier strip (wait),
// which is exactly the reference's order of updates.  Strips trail each other
// by >= 32 columns through per-strip progress counters (release/acquire), so
// consecutive sweeps pipeline; every strip is co-resident (cooperative
// launch), and the waits only point to earlier rows in this sweep or later
// rows in the previous one, so they cannot deadlock.  Operands are loaded
// kPF steps ahead into a register ring (kPF = 14 in 2D / 6 in 3D for constant
// stencils when every strip fits at that occupancy, else 4); right and down
// come from the ring.  Per-cell arithmetic and the masks are the reference's.
#pragma once
#include "srj_device.cuh"

namespace srj {

struct GSParams {
  double *u;             // interior origin (cell (0,0[,0])), updated in place
  const double *f;       // source
  const uint8_t *act;    // mask or nullptr
  const double *coef[7]; // per-cell c, am0, ap0, am1, ap1[, am2, ap2] (VAR)
  double kc[7];          // constant stencil
  double kinv, kinv_lo;  // double-word reciprocal of kc[0] (constant stencil)
  int64_t pitch, plane;
  int n1;                // 3D: rows per plane (axis 1); 2D: unused
  int64_t nrows;         // flattened interior rows
  int ncols;             // last-axis extent
  int nstrips;
  double omega;
  int nsweeps;
  unsigned long long *prog;  // [nstrips] steps completed (zeroed per launch)
  double *norms;             // [nsweeps][2]: (dmax, rmax)
};

// progress is published every kGSPublish<ND> steps (the release is a full
// memory barrier): 32 in 2D (4096^2: 9.9 GLUPS vs 9.5 at 16, 8.9 at 8); 16 in
// 3D, where the next plane's strips wait on it (128^3: 8.5 vs 7.2 at 32)
template <int ND>
constexpr int kGSPublish = ND == 2 ? 32 : 16;
constexpr int kGSPrefetch = 96;  // columns ahead for the L1 prefetch of a lane's rows

__device__ __forceinline__ void prefetch_l1(const void *ptr) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(ptr));
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

// spin until *p >= need (monotone counters), with back-off; traps if stuck
__device__ __forceinline__ unsigned long long wait_ge(const unsigned long long *p,
                                                      unsigned long long need,
                                                      unsigned long long have) {
  uint32_t spins = 0;
  while (have < need) {
    have = ld_acquire_u64(p);
    if (have >= need) break;
    __nanosleep(64);
    if (++spins > (1u << 28)) __trap();
  }
  return have;
}

template <int ND, bool VAR, bool RECIP, bool DEEP>
__global__ void __launch_bounds__(32, (DEEP || VAR) ? 1 : 12) gs_sweep(const __grid_constant__ GSParams p) {
  const int lane = threadIdx.x;
  const int s = blockIdx.x;
  const int64_t R = int64_t(s) * 32 + lane;
  const bool row_ok = R < p.nrows;
  const int64_t Rc = row_ok ? R : p.nrows - 1;
  int64_t off;          // element offset of (row R, column 0)
  bool up_ghost;        // 3D: first row of a plane -> up neighbour is a ghost row
  if (ND == 2) {
    off = Rc * p.pitch;
    up_ghost = false;
  } else {
    const int64_t i = Rc / p.n1, j = Rc % p.n1;
    off = i * p.plane + j * p.pitch;
    up_ghost = (j == 0);
  }
  const int64_t W = int64_t(p.ncols) + 31;  // steps per sweep
  double *u = p.u;
  // strips holding the previous / next plane of this strip's rows (3D)
  int sa0 = -1, sa1 = -1, sb0 = -1, sb1 = -1;
  if (ND == 3) {
    const int64_t r0 = int64_t(s) * 32, r1 = min(r0 + 31, p.nrows - 1);
    if (r0 - p.n1 >= 0) {
      sa0 = int((r0 - p.n1) / 32);
      sa1 = int((r1 - p.n1) / 32);
    }
    if (r0 + p.n1 < p.nrows) {
      sb0 = int((r0 + p.n1) / 32);
      sb1 = int(min(r1 + p.n1, p.nrows - 1) / 32);
    }
  }
  unsigned long long have_up = 0, have_dn = 0, have_pa = 0, have_pb = 0;

  // 3D: last row of a plane -> the down neighbour is a ghost row, not lane r+1
  const bool dn_ghost = (ND == 3) && ((Rc % p.n1) == p.n1 - 1);
  auto clampj = [&](int64_t j) { return min(max(j, int64_t(-1)), int64_t(p.ncols)); };
  const bool need_up_mem = (lane == 0) || up_ghost;
  // ... and the last interior row's down neighbour is the ghost row
  const bool need_dn_mem = (lane == 31) || dn_ghost || (R + 1 >= p.nrows);
  // 3D, planes of < 32 rows: the previous-plane row of some lanes lies in this
  // strip and is written fewer than kPF steps before use -> read it late
  const bool pa_late = (ND == 3) && (R - p.n1 >= int64_t(s) * 32);
  const bool pa_any = __any_sync(kFull, pa_late);  // warp-uniform

  // operands of one step, loaded kPF steps ahead into a register ring
  struct Ops {
    double uc, f, up_mem, dn_mem, pa, pb;
    double c[1 + 2 * ND];
    bool act;
  };
  // ring depth: deeper rings hide more of the per-step latency (4096^2:
  // kPF 4 / 6 / 9 / 14 -> 9.9 / 10.8 / 11.8 / 12.4 GLUPS) within 255
  // registers (2D constant 240-250; the 3D and per-cell rings hold more).
  // The deep rings cost occupancy (8 co-resident warps per SM instead of
  // ~12): grids whose strips do not all fit then take the DEEP=false copy
  // (kPF 4), chosen at launch from the occupancy query (srj_capi.cu launch_gs)
  constexpr int kPF = (VAR || !DEEP) ? 4 : (ND == 2 ? 14 : 6);

#pragma unroll 1
  for (int k = 0; k < p.nsweeps; ++k) {
    const unsigned long long base = (unsigned long long)k * W;
    // wait until step d's operands are final (lane 0 polls, warp-uniform)
    auto wait_for = [&](int64_t d) {
      if (lane == 0) {
        // (the column is clamped to the last one, not skipped: one call
        // covers every step up to d, so the requirement must be monotone)
        const int64_t jl = min(d, int64_t(p.ncols) - 1);
        if (s > 0)  // (a) previous strip's last row, this sweep
          have_up = wait_ge(p.prog + s - 1, base + jl + 32, have_up);
        if (k > 0 && s + 1 < p.nstrips && d - 31 >= 0)  // (b) next strip
          have_dn = wait_ge(p.prog + s + 1, base - W + min(d - 31, int64_t(p.ncols) - 1) + 1,
                            have_dn);
        if (ND == 3) {
          // (c) previous plane, this sweep: rows R-n1 finished column d-lane
          // by their step <= d+31 (capped at the end of the sweep -- never
          // ask for the next one, whose start may wait on this strip)
          const unsigned long long nc = min(base + d + 32, base + W);
          if (sa0 >= 0 && sa0 != s) have_pa = wait_ge(p.prog + sa0, nc, have_pa);
          if (sa1 >= 0 && sa1 != s && sa1 != sa0) wait_ge(p.prog + sa1, nc, 0);
          // (d) next plane, previous sweep: rows R+n1 hold their sweep-(k-1)
          // values at column d-lane
          if (k > 0) {
            const unsigned long long nd = min(base - W + d + 32, base);
            if (sb0 >= 0 && sb0 != s) have_pb = wait_ge(p.prog + sb0, nd, have_pb);
            if (sb1 >= 0 && sb1 != s && sb1 != sb0) wait_ge(p.prog + sb1, nd, 0);
          }
        }
      }
      __syncwarp();
    };
    auto load = [&](int64_t d, Ops &o) {
      const int64_t j = d - lane;
      const int64_t jc = clampj(j);
      const double *row = u + off;
      // own-strip rows are written only by this warp (this SM), so the L1
      // path is coherent for them: one 128-B line serves 16 steps of a lane
      o.uc = row[jc];
      if (need_up_mem) o.up_mem = __ldcg(row - p.pitch + jc);
      if (need_dn_mem) o.dn_mem = __ldcg(row + p.pitch + jc);
      if (ND == 3) {
        if (!pa_late) o.pa = __ldcg(row - p.plane + jc);
        o.pb = __ldcg(row + p.plane + jc);
      }
      const int64_t q = off + jc;
      o.f = __ldg(p.f + q);
      if (VAR) {
#pragma unroll
        for (int a = 0; a < 1 + 2 * ND; ++a) o.c[a] = __ldg(p.coef[a] + q);
      }
      o.act = row_ok && j >= 0 && j < p.ncols && (!p.act || __ldg(p.act + q) != 0);
    };

    double rmx = 0.0, dmx = 0.0;
    double yprev = 0.0;  // this lane's result of the previous step (column j-1)
    // the row's ghost columns are constant during a sweep: keep them in
    // registers so no load sits in the per-step dependency chain
    const double ghost_l = __ldcg(u + off - 1), ghost_r = __ldcg(u + off + p.ncols);
    Ops ring[kPF + 1];
    wait_for(kPF);  // requirements are monotone in the step: one wait covers 0..kPF
#pragma unroll
    for (int q = 0; q <= kPF; ++q) load(q, ring[q]);
#pragma unroll 1
    for (int64_t d0 = 0; d0 < W; d0 += kPF + 1) {
      // one progress wait per ring round, for the farthest step it prefetches
      if (d0 + kPF + 1 < W) wait_for(min(d0 + 2 * kPF + 1, W - 1));
#pragma unroll
      for (int q = 0; q <= kPF; ++q) {
        const int64_t d = d0 + q;
        if (d >= W) break;
        Ops &cur = ring[q];
        const Ops &nxt = ring[(q + 1) % (kPF + 1)];  // step d+1 (column j+1)
        const int64_t j = d - lane;
        // down (row R+1, column j, old) is lane r+1's centre of step d+1
        const double dn_sh = __shfl_down_sync(kFull, nxt.uc, 1);
        const double upn = __shfl_up_sync(kFull, yprev, 1);  // lane r-1, step d-1 = (R-1, j)
        const double upv = need_up_mem ? cur.up_mem : upn;
        const double dnv = need_dn_mem ? cur.dn_mem : dn_sh;
        const double left = (j == 0) ? ghost_l : yprev;
        // own centre of step d+1 = column j+1 (old); the last column's right
        // neighbour is the ghost column (lane 31 reaches it at the sweep's
        // final step, whose successor is never loaded into the ring)
        const double right = (j == p.ncols - 1) ? ghost_r : nxt.uc;
        if (ND == 3 && pa_late) cur.pa = __ldcg(u + off - p.plane + clampj(j));
        double k7[1 + 2 * ND];
#pragma unroll
        for (int a = 0; a < 1 + 2 * ND; ++a) k7[a] = VAR ? cur.c[a] : p.kc[a];
        double rr;
        if (ND == 2)
          rr = resid5(cur.f, k7[0], cur.uc, k7[1], upv, k7[2], dnv, k7[3], left, k7[4], right);
        else
          rr = resid7(cur.f, k7[0], cur.uc, k7[1], cur.pa, k7[2], cur.pb, k7[3], upv, k7[4], dnv,
                      k7[5], left, k7[6], right);
        const double num = __dmul_rn(p.omega, cur.act ? rr : 0.0);
        double dd;
        if (RECIP) {
          dd = div_recip(num, p.kc[0], p.kinv, p.kinv_lo);
          if (recip_unsafe(num)) dd = div_ieee(num, p.kc[0]);
        } else {
          dd = __ddiv_rn(num, cur.act ? k7[0] : 1.0);
        }
        const double y = cur.act ? __dadd_rn(cur.uc, dd) : cur.uc;
        if (cur.act) {
          u[off + j] = y;
          acc_absmax(rmx, rr);
          acc_absmax(dmx, dd);
        }
        yprev = y;
        if (ND == 3 && pa_any) __syncwarp();  // stores before late same-strip plane reads
        // publish (stores of every lane ordered before the release by the
        // warp barrier), then refill this slot with step d+kPF+1
        if ((d % kGSPublish<ND>) == kGSPublish<ND> - 1 || d == W - 1) {
          __syncwarp();
          if (lane == 0) st_release_u64(p.prog + s, base + d + 1);
        }
        if (d + kPF + 1 < W) load(d + kPF + 1, cur);
        // the register ring covers L1/L2 latency only; the lane's own row and
        // its source/coefficient rows stream from HBM (a 4096^2 field is
        // larger than L2), so pull the line kGSPrefetch columns ahead into L1
        // once per line (own rows only: they are written by this warp alone)
        const int64_t jp = j + kGSPrefetch;
        if ((jp & 15) == 0 && jp >= 0 && jp < p.ncols && row_ok) {
          prefetch_l1(u + off + jp);
          prefetch_l1(p.f + off + jp);
          if (VAR) {
#pragma unroll
            for (int a = 0; a < 1 + 2 * ND; ++a) prefetch_l1(p.coef[a] + off + jp);
          }
        }
      }
    }
    const double rm = warp_max(fabs(rmx));
    const double dm = warp_max(fabs(dmx));
    if (lane == 0) {
      global_max(p.norms + 2 * k, dm);
      global_max(p.norms + 2 * k + 1, rm);
    }
  }
}

}  // namespace srj
