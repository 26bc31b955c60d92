// srj_cluster2d.cuh -- persistent small-grid 2D sweep on one thread-block
// cluster (distributed shared memory).
//
// For grids that fit in the cluster's shared memory (e.g. the BASELINE cfg1
// 256^2 and the paper's 300^2 Grad-Shafranov runs) a sweep costs a few hundred
// nanoseconds of work, so separate launches are latency-bound.  Here one
// cluster of C CTAs (up to 16, non-portable size) keeps the whole field on
// chip: CTA c owns rows [c*R, (c+1)*R) in two shared-memory buffers (plus one
// halo row above and below and the ghost columns), and runs every step of a
// chunk inside ONE launch:
//
//   cluster barrier -> pull the neighbours' boundary rows of the current
//   buffer over DSMEM into the halo rows, refresh the physical ghost layers
//   (FIXED / mirror / periodic / face-Dirichlet: refresh_ghosts,
//   grids.py:225-247) -> CTA barrier -> relax all owned cells into the other
//   buffer (the reference's _wj2 arithmetic, grids.py:351-376) -> per-step
//   (dmax, rmax) by warp/CTA max + one atomicMax -> next step.
//
// The source/kappa, per-cell coefficients and mask stay in global memory
// (read-only, L2-resident for these sizes).  At the end the final buffer (with
// refreshed ghosts) is written to the destination field in the padded layout.
#pragma once
#include <cooperative_groups.h>

#include "srj_device.cuh"

namespace srj {

namespace cg = cooperative_groups;

constexpr int kClusterMax = 16;
constexpr int kClusterThreads = 1024;
constexpr int kTX = 128, kTY = 8;    // thread grid over (columns, rows) of a CTA
constexpr int kMaxA = 4, kMaxB = 4;  // => at most 32 rows per CTA, 512 columns

struct Cluster2DParams {
  const double *src;       // interior origin of the input field (padded layout)
  double *dst;             // interior origin of the output field
  const double *f;         // source or kappa
  const uint8_t *act;
  const double *c, *am0, *ap0, *am1, *ap1;  // VAR coefficients (padded layout)
  double kc, kam0, kap0, kam1, kap1;
  double kinv;             // RN(1/kc) for the reciprocal division (RECIP)
  double kinv_lo;      // RN(1/c - kinv): low word of the reciprocal
  int64_t pitch;           // global row pitch (elements)
  int n0, n1;
  int R;                   // rows per CTA
  int sp;                  // shared row pitch (n1 + 2)
  int bc_kind[2][2];
  double bc_value[2][2];
  const double *bc_values[2][2];
  const double *omegas;    // [nsteps] device
  int nsteps;
  double *norms;           // [nsteps][2]
};

template <bool VAR, bool NL, bool RECIP>
__global__ void __launch_bounds__(kClusterThreads, 1)
    sweep2d_cluster(const __grid_constant__ Cluster2DParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smem_d[];
  const int rank = int(cluster.block_rank());
  const int C = int(cluster.num_blocks());
  const int sp = p.sp;
  const int R = p.R;
  const int slab = (R + 2) * sp;  // one buffer: halo row, R rows, halo row
  double *buf[2] = {smem_d, smem_d + slab};
  const int r0 = rank * R;
  const int rows = max(0, min(R, p.n0 - r0));  // owned rows of this CTA
  const int tid = threadIdx.x;
  __shared__ double red[2][kClusterThreads / 32];

  // local (lr, gc) <-> buffer offset: lr in [-1, rows], gc in [-1, n1]
  auto at = [&](int b, int lr, int gc) -> double & { return buf[b][(lr + 1) * sp + gc + 1]; };

  // load owned rows + the ghost/halo rows below and above from the source
  for (int q = tid; q < (rows + 2) * sp; q += blockDim.x) {
    const int lr = q / sp - 1, gc = q % sp - 1;
    const double v = p.src[int64_t(r0 + lr) * p.pitch + gc];
    at(0, lr, gc) = v;
    at(1, lr, gc) = v;
  }

  const int tx = tid % kTX, ty = tid / kTX;
  int cur = 0;
  for (int s = 0; s <= p.nsteps; ++s) {
    cluster.sync();  // every CTA finished writing buffer `cur`
    double *mine = buf[cur];
    // step 0 relaxes the field as loaded: its halo rows came from memory and
    // its ghosts are the caller's (the reference sweeps the given ghosts and
    // refreshes only after each sweep, grids.py:557-558)
    if (s > 0) {
    // ---- halo rows from the neighbours (interior columns only) ----------
    if (rank > 0) {
      const double *up = cluster.map_shared_rank(buf[cur], rank - 1);
      const int urows = R;  // upper neighbour is full
      for (int gc = tid; gc < p.n1; gc += blockDim.x) mine[gc + 1] = up[urows * sp + gc + 1];
    }
    if (r0 + rows < p.n0) {  // a lower neighbour owns row r0+rows
      const double *dn = cluster.map_shared_rank(buf[cur], rank + 1);
      for (int gc = tid; gc < p.n1; gc += blockDim.x)
        mine[(rows + 1) * sp + gc + 1] = dn[1 * sp + gc + 1];
    }
    // ---- physical ghost rows (axis 0) --------------------------------------
    if (rank == 0 && p.bc_kind[0][0] != 0) {
      const int k = p.bc_kind[0][0];
      const double *src_row;
      if (k == 2) {  // periodic: ghost row -1 = global row n0-1 (last owner)
        const int owner = (p.n0 - 1) / R;
        const double *o = cluster.map_shared_rank(buf[cur], owner);
        src_row = o + ((p.n0 - 1 - owner * R) + 1) * sp + 1;
      } else {
        src_row = mine + 1 * sp + 1;  // own row 0
      }
      for (int gc = tid; gc < p.n1; gc += blockDim.x) {
        double g = src_row[gc];
        if (k == 3) {
          const double v = p.bc_values[0][0] ? p.bc_values[0][0][gc] : p.bc_value[0][0];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        mine[gc + 1] = g;
      }
    }
    if (r0 + rows == p.n0 && p.bc_kind[0][1] != 0) {
      const int k = p.bc_kind[0][1];
      const double *src_row;
      if (k == 2) {  // periodic: ghost row n0 = global row 0 (CTA 0)
        const double *o = cluster.map_shared_rank(buf[cur], 0);
        src_row = o + 1 * sp + 1;
      } else {
        src_row = mine + rows * sp + 1;  // own row rows-1
      }
      for (int gc = tid; gc < p.n1; gc += blockDim.x) {
        double g = src_row[gc];
        if (k == 3) {
          const double v = p.bc_values[0][1] ? p.bc_values[0][1][gc] : p.bc_value[0][1];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        mine[(rows + 1) * sp + gc + 1] = g;
      }
    }
    // ---- ghost columns (axis 1) of the owned rows --------------------------
    for (int lr = tid; lr < rows; lr += blockDim.x) {
      for (int side = 0; side < 2; ++side) {
        const int k = p.bc_kind[1][side];
        if (k == 0) continue;
        const int adj = side ? p.n1 - 1 : 0;
        double g = (k == 2) ? at(cur, lr, side ? 0 : p.n1 - 1) : at(cur, lr, adj);
        if (k == 3) {
          const double v =
              p.bc_values[1][side] ? p.bc_values[1][side][r0 + lr] : p.bc_value[1][side];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        at(cur, lr, side ? p.n1 : -1) = g;
      }
    }
    }  // s > 0
    __syncthreads();
    if (s == p.nsteps) break;  // final buffer refreshed; write-out below

    // ---- relax the owned cells into the other buffer -----------------------
    // thread (ty, tx) owns rows ty + kTY*a and columns tx + kTX*b; the source
    // is re-read each step from L1 (the CTA's share is a few tens of KB)
    const double om = p.omegas[s];
    const int nxt = cur ^ 1;
    double dm = 0.0, rm = 0.0;
    bool bad = false;
    auto cell = [&](int lr, int gc, bool ieee) {
      const int64_t g = int64_t(r0 + lr) * p.pitch + gc;
      const double uc = at(cur, lr, gc);
      bool active = true;
      double c = p.kc, a0 = p.kam0, b0 = p.kap0, a1 = p.kam1, b1 = p.kap1;
      if (VAR) {
        c = __ldg(p.c + g);
        a0 = __ldg(p.am0 + g);
        b0 = __ldg(p.ap0 + g);
        a1 = __ldg(p.am1 + g);
        b1 = __ldg(p.ap1 + g);
        if (p.act) active = __ldg(p.act + g) != 0;
      }
      double out = uc;
      if (active) {
        const double fval = __ldg(p.f + g);
        const double s_ = NL ? nl_source(fval, uc) : fval;
        const double rr = resid5(s_, c, uc, a0, at(cur, lr - 1, gc), b0, at(cur, lr + 1, gc), a1,
                                 at(cur, lr, gc - 1), b1, at(cur, lr, gc + 1));
        const double nm = __dmul_rn(om, rr);
        double d;
        if (RECIP && !ieee) {
          d = div_recip(nm, p.kc, p.kinv, p.kinv_lo);
          bad |= recip_unsafe(nm);
        } else {
          d = (RECIP ? div_ieee(nm, c) : __ddiv_rn(nm, c));
        }
        out = __dadd_rn(uc, d);
        acc_max(dm, d);
        acc_max(rm, rr);
      }
      at(nxt, lr, gc) = out;
    };
#pragma unroll
    for (int a = 0; a < kMaxA; ++a)
#pragma unroll
      for (int b = 0; b < kMaxB; ++b) {
        const int lr = ty + kTY * a, gc = tx + kTX * b;
        if (lr < rows && gc < p.n1) cell(lr, gc, false);
      }
    if (RECIP && __any_sync(kFull, bad)) {
      // rare (zero/subnormal/huge/inf/NaN numerators): redo the thread's
      // cells with the IEEE division; the norms are recomputed with them
      dm = 0.0;
      rm = 0.0;
#pragma unroll 1
      for (int a = 0; a < kMaxA; ++a)
#pragma unroll 1
        for (int b = 0; b < kMaxB; ++b) {
          const int lr = ty + kTY * a, gc = tx + kTX * b;
          if (lr < rows && gc < p.n1) cell(lr, gc, true);
        }
    }
    dm = warp_max(dm);
    rm = warp_max(rm);
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = dm;
      red[1][tid >> 5] = rm;
    }
    __syncthreads();
    if (tid < 32) {
      const int nw = blockDim.x / 32;
      double a = tid < nw ? red[0][tid] : 0.0, b = tid < nw ? red[1][tid] : 0.0;
      a = warp_max(a);
      b = warp_max(b);
      if (tid == 0) {
        global_max(p.norms + 2 * s, a);
        global_max(p.norms + 2 * s + 1, b);
      }
    }
    cur = nxt;
  }

  // ---- write the final buffer: owned rows (with ghost columns) and the
  // physical ghost rows of the first / last CTA --------------------------------
  const int lo = (rank == 0) ? -1 : 0;
  const int hi = (r0 + rows == p.n0) ? rows + 1 : rows;
  for (int q = tid; q < (hi - lo) * sp; q += blockDim.x) {
    const int lr = lo + q / sp, gc = q % sp - 1;
    p.dst[int64_t(r0 + lr) * p.pitch + gc] = at(cur, lr, gc);
  }
}

}  // namespace srj
