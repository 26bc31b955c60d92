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
//   relax the CTA's cells into the other buffer (the reference's _wj2
//   arithmetic, grids.py:351-376); the cells of the first / last owned row
//   are also STORED straight into the neighbours' halo rows of that buffer
//   over DSMEM (push: no remote load on the critical path) -> per-warp
//   (dmax, rmax) into a shared slot -> cluster barrier (split arrive / wait)
//   -> warp 0 folds the previous step's slots into the norm buffer while the
//   others go on -> refresh the physical ghost layers when a face is not
//   FIXED (mirror / periodic / face-Dirichlet: refresh_ghosts,
//   grids.py:225-247; one CTA barrier) -> next step.
// Cells are spread densely over the 1024 threads (cell q = tid + 1024 k of
// the CTA's rows x n1, row = q * ceil(2^32 / n1) >> 32), and both buffers are
// indexed off the shared-memory symbol, so every field access is an LDS with
// an immediate neighbour offset.
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
  int f_smem;              // the source (or kappa) of the owned cells sits in a third shared slab
  unsigned n1_magic;       // ceil(2^32 / n1): row of cell q = umulhi(q, n1_magic)
  double *norms;           // [nsteps][2]
};

template <bool VAR, bool NL, bool RECIP>
__global__ void __launch_bounds__(kClusterThreads, 1)
    sweep2d_cluster(const __grid_constant__ Cluster2DParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smem_d[];
  const int rank = int(cluster.block_rank());
  const int sp = p.sp;
  const int R = p.R;
  const int slab = (R + 2) * sp;  // one buffer: halo row, R rows, halo row
  const int r0 = rank * R;
  const int rows = max(0, min(R, p.n0 - r0));  // owned rows of this CTA
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  __shared__ double red[2][2][kClusterThreads / 32];  // [step parity][dmax, rmax][warp]
  const bool has_up = rank > 0, has_dn = r0 + rows < p.n0;
  // neighbours' buffers (DSMEM): the push targets of the first / last row
  double *up_buf = has_up ? cluster.map_shared_rank(smem_d, rank - 1) : nullptr;
  double *dn_buf = has_dn ? cluster.map_shared_rank(smem_d, rank + 1) : nullptr;
  // local (lr, gc) -> buffer offset: lr in [-1, rows], gc in [-1, n1]
  auto off = [&](int lr, int gc) { return (lr + 1) * sp + gc + 1; };

  // load owned rows + the ghost/halo rows below and above from the source
  for (int q = tid; q < (rows + 2) * sp; q += blockDim.x) {
    const int lr = q / sp - 1, gc = q % sp - 1;
    const double v = p.src[int64_t(r0 + lr) * p.pitch + gc];
    smem_d[off(lr, gc)] = v;
    smem_d[slab + off(lr, gc)] = v;
    // the source does not change between steps: one global read per launch
    // instead of one (L2 latency, every step) per cell and step
    if (p.f_smem)
      smem_d[2 * slab + off(lr, gc)] = (lr >= 0 && lr < rows && gc >= 0 && gc < p.n1)
                                           ? p.f[int64_t(r0 + lr) * p.pitch + gc]
                                           : 0.0;
  }
  cluster.sync();  // every buffer loaded before the first pushes land in it

  const bool phys = p.bc_kind[0][0] | p.bc_kind[0][1] | p.bc_kind[1][0] | p.bc_kind[1][1];
  const int ncell = rows * p.n1;
  const int kfull = ncell / kClusterThreads;   // passes in which every thread has a cell
  const int tail = ncell - kfull * kClusterThreads;
  int cur = 0;
#pragma unroll 1
  for (int s = 0; s < p.nsteps; ++s) {
    // ---- relax the owned cells into the other buffer -----------------------
    const double om = p.omegas[s];
    const int bc = cur * slab, bn = slab - bc;  // current / next buffer offsets
    double dm = 0.0, rm = 0.0;
    bool bad = false;
    auto cell = [&](int q, bool ieee) {
      const int lr = int(__umulhi(unsigned(q), p.n1_magic));
      const int gc = q - lr * p.n1;
      const int o = off(lr, gc);
      const int g = (r0 + lr) * int(p.pitch) + gc;  // small grids: 32-bit index
      const double uc = smem_d[bc + o];
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
        const double fval = p.f_smem ? smem_d[2 * slab + o] : __ldg(p.f + g);
        const double s_ = NL ? nl_source(fval, uc) : fval;
        const double rr = resid5(s_, c, uc, a0, smem_d[bc + o - sp], b0, smem_d[bc + o + sp], a1,
                                 smem_d[bc + o - 1], b1, smem_d[bc + o + 1]);
        const double nm = __dmul_rn(om, rr);
        double d;
        if (RECIP && !ieee) {
          d = div_recip(nm, p.kc, p.kinv, p.kinv_lo);
          bad |= recip_maybe_unsafe(nm);
        } else {
          d = (RECIP ? (recip_unsafe(nm) ? div_ieee(nm, c) : div_recip(nm, p.kc, p.kinv,
                                                                        p.kinv_lo))
                     : __ddiv_rn(nm, c));
        }
        out = __dadd_rn(uc, d);
        acc_max(dm, d);
        acc_max(rm, rr);
      }
      smem_d[bn + o] = out;
      // push the first / last owned row into the neighbours' halo rows
      if (lr == 0 && has_up) up_buf[bn + off(R, gc)] = out;
      if (lr == rows - 1 && has_dn) dn_buf[bn + off(-1, gc)] = out;
    };
#pragma unroll 4
    for (int k = 0; k < kfull; ++k) cell(tid + k * kClusterThreads, false);
    if (tid < tail) cell(tid + kfull * kClusterThreads, false);
    if (RECIP && __any_sync(kFull, bad)) {
      // rare (zero/subnormal/huge/inf/NaN numerators): redo the thread's
      // cells with the exact test; the norms are recomputed with them
      dm = 0.0;
      rm = 0.0;
#pragma unroll 1
      for (int k = 0; k < kfull; ++k) cell(tid + k * kClusterThreads, true);
      if (tid < tail) cell(tid + kfull * kClusterThreads, true);
    }
    dm = warp_max(dm);
    rm = warp_max(rm);
    if ((tid & 31) == 0) {
      red[s & 1][0][warp] = dm;
      red[s & 1][1][warp] = rm;
    }
    // every CTA finished writing (and pushing into) buffer `bn`
    cluster.barrier_arrive();
    cluster.barrier_wait();
    if (warp == 0) {  // fold this step's warp maxima (slots of the other parity stay free)
      const int nw = blockDim.x / 32;
      double a = tid < nw ? red[s & 1][0][tid] : 0.0, b = tid < nw ? red[s & 1][1][tid] : 0.0;
      a = warp_max(a);
      b = warp_max(b);
      if (tid == 0) {
        global_max(p.norms + 2 * s, a);
        global_max(p.norms + 2 * s + 1, b);
      }
    }
    cur ^= 1;
    if (!phys) continue;
    // ---- physical ghost layers of the new buffer (non-FIXED faces) ---------
    const int bm = cur * slab;
    if (rank == 0 && p.bc_kind[0][0] != 0) {
      const int k = p.bc_kind[0][0];
      const double *src_row;
      if (k == 2) {  // periodic: ghost row -1 = global row n0-1 (last owner)
        const int owner = (p.n0 - 1) / R;
        const double *o = cluster.map_shared_rank(smem_d, owner);
        src_row = o + bm + off(p.n0 - 1 - owner * R, 0);
      } else {
        src_row = smem_d + bm + off(0, 0);  // own row 0
      }
      for (int gc = tid; gc < p.n1; gc += blockDim.x) {
        double g = src_row[gc];
        if (k == 3) {
          const double v = p.bc_values[0][0] ? p.bc_values[0][0][gc] : p.bc_value[0][0];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        smem_d[bm + off(-1, gc)] = g;
      }
    }
    if (r0 + rows == p.n0 && p.bc_kind[0][1] != 0) {
      const int k = p.bc_kind[0][1];
      const double *src_row;
      if (k == 2) {  // periodic: ghost row n0 = global row 0 (CTA 0)
        const double *o = cluster.map_shared_rank(smem_d, 0);
        src_row = o + bm + off(0, 0);
      } else {
        src_row = smem_d + bm + off(rows - 1, 0);  // own row rows-1
      }
      for (int gc = tid; gc < p.n1; gc += blockDim.x) {
        double g = src_row[gc];
        if (k == 3) {
          const double v = p.bc_values[0][1] ? p.bc_values[0][1][gc] : p.bc_value[0][1];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        smem_d[bm + off(rows, gc)] = g;
      }
    }
    // ghost columns (axis 1) of the owned rows
    for (int lr = tid; lr < rows; lr += blockDim.x) {
      for (int side = 0; side < 2; ++side) {
        const int k = p.bc_kind[1][side];
        if (k == 0) continue;
        const int adj = side ? p.n1 - 1 : 0;
        double g = (k == 2) ? smem_d[bm + off(lr, side ? 0 : p.n1 - 1)] : smem_d[bm + off(lr, adj)];
        if (k == 3) {
          const double v =
              p.bc_values[1][side] ? p.bc_values[1][side][r0 + lr] : p.bc_value[1][side];
          g = __dsub_rn(__dmul_rn(2.0, v), g);
        }
        smem_d[bm + off(lr, side ? p.n1 : -1)] = g;
      }
    }
    // the periodic ghost rows read another CTA's rows: no CTA may overwrite
    // its buffer (next step) before they are read -> cluster barrier
    if (p.bc_kind[0][0] == 2) cluster.sync();
    else __syncthreads();
  }

  // ---- write the final buffer: owned rows (with ghost columns) and the
  // physical ghost rows of the first / last CTA --------------------------------
  const int lo = (rank == 0) ? -1 : 0;
  const int hi = (r0 + rows == p.n0) ? rows + 1 : rows;
  const int bf = cur * slab;
  for (int q = tid; q < (hi - lo) * sp; q += blockDim.x) {
    const int lr = lo + q / sp, gc = q % sp - 1;
    p.dst[int64_t(r0 + lr) * p.pitch + gc] = smem_d[bf + off(lr, gc)];
  }
}

}  // namespace srj
