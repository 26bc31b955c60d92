// srj_reduce.cuh -- true-residual norms and the dense-layout single step.
//
// residual_partial / residual_final: (sum r^2, max |r|) of r = s - A u over
// the owned active cells (GridProblem.residual_field, grids.py:249-266, same
// association as the sweep).  Warp-shuffle -> block -> grid reduction in a
// FIXED order (thread-strided partial sums, shuffle tree, shared-memory tree,
// then one block summing the per-block partials in index order), so the L2
// norm is bit-reproducible run to run.
//
// wj_dense: one weighted-Jacobi step on the reference's dense layout, the
// drop-in for one call of _WJ_KERNELS[ndim] (grids.py:478, :547-554).
#pragma once
#include "srj_device.cuh"

namespace srj {

struct ResidParams {
  const double *u;       // interior origin
  const double *f;       // source or kappa
  const uint8_t *act;
  const double *coef[7];
  double kc[7];
  int64_t pitch, plane;  // 2D: plane == pitch
  int ndim, n0, n1, n2;  // 2D: n2 == 1 and the grid is (n0, n1)
  int own_b, own_e;
  double *partials;      // [gridDim.x][2]
};

constexpr int kResidThreads = 256;
constexpr int kResidBlocksMax = 4096;  // grid = min(4 x SMs, this): fixed per device

template <bool VAR, bool NL>
__global__ void __launch_bounds__(kResidThreads) residual_partial(const __grid_constant__ ResidParams p) {
  double ss = 0.0, mx = 0.0;
  const int ncols = (p.ndim == 2) ? p.n1 : p.n2;
  const long nrows = (p.ndim == 2) ? long(p.own_e - p.own_b) : long(p.own_e - p.own_b) * p.n1;
  for (long row = blockIdx.x; row < nrows; row += gridDim.x) {
    int i, j;
    int64_t base;
    if (p.ndim == 2) {
      i = p.own_b + int(row);
      j = 0;
      base = int64_t(i) * p.pitch;
    } else {
      i = p.own_b + int(row / p.n1);
      j = int(row % p.n1);
      base = int64_t(i) * p.plane + int64_t(j) * p.pitch;
    }
    for (int k = threadIdx.x; k < ncols; k += blockDim.x) {
      const int64_t q = base + k;
      if (p.act && !p.act[q]) continue;
      double kk[7];
      if constexpr (VAR) {
        for (int a = 0; a < 7; ++a) kk[a] = (a < 1 + 2 * p.ndim) ? p.coef[a][q] : 0.0;
      } else {
        for (int a = 0; a < 7; ++a) kk[a] = p.kc[a];
      }
      const double *c = p.u + q;
      const double uc = c[0];
      const double s = NL ? nl_source(p.f[q], uc) : p.f[q];
      double r;
      if (p.ndim == 2)
        r = resid5(s, kk[0], uc, kk[1], c[-p.pitch], kk[2], c[p.pitch], kk[3], c[-1], kk[4], c[1]);
      else
        r = resid7(s, kk[0], uc, kk[1], c[-p.plane], kk[2], c[p.plane], kk[3], c[-p.pitch],
                   kk[4], c[p.pitch], kk[5], c[-1], kk[6], c[1]);
      ss = __dadd_rn(ss, __dmul_rn(r, r));
      acc_max(mx, r);
    }
  }
  // block reduction, fixed tree
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss = __dadd_rn(ss, __shfl_down_sync(kFull, ss, o));
    const double w = __shfl_down_sync(kFull, mx, o);
    mx = (w > mx) ? w : mx;
  }
  __shared__ double s_ss[kResidThreads / 32], s_mx[kResidThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_ss[warp] = ss;
    s_mx[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, m = 0.0;
    for (int w = 0; w < kResidThreads / 32; ++w) {
      a = __dadd_rn(a, s_ss[w]);
      m = (s_mx[w] > m) ? s_mx[w] : m;
    }
    p.partials[2 * blockIdx.x] = a;
    p.partials[2 * blockIdx.x + 1] = m;
  }
}

__global__ void __launch_bounds__(32) residual_final(const double *partials, int n, double *out) {
  // one warp, fixed order: lane l sums partials l, l+32, ... then a shuffle tree
  double ss = 0.0, mx = 0.0;
  for (int b = threadIdx.x; b < n; b += 32) {
    ss = __dadd_rn(ss, partials[2 * b]);
    const double m = partials[2 * b + 1];
    mx = (m > mx) ? m : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss = __dadd_rn(ss, __shfl_down_sync(kFull, ss, o));
    const double w = __shfl_down_sync(kFull, mx, o);
    mx = (w > mx) ? w : mx;
  }
  if (threadIdx.x == 0) {
    out[0] = ss;
    out[1] = mx;
  }
}

// residual_rows / residual_layers: the same (sum r^2, max |r|) per axis-0
// LAYER (2D: a row; 3D: a plane) of the owned rows, written to
// out[layer - own_b][2].  A warp reduces one last-axis row (lane-strided
// double2 loads, xor-shuffle tree); in 3D a second kernel folds a plane's
// row partials in a fixed order (one warp per plane).  Every layer's value
// depends only on the layer's cells, not on how the grid is split across
// ranks, so the host's exactly rounded sum over layers (math.fsum) gives the
// same L2 norm on 1 or N GPUs (distributed.srj_solve's residual-L2 rule).
template <bool VAR, bool NL>
__global__ void __launch_bounds__(256) residual_rows(const __grid_constant__ ResidParams p,
                                                     double *rows_out) {
  const int lane = threadIdx.x & 31;
  const int ncols = (p.ndim == 2) ? p.n1 : p.n2;
  const long nrows = (p.ndim == 2) ? long(p.own_e - p.own_b) : long(p.own_e - p.own_b) * p.n1;
  const long warp0 = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (long(gridDim.x) * blockDim.x) >> 5;
  for (long row = warp0; row < nrows; row += nwarps) {
    int64_t base;
    if (p.ndim == 2) {
      base = int64_t(p.own_b + int(row)) * p.pitch;
    } else {
      const int i = p.own_b + int(row / p.n1), j = int(row % p.n1);
      base = int64_t(i) * p.plane + int64_t(j) * p.pitch;
    }
    double ss = 0.0, mx = 0.0;
#pragma unroll 4
    for (int k = lane; k < ncols; k += 32) {
      const int64_t q = base + k;
      if (p.act && !p.act[q]) continue;
      double kk[7];
      if constexpr (VAR) {
        for (int a = 0; a < 7; ++a) kk[a] = (a < 1 + 2 * p.ndim) ? p.coef[a][q] : 0.0;
      } else {
        for (int a = 0; a < 7; ++a) kk[a] = p.kc[a];
      }
      const double *c = p.u + q;
      const double uc = c[0];
      const double s = NL ? nl_source(p.f[q], uc) : p.f[q];
      double r;
      if (p.ndim == 2)
        r = resid5(s, kk[0], uc, kk[1], c[-p.pitch], kk[2], c[p.pitch], kk[3], c[-1], kk[4], c[1]);
      else
        r = resid7(s, kk[0], uc, kk[1], c[-p.plane], kk[2], c[p.plane], kk[3], c[-p.pitch],
                   kk[4], c[p.pitch], kk[5], c[-1], kk[6], c[1]);
      ss = __dadd_rn(ss, __dmul_rn(r, r));
      acc_max(mx, r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss = __dadd_rn(ss, __shfl_xor_sync(kFull, ss, o));
      const double w = __shfl_xor_sync(kFull, mx, o);
      mx = (w > mx) ? w : mx;
    }
    if (lane == 0) {
      rows_out[2 * row] = ss;
      rows_out[2 * row + 1] = mx;
    }
  }
}

// 3D: out[layer] = fixed-order fold of the plane's n1 row partials
__global__ void __launch_bounds__(256) residual_layers(const double *rows, int nlayers, int n1,
                                                       double *out) {
  const int lane = threadIdx.x & 31;
  const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int layer = warp0; layer < nlayers; layer += nwarps) {
    const double *r = rows + 2 * int64_t(layer) * n1;
    double ss = 0.0, mx = 0.0;
    for (int j = lane; j < n1; j += 32) {
      ss = __dadd_rn(ss, r[2 * j]);
      const double m = r[2 * j + 1];
      mx = (m > mx) ? m : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss = __dadd_rn(ss, __shfl_xor_sync(kFull, ss, o));
      const double w = __shfl_xor_sync(kFull, mx, o);
      mx = (w > mx) ? w : mx;
    }
    if (lane == 0) {
      out[2 * layer] = ss;
      out[2 * layer + 1] = mx;
    }
  }
}

// Ghost-layer refresh after a sweep: GridProblem.refresh_ghosts
// (grids.py:225-247).  Every face writes only its ghost layer with the other
// axes restricted to the interior (corners untouched, as the reference) and
// reads only interior cells, so the faces are independent.  face_dirichlet is
// RN(RN(2*v) - u) like numpy's `2.0 * values - u[...]`.
struct GhostParams {
  double *u;              // interior origin of the buffer to refresh
  int64_t stride[3];      // element stride per axis (padded layout)
  int n[3];               // interior extents (unused axes = 1)
  int ndim;
  int kind[3][2];
  double value[3][2];
  const double *values[3][2];
  int64_t face_start[7];  // prefix sums of face sizes over the 2*ndim faces
};

// One face per blockIdx.y (2*ndim faces); blocks stride over the face's
// cells in C order of the other axes, 32-bit index math (faces are far below
// 2^31 cells; int64 division per cell made this kernel 4x slower).
__global__ void __launch_bounds__(256) ghost_refresh(const __grid_constant__ GhostParams p) {
  const int f = blockIdx.y;
  const int ax = f >> 1, side = f & 1;
  const int kind = p.kind[ax][side];
  if (kind == 0) return;
  // the other axes: (a0 outer, a1 inner); 2D has only a1
  const int a1 = (ax == p.ndim - 1) ? p.ndim - 2 : p.ndim - 1;
  const int a0 = (p.ndim == 3) ? ((ax == 0) ? 1 : 0) : -1;
  const int n1 = p.n[a1];
  const int ncell = int(p.face_start[f + 1] - p.face_start[f]);
  const int64_t sa = p.stride[ax];
  const int64_t s1 = p.stride[a1], s0 = a0 >= 0 ? p.stride[a0] : 0;
  const int64_t ghost_off = (side ? int64_t(p.n[ax]) : -1) * sa;
  const int64_t adj_off = (side ? int64_t(p.n[ax] - 1) : 0) * sa;
  const int64_t per_off = (side ? 0 : int64_t(p.n[ax] - 1)) * sa;  // periodic source
  const double *vals = p.values[ax][side];
  const double val = p.value[ax][side];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < ncell; q += gridDim.x * blockDim.x) {
    const int i0 = (a0 >= 0) ? q / n1 : 0;
    const int i1 = q - i0 * n1;
    const int64_t off = int64_t(i0) * s0 + int64_t(i1) * s1;
    double g;
    if (kind == 1) {
      g = p.u[off + adj_off];
    } else if (kind == 2) {
      g = p.u[off + per_off];
    } else {
      const double v = vals ? vals[q] : val;
      g = __dsub_rn(__dmul_rn(2.0, v), p.u[off + adj_off]);
    }
    p.u[off + ghost_off] = g;
  }
}

// Post-sweep gather (srj_plan_set_post_gather): phase 0 copies (or stages
// into tmp when destinations overlap sources), phase 1 scatters tmp.
__global__ void __launch_bounds__(256)
    post_gather(double *u, const int64_t *dst, const int64_t *src, int64_t n, double *tmp,
                int phase) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (phase == 1)
      u[dst[i]] = tmp[i];
    else if (tmp)
      tmp[i] = u[src[i]];
    else
      u[dst[i]] = u[src[i]];
  }
}

struct DenseParams {
  const double *u;
  double *un;
  const double *s, *c;
  const double *lo[3], *hi[3];
  const uint8_t *act;
  int ndim;
  int64_t n0, n1, n2;  // 1D: n1 == n2 == 1; 2D: n2 == 1
  double omega;
  double *norms;
};

__global__ void __launch_bounds__(256) wj_dense(const __grid_constant__ DenseParams p) {
  const int64_t total = p.n0 * p.n1 * p.n2;
  double dmx = 0.0, rmx = 0.0;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    int64_t g;  // offset of the cell in the ghosted array
    int64_t s0, s1;  // ghosted strides of axis 0 / axis 1
    if (p.ndim == 1) {
      s0 = s1 = 1;
      g = q + 1;
    } else if (p.ndim == 2) {
      const int64_t i = q / p.n1, j = q % p.n1;
      s1 = 1;
      s0 = p.n1 + 2;
      g = (i + 1) * s0 + (j + 1);
    } else {
      const int64_t k = q % p.n2, ij = q / p.n2;
      const int64_t j = ij % p.n1, i = ij / p.n1;
      s1 = p.n2 + 2;
      s0 = (p.n1 + 2) * s1;
      g = (i + 1) * s0 + (j + 1) * s1 + (k + 1);
    }
    const double uc = p.u[g];
    if (p.act && !p.act[q]) {
      p.un[g] = uc;
      continue;
    }
    double r;
    if (p.ndim == 1)
      r = resid3(p.s[q], p.c[q], uc, p.lo[0][q], p.u[g - 1], p.hi[0][q], p.u[g + 1]);
    else if (p.ndim == 2)
      r = resid5(p.s[q], p.c[q], uc, p.lo[0][q], p.u[g - s0], p.hi[0][q], p.u[g + s0],
                 p.lo[1][q], p.u[g - 1], p.hi[1][q], p.u[g + 1]);
    else
      r = resid7(p.s[q], p.c[q], uc, p.lo[0][q], p.u[g - s0], p.hi[0][q], p.u[g + s0],
                 p.lo[1][q], p.u[g - s1], p.hi[1][q], p.u[g + s1], p.lo[2][q], p.u[g - 1],
                 p.hi[2][q], p.u[g + 1]);
    const double d = relax(p.omega, r, p.c[q]);
    p.un[g] = __dadd_rn(uc, d);
    acc_max(dmx, d);
    acc_max(rmx, r);
  }
  dmx = warp_max(dmx);
  rmx = warp_max(rmx);
  if ((threadIdx.x & 31) == 0) {
    global_max(p.norms, dmx);
    global_max(p.norms + 1, rmx);
  }
}

}  // namespace srj
