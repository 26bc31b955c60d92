/*
 * srj.h -- C ABI of the B200 (sm_100a) SRJ weighted-Jacobi sweep library
 * (libsrj.so).  Plain pointers and sizes only; no torch or Python types.
 *
 * The reference (arXiv:1511.04292 package, /root/reference/pkg/src/srj) has no
 * FFI: its hot path is the numba kernel dispatch in grids.py.  Each entry point
 * below names the reference interface it replaces (file:line relative to
 * pkg/src/srj/).  INTEGRATION.md shows the ctypes binding a maintainer adds.
 *
 * Conventions
 *   - Every function returns an int status: SRJ_OK (0) or a negative SRJ_E*
 *     code; srj_last_error() returns a thread-local message for the last
 *     failure.  The Python host maps failures to RuntimeError/ValueError with
 *     the reference's messages.
 *   - "device" pointers are CUDA global-memory pointers on the current device;
 *     "host" pointers are CPU memory (pinned for full copy bandwidth).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Arithmetic is fp64 and bit-identical to the reference kernels _wj2/_wj3
 *     (grids.py:351-408): r = s - ((((c*u + am0*u[i-1]) + ap0*u[i+1]) +
 *     am1*u[j-1]) + ap1*u[j+1]) [+ am2*u[k-1] + ap2*u[k+1] in 3D],
 *     d = (omega*r)/c, un = u + d; no FMA contraction; NaNs never enter the
 *     max-norms (same as "if abs(d) > dmax").
 */
#ifndef SRJ_H
#define SRJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRJ_ABI_VERSION 7

enum {
    SRJ_OK = 0,
    SRJ_EINVAL = -1,       /* bad argument (maps to ValueError)            */
    SRJ_ECUDA = -2,        /* CUDA runtime/launch failure                  */
    SRJ_ENOMEM = -3,       /* device allocation failed                     */
    SRJ_EUNSUPPORTED = -4  /* feature outside the GPU path (NotImplemented) */
};

/* ------------------------------------------------------------------------
 * Device field layout ("padded layout").
 *
 * A ghosted field of interior extents n[0..ndim) (axis 0 slowest, as the
 * reference's C-order arrays) is stored with a 128-byte aligned row pitch so
 * the first interior cell of every row sits on a 128 B boundary.  Element
 * (g0, g1[, g2]) in ghost-inclusive reference indices (g = interior index + 1)
 * lives at   base + origin_shift + g0*plane0 + g1*pitch + g2      (3D)
 *            base + origin_shift + g0*pitch  + g1                 (2D)
 * where origin_shift puts g_last = 1 on an aligned address.  Rows along
 * axis 0 may carry `halo0` >= 1 ghost layers (multi-GPU slabs); the reference
 * layout corresponds to halo0 = 1.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t ndim;          /* 2 or 3                                          */
    int32_t halo0;         /* ghost layers on axis 0 (>= 1)                   */
    int64_t n[3];          /* interior extents                                */
    int64_t pitch;         /* elements between consecutive last-axis rows      */
    int64_t plane;         /* elements between axis-0 layers (3D; 2D: = pitch) */
    int64_t rows0;         /* axis-0 layers allocated = n[0] + 2*halo0         */
    int64_t origin;        /* element offset of (layer 0, row 0, ghost col 0);
                              reference index (g0, g1[, g2]) is at layer
                              g0 + halo0 - 1, so with halo0 == 1 this is the
                              reference's (0, 0[, 0])                         */
    int64_t elems;         /* elements to allocate per field                   */
} srj_layout_t;

/* Computes the padded layout for a grid.  Pure host arithmetic. */
int srj_layout(int32_t ndim, const int64_t *n, int32_t halo0,
               srj_layout_t *out);

/* ------------------------------------------------------------------------
 * Kernel-level entry point: one weighted-Jacobi step on the REFERENCE's dense
 * layout, replacing one call of the numba dispatch
 *     _WJ_KERNELS[ndim](u, scratch, *_coefficient_args(problem), omega, reverse)
 *     (grids.py:478, :547-554; argument order = _coefficient_args,
 *      grids.py:482-488)
 * for ndim = 1, 2, 3 (_wj1 / _wj2 / _wj3, grids.py:331-408).
 * u/un: device, shape n+2 per axis (dense C order).  s, c, lower[ax],
 * upper[ax]: device, interior-shaped dense.  act: device uint8 interior mask or
 * NULL.  Writes only the interior of un.  d_norms (device, 2 doubles) receives
 * (dmax, rmax) of this step.  The reference's `reverse` flag has no effect on
 * a two-buffer update and is therefore not an argument.
 * ---------------------------------------------------------------------- */
int srj_wj_dense(int32_t ndim, const int64_t *n, const double *u, double *un,
                 const double *s, const double *c, const double *const *lower,
                 const double *const *upper, const uint8_t *act, double omega,
                 double *d_norms, void *stream);

/* ------------------------------------------------------------------------
 * Solver plan: the device side of srj_solve / jacobi_solve / _Sweeper
 * (grids.py:535-559, :602-694).  Buffers are owned by the caller.
 * ---------------------------------------------------------------------- */
enum {
    SRJ_BC_FIXED = 0,          /* ghosts never touched                       */
    SRJ_BC_MIRROR = 1,         /* ghost = adjacent interior cell              */
    SRJ_BC_PERIODIC = 2,       /* ghost = interior cell at the opposite face  */
    SRJ_BC_FACE_DIRICHLET = 3  /* ghost = 2*value - adjacent interior cell    */
};

typedef struct {
    int32_t kind;              /* SRJ_BC_*                                    */
    double value;              /* face_dirichlet scalar (when values == NULL) */
    const double *values;      /* face_dirichlet: device array, dense, shaped
                                  like the interior without this axis         */
} srj_face_rule;

typedef struct {
    srj_layout_t layout;         /* from srj_layout()                         */
    int32_t coef_mode;           /* 0: constant stencil (scalars below)       */
                                 /* 1: per-cell arrays (coef_arrays)          */
    double coef[7];              /* center, lower0, upper0, lower1, upper1,
                                    lower2, upper2 (constant mode)            */
    const double *coef_arrays[7];/* same order, device, padded layout         */
    const uint8_t *act;          /* device uint8 mask in padded layout or NULL */
    const double *source;        /* device, padded layout (interior used)     */
    const double *kappa;         /* device, padded: nonlinear source
                                    s = kappa*u^5 from the current iterate
                                    (source ignored), or NULL                 */
    int64_t own0_begin;          /* axis-0 interior rows this plan owns for   */
    int64_t own0_end;            /*   stores and norms (default 0, n[0])      */
    int32_t physical_lo0;        /* 1: layer below row 0 is a FIXED boundary  */
    int32_t physical_hi0;        /* 1: layer above row n0-1 is a FIXED bound. */
    srj_face_rule bc[3][2];      /* per axis (low, high) ghost rule; all-zero =
                                    FIXED everywhere.  Non-FIXED faces refresh
                                    the ghosts after every launch (BoundaryRule,
                                    grids.py:73-112, refresh_ghosts :225-247);
                                    MIRROR / FACE_DIRICHLET faces keep fusing
                                    sweeps (2D up to 4, 3D up to 3; the ghosts
                                    between fused sweeps are formed on chip),
                                    PERIODIC runs one sweep per launch;
                                    single-slab only */
} srj_plan_desc;

typedef struct srj_plan srj_plan;

/* Validates the descriptor, allocates small device scratch. */
int srj_plan_create(const srj_plan_desc *desc, srj_plan **out);
int srj_plan_destroy(srj_plan *plan);

/* Post-sweep gather: the device form of the reference's `post_sweep` hooks
 * that copy field values (GridProblem.post_sweep, grids.py:146-163, called by
 * refresh_ghosts :246-247; e.g. the spherical tie_origin u[1] = u[2],
 * u[0] = u[2], problems.py:586-589).  After every sweep and its ghost
 * refresh, field[dst[i]] = field[src[i]] for i < n with simultaneous
 * semantics (all sources read before any destination is written).  dst/src
 * are HOST arrays of element offsets from the start of a field buffer in the
 * padded layout; the plan keeps a device copy.  n = 0 removes the gather.
 * Like a non-FIXED face, it makes every launch a single sweep. */
int srj_plan_set_post_gather(srj_plan *plan, const int64_t *dst,
                             const int64_t *src, int64_t n);

/* Coefficient array classes (ABI v6).  Per-cell coefficient arrays that are
 * constant along an axis -- the reference's problem builders broadcast radial
 * / polar profiles over the grid, e.g. spherical_poisson's center and lower /
 * upper (problems.py:489-560), and a constant stencil under a mask is
 * constant along every axis -- are read once per row instead of once per cell
 * by the 3D per-cell sweep kernel (srj_sweep3d.cuh; the reference's
 * spherical problem at 512^3: 69 -> 96 G updates/s).  The 2D per-cell kernels
 * read every cell (measured: no gain).  cls[a] for
 * coefficient a (order of coef_arrays) is a bit set:
 *   SRJ_COEF_CONST_AXIS0: value(i, ...) == value(0, ...) for every i;
 *   SRJ_COEF_CONST_LAST:  value(..., k) == value(..., 0) for every k.
 * The arrays stay in coef_arrays (padded layout, every cell present), so the
 * other kernels and the residual kernels read them as before; the caller
 * guarantees the equalities bit for bit (engine.py detects them), so every
 * result is unchanged.  All zero (the default) = read every cell. */
enum { SRJ_COEF_FULL = 0, SRJ_COEF_CONST_AXIS0 = 1, SRJ_COEF_CONST_LAST = 2 };
int srj_plan_set_coef_classes(srj_plan *plan, const int32_t *cls);

/* Maximum fused-sweep depth (temporal blocking) supported by srj_plan_run. */
int srj_max_fuse(void);

/* Runs `nsteps` elementary steps k = first .. first+nsteps-1 with
 * omega_k = weights[k mod m] (weights: HOST array of the cycle's M weights,
 * CycleSchedule.weight_sequence, schedule.py:33-83), starting from the field
 * in `src` and ping-ponging between buf_a and buf_b (both distinct from src,
 * so src survives as a snapshot).  `fuse` = sweeps fused per launch
 * (0 = plan default; 1..srj_max_fuse()).  d_norms (device, 2*nsteps doubles)
 * receives per-step (dmax, rmax) exactly as _wj* returns them; it is
 * zero-initialised by this call.  *final_buf = 0 (src, nsteps==0), 1 (buf_a)
 * or 2 (buf_b) tells where the last iterate is.  Asynchronous on `stream`.
 * Replaces the per-step loop of _iterate/_Sweeper.jacobi
 * (grids.py:613-617, :544-559). */
int srj_plan_run(srj_plan *plan, const double *src, double *buf_a,
                 double *buf_b, const double *weights, int64_t m,
                 int64_t first, int64_t nsteps, int32_t fuse, double *d_norms,
                 int32_t *final_buf, void *stream);

/* True residual of field u: d_out[0] = sum r^2, d_out[1] = max |r| over the
 * owned active cells, r = s - A u (GridProblem.residual_field,
 * grids.py:249-266; same operator association as the sweep).  Deterministic
 * two-pass reduction (fixed order).  d_out: device, 2 doubles. */
int srj_plan_residual(srj_plan *plan, const double *u, double *d_out,
                      void *stream);

/* Per-layer true residual: d_layers[2*(i - own0_begin) + {0, 1}] = (sum r^2,
 * max |r|) over the owned active cells of axis-0 layer i (2D: a row, 3D: a
 * plane), for every owned layer i (GridProblem.residual_field,
 * grids.py:249-266).  A layer's value depends only on its cells (fixed
 * reduction order per layer), so a host sum over layers is independent of how
 * the grid is split across GPUs.  d_layers: device, 2*(own0_end-own0_begin). */
int srj_plan_residual_layers(srj_plan *plan, const double *u, double *d_layers,
                             void *stream);

/* Gauss-Seidel / SOR: `nsweeps` in-place lexicographic sweeps of field `u`
 * (a buffer in the plan's layout) with relaxation factor omega (1 = GS),
 * bitwise the reference's _gs2 / _gs3 (grids.py:426-474) followed by its ghost
 * refresh (and copy hook) after every sweep (_Sweeper.gauss_seidel,
 * grids.py:561-571).  d_norms (device, 2*nsweeps doubles): per-sweep (dmax,
 * rmax).  A GPU wavefront: 32-row strips must all be co-resident (cooperative
 * launch), else SRJ_EUNSUPPORTED; whole-grid plans, no nonlinear source. */
int srj_plan_gs(srj_plan *plan, double *u, double omega, int64_t nsweeps,
                double *d_norms, void *stream);

/* Host <-> device transfers between the reference's dense layout and the
 * padded layout (cudaMemcpy2DAsync; host memory should be pinned).
 *   field:    ghosted array, shape n+2 per axis (problem.u)
 *   interior: interior-shaped array (problem.source / center / ...); written
 *             into the interior positions of a padded field-shaped buffer
 *   elem_size: 8 for fp64 fields, 1 for the uint8 mask.
 * For halo0 > 1 layouts only layers [halo0-1, halo0+n0] are transferred. */
int srj_upload_field(const srj_layout_t *lay, const double *host, double *dev,
                     void *stream);
int srj_download_field(const srj_layout_t *lay, const double *dev, double *host,
                       void *stream);
int srj_upload_interior(const srj_layout_t *lay, const void *host, void *dev,
                        int32_t elem_size, void *stream);

/* Copies `count` axis-0 layers starting at layer `first_layer` (padded-layout
 * layer index, 0 = lowest allocated layer) between two padded buffers of the
 * same layout, possibly on different devices via peer access (halo exchange
 * for slab decomposition). */
int srj_copy_layers(const srj_layout_t *lay, const double *src,
                    int64_t src_layer, double *dst, int64_t dst_layer,
                    int64_t count, void *stream);

/* ------------------------------------------------------------------------
 * Slab decomposition across GPUs (the reference has no parallel
 * path -- SPEC.md:305 -- and relies on Jacobi's insensitivity to domain
 * decomposition).  Each rank owns a block of axis-0 rows of
 * the global grid plus `halo` >= fuse exchanged rows per neighbour side, held
 * as interior rows of its local plan (desc.own0_begin/end = the owned rows).
 * srj_slab_run replaces the per-step loop of _iterate/_Sweeper.jacobi
 * (grids.py:613-617, :544-559) for one rank.  Ranks order each other on the
 * device through flag words in each other's memory (stream memory operations:
 * "halo of my source delivered", "neighbour finished the launch that read the
 * buffer I write into"), so the host only enqueues work.  Two data paths:
 *  - direct (default; constant stencil at 2D fused depth <= 4 / 3D depth <= 2,
 *    per-cell coefficients at depth 1):
 *    ONE launch per fused step over all owned rows; the sweep kernel itself
 *    stores the rows next to a neighbour into that neighbour's halo rows of
 *    the destination buffer (peer memory over NVLink) -- no edge launches, no
 *    copies, one batch of flag operations per launch;
 *  - staged (fused per-cell sweeps, deeper fusion; SRJ_SLAB_DIRECT=0): the
 *    edge rows run on an internal edge stream, are copied into the
 *    neighbours' halo rows (peer cudaMemcpyAsync on a comm stream) while the
 *    inner rows run concurrently on the caller's stream.
 * ------------------------------------------------------------------------ */
#define SRJ_SLAB_FLAG_WORDS 8   /* uint32 flag words per rank (device)       */

typedef struct srj_slab srj_slab;

typedef struct {
    double *bufs[3];     /* the neighbour's three field buffers, addressable
                            from this rank's device (IPC-mapped peer memory,
                            or the same device when ranks are emulated)      */
    uint32_t *flags;     /* the neighbour's flag block                        */
    int64_t dst_row;     /* neighbour-local interior row where the rows this
                            rank sends land (lower neighbour: its own0_end;
                            upper neighbour: 0)                               */
} srj_slab_peer;

/* desc: the rank's local plan (FIXED faces only); bufs: its three field
 * buffers (the same three every srj_slab_run call uses by index); flags:
 * SRJ_SLAB_FLAG_WORDS device words; has_lo/has_hi: neighbours exist. */
int srj_slab_create(const srj_plan_desc *desc, int32_t halo, double *const *bufs,
                    uint32_t *flags, int32_t has_lo, int32_t has_hi,
                    srj_slab **out);
/* side 0 = lower neighbour (rank-1), 1 = upper (rank+1). */
int srj_slab_connect(srj_slab *slab, int32_t side, const srj_slab_peer *peer);
/* Zero this rank's flags and launch counter (all ranks, then a host barrier,
 * before the first srj_slab_run). */
int srj_slab_reset(srj_slab *slab, void *stream);
int srj_slab_destroy(srj_slab *slab);
/* The slab's plan (for srj_plan_residual_layers etc.; owned by the slab). */
srj_plan *srj_slab_plan(srj_slab *slab);
/* Sweeps per fused launch srj_slab_run runs for this `fuse` (0 = the plan's
 * default), capped by the halo.  A plan's default depends on its local size
 * and coefficient mode: the ranks of a run must agree on ONE depth (their
 * minimum) and pass it as `fuse`, or their exchanges fall out of step. */
int srj_slab_depth(srj_slab *slab, int32_t fuse);
/* 1 if srj_slab_run with this `fuse` takes the direct data path (one launch
 * per fused step, edge rows stored into the neighbours' halos by the sweep
 * kernel), 0 for the staged path (edge launches + peer copies), < 0 on error. */
int srj_slab_direct(srj_slab *slab, int32_t fuse);
/* Steps first .. first+nsteps-1 (omega_k = weights[k mod m]) from field buffer
 * `src` (0..2, left untouched) ping-ponging over the other two; *final_buf =
 * the buffer index holding the result.  d_norms[i]: device, 2*nsteps doubles
 * of per-step (dmax, rmax) over slab i's owned rows (MAX over ranks is the
 * caller's all-reduce).  n == 1: this process's rank on streams[0] (+ an
 * internal comm stream).  n > 1 slabs in one call = ranks emulated on one
 * device: with one shared stream everything is enqueued on it in dependency
 * order; with pairwise distinct streams[i] every slab runs as a rank would
 * (its stream + its comm stream, ordered against the others only by the
 * flag words). */
int srj_slab_run(srj_slab *const *slabs, int32_t n, int32_t src,
                 const double *weights, int64_t m, int64_t first, int64_t nsteps,
                 int32_t fuse, double *const *d_norms, int32_t *final_buf,
                 void *const *streams);

/* CUDA IPC between the ranks' processes: handle (64 bytes) + byte offset of
 * dev_ptr inside its allocation; srj_ipc_open maps it (peer access enabled
 * lazily) and returns the address of the same byte; srj_ipc_close unmaps
 * (pass ptr - offset, the mapped base). */
int srj_ipc_get_handle(const void *dev_ptr, void *handle, int64_t *offset);
int srj_ipc_open(const void *handle, int64_t offset, void **dev_ptr);
int srj_ipc_close(void *base);

/* Diagnostic: out[i] = a[i]/c through the reciprocal-refinement division the
 * constant-stencil kernels use (y = RN(1/c), two Markstein corrections), and
 * ref[i] = the IEEE-754 quotient; device arrays of n doubles.  Tests assert
 * out == ref bit for bit. */
int srj_selftest_div(const double *a, int64_t n, double c, double *out,
                     double *ref, void *stream);

int srj_abi_version(void);
const char *srj_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SRJ_H */
