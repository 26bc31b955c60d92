// srj_capi.cu -- C ABI (include/srj.h) over the sm_100a SRJ kernels.
//
// Host-side launch logic for the reference's hot loop (grids.py:535-559,
// :602-687): the caller (Python, ctypes) owns all device buffers; this layer
// plans the launch geometry, picks the fused-sweep depth, launches the
// kernels on the caller's stream and reports errors as status codes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/srj.h"
#include "srj_host.cuh"
#include "srj_reduce.cuh"
#include "srj_cluster2d.cuh"
#include "srj_sweep2d_var.cuh"

using namespace srj;
using namespace srj_host;

namespace {

constexpr int64_t kAlign = 16;        // elements (128 B)
constexpr int64_t kXOff = kAlign - 1; // last-axis ghost g=0 sits at offset 15
constexpr int64_t kSlack = 256;       // tail elements for band over-reads

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// y = RN(1/c) for the reciprocal division path (srj_sweep2d.cuh div_by_const),
// or 0 to keep the IEEE division when c is outside [2^-100, 2^100].
// low word of the double-word reciprocal: yl = RN(1/c - yh), via the exact
// FMA remainder 1 - c*yh
double recip_lo(double c, double yh) {
  if (yh == 0.0) return 0.0;
  return std::fma(-c, yh, 1.0) / c;
}

double recip_or_zero(double c) {
  if (!(c >= 0x1p-100 && c <= 0x1p+100)) return 0.0;  // c > 0 only (div_recip sign rule)
  return 1.0 / c;
}

// offset of interior cell (0,0[,0])
int64_t interior_offset(const srj_layout_t &l) {
  return l.origin + int64_t(l.halo0) * l.plane + (l.ndim == 3 ? l.pitch : 0) + 1;
}

// SRJ_WAVES=<n>: launch n waves of band warps instead of one (tuning knob)
int waves_2d() {
  static int w = 0;
  if (w == 0) {
    const char *e = getenv("SRJ_WAVES");
    w = e ? atoi(e) : 1;
    if (w < 1 || w > 64) w = 1;
  }
  return w;
}

// SRJ_SLAB_SPLIT=0: slab ranks run edge and inner rows on one stream (A/B knob)
// (read on every srj_slab_run call, so a probe can toggle it in-process)
bool slab_split_enabled() {
  const char *e = getenv("SRJ_SLAB_SPLIT");
  return !(e && *e && atoi(e) == 0);
}

// SRJ_SLAB_DIRECT=0: slab ranks exchange by edge launches + peer copies
// instead of storing edge rows from the sweep kernel (A/B knob)
bool slab_direct_enabled() {
  const char *e = getenv("SRJ_SLAB_DIRECT");
  return !(e && *e && atoi(e) == 0);
}

// SRJ_MIN_PLANES=<n>: least planes per persistent CTA of the 3D T = 2 kernel (tuning knob)
long min_planes_3d() {
  const char *e = getenv("SRJ_MIN_PLANES");
  const long v = e ? atol(e) : 2;
  return v >= 1 ? v : 2;
}

// SRJ_BPS=<n>: size the 2D grid for n resident blocks per SM (tuning knob)
int bps_override() {
  static int b = -1;
  if (b < 0) {
    const char *e = getenv("SRJ_BPS");
    b = e ? atoi(e) : 0;
  }
  return b;
}

// 2D per-cell coefficients, one sweep (HBM-bound streaming kernel)
template <bool NL>
struct KVar2D {
  static int bps() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep2d_var<NL>, kWarps2DVar * 32, 0);
      return n > 0 ? n : 1;
    });
  }
};

// row / plane stride and column multiplier of coefficient array `a` under
// its class (srj_plan_set_coef_classes)
static void class_strides(const int32_t *cls, int a, int64_t stride, int64_t &rs, int &cm) {
  rs = (cls[a] & SRJ_COEF_CONST_AXIS0) ? 0 : stride;
  cm = (cls[a] & SRJ_COEF_CONST_LAST) ? 0 : 1;
}

static int launch_var2d(const srj_plan_desc &d, int64_t own_b, int64_t own_e, const double *cur,
                        double *nxt, const double *f, int ld_lo, int ld_hi, double omega,
                        double *norms, cudaStream_t st, const PeerSend *send = nullptr) {
  const srj_layout_t &l = d.layout;
  const int64_t ioff = interior_offset(l);
  const bool nl = d.kappa != nullptr;
  Var2DParams p{};
  p.src = cur + ioff;
  p.dst = nxt + ioff;
  p.f = f + ioff;
  p.act = d.act ? d.act + ioff : nullptr;
  p.c = d.coef_arrays[0] + ioff;
  p.am0 = d.coef_arrays[1] + ioff;
  p.ap0 = d.coef_arrays[2] + ioff;
  p.am1 = d.coef_arrays[3] + ioff;
  p.ap1 = d.coef_arrays[4] + ioff;
  p.pitch = l.pitch;
  p.n0 = int(l.n[0]);
  p.n1 = int(l.n[1]);
  p.ld_lo = ld_lo;
  p.ld_hi = ld_hi;
  p.own_b = int(own_b);
  p.own_e = int(own_e);
  p.nbands = int((l.n[1] + 63) / 64);
  p.omega = omega;
  p.norms = norms;
  const int rows = p.own_e - p.own_b;
  const long capacity = long(sm_count()) * (nl ? KVar2D<true>::bps() : KVar2D<false>::bps()) *
                        kWarps2DVar;
  // strips: best fill of whole waves, discounting the 2 halo rows per strip
  int nstrips = 1;
  double best = -1.0;
  for (int ns = 1; ns <= std::max(1, std::min(256, rows / 8)); ++ns) {
    const long w = long(p.nbands) * ns;
    const long waves = (w + capacity - 1) / capacity;
    const double hh = double(rows) / ns;
    const double eff = double(w) / double(waves * capacity) * hh / (hh + 2.0);
    if (eff > best + 1e-9) {
      best = eff;
      nstrips = ns;
    }
  }
  p.H = (rows + nstrips - 1) / nstrips;
  p.nstrips = (rows + p.H - 1) / p.H;
  const long warps = long(p.nbands) * p.nstrips;
  const int blocks = int((warps + kWarps2DVar - 1) / kWarps2DVar);
  if (send) {
    p.send = *send;
    if (nl)
      sweep2d_var<true, true><<<blocks, kWarps2DVar * 32, 0, st>>>(p);
    else
      sweep2d_var<false, true><<<blocks, kWarps2DVar * 32, 0, st>>>(p);
  } else if (nl) {
    sweep2d_var<true><<<blocks, kWarps2DVar * 32, 0, st>>>(p);
  } else {
    sweep2d_var<false><<<blocks, kWarps2DVar * 32, 0, st>>>(p);
  }
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

Kernel2D pick2d(int T, bool var, bool nl, bool recip, int bcf, bool send = false) {
  switch (T) {
    case 1: return pick2d_t<1>(var, nl, recip, bcf, send);
    case 2: return pick2d_t<2>(var, nl, recip, bcf, send);
    case 3: return pick2d_t<3>(var, nl, recip, bcf, send);
    case 4: return pick2d_t<4>(var, nl, recip, bcf, send);
    case 5: return pick2d_t<5>(var, nl, recip, bcf, send);
    case 6: return pick2d_t<6>(var, nl, recip, bcf, send);
    case 7: return pick2d_t<7>(var, nl, recip, bcf, send);
    default: return pick2d_t<8>(var, nl, recip, bcf, send);
  }
}

// 2D tensor map over a whole padded 2D field: rows0 rows of `pitch` doubles,
// box = box_cols x 3 rows (one TMA group of the band kernel).
int make_tmap(CUtensorMap *m, const double *base, const srj_layout_t &l, int box_cols,
              int box_rows = 3) {
  auto fn = encode_fn();
  if (!fn) return fail(SRJ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  // every last-axis row of the field is one tensor row (3D: planes x rows)
  const int64_t rows = l.ndim == 3 ? l.rows0 * (l.n[1] + 2) : l.rows0;
  cuuint64_t dims[2] = {cuuint64_t(l.pitch), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(l.pitch) * 8};
  cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SRJ_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SRJ_OK;
}

}  // namespace

__global__ void selftest_div(const double *a, int64_t n, double c, double y, double yl,
                             double *out, double *ref) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double q = __ddiv_rn(a[i], c);
    if (y != 0.0) {  // exactly what the RECIP sweep kernels compute
      q = div_recip(a[i], c, y, yl);
      if (recip_unsafe(a[i])) q = div_ieee(a[i], c);
    }
    out[i] = q;
    ref[i] = __ddiv_rn(a[i], c);
  }
}

struct srj_plan {
  srj_plan_desc d;
  bool has_bc;       // some face is not FIXED: refresh ghosts after each launch
  bool bc_fusable;   // ...and none is PERIODIC: fused launches form the ghosts on chip
  int default_fuse;
  double *partials;  // [resid_blocks][2] device scratch
  int resid_blocks;  // 4 x SMs (fixed per device, so a fixed reduction order)
  double *row_parts = nullptr;  // 3D per-(i,j)-row residual partials (srj_plan_residual_layers)
  int64_t row_parts_cap = 0;
  double *vtb_yh = nullptr, *vtb_yl = nullptr;  // per-cell reciprocal of c (sweep2d_vtb)
  int32_t cls[7] = {};  // coefficient classes (srj_plan_set_coef_classes)
  double *bc_scalars;  // [3][2] device copies of the faces' scalar values (fused BCs)
  // small-grid cluster path: per-chunk omegas (device + pinned staging)
  double *d_omegas = nullptr, *h_omegas = nullptr;
  int64_t omega_cap = 0;
  cudaEvent_t omega_ev = nullptr;
  // Gauss-Seidel wavefront progress counters (one per 32-row strip)
  unsigned long long *gs_prog = nullptr;
  int64_t gs_prog_cap = 0;
  // post-sweep gather (device copies; tmp only when dst and src overlap)
  int64_t *g_dst = nullptr, *g_src = nullptr;
  double *g_tmp = nullptr;
  int64_t g_n = 0;
  // encoded TMA descriptors by (base, box): a solve cycles through 3 field
  // buffers and one source array, so a handful of entries avoids re-encoding
  // two descriptors per launch on the host
  struct Tmap {
    CUtensorMap m;
    const void *base = nullptr;
    int cols = 0, rows = 0;
  };
  Tmap tmaps[8];
  int tmap_next = 0;
};

static int plan_tmap(srj_plan &plan, CUtensorMap *out, const double *base, int box_cols, int box_rows) {
  for (const auto &t : plan.tmaps)
    if (t.base == base && t.cols == box_cols && t.rows == box_rows) {
      *out = t.m;
      return SRJ_OK;
    }
  srj_plan::Tmap &t = plan.tmaps[plan.tmap_next];
  plan.tmap_next = (plan.tmap_next + 1) % 8;
  const int rc = make_tmap(&t.m, base, plan.d.layout, box_cols, box_rows);
  if (rc != SRJ_OK) {
    t.base = nullptr;
    return rc;
  }
  t.base = base;
  t.cols = box_cols;
  t.rows = box_rows;
  *out = t.m;
  return SRJ_OK;
}

// ---------------------------------------------------------------- scratch
// Small device / pinned-host work buffers of a plan (norm partials, per-chunk
// weights, gather indices, GS progress counters) come from a process-wide
// cache instead of cudaMalloc / cudaFree per plan: a solve on a small grid
// spent ~10 ms of its ~13 ms in those calls (each cudaFree also synchronises
// the device).  Blocks are recycled by (device, power-of-two size); blocks
// above kScratchMax bytes bypass the cache.  srj_plan_destroy synchronises the
// device once before returning blocks, as cudaFree did implicitly.
constexpr size_t kScratchMax = size_t(4) << 20;

struct ScratchCache {
  struct Block {
    void *ptr;
    size_t bytes;
    int device;  // -1: pinned host
  };
  std::mutex mu;
  std::vector<Block> free_list, live;
};

static ScratchCache &scratch_cache() {
  static ScratchCache *c = new ScratchCache;  // never destroyed: no CUDA calls at exit
  return *c;
}

static size_t scratch_round(size_t bytes) {
  size_t r = 256;
  while (r < bytes) r <<= 1;
  return r;
}

static cudaError_t scratch_alloc_impl(void **out, size_t bytes, bool host) {
  *out = nullptr;
  const size_t want = bytes > kScratchMax ? bytes : scratch_round(bytes);
  const int dev = host ? -1 : current_device();
  ScratchCache &c = scratch_cache();
  if (bytes <= kScratchMax) {
    std::lock_guard<std::mutex> lk(c.mu);
    for (size_t i = 0; i < c.free_list.size(); ++i)
      if (c.free_list[i].device == dev && c.free_list[i].bytes == want) {
        *out = c.free_list[i].ptr;
        c.live.push_back(c.free_list[i]);
        c.free_list.erase(c.free_list.begin() + long(i));
        return cudaSuccess;
      }
  }
  void *ptr = nullptr;
  const cudaError_t e = host ? cudaMallocHost(&ptr, want) : cudaMalloc(&ptr, want);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    c.live.push_back({ptr, want, dev});
  }
  *out = ptr;
  return cudaSuccess;
}

template <class T>
static cudaError_t scratch_alloc(T **out, size_t bytes) {
  return scratch_alloc_impl(reinterpret_cast<void **>(out), bytes, false);
}
template <class T>
static cudaError_t scratch_alloc_host(T **out, size_t bytes) {
  return scratch_alloc_impl(reinterpret_cast<void **>(out), bytes, true);
}

// The caller guarantees no work in flight still uses the block.
static void scratch_free(void *ptr) {
  if (!ptr) return;
  ScratchCache &c = scratch_cache();
  ScratchCache::Block b{nullptr, 0, 0};
  {
    std::lock_guard<std::mutex> lk(c.mu);
    for (size_t i = 0; i < c.live.size(); ++i)
      if (c.live[i].ptr == ptr) {
        b = c.live[i];
        c.live.erase(c.live.begin() + long(i));
        break;
      }
    if (b.ptr && b.bytes <= kScratchMax && c.free_list.size() < 256) {
      c.free_list.push_back(b);
      return;
    }
  }
  if (!b.ptr) return;  // not ours
  if (b.device < 0)
    cudaFreeHost(ptr);
  else
    cudaFree(ptr);
}

static void free_gather(srj_plan *p) {
  scratch_free(p->g_dst);
  scratch_free(p->g_src);
  scratch_free(p->g_tmp);
  p->g_dst = p->g_src = nullptr;
  p->g_tmp = nullptr;
  p->g_n = 0;
}

static int launch_gather(const srj_plan &plan, double *field, cudaStream_t st) {
  const int blocks = int(std::min<int64_t>((plan.g_n + 255) / 256, int64_t(sm_count()) * 8));
  post_gather<<<blocks, 256, 0, st>>>(field, plan.g_dst, plan.g_src, plan.g_n, plan.g_tmp, 0);
  if (plan.g_tmp)
    post_gather<<<blocks, 256, 0, st>>>(field, plan.g_dst, plan.g_src, plan.g_n, plan.g_tmp, 1);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

extern "C" {

int srj_abi_version(void) { return SRJ_ABI_VERSION; }

int srj_selftest_div(const double *a, int64_t n, double c, double *out, double *ref,
                     void *stream) {
  if (!a || !out || !ref || n < 0) return fail(SRJ_EINVAL, "bad argument");
  if (n == 0) return SRJ_OK;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 32));
  const double yh = recip_or_zero(c);
  selftest_div<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, n, c, yh,
                                                                       recip_lo(c, yh), out, ref);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}
const char *srj_last_error(void) { return g_err; }
int srj_max_fuse(void) { return kMaxFuse; }

int srj_layout(int32_t ndim, const int64_t *n, int32_t halo0, srj_layout_t *out) {
  if (!out || !n) return fail(SRJ_EINVAL, "null argument");
  if (ndim != 2 && ndim != 3)
    return fail(SRJ_EUNSUPPORTED, "the GPU path supports 2- and 3-dimensional grids (got %d)", ndim);
  if (halo0 < 1 || halo0 > kMaxFuse) return fail(SRJ_EINVAL, "halo0 must be in [1, %d]", kMaxFuse);
  srj_layout_t l;
  std::memset(&l, 0, sizeof(l));
  l.ndim = ndim;
  l.halo0 = halo0;
  for (int a = 0; a < ndim; ++a) {
    if (n[a] < 1 || n[a] > (int64_t(1) << 30)) return fail(SRJ_EINVAL, "bad extent n[%d]=%lld", a, (long long)n[a]);
    l.n[a] = n[a];
  }
  const int64_t last = n[ndim - 1];
  l.pitch = kAlign + round_up(last + 1, 64);
  l.plane = (ndim == 3) ? (n[1] + 2) * l.pitch : l.pitch;
  l.rows0 = n[0] + 2 * int64_t(halo0);
  l.origin = kXOff;
  l.elems = l.rows0 * l.plane + kSlack + kAlign;
  *out = l;
  return SRJ_OK;
}

int srj_wj_dense(int32_t ndim, const int64_t *n, const double *u, double *un, const double *s,
                 const double *c, const double *const *lower, const double *const *upper,
                 const uint8_t *act, double omega, double *d_norms, void *stream) {
  if (ndim < 1 || ndim > 3)
    return fail(SRJ_EUNSUPPORTED, "the dense kernel supports 1- to 3-dimensional grids (got %d)", ndim);
  if (!u || !un || !s || !c || !lower || !upper || !d_norms) return fail(SRJ_EINVAL, "null argument");
  DenseParams p{};
  p.u = u;
  p.un = un;
  p.s = s;
  p.c = c;
  for (int a = 0; a < ndim; ++a) {
    p.lo[a] = lower[a];
    p.hi[a] = upper[a];
  }
  p.act = act;
  p.ndim = ndim;
  p.n0 = n[0];
  p.n1 = (ndim >= 2) ? n[1] : 1;
  p.n2 = (ndim == 3) ? n[2] : 1;
  p.omega = omega;
  p.norms = d_norms;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SRJ_CUDA(cudaMemsetAsync(d_norms, 0, 2 * sizeof(double), st));
  const int64_t total = p.n0 * p.n1 * p.n2;
  if (total == 0) return SRJ_OK;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(sm_count()) * 16));
  wj_dense<<<blocks, 256, 0, st>>>(p);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

int srj_plan_create(const srj_plan_desc *desc, srj_plan **out) {
  if (!desc || !out) return fail(SRJ_EINVAL, "null argument");
  const srj_layout_t &l = desc->layout;
  if (l.ndim != 2 && l.ndim != 3) return fail(SRJ_EUNSUPPORTED, "ndim must be 2 or 3");
  if (!desc->source && !desc->kappa) return fail(SRJ_EINVAL, "source (or kappa) required");
  if (desc->coef_mode != 0 && desc->coef_mode != 1) return fail(SRJ_EINVAL, "coef_mode must be 0 or 1");
  if (desc->coef_mode == 1)
    for (int a = 0; a < 1 + 2 * l.ndim; ++a)
      if (!desc->coef_arrays[a]) return fail(SRJ_EINVAL, "coefficient array %d missing", a);
  if (desc->coef_mode == 0 && desc->coef[0] == 0.0)
    return fail(SRJ_EINVAL, "center coefficient vanishes on an active cell");
  srj_plan *p = new (std::nothrow) srj_plan;
  if (!p) return fail(SRJ_ENOMEM, "host allocation failed");
  p->d = *desc;
  if (p->d.own0_end <= p->d.own0_begin) {
    p->d.own0_begin = 0;
    p->d.own0_end = l.n[0];
  }
  if (p->d.own0_begin < 0 || p->d.own0_end > l.n[0]) {
    delete p;
    return fail(SRJ_EINVAL, "owned rows out of range");
  }
  p->has_bc = false;
  for (int a = 0; a < 3; ++a)
    for (int side = 0; side < 2; ++side) {
      const int k = desc->bc[a][side].kind;
      if (k < SRJ_BC_FIXED || k > SRJ_BC_FACE_DIRICHLET || (k != SRJ_BC_FIXED && a >= l.ndim)) {
        delete p;
        return fail(SRJ_EINVAL, "bad boundary rule on axis %d", a);
      }
      if (k != SRJ_BC_FIXED) p->has_bc = true;
    }
  for (int a = 0; a < l.ndim; ++a)
    if ((desc->bc[a][0].kind == SRJ_BC_PERIODIC) != (desc->bc[a][1].kind == SRJ_BC_PERIODIC)) {
      delete p;
      return fail(SRJ_EINVAL, "periodic axes need the rule on both faces");
    }
  if (p->has_bc && (!desc->physical_lo0 || !desc->physical_hi0 || p->d.own0_begin != 0 ||
                    p->d.own0_end != l.n[0])) {
    delete p;
    return fail(SRJ_EUNSUPPORTED, "non-FIXED boundary rules need the whole grid on one plan");
  }
  // non-FIXED ghosts change every step.  MIRROR and FACE_DIRICHLET ghosts are a
  // function of the adjacent cell, so the 2D band kernel and the 3D tile
  // kernel fold them into their fused stages; PERIODIC (the opposite face)
  // runs one sweep per launch
  p->bc_fusable = p->has_bc && (l.ndim == 2 || (l.n[1] < (1 << 15) && l.n[2] < (1 << 16)));
  for (int a = 0; a < l.ndim; ++a)
    if (desc->bc[a][0].kind == SRJ_BC_PERIODIC) p->bc_fusable = false;
  p->default_fuse = (desc->coef_mode == 0 && (!p->has_bc || p->bc_fusable))
                        ? (l.ndim == 2 ? 4 : 2)
                        // per-cell coefficients (2D, FIXED faces): the fused T=2 kernel
                        // (srj_sweep2d_vtb.cuh) from 2M cells up, where it beats one sweep
                        // per launch
                        : (desc->coef_mode == 1 && l.ndim == 2 && !p->has_bc &&
                                   l.n[0] * l.n[1] >= (int64_t(1) << 21)
                               ? 2
                               : 1);
  p->partials = nullptr;
  p->bc_scalars = nullptr;
  p->resid_blocks = std::min(4 * sm_count(), kResidBlocksMax);
  cudaError_t e = scratch_alloc(&p->partials, sizeof(double) * 2 * p->resid_blocks);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(partials)");
  }
  if (p->bc_fusable) {
    double v[6];
    for (int f = 0; f < 6; ++f) v[f] = desc->bc[f >> 1][f & 1].value;
    e = scratch_alloc(&p->bc_scalars, sizeof(v));
    if (e == cudaSuccess) e = cudaMemcpy(p->bc_scalars, v, sizeof(v), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      scratch_free(p->partials);
      scratch_free(p->bc_scalars);
      delete p;
      return cuda_fail(e, "cudaMalloc(bc scalars)");
    }
  }
  *out = p;
  return SRJ_OK;
}

int srj_plan_set_post_gather(srj_plan *p, const int64_t *dst, const int64_t *src, int64_t n) {
  if (!p) return fail(SRJ_EINVAL, "null plan");
  if (n < 0 || (n > 0 && (!dst || !src))) return fail(SRJ_EINVAL, "bad gather arguments");
  free_gather(p);
  if (n == 0) return SRJ_OK;
  const srj_layout_t &l = p->d.layout;
  if (!p->d.physical_lo0 || !p->d.physical_hi0 || p->d.own0_begin != 0 || p->d.own0_end != l.n[0])
    return fail(SRJ_EUNSUPPORTED, "post-sweep gathers need the whole grid on one plan");
  std::vector<int64_t> sorted_dst(dst, dst + n);
  for (int64_t i = 0; i < n; ++i)
    if (dst[i] < 0 || dst[i] >= l.elems || src[i] < 0 || src[i] >= l.elems)
      return fail(SRJ_EINVAL, "gather offset %lld out of range", (long long)i);
  std::sort(sorted_dst.begin(), sorted_dst.end());
  if (std::adjacent_find(sorted_dst.begin(), sorted_dst.end()) != sorted_dst.end())
    return fail(SRJ_EINVAL, "gather destinations must be distinct");
  bool overlap = false;
  for (int64_t i = 0; i < n && !overlap; ++i)
    overlap = std::binary_search(sorted_dst.begin(), sorted_dst.end(), src[i]);
  const size_t bytes = sizeof(int64_t) * size_t(n);
  cudaError_t e = scratch_alloc(&p->g_dst, bytes);
  if (e == cudaSuccess) e = scratch_alloc(&p->g_src, bytes);
  if (e == cudaSuccess && overlap) e = scratch_alloc(&p->g_tmp, sizeof(double) * size_t(n));
  if (e == cudaSuccess) e = cudaMemcpy(p->g_dst, dst, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->g_src, src, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    free_gather(p);
    return cuda_fail(e, "post-gather setup");
  }
  p->g_n = n;
  return SRJ_OK;
}

int srj_plan_set_coef_classes(srj_plan *p, const int32_t *cls) {
  if (!p || !cls) return fail(SRJ_EINVAL, "null argument");
  const srj_layout_t &l = p->d.layout;  // read by the 3D per-cell kernel (srj_sweep3d.cuh)
  for (int a = 0; a < 7; ++a)
    if (cls[a] < 0 || cls[a] > (SRJ_COEF_CONST_AXIS0 | SRJ_COEF_CONST_LAST))
      return fail(SRJ_EINVAL, "bad coefficient class %d for array %d", int(cls[a]), a);
  for (int a = 0; a < 7; ++a) {
    p->cls[a] = (a < 1 + 2 * l.ndim) ? cls[a] : 0;
  }
  return SRJ_OK;
}

int srj_plan_destroy(srj_plan *p) {
  if (!p) return SRJ_OK;
  free_gather(p);
  cudaDeviceSynchronize();  // nothing in flight uses the plan's buffers (cudaFree's implicit sync)
  scratch_free(p->gs_prog);
  scratch_free(p->partials);
  scratch_free(p->row_parts);
  scratch_free(p->vtb_yh);
  scratch_free(p->vtb_yl);
  scratch_free(p->bc_scalars);
  scratch_free(p->d_omegas);
  scratch_free(p->h_omegas);
  if (p->omega_ev) cudaEventDestroy(p->omega_ev);
  delete p;
  return SRJ_OK;
}

static void row_ranges(const srj_plan_desc &d, int &lo_c, int &hi_c, int &ld_lo, int &ld_hi) {
  const srj_layout_t &l = d.layout;
  const int n0 = int(l.n[0]), h = l.halo0;
  if (d.physical_lo0) {
    lo_c = 0;
    ld_lo = -1;
  } else {
    lo_c = -h;
    ld_lo = -h;
  }
  if (d.physical_hi0) {
    hi_c = n0;
    ld_hi = n0;
  } else {
    hi_c = n0 + h;
    ld_hi = n0 + h - 1;
  }
}

static int launch_ghosts(const srj_plan_desc &d, double *u0, cudaStream_t st) {
  const srj_layout_t &l = d.layout;
  GhostParams g{};
  g.u = u0;
  g.ndim = l.ndim;
  g.stride[l.ndim - 1] = 1;
  g.stride[l.ndim - 2] = l.pitch;
  if (l.ndim == 3) g.stride[0] = l.plane;
  for (int a = 0; a < 3; ++a) g.n[a] = a < l.ndim ? int(l.n[a]) : 1;
  g.face_start[0] = 0;
  for (int f = 0; f < 2 * l.ndim; ++f) {
    const int ax = f >> 1, side = f & 1;
    int64_t size = 1;
    for (int a = 0; a < l.ndim; ++a)
      if (a != ax) size *= l.n[a];
    g.face_start[f + 1] = g.face_start[f] + size;
    g.kind[ax][side] = d.bc[ax][side].kind;
    g.value[ax][side] = d.bc[ax][side].value;
    g.values[ax][side] = d.bc[ax][side].values;
  }
  int64_t biggest = 1;
  for (int f = 0; f < 2 * l.ndim; ++f)
    biggest = std::max<int64_t>(biggest, g.face_start[f + 1] - g.face_start[f]);
  const int blocks = int(std::min<int64_t>((biggest + 255) / 256, int64_t(sm_count())));
  ghost_refresh<<<dim3(std::max(blocks, 1), 2 * l.ndim), 256, 0, st>>>(g);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

}  // extern "C" (the small-grid helpers below are C++)

// SRJ_SMALL=0 disables, =1 forces (when it fits) the cluster path; default:
// used for whole-grid 2D plans of at most kSmallCells cells
constexpr int64_t kSmallCells = 1 << 18;

int small_mode() {
  static int v = -2;
  if (v == -2) {
    const char *e = getenv("SRJ_SMALL");
    v = e ? atoi(e) : -1;
  }
  return v;
}

template <bool VAR, bool NL, bool RECIP>
static void configure_cluster() {
  static std::atomic<uint64_t> configured{0};
  once_per_device(configured, [] {
    cudaFuncSetAttribute(sweep2d_cluster<VAR, NL, RECIP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(sweep2d_cluster<VAR, NL, RECIP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  });
}

static cudaLaunchConfig_t cluster_config(int C, size_t smem, cudaStream_t st, cudaLaunchAttribute *attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(kClusterThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// Can a C-CTA cluster with `smem` bytes per CTA be co-scheduled on this
// device at all (a MIG slice or a partly busy GPC may not hold 16 CTAs)?
// Cached per (device, C, smem); a "no" sends the plan to the band kernel.
template <bool VAR, bool NL, bool RECIP>
static bool cluster_schedulable_t(int C, size_t smem) {
  static std::mutex mu;
  static std::vector<std::array<int64_t, 4>> cache;  // device, C, smem, ok
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto &e : cache)
      if (e[0] == dev && e[1] == C && e[2] == int64_t(smem)) return e[3] != 0;
  }
  configure_cluster<VAR, NL, RECIP>();
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = cluster_config(C, smem, nullptr, attr);
  int n = 0;
  const bool ok = cudaOccupancyMaxActiveClusters(&n, sweep2d_cluster<VAR, NL, RECIP>, &cfg) == cudaSuccess && n >= 1;
  cudaGetLastError();
  std::lock_guard<std::mutex> lk(mu);
  cache.push_back({dev, C, int64_t(smem), ok ? 1 : 0});
  return ok;
}

// Shared bytes per CTA: two field slabs, plus a third with the source of the
// owned cells when it fits (f_smem).
constexpr size_t kClusterSmemMax = 200 * 1024;
static size_t cluster_smem(int R, int64_t n1, bool *f_smem) {
  const size_t slab = size_t(R + 2) * size_t(n1 + 2) * 8;
  const bool fits = 3 * slab <= kClusterSmemMax;
  if (f_smem) *f_smem = fits;
  return (fits ? 3 : 2) * slab;
}

static bool cluster_schedulable(const srj_plan &plan, int C, int R) {
  const srj_plan_desc &d = plan.d;
  const bool var = d.coef_mode == 1, nl = d.kappa != nullptr;
  const bool recip = !var && recip_or_zero(d.coef[0]) != 0.0;
  const size_t smem = cluster_smem(R, d.layout.n[1], nullptr);
  if (var) return nl ? cluster_schedulable_t<true, true, false>(C, smem) : cluster_schedulable_t<true, false, false>(C, smem);
  if (recip) return nl ? cluster_schedulable_t<false, true, true>(C, smem) : cluster_schedulable_t<false, false, true>(C, smem);
  return nl ? cluster_schedulable_t<false, true, false>(C, smem) : cluster_schedulable_t<false, false, false>(C, smem);
}

static bool cluster_fits(const srj_plan &plan, int &C, int &R) {
  const srj_plan_desc &d = plan.d;
  const srj_layout_t &l = d.layout;
  if (l.ndim != 2 || !d.physical_lo0 || !d.physical_hi0 || l.halo0 != 1) return false;
  if (d.own0_begin != 0 || d.own0_end != l.n[0]) return false;
  const int mode = small_mode();
  if (mode == 0) return false;
  if (mode < 0 && l.n[0] * l.n[1] > kSmallCells) return false;
  const int n0 = int(l.n[0]);
  C = std::min(kClusterMax, n0);
  R = (n0 + C - 1) / C;
  C = (n0 + R - 1) / R;
  // cells per CTA <= 16 x 1024 threads (the row division by n1_magic is exact
  // for them); n1 >= 2 keeps ceil(2^32 / n1) in 32 bits
  if (R > kTY * kMaxA || l.n[1] > kTX * kMaxB || l.n[1] < 2) return false;
  const size_t bytes = 2 * size_t(R + 2) * size_t(l.n[1] + 2) * 8;
  return bytes <= 200 * 1024 && cluster_schedulable(plan, C, R);
}

template <bool VAR, bool NL, bool RECIP>
static int launch_cluster(const Cluster2DParams &p, int C, size_t smem, cudaStream_t st) {
  configure_cluster<VAR, NL, RECIP>();
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = cluster_config(C, smem, st, attr);
  SRJ_CUDA(cudaLaunchKernelEx(&cfg, sweep2d_cluster<VAR, NL, RECIP>, p));
  return SRJ_OK;
}

static int run_cluster2d(srj_plan &plan, const double *src, double *dst, const double *weights,
                         int64_t m, int64_t first, int64_t nsteps, double *d_norms,
                         int32_t *final_buf, cudaStream_t st, int C, int R) {
  const srj_plan_desc &d = plan.d;
  const srj_layout_t &l = d.layout;
  if (nsteps > plan.omega_cap) {
    if (plan.d_omegas || plan.h_omegas) cudaDeviceSynchronize();  // the old staging buffers
    scratch_free(plan.d_omegas);
    scratch_free(plan.h_omegas);
    plan.d_omegas = plan.h_omegas = nullptr;
    plan.omega_cap = 0;
    SRJ_CUDA(scratch_alloc(&plan.d_omegas, sizeof(double) * size_t(nsteps)));
    SRJ_CUDA(scratch_alloc_host(&plan.h_omegas, sizeof(double) * size_t(nsteps)));
    if (!plan.omega_ev) SRJ_CUDA(cudaEventCreateWithFlags(&plan.omega_ev, cudaEventDisableTiming));
    plan.omega_cap = nsteps;
  } else if (plan.omega_ev) {
    SRJ_CUDA(cudaEventSynchronize(plan.omega_ev));  // staging buffer free again
  }
  for (int64_t k = 0; k < nsteps; ++k) plan.h_omegas[k] = weights[(first + k) % m];
  SRJ_CUDA(cudaMemcpyAsync(plan.d_omegas, plan.h_omegas, sizeof(double) * size_t(nsteps),
                           cudaMemcpyHostToDevice, st));
  SRJ_CUDA(cudaEventRecord(plan.omega_ev, st));
  const int64_t ioff = interior_offset(l);
  Cluster2DParams p{};
  p.src = src + ioff;
  p.dst = dst + ioff;
  const bool nl = d.kappa != nullptr, var = d.coef_mode == 1;
  p.f = (nl ? d.kappa : d.source) + ioff;
  p.act = d.act ? d.act + ioff : nullptr;
  if (var) {
    p.c = d.coef_arrays[0] + ioff;
    p.am0 = d.coef_arrays[1] + ioff;
    p.ap0 = d.coef_arrays[2] + ioff;
    p.am1 = d.coef_arrays[3] + ioff;
    p.ap1 = d.coef_arrays[4] + ioff;
  }
  p.kc = d.coef[0];
  p.kam0 = d.coef[1];
  p.kap0 = d.coef[2];
  p.kam1 = d.coef[3];
  p.kap1 = d.coef[4];
  p.pitch = l.pitch;
  p.n0 = int(l.n[0]);
  p.n1 = int(l.n[1]);
  p.R = R;
  p.sp = int(l.n[1]) + 2;
  for (int a = 0; a < 2; ++a)
    for (int side = 0; side < 2; ++side) {
      p.bc_kind[a][side] = d.bc[a][side].kind;
      p.bc_value[a][side] = d.bc[a][side].value;
      p.bc_values[a][side] = d.bc[a][side].values;
    }
  p.omegas = plan.d_omegas;
  p.nsteps = int(nsteps);
  p.n1_magic = unsigned(((uint64_t(1) << 32) + uint64_t(l.n[1]) - 1) / uint64_t(l.n[1]));
  p.norms = d_norms;
  bool f_smem = false;
  const size_t smem = cluster_smem(R, l.n[1], &f_smem);
  p.f_smem = f_smem ? 1 : 0;
  p.kinv = var ? 0.0 : recip_or_zero(d.coef[0]);
  p.kinv_lo = recip_lo(d.coef[0], p.kinv);
  const bool recip = !var && p.kinv != 0.0;
  int rc;
  if (var)
    rc = nl ? launch_cluster<true, true, false>(p, C, smem, st)
            : launch_cluster<true, false, false>(p, C, smem, st);
  else if (recip)
    rc = nl ? launch_cluster<false, true, true>(p, C, smem, st)
            : launch_cluster<false, false, true>(p, C, smem, st);
  else
    rc = nl ? launch_cluster<false, true, false>(p, C, smem, st)
            : launch_cluster<false, false, false>(p, C, smem, st);
  if (rc != SRJ_OK) return rc;
  *final_buf = 1;
  return SRJ_OK;
}

// One launch of t fused sweeps (weights om[0..t)) from `cur` into `nxt`,
// relaxing, storing and counting local axis-0 rows [own_b, own_e) only (the
// plan's own range, or a part of it: the slab exchange's edge / inner
// launches).  Per-step (dmax, rmax) are folded into norms[2*q..] with
// atomicMax, so several parts of one step may share a norm slot.
// Which launches can store slab edge rows straight into the neighbours' halos
// (PeerSend): the constant-stencil 2D band kernel up to depth kMaxFuseSend, in
// 3D the register-streaming T = 2 kernel plus the one-sweep kernel for a
// chunk's odd last step, and the per-cell one-sweep kernels (2D and 3D).
static bool direct_send_ok(const srj_plan &plan, int T) {
  const srj_plan_desc &d = plan.d;
  if (plan.has_bc) return false;
  if (d.coef_mode != 0) return T == 1;
  if (d.layout.ndim == 2) return T <= kMaxFuseSend;
  return T <= 2 && !rs3d_disabled();
}

static int launch_fused(srj_plan &plan, int64_t own_b, int64_t own_e, const double *cur,
                        double *nxt, const double *om, int t, double *norms, cudaStream_t st,
                        const PeerSend *send = nullptr) {
  const srj_plan_desc &d = plan.d;
  const srj_layout_t &l = d.layout;
  const int64_t ioff = interior_offset(l);
  const bool var = d.coef_mode == 1;
  if (send && !direct_send_ok(plan, t))
    return fail(SRJ_EINVAL, "direct halo stores are not available for this launch");
  const bool nl = d.kappa != nullptr;
  const double *f = nl ? d.kappa : d.source;
  int lo_c, hi_c, ld_lo, ld_hi;
  row_ranges(d, lo_c, hi_c, ld_lo, ld_hi);
  const int rows = int(own_e - own_b);
  if (l.ndim == 2 && var && t == 1) {
    const int rc = launch_var2d(d, own_b, own_e, cur, nxt, f, ld_lo, ld_hi, om[0], norms, st, send);
    if (rc != SRJ_OK) return rc;
  } else if (l.ndim == 2 && var && t == 2 && !plan.has_bc) {
    // two fused steps on per-cell coefficients (srj_sweep2d_vtb.cuh)
    VarTB2DParams p{};
    p.src = cur + ioff;
    p.dst = nxt + ioff;
    p.f = f + ioff;
    p.act = d.act ? d.act + ioff : nullptr;
    p.c = d.coef_arrays[0] + ioff;
    p.am0 = d.coef_arrays[1] + ioff;
    p.ap0 = d.coef_arrays[2] + ioff;
    p.am1 = d.coef_arrays[3] + ioff;
    p.ap1 = d.coef_arrays[4] + ioff;
    if (!plan.vtb_yh) {  // first fused per-cell launch: reciprocals of the centre
      const size_t bytes = sizeof(double) * size_t(l.elems);
      SRJ_CUDA(scratch_alloc(&plan.vtb_yh, bytes));
      SRJ_CUDA(scratch_alloc(&plan.vtb_yl, bytes));
      SRJ_CUDA(cudaMemsetAsync(plan.vtb_yh, 0, bytes, st));
      SRJ_CUDA(cudaMemsetAsync(plan.vtb_yl, 0, bytes, st));
      vtb_recip<<<sm_count() * 8, 256, 0, st>>>(d.coef_arrays[0] + ioff, plan.vtb_yh + ioff,
                                                plan.vtb_yl + ioff, l.pitch, int(l.n[0]),
                                                int(l.n[1]));
      SRJ_CUDA(cudaGetLastError());
    }
    p.yh = plan.vtb_yh + ioff;
    p.yl = plan.vtb_yl + ioff;
    p.pitch = l.pitch;
    p.n0 = int(l.n[0]);
    p.n1 = int(l.n[1]);
    p.lo_c = lo_c;
    p.hi_c = hi_c;
    p.ld_lo = ld_lo;
    p.ld_hi = ld_hi;
    p.own_b = int(own_b);
    p.own_e = int(own_e);
    // last interior column (relative to the row origin) a double2 load may
    // start at: element origin+1+col+1 stays inside the padded row
    p.col_max = int(l.pitch - (l.origin + 1) - 2) & ~1;
    p.mcol_max = int(l.pitch - (l.origin + 1) - 4) & ~3;
    p.omega[0] = om[0];
    p.omega[1] = om[1];
    p.norms = norms;
    const int rc = launch_var2d_tb(p, nl, st);
    if (rc != SRJ_OK) return rc;
  } else if (l.ndim == 2) {
    Sweep2DParams p{};
    p.src = cur + ioff;
    p.dst = nxt + ioff;
    p.f = f + ioff;
    p.act = d.act ? d.act + ioff : nullptr;
    if (var) {
      p.c = d.coef_arrays[0] + ioff;
      p.am0 = d.coef_arrays[1] + ioff;
      p.ap0 = d.coef_arrays[2] + ioff;
      p.am1 = d.coef_arrays[3] + ioff;
      p.ap1 = d.coef_arrays[4] + ioff;
    }
    p.kc = d.coef[0];
    p.kam0 = d.coef[1];
    p.kap0 = d.coef[2];
    p.kam1 = d.coef[3];
    p.kap1 = d.coef[4];
    p.kinv = recip_or_zero(d.coef[0]);
    p.kinv_lo = recip_lo(d.coef[0], p.kinv);
    p.pitch = l.pitch;
    p.n0 = int(l.n[0]);
    p.n1 = int(l.n[1]);
    p.lo_c = lo_c;
    p.hi_c = hi_c;
    p.ld_lo = ld_lo;
    p.ld_hi = ld_hi;
    p.own_b = int(own_b);
    p.own_e = int(own_e);
    if (send) p.send = *send;
    int bcf = 0;
    if (plan.has_bc && t > 1) {
      bcf = 2;
      for (int side = 0; side < 2; ++side)
        if (d.bc[1][side].kind == SRJ_BC_FACE_DIRICHLET) bcf = 1;
    }
    const Kernel2D k2 = pick2d(t, var, nl, !var && p.kinv != 0.0, bcf, send != nullptr);
    p.nbands = int((l.n[1] + k2.own - 1) / k2.own);
    // strips x bands = waves x resident warps (default one wave)
    const int bps = bps_override() > 0 ? std::min(bps_override(), k2.blocks_per_sm())
                                       : k2.blocks_per_sm();
    const int capacity = sm_count() * bps * Band2D<1, 2>::WARPS * waves_2d();
    int nstrips = std::max(1, capacity / p.nbands);
    nstrips = std::min(nstrips, std::max(1, rows / std::max(2 * t, 8)));
    p.H = (rows + nstrips - 1) / nstrips;
    p.nstrips = (rows + p.H - 1) / p.H;
    for (int q = 0; q < t; ++q) p.omega[q] = om[q];
    p.norms = norms;
    p.tma_col0 = int(l.origin + 1);
    p.tma_row0 = l.halo0;
    for (int a = 0; a < 2; ++a)
      for (int side = 0; side < 2; ++side) {
        const srj_face_rule &b = d.bc[a][side];
        p.bc_kind[a][side] = b.kind;
        const bool arr = b.kind == SRJ_BC_FACE_DIRICHLET && b.values;
        p.bc_ptr[a][side] = arr ? b.values : plan.bc_scalars + 2 * a + side;
        p.bc_step[a][side] = arr ? 1 : 0;
      }
    CUtensorMap tu, tf;
    int rc = plan_tmap(plan, &tu, cur, k2.box_cols, 3);
    if (rc != SRJ_OK) return rc;
    rc = plan_tmap(plan, &tf, f, k2.box_cols, 3);
    if (rc != SRJ_OK) return rc;
    const int warps = p.nbands * p.nstrips;
    const int blocks = (warps + Band2D<1, 2>::WARPS - 1) / Band2D<1, 2>::WARPS;
    k2.launch(p, tu, tf, blocks, st);
  } else if (t > 1) {
    // temporally blocked 3D (constant stencil): t fused sweeps per launch
    Sweep3DTBParams p{};
    p.dst = nxt + ioff;
    for (int a = 0; a < 7; ++a) p.kc[a] = d.coef[a];
    p.kinv = recip_or_zero(d.coef[0]);
    p.kinv_lo = recip_lo(d.coef[0], p.kinv);
    p.pitch = l.pitch;
    p.plane = l.plane;
    p.n0 = int(l.n[0]);
    p.n1 = int(l.n[1]);
    p.n2 = int(l.n[2]);
    p.ld_lo = ld_lo;
    p.ld_hi = ld_hi;
    p.own_b = int(own_b);
    p.own_e = int(own_e);
    p.tma_col0 = int(l.origin + 1);
    p.rows_per_plane = int(l.n[1] + 2);
    p.tma_row0 = l.halo0 * p.rows_per_plane + 1;  // row of (i=0, j=0)
    for (int q = 0; q < t; ++q) p.omega[q] = om[q];
    p.norms = norms;
    if (send) p.send = *send;
    for (int a = 0; a < 3; ++a)
      for (int side = 0; side < 2; ++side) {
        const srj_face_rule &b = d.bc[a][side];
        p.bc_kind[a][side] = b.kind;
        const bool arr = b.kind == SRJ_BC_FACE_DIRICHLET && b.values;
        p.bc_ptr[a][side] = arr ? b.values : plan.bc_scalars + 2 * a + side;
        p.bc_step[a][side] = arr ? 1 : 0;
      }
    int bcf = 0;
    if (plan.has_bc) {
      bcf = 2;
      for (int a = 0; a < 3; ++a)
        for (int side = 0; side < 2; ++side)
          if (d.bc[a][side].kind == SRJ_BC_FACE_DIRICHLET) bcf = 1;
    }
    const Kernel3DTB k3 = pick3d_tb(t, nl, p.kinv != 0.0, bcf, send != nullptr);
    if (send && !k3.persistent)
      return fail(SRJ_EINVAL, "direct halo stores need the register-streaming 3D kernel");
    p.ntj = int((l.n[1] + k3.tj - 1) / k3.tj);
    p.ntk = int((l.n[2] + k3.tk - 1) / k3.tk);
    const long tiles = long(p.ntj) * p.ntk;
    const long capacity = long(sm_count()) * k3.blocks_per_sm();
    int nstrips = 1;
    double best = -1.0;
    for (int ns = 1; ns <= std::max(1, std::min(64, rows / (4 * t))); ++ns) {
      const long w = tiles * ns;
      const long waves = (w + capacity - 1) / capacity;
      const double hh = double(rows) / ns;
      const double eff = double(w) / double(waves * capacity) * hh / (hh + 2.0 * t);
      if (eff > best + 1e-9) {
        best = eff;
        nstrips = ns;
      }
    }
    p.H = (rows + nstrips - 1) / nstrips;
    p.nstrips = (rows + p.H - 1) / p.H;
    CUtensorMap tu, tf;
    int rc = plan_tmap(plan, &tu, cur, k3.box_cols, k3.box_rows);
    if (rc != SRJ_OK) return rc;
    rc = plan_tmap(plan, &tf, f, k3.box_cols, k3.f_box_rows);
    if (rc != SRJ_OK) return rc;
    long blocks = tiles * p.nstrips;
    if (k3.persistent) {
      // one CTA per resident slot, at least kMinPlanes planes each: a small
      // grid is spread over more CTAs (each pays the 5-tick pipeline fill, but
      // on SMs that would idle) -- 2 instead of 8: 64^3 12.5 -> ~7 us per sweep
      const long min_planes = min_planes_3d();
      blocks = std::max(1L, std::min(capacity, (tiles * rows + min_planes - 1) / min_planes));
    }
    k3.launch(p, tu, tf, int(blocks), st);
  } else {
    Sweep3DParams p{};
    p.src = cur + ioff;
    p.dst = nxt + ioff;
    p.f = f + ioff;
    p.act = d.act ? d.act + ioff : nullptr;
    bool cls = false;
    for (int a = 0; a < 7; ++a) {
      p.coef[a] = var ? d.coef_arrays[a] + ioff : nullptr;
      p.kc[a] = d.coef[a];
      class_strides(plan.cls, a, l.plane, p.cplane[a], p.ccol[a]);
      cls |= var && plan.cls[a] != 0;
    }
    p.pitch = l.pitch;
    p.plane = l.plane;
    p.n0 = int(l.n[0]);
    p.n1 = int(l.n[1]);
    p.n2 = int(l.n[2]);
    // one-deep stencil: only owned rows relax; exchanged halos are inputs
    p.lo_c = 0;
    p.hi_c = p.n0;
    p.ld_lo = ld_lo;
    p.ld_hi = ld_hi;
    p.own_b = int(own_b);
    p.own_e = int(own_e);
    if (send) p.send = *send;
    p.nbands = int((l.n[2] + 63) / 64);
    p.njg = int((l.n[1] + kRows3D - 1) / kRows3D);
    p.kinv = var ? 0.0 : recip_or_zero(d.coef[0]);
    p.kinv_lo = recip_lo(d.coef[0], p.kinv);
    const bool recip = !var && p.kinv != 0.0;
    const Kernel3D k3 = pick3d(var, nl, recip, cls, send != nullptr);
    const long per_strip = long(p.njg) * p.nbands;
    const long capacity = long(sm_count()) * k3.blocks_per_sm() * kWarps3D;
    // strips: best fill of whole waves, discounting the 2 halo planes per strip
    int nstrips = 1;
    double best = -1.0;
    for (int ns = 1; ns <= std::max(1, std::min(64, rows / 8)); ++ns) {
      const long w = per_strip * ns;
      const long waves = (w + capacity - 1) / capacity;
      const double hh = double(rows) / ns;
      const double eff = double(w) / double(waves * capacity) * hh / (hh + 2.0);
      if (eff > best + 1e-9) {
        best = eff;
        nstrips = ns;
      }
    }
    p.H = (rows + nstrips - 1) / nstrips;
    p.nstrips = (rows + p.H - 1) / p.H;
    p.omega = om[0];
    p.norms = norms;
    const long warps = per_strip * p.nstrips;
    k3.launch(p, int((warps + kWarps3D - 1) / kWarps3D), st);
  }
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

// effective fused depth for a plan (srj_plan_run's rules)
static int plan_depth(const srj_plan &plan, int fuse) {
  const srj_plan_desc &d = plan.d;
  const srj_layout_t &l = d.layout;
  int T = fuse > 0 ? fuse : plan.default_fuse;
  if ((plan.has_bc && !plan.bc_fusable) || plan.g_n > 0 || (l.ndim == 3 && d.coef_mode == 1)) T = 1;
  if (plan.has_bc && T > kMaxFuseBC) T = kMaxFuseBC;
  if (l.ndim == 3 && T > kMaxFuse3D) T = kMaxFuse3D;
  return T;
}

// ------------------------------------------------------- slab exchange
// Driver entry points (no -lcuda): stream memory operations order the halo
// exchange between ranks on the device, with no host round trip per launch.
struct DriverOps {
  PFN_cuStreamWaitValue32_v11070 wait32 = nullptr;
  PFN_cuStreamWriteValue32_v11070 write32 = nullptr;
  PFN_cuMemGetAddressRange_v3020 addr_range = nullptr;
  PFN_cuStreamBatchMemOp_v11070 batch = nullptr;
  bool ok = false;
  bool ops64 = false;  // 64-bit wait / write stream operations on the current device
};

static const DriverOps &driver_ops() {
  static DriverOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void *a = nullptr, *b = nullptr, *c = nullptr, *e = nullptr;
    cudaDriverEntryPointQueryResult q1, q2, q3, q4;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &a, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &b, cudaEnableDefault, &q2) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuMemGetAddressRange", &c, cudaEnableDefault, &q3) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamBatchMemOp", &e, cudaEnableDefault, &q4) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess &&
        q3 == cudaDriverEntryPointSuccess && q4 == cudaDriverEntryPointSuccess) {
      ops.wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(a);
      ops.write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(b);
      ops.addr_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(c);
      ops.batch = reinterpret_cast<PFN_cuStreamBatchMemOp_v11070>(e);
      ops.ok = true;
      void *g = nullptr;
      cudaDriverEntryPointQueryResult q5;
      int dev = 0, v = 0;
      if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &g, cudaEnableDefault, &q5) == cudaSuccess &&
          q5 == cudaDriverEntryPointSuccess && cudaGetDevice(&dev) == cudaSuccess &&
          reinterpret_cast<PFN_cuDeviceGetAttribute_v2000>(g)(
              &v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev) == CUDA_SUCCESS)
        ops.ops64 = v != 0;
    }
    cudaGetLastError();
  });
  return ops;
}

// flag words of a rank's block (written by its neighbours)
// Flag words of a rank: per side (0 = written by the lower, 1 = by the upper
// neighbour) an adjacent pair {arrived, done} -- one aligned 64-bit word, so
// the direct path waits for / writes both with one stream operation.
enum { kFlagArrived = 0, kFlagDone = 1 };  // + 2 * side

struct srj_slab {
  srj_plan *plan = nullptr;   // the rank's plan (owned rows = desc own range)
  double *bufs[3] = {};
  uint32_t *flags = nullptr;  // SRJ_SLAB_FLAG_WORDS words, device
  int halo = 1;
  bool has[2] = {false, false};
  srj_slab_peer peer[2] = {};
  uint32_t epoch = 0;         // launches run since the last reset (all ranks agree)
  int device = 0;
  cudaStream_t comm = nullptr, edge = nullptr;  // peer copies; edge-row launches
  cudaEvent_t ev_edge = nullptr, ev_copy = nullptr, ev_inner = nullptr;
  // local interior row ranges: edges (sent after every launch) and inner
  int64_t part_b[3] = {}, part_e[3] = {};  // [0] lower edge, [1] upper edge, [2] inner (empty: b == e)
};

// Flag writes as a one-thread kernel: the fallback when the driver refuses a
// stream write operation on a peer-mapped address (and SRJ_SLAB_FLAG_KERNEL=1
// forces it, so the path is tested on one GPU).  System-scope release order
// after the preceding kernel's stores is the stream order itself.
struct FlagWrites {
  unsigned long long addr[8];
  unsigned long long value[8];
  int width[8];  // 4 or 8 bytes
  int n;
};

__global__ void flag_write_kernel(const FlagWrites w) {
  __threadfence_system();
  for (int i = 0; i < w.n; ++i) {
    if (w.width[i] == 8)
      *reinterpret_cast<volatile unsigned long long *>(w.addr[i]) = w.value[i];
    else
      *reinterpret_cast<volatile unsigned int *>(w.addr[i]) = static_cast<unsigned int>(w.value[i]);
  }
  __threadfence_system();
}

static std::atomic<int> g_flag_kernel{-1};  // -1: not decided, 0: stream operations, 1: kernel
static bool flag_kernel_mode() {
  int v = g_flag_kernel.load();
  if (v < 0) {
    const char *e = getenv("SRJ_SLAB_FLAG_KERNEL");
    v = (e && atoi(e) == 1) ? 1 : 0;
    g_flag_kernel.store(v);
  }
  return v == 1;
}

// Flag operations of one phase, enqueued with ONE cuStreamBatchMemOp call
// (executed in array order): halves the host API calls per fused launch.
struct FlagOps {
  CUstreamBatchMemOpParams p[8];
  unsigned n = 0;
  void wait(uint32_t *addr, uint32_t v) {
    CUstreamBatchMemOpParams &x = p[n++];
    std::memset(&x, 0, sizeof(x));
    x.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    x.waitValue.address = CUdeviceptr(addr);
    x.waitValue.value = v;
    x.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  }
  void write(uint32_t *addr, uint32_t v) {
    CUstreamBatchMemOpParams &x = p[n++];
    std::memset(&x, 0, sizeof(x));
    x.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    x.writeValue.address = CUdeviceptr(addr);
    x.writeValue.value = v;
    x.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  }
  // both flags of a side at once: {arrived, done} as one 64-bit word, done in
  // the high half.  "arrived >= v and done >= v" is the unsigned 64-bit test
  // word >= (v, v): a neighbour's done flag never runs more than one launch
  // ahead of its arrived flag (its launch j+1 starts after its rows of launch
  // j were delivered), so done > v implies arrived >= v.
  void wait_pair(uint32_t *pair, uint32_t v) {
    if (!driver_ops().ops64) {
      wait(pair + kFlagArrived, v);
      wait(pair + kFlagDone, v);
      return;
    }
    CUstreamBatchMemOpParams &x = p[n++];
    std::memset(&x, 0, sizeof(x));
    x.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
    x.waitValue.address = CUdeviceptr(pair);
    x.waitValue.value64 = (uint64_t(v) << 32) | v;
    x.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  }
  void write_pair(uint32_t *pair, uint32_t v) {
    if (!driver_ops().ops64) {
      write(pair + kFlagArrived, v);
      write(pair + kFlagDone, v);
      return;
    }
    CUstreamBatchMemOpParams &x = p[n++];
    std::memset(&x, 0, sizeof(x));
    x.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    x.writeValue.address = CUdeviceptr(pair);
    x.writeValue.value64 = (uint64_t(v) << 32) | v;
    x.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  }
  int flush(cudaStream_t st) {
    if (n == 0) return SRJ_OK;
    if (getenv("SRJ_SLAB_NOFLAGS")) {  // timing experiments only: results are undefined
      n = 0;
      return SRJ_OK;
    }
    if (!flag_kernel_mode()) {
      const CUresult r = driver_ops().batch(reinterpret_cast<CUstream>(st), n, p, 0);
      if (r == CUDA_SUCCESS) {
        n = 0;
        return SRJ_OK;
      }
      bool has_write = false;
      for (unsigned i = 0; i < n; ++i)
        has_write |= p[i].operation != CU_STREAM_MEM_OP_WAIT_VALUE_32 &&
                     p[i].operation != CU_STREAM_MEM_OP_WAIT_VALUE_64;
      if (!has_write) {
        n = 0;
        return fail(SRJ_ECUDA, "cuStreamBatchMemOp failed (%d)", int(r));
      }
      // a refused write (peer-mapped flag word): from now on write by kernel
      cudaGetLastError();
      g_flag_kernel.store(1);
    }
    // array order is kept: runs of waits go through the batch call, runs of
    // writes through the one-thread kernel
    unsigned i = 0;
    while (i < n) {
      const bool is_wait = p[i].operation == CU_STREAM_MEM_OP_WAIT_VALUE_32 ||
                           p[i].operation == CU_STREAM_MEM_OP_WAIT_VALUE_64;
      unsigned j = i;
      if (is_wait) {
        while (j < n && (p[j].operation == CU_STREAM_MEM_OP_WAIT_VALUE_32 ||
                         p[j].operation == CU_STREAM_MEM_OP_WAIT_VALUE_64))
          ++j;
        const CUresult r = driver_ops().batch(reinterpret_cast<CUstream>(st), j - i, p + i, 0);
        if (r != CUDA_SUCCESS) {
          n = 0;
          return fail(SRJ_ECUDA, "cuStreamBatchMemOp (waits) failed (%d)", int(r));
        }
      } else {
        FlagWrites w{};
        while (j < n && (p[j].operation == CU_STREAM_MEM_OP_WRITE_VALUE_32 ||
                         p[j].operation == CU_STREAM_MEM_OP_WRITE_VALUE_64)) {
          const bool wide = p[j].operation == CU_STREAM_MEM_OP_WRITE_VALUE_64;
          w.addr[w.n] = static_cast<unsigned long long>(p[j].writeValue.address);
          w.value[w.n] = wide ? p[j].writeValue.value64 : p[j].writeValue.value;
          w.width[w.n] = wide ? 8 : 4;
          ++w.n;
          ++j;
        }
        flag_write_kernel<<<1, 1, 0, st>>>(w);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
          n = 0;
          return cuda_fail(e, "flag_write_kernel");
        }
      }
      i = j;
    }
    n = 0;
    return SRJ_OK;
  }
};

// element offset of local interior row `row` (layer row + halo0) in a field buffer
static int64_t layer_offset(const srj_layout_t &l, int64_t row) {
  return l.origin + (row + l.halo0) * l.plane;
}

extern "C" {

int srj_plan_run(srj_plan *plan, const double *src, double *buf_a, double *buf_b,
                 const double *weights, int64_t m, int64_t first, int64_t nsteps, int32_t fuse,
                 double *d_norms, int32_t *final_buf, void *stream) {
  if (!plan || !src || !buf_a || !buf_b || !weights || !final_buf)
    return fail(SRJ_EINVAL, "null argument");
  if (m < 1) return fail(SRJ_EINVAL, "weight cycle must be non-empty");
  if (nsteps < 0 || first < 0) return fail(SRJ_EINVAL, "negative step range");
  if (src == buf_a || src == buf_b || buf_a == buf_b)
    return fail(SRJ_EINVAL, "src, buf_a and buf_b must be distinct");
  *final_buf = 0;
  if (nsteps == 0) return SRJ_OK;
  if (!d_norms) return fail(SRJ_EINVAL, "null norms buffer");
  const srj_plan_desc &d = plan->d;
  const srj_layout_t &l = d.layout;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int T = plan_depth(*plan, fuse);
  if (T > kMaxFuse) return fail(SRJ_EINVAL, "fuse depth %d exceeds %d", T, kMaxFuse);
  if ((!d.physical_lo0 || !d.physical_hi0) && T > l.halo0 && T > 1)
    return fail(SRJ_EINVAL, "fuse depth %d needs halo0 >= %d on exchanged faces", T, T);

  SRJ_CUDA(cudaMemsetAsync(d_norms, 0, sizeof(double) * 2 * size_t(nsteps), st));
  const int64_t ioff = interior_offset(l);
  if (l.ndim == 2 && plan->g_n == 0) {
    int C = 0, R = 0;
    if (cluster_fits(*plan, C, R)) return run_cluster2d(*plan, src, buf_a, weights, m, first, nsteps, d_norms, final_buf, st, C, R);
  }
  const double *cur = src;
  double *nxt = buf_a;
  int which = 1;
  int64_t k = 0;
  while (k < nsteps) {
    const int t = int(std::min<int64_t>(T, nsteps - k));
    double om[kMaxFuse];
    for (int q = 0; q < t; ++q) om[q] = weights[(first + k + q) % m];
    int rc = launch_fused(*plan, d.own0_begin, d.own0_end, cur, nxt, om, t, d_norms + 2 * k, st);
    if (rc != SRJ_OK) return rc;
    if (plan->has_bc) {
      rc = launch_ghosts(d, nxt + ioff, st);
      if (rc != SRJ_OK) return rc;
    }
    if (plan->g_n > 0) {
      rc = launch_gather(*plan, nxt, st);
      if (rc != SRJ_OK) return rc;
    }
    k += t;
    *final_buf = which;
    cur = nxt;
    nxt = (which == 1) ? buf_b : buf_a;
    which = (which == 1) ? 2 : 1;
  }
  return SRJ_OK;
}

static ResidParams resid_params(const srj_plan &plan, const double *u) {
  const srj_plan_desc &d = plan.d;
  const srj_layout_t &l = d.layout;
  const int64_t ioff = interior_offset(l);
  ResidParams p{};
  p.u = u + ioff;
  const bool nl = d.kappa != nullptr;
  p.f = (nl ? d.kappa : d.source) + ioff;
  p.act = d.act ? d.act + ioff : nullptr;
  const bool var = d.coef_mode == 1;
  for (int a = 0; a < 7; ++a) {
    p.coef[a] = (var && a < 1 + 2 * l.ndim) ? d.coef_arrays[a] + ioff : nullptr;
    p.kc[a] = d.coef[a];
  }
  p.pitch = l.pitch;
  p.plane = l.plane;
  p.ndim = l.ndim;
  p.n0 = int(l.n[0]);
  p.n1 = int(l.n[1]);
  p.n2 = (l.ndim == 3) ? int(l.n[2]) : 1;
  p.own_b = int(d.own0_begin);
  p.own_e = int(d.own0_end);
  p.partials = plan.partials;
  return p;
}

int srj_plan_residual(srj_plan *plan, const double *u, double *d_out, void *stream) {
  if (!plan || !u || !d_out) return fail(SRJ_EINVAL, "null argument");
  const srj_plan_desc &d = plan->d;
  const ResidParams p = resid_params(*plan, u);
  const bool nl = d.kappa != nullptr, var = d.coef_mode == 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (var)
    nl ? residual_partial<true, true><<<plan->resid_blocks, kResidThreads, 0, st>>>(p)
       : residual_partial<true, false><<<plan->resid_blocks, kResidThreads, 0, st>>>(p);
  else
    nl ? residual_partial<false, true><<<plan->resid_blocks, kResidThreads, 0, st>>>(p)
       : residual_partial<false, false><<<plan->resid_blocks, kResidThreads, 0, st>>>(p);
  residual_final<<<1, 32, 0, st>>>(plan->partials, plan->resid_blocks, d_out);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

int srj_plan_residual_layers(srj_plan *plan, const double *u, double *d_layers, void *stream) {
  if (!plan || !u || !d_layers) return fail(SRJ_EINVAL, "null argument");
  const srj_plan_desc &d = plan->d;
  const srj_layout_t &l = d.layout;
  const ResidParams p = resid_params(*plan, u);
  const bool nl = d.kappa != nullptr, var = d.coef_mode == 1;
  const int64_t layers = d.own0_end - d.own0_begin;
  if (layers <= 0) return SRJ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *rows_out = d_layers;
  if (l.ndim == 3) {
    const int64_t need = 2 * layers * l.n[1];
    if (need > plan->row_parts_cap) {
      if (plan->row_parts) {
        cudaDeviceSynchronize();
        scratch_free(plan->row_parts);
      }
      plan->row_parts = nullptr;
      plan->row_parts_cap = 0;
      SRJ_CUDA(scratch_alloc(&plan->row_parts, sizeof(double) * size_t(need)));
      plan->row_parts_cap = need;
    }
    rows_out = plan->row_parts;
  }
  const int blocks = sm_count() * 8;  // 64 warps per SM, grid-stride over rows
  if (var)
    nl ? residual_rows<true, true><<<blocks, 256, 0, st>>>(p, rows_out)
       : residual_rows<true, false><<<blocks, 256, 0, st>>>(p, rows_out);
  else
    nl ? residual_rows<false, true><<<blocks, 256, 0, st>>>(p, rows_out)
       : residual_rows<false, false><<<blocks, 256, 0, st>>>(p, rows_out);
  if (l.ndim == 3) {
    const int lb = int(std::min<int64_t>((layers + 7) / 8, int64_t(sm_count()) * 4));
    residual_layers<<<lb, 256, 0, st>>>(plan->row_parts, int(layers), int(l.n[1]), d_layers);
  }
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

int srj_plan_gs(srj_plan *plan, double *u, double omega, int64_t nsweeps, double *d_norms,
                void *stream) {
  if (!plan || !u || (nsweeps > 0 && !d_norms)) return fail(SRJ_EINVAL, "null argument");
  if (nsweeps < 0) return fail(SRJ_EINVAL, "negative sweep count");
  if (nsweeps == 0) return SRJ_OK;
  const srj_plan_desc &d = plan->d;
  const srj_layout_t &l = d.layout;
  if (d.kappa) return fail(SRJ_EUNSUPPORTED, "Gauss-Seidel has no nonlinear source");
  if (!d.physical_lo0 || !d.physical_hi0 || d.own0_begin != 0 || d.own0_end != l.n[0])
    return fail(SRJ_EUNSUPPORTED, "Gauss-Seidel needs the whole grid on one plan");
  if (l.ndim == 3 && l.n[1] < 2)
    return fail(SRJ_EUNSUPPORTED, "3-D Gauss-Seidel needs n[1] >= 2");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ioff = interior_offset(l);
  const bool var = d.coef_mode == 1;
  GSParams p{};
  p.u = u + ioff;
  p.f = d.source + ioff;
  p.act = d.act ? d.act + ioff : nullptr;
  for (int a = 0; a < 7; ++a) {
    p.coef[a] = (var && a < 1 + 2 * l.ndim) ? d.coef_arrays[a] + ioff : nullptr;
    p.kc[a] = d.coef[a];
  }
  p.kinv = var ? 0.0 : recip_or_zero(d.coef[0]);
  p.kinv_lo = recip_lo(d.coef[0], p.kinv);
  p.pitch = l.pitch;
  p.plane = l.plane;
  p.n1 = l.ndim == 3 ? int(l.n[1]) : 0;
  p.nrows = l.ndim == 3 ? l.n[0] * l.n[1] : l.n[0];
  p.ncols = int(l.n[l.ndim - 1]);
  const int nstrips = int((p.nrows + 31) / 32);
  p.nstrips = nstrips;
  p.omega = omega;
  if (nstrips > plan->gs_prog_cap) {
    if (plan->gs_prog) {
      cudaDeviceSynchronize();
      scratch_free(plan->gs_prog);
    }
    plan->gs_prog = nullptr;
    plan->gs_prog_cap = 0;
    SRJ_CUDA(scratch_alloc(&plan->gs_prog, sizeof(unsigned long long) * size_t(nstrips)));
    plan->gs_prog_cap = nstrips;
  }
  p.prog = plan->gs_prog;
  SRJ_CUDA(cudaMemsetAsync(d_norms, 0, sizeof(double) * 2 * size_t(nsweeps), st));
  const bool recip = !var && p.kinv != 0.0;
  // non-FIXED faces / copy hooks: the reference refreshes ghosts after every
  // sweep (_Sweeper.gauss_seidel, grids.py:561-571) -> one sweep per launch
  const bool per_sweep = plan->has_bc || plan->g_n > 0;
  const int64_t chunk = per_sweep ? 1 : (int64_t(1) << 20);
  for (int64_t k = 0; k < nsweeps; k += chunk) {
    p.nsweeps = int(std::min<int64_t>(chunk, nsweeps - k));
    p.norms = d_norms + 2 * k;
    SRJ_CUDA(cudaMemsetAsync(plan->gs_prog, 0, sizeof(unsigned long long) * size_t(nstrips), st));
    const int rc = launch_gs(p, l.ndim, var, recip, nstrips, st);
    if (rc != SRJ_OK) return rc;
    if (plan->has_bc) {
      const int rg = launch_ghosts(d, u + ioff, st);
      if (rg != SRJ_OK) return rg;
    }
    if (plan->g_n > 0) {
      const int rg = launch_gather(*plan, u, st);
      if (rg != SRJ_OK) return rg;
    }
  }
  return SRJ_OK;
}

int srj_upload_field(const srj_layout_t *lay, const double *host, double *dev, void *stream) {
  if (!lay || !host || !dev) return fail(SRJ_EINVAL, "null argument");
  const srj_layout_t &l = *lay;
  const int64_t last = l.n[l.ndim - 1] + 2;
  const int64_t rows = (l.ndim == 3) ? (l.n[0] + 2) * (l.n[1] + 2) : (l.n[0] + 2);
  double *dst = dev + l.origin + int64_t(l.halo0 - 1) * l.plane;
  SRJ_CUDA(cudaMemcpy2DAsync(dst, l.pitch * 8, host, last * 8, last * 8, rows,
                             cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  return SRJ_OK;
}

int srj_download_field(const srj_layout_t *lay, const double *dev, double *host, void *stream) {
  if (!lay || !host || !dev) return fail(SRJ_EINVAL, "null argument");
  const srj_layout_t &l = *lay;
  const int64_t last = l.n[l.ndim - 1] + 2;
  const int64_t rows = (l.ndim == 3) ? (l.n[0] + 2) * (l.n[1] + 2) : (l.n[0] + 2);
  const double *src = dev + l.origin + int64_t(l.halo0 - 1) * l.plane;
  SRJ_CUDA(cudaMemcpy2DAsync(host, last * 8, src, l.pitch * 8, last * 8, rows,
                             cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  return SRJ_OK;
}

int srj_upload_interior(const srj_layout_t *lay, const void *host, void *dev, int32_t elem_size,
                        void *stream) {
  if (!lay || !host || !dev) return fail(SRJ_EINVAL, "null argument");
  if (elem_size != 1 && elem_size != 8) return fail(SRJ_EINVAL, "elem_size must be 1 or 8");
  const srj_layout_t &l = *lay;
  const int64_t e = elem_size;
  const int64_t ioff = interior_offset(l);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char *h = static_cast<const char *>(host);
  char *dv = static_cast<char *>(dev);
  if (l.ndim == 2) {
    SRJ_CUDA(cudaMemcpy2DAsync(dv + ioff * e, l.pitch * e, h, l.n[1] * e, l.n[1] * e, l.n[0],
                               cudaMemcpyHostToDevice, st));
  } else {
    const int64_t layer = l.n[1] * l.n[2] * e;
    for (int64_t i = 0; i < l.n[0]; ++i)
      SRJ_CUDA(cudaMemcpy2DAsync(dv + (ioff + i * l.plane) * e, l.pitch * e, h + i * layer,
                                 l.n[2] * e, l.n[2] * e, l.n[1], cudaMemcpyHostToDevice, st));
  }
  return SRJ_OK;
}

int srj_copy_layers(const srj_layout_t *lay, const double *src, int64_t src_layer, double *dst,
                    int64_t dst_layer, int64_t count, void *stream) {
  if (!lay || !src || !dst) return fail(SRJ_EINVAL, "null argument");
  const srj_layout_t &l = *lay;
  if (count < 0 || src_layer < 0 || dst_layer < 0 || src_layer + count > l.rows0 ||
      dst_layer + count > l.rows0)
    return fail(SRJ_EINVAL, "layer range out of bounds");
  if (count == 0) return SRJ_OK;
  SRJ_CUDA(cudaMemcpyAsync(dst + l.origin + dst_layer * l.plane, src + l.origin + src_layer * l.plane,
                           sizeof(double) * size_t(count * l.plane), cudaMemcpyDefault,
                           static_cast<cudaStream_t>(stream)));
  return SRJ_OK;
}

/* ------------------------------------------------------------ slab API */

int srj_slab_create(const srj_plan_desc *desc, int32_t halo, double *const *bufs, uint32_t *flags,
                    int32_t has_lo, int32_t has_hi, srj_slab **out) {
  if (!desc || !bufs || !flags || !out) return fail(SRJ_EINVAL, "null argument");
  if (!bufs[0] || !bufs[1] || !bufs[2]) return fail(SRJ_EINVAL, "null field buffer");
  if (halo < 1 || halo > kMaxFuse) return fail(SRJ_EINVAL, "halo must be in [1, %d]", kMaxFuse);
  if (!driver_ops().ok) return fail(SRJ_EUNSUPPORTED, "CUDA stream memory operations unavailable");
  srj_plan *plan = nullptr;
  int rc = srj_plan_create(desc, &plan);
  if (rc != SRJ_OK) return rc;
  if (plan->has_bc || plan->g_n > 0) {
    srj_plan_destroy(plan);
    return fail(SRJ_EUNSUPPORTED, "slab decomposition supports FIXED faces only");
  }
  const int64_t ob = plan->d.own0_begin, oe = plan->d.own0_end;
  const int64_t n0 = plan->d.layout.n[0];
  if ((has_lo && ob < halo) || (has_hi && n0 - oe < halo) || oe - ob < halo) {
    srj_plan_destroy(plan);
    return fail(SRJ_EINVAL, "owned rows [%lld, %lld) of %lld leave no room for %d halo rows",
                (long long)ob, (long long)oe, (long long)n0, halo);
  }
  srj_slab *sl = new (std::nothrow) srj_slab;
  if (!sl) {
    srj_plan_destroy(plan);
    return fail(SRJ_ENOMEM, "host allocation failed");
  }
  sl->plan = plan;
  for (int i = 0; i < 3; ++i) sl->bufs[i] = bufs[i];
  sl->flags = flags;
  sl->halo = halo;
  sl->has[0] = has_lo != 0;
  sl->has[1] = has_hi != 0;
  sl->device = current_device();
  const int64_t a = ob + (sl->has[0] ? halo : 0), b = oe - (sl->has[1] ? halo : 0);
  if (a >= b) {  // thin slab: one edge launch covers every owned row
    sl->part_b[0] = ob;
    sl->part_e[0] = oe;
    sl->part_b[1] = sl->part_e[1] = sl->part_b[2] = sl->part_e[2] = 0;
  } else {
    sl->part_b[0] = ob;
    sl->part_e[0] = a;
    sl->part_b[1] = b;
    sl->part_e[1] = oe;
    sl->part_b[2] = a;
    sl->part_e[2] = b;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&sl->comm, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sl->edge, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl->ev_edge, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl->ev_copy, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl->ev_inner, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    srj_slab_destroy(sl);
    return cuda_fail(e, "slab stream/event creation");
  }
  *out = sl;
  return SRJ_OK;
}

int srj_slab_connect(srj_slab *sl, int32_t side, const srj_slab_peer *peer) {
  if (!sl || !peer || side < 0 || side > 1) return fail(SRJ_EINVAL, "bad argument");
  if (!sl->has[side]) return fail(SRJ_EINVAL, "this slab has no neighbour on side %d", side);
  if (!peer->bufs[0] || !peer->bufs[1] || !peer->bufs[2] || !peer->flags)
    return fail(SRJ_EINVAL, "null peer pointer");
  if (peer->dst_row < 0) return fail(SRJ_EINVAL, "negative peer row");
  sl->peer[side] = *peer;
  return SRJ_OK;
}

int srj_slab_reset(srj_slab *sl, void *stream) {
  if (!sl) return fail(SRJ_EINVAL, "null slab");
  SRJ_CUDA(cudaMemsetAsync(sl->flags, 0, sizeof(uint32_t) * SRJ_SLAB_FLAG_WORDS,
                           static_cast<cudaStream_t>(stream)));
  sl->epoch = 0;
  return SRJ_OK;
}

int srj_slab_destroy(srj_slab *sl) {
  if (!sl) return SRJ_OK;
  if (sl->comm) cudaStreamDestroy(sl->comm);
  if (sl->edge) cudaStreamDestroy(sl->edge);
  if (sl->ev_edge) cudaEventDestroy(sl->ev_edge);
  if (sl->ev_copy) cudaEventDestroy(sl->ev_copy);
  if (sl->ev_inner) cudaEventDestroy(sl->ev_inner);
  if (sl->plan) srj_plan_destroy(sl->plan);
  delete sl;
  return SRJ_OK;
}

srj_plan *srj_slab_plan(srj_slab *sl) { return sl ? sl->plan : nullptr; }

int srj_slab_depth(srj_slab *sl, int32_t fuse) {
  if (!sl) return fail(SRJ_EINVAL, "null slab");
  return std::min(plan_depth(*sl->plan, fuse), sl->halo);
}

int srj_slab_direct(srj_slab *sl, int32_t fuse) {
  if (!sl) return fail(SRJ_EINVAL, "null slab");
  const int T = std::min(plan_depth(*sl->plan, fuse), sl->halo);
  return (slab_direct_enabled() && direct_send_ok(*sl->plan, T)) ? 1 : 0;
}

int srj_slab_run(srj_slab *const *slabs, int32_t n, int32_t src, const double *weights, int64_t m,
                 int64_t first, int64_t nsteps, int32_t fuse, double *const *d_norms,
                 int32_t *final_buf, void *const *streams) {
  if (!slabs || n < 1 || !weights || !d_norms || !final_buf || !streams)
    return fail(SRJ_EINVAL, "null argument");
  if (src < 0 || src > 2) return fail(SRJ_EINVAL, "src must be buffer 0, 1 or 2");
  if (m < 1) return fail(SRJ_EINVAL, "weight cycle must be non-empty");
  if (nsteps < 0 || first < 0) return fail(SRJ_EINVAL, "negative step range");
  *final_buf = src;
  if (nsteps == 0) return SRJ_OK;
  // several slabs in one call (ranks emulated on one device) that share one
  // stream: everything is enqueued on it in dependency order, so every flag
  // wait is already satisfied when the stream reaches it.  Slabs with
  // distinct streams run exactly as separate ranks do (own stream + comm
  // stream each, ordered only by the flag words).
  bool serial = n > 1;
  for (int i = 1; i < n; ++i)
    if (streams[i] != streams[0]) serial = false;
  int T = kMaxFuse;
  for (int i = 0; i < n; ++i) {
    srj_slab *sl = slabs[i];
    if (!sl) return fail(SRJ_EINVAL, "null slab %d", i);
    for (int sd = 0; sd < 2; ++sd)
      if (sl->has[sd] && !sl->peer[sd].flags) return fail(SRJ_EINVAL, "slab %d is not connected", i);
    T = std::min(T, plan_depth(*sl->plan, fuse));
    if (T > sl->halo) T = sl->halo;
    SRJ_CUDA(cudaMemsetAsync(d_norms[i], 0, sizeof(double) * 2 * size_t(nsteps),
                             static_cast<cudaStream_t>(streams[serial ? 0 : i])));
  }
  const int others[3][2] = {{1, 2}, {0, 2}, {0, 1}};
  // Direct mode (default where every launch of the run supports it): ONE
  // launch per fused step over all owned rows; the sweep kernel stores the
  // edge rows into the neighbours' halo rows of the destination buffer as it
  // produces them (PeerSend, peer memory over NVLink), and two flag writes
  // follow the kernel.  Per launch: wait "halo of my source delivered" and
  // "neighbour finished the launch that read the buffer I write into", the
  // kernel, then "my rows arrived" + "I finished this launch".
  bool direct = slab_direct_enabled();
  for (int i = 0; i < n; ++i) direct = direct && direct_send_ok(*slabs[i]->plan, T);
  if (direct) {
    int cur = src, flip = 0;
    // flag operations pending per slab: the writes that follow launch j travel
    // in one batch with the waits that precede launch j+1
    std::vector<FlagOps> pend(static_cast<size_t>(n));
    for (int64_t k = 0; k < nsteps;) {
      const int t = int(std::min<int64_t>(T, nsteps - k));
      const int dst = others[src][flip];
      double om[kMaxFuse];
      for (int q = 0; q < t; ++q) om[q] = weights[(first + k + q) % m];
      for (int i = 0; i < n; ++i) {
        srj_slab *sl = slabs[i];
        cudaStream_t st = static_cast<cudaStream_t>(streams[serial ? 0 : i]);
        const srj_plan_desc &d = sl->plan->d;
        const int64_t ioff = interior_offset(d.layout);
        FlagOps &ops = pend[size_t(i)];
        PeerSend ps;
        for (int sd = 0; sd < 2; ++sd) {
          if (!sl->has[sd]) continue;
          ops.wait_pair(sl->flags + 2 * sd, sl->epoch);
          const srj_slab_peer &pr = sl->peer[sd];
          if (sd == 0) {
            ps.lo = pr.bufs[dst] + ioff;
            ps.lo_end = int(d.own0_begin) + sl->halo;
            ps.lo_shift = int(pr.dst_row - d.own0_begin);
          } else {
            ps.hi = pr.bufs[dst] + ioff;
            ps.hi_beg = int(d.own0_end) - sl->halo;
            ps.hi_shift = int(pr.dst_row - (d.own0_end - sl->halo));
          }
        }
        int rc = ops.flush(st);
        if (rc != SRJ_OK) return rc;
        rc = launch_fused(*sl->plan, d.own0_begin, d.own0_end, sl->bufs[cur], sl->bufs[dst], om, t,
                          d_norms[i] + 2 * k, st, (sl->has[0] || sl->has[1]) ? &ps : nullptr);
        if (rc != SRJ_OK) return rc;
        for (int sd = 0; sd < 2; ++sd) {
          if (!sl->has[sd]) continue;
          // the neighbour sees this rank on its opposite side
          ops.write_pair(sl->peer[sd].flags + 2 * (1 - sd), sl->epoch + 1);
        }
        // Ranks emulated in one process (n > 1) flush at once: the next slab's
        // waits need these writes ahead of them, on one shared stream and
        // also on distinct streams, which may share a hardware queue (a wait
        // at its head would block the write behind it for ever -- caught by
        // tests/test_gpu_slab_streams.py).  A real rank (n == 1) has only its
        // own operations on the device.
        if (n > 1 || k + t >= nsteps) {
          rc = ops.flush(st);
          if (rc != SRJ_OK) return rc;
        }
        sl->epoch += 1;
      }
      k += t;
      cur = dst;
      flip ^= 1;
    }
    *final_buf = cur;
    return SRJ_OK;
  }
  // A rank with neighbours (not serial) runs on three streams: its edge-row
  // launches on sl->edge, the peer copies on sl->comm and the inner-row
  // launches on the caller's stream.  The inner rows of launch j read no halo
  // row, so they run concurrently with launch j's edge rows; the two streams
  // meet once per launch (each waits for the other's previous launch, whose
  // rows its dependency cone reads and whose source rows it overwrites).
  // (SRJ_SLAB_SPLIT=0: edge and inner rows back to back on one stream.)
  const bool split_on = slab_split_enabled();
  auto split = [&](const srj_slab *sl) {
    return split_on && !serial && (sl->has[0] || sl->has[1]);
  };
  for (int i = 0; i < n; ++i) {
    srj_slab *sl = slabs[i];
    if (!split(sl)) continue;
    // the edge stream starts after everything queued on the caller's stream
    // (the norm memset above, the previous chunk, uploads)
    cudaStream_t st = static_cast<cudaStream_t>(streams[i]);
    SRJ_CUDA(cudaEventRecord(sl->ev_inner, st));
    SRJ_CUDA(cudaStreamWaitEvent(sl->edge, sl->ev_inner, 0));
  }
  int cur = src, flip = 0;
  int64_t k = 0;
  while (k < nsteps) {
    const int t = int(std::min<int64_t>(T, nsteps - k));
    const int dst = others[src][flip];
    double om[kMaxFuse];
    for (int q = 0; q < t; ++q) om[q] = weights[(first + k + q) % m];
    // phase A: halo of `cur` delivered (previous launch) -> edge rows
    for (int i = 0; i < n; ++i) {
      srj_slab *sl = slabs[i];
      cudaStream_t st = static_cast<cudaStream_t>(streams[serial ? 0 : i]);
      cudaStream_t es = split(sl) ? sl->edge : st;
      FlagOps ops;
      for (int sd = 0; sd < 2; ++sd)
        if (sl->has[sd]) ops.wait(sl->flags + kFlagArrived + 2 * sd, sl->epoch);
      int rc = ops.flush(es);
      if (rc != SRJ_OK) return rc;
      if (split(sl) && k > 0) {
        // the previous launch's inner rows (read by this cone, and the last
        // readers of the rows written now) and its peer copy (reads the
        // buffer the launch after this one overwrites)
        SRJ_CUDA(cudaStreamWaitEvent(es, sl->ev_inner, 0));
        SRJ_CUDA(cudaStreamWaitEvent(es, sl->ev_copy, 0));
      }
      for (int part = 0; part < 2; ++part)
        if (sl->part_e[part] > sl->part_b[part]) {
          rc = launch_fused(*sl->plan, sl->part_b[part], sl->part_e[part], sl->bufs[cur],
                            sl->bufs[dst], om, t, d_norms[i] + 2 * k, es);
          if (rc != SRJ_OK) return rc;
        }
      if (!serial) SRJ_CUDA(cudaEventRecord(sl->ev_edge, es));
    }
    // phase B: send the edge rows into the neighbours' halo rows of `dst`
    // once they finished every launch that read that buffer
    for (int i = 0; i < n; ++i) {
      srj_slab *sl = slabs[i];
      if (!sl->has[0] && !sl->has[1]) continue;
      cudaStream_t cs = serial ? static_cast<cudaStream_t>(streams[0]) : sl->comm;
      if (!serial) SRJ_CUDA(cudaStreamWaitEvent(cs, sl->ev_edge, 0));
      const srj_layout_t &l = sl->plan->d.layout;
      FlagOps ops;
      for (int sd = 0; sd < 2; ++sd)
        if (sl->has[sd]) ops.wait(sl->flags + kFlagDone + 2 * sd, sl->epoch);
      int rc = ops.flush(cs);
      if (rc != SRJ_OK) return rc;
      for (int sd = 0; sd < 2; ++sd) {
        if (!sl->has[sd]) continue;
        const srj_slab_peer &pr = sl->peer[sd];
        const int64_t row = sd == 0 ? sl->plan->d.own0_begin : sl->plan->d.own0_end - sl->halo;
        SRJ_CUDA(cudaMemcpyAsync(pr.bufs[dst] + layer_offset(l, pr.dst_row),
                                 sl->bufs[dst] + layer_offset(l, row),
                                 sizeof(double) * size_t(sl->halo * l.plane), cudaMemcpyDefault, cs));
        // the neighbour sees this rank on its opposite side
        ops.write(pr.flags + kFlagArrived + 2 * (1 - sd), sl->epoch + 1);
      }
      rc = ops.flush(cs);
      if (rc != SRJ_OK) return rc;
      if (!serial) SRJ_CUDA(cudaEventRecord(sl->ev_copy, cs));
    }
    // phase C: inner rows (concurrent with this launch's edge rows and
    // their transfer); then tell the neighbours this launch (and its reads
    // of `cur`) is complete
    for (int i = 0; i < n; ++i) {
      srj_slab *sl = slabs[i];
      cudaStream_t st = static_cast<cudaStream_t>(streams[serial ? 0 : i]);
      // first launch of a call: one-time set-up inside launch_fused (e.g. the
      // reciprocal arrays of the fused per-cell kernel) is queued on the edge
      // stream, so the inner rows follow it
      if (split(sl) && k == 0) SRJ_CUDA(cudaStreamWaitEvent(st, sl->ev_edge, 0));
      if (sl->part_e[2] > sl->part_b[2]) {
        const int rc = launch_fused(*sl->plan, sl->part_b[2], sl->part_e[2], sl->bufs[cur],
                                    sl->bufs[dst], om, t, d_norms[i] + 2 * k, st);
        if (rc != SRJ_OK) return rc;
      }
      if (split(sl)) {
        SRJ_CUDA(cudaEventRecord(sl->ev_inner, st));
        SRJ_CUDA(cudaStreamWaitEvent(st, sl->ev_edge, 0));  // launch complete = both parts
      }
      FlagOps ops;
      for (int sd = 0; sd < 2; ++sd)
        if (sl->has[sd]) ops.write(sl->peer[sd].flags + kFlagDone + 2 * (1 - sd), sl->epoch + 1);
      const int rc = ops.flush(st);
      if (rc != SRJ_OK) return rc;
      // one stream for both parts: the next launches overwrite rows the
      // copy of this one reads
      if (!serial && !split(sl) && (sl->has[0] || sl->has[1]))
        SRJ_CUDA(cudaStreamWaitEvent(st, sl->ev_copy, 0));
      sl->epoch += 1;
    }
    k += t;
    cur = dst;
    flip ^= 1;
  }
  // the caller's stream ends behind the last peer copy: whatever it runs next
  // (the norm all-reduce, which every rank joins only after this point, a
  // residual pass, the next chunk) sees every halo row delivered by THIS rank
  for (int i = 0; i < n; ++i)
    if (split(slabs[i]))
      SRJ_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[i]), slabs[i]->ev_copy, 0));
  *final_buf = cur;
  return SRJ_OK;
}

/* IPC: export a device allocation to another process of the same node */
int srj_ipc_get_handle(const void *dev_ptr, void *handle, int64_t *offset) {
  if (!dev_ptr || !handle || !offset) return fail(SRJ_EINVAL, "null argument");
  if (!driver_ops().ok) return fail(SRJ_EUNSUPPORTED, "CUDA driver entry points unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  const CUresult r = driver_ops().addr_range(&base, &size, CUdeviceptr(dev_ptr));
  if (r != CUDA_SUCCESS) return fail(SRJ_ECUDA, "cuMemGetAddressRange failed (%d)", int(r));
  cudaIpcMemHandle_t h;
  SRJ_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
  std::memcpy(handle, &h, sizeof(h));
  *offset = int64_t(CUdeviceptr(dev_ptr) - base);
  return SRJ_OK;
}

int srj_ipc_open(const void *handle, int64_t offset, void **dev_ptr) {
  if (!handle || !dev_ptr || offset < 0) return fail(SRJ_EINVAL, "bad argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void *base = nullptr;
  SRJ_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = static_cast<char *>(base) + offset;
  return SRJ_OK;
}

int srj_ipc_close(void *base) {
  if (!base) return fail(SRJ_EINVAL, "null argument");
  SRJ_CUDA(cudaIpcCloseMemHandle(base));
  return SRJ_OK;
}

}  // extern "C"
