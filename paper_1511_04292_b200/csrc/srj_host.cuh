// srj_host.cuh -- host-side helpers shared by the translation units of
// libsrj.so: error reporting (srj_last_error), per-device caches, and the
// dispatch tables of the kernel families.  The kernel instantiations live in
// separate .cu files (srj_k2d_t*.cu, srj_k3d.cu, srj_kgs.cu) so nvcc compiles
// them in parallel; srj_capi.cu holds the C ABI.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include "../../include/srj.h"
#include "srj_gs.cuh"
#include "srj_sweep2d.cuh"
#include "srj_sweep3d.cuh"
#include "srj_sweep3d_tb.cuh"
#include "srj_sweep3d_rs.cuh"
#include "srj_sweep2d_vtb.cuh"

namespace srj_host {
using namespace srj;

inline thread_local char g_err[512] = "";

inline int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

inline int cuda_fail(cudaError_t e, const char *what) {
  return fail(e == cudaErrorMemoryAllocation ? SRJ_ENOMEM : SRJ_ECUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define SRJ_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// Per-device caches: function attributes and occupancy belong to a device
// context, so one process may drive several GPUs (from several threads).
// Races only repeat idempotent work.
constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & (kMaxDevices - 1);
}

// Runs f() once per device for the given cache of flags.
template <typename F>
void once_per_device(std::atomic<uint64_t> &done, F &&f) {
  const uint64_t bit = uint64_t(1) << current_device();
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// Per-device integer cache filled by f() (0 = not yet computed).
template <typename F>
int cached_per_device(std::atomic<int> (&slot)[kMaxDevices], F &&f) {
  std::atomic<int> &v = slot[current_device()];
  int n = v.load(std::memory_order_acquire);
  if (n == 0) {
    n = f();
    v.store(n, std::memory_order_release);
  }
  return n;
}

// SRJ_RS3D=0: use the shared-memory tile kernel (sweep3d_tb) for T=2 too
inline bool rs3d_disabled() {
  static const bool off = [] {
    const char *e = getenv("SRJ_RS3D");
    return e && e[0] == '0';
  }();
  return off;
}

inline int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  return cached_per_device(cache, [] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
    return n > 0 ? n : 148;
  });
}


// ------------------------------------------------------------ 2D dispatch
constexpr int kMaxFuseBC = 4;  // 2D fused depth with MIRROR / FACE_DIRICHLET faces
constexpr int kMaxFuseSend = 4;  // 2D fused depth of the kernels with direct halo stores (PeerSend)

// One entry per kernel instantiation: launcher + resident blocks per SM
// (registers and shared memory both counted, from the occupancy API), so the
// launch can be sized to exactly one wave.
struct Kernel2D {
  void (*launch)(const Sweep2DParams &, const CUtensorMap &, const CUtensorMap &, int blocks,
                 cudaStream_t);
  int box_cols;
  int (*blocks_per_sm)();
  int own;  // columns owned per band
};

// one TU per depth group instantiates these (srj_k2d_t*.cu)
template <int T>
Kernel2D pick2d_t(bool var, bool nl, bool recip, int bcf, bool send);

// ------------------------------------------------------------ 3D dispatch
struct Kernel3D {
  void (*launch)(const Sweep3DParams &, int blocks, cudaStream_t);
  int (*blocks_per_sm)();
};

// temporally blocked 3D (constant stencil only)
constexpr int kMaxFuse3D = 3;  // T=4 tiles exceed shared memory

struct Kernel3DTB {
  void (*launch)(const Sweep3DTBParams &, const CUtensorMap &, const CUtensorMap &, int,
                 cudaStream_t);
  int (*blocks_per_sm)();
  int tj, tk, box_cols, box_rows;
  int f_box_rows;  // source box rows (sweep3d_rs loads fewer than for u)
  bool persistent; // sweep3d_rs: grid = resident CTAs, equal (tile, plane) shares
};

// send: the instantiation that stores slab edge planes into the neighbours'
// halos (PeerSend; constant stencil; T = 2: sweep3d_rs only)
Kernel3D pick3d(bool var, bool nl, bool recip, bool cls, bool send = false);  // srj_k3d.cu
Kernel3DTB pick3d_tb(int T, bool nl, bool recip, int bcf, bool send = false);  // srj_k3d.cu
// fused T = 2 per-cell-coefficient 2D sweep (srj_kvar.cu); sets H/nbands/nstrips
int launch_var2d_tb(VarTB2DParams p, bool nl, cudaStream_t st);
int launch_gs(const GSParams &p, int nd, bool var, bool recip, int nstrips, cudaStream_t st);  // srj_kgs.cu

}  // namespace srj_host
