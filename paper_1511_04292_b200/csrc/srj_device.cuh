// srj_device.cuh -- device helpers shared by the SRJ sweep kernels (sm_100a).
//
// Arithmetic contract: bit-identical to the reference kernels _wj2/_wj3
// (pkg/src/srj/grids.py:351-408).  Every operation is an explicit
// round-to-nearest intrinsic, so ptxas can never contract a multiply-add into
// an FMA (the library is also built with -fmad=false as a second guard):
//     acc = c*u ; acc += am0*u[i-1] ; acc += ap0*u[i+1] ; acc += am1*u[j-1] ;
//     acc += ap1*u[j+1] [; acc += am2*u[k-1] ; acc += ap2*u[k+1]]
//     r = s - acc ; d = (omega*r)/c ; un = u + d
#pragma once
#include <cstdint>

namespace srj {

constexpr int kMaxFuse = 8;       // deepest temporal blocking supported
constexpr unsigned kFull = 0xffffffffu;

// Direct halo stores of a slab rank (srj_slab_run): the sweep kernel writes
// the axis-0 rows / planes it owns next to a neighbour rank ALSO into that
// neighbour's halo rows of the destination buffer -- peer memory over NVLink
// (CUDA IPC mapping) -- so the exchange is part of the sweep itself: no edge
// launches, no copies, one flag write after the kernel.  Rows [own_b, lo_end)
// land `lo_shift` rows away in `lo`, rows [hi_beg, own_e) `hi_shift` rows away
// in `hi` (both the neighbour buffers' interior origins, same pitch / plane).
// No neighbour: lo_end = INT_MIN / hi_beg = INT_MAX, so the tests never pass.
struct PeerSend {
  double *lo = nullptr, *hi = nullptr;
  int lo_end = -2147483647 - 1, hi_beg = 2147483647;
  int lo_shift = 0, hi_shift = 0;
};

// Nonlinear source s(psi) = kappa * psi^5, fixed order:
//   p2 = psi*psi ; p4 = p2*p2 ; s = kappa * (p4*psi)
__device__ __forceinline__ double nl_source(double kappa, double psi) {
  double p2 = __dmul_rn(psi, psi);
  double p4 = __dmul_rn(p2, p2);
  return __dmul_rn(kappa, __dmul_rn(p4, psi));
}

// 5-point residual in the reference association order (grids.py:361-367).
// _wj1 (grids.py:331-348): r = s - ((c*u + am0*u[i-1]) + ap0*u[i+1])
__device__ __forceinline__ double resid3(double s, double c, double uc, double am0, double um0,
                                         double ap0, double up0) {
  double acc = __dmul_rn(c, uc);
  acc = __dadd_rn(acc, __dmul_rn(am0, um0));
  acc = __dadd_rn(acc, __dmul_rn(ap0, up0));
  return __dsub_rn(s, acc);
}

__device__ __forceinline__ double resid5(double s, double c, double uc,
                                         double am0, double um, double ap0,
                                         double up, double am1, double uw,
                                         double ap1, double ue) {
  double acc = __dmul_rn(c, uc);
  acc = __dadd_rn(acc, __dmul_rn(am0, um));
  acc = __dadd_rn(acc, __dmul_rn(ap0, up));
  acc = __dadd_rn(acc, __dmul_rn(am1, uw));
  acc = __dadd_rn(acc, __dmul_rn(ap1, ue));
  return __dsub_rn(s, acc);
}

// 7-point residual (grids.py:391-399).
__device__ __forceinline__ double resid7(double s, double c, double uc,
                                         double am0, double um, double ap0,
                                         double up, double am1, double un_,
                                         double ap1, double us, double am2,
                                         double uw, double ap2, double ue) {
  double acc = __dmul_rn(c, uc);
  acc = __dadd_rn(acc, __dmul_rn(am0, um));
  acc = __dadd_rn(acc, __dmul_rn(ap0, up));
  acc = __dadd_rn(acc, __dmul_rn(am1, un_));
  acc = __dadd_rn(acc, __dmul_rn(ap1, us));
  acc = __dadd_rn(acc, __dmul_rn(am2, uw));
  acc = __dadd_rn(acc, __dmul_rn(ap2, ue));
  return __dsub_rn(s, acc);
}

// d = (omega*r)/c with IEEE round-to-nearest division (grids.py:368).
__device__ __forceinline__ double relax(double omega, double r, double c) {
  return __ddiv_rn(__dmul_rn(omega, r), c);
}

// "if abs(x) > m: m = abs(x)" -- NaN never enters (grids.py:370-373).
__device__ __forceinline__ void acc_max(double &m, double x) {
  double a = fabs(x);
  m = (a > m) ? a : m;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(kFull, v, o);
    v = (w > v) ? w : v;
  }
  return v;
}

// Max-combine of a non-negative, non-NaN double into global memory.  The bit
// patterns of non-negative doubles (incl. +inf) order like unsigned integers.
__device__ __forceinline__ void global_max(double *slot, double v) {
  if (v > 0.0)
    atomicMax(reinterpret_cast<unsigned long long *>(slot),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

// RN(a/c) for a fixed divisor c > 0 from a double-word reciprocal
// (yh = RN(1/c), yl = RN(1/c - yh), host-computed), branch-free, 4 FP64 ops.  The sign is copied from a, which is exact for
// c > 0 and restores IEEE's -0/c = -0.  Valid for a = +-0 and for normal a
// with exponent in [-899, 899] (no overflow/underflow in q, r); other inputs
// (subnormal, huge, inf, NaN) are flagged by recip_unsafe() and redone with
// the IEEE division after a warp vote (see stage2d).
__device__ __forceinline__ double div_recip(double a, double c, double yh, double yl) {
  // q0 = RN(a*yh + RN(a*yl)) with yh + yl = 1/c to ~2^-106 is faithful (within
  // 1 ulp of a/c); Markstein's theorem (yh within 1/2 ulp of 1/c, q0 faithful)
  // then makes the remainder exact and one correction correctly rounded.
  double q = __fma_rn(a, yh, __dmul_rn(a, yl));
  const double r = __fma_rn(-q, c, a);
  q = __fma_rn(r, yh, q);
  // hi = (q.hi & 0x7fffffff) | (a.hi & 0x80000000): one bitwise select (LOP3)
  int hi;
  asm("lop3.b32 %0, %1, 0x7fffffff, %2, 0xE2;" : "=r"(hi) : "r"(__double2hiint(q)),
      "r"(__double2hiint(a)));
  return __hiloint2double(hi, __double2loint(q));
}

__device__ __forceinline__ bool recip_unsafe(double a) {
  const unsigned hi = unsigned(__double2hiint(a)) & 0x7fffffffu;
  const unsigned e = hi >> 20;
  const bool zero = (hi | unsigned(__double2loint(a))) == 0u;
  return (e - 124u > 1798u) && !zero;  // exponent outside [-899, 899], nonzero
}

// Superset of recip_unsafe() in three integer ops (also flags a = 0): the
// per-tick votes use it, the fix-up passes apply the exact test.
__device__ __forceinline__ bool recip_maybe_unsafe(double a) {
  const unsigned h2 = unsigned(__double2hiint(a)) << 1;  // exponent on top, sign dropped
  return h2 - (124u << 21) > (1798u << 21) + ((1u << 21) - 1u);
}

// out of line: the IEEE division is the rare path and its inline expansion
// would triple the size of the unrolled fast loop
static __device__ __noinline__ double div_ieee(double a, double c) { return __ddiv_rn(a, c); }

// keep the entry of larger magnitude (signed); NaN never replaces m
__device__ __forceinline__ void acc_absmax(double &m, double x) {
  m = (fabs(x) > fabs(m)) ? x : m;
}

// ---------------------------------------------------------------- mbarrier /
// bulk-copy (TMA engine, non-tensor form) helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
          smem_addr(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src,
                                         uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];\n" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Blocking wait with a hard bound: a pipeline bug traps (launch error) instead
// of hanging the GPU.  try_wait already suspends in hardware between probes.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > (1u << 24)) __trap();
  }
}

}  // namespace srj
