// srj_k2d_impl.cuh -- instantiation table of the 2D band kernel
// (srj_sweep2d.cuh): one launcher per (T, VAR, NL, RECIP, BCF), included by
// the srj_k2d_t*.cu translation units, each instantiating some depths T.
#pragma once
#include "srj_host.cuh"

namespace srj_host {

template <int T, bool VAR, bool NL, bool RECIP, int BCF = 0, bool SEND = false>
struct K2 {
  static constexpr int V = 2;
  using B = Band2D<T, V>;
  static void configure() {
    static std::atomic<uint64_t> done{0};
    once_per_device(done, [] {
      cudaFuncSetAttribute(sweep2d_tb<T, V, VAR, NL, RECIP, BCF, SEND>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(B::smem_bytes()));
    });
  }
  static void launch(const Sweep2DParams &p, const CUtensorMap &tu, const CUtensorMap &tf,
                     int blocks, cudaStream_t s) {
    configure();
    sweep2d_tb<T, V, VAR, NL, RECIP, BCF, SEND><<<blocks, B::WARPS * 32, B::smem_bytes(), s>>>(p, tu, tf);
  }
  static int bps() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
      configure();
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep2d_tb<T, V, VAR, NL, RECIP, BCF, SEND>,
                                                    B::WARPS * 32, B::smem_bytes());
      return n > 0 ? n : 1;
    });
  }
  static Kernel2D get() { return Kernel2D{launch, B::BAND, bps, B::OWN}; }
};

template <int T, int BCF>
Kernel2D pick2d_bc(bool var, bool nl, bool recip) {
  if (var) return nl ? K2<T, true, true, false, BCF>::get() : K2<T, true, false, false, BCF>::get();
  if (recip) return nl ? K2<T, false, true, true, BCF>::get() : K2<T, false, false, true, BCF>::get();
  return nl ? K2<T, false, true, false, BCF>::get() : K2<T, false, false, false, BCF>::get();
}

// bcf: 0 = FIXED faces; 1 = fused MIRROR / FACE_DIRICHLET faces; 2 = the same
// with MIRROR-or-FIXED column faces (no face values in the edge-band path)
// send: the copy that stores slab edge rows into the neighbours' halos
// (constant stencil, FIXED faces, T <= kMaxFuseSend)
template <int T>
Kernel2D pick2d_t(bool var, bool nl, bool recip, int bcf, bool send) {
  if constexpr (T <= kMaxFuseSend) {
    if (send && !var && bcf == 0) {
      if (recip) return nl ? K2<T, false, true, true, 0, true>::get() : K2<T, false, false, true, 0, true>::get();
      return nl ? K2<T, false, true, false, 0, true>::get() : K2<T, false, false, false, 0, true>::get();
    }
  }
  if constexpr (T >= 2 && T <= kMaxFuseBC) {
    if (bcf == 1) return pick2d_bc<T, 1>(var, nl, recip);
    if (bcf == 2) return pick2d_bc<T, 2>(var, nl, recip);
  }
  if (var) return nl ? K2<T, true, true, false>::get() : K2<T, true, false, false>::get();
  if (recip) return nl ? K2<T, false, true, true>::get() : K2<T, false, false, true>::get();
  return nl ? K2<T, false, true, false>::get() : K2<T, false, false, false>::get();
}


}  // namespace srj_host
