// srj_k3d.cu -- instantiation table of the 3D kernels: the one-sweep
// streaming kernel (srj_sweep3d.cuh) and the temporally blocked CTA-tile
// kernel (srj_sweep3d_tb.cuh).
#include "srj_host.cuh"

namespace srj_host {

template <bool VAR, bool NL, bool RECIP, bool CLS = false, bool SEND = false>
struct K3 {
  static void launch(const Sweep3DParams &p, int blocks, cudaStream_t s) {
    sweep3d<VAR, NL, RECIP, CLS, SEND><<<blocks, kWarps3D * 32, 0, s>>>(p);
  }
  static int bps() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep3d<VAR, NL, RECIP, CLS, SEND>, kWarps3D * 32, 0);
      return n > 0 ? n : 1;
    });
  }
  static Kernel3D get() { return Kernel3D{launch, bps}; }
};


template <int T, bool NL, bool RECIP, int BCF = 0>
struct K3TB {
  using B = Tile3D<T>;
  static void configure() {
    static std::atomic<uint64_t> done{0};
    once_per_device(done, [] {
      cudaFuncSetAttribute(sweep3d_tb<T, NL, RECIP, BCF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(B::smem_bytes()));
    });
  }
  static void launch(const Sweep3DTBParams &p, const CUtensorMap &tu, const CUtensorMap &tf,
                     int blocks, cudaStream_t s) {
    configure();
    sweep3d_tb<T, NL, RECIP, BCF><<<blocks, B::THREADS, B::smem_bytes(), s>>>(p, tu, tf);
  }
  static int bps() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
      configure();
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep3d_tb<T, NL, RECIP, BCF>, B::THREADS,
                                                    B::smem_bytes());
      return n > 0 ? n : 1;
    });
  }
  static Kernel3DTB get() { return Kernel3DTB{launch, bps, B::TJ, B::TK, B::HS, B::HJ, B::HJ, false}; }
};

template <int T, int BCF>
Kernel3DTB pick3d_tb_bc(bool nl, bool recip) {
  if (recip) return nl ? K3TB<T, true, true, BCF>::get() : K3TB<T, false, true, BCF>::get();
  return nl ? K3TB<T, true, false, BCF>::get() : K3TB<T, false, false, BCF>::get();
}

// bcf: 0 = FIXED faces; 1 = fused MIRROR / FACE_DIRICHLET faces; 2 = MIRROR only
template <int T>
Kernel3DTB pick3d_tb_t(bool nl, bool recip, int bcf) {
  if (bcf == 1) return pick3d_tb_bc<T, 1>(nl, recip);
  if (bcf == 2) return pick3d_tb_bc<T, 2>(nl, recip);
  if (recip) return nl ? K3TB<T, true, true>::get() : K3TB<T, false, true>::get();
  return nl ? K3TB<T, true, false>::get() : K3TB<T, false, false>::get();
}

// register-streaming T = 2 kernel (srj_sweep3d_rs.cuh): FIXED faces
template <bool NL, bool RECIP, bool SEND = false>
struct K3RS {
  using B = RS3D;
  static void configure() {
    static std::atomic<uint64_t> done{0};
    once_per_device(done, [] {
      cudaFuncSetAttribute(sweep3d_rs<NL, RECIP, SEND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(B::smem_bytes()));
    });
  }
  static void launch(const Sweep3DTBParams &p, const CUtensorMap &tu, const CUtensorMap &tf,
                     int blocks, cudaStream_t s) {
    configure();
    sweep3d_rs<NL, RECIP, SEND><<<blocks, B::THREADS, B::smem_bytes(), s>>>(p, tu, tf);
  }
  static int bps() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
      configure();
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep3d_rs<NL, RECIP, SEND>, B::THREADS,
                                                    B::smem_bytes());
      return n > 0 ? n : 1;
    });
  }
  static Kernel3DTB get() {
    return Kernel3DTB{launch, bps, B::TJ, B::TK, B::UC, B::UR, B::FR, true};
  }
};

Kernel3DTB pick3d_tb(int T, bool nl, bool recip, int bcf, bool send) {
  if (send && T == 2 && bcf == 0 && !rs3d_disabled()) {
    if (recip) return nl ? K3RS<true, true, true>::get() : K3RS<false, true, true>::get();
    return nl ? K3RS<true, false, true>::get() : K3RS<false, false, true>::get();
  }
  if (T == 2 && bcf == 0 && !rs3d_disabled()) {
    if (recip) return nl ? K3RS<true, true>::get() : K3RS<false, true>::get();
    return nl ? K3RS<true, false>::get() : K3RS<false, false>::get();
  }
  switch (T) {
    case 2: return pick3d_tb_t<2>(nl, recip, bcf);
    default: return pick3d_tb_t<3>(nl, recip, bcf);
  }
}

Kernel3D pick3d(bool var, bool nl, bool recip, bool cls, bool send) {
  if (send && var && cls) return nl ? K3<true, true, false, true, true>::get() : K3<true, false, false, true, true>::get();
  if (send && var) return nl ? K3<true, true, false, false, true>::get() : K3<true, false, false, false, true>::get();
  if (send) {
    if (recip) return nl ? K3<false, true, true, false, true>::get() : K3<false, false, true, false, true>::get();
    return nl ? K3<false, true, false, false, true>::get() : K3<false, false, false, false, true>::get();
  }
  if (var && cls) return nl ? K3<true, true, false, true>::get() : K3<true, false, false, true>::get();
  if (var) return nl ? K3<true, true, false>::get() : K3<true, false, false>::get();
  if (recip) return nl ? K3<false, true, true>::get() : K3<false, false, true>::get();
  return nl ? K3<false, true, false>::get() : K3<false, false, false>::get();
}


}  // namespace srj_host
