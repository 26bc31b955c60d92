// srj_kvar.cu -- launcher of the fused (T = 2) per-cell-coefficient 2D kernel
// (srj_sweep2d_vtb.cuh).
#include "srj_host.cuh"

namespace srj_host {

template <bool NL, bool MASK>
static int vtb_bps() {
  static std::atomic<int> cache[kMaxDevices];
  return cached_per_device(cache, [] {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep2d_vtb<NL>, kWarps2DVTB * 32,
                                                  MASK ? kVTBSmemMask : kVTBSmem);
    return n > 0 ? n : 1;
  });
}

int launch_var2d_tb(VarTB2DParams p, bool nl, cudaStream_t st) {
  const int rows = p.own_e - p.own_b;
  p.nbands = (p.n1 + kVTBOwn - 1) / kVTBOwn;  // owned columns cover [0, n1)
  const bool mask = p.act != nullptr;
  const int bps = nl ? (mask ? vtb_bps<true, true>() : vtb_bps<true, false>())
                     : (mask ? vtb_bps<false, true>() : vtb_bps<false, false>());
  const long capacity = long(sm_count()) * bps * kWarps2DVTB;
  const size_t smem = mask ? kVTBSmemMask : kVTBSmem;
  // strips: best fill of whole waves, discounting the 3 fill ticks per strip
  int nstrips = 1;
  double best = -1.0;
  for (int ns = 1; ns <= std::max(1, std::min(256, rows / 8)); ++ns) {
    const long w = long(p.nbands) * ns;
    const long waves = (w + capacity - 1) / capacity;
    const double hh = double(rows) / ns;
    const double eff = double(w) / double(waves * capacity) * hh / (hh + 3.0);
    if (eff > best + 1e-9) {
      best = eff;
      nstrips = ns;
    }
  }
  p.H = (rows + nstrips - 1) / nstrips;
  p.nstrips = (rows + p.H - 1) / p.H;
  const long warps = long(p.nbands) * p.nstrips;
  const int blocks = int((warps + kWarps2DVTB - 1) / kWarps2DVTB);
  if (nl)
    sweep2d_vtb<true><<<blocks, kWarps2DVTB * 32, smem, st>>>(p);
  else
    sweep2d_vtb<false><<<blocks, kWarps2DVTB * 32, smem, st>>>(p);
  SRJ_CUDA(cudaGetLastError());
  return SRJ_OK;
}

}  // namespace srj_host
