// srj_kgs.cu -- Gauss-Seidel / SOR wavefront launchers (srj_gs.cuh).
#include "srj_host.cuh"

namespace srj_host {

// Gauss-Seidel / SOR wavefront (srj_gs.cuh): nsweeps in-place sweeps, one
// cooperative launch (every strip co-resident).  The deep operand ring
// (DEEP) is used when every strip fits at its occupancy, else the kPF=4 copy
template <int ND, bool VAR, bool RECIP, bool DEEP>
static int gs_per_sm() {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_sweep<ND, VAR, RECIP, DEEP>, 32, 0) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm;
}

template <int ND, bool VAR, bool RECIP, bool DEEP>
static int launch_gs_t(const GSParams &p, int nstrips, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nstrips);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, gs_sweep<ND, VAR, RECIP, DEEP>, p);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // clear the launch error so later checks do not see it
    return fail(SRJ_EUNSUPPORTED, "Gauss-Seidel wavefront needs %d co-resident strips of 32 rows; "
                "the grid has too many rows for one GPU (%d warps per SM x %d SMs)", nstrips,
                gs_per_sm<ND, VAR, RECIP, DEEP>(), sm_count());
  }
  SRJ_CUDA(e);
  return SRJ_OK;
}

template <int ND, bool VAR, bool RECIP>
static int launch_gs_pick(const GSParams &p, int nstrips, cudaStream_t st) {
  if constexpr (!VAR) {
    if (long(gs_per_sm<ND, VAR, RECIP, true>()) * sm_count() >= nstrips) {
      const int rc = launch_gs_t<ND, VAR, RECIP, true>(p, nstrips, st);
      if (rc != SRJ_EUNSUPPORTED) return rc;  // else retry with the shallow ring
    }
  }
  return launch_gs_t<ND, VAR, RECIP, false>(p, nstrips, st);
}

int launch_gs(const GSParams &p, int nd, bool var, bool recip, int nstrips, cudaStream_t st) {
  if (nd == 2) {
    if (var) return launch_gs_pick<2, true, false>(p, nstrips, st);
    return recip ? launch_gs_pick<2, false, true>(p, nstrips, st)
                 : launch_gs_pick<2, false, false>(p, nstrips, st);
  }
  if (var) return launch_gs_pick<3, true, false>(p, nstrips, st);
  return recip ? launch_gs_pick<3, false, true>(p, nstrips, st)
               : launch_gs_pick<3, false, false>(p, nstrips, st);
}


}  // namespace srj_host
