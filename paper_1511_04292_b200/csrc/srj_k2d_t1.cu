// Instantiates the 2D band kernel for fused depth(s) 1 (see srj_k2d_impl.cuh).
#include "srj_k2d_impl.cuh"

namespace srj_host {
template Kernel2D pick2d_t<1>(bool, bool, bool, int, bool);
}  // namespace srj_host
