// Instantiates the 2D band kernel for fused depth(s) 5, 6, 7, 8 (see srj_k2d_impl.cuh).
#include "srj_k2d_impl.cuh"

namespace srj_host {
template Kernel2D pick2d_t<5>(bool, bool, bool, int, bool);
template Kernel2D pick2d_t<6>(bool, bool, bool, int, bool);
template Kernel2D pick2d_t<7>(bool, bool, bool, int, bool);
template Kernel2D pick2d_t<8>(bool, bool, bool, int, bool);
}  // namespace srj_host
