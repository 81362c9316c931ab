// mf_small63.cu -- the small-k kernel's 33 <= k <= 63 instantiations (32-bit keys, 64-bit
// live masks), in their own translation unit so they compile in parallel with mf_small.cu.
#include "mf_launch.h"
#include "mf_small.cuh"

namespace mf {

namespace {
template <int DT>
cudaError_t launch_dt63(const Geom& g, cudaStream_t s) {
  switch (g.k) {
#define MF_K(KK) case KK: return small_launch_k<DT, KK>(g, s);
    MF_K(33) MF_K(35) MF_K(37) MF_K(39) MF_K(41) MF_K(43) MF_K(45) MF_K(47)
    MF_K(49) MF_K(51) MF_K(53)
#if MF_SMALL_MAXK32 > 53
    MF_K(55) MF_K(57) MF_K(59) MF_K(61) MF_K(63)
#endif
#undef MF_K
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_small_k63(int dt, const Geom& g, cudaStream_t s) {
  switch (dt) {
    case DT_I32: return launch_dt63<DT_I32>(g, s);
    case DT_F32: return launch_dt63<DT_F32>(g, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mf
