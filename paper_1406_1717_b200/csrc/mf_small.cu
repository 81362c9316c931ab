// mf_small.cu -- instantiations and launcher of the fused small-k kernel.
#include <algorithm>

#include "mf_launch.h"
#include "mf_small.cuh"

namespace mf {

namespace {
template <int DT, int K>
cudaError_t launch_k(const Geom& g, cudaStream_t s) {
  constexpr int kSmallThreads = SmallShape<DT, K>::T;
  using C = SmallCfg<DT, K, kSmallThreads>;
  auto kern = mf_small_kernel<DT, K, kSmallThreads>;
  static int resident = 0;  // CTAs per SM (per process; the attribute is idempotent)
  static int sms = 0;
  if (!resident) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, kSmallThreads, C::smem);
    if (e != cudaSuccess) return e;
    if (resident < 1) resident = 1;
  }
  const uint64_t tiles_per_row = (g.units + C::TU - 1) / C::TU;
  const uint64_t total = tiles_per_row * g.rows;
  // persistent grid: each CTA streams a contiguous range of tiles with a prefetch
  const uint64_t ctas = std::min<uint64_t>(total, (uint64_t)sms * resident);
  kern<<<(unsigned)ctas, kSmallThreads, C::smem, s>>>(g, tiles_per_row, total);
  return cudaGetLastError();
}

template <int DT>
cudaError_t launch_dt(const Geom& g, cudaStream_t s) {
  switch (g.k) {
#define MF_K(KK) case KK: return launch_k<DT, KK>(g, s);
    MF_K(1) MF_K(3) MF_K(5) MF_K(7) MF_K(9) MF_K(11) MF_K(13) MF_K(15)
    MF_K(17) MF_K(19) MF_K(21) MF_K(23) MF_K(25) MF_K(27) MF_K(29) MF_K(31)
#undef MF_K
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_small(int dt, const Geom& g, cudaStream_t s, uint64_t* launches) {
  cudaError_t e;
  switch (dt) {
    case DT_I32: e = launch_dt<DT_I32>(g, s); break;
    case DT_I64: e = launch_dt<DT_I64>(g, s); break;
    case DT_F32: e = launch_dt<DT_F32>(g, s); break;
    case DT_F64: e = launch_dt<DT_F64>(g, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace mf
