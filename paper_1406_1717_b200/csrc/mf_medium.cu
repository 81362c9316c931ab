// mf_medium.cu -- instantiations and launcher of the fused medium-k kernel.
#include <algorithm>
#include "mf_launch.h"
#include "mf_medium.cuh"

namespace mf {

namespace {
// Warps per CTA by (R, key width): a few hundred CTA-resident pairs per SM at most;
// smaller R has a smaller footprint and gets more warps.
template <int DT, int R> struct WarpsFor {
  static constexpr bool wide = sizeof(typename Traits<DT>::U) == 8;
#ifndef MF_W_R16
#define MF_W_R16 4  // teams per CTA for R = 16 (8 teams: k = 511 1.20 ms with the payload sort; 4 with the key sort: 1.04 ms)
#endif
#ifndef MF_W_R8
#define MF_W_R8 4   // ... for R = 8 (4 teams x 8 CTAs/SM: k = 255 1.00 -> 0.985 ms)
#endif
#ifndef MF_W_R4
#define MF_W_R4 8   // ... for R <= 4
#endif
#ifndef MF_W_R32
#define MF_W_R32 2
#endif
#ifndef MF_W_R4_WIDE
#define MF_W_R4_WIDE 4  // ... for R <= 4 and 64-bit keys (config 1, f64 k = 101: 0.0646 -> 0.0600 ms)
#endif
#ifndef MF_W_R2
#define MF_W_R2 2  // ... for R = 2 and 32-bit keys, k = 49..63 (8 teams: k = 49 1.71 ms, 2 teams: 1.64 ms)
#endif
  static constexpr int value =
      R >= 32 ? MF_W_R32
              : (R >= 16 ? MF_W_R16 : R >= 8 ? MF_W_R8 : (wide ? MF_W_R4_WIDE : R == 2 ? MF_W_R2 : MF_W_R4));
};

template <int DT, int R>
cudaError_t launch_r(const Geom& g, cudaStream_t s) {
  constexpr int W = WarpsFor<DT, R>::value;
#ifndef MF_WP_R16
#define MF_WP_R16 1
#endif
#ifndef MF_WP_R8
#define MF_WP_R8 1
#endif
  // warps per block pair (team); k <= 511 measured faster with 1
  constexpr int WP = R >= 32 ? 2 : R == 16 ? MF_WP_R16 : R == 8 ? MF_WP_R8 : 1;
  using C = MediumCfg<DT, R, W, WP>;
  auto kern = mf_medium_kernel<DT, R, W, WP>;
  LaunchInfo li;
  cudaError_t e = kernel_setup((const void*)kern, C::smem, 32 * W * WP, &li);
  if (e != cudaSuccess) return e;
  const int sms = li.sms, resident = li.resident;
  const uint64_t tiles_per_row = (g.units + W - 1) / W;
  const uint64_t total = tiles_per_row * g.rows;
  // persistent grid: each CTA walks a contiguous range of tiles (ring-carried blocks)
  const uint64_t ctas = std::min<uint64_t>(total, (uint64_t)sms * resident);
  kern<<<(unsigned)ctas, 32 * W * WP, C::smem, s>>>(g, tiles_per_row, total);
  return cudaGetLastError();
}

template <int DT>
cudaError_t launch_dt(const Geom& g, cudaStream_t s) {
  if (g.k <= 64) return launch_r<DT, 2>(g, s);
  if (g.k <= 128) return launch_r<DT, 4>(g, s);
  if (g.k <= 256) return launch_r<DT, 8>(g, s);
  if (g.k <= 512) return launch_r<DT, 16>(g, s);
  if (g.k <= 1024) return launch_r<DT, 32>(g, s);
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_medium(int dt, const Geom& g, cudaStream_t s, uint64_t* launches) {
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
