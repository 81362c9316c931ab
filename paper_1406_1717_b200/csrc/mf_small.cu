// mf_small.cu -- instantiations and launcher of the fused small-k kernel.
#include <algorithm>
#include <cstring>

#include "mf_launch.h"
#include "mf_small.cuh"

namespace mf {

namespace {
template <int DT, int K>
cudaError_t launch_k(const Geom& g, cudaStream_t s) { return small_launch_k<DT, K>(g, s); }

// ---- k = 3: direct selection ------------------------------------------------------------
// With k = 3 the paper's blocks hold three samples and every window spans two blocks, so the
// sort + Figure-7 walk degenerate to one compare-exchange chain per output: the median of
// (x[i], x[i+1], x[i+2]) under the sample order is max(min(a, b), min(max(a, b), c)) on the
// signed keys below.  The result is the same sample the reference picks (equal
// keys are equal bit patterns, so tie-breaking cannot change the emitted value), at ~4 key
// ops per output, so the kernel streams at HBM speed.  A warp owns 32*Q 16-byte groups of
// consecutive outputs; its Q loads and Q stores are each one contiguous 512-byte run, and a
// group's two samples past its end come from the next lane by shuffle (for lane 31, from lane
// 0's next group, or from two samples lane 0 loads past the warp's run).
#ifndef MF_MED3
#define MF_MED3 1  // 0: k = 3 runs the generic small kernel
#endif
constexpr int kMed3Threads = 256;
#ifndef MF_MED3_CS
#define MF_MED3_CS 0  // 1: ld.global.cs / st.global.cs (streaming) for the vector loads and stores
#endif
#ifndef MF_MED3_Q
#define MF_MED3_Q 2  // 16-byte loads per thread and chunk (a warp's loads are contiguous)
#endif
#ifndef MF_MED3_CTAS
#define MF_MED3_CTAS 8  // CTAs per SM of the grid
#endif
constexpr int kMed3Q = MF_MED3_Q, kMed3CtasPerSm = MF_MED3_CTAS;

// Signed keys: an involution on the sample bits whose signed order is the sample order
// (floats map negative patterns through x ^ 0x7F..F; integers are their own
// key), so one shift + one LOP3 encodes and the same two decode.
template <int DT> struct SKey;
template <> struct SKey<DT_I32> {
  using S = int32_t;
  __device__ __forceinline__ static S f(int32_t v) { return v; }
  __device__ __forceinline__ static int32_t g(S s) { return s; }
};
template <> struct SKey<DT_I64> {
  using S = int64_t;
  __device__ __forceinline__ static S f(int64_t v) { return v; }
  __device__ __forceinline__ static int64_t g(S s) { return s; }
};
template <> struct SKey<DT_F32> {
  using S = int32_t;
  __device__ __forceinline__ static S f(uint32_t b) { const S s = (S)b; return s ^ ((s >> 31) & 0x7FFFFFFF); }
  __device__ __forceinline__ static uint32_t g(S s) { return (uint32_t)(s ^ ((s >> 31) & 0x7FFFFFFF)); }
};
template <> struct SKey<DT_F64> {
  using S = int64_t;
  __device__ __forceinline__ static S f(uint64_t b) {
    const S s = (S)b;
    return s ^ ((s >> 63) & 0x7FFFFFFFFFFFFFFFll);
  }
  __device__ __forceinline__ static uint64_t g(S s) { return (uint64_t)(s ^ ((s >> 63) & 0x7FFFFFFFFFFFFFFFll)); }
};

template <typename U>
__device__ __forceinline__ U med3(U a, U b, U c) {
  const U lo = a < b ? a : b, hi = a < b ? b : a;
  const U m = hi < c ? hi : c;
  return lo < m ? m : lo;
}

template <int DT>
__global__ void __launch_bounds__(kMed3Threads) mf_med3_kernel(Geom g, uint64_t cpr, bool vec) {
  using T = typename Traits<DT>::T;
  using K = SKey<DT>;
  using U = typename K::S;
  constexpr int E4 = 16 / sizeof(T), Q = kMed3Q;
  constexpr uint64_t WSPAN = 32ull * Q * E4, SPAN = WSPAN * (kMed3Threads / 32);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t row = blockIdx.y; row < g.rows; row += gridDim.y) {
    const T* x = reinterpret_cast<const T*>(g.x) + row * g.ld_x;
    T* y = reinterpret_cast<T*>(g.y) + row * g.ld_y;
    for (uint64_t c = blockIdx.x; c < cpr; c += gridDim.x) {
      const uint64_t wb = c * SPAN + warp * WSPAN;                 // warp-uniform
      if (wb >= g.keep) continue;
      if (vec && wb + WSPAN <= g.keep) {                           // then wb + WSPAN + 2 <= n
        uint4 q[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
#if MF_MED3_CS
          q[j] = __ldcs(reinterpret_cast<const uint4*>(x + wb) + j * 32 + lane);   // streamed once: evict first
#else
          q[j] = __ldg(reinterpret_cast<const uint4*>(x + wb) + j * 32 + lane);
#endif
        }
        T h0 = T(0), h1 = T(0);                                    // the two samples past the warp's run
        if (lane == 0) { h0 = __ldg(x + wb + WSPAN); h1 = __ldg(x + wb + WSPAN + 1); }
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          T v[E4 + 2];
          memcpy(&v[0], &q[j], 16);
          T n0 = __shfl_down_sync(0xFFFFFFFFu, v[0], 1), n1 = __shfl_down_sync(0xFFFFFFFFu, v[1], 1);
          if (j + 1 < Q) {                                          // lane 31: lane 0's next group
            T w[E4];
            memcpy(&w[0], &q[j + 1 < Q ? j + 1 : j], 16);
            const T f0 = __shfl_sync(0xFFFFFFFFu, w[0], 0), f1 = __shfl_sync(0xFFFFFFFFu, w[1], 0);
            if (lane == 31) { n0 = f0; n1 = f1; }
          } else {
            const T f0 = __shfl_sync(0xFFFFFFFFu, h0, 0), f1 = __shfl_sync(0xFFFFFFFFu, h1, 0);
            if (lane == 31) { n0 = f0; n1 = f1; }
          }
          v[E4] = n0;
          v[E4 + 1] = n1;
          U kk[E4 + 2];
#pragma unroll
          for (int i = 0; i < E4 + 2; ++i) kk[i] = K::f(v[i]);
          T out[E4];
#pragma unroll
          for (int i = 0; i < E4; ++i) out[i] = K::g(med3<U>(kk[i], kk[i + 1], kk[i + 2]));
          uint4 o;
          memcpy(&o, &out[0], 16);
#if MF_MED3_CS
          __stcs(reinterpret_cast<uint4*>(y + wb) + j * 32 + lane, o);
#else
          reinterpret_cast<uint4*>(y + wb)[j * 32 + lane] = o;
#endif
        }
      } else {                                                     // ragged tail or unaligned rows
        for (uint64_t o = wb + lane; o < min(wb + WSPAN, g.keep); o += 32)
          y[o] = K::g(med3<U>(K::f(__ldg(x + o)), K::f(__ldg(x + o + 1)), K::f(__ldg(x + o + 2))));
      }
    }
  }
}

template <int DT>
cudaError_t launch_med3(const Geom& g, cudaStream_t s) {
  using T = typename Traits<DT>::T;
  constexpr uint64_t SPAN = (uint64_t)kMed3Threads * kMed3Q * (16 / sizeof(T));
  LaunchInfo li;
  cudaError_t e = kernel_setup((const void*)mf_med3_kernel<DT>, 0, 0, &li);
  if (e != cudaSuccess) return e;
  const int sms = li.sms;
  const uint64_t cpr = (g.keep + SPAN - 1) / SPAN;
  const bool vec = (reinterpret_cast<uintptr_t>(g.x) % 16 == 0) && (reinterpret_cast<uintptr_t>(g.y) % 16 == 0) &&
                   (g.ld_x * sizeof(T)) % 16 == 0 && (g.ld_y * sizeof(T)) % 16 == 0;
  const uint64_t want = (uint64_t)sms * kMed3CtasPerSm;        // resident CTAs to fill the GPU
  const unsigned gy = (unsigned)std::min<uint64_t>(g.rows, 65535);
  const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cpr, (want + gy - 1) / gy));
  mf_med3_kernel<DT><<<dim3(gx, gy), kMed3Threads, 0, s>>>(g, cpr, vec);
  return cudaGetLastError();
}

template <int DT>
cudaError_t launch_dt(const Geom& g, cudaStream_t s) {
#if MF_MED3
  if (g.k == 3) return launch_med3<DT>(g, s);
#endif
  switch (g.k) {
#define MF_K(KK) case KK: return launch_k<DT, KK>(g, s);
    MF_K(1) MF_K(3) MF_K(5) MF_K(7) MF_K(9) MF_K(11) MF_K(13) MF_K(15)
    MF_K(17) MF_K(19) MF_K(21) MF_K(23) MF_K(25) MF_K(27) MF_K(29) MF_K(31)
#undef MF_K
    default:
      if (sizeof(typename Traits<DT>::U) == 4 && g.k <= kSmallMaxK32) return launch_small_k63(DT, g, s);
      return cudaErrorInvalidValue;
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
