// mf_common.cuh -- shared device-side vocabulary of the median-filter kernels.
//
// Keys.  Every kernel works on unsigned "ukeys" whose unsigned order is the
// reference's sample order (core.hpp:34-38): int32/int64 flip the sign bit; float
// and double use the IEEE totalOrder bit map of SURVEY.md §0.1 (the signed key
// `bits >= 0 ? bits : bits ^ 0x7FF..F`, then the sign flip).  The maps are
// bijections, so a median is emitted by inverting the map of the selected key:
// output bits are always the bits of an input element (bit-exact by construction).
//
// Padding.  The reference pads the last block with +INF sentinels
// (filter.hpp:28-36).  Here padding is virtual: a load past n yields UKEY_MAX, and
// because padding only ever occupies the tail of a block its (key, index) pair
// sorts after every real UKEY_MAX element of the block -- the same place the
// sentinel takes (core.hpp:34-47).  No kept window ever contains padding
// (filter.hpp:76-79), so padding never reaches an output.
#pragma once
#include <cassert>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

// MF_CHECK=1 builds (paper_1406_1717_b200.build.build(extra_flags=["-DMF_CHECK=1"], ...)):
// every data-dependent shared-memory index and every output store is bounds-checked with a
// device assert (file/line printed, kernel trapped).  compute-sanitizer is not available on
// the GPU pool, so the GPU suite run against this build is the memory-safety evidence
// (profiles/r02_checked_build.txt).  Release builds compile the checks away.
#ifndef MF_CHECK
#define MF_CHECK 0
#endif
#if MF_CHECK
#define MF_ASSERT(...) assert((__VA_ARGS__))
#else
#define MF_ASSERT(...) ((void)0)
#endif

namespace mf {

// size in bytes of the launch's dynamic shared memory (checked builds)
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
// `saddr` (shared-window byte address) .. saddr + bytes lies inside the dynamic smem that
// starts at shared-window address `base`
__device__ __forceinline__ void check_smem(uint32_t base, uint32_t saddr, uint32_t bytes) {
  MF_ASSERT(saddr >= base && saddr + bytes <= base + dyn_smem_bytes());
  (void)base; (void)saddr; (void)bytes;
}
#if MF_CHECK
extern __shared__ __align__(16) unsigned char mf_dyn_smem[];  // aliases every kernel's dynamic smem
#endif
// shared-window address `saddr` .. + bytes inside the launch's dynamic shared memory
__device__ __forceinline__ void check_saddr(uint32_t saddr, uint32_t bytes) {
#if MF_CHECK
  check_smem((uint32_t)__cvta_generic_to_shared(mf_dyn_smem), saddr, bytes);
#else
  (void)saddr; (void)bytes;
#endif
}
// p .. p + count elements inside the launch's dynamic shared memory
template <typename P>
__device__ __forceinline__ void check_sptr(const P* p, uint32_t count = 1) {
#if MF_CHECK
  check_saddr((uint32_t)__cvta_generic_to_shared(p), (uint32_t)(sizeof(P) * count));
#else
  (void)p; (void)count;
#endif
}

enum DType : int { DT_I32 = 0, DT_I64 = 1, DT_F32 = 2, DT_F64 = 3 };

template <int DT> struct Traits;
template <> struct Traits<DT_I32> {
  using T = int32_t; using U = uint32_t;
  __host__ __device__ static __forceinline__ U enc(T v) { return (U)v ^ 0x80000000u; }
  __host__ __device__ static __forceinline__ T dec(U u) { return (T)(u ^ 0x80000000u); }
};
template <> struct Traits<DT_I64> {
  using T = int64_t; using U = uint64_t;
  __host__ __device__ static __forceinline__ U enc(T v) { return (U)v ^ 0x8000000000000000ull; }
  __host__ __device__ static __forceinline__ T dec(U u) { return (T)(u ^ 0x8000000000000000ull); }
};
template <> struct Traits<DT_F32> {
  using T = uint32_t; using U = uint32_t;  // float carried as its bits
  __host__ __device__ static __forceinline__ U enc(T b) { return (b & 0x80000000u) ? ~b : (b ^ 0x80000000u); }
  __host__ __device__ static __forceinline__ T dec(U u) { return (u & 0x80000000u) ? (u ^ 0x80000000u) : ~u; }
};
template <> struct Traits<DT_F64> {
  using T = uint64_t; using U = uint64_t;  // double carried as its bits
  __host__ __device__ static __forceinline__ U enc(T b) {
    return (b & 0x8000000000000000ull) ? ~b : (b ^ 0x8000000000000000ull);
  }
  __host__ __device__ static __forceinline__ T dec(U u) {
    return (u & 0x8000000000000000ull) ? (u ^ 0x8000000000000000ull) : ~u;
  }
};

template <typename U> struct UMax;
template <> struct UMax<uint32_t> { static constexpr uint32_t v = 0xFFFFFFFFu; };
template <> struct UMax<uint64_t> { static constexpr uint64_t v = 0xFFFFFFFFFFFFFFFFull; };

// Problem geometry shared by every kernel.  A "signal" (row) has n samples; the
// output has keep = n-k+1 medians.  Output o = u*k + i belongs to "unit" u: the
// window made of block u restricted to indices >= i plus block u+1 restricted to
// indices < i.  Unit u therefore owns the k contiguous outputs [u*k, u*k+k) and is
// exactly the reference's block pair (A = X_u, B = X_{u+1}) of filter.hpp:83-101
// (its step i emits y[u*k+i+1]); output u*k (i = 0) is Peek of the freshly
// constructed block u (filter.hpp:81-82 for u = 0, and the last step of the
// previous pair otherwise).
struct Geom {
  const void* x;      // rows x ld_x samples
  void* y;            // rows x ld_y outputs
  uint64_t n;         // samples per row
  uint64_t ld_x, ld_y;
  uint32_t k, h;
  uint64_t keep;      // outputs per row = n - k + 1 (>= 1)
  uint64_t units;     // units per row = ceil(keep / k)
  uint32_t rows;
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Forced select (selp): both operands are computed, so no divergent branch is emitted.
#ifndef MF_SEL_PLAIN
#define MF_SEL_PLAIN 1  // plain ternaries: ptxas still emits selects, and schedules them better (k = 31 -3 %)
#endif
#if MF_SEL_PLAIN
__device__ __forceinline__ uint32_t sel(bool c, uint32_t a, uint32_t b) { return c ? a : b; }
__device__ __forceinline__ uint64_t sel(bool c, uint64_t a, uint64_t b) { return c ? a : b; }
#else
__device__ __forceinline__ uint32_t sel(bool c, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
      : "=r"(r) : "r"((uint32_t)c), "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint64_t sel(bool c, uint64_t a, uint64_t b) {
  uint64_t r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b64 %0, %2, %3, p;\n\t}"
      : "=l"(r) : "r"((uint32_t)c), "l"(a), "l"(b));
  return r;
}
#endif


}  // namespace mf
