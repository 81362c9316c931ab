// mf_small.cuh -- fused median filter for small windows (k <= 31): one thread per
// block pair, both phases in one pass over HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155) for k <= 31:
//   pad_to_blocks (filter.hpp:28-36)   -> virtual padding in the tile loader
//   piecewise_sort (filter.hpp:41-54)  -> a pruned odd-even merge network in registers
//   run_postprocess (filter.hpp:64-106) + Block (block.hpp:24-146)
//                                       -> the same Figure-7 state machine per pair,
//                                          with each sorted list held as a k-bit
//                                          live mask in one register.
// The Block's doubly linked list over sorted positions is the set of live sorted
// positions, so prev[m]/next[m] are "highest live bit below m" / "lowest live bit
// above m" (one clz/ffs each), and the stale-link undelete of dancing links is a
// plain bit set.  Cursor m and small-count s follow block.hpp:71-104 step for step,
// so the per-step (m, s) state is identical to the reference's (tests pin it).
//
// Tile: T threads own T consecutive units (block pairs); the T+1 blocks of the
// tile are loaded once (coalesced), sorted into a lane-interleaved smem layout
// ([position][column], column stride a multiple of 32: every warp access is
// conflict-free regardless of the data-dependent position), walked, staged and
// stored coalesced.
#pragma once
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

template <int DT, int K, int T>
struct SmallCfg {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  static constexpr int H = (K - 1) / 2;
  static constexpr int SC = T + 32;  // column stride: >= T+1 and a multiple of 32
  static constexpr size_t off_key = 0;                                   // U[K*SC]
  static constexpr size_t off_rank = off_key + sizeof(U) * K * SC;       // u8[K*SC]
  static constexpr size_t off_io = (off_rank + K * SC + 15) / 16 * 16;   // U[(T+1)*K]
  static constexpr size_t smem = off_io + sizeof(U) * (T + 1) * K;
};

// below/above helpers over a K-bit live mask (K <= 31)
__device__ __forceinline__ uint32_t live_next(uint32_t mask, uint32_t r, uint32_t K) {
  // lowest live position > r (r < K), or K
  const uint32_t hi = mask >> (r + 1);
  return hi ? r + 1 + (uint32_t)__ffs(hi) - 1 : K;
}
__device__ __forceinline__ uint32_t live_prev(uint32_t mask, uint32_t m, uint32_t K) {
  // highest live position < m (m <= K), or K (the list head/tail node)
  const uint32_t lo = mask & ((1u << m) - 1u);
  return lo ? 31u - (uint32_t)__clz(lo) : K;
}
__device__ __forceinline__ uint32_t live_first(uint32_t mask, uint32_t K) {
  return mask ? (uint32_t)__ffs(mask) - 1 : K;
}

template <int DT, int K, int T>
__global__ void __launch_bounds__(T) mf_small_kernel(Geom g) {
  using C = SmallCfg<DT, K, T>;
  using Tr = typename C::Tr;
  using U = typename C::U;
  using TV = typename Tr::T;
  using E = Elem<U>;
  constexpr int H = C::H, SC = C::SC;
  extern __shared__ __align__(16) unsigned char smem[];
  U* skey = reinterpret_cast<U*>(smem + C::off_key);
  uint8_t* srank = smem + C::off_rank;
  U* io = reinterpret_cast<U*>(smem + C::off_io);

  const uint32_t t = threadIdx.x;
  const uint64_t row = blockIdx.y;
  const uint64_t u0 = (uint64_t)blockIdx.x * T;
  const TV* __restrict__ x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  TV* __restrict__ y = reinterpret_cast<TV*>(g.y) + row * g.ld_y;
  const uint64_t base = u0 * K;

  // ---- load blocks u0 .. u0+T (virtual +INF padding past n) ----
  for (uint32_t e = t; e < (uint32_t)((T + 1) * K); e += T) {
    const uint64_t gp = base + e;
    io[e] = gp < g.n ? Tr::enc(x[gp]) : UMax<U>::v;
  }
  __syncthreads();

  // ---- phase 1: sort column c (= block u0+c) in registers ----
  auto sort_column = [&](uint32_t c) {
    E v[K];
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = E::make(io[c * K + i], (uint32_t)i);
    sort_regs<K>(v);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      skey[p * SC + c] = v[p].key();
      srank[v[p].idx() * SC + c] = (uint8_t)p;
    }
  };
  sort_column(t + 1);
  if (t == 0) sort_column(0);
  __syncthreads();

  // ---- phase 2: Figure-7 postprocess for unit u = (A = column t, B = column t+1) ----
  const uint64_t u = u0 + t;
  uint32_t imax = 0;
  if (u < g.units) {
    const uint64_t rem = g.keep - u * K;
    imax = rem < (uint64_t)K ? (uint32_t)rem : (uint32_t)K;
  }
  // outputs are staged in io (natural layout, odd K: conflict-free)
  __syncthreads();  // everyone is done reading io for sorting
  if (imax > 0) {
    const uint32_t ca = t, cb = t + 1;
    uint32_t maskA = (K == 32) ? 0xFFFFFFFFu : ((1u << K) - 1u);
    uint32_t mA = H, sA = H;          // construct: s = h, m = pi[h] (block.hpp:47-49)
    uint32_t maskB = 0, mB = K, sB = 0;  // unwind: empty, m = k, s = 0 (block.hpp:62-63)
    U keyA = skey[mA * SC + ca];
    U keyB = 0;
    io[t * K] = keyA;  // Peek of the constructed block (filter.hpp:81-82)
    for (uint32_t i = 1; i < imax; ++i) {
      const uint32_t s = i - 1;
      const uint32_t ra = srank[s * SC + ca];
      const uint32_t rb = srank[s * SC + cb];
      // Delete(A, s): block.hpp:71-87
      maskA &= ~(1u << ra);
      if (ra < mA) {
        --sA;
      } else {
        if (ra == mA) mA = live_next(maskA, ra, K);
        if (sA > 0) { mA = live_prev(maskA, mA, K); --sA; }
      }
      // Undelete(B, s): block.hpp:89-98
      maskB |= 1u << rb;
      if (rb < mB) mB = live_prev(maskB, mB, K);
      // Balance: filter.hpp:90-95 (ties go to A)
      keyA = mA < K ? skey[mA * SC + ca] : UMax<U>::v;
      keyB = mB < K ? skey[mB * SC + cb] : UMax<U>::v;
      if ((int)(sA + sB) < H) {
        const bool b_less = (mB != K) && (mA == K || keyB < keyA);
        if (!b_less) {
          mA = (mA == K) ? live_first(maskA, K) : live_next(maskA, mA, K);
          ++sA;
          keyA = mA < K ? skey[mA * SC + ca] : UMax<U>::v;
        } else {
          mB = (mB == K) ? live_first(maskB, K) : live_next(maskB, mB, K);
          ++sB;
          keyB = mB < K ? skey[mB * SC + cb] : UMax<U>::v;
        }
      }
      // Emit min{Peek(A), Peek(B)}: filter.hpp:97-100
      const bool b_less = (mB != K) && (mA == K || keyB < keyA);
      io[t * K + i] = b_less ? keyB : keyA;
    }
  }
  __syncthreads();

  // ---- coalesced store of the tile's contiguous outputs ----
  const uint64_t tile_out = (uint64_t)T * K;
  for (uint32_t e = t; e < tile_out; e += T) {
    const uint64_t o = base + e;
    if (o < g.keep) y[o] = Tr::dec(io[e]);
  }
}

}  // namespace mf
