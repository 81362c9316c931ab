// mf_small.cuh -- fused median filter for small windows (k <= 31, and k <= 63 for 32-bit
// keys): one thread per block pair, both phases in one pass over HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155) for k <= 31:
//   pad_to_blocks (filter.hpp:28-36)   -> virtual padding in the tile loader
//   piecewise_sort (filter.hpp:41-54)  -> a pruned odd-even merge network in registers
//   run_postprocess (filter.hpp:64-106) + Block (block.hpp:24-146)
//                                       -> the same Figure-7 state machine per pair,
//                                          with each sorted list held as a k-bit
//                                          live mask in one register (64-bit past k = 31).
// The Block's doubly linked list over sorted positions is the set of live sorted
// positions, so prev[m]/next[m] are "highest live bit below m" / "lowest live bit
// above m" (one clz/ffs each), and the stale-link undelete of dancing links is a
// plain bit set.  Cursor m and small-count s follow block.hpp:71-104 step for step,
// so the per-step (m, s) state is the reference's (up to the order of equal keys inside
// a block, which the key-ordered sort leaves open and which no emitted median depends on).  Every step is
// evaluated branch-free (selects, no divergence), fully unrolled over the K steps.
//
// Persistent CTAs stream tiles of T consecutive units: while a tile is sorted and
// walked, the next tile's T+1 blocks are already in flight into the other half of a
// double buffer (one TMA bulk copy per tile, completing on an mbarrier), so HBM reads
// overlap the compute.  The
// sorted keys and ranks use a lane-interleaved [position][column] layout whose column
// stride is a multiple of 32, so every warp access is conflict-free regardless of
// the data-dependent cursor positions.
#pragma once
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

// Tile shape by (key width, k): threads per CTA and units (block pairs) per thread per
// tile, measured on config 2 (f32, 2^26 samples) for every odd k <= 31.  8-byte keys keep
// 128 threads so that two tiles of input still fit the shared-memory budget.
template <int DT, int K> struct SmallShape {
  static constexpr bool wide = sizeof(typename Traits<DT>::U) == 8;
#ifndef MF_SMALL_T_K31
#define MF_SMALL_T_K31 512  // (experiments: tile shape of k = 24..31, 32-bit keys)
#endif
#ifndef MF_SMALL_T_K23
#define MF_SMALL_T_K23 256  // k = 9..23
#endif
#ifndef MF_SMALL_UPT_K31
#define MF_SMALL_UPT_K31 1
#endif
#ifndef MF_SMALL_T_K3
#define MF_SMALL_T_K3 256   // (experiments: tile shape of k <= 5, 32-bit keys)
#endif
#ifndef MF_SMALL_UPT_K3
#define MF_SMALL_UPT_K3 4
#endif
  // 33 <= k <= 53, re-measured after the column sort became a single inlined call site (no
  // local-memory element array any more): T = 64 / 96 / 128 / 256 gave, in ms on the c2 signal,
  //   k = 37: 1.10 / 1.07 / 1.02 / 0.70    k = 41: 1.31 / 1.27 / 0.94 / 0.73    k = 43: 1.28 / 1.29 / 0.91 / 0.83
  //   k = 45: 1.30 / 1.26 / 0.97 / 1.02    k = 47: 1.12 / 1.21 / 1.10 / 1.12    k = 49: 1.15 / 1.20 / 1.15 / 1.15
  //   k = 51: 1.14 / 1.08 / 1.14 / 1.14    k = 53: 1.14 / 1.11 / 1.15 / 1.16
#ifndef MF_SMALL_T_K35
#define MF_SMALL_T_K35 256  // k = 33, 35: 0.64 / 0.71 ms (128: 1.02 / 1.03)
#endif
#ifndef MF_SMALL_T_K43
#define MF_SMALL_T_K43 256  // k = 37..43
#endif
#ifndef MF_SMALL_T_K47
#define MF_SMALL_T_K47 128  // k = 45, 47
#endif
#ifndef MF_SMALL_T_K49
#define MF_SMALL_T_K49 128  // k = 49
#endif
#ifndef MF_SMALL_T_K53
#define MF_SMALL_T_K53 96   // k = 51, 53
#endif
#ifndef MF_SMALL_T_K63
#define MF_SMALL_T_K63 128  // k = 55..63: 1.17 ms each (96: 1.48 / 1.51 / 1.49; 256: 1.18; the medium kernel: 1.38 / 1.30 / 1.22)
#endif
  static constexpr int T = wide ? 128
                                : (K <= 5 ? MF_SMALL_T_K3 : K <= 7 ? 512 : K <= 23 ? MF_SMALL_T_K23 : K <= 31 ? MF_SMALL_T_K31
                                   : K <= 35 ? MF_SMALL_T_K35 : K <= 43 ? MF_SMALL_T_K43
                                   : K <= 47 ? MF_SMALL_T_K47 : K <= 49 ? MF_SMALL_T_K49 : K <= 53 ? MF_SMALL_T_K53 : MF_SMALL_T_K63);
  static constexpr int UPT = wide ? (K <= 7 ? 4 : K <= 15 ? 2 : 1)
                                  : (K <= 5 ? MF_SMALL_UPT_K3 : K <= 11 ? 2 : K <= 23 ? 1 : MF_SMALL_UPT_K31);
  // the cross-tile carry of the last block is spread over the first K threads (t < K)
  static_assert(T >= K, "small-kernel CTA must have at least K threads");
};

#ifndef MF_SMALL_FAST_MAXK
#define MF_SMALL_FAST_MAXK 31  // largest k with the sentinel-row walk variant (k = 5..31: 10-16 % faster; past 31 the
                               // second copy of the unrolled walk and the extra key row cost more than they save)
#endif
template <int DT, int K, int T>
struct SmallCfg {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  static constexpr int H = (K - 1) / 2;
  static constexpr int UPT = SmallShape<DT, K>::UPT;  // units (block pairs) per thread per tile
  static constexpr int TU = T * UPT;                    // units per tile
  static constexpr int NB = TU + 1;                     // blocks (columns) per tile
  static constexpr int SC = TU + 32;                    // column stride: >= NB, a multiple of 32
  // one input buffer (bytes): NB*K elements plus up to 16 bytes of alignment shift
  static constexpr int IO = (NB * K * (int)sizeof(U) + 15) / 16 * 16 + 16;
  static constexpr bool FAST = K <= MF_SMALL_FAST_MAXK;                         // sentinel row + fast walk variant
  static constexpr size_t off_key = 0;                                          // U[K*SC] (+ the sentinel row K)
  static constexpr size_t off_rank = off_key + sizeof(U) * (K + (FAST ? 1 : 0)) * SC;  // u8[K*SC]
  static constexpr size_t off_io = (off_rank + K * SC + 15) / 16 * 16;          // 2 x IO bytes
  static constexpr size_t smem = off_io + 2 * (size_t)IO;
};

// Live masks carry a sentinel bit at position K (the reference's list node k,
// block.hpp:21-24), so "next live" always exists and needs no branch.  K <= 31 uses 32-bit
// masks, 33 <= K <= 63 64-bit ones.
__device__ __forceinline__ uint32_t ffs_m(uint32_t m) { return (uint32_t)__ffs(m); }
__device__ __forceinline__ uint32_t ffs_m(uint64_t m) { return (uint32_t)__ffsll((long long)m); }
__device__ __forceinline__ uint32_t top_m(uint32_t m) { return 31u - (uint32_t)__clz(m); }
__device__ __forceinline__ uint32_t top_m(uint64_t m) { return 63u - (uint32_t)__clzll((long long)m); }
template <typename M>
__device__ __forceinline__ uint32_t live_next(M mask, uint32_t r) {
  // lowest live position > r (r < K): the sentinel K when none
  return r + ffs_m((M)(mask >> (r + 1)));
}
template <typename M>
__device__ __forceinline__ uint32_t live_prev(M mask, uint32_t m, uint32_t K) {
  // highest live position < m (m <= K), or K (the list head/tail node)
  const M lo = mask & (((M)1 << m) - (M)1);
  return sel(lo != 0, top_m(lo), K);
}
template <typename M>
__device__ __forceinline__ uint32_t live_succ(M mask, uint32_t m, uint32_t K) {
  // next[m] of the reference list: lowest live > m, or the list head when m = k
  const uint32_t nx = live_next(mask, m < K ? m : K - 1);
  return sel(m == K, ffs_m(mask) - 1, nx);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Element e of a staged tile sits at buf[e + misalign(x + base)], so smem and global
// addresses agree modulo 16 bytes and whole chunks can move with cp.async.
template <typename TV>
__device__ __forceinline__ int misalign(const TV* p) {
  return (int)((reinterpret_cast<uintptr_t>(p) & 15) / sizeof(TV));
}

// TMA bulk copy (cp.async.bulk, the 1-D form of the tensor memory accelerator): one thread
// issues one asynchronous global -> shared copy for the whole aligned body of a tile and the
// copy engine signals an mbarrier with the bytes it wrote, so no thread spends issue slots or
// address arithmetic on the staging loads.
#ifndef MF_SMALL_TMA
#define MF_SMALL_TMA 1  // 0: per-thread 16-byte cp.async chunks (the round-1 loader)
#endif
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
// orders this CTA's earlier generic-proxy accesses of shared memory before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(d), "l"(gmem_src), "r"(bytes), "r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  } while (!ok);
}

// Stage NE elements (raw input bits from x + base) into `buf`.  The whole 16-byte chunks
// inside [0, n) move as one TMA bulk copy that completes on `bar` (every call arms one phase
// of it, with zero bytes when the tile has no aligned body); the ragged head/tail and the
// padding past n (the reference's +INF sentinels, filter.hpp:28-36) are written directly.
// The padding value 0x7FF..F maps to the all-ones ukey for every dtype.  The caller has
// synchronised the CTA after its last generic access of `buf`.
template <typename TV, int NE, int T>
__device__ __forceinline__ void stage_tile(TV* buf, const TV* x, uint64_t n, uint64_t base, uint64_t* bar) {
  constexpr int EPC = 16 / (int)sizeof(TV);  // elements per 16-byte chunk
  const TV pad = (TV)(~(std::make_unsigned_t<TV>)0 >> 1);
  const int mis = misalign(x + base);
  TV* dst = buf + mis;
  const TV* src = x + base;
  const int real = n > base ? (int)(n - base < (uint64_t)NE ? n - base : (uint64_t)NE) : 0;
  const int h0 = min((EPC - mis) % EPC, real);   // unaligned head elements
  const int nchunks = (real - h0) / EPC;
  const int tail0 = h0 + nchunks * EPC;
#if MF_SMALL_TMA
  if (threadIdx.x == 0) {
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)nchunks * 16u);
    if (nchunks > 0) tma_load_1d(dst + h0, src + h0, (uint32_t)nchunks * 16u, bar);
  }
#else
  (void)bar;
  for (int c = threadIdx.x; c < nchunks; c += T) cp_async16(dst + h0 + c * EPC, src + h0 + c * EPC);
#endif
  if ((int)threadIdx.x < h0) dst[threadIdx.x] = src[threadIdx.x];
  for (int e = tail0 + threadIdx.x; e < NE; e += T) dst[e] = e < real ? src[e] : pad;
#if !MF_SMALL_TMA
  cp_async_commit();
#endif
}

#ifndef MF_SMALL_ONE_SUCC
#define MF_SMALL_ONE_SUCC 1  // one live_succ per step on the side that may advance
#endif
template <int DT, int K, int T>
__global__ void __launch_bounds__(T) mf_small_kernel(Geom g, uint64_t tiles_per_row, uint64_t total_tiles) {
  using C = SmallCfg<DT, K, T>;
  using Tr = typename C::Tr;
  using U = typename C::U;
  using TV = typename Tr::T;
#ifndef MF_SMALL_KEYORD_MAXK
#define MF_SMALL_KEYORD_MAXK 31  // (measured: k = 3..15 4-8 %, k = 23..31 8-12 % faster)
#endif
  // key-ordered elements (one compare per exchange): equal keys may take either order
  // inside a block, which changes no emitted median
  using E = std::conditional_t<(K <= MF_SMALL_KEYORD_MAXK), typename KeyOrd<U>::E, Elem<U>>;
  constexpr int H = C::H, SC = C::SC, UPT = C::UPT, TU = C::TU, NB = C::NB;
  extern __shared__ __align__(16) unsigned char smem[];
  U* skey = reinterpret_cast<U*>(smem + C::off_key);
  uint8_t* srank = smem + C::off_rank;
  auto io = [&](int which) { return reinterpret_cast<TV*>(smem + C::off_io + which * C::IO); };

  const uint32_t t = threadIdx.x;
  const uint64_t t_begin = total_tiles * blockIdx.x / gridDim.x;
  const uint64_t t_end = total_tiles * (blockIdx.x + 1) / gridDim.x;
  // (row, tile-in-row) of the current tile, advanced incrementally (no 64-bit division)
  uint64_t row = t_begin / tiles_per_row, tr = t_begin % tiles_per_row;
  auto xrow = [&](uint64_t r) { return reinterpret_cast<const TV*>(g.x) + r * g.ld_x; };
  // one mbarrier per input buffer; buffer b's phase flips every time it is refilled
  __shared__ __align__(8) uint64_t tile_bar[2];
  uint32_t bar_phase = 0;                 // bit b: parity to wait for on tile_bar[b]
  if (t == 0) {
    mbar_init(&tile_bar[0], 1);
    mbar_init(&tile_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (t_begin < t_end) stage_tile<TV, NB * K, T>(io(0), xrow(row), g.n, tr * TU * K, &tile_bar[0]);
  // sorted position K of every column: the list's sentinel node k (block.hpp:21-24), an all-ones key
  if constexpr (C::FAST)
    for (int c = t; c < SC; c += T) skey[K * SC + c] = UMax<U>::v;
  int cur = 0;
  bool carried = false;                   // column 0 already holds this tile's first block
  for (uint64_t tt = t_begin; tt < t_end; ++tt, cur ^= 1) {
    const TV* x = xrow(row);
    TV* y = reinterpret_cast<TV*>(g.y) + row * g.ld_y;
    const uint64_t u0 = tr * TU;
    uint64_t nrow = row, ntr = tr + 1;
    if (ntr == tiles_per_row) { ntr = 0; ++nrow; }
#if MF_SMALL_TMA
    mbar_wait(&tile_bar[cur], (bar_phase >> cur) & 1u);
    bar_phase ^= 1u << cur;
#else
    cp_async_wait_all();
#endif
    __syncthreads();                      // tile tt landed; previous tile fully consumed
    if (tt + 1 < t_end) stage_tile<TV, NB * K, T>(io(cur ^ 1), xrow(nrow), g.n, ntr * TU * K, &tile_bar[cur ^ 1]);  // prefetch
    TV* in = io(cur) + misalign(x + u0 * K);

    // ---- phase 1: sort column c (= block u0+c) in registers ----
    auto sort_column = [&](uint32_t c) {
      E v[K];
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = E::make(Tr::enc(in[c * K + i]), (uint32_t)i);
      sort_regs<K>(v);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        MF_ASSERT(v[p].idx() < (uint32_t)K && c < (uint32_t)SC);
        skey[p * SC + c] = v[p].key();
        srank[v[p].idx() * SC + c] = (uint8_t)p;
      }
    };
    // one call site, not unrolled: a single copy of the network, always inlined (with two call
    // sites nvcc outlined the column sort at k = 29, 31 and the element array went through
    // local memory).  Thread 0 also sorts column 0 when the previous tile did not carry it.
#pragma unroll 1
    for (int j = (!carried && t == 0) ? -1 : 0; j < UPT; ++j) sort_column(j < 0 ? 0u : t + T * j + 1);
    __syncthreads();                      // columns ready; `in` is free for output staging

    // ---- phase 2: Figure-7 postprocess for unit (A = column c, B = column c+1) ----
    // Steps past the last kept output run on padding harmlessly; only the store is bounded.
    // output staging, offset like the output row so whole 16-byte chunks store at once
    const uint64_t obase = u0 * K;
    const int omis = misalign(y + obase);
    U* ost = reinterpret_cast<U*>(io(cur) + omis);  // natural layout, odd K: conflict-free
    // The walk of one unit.  EXACT = false: neither block holds a real all-ones key (the usual
    // case), so the sentinel row orders Peek(A) against Peek(B) by a plain key compare -- an
    // exhausted list peeks the all-ones key, which no live element ties with -- and the
    // emitted value is the smaller peek.  EXACT = true keeps the explicit sentinel tests
    // (ties go to A; the sentinel is never smaller, filter.hpp:90-95).
    auto walk_unit = [&](auto exact_tag, uint32_t c) {
      constexpr bool EXACT = decltype(exact_tag)::value;
      const U* kA = skey + c;
      const U* kB = skey + c + 1;
      const uint8_t* rA = srank + c;
      const uint8_t* rB = srank + c + 1;
      constexpr uint32_t KK = K;
      using M = std::conditional_t<(K < 32), uint32_t, uint64_t>;
      constexpr M SENT = (M)1 << K;
      M maskA = SENT | (SENT - 1u);  // construct: all live, s = h, m = pi[h] (block.hpp:47-49)
      uint32_t mA = H, sA = H;
      M maskB = SENT;
      uint32_t mB = K;          // unwind: empty, m = k, s = 0 (block.hpp:62-63)
      U keyA = kA[H * SC], keyB = UMax<U>::v;
      ost[c * K] = keyA;                      // Peek of the constructed block (filter.hpp:81-82)
#pragma unroll
      for (int i = 1; i < K; ++i) {
        const uint32_t ra = rA[(i - 1) * SC];
        const uint32_t rb = rB[(i - 1) * SC];
        MF_ASSERT(ra < KK && rb < KK);
        // Delete(A, i-1): block.hpp:71-87
        maskA &= ~((M)1 << ra);
        const bool belowA = ra < mA;
        const uint32_t m1 = sel(ra == mA, live_next(maskA, ra), mA);
        // (prev of the moved cursor = highest live below the old one: ra itself is deleted and
        // nothing live lies between it and its successor -- one step off the dependency chain)
        const uint32_t pv = live_prev(maskA, mA, KK);
        mA = sel(!belowA && sA > 0, pv, m1);
        // s_A + s_B = h holds before every step (Balance restores it with its single advance), so
        // Balance must advance exactly when Delete took a small element away; s_B = h - s_A is
        // not carried
        // (s_A then changes by advA - need = -advB: need && !advB is need && advA)
        const bool need = belowA || sA > 0;
        // Undelete(B, i-1): block.hpp:89-98
        maskB |= (M)1 << rb;
        mB = sel(rb < mB, live_prev(maskB, mB, KK), mB);
        // Balance: filter.hpp:90-95 (ties go to A; the sentinel is never smaller)
        if constexpr (EXACT) {
          keyA = sel(mA == KK, UMax<U>::v, kA[min(mA, KK - 1) * SC]);
          keyB = sel(mB == KK, UMax<U>::v, kB[min(mB, KK - 1) * SC]);
        } else {
          keyA = kA[mA * SC];
          keyB = kB[mB * SC];
        }
        const bool bLess = EXACT ? (mB != KK) && (mA == KK || keyB < keyA) : keyB < keyA;
        const bool advA = need && !bLess, advB = need && bLess;
#if MF_SMALL_ONE_SUCC
        // at most one side advances: one successor search on the selected list.  Without real
        // all-ones keys a list that must advance is never at its sentinel (keyB < keyA rules it out
        // for B; for A both peeks would be sentinels, i.e. every live element is already small and
        // `need` is false), so the successor is the next live position above the cursor; the two
        // one-position shifts keep the unused result of a cursor at K defined.
        uint32_t nxt;
        if constexpr (EXACT) {
          nxt = live_succ(bLess ? maskB : maskA, bLess ? mB : mA, KK);
        } else {
          const uint32_t ms = bLess ? mB : mA;
          nxt = ms + ffs_m((M)((M)((bLess ? maskB : maskA) >> 1) >> ms));
        }
        mA = sel(advA, nxt, mA);
        mB = sel(advB, nxt, mB);
#else
        mA = sel(advA, live_succ(maskA, mA, KK), mA);
        mB = sel(advB, live_succ(maskB, mB, KK), mB);
#endif
        sA -= advB ? 1u : 0u;
        if constexpr (EXACT) {
          const U* kp = advA ? kA + min(mA, KK - 1) * SC : kB + min(mB, KK - 1) * SC;
          const U kn = *kp;
          keyA = sel(mA == KK, UMax<U>::v, sel(advA, kn, keyA));
          keyB = sel(mB == KK, UMax<U>::v, sel(advB, kn, keyB));
          // Emit min{Peek(A), Peek(B)}: filter.hpp:97-100
          const bool bLess2 = (mB != KK) && (mA == KK || keyB < keyA);
          ost[c * K + i] = sel(bLess2, keyB, keyA);
        } else {
          const U* kp = advA ? kA + mA * SC : kB + mB * SC;
          const U kn = *kp;
          keyA = sel(advA, kn, keyA);
          keyB = sel(advB, kn, keyB);
          ost[c * K + i] = min(keyA, keyB);   // Emit min{Peek(A), Peek(B)}: filter.hpp:97-100
        }
      }
    };
#pragma unroll 1
    for (int j = 0; j < UPT; ++j) {
      const uint32_t c = t + T * j;
      // a block's largest key sits at sorted position K-1
      if constexpr (C::FAST) {
        const bool exact = skey[(K - 1) * SC + c] == UMax<U>::v || skey[(K - 1) * SC + c + 1] == UMax<U>::v;
        if (exact) walk_unit(std::true_type{}, c);
        else walk_unit(std::false_type{}, c);
      } else {
        walk_unit(std::true_type{}, c);
      }
    }
    __syncthreads();

    // ---- carry the tile's last block to column 0 when the next tile continues the row ----
    carried = (nrow == row);
    if (carried && t < (uint32_t)K) {
      skey[t * SC] = skey[t * SC + TU];
      srank[t * SC] = srank[t * SC + TU];
    }

    // ---- coalesced 16-byte stores of the tile's contiguous outputs ----
    {
      constexpr int EPC = 16 / (int)sizeof(U);
      const uint64_t left = g.keep > obase ? g.keep - obase : 0;
      const uint32_t n_out = (uint32_t)(left < (uint64_t)TU * K ? left : (uint64_t)TU * K);
      MF_ASSERT(obase + n_out <= g.keep);
      check_sptr(ost, n_out);
      const uint32_t head = min((uint32_t)((EPC - omis) % EPC), n_out);
      const uint32_t nvec = (n_out - head) / EPC;
      TV* yo = y + obase;
      if (t < head) yo[t] = Tr::dec(ost[t]);
      for (uint32_t v = t; v < nvec; v += T) {
        union { uint4 q; U u[EPC]; TV o[EPC]; } w;
        w.q = *reinterpret_cast<const uint4*>(ost + head + v * EPC);
#pragma unroll
        for (int j = 0; j < EPC; ++j) w.o[j] = Tr::dec(w.u[j]);
        *reinterpret_cast<uint4*>(yo + head + v * EPC) = w.q;
      }
      for (uint32_t e = head + nvec * EPC + t; e < n_out; e += T) yo[e] = Tr::dec(ost[e]);
    }
    row = nrow;
    tr = ntr;
  }
}

// Launch the small kernel for one (dtype, K): persistent grid over the row-major tiles.
template <int DT, int K>
cudaError_t small_launch_k(const Geom& g, cudaStream_t s) {
  constexpr int kSmallThreads = SmallShape<DT, K>::T;
  using C = SmallCfg<DT, K, kSmallThreads>;
  auto kern = mf_small_kernel<DT, K, kSmallThreads>;
  LaunchInfo li;
  cudaError_t e = kernel_setup((const void*)kern, C::smem, kSmallThreads, &li);
  if (e != cudaSuccess) return e;
  const int sms = li.sms, resident = li.resident;
  const uint64_t tiles_per_row = (g.units + C::TU - 1) / C::TU;
  const uint64_t total = tiles_per_row * g.rows;
  // persistent grid: each CTA streams a contiguous range of tiles with a prefetch
  const uint64_t ctas = total < (uint64_t)sms * resident ? total : (uint64_t)sms * resident;
  kern<<<(unsigned)ctas, kSmallThreads, C::smem, s>>>(g, tiles_per_row, total);
  return cudaGetLastError();
}

}  // namespace mf
