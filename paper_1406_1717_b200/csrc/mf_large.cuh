// mf_large.cuh -- median filter for large windows (k beyond the fused kernels'
// shared-memory budget, e.g. k = 10,001 and 100,001): multi-kernel pipeline with
// the per-pair state in L2/HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155).
//   piecewise_sort (filter.hpp:41-54) -> segmented global merge sort: a CTA sorts a
//       tile of TS elements (8 warp sorts + 3 CTA merge-path levels in padded smem),
//       then ceil(log2(k/TS)) global merge-path passes; blocks are segments and the
//       (key, index) elements keep it stable.
//   run_postprocess (filter.hpp:64-106) -> per block pair (unit):
//     ml_unit_merge   merge path of sorted A and sorted B: merged keys,
//                     merged-position -> (block, index), index -> merged position
//                     (the Delete(A,i) / Undelete(B,i) targets), and, fused, the live
//                     counts of every 1024-position "superword" at every chunk start;
//     ml_walk         one thread per chunk of CL steps.  The state before step i is the
//                     live set {A: idx >= i} u {B: idx < i} (Eq. 4 / Lemma 1,
//                     SURVEY.md §0.6); the thread keeps only the cursor p and the one
//                     32-position word of the live set around it, recomputing a word
//                     from the origin table when the cursor leaves it, so per-thread state
//                     is O(1) however large k is.
#pragma once
#include "mf_blocksort.cuh"
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

constexpr int LNT = 256;         // threads per CTA
constexpr int LR2 = 16;          // outputs per thread in merge tiles
constexpr int LQ = LNT * LR2;    // merge tile (elements), a multiple of 1024
constexpr int LPS = 4;           // pad shift of merge tiles (R = 16)
template <typename U>
constexpr size_t merge_tile_smem() { return sizeof(Elem<U>) * (LQ + (LQ >> LPS) + 1); }
// 64-bit keys in key order (the filter's passes, not the phase API) keep their tiles as
// struct-of-arrays in shared memory: keys and indices in two padded arrays, 12 bytes per
// element instead of 16, key-only merge compares (ml_tile_sort_soa, merge_tile_soa).
#ifndef MF_TS_SOA
#define MF_TS_SOA 1
#endif
#ifndef MF_SOA32
#define MF_SOA32 0  // 1: 32-bit keys too (4-byte key compares in the merge tiles): measured c5 +0.6 %
#endif
template <typename U, bool KO>
constexpr bool kSoa = MF_TS_SOA && KO && (sizeof(U) == 8 || MF_SOA32);
template <typename U, bool SOA>
constexpr size_t merge_tile_bytes() {
  return (SOA ? sizeof(U) + sizeof(uint32_t) : sizeof(Elem<U>)) * (LQ + (LQ >> LPS) + 1);
}

// tile sort geometry by key width: 8 warps x 32R elements
template <typename U> struct TileSortCfg;
template <> struct TileSortCfg<uint32_t> { static constexpr int R = 32; };
template <> struct TileSortCfg<uint64_t> { static constexpr int R = 16; };
#ifndef MF_TS_PS
#define MF_TS_PS 0  // pad shift of the tile sort's shared tile (0: pad_shift<R>())
#endif
template <typename U> struct TileSort {
  static constexpr int R = TileSortCfg<U>::R;
  static constexpr int PS = MF_TS_PS ? MF_TS_PS : pad_shift<R>();
  static constexpr int TS = 8 * 32 * R;
  static constexpr size_t smem = sizeof(Elem<U>) * (TS + (TS >> PS) + 1) + sizeof(uint32_t) * (LNT / 32);
};

struct LargeGeom {
  Geom g;
  uint64_t nb;        // blocks per row (= units + 1)
  uint32_t TS;        // tile-sort size (elements)
  uint32_t tiles;     // tile sorts per block = ceil(k / TS)
  uint32_t mtiles;    // merge tiles per block = ceil(k / LQ)
  uint32_t nq;        // merged positions per unit = 2k
  uint32_t nqp;       // padded stride (multiple of 32)
  uint32_t tiles2;    // unit-merge tiles per unit = ceil(2k / LQ)
  uint32_t CL;        // steps per walk chunk (a power of two)
  uint32_t CLshift;   // log2(CL)
  uint32_t C;         // chunks per unit
  uint32_t NS;        // superwords (1024 positions) per unit
};

// Sort element of the large-k passes.  The filter sorts by key only (KO: equal keys in any
// order, which no emitted median depends on; KElem* keep Elem's memory layout and compare
// one key instead of (key, index)); the phase API (mf_block_sort_*) needs piecewise_sort's
// exact permutation and sorts by (key, index).
template <typename U, bool KO> using SortElem = std::conditional_t<KO, typename KeyOrd<U>::E, Elem<U>>;

// ---- phase 1a: sort TS-element tiles of every block ----------------------------------
template <int DT, bool KO>
__global__ void __launch_bounds__(LNT, 3) ml_tile_sort(LargeGeom L, Elem<typename Traits<DT>::U>* out_) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using E = SortElem<U, KO>;
  static_assert(sizeof(E) == sizeof(Elem<U>), "same memory layout");
  E* out = reinterpret_cast<E*>(out_);
  using TV = typename Tr::T;
  using C = TileSort<U>;
  constexpr int R = C::R, PS = C::PS, TS = C::TS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* s = reinterpret_cast<E*>(smem_raw);
  const Geom& g = L.g;
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.tiles;
  const uint32_t t = blockIdx.x % L.tiles;
  const TV* x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  const uint32_t k = g.k;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  E v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t e = t * TS + warp * 32 * R + lane + 32 * r;  // coalesced across the warp
    const uint64_t gp = b * k + e;
    const U key = (e < k && gp < g.n) ? Tr::enc(__ldg(x + gp)) : UMax<U>::v;
    v[r] = E::make(key, e);
  }
#ifndef MF_BL_LARGE
#define MF_BL_LARGE 2  // bitonic register levels of the tile sort (experiments)
#endif
  warp_sort_regs<E, R, PS, MF_BL_LARGE>(v, s, warp * 32 * R, lane);
  __syncthreads();
  merge_levels<E, R, PS, true>(s, 0, threadIdx.x, 32 * R, TS, v);
  const uint32_t len = min((uint32_t)TS, k - t * TS);
  E* o = out + (row * L.nb + b) * k + (uint64_t)t * TS;
  if (E::kFull || len == (uint32_t)TS) {
    for (uint32_t i = threadIdx.x; i < len; i += LNT) o[i] = s[pad<PS>(i)];
    return;
  }
  // Key order leaves the slot fillers past the block's end (index >= k, key UKEY_MAX) mixed
  // with real UKEY_MAX elements: keep only real elements, in sorted order (stable
  // compaction; one thread per run of TS / LNT positions, CTA scan of the run counts).
  constexpr int RUN = TS / LNT;
  uint32_t* wsum = reinterpret_cast<uint32_t*>(s + TS + (TS >> PS) + 1);  // past the tile
  const uint32_t i0 = threadIdx.x * RUN;
  uint32_t c = 0;
#pragma unroll 4
  for (int j = 0; j < RUN; ++j) c += s[pad<PS>(i0 + j)].idx() < k;
  uint32_t inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= (uint32_t)d) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t q = inc - c;
  for (uint32_t w = 0; w < warp; ++w) q += wsum[w];
#pragma unroll 4
  for (int j = 0; j < RUN; ++j) {
    const E e = s[pad<PS>(i0 + j)];
    if (e.idx() < k) o[q++] = e;
  }
}

// ---- phase 1a (experiment, MF_TILE_RADIX=1): LSD radix sort of a TS-element tile ------
// 5-bit digits, least significant first.  Every pass is stable and the tile starts in index
// order, so the result is the (key, index) order of E::less without comparing indices.
// Ranking is warp-level multisplit with the 32 bin counters in registers, one bin per
// lane: five ballots give each lane the mask of lanes holding its bin, a shuffle from lane
// `digit` gives an element its peers and the running count of its bin, so no pass has a
// shared-memory read -> write chain.  A bin-major, warp-minor exclusive scan of the NB x W
// warp totals turns ranks into positions.  Digits on which every key of the tile agrees are
// skipped (AND/OR test).  (Measured: 8-bit digits with warp counters in shared memory were
// slower than the comparison network, with match.any or with ballots.)
template <typename U> struct TileRadixCfg;
template <> struct TileRadixCfg<uint32_t> { static constexpr int NT = 1024, R = 8, MINB = 1; };
template <> struct TileRadixCfg<uint64_t> { static constexpr int NT = 256, R = 16, MINB = 3; };
template <typename U> struct TileRadix {
  static constexpr int NT = TileRadixCfg<U>::NT, R = TileRadixCfg<U>::R, W = NT / 32, MINB = TileRadixCfg<U>::MINB;
  static constexpr int DB = 5, NB = 1 << DB;
  static constexpr int WS = 32 * R, TS = NT * R;
  static_assert(NB * W == NT, "one scan entry (bin, warp) per thread");
  static constexpr size_t smem = sizeof(U) * TS + sizeof(uint16_t) * TS + sizeof(uint32_t) * NT +
                                 sizeof(U) * 2 * W + sizeof(uint32_t) * W;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t red_and(uint32_t v) { return __reduce_and_sync(0xFFFFFFFFu, v); }
__device__ __forceinline__ uint32_t red_or(uint32_t v) { return __reduce_or_sync(0xFFFFFFFFu, v); }
__device__ __forceinline__ uint64_t red_and(uint64_t v) {
  return ((uint64_t)red_and((uint32_t)(v >> 32)) << 32) | red_and((uint32_t)v);
}
__device__ __forceinline__ uint64_t red_or(uint64_t v) {
  return ((uint64_t)red_or((uint32_t)(v >> 32)) << 32) | red_or((uint32_t)v);
}
// full 16-byte stores for 64-bit keys: a partially written sector costs a DRAM fill read
__device__ __forceinline__ void store_elem(Elem<uint32_t>* o, uint32_t key, uint32_t idx) {
  *o = Elem<uint32_t>::make(key, idx);
}
__device__ __forceinline__ void store_elem(Elem<uint64_t>* o, uint64_t key, uint32_t idx) {
  static_assert(sizeof(Elem<uint64_t>) == 16, "16-byte element");
  *reinterpret_cast<uint4*>(o) = make_uint4((uint32_t)key, (uint32_t)(key >> 32), idx, 0u);
}

// ---- phase 1a, 64-bit keys in key order: struct-of-arrays tile sort ------------------------
// The filter's tile sort for 64-bit keys keeps keys and indices in two padded shared
// arrays instead of 16-byte {key, index} elements: a merge step compares keys only (one
// 8-byte load refills the consumed side), and the index of the taken element is loaded off
// the dependency chain.  8-byte keys at the pad<4> stride store conflict-free, and the tile
// takes 12 bytes per element of shared memory instead of 16.  Ties between equal keys may
// land in any order (key order, KElem64); the slot fillers of the last tile are compacted
// as in ml_tile_sort.
#ifndef MF_TS_SOA_MINB
#define MF_TS_SOA_MINB 3
#endif
struct TileSoa {
  static constexpr int R = 16, PS = 4, TS = 8 * 32 * R;
  static constexpr int NSLOT = TS + (TS >> PS) + 1;
  static constexpr size_t smem = (sizeof(uint64_t) + sizeof(uint32_t)) * NSLOT + sizeof(uint32_t) * (LNT / 32);
};

template <int DT>
__global__ void __launch_bounds__(LNT, MF_TS_SOA_MINB) ml_tile_sort_soa(LargeGeom L, Elem<uint64_t>* out) {
  using Tr = Traits<DT>;
  using TV = typename Tr::T;
  static_assert(sizeof(typename Tr::U) == 8, "64-bit keys");
  constexpr int R = TileSoa::R, PS = TileSoa::PS, TS = TileSoa::TS, NSLOT = TileSoa::NSLOT;
  static_assert(TS == TileSort<uint64_t>::TS, "same tiles as the merge passes expect");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* si = reinterpret_cast<uint32_t*>(sk + NSLOT);
  uint32_t* wsum = si + NSLOT;
  const Geom& g = L.g;
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.tiles;
  const uint32_t t = blockIdx.x % L.tiles;
  const TV* x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  const uint32_t k = g.k;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    KElem64 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t e = t * TS + warp * 32 * R + lane + 32 * r;  // coalesced across the warp
      const uint64_t gp = b * k + e;
      const uint64_t key = (e < k && gp < g.n) ? Tr::enc(__ldg(x + gp)) : UMax<uint64_t>::v;
      v[r] = KElem64::make(key, e);
    }
    sort_regs<R>(v);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = pad<PS>((int)(warp * 32 * R + lane * R + r));
      sk[p] = v[r].k;
      si[p] = v[r].i;
    }
  }
  __syncwarp();
  uint64_t vk[R];
  uint32_t vi[R];
  merge_levels_soa<R, PS>(sk, si, warp * 32 * R, lane, R, 32 * R, vk, vi, SyncWarp{});
  __syncthreads();
  merge_levels_soa<R, PS>(sk, si, 0, threadIdx.x, 32 * R, TS, vk, vi, SyncCta{});
  const uint32_t len = min((uint32_t)TS, k - t * TS);
  Elem<uint64_t>* o = out + (row * L.nb + b) * k + (uint64_t)t * TS;
  if (len == (uint32_t)TS) {
    for (uint32_t i = threadIdx.x; i < len; i += LNT) store_elem(o + i, sk[pad<PS>(i)], si[pad<PS>(i)]);
    return;
  }
  // last tile of a block: keep the real elements (index < k) in sorted order (see ml_tile_sort)
  constexpr int RUN = TS / LNT;
  const uint32_t i0 = threadIdx.x * RUN;
  uint32_t c = 0;
#pragma unroll 4
  for (int j = 0; j < RUN; ++j) c += si[pad<PS>(i0 + j)] < k;
  uint32_t inc = c;
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, dd);
    if (lane >= (uint32_t)dd) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t q = inc - c;
  for (uint32_t w = 0; w < warp; ++w) q += wsum[w];
#pragma unroll 4
  for (int j = 0; j < RUN; ++j) {
    const uint32_t e = si[pad<PS>(i0 + j)];
    if (e < k) {
      MF_ASSERT(q < len);
      store_elem(o + q++, sk[pad<PS>(i0 + j)], e);
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(TileRadix<typename Traits<DT>::U>::NT, TileRadix<typename Traits<DT>::U>::MINB)
    ml_tile_radix(LargeGeom L, Elem<typename Traits<DT>::U>* out) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using TV = typename Tr::T;
  using C = TileRadix<U>;
  constexpr int R = C::R, W = C::W, WS = C::WS, TS = C::TS, DB = C::DB, NB = C::NB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  U* sk = reinterpret_cast<U*>(smem_raw);
  uint16_t* si = reinterpret_cast<uint16_t*>(sk + TS);
  uint32_t* tot = reinterpret_cast<uint32_t*>(si + TS);         // [NB][W] warp totals -> bases
  U* wred = reinterpret_cast<U*>(tot + C::NT);                   // [W][2] AND / OR
  uint32_t* wsum = reinterpret_cast<uint32_t*>(wred + 2 * W);    // [W] scan carries
  const Geom& g = L.g;
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.tiles;
  const uint32_t t = blockIdx.x % L.tiles;
  const TV* x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  const uint32_t k = g.k;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = warp * WS + lane;                        // position of item r: base + 32r
  U key[R];
  uint32_t rix[R];                                               // index (low 16) | rank (high 16)
  U kand = UMax<U>::v, kor = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t e = t * TS + base + 32 * r;
    const uint64_t gp = b * k + e;
    key[r] = (e < k && gp < g.n) ? Tr::enc(__ldg(x + gp)) : UMax<U>::v;
    rix[r] = base + 32 * r;
    kand &= key[r];
    kor |= key[r];
  }
  kand = red_and(kand);
  kor = red_or(kor);
  if (lane == 0) { wred[2 * warp] = kand; wred[2 * warp + 1] = kor; }
  __syncthreads();
  U diff = 0;
  {
    U a = UMax<U>::v, o = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) { a &= wred[2 * w]; o |= wred[2 * w + 1]; }
    diff = a ^ o;                                                // bits that vary in the tile
  }
  const uint32_t lt = lanemask_lt();
  uint32_t xm[DB];                                               // ~0 where this lane's bin has a 0 bit
#pragma unroll
  for (int bit = 0; bit < DB; ++bit) xm[bit] = ((lane >> bit) & 1u) ? 0u : 0xFFFFFFFFu;
#pragma unroll 1
  for (int d = 0; d < (int)(8 * sizeof(U)); d += DB) {
    if (((diff >> d) & (NB - 1)) == 0) continue;                // uniform across the CTA
    uint32_t cnt = 0;                                            // this warp's count of bin `lane`
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t dg = (uint32_t)(key[r] >> d) & (NB - 1);
      uint32_t m = 0xFFFFFFFFu;                                  // lanes whose digit is `lane`
#pragma unroll
      for (int bit = 0; bit < DB; ++bit) m &= __ballot_sync(0xFFFFFFFFu, (dg >> bit) & 1u) ^ xm[bit];
      const uint32_t peers = __shfl_sync(0xFFFFFFFFu, m, dg);
      const uint32_t cb = __shfl_sync(0xFFFFFFFFu, cnt, dg);
      rix[r] = (rix[r] & 0xFFFFu) | ((cb + __popc(peers & lt)) << 16);
      cnt += __popc(m);
    }
    tot[lane * W + warp] = cnt;
    __syncthreads();
    {  // exclusive scan of tot in (bin, warp) order, one entry per thread
      const uint32_t v = tot[threadIdx.x];
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      uint32_t pre = inc - v;
      for (uint32_t w = 0; w < warp; ++w) pre += wsum[w];
      tot[threadIdx.x] = pre;
    }
    __syncthreads();
    const uint32_t bw = tot[lane * W + warp];                    // this warp's base of bin `lane`
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t dg = (uint32_t)(key[r] >> d) & (NB - 1);
      const uint32_t pos = __shfl_sync(0xFFFFFFFFu, bw, dg) + (rix[r] >> 16);
      sk[pos] = key[r];
      si[pos] = (uint16_t)rix[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      key[r] = sk[base + 32 * r];
      rix[r] = si[base + 32 * r];
    }
  }
  const uint32_t len = min((uint32_t)TS, k - t * TS);
  Elem<U>* o = out + (row * L.nb + b) * k + (uint64_t)t * TS;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t p = base + 32 * r;
    if (p < len) store_elem(o + p, key[r], t * TS + (rix[r] & 0xFFFFu));
  }
}

// Warp-cooperative merge-path split: the number of X elements among the first d merged
// elements of X[0,lx) and Y[0,ly) under `before(x, y)` (x goes first).  Each round probes
// 32 diagonal points at once, so a split over 10^5 costs 4 rounds of loads, not 17.
template <typename E, typename Before>
__device__ __forceinline__ uint32_t warp_split(const E* X, uint32_t lx, const E* Y, uint32_t ly, uint32_t d,
                                               Before before, uint32_t lane) {
  uint32_t lo = d > ly ? d - ly : 0, hi = d < lx ? d : lx;
  while (lo < hi) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t mid = lo + lane * step;
    const bool p = mid < hi && before(X[mid], Y[d - 1 - mid]);
    const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, p));  // a prefix of lanes: monotone
    const uint32_t nlo = c ? lo + (c - 1) * step + 1 : lo;
    hi = min(hi, lo + c * step);
    lo = nlo;
  }
  return lo;
}

// One LQ-output tile of a merge of X[0,lx) and Y[0,ly), outputs [d0, d1): the inputs go
// through padded smem; thread `tid` merges outputs [tid*LR2, tid*LR2 + LR2) into v and
// returns how many it produced; `srcB[r]` tells which side each came from.
template <typename E, typename Before>
__device__ __forceinline__ int merge_tile(E* s, const E* X, const E* Y, uint32_t d0, uint32_t d1, uint2 sp,
                                          Before before, E (&v)[LR2], bool (&srcB)[LR2], uint32_t& nx_out) {
  const uint32_t a0 = sp.x, a1 = sp.y;   // merge-path splits, precomputed by ml_partition_*
  const uint32_t b0 = d0 - a0, b1 = d1 - a1;
  const uint32_t nx = a1 - a0, ny = b1 - b0;
  const uint32_t yoff = (uint32_t)(Y - X);  // Y follows X in the same buffer (runs / blocks)
  {  // stage the tile's inputs: all LR2 global loads in flight before the shared stores
    E tmp[LR2];
#pragma unroll
    for (int j = 0; j < LR2; ++j) {
      const uint32_t i = threadIdx.x + j * LNT;
      const E* src = X + (i < nx ? a0 + i : yoff + b0 + (i - nx));  // 32-bit offset, one 64-bit add
      if (i < nx + ny) tmp[j] = ldg_elem(src);
    }
#pragma unroll
    for (int j = 0; j < LR2; ++j) {
      const uint32_t i = threadIdx.x + j * LNT;
      if (i < nx + ny) s[pad<LPS>(i)] = tmp[j];
    }
  }
  __syncthreads();
  nx_out = nx;
  const int dd = threadIdx.x * LR2;
  const int tot = (int)(nx + ny);
  int cnt = 0;
  if (dd < tot) {
    const int NX = (int)nx, NY = (int)ny;
    int lo = dd > NY ? dd - NY : 0, hi = dd < NX ? dd : NX;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (before(s[pad<LPS>(mid)], s[pad<LPS>(NX + dd - 1 - mid)])) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = dd - lo;
    // unclamped cursors: past X reads Y's head, past Y the slot after the tile (never taken)
    E xa = s[pad<LPS>(ia)], yv = s[pad<LPS>(NX + ib)];
    cnt = min(LR2, tot - dd);
#pragma unroll
    for (int r = 0; r < LR2; ++r) {
      const bool takeA = sizeof(E) == 8 ? (bool)((ib >= NY) | ((ia < NX) & before(xa, yv)))  // no branch per step
                                        : (ib >= NY) || (ia < NX && before(xa, yv));
      v[r] = E::select(takeA, xa, yv);
      srcB[r] = !takeA;
      ia += takeA;
      ib += !takeA;
      const E nv = s[pad<LPS>(takeA ? ia : NX + ib)];
      xa = E::select(takeA, nv, xa);
      yv = E::select(takeA, yv, nv);
    }
  }
  return cnt;
}

// merge_tile over struct-of-arrays shared tiles (64-bit keys): keys in sk, indices in si,
// key compares only (LE: x goes first on ties, else y does); the taken element's index is
// loaded off the dependency chain.
template <bool LE, typename U, typename E>
__device__ __forceinline__ int merge_tile_soa(U* sk, uint32_t* si, const E* X, const E* Y, uint32_t d0,
                                              uint32_t d1, uint2 sp, U (&vk)[LR2], uint32_t (&vi)[LR2],
                                              bool (&srcB)[LR2], uint32_t& nx_out) {
  const uint32_t a0 = sp.x, a1 = sp.y;
  const uint32_t b0 = d0 - a0, b1 = d1 - a1;
  const uint32_t nx = a1 - a0, ny = b1 - b0;
  const uint32_t yoff = (uint32_t)(Y - X);  // Y follows X in the same buffer (runs / blocks)
  {
    E tmp[LR2];
#pragma unroll
    for (int j = 0; j < LR2; ++j) {
      const uint32_t i = threadIdx.x + j * LNT;
      const E* src = X + (i < nx ? a0 + i : yoff + b0 + (i - nx));  // 32-bit offset, one 64-bit add
      if (i < nx + ny) tmp[j] = ldg_elem(src);
    }
#pragma unroll
    for (int j = 0; j < LR2; ++j) {
      const uint32_t i = threadIdx.x + j * LNT;
      if (i < nx + ny) {
        sk[pad<LPS>(i)] = tmp[j].key();
        si[pad<LPS>(i)] = tmp[j].idx();
      }
    }
  }
  __syncthreads();
  nx_out = nx;
  auto before = [](U x, U y) { return LE ? x <= y : x < y; };
  const int dd = threadIdx.x * LR2;
  const int tot = (int)(nx + ny);
  int cnt = 0;
  if (dd < tot) {
    const int NX = (int)nx, NY = (int)ny;
    int lo = dd > NY ? dd - NY : 0, hi = dd < NX ? dd : NX;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (before(sk[pad<LPS>(mid)], sk[pad<LPS>(NX + dd - 1 - mid)])) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = dd - lo;
    U xa = sk[pad<LPS>(ia)], yv = sk[pad<LPS>(NX + ib)];  // unclamped, as in merge_tile
    cnt = min(LR2, tot - dd);
#pragma unroll
    for (int r = 0; r < LR2; ++r) {
      const bool takeA = (ib >= NY) || (ia < NX && before(xa, yv));
      vk[r] = takeA ? xa : yv;
      vi[r] = si[pad<LPS>(takeA ? ia : NX + ib)];
      srcB[r] = !takeA;
      ia += takeA;
      ib += !takeA;
      const U nv = sk[pad<LPS>(takeA ? ia : NX + ib)];
      xa = takeA ? nv : xa;
      yv = takeA ? yv : nv;
    }
  }
  return cnt;
}

// merge-path split of diagonal d over X[0,lx) and Y[0,ly) under `before(x, y)`
template <typename E, typename Before>
__device__ __forceinline__ uint32_t merge_split(const E* X, uint32_t lx, const E* Y, uint32_t ly, uint32_t d,
                                                Before before) {
  uint32_t lo = d > ly ? d - ly : 0, hi = d < lx ? d : lx;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (before(X[mid], Y[d - 1 - mid])) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- merge-path partitions: the (start, end) split of every merge tile, computed up front
// by one thread per tile so the merge kernels start streaming immediately ---------------
template <int DT, bool KO>
__global__ void ml_partition_pass(LargeGeom L, const Elem<typename Traits<DT>::U>* in_, uint2* splits, uint32_t run,
                                  uint64_t total) {
  using E = SortElem<typename Traits<DT>::U, KO>;
  const E* in = reinterpret_cast<const E*>(in_);
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= total) return;
  const uint32_t t = id % L.mtiles;
  const uint64_t rb = id / L.mtiles;                 // row * nb + b
  const uint32_t k = L.g.k;
  const uint32_t p0 = t * LQ;
  const uint32_t x0 = p0 / (2 * run) * (2 * run);
  const uint32_t lx = min(run, k - x0);
  const uint32_t y0 = x0 + lx;
  const uint32_t ly = y0 < k ? min(run, k - y0) : 0;
  const uint32_t d0 = p0 - x0, d1 = min(d0 + LQ, lx + ly);
  const E* X = in + rb * k + x0;
  const E* Y = in + rb * k + y0;
  auto before = [](const E& a, const E& c) { return E::less(a, c); };
  splits[id] = make_uint2(merge_split(X, lx, Y, ly, d0, before), merge_split(X, lx, Y, ly, d1, before));
}

template <int DT>
__global__ void ml_partition_units(LargeGeom L, const Elem<typename Traits<DT>::U>* S, uint2* splits,
                                   uint64_t total) {
  using E = Elem<typename Traits<DT>::U>;
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= total) return;
  const uint32_t t = id % L.tiles2;
  const uint64_t ug = id / L.tiles2;                 // row * units + u
  const uint64_t row = ug / L.g.units, u = ug % L.g.units;
  const uint32_t k = L.g.k;
  const E* A = S + (row * L.nb + u) * k;
  const E* B = A + k;
  const uint32_t d0 = t * LQ, d1 = min(d0 + LQ, L.nq);
  auto before = [](const E& a, const E& c) { return a.key() <= c.key(); };
  splits[id] = make_uint2(merge_split(A, k, B, k, d0, before), merge_split(A, k, B, k, d1, before));
}

// ---- phase 1b: one global merge pass (runs of length `run` within every block) --------
template <int DT, bool KO>
__global__ void __launch_bounds__(LNT) ml_merge_pass(LargeGeom L, const Elem<typename Traits<DT>::U>* in_,
                                                     Elem<typename Traits<DT>::U>* out_, uint32_t run,
                                                     const uint2* splits) {
  using U = typename Traits<DT>::U;
  using E = SortElem<U, KO>;
  const E* in = reinterpret_cast<const E*>(in_);
  E* out = reinterpret_cast<E*>(out_);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* s = reinterpret_cast<E*>(smem_raw);
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.mtiles;
  const uint32_t t = blockIdx.x % L.mtiles;
  const uint32_t k = L.g.k;
  const uint64_t base = (row * L.nb + b) * k;
  const uint32_t p0 = t * LQ;
  const uint32_t x0 = p0 / (2 * run) * (2 * run);
  const uint32_t lx = min(run, k - x0);
  const uint32_t y0 = x0 + lx;
  const uint32_t ly = y0 < k ? min(run, k - y0) : 0;
  const uint32_t d0 = p0 - x0;
  const uint32_t d1 = min(d0 + LQ, lx + ly);
  bool srcB[LR2];
  uint32_t nx;
  const uint2 sp = splits[(row * L.nb + b) * L.mtiles + t];
  const int dd = threadIdx.x * LR2;
  if constexpr (kSoa<U, KO>) {
    U* sk = reinterpret_cast<U*>(smem_raw);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + LQ + (LQ >> LPS) + 1);
    U vk[LR2];
    uint32_t vi[LR2];
    const int cnt = merge_tile_soa<false>(sk, si, in + base + x0, in + base + y0, d0, d1, sp, vk, vi, srcB, nx);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < LR2; ++r)
      if (r < cnt) {
        sk[pad<LPS>(dd + r)] = vk[r];
        si[pad<LPS>(dd + r)] = vi[r];
      }
    __syncthreads();
    Elem<U>* o = reinterpret_cast<Elem<U>*>(out + base + x0 + d0);
    for (uint32_t i = threadIdx.x; i < d1 - d0; i += LNT) store_elem(o + i, sk[pad<LPS>(i)], si[pad<LPS>(i)]);
  } else {
    auto before = [](const E& a, const E& c) { return E::less(a, c); };
    E v[LR2];
    const int cnt = merge_tile(s, in + base + x0, in + base + y0, d0, d1, sp, before, v, srcB, nx);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < LR2; ++r)
      if (r < cnt) s[pad<LPS>(dd + r)] = v[r];
    __syncthreads();
    E* o = out + base + x0 + d0;
    for (uint32_t i = threadIdx.x; i < d1 - d0; i += LNT) o[i] = s[pad<LPS>(i)];
  }
}

// ---- phase 2a: merge each pair (A = block u, B = block u+1) + live counts -------------
template <int DT>
__global__ void __launch_bounds__(LNT, sizeof(typename Traits<DT>::U) == 8 ? 3 : 4) ml_unit_merge(LargeGeom L, const Elem<typename Traits<DT>::U>* S,
                                                     typename Traits<DT>::U* mk, uint32_t* org, uint2* rab,
                                                     uint32_t* live, const uint2* splits) {
  using U = typename Traits<DT>::U;
  using E = Elem<U>;
  constexpr bool SOA = kSoa<U, true>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* s = reinterpret_cast<E*>(smem_raw);                                     // merge tile
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw + merge_tile_bytes<U, SOA>());  // [4][2][C]
  const uint64_t row = blockIdx.y;
  const uint64_t u = blockIdx.x / L.tiles2;
  const uint32_t t = blockIdx.x % L.tiles2;
  const uint32_t k = L.g.k;
  const E* A = S + (row * L.nb + u) * k;
  const E* B = A + k;
  const uint64_t ug = row * L.g.units + u;
  const uint32_t d0 = t * LQ, d1 = min(d0 + LQ, L.nq);
  const uint32_t C = L.C;
  for (uint32_t i = threadIdx.x; i < 8 * C; i += LNT) hist[i] = 0;
  U vk[LR2];
  uint32_t vi[LR2];
  bool srcB[LR2];
  uint32_t nx;
  const uint2 sp = splits[(row * L.g.units + u) * L.tiles2 + t];
  int cnt;
  if constexpr (SOA) {
    U* tk = reinterpret_cast<U*>(smem_raw);
    uint32_t* ti = reinterpret_cast<uint32_t*>(tk + LQ + (LQ >> LPS) + 1);
    cnt = merge_tile_soa<true>(tk, ti, A, B, d0, d1, sp, vk, vi, srcB, nx);  // A first on key ties
  } else {
    auto before = [](const E& a, const E& c) { return a.key() <= c.key(); };  // A first on key ties
    E v[LR2];
    cnt = merge_tile(s, A, B, d0, d1, sp, before, v, srcB, nx);
#pragma unroll
    for (int r = 0; r < LR2; ++r) {
      vk[r] = v[r].key();
      vi[r] = v[r].idx();
    }
  }
  const int dd = threadIdx.x * LR2;
  uint2* ro = rab + ug * (uint64_t)L.C * L.CL;
  __syncthreads();
  // staging: keys, then origins, both padded (pad<LPS>): a thread's LR2 consecutive slots
  // would otherwise put every other lane on the same bank (16-way conflicts)
  static_assert((sizeof(U) + 4) * (LQ + (LQ >> LPS)) <= merge_tile_bytes<U, SOA>(), "staging fits the merge tile");
  U* sk = reinterpret_cast<U*>(s);
  uint32_t* so = reinterpret_cast<uint32_t*>(sk + LQ + (LQ >> LPS));
#pragma unroll
  for (int r = 0; r < LR2; ++r) {
    if (r < cnt) {
      const uint32_t q = d0 + dd + r;
      const uint32_t idx = vi[r];
      sk[pad<LPS>(dd + r)] = vk[r];
      so[pad<LPS>(dd + r)] = idx | (srcB[r] ? 0x80000000u : 0u);
      uint2* slot = ro + ((idx & (L.CL - 1)) * C + (idx >> L.CLshift));  // transposed [t][c] (< C*CL: 32-bit)
      MF_ASSERT(idx < k && q < L.nq && (idx >> L.CLshift) < C);
      if (srcB[r]) slot->y = q; else slot->x = q;
      const uint32_t sw = (dd + r) >> 10;                   // superword within the tile
      MF_ASSERT(sw < 4);
      check_sptr(&hist[(sw * 2 + (srcB[r] ? 1 : 0)) * C + (idx >> L.CLshift)]);
      atomicAdd(&hist[(sw * 2 + (srcB[r] ? 1 : 0)) * C + (idx >> L.CLshift)], 1u);
    }
  }
  __syncthreads();
  U* mko = mk + ug * L.nqp + d0;
  uint32_t* oo = org + ug * L.nqp + d0;
  for (uint32_t i = threadIdx.x; i < d1 - d0; i += LNT) {
    mko[i] = sk[pad<LPS>(i)];
    oo[i] = so[pad<LPS>(i)];
  }
  // live count of each superword at every chunk start c: A elements with chunk >= c plus
  // B elements with chunk < c.  One warp per superword; lanes scan 32 chunks at a time.
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nsw = (d1 - d0 + 1023) / 1024;
  if (warp < nsw) {
    const uint32_t* hA = hist + (warp * 2) * C;
    const uint32_t* hB = hist + (warp * 2 + 1) * C;
    const uint32_t S = d0 / 1024 + warp;
    uint32_t totA = 0;
    for (uint32_t c = lane; c < C; c += 32) totA += hA[c];
    for (int o = 16; o; o >>= 1) totA += __shfl_xor_sync(0xFFFFFFFFu, totA, o);
    uint32_t preA = 0, preB = 0;  // exclusive prefixes over chunks < c0
    for (uint32_t c0 = 0; c0 < C; c0 += 32) {
      const uint32_t c = c0 + lane;
      const uint32_t a = c < C ? hA[c] : 0, bb = c < C ? hB[c] : 0;
      uint32_t ia = a, ib = bb;  // inclusive warp scans
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ta = __shfl_up_sync(0xFFFFFFFFu, ia, o), tb = __shfl_up_sync(0xFFFFFFFFu, ib, o);
        if (lane >= (uint32_t)o) { ia += ta; ib += tb; }
      }
      if (c < C) live[(ug * L.NS + S) * C + c] = (totA - (preA + ia - a)) + (preB + ib - bb);
      preA += __shfl_sync(0xFFFFFFFFu, ia, 31);
      preB += __shfl_sync(0xFFFFFFFFu, ib, 31);
    }
  }
}

// live bits of merged positions [32w, 32w+32) just before step i (output i).
// org = idx | isB << 31, and a position is live iff (A and idx >= i) or (B and idx < i),
// which is exactly "org - i has bit 31 clear": for A, org - i = idx - i underflows iff
// idx < i; for B, org - i = 2^31 + (idx - i) stays below 2^31 iff idx < i.  One subtract
// and one shift-or per position; positions past 2k are masked off.
__device__ __forceinline__ uint32_t live_word(const uint32_t* og, uint32_t w, uint32_t i, uint32_t nq) {
  uint32_t dead = 0;
  const uint4* v4 = reinterpret_cast<const uint4*>(og + w * 32);
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    const uint4 v = __ldg(v4 + j);
    dead = (dead << 1) | ((v.w - i) >> 31);
    dead = (dead << 1) | ((v.z - i) >> 31);
    dead = (dead << 1) | ((v.y - i) >> 31);
    dead = (dead << 1) | ((v.x - i) >> 31);
  }
  const uint32_t q0 = w * 32;
  const uint32_t valid = q0 + 32 <= nq ? 0xFFFFFFFFu : (q0 < nq ? (1u << (nq - q0)) - 1u : 0u);
  return ~dead & valid;
}

// ---- phase 2c: chunked walk -----------------------------------------------------------
// Thread id = ug*C + c walks chunk c of unit ug: outputs [c*CL, c*CL + CL).  Consecutive
// lanes take consecutive chunks, so the per-step Delete/Undelete targets (stored
// transposed, rab[t*C + c]) are read coalesced; outputs are gathered 8 steps at a time
// in shared memory and written back as 32-byte runs, four chunks per warp store.
template <int DT>
__global__ void __launch_bounds__(LNT) ml_walk(LargeGeom L, const typename Traits<DT>::U* mk, const uint32_t* org,
                                               const uint2* rab, const uint32_t* live, uint64_t total) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using TV = typename Tr::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  U* stage = reinterpret_cast<U*>(smem_raw) + warp * 32 * 9;    // [lane][step] with stride 9
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const Geom& g = L.g;
  const uint32_t k = g.k, h = g.h;
  uint64_t ug = 0, row = 0, u = 0;
  uint32_t c = 0, i0 = 0, i1 = 0;
  if (id < total) {
    ug = id / L.C;
    c = id % L.C;
    row = ug / g.units;
    u = ug % g.units;
    const uint64_t rem = g.keep - u * k;
    const uint32_t imax = rem < (uint64_t)k ? (uint32_t)rem : k;
    i0 = c * L.CL;
    i1 = min(imax, i0 + L.CL);
    if (i0 > i1) i0 = i1;
  }
  const bool active = i0 < i1;
  const uint32_t* og = org + ug * L.nqp;
  const U* mkg = mk + ug * L.nqp;
  const uint2* rb = rab + ug * (uint64_t)L.C * L.CL + c;      // step t at rb[t * C]
  TV* y = reinterpret_cast<TV*>(g.y) + row * g.ld_y + u * k + i0;

  // The cursor's neighbourhood is a 64-position window: words cw0 and cw0+1 of the live set.
  // When the cursor leaves it the window slides by one word (one live_word), so the cursor
  // sits mid-window afterwards and small back-and-forth moves never recompute a word.
  const uint32_t nwq = L.nqp / 32;                             // words per unit
  auto word = [&](uint32_t w, uint32_t i) -> uint32_t { return w < nwq ? live_word(og, w, i, L.nq) : 0u; };
  uint32_t p = 0, cw0 = 0;
  uint64_t win = 0;
  if (active) {
    // select: superword S with prefix(S) <= h < prefix(S+1) (prefix of the live counts,
    // read 8 superwords at a time), then the words inside it
    const uint32_t* cnt = live + ug * L.NS * L.C + c;          // stride C over superwords
    uint32_t acc = 0, S = 0;
    for (; S < L.NS; S += 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = S + j < L.NS ? __ldg(cnt + (uint64_t)(S + j) * L.C) : 0xFFFFFFFFu;
      uint32_t s8 = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) s8 += (S + j < L.NS) ? v[j] : 0;
      if (acc + s8 > h) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (acc + v[j] > h) { S += j; break; }
          acc += v[j];
        }
        break;
      }
      acc += s8;
    }
    uint32_t r = h - acc;
    uint32_t cw = S * 32, cb = 0;
    for (;; ++cw) {
      MF_ASSERT(cw < nwq);
      cb = live_word(og, cw, i0, L.nq);
      const uint32_t pc = __popc(cb);
      if (r < pc) break;
      r -= pc;
    }
    p = cw * 32 + __fns(cb, 0, (int)r + 1);
    cw0 = cw;
    win = (uint64_t)cb | ((uint64_t)word(cw + 1, i0) << 32);
  }
  const uint32_t my_n = active ? i1 - i0 : 0u;
  // Steps run in groups of 8.  The group's Delete/Undelete targets (rab) are loaded one group
  // ahead, and its 8 median keys are gathered into registers and staged after the group, so a
  // thread has up to 16 independent loads in flight instead of stalling on each step's two
  // (the kernel was bound by long-scoreboard stalls: 14 per issued instruction).
#ifndef MF_WALK_PREFETCH
#define MF_WALK_PREFETCH 1
#endif
  auto load_group = [&](uint32_t t0, uint2 (&ab)[8]) {
#pragma unroll
    for (uint32_t tt = 0; tt < 8; ++tt) {
      const uint32_t t = t0 + tt;
      ab[tt] = (t > 0 && t < my_n) ? __ldg(rb + (uint64_t)(t - 1) * L.C) : make_uint2(0u, 0u);
    }
  };
  uint2 abn[8];
  if (MF_WALK_PREFETCH) load_group(0, abn);
  for (uint32_t t0 = 0; t0 < L.CL; t0 += 8) {
    uint2 abc[8];
    U kv[8];
    if (MF_WALK_PREFETCH) {
#pragma unroll
      for (int j = 0; j < 8; ++j) abc[j] = abn[j];
      if (t0 + 8 < L.CL) load_group(t0 + 8, abn);
    }
#pragma unroll
    for (uint32_t tt = 0; tt < 8; ++tt) {
      const uint32_t t = t0 + tt;
      const uint32_t i = i0 + t;
      kv[tt] = 0;
      if (t < my_n) {
        if (t > 0) {
          const uint2 ab = MF_WALK_PREFETCH ? abc[tt] : __ldg(rb + (uint64_t)(t - 1) * L.C);
          const uint32_t a = ab.x, b = ab.y;
          MF_ASSERT(a < L.nq && b < L.nq);
          const uint32_t base = cw0 * 32;
          const uint32_t oa = a - base, ob = b - base, off = p - base;   // window offsets
          win &= ~(oa < 64 ? 1ull << oa : 0ull);
          win |= ob < 64 ? 1ull << ob : 0ull;
          const bool up = a <= p && b > p;
          const bool down = a >= p && b < p;
          uint64_t m = sel(up, (uint64_t)(win & (0xFFFFFFFFFFFFFFFEull << off)), (uint64_t)(win & ((1ull << off) - 1ull)));
          if ((up || down) && m == 0) {  // slide the window one word at a time (rare)
            do {
              if (up) {
                ++cw0;
                win = (win >> 32) | ((uint64_t)word(cw0 + 1, i) << 32);
                m = win & 0xFFFFFFFF00000000ull;
              } else {
                --cw0;
                win = (win << 32) | word(cw0, i);
                m = win & 0xFFFFFFFFull;
              }
            } while (m == 0);
          }
          p = sel(up, cw0 * 32 + __ffsll((long long)m) - 1, sel(down, cw0 * 32 + 63 - __clzll((long long)m), p));
        }
        MF_ASSERT(p < L.nq);
        kv[tt] = __ldg(mkg + p);
      }
    }
#pragma unroll
    for (uint32_t tt = 0; tt < 8; ++tt) stage[lane * 9 + tt] = kv[tt];
    __syncwarp();
    // 8 outputs of 4 chunks per warp store: lane l -> chunk 4j + l/8, step l%8
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
      const uint32_t src = 4 * j + (lane >> 3), st = lane & 7;
      const uint32_t jn = __shfl_sync(0xFFFFFFFFu, my_n, src);
      TV* yj = reinterpret_cast<TV*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(y), src));
      if (t0 + st < jn) {
        MF_ASSERT(yj + t0 + st < reinterpret_cast<TV*>(g.y) + (uint64_t)(g.rows - 1) * g.ld_y + g.keep);
        yj[t0 + st] = Tr::dec(stage[src * 9 + st]);
      }
    }
    __syncwarp();
    if (__all_sync(0xFFFFFFFFu, t0 + 8 >= my_n)) break;
  }
}

}  // namespace mf
