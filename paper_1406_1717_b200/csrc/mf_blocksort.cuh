// mf_blocksort.cuh -- segmented block sort primitives (phase 1, piecewise_sort,
// filter.hpp:41-54) shared by the medium-k and large-k pipelines.
//
// Elements are (key, index) pairs in one total order (mf_sortnet.cuh), so every sort
// here is stable in the reference's sense.  A group of NT threads sorts NT*R elements:
// each thread sorts R in registers (odd-even merge network), then log2(NT) merge-path
// levels run through shared memory.  Shared arrays use the padded index
// p + (p >> PS), which makes the blocked per-thread writes bank-conflict free for
// 8-byte elements (PS = 5 when R >= 32, else 4).
#pragma once
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

template <int PS>
__device__ __forceinline__ int pad(int p) { return p + (p >> PS); }

template <int R>
constexpr int pad_shift() { return R >= 32 ? 5 : 4; }

// Merge-path levels: runs of length run0, 2*run0, ... < run_end (a power-of-two
// multiple of R) inside s[b0 .. b0 + NT*R), NT threads, thread `tid` produces the R
// outputs [tid*R, tid*R + R) of its merged pair.  On entry s holds sorted runs of
// length run0; v is scratch.  CTA = true syncs the CTA, else the warp.
struct SyncWarp { __device__ __forceinline__ void operator()() const { __syncwarp(); } };
struct SyncCta { __device__ __forceinline__ void operator()() const { __syncthreads(); } };
// named barrier over `count` threads (a team of warps), id != 0
struct SyncTeam {
  uint32_t id, count;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
  // barrier that also ORs a predicate over the team
  __device__ __forceinline__ bool any(bool v) const {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.or.pred p, %2, %3, q;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r) : "r"((uint32_t)v), "r"(id), "r"(count) : "memory");
    return r != 0;
  }
};

template <typename E, int R, int PS, typename Sync>
__device__ __forceinline__ void merge_levels_s(E* s, int b0, int tid, int run0, int run_end, E (&v)[R], Sync sync) {
#pragma unroll 1
  for (int run = run0; run < run_end; run *= 2) {
    const int gl = (2 * run) / R;                // threads per merged run
    const int j = tid & (gl - 1);
    const int xb = b0 + (tid / gl) * (2 * run);  // X = [xb, xb+run), Y = [xb+run, xb+2run)
    const int yb0 = xb + run;
    const int d = j * R;
    int lo = d > run ? d - run : 0, hi = d < run ? d : run;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (E::less(s[pad<PS>(xb + mid)], s[pad<PS>(yb0 + d - 1 - mid)])) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d - lo;
    // An exhausted side's cursor reads the element after its run: Y's head for X, the next
    // run pair's head (or the tile's spare slot) for Y -- always inside the buffer, and never
    // taken (the bounds tests decide), so no clamps are needed.
    E xa = s[pad<PS>(xb + ia)], yv = s[pad<PS>(yb0 + ib)];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      // branch-free step: one shared load refills whichever side was consumed
      // 8-byte elements (32-bit keys): bitwise, so no branch per step (c5 50.7 -> 49.0 ms); with 64-bit
      // keys the short-circuit form measured faster (c1 0.0466 against 0.0498 ms)
      const bool takeA = sizeof(E) == 8 ? (bool)((ib >= run) | ((ia < run) & E::less(xa, yv)))
                                        : (ib >= run) || (ia < run && E::less(xa, yv));
      v[r] = E::select(takeA, xa, yv);
      ia += takeA;
      ib += !takeA;
      const E nv = s[pad<PS>(takeA ? xb + ia : yb0 + ib)];
      xa = E::select(takeA, nv, xa);
      yv = E::select(takeA, yv, nv);
    }
    sync();
#pragma unroll
    for (int r = 0; r < R; ++r) s[pad<PS>(xb + d + r)] = v[r];
    sync();
  }
}

template <typename E, int R, int PS, bool CTA>
__device__ __forceinline__ void merge_levels(E* s, int b0, int tid, int run0, int run_end, E (&v)[R]) {
  if constexpr (CTA) merge_levels_s<E, R, PS>(s, b0, tid, run0, run_end, v, SyncCta{});
  else merge_levels_s<E, R, PS>(s, b0, tid, run0, run_end, v, SyncWarp{});
}

// Warp sort of 32*R register-loaded elements (v, any distribution over lanes) into
// s[b0 .. b0 + 32R) (padded layout, sorted ascending).
// Bitonic merge levels in registers: after it, every group of G = 2^levels lanes holds one
// sorted run of G*R elements (lane offset o of the group holds elements [o*R, o*R + R)).
// Each level is a mirror stage (element i against element G*R-1-i of the partner lane
// o ^ (G-1)), then half-cleaners: across lanes for distances >= R (partner o ^ (d/R)) and
// inside the lane below that.  No shared memory, no searches; the elements are totally
// ordered, so the result equals any other sort's.
template <typename E, int R, int LEVELS>
__device__ __forceinline__ void warp_bitonic_levels(E (&v)[R], uint32_t lane) {
#pragma unroll
  for (int m = 1; m <= LEVELS; ++m) {
    const int G = 1 << m;
    {  // mirror stage
      const bool lower = (lane & (G >> 1)) == 0;
      E t[R];
#pragma unroll
      for (int r = 0; r < R; ++r) t[r] = shfl_xor(v[R - 1 - r], G - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool lt = E::less_full(v[r], t[r]);
        v[r] = E::select(lt == lower, v[r], t[r]);
      }
    }
#pragma unroll
    for (int dl = G >> 2; dl >= 1; dl >>= 1) {  // cross-lane half-cleaners, lane distance dl
      const bool lower = (lane & dl) == 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const E p = shfl_xor(v[r], dl);
        const bool lt = E::less_full(v[r], p);
        v[r] = E::select(lt == lower, v[r], p);
      }
    }
#pragma unroll
    for (int d = R >> 1; d >= 1; d >>= 1) {      // in-lane half-cleaners
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & d) == 0) E::cswap(v[r], v[r + d]);
    }
  }
}

// Warp sort: register network per lane, then BLV register bitonic levels (shuffles; 5 =
// the whole warp), then shared-memory merge-path levels up to 32R.  16-byte elements skip
// the bitonic levels (measured: no gain for 64-bit keys).
template <typename E, int R, int PS, int BLV>
__device__ __forceinline__ void warp_sort_regs(E (&v)[R], E* s, int b0, uint32_t lane) {
  constexpr int BL = sizeof(E) > 8 ? 0 : BLV;
  sort_regs<R>(v);
  warp_bitonic_levels<E, R, BL>(v, lane);
#pragma unroll
  for (int r = 0; r < R; ++r) s[pad<PS>(b0 + lane * R + r)] = v[r];
  __syncwarp();
  merge_levels<E, R, PS, false>(s, b0, lane, R << BL, 32 * R, v);
}

// Merge-path levels over the SoA arrays (runs run0, 2*run0, ... < run_end); thread `tid`
// produces outputs [j*R, j*R + R) of its merged run pair.  Key compares are strict in both
// the search and the steps, so the lanes' ranges tile each merged run exactly.
// With `aos` set, the last level writes its outputs as 16-byte {key, index} elements into
// `aos` (which may overlap sk/si: every read of the level precedes the write-back barrier).
template <int R, int PS, typename Sync, typename EA = KElem64>
__device__ __forceinline__ void merge_levels_soa(uint64_t* sk, uint32_t* si, int b0, int tid, int run0, int run_end,
                                                 uint64_t (&vk)[R], uint32_t (&vi)[R], Sync sync,
                                                 EA* aos = nullptr) {
#pragma unroll 1
  for (int run = run0; run < run_end; run *= 2) {
    const int gl = (2 * run) / R;                // threads per merged run
    const int j = tid & (gl - 1);
    const int xb = b0 + (tid / gl) * (2 * run);  // X = [xb, xb+run), Y = [xb+run, xb+2run)
    const int yb0 = xb + run;
    const int d = j * R;
    int lo = d > run ? d - run : 0, hi = d < run ? d : run;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sk[pad<PS>(xb + mid)] < sk[pad<PS>(yb0 + d - 1 - mid)]) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d - lo;
    uint64_t xa = sk[pad<PS>(xb + ia)], yv = sk[pad<PS>(yb0 + ib)];  // unclamped: see merge_levels_s
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool takeA = (ib >= run) || (ia < run && xa < yv);
      vk[r] = takeA ? xa : yv;
      vi[r] = si[pad<PS>(takeA ? xb + ia : yb0 + ib)];   // off the chain
      ia += takeA;
      ib += !takeA;
      const uint64_t nv = sk[pad<PS>(takeA ? xb + ia : yb0 + ib)];
      xa = takeA ? nv : xa;
      yv = takeA ? yv : nv;
    }
    sync();
    if (aos && 2 * run >= run_end) {
#pragma unroll
      for (int r = 0; r < R; ++r) aos[pad<PS>(xb + d + r)] = EA::make(vk[r], vi[r]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sk[pad<PS>(xb + d + r)] = vk[r];
        si[pad<PS>(xb + d + r)] = vi[r];
      }
    }
    sync();
  }
}

// Warp-wide stable compaction of the elements with idx < k to the front of sb[0, NS).
// Needed after a key-ordered sort (KElem) when the block holds samples whose key is the
// all-ones padding key (real maxima or the reference's +INF padding, filter.hpp:28-36):
// the slot fillers past k share that key and may have landed among the first k sorted
// positions.  Fillers only ever sit in the all-ones run at the end, so everything before
// it stays where it is.  Positions past k are left as they are (nothing reads them).
template <typename E, int PS>
__device__ __noinline__ void compact_block(E* sb, int NS, uint32_t k, uint32_t lane) {
  uint32_t base = 0;
  for (int p0 = 0; p0 < NS; p0 += 32) {
    const E e = sb[pad<PS>(p0 + (int)lane)];
    const bool real = e.idx() < k;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, real);
    __syncwarp();
    MF_ASSERT(!real || base + __popc(bal & ((1u << lane) - 1u)) < k);
    if (real) sb[pad<PS>((int)(base + __popc(bal & ((1u << lane) - 1u))))] = e;
    base += __popc(bal);
    __syncwarp();
  }
}

// Team sort: WP warps sort one block of 32*RS*WP slots.  Warp `sub` of the team holds the
// elements [sub*32*RS, (sub+1)*32*RS) (element e = sub*32*RS + lane + 32r), sorts them
// into its part of sb, then the team merges the WP sorted parts.  Slots e >= k hold the
// padding value; with key-ordered elements they are moved behind the k real ones.
template <int DT, int RS, int WP, int BL, typename E>
__device__ __forceinline__ void team_sort_raw(E* sb, const typename Traits<DT>::T (&raw)[RS], uint32_t k,
                                              uint32_t sub, uint32_t lane, SyncTeam bar) {
  using TV = typename Traits<DT>::T;
  constexpr int PS = pad_shift<RS>();
  const TV padv = (TV)(~(std::make_unsigned_t<TV>)0 >> 1);
  E v[RS];
  bool maxkey = false;  // a slot e < k carries the padding key
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const uint32_t e = sub * 32 * RS + lane + 32 * r;
    v[r] = E::make(Traits<DT>::enc(raw[r]), e);
    maxkey |= e < k && raw[r] == padv;
  }
#ifndef MF_MED_SOA64
#define MF_MED_SOA64 1  // one-warp 64-bit key sorts merge through SoA scratch (keys, indices) inside the slot
#endif
  if constexpr (MF_MED_SOA64 && WP == 1 && std::is_same_v<E, KElem64> && RS < 32) {
    // register network, then the merge levels over struct-of-arrays scratch laid in the slot's
    // own bytes (12 bytes per element fit in its 16); the last level writes the slot's
    // {key, index} elements
    constexpr int NSL = 32 * RS + ((32 * RS) >> PS) + 1;
    static_assert(12 * NSL <= 16 * NSL, "SoA scratch fits the slot");
    sort_regs<RS>(v);
    uint64_t* sk = reinterpret_cast<uint64_t*>(sb);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + NSL);
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int p = pad<PS>((int)(lane * RS + r));
      sk[p] = v[r].k;
      si[p] = v[r].i;
    }
    __syncwarp();
    uint64_t vk[RS];
    uint32_t vi[RS];
    merge_levels_soa<RS, PS>(sk, si, 0, (int)lane, RS, 32 * RS, vk, vi, SyncWarp{}, sb);
  } else {
    warp_sort_regs<E, RS, PS, BL>(v, sb, sub * 32 * RS, lane);
  }
  if constexpr (WP > 1) {
    maxkey = bar.any(maxkey);
    merge_levels_s<E, RS, PS>(sb, 0, sub * 32 + lane, 32 * RS, 32 * RS * WP, v, bar);
  } else {
    maxkey = __any_sync(0xFFFFFFFFu, maxkey);
  }
  if constexpr (!E::kFull) {
    if (maxkey && sub == 0) compact_block<E, PS>(sb, 32 * RS * WP, k, lane);
  }
}

// ---- key-only team sort (32-bit keys) -------------------------------------------------
// The sorting network moves bare 32-bit keys: a compare-exchange is two min/max ops
// (VIMNMX), a cross-lane stage one shuffle and a lane-directed min/max, where carrying the
// index would cost a compare and four selects per exchange on the ALU pipe (the medium
// kernel's limiter).  The permutation is recovered afterwards: each element's sorted
// position is the number of smaller keys (a branch-free lower-bound search in the sorted
// keys of every warp of the team) plus a tie slot claimed with a shared atomic, so equal
// keys take distinct consecutive positions in some order -- the key order the medium
// kernel needs (mf_sortnet.cuh, KElem32).  Slot fillers (e >= k) claim nothing, so the k
// real elements (virtual +INF padding included, filter.hpp:28-36) fill positions [0, k).
struct KeyU32 {
  uint32_t v;
  __device__ __forceinline__ static void cswap(KeyU32& x, KeyU32& y) {
    const uint32_t lo = min(x.v, y.v), hi = max(x.v, y.v);
    x.v = lo; y.v = hi;
  }
};

// register bitonic levels on bare keys (layout as warp_bitonic_levels)
template <int R, int LEVELS>
__device__ __forceinline__ void warp_bitonic_keys(KeyU32 (&v)[R], uint32_t lane) {
#pragma unroll
  for (int m = 1; m <= LEVELS; ++m) {
    const int G = 1 << m;
    {  // mirror stage
      const bool lower = (lane & (G >> 1)) == 0;
      uint32_t t[R];
#pragma unroll
      for (int r = 0; r < R; ++r) t[r] = __shfl_xor_sync(0xFFFFFFFFu, v[R - 1 - r].v, G - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) v[r].v = lower ? min(v[r].v, t[r]) : max(v[r].v, t[r]);
    }
#pragma unroll
    for (int dl = G >> 2; dl >= 1; dl >>= 1) {  // cross-lane half-cleaners
      const bool lower = (lane & dl) == 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t p = __shfl_xor_sync(0xFFFFFFFFu, v[r].v, dl);
        v[r].v = lower ? min(v[r].v, p) : max(v[r].v, p);
      }
    }
#pragma unroll
    for (int d = R >> 1; d >= 1; d >>= 1) {      // in-lane half-cleaners
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & d) == 0) KeyU32::cswap(v[r], v[r + d]);
    }
  }
}

// number of keys < x in the sorted run s[pad5(0 .. N)), N a power of two (branch-free).
// The search walks the padded index P = pad5(p) directly: at a step of size st the
// position p is a multiple of 2*st, so the probe p + st - 1 sits at P + pad5(st - 1) (an
// immediate load offset) and the step adds pad5(st) -- one compare and one predicated add
// per step.  p is recovered at the end: P = 33a + b (b < 32) gives p = P - (P + 1) / 33.
constexpr uint32_t cpad5(uint32_t q) { return q + (q >> 5); }
// Plain (reorderable) shared load by shared-window address.  It is ordered after a barrier
// only through its address: callers add order_token(), read after the barrier.
__device__ __forceinline__ uint32_t lds32(uint32_t saddr) {
  check_saddr(saddr, 4);
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint32_t order_token() {
  uint32_t z;
  asm volatile("mov.u32 %0, 0;" : "=r"(z)::"memory");
  return z;
}

template <int N>
__device__ __forceinline__ uint32_t lower_bound_keys(uint32_t s0, uint32_t x) {
  uint32_t q = s0;  // s0: shared-window byte address of the run  // shared-window byte address of padded position P
#pragma unroll
  for (uint32_t st = N / 2; st >= 1; st >>= 1)
    if (lds32(q + 4 * cpad5(st - 1)) < x) q += 4 * cpad5(st);
  const uint32_t P = (q - s0) >> 2;
  return P - (P + 1) / 33 + (lds32(q) < x ? 1u : 0u);
}

// the same count with 4-way steps: three independent loads per step, half the dependent chain
template <int N>
__device__ __forceinline__ uint32_t lower_bound_keys4(uint32_t s0, uint32_t x) {
  uint32_t q = s0;
#pragma unroll
  for (uint32_t st = N / 4; st >= 1; st >>= 2) {
    const uint32_t c = (lds32(q + 4 * cpad5(st - 1)) < x ? 1u : 0u) + (lds32(q + 4 * cpad5(2 * st - 1)) < x ? 1u : 0u) +
                       (lds32(q + 4 * cpad5(3 * st - 1)) < x ? 1u : 0u);
    const uint32_t a = c * st;
    q += 4 * (st >= 16 ? a + (a >> 5) : a);
  }
  if constexpr ((__builtin_ctz(N) & 1) != 0)
    if (lds32(q) < x) q += 4;
  const uint32_t P = (q - s0) >> 2;
  return P - (P + 1) / 33 + (lds32(q) < x ? 1u : 0u);
}

#ifndef MF_LB4_MIN
#define MF_LB4_MIN 2048  // smallest run searched with 4-way steps.  Round 1 (latency-bound): 4-way at 1024 keys, k = 1023
                         // 1.70 -> 1.64 ms.  Round 2: the kernel is bound by shared-memory wavefronts (75 % of peak), and the
                         // binary search issues 11 loads per key instead of 16: k = 1023 1.335 -> 1.245 ms
#endif
template <int N>
__device__ __forceinline__ uint32_t lower_bound_sel(uint32_t s, uint32_t x) {
  if constexpr (N >= MF_LB4_MIN) return lower_bound_keys4<N>(s, x);
  else return lower_bound_keys<N>(s, x);
}

#ifndef MF_TEAM_KEYMERGE
#define MF_TEAM_KEYMERGE 1
#endif
// Team sort of one block into sb (KElem32, key order): WP warps, warp `sub` holds the
// elements e = sub*32*RS + lane + 32r.  sk: team scratch of 2*WP*(32*RS + RS) words; cnt: team
// scratch of WP*32*RS words.  Position k of sb gets the merge sentinel.
// The element's index is stored as ridx = (e % SRr) * CHr + e / SRr (the walk's transposed
// [step][chunk] slot of e; SRr = 0 stores e itself).  The sentinel's low word is 0xFFFFFFFF
// when a real element of the block has the all-ones key (it would tie with the sentinel),
// else 0xFFFFFFFE; both have bit 31 set (KElem32::merge_le).
template <int DT, int RS, int WP, int PS, int SRr = 0, int CHr = 1>
__device__ __forceinline__ void team_sort_keys(KElem32* sb, const typename Traits<DT>::T (&raw)[RS], uint32_t k,
                                               uint32_t sub, uint32_t lane, SyncTeam bar, uint32_t* sk,
                                               uint32_t* cnt) {
  constexpr int NS = 32 * RS;             // keys per warp
  constexpr int SKW = NS + NS / 32;       // padded words per warp
  constexpr uint32_t BS = WP * NS;
  const uint32_t tl = sub * 32 + lane;
  uint32_t key[RS];
  KeyU32 v[RS];
  bool maxkey = false;                    // a real element (e < k) has the all-ones key
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    key[r] = Traits<DT>::enc(raw[r]);
    v[r].v = key[r];
    maxkey |= sub * NS + lane + 32 * r < k && key[r] == 0xFFFFFFFFu;
  }
  sort_regs<RS>(v);
  warp_bitonic_keys<RS, 5>(v, lane);
  uint32_t* mine = sk + sub * SKW;
#pragma unroll
  for (int r = 0; r < RS; ++r) mine[pad<5>((int)lane * RS + r)] = v[r].v;
  // `ties`: two equal keys below the all-ones key sit next to each other in the sorted block,
  // or a real element has the all-ones key (it ties with the slot fillers).  Without ties every
  // real element's position is its count of smaller keys, and the tie-slot counters are skipped.
#ifndef MF_TIE_SKIP
#define MF_TIE_SKIP 1
#endif
  bool ties = maxkey || !MF_TIE_SKIP;
  // two warps: one merge-path level joins their runs, so each element searches once
  constexpr bool MERGE = WP == 2 && MF_TEAM_KEYMERGE;
  const uint32_t* srch = sk;
  if constexpr (MERGE) {
    bar();
    uint32_t* skm = sk + 2 * SKW;
    const uint32_t* X = sk;
    const uint32_t* Y = sk + SKW;
    const int d = tl * RS;
    int lo = d > NS ? d - NS : 0, hi = d < NS ? d : NS;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (X[pad<5>(mid)] <= Y[pad<5>(d - 1 - mid)]) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d - lo;
    uint32_t xa = X[pad<5>(min(ia, NS - 1))], yb = Y[pad<5>(min(ib, NS - 1))];
    uint32_t o[RS];
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const bool takeA = (ib >= NS) | ((ia < NS) & (xa <= yb));
      o[r] = takeA ? xa : yb;
      ia += takeA;
      ib += !takeA;
      const uint32_t nv = takeA ? X[pad<5>(min(ia, NS - 1))] : Y[pad<5>(min(ib, NS - 1))];
      xa = takeA ? nv : xa;
      yb = takeA ? yb : nv;
    }
#pragma unroll
    for (int r = 0; r < RS; ++r) skm[pad<5>(d + r)] = o[r];
    // (two-warp teams always count tie slots: detecting ties across the merged run measured
    // slower than the counters it saves, k = 1023 1.318 -> 1.338 ms)
    ties = true;
    bar();
    srch = skm;
  } else if constexpr (WP == 1) {
    const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, v[0].v, 1);
#pragma unroll
    for (int r = 0; r + 1 < RS; ++r) ties |= v[r].v == v[r + 1].v && v[r].v != 0xFFFFFFFFu;
    ties |= lane < 31 && v[RS - 1].v == nxt && nxt != 0xFFFFFFFFu;
    ties = __any_sync(0xFFFFFFFFu, ties);
    __syncwarp();                           // the stores to `mine` before the searches
  } else {
    ties = bar.any(true);                   // separate runs per warp: always count tie slots
  }
  if (ties) {
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    for (uint32_t i = tl; i < (uint32_t)(WP * NS / 4); i += 32 * WP) c4[i] = make_uint4(0, 0, 0, 0);
    if constexpr (WP > 1) bar(); else __syncwarp();
  }
  // shared-window addresses of the sorted runs, tied to the barrier above
  const uint32_t tok = order_token();
  const uint32_t srch0 = (uint32_t)__cvta_generic_to_shared(srch) + tok;
  uint32_t pos[RS];
#pragma unroll
  for (int r = 0; r < RS; ++r) {  // independent searches (no branch: they interleave)
    pos[r] = 0;
    if constexpr (MERGE) {
      pos[r] = lower_bound_sel<2 * NS>(srch0, key[r]);
    } else {
#pragma unroll
      for (int w = 0; w < WP; ++w) pos[r] += lower_bound_sel<NS>(srch0 + 4 * w * SKW, key[r]);
    }
  }
  // tie slots and the scatter, branch-free: slot fillers count on cnt[BS-1] (never a real
  // element's rank, which is < k <= BS-1) and write the unused slot position BS
  if (ties) {
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const uint32_t e = sub * NS + lane + 32 * r;
      const bool real = e < k;
      MF_ASSERT(!real || pos[r] < k);
      check_sptr(&cnt[real ? pos[r] : BS - 1]);
      const uint32_t t = atomicAdd(&cnt[real ? pos[r] : BS - 1], 1u);
      uint32_t ri = e;
      if constexpr (SRr > 0) ri = (e & (SRr - 1)) * CHr + e / SRr;
      MF_ASSERT(!real || pos[r] + t < k);
      check_sptr(&sb[pad<PS>((int)(real ? pos[r] + t : BS))]);
      sb[pad<PS>((int)(real ? pos[r] + t : BS))] = KElem32::make(key[r], ri);
    }
  } else {
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const uint32_t e = sub * NS + lane + 32 * r;
      const bool real = e < k;
      uint32_t ri = e;
      if constexpr (SRr > 0) ri = (e & (SRr - 1)) * CHr + e / SRr;
      MF_ASSERT(!real || pos[r] < k);
      check_sptr(&sb[pad<PS>((int)(real ? pos[r] : BS))]);
      sb[pad<PS>((int)(real ? pos[r] : BS))] = KElem32::make(key[r], ri);
    }
  }
  // the scratch is reused by the next sort
  if constexpr (WP > 1) maxkey = bar.any(maxkey); else maxkey = __any_sync(0xFFFFFFFFu, maxkey);
  if (tl == 0) {
    KElem32 s = KElem32::sentinel();
    if (!maxkey) s.v &= ~1ull;
    sb[pad<PS>((int)k)] = s;
  }
}

template <typename TV, int RS, int WP>
__device__ __forceinline__ void team_load_block(TV (&raw)[RS], const TV* x, uint64_t n, uint32_t k, uint64_t blk,
                                                uint32_t sub, uint32_t lane) {
  const TV padv = (TV)(~(std::make_unsigned_t<TV>)0 >> 1);
  const uint64_t b0 = blk * k;
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const uint32_t e = sub * 32 * RS + lane + 32 * r;
    const uint64_t gp = b0 + e;
    raw[r] = (e < k && gp < n) ? __ldg(x + gp) : padv;
  }
}

}  // namespace mf
