// mf_medium.cuh -- fused median filter for medium windows (32 < k <= 32*R):
// one warp per block pair, both phases in one pass over HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155).
//   pad_to_blocks (filter.hpp:28-36)  -> virtual padding in the warp's loader
//   piecewise_sort (filter.hpp:41-54) -> warp block sort: every lane sorts R
//        (key, index) elements in registers (odd-even merge network), then five
//        warp-wide merge-path passes in shared memory produce the sorted block.
//   run_postprocess (filter.hpp:64-106) + Block (block.hpp:24-146) -> per pair:
//     (1) merge path over sorted A and sorted B gives every element its position in
//         the pair's merged order, so Peek(A) vs Peek(B) comparisons become position
//         comparisons (ties between A and B can go either way: the emitted value is
//         the same);
//     (2) the k steps of the pair are cut into 32 chunks of R steps, one per lane.
//         The state before any step is a pure function of (pi_A, pi_B, step)
//         (Eq. 4 / Lemma 1): the live set is {A: idx >= i} u
//         {B: idx < i}, and the median is its (h+1)-th smallest element.  Each
//         lane gets that live set as a 2k-bit row of the merged order (built for all
//         lanes at once by an XOR prefix over the per-chunk toggle sets), selects
//         its first median, then walks its R steps with Delete(A,i)/Undelete(B,i)
//         as bit clear/set and the median cursor moved to the next/previous live bit
//         -- the dancing-links list and the pair of cursors of Figure 7 folded into
//         one cursor over the merged order.  The word holding the cursor is cached in
//         a register, so most steps touch no shared memory on the dependency chain.
//
// Persistent CTAs own a contiguous range of tiles (W pairs each); the sorted blocks
// live in a ring of W+1 slots, so the block shared by two consecutive tiles is loaded
// and sorted once.  Each input block is read from HBM once per CTA range and every
// median is written once, coalesced.
#pragma once
#include "mf_common.cuh"
#include "mf_blocksort.cuh"
#include "mf_sortnet.cuh"

namespace mf {

#ifndef MF_MEDIUM_KEYORD_MAXR
#define MF_MEDIUM_KEYORD_MAXR 16  // largest R sorted with key-ordered elements (R = 32: measured slower)
#endif

#ifndef MF_WALK_WT
#define MF_WALK_WT 1  // how the walk keeps the rows current.  1: every Delete/Undelete is written through (two
                      // atomics per step on random words of the lane's row).  2: only the three words around
                      // the chunk's first cursor word are written through; a word outside that window keeps its
                      // chunk-start value and is rebuilt by replaying the chunk's steps when the cursor enters
                      // it -- fewer shared-memory wavefronts, but measured slower (k = 1023 1.229 -> 1.306 ms,
                      // k = 255 0.927 -> 0.964 ms: the window tests cost more than the atomics).  0: no
                      // write-through at all (k = 1023 1.41 -> 1.84 ms)
#endif
#ifndef MF_ROWS_PAD
#define MF_ROWS_PAD 1
#endif

template <int DT, int R, int W, int WP = 1>
struct MediumCfg {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  // key-ordered elements: ties in any order (mf_sortnet.cuh)
#ifndef MF_KEYSORT
#define MF_KEYSORT 1  // 32-bit keys: key-only network + rank recovery (team_sort_keys)
#endif
#ifndef MF_KS_R16
#define MF_KS_R16 1  // R = 16 (k = 257..511) on the key-only sort too: with 4 teams per CTA and 4 CTAs per SM,
                     // k = 257 / 385 / 511 2.30 / 1.58 / 1.20 -> 1.90 / 1.32 / 1.04 ms (round 1 had it 2 % slower)
#endif
  static constexpr bool KS = MF_KEYSORT && sizeof(U) == 4 && (R != 16 || MF_KS_R16);
  using E = std::conditional_t<(KS || R <= MF_MEDIUM_KEYORD_MAXR), typename KeyOrd<U>::E, Elem<U>>;
  static constexpr int BS = 32 * R;        // block slot capacity (>= k)
  static constexpr int NW = 2 * R;         // words per merged row (2k bits <= 64R)
  static constexpr int RS = R / WP;        // elements per lane in the team block sort
#ifndef MF_WALK_WARPS_R32
#define MF_WALK_WARPS_R32 2  // warps of a 2-warp team that walk at R = 32 (1: 32 chunks, half the rows; measured 12 % slower at equal occupancy)
#endif
  static constexpr int WW = (R == 32 && WP == 2) ? MF_WALK_WARPS_R32 : WP;  // walking warps
  static constexpr int CH = 32 * WW;       // walk chunks per pair (one per walking lane)
  static constexpr int SR = R / WW;        // steps per chunk
#ifndef MF_BL_TEAM
#define MF_BL_TEAM 3  // register bitonic levels of the warp sorts in 2-warp teams (experiments)
#endif
#ifndef MF_BL_WARP
#define MF_BL_WARP 5  // ... in 1-warp teams (5: the whole block in registers)
#endif
  static constexpr int BL = WP > 1 ? MF_BL_TEAM : MF_BL_WARP;
  // padded element index: blocked per-lane writes hit distinct banks (8-byte elements);
  // the key sort scatters, so its slots are unpadded (the merge walks byte addresses)
#ifndef MF_KS_PAD_MINR
#define MF_KS_PAD_MINR 32  // smallest R whose key-sorted slots are padded one element per 16, so the lanes' merge
                           // cursors (16 elements apart at R = 32) hit distinct banks.  With the kernel bound by
                           // shared-memory wavefronts, R = 32 gains 2 % (k = 1023 1.344 -> 1.318 ms); R = 8 loses
                           // 2.6 % (k = 255; the padded cursor arithmetic costs more than its conflicts did)
#endif
  static constexpr int PS = KS ? (R >= MF_KS_PAD_MINR ? 4 : 30) : pad_shift<RS>();
  static constexpr int SLOT = BS + (BS >> PS) + 1;
  static constexpr size_t sz_sorted = (sizeof(E) * SLOT * (W + 1) + 15) / 16 * 16;
  // merged pos -> key (MK), or -> (isB, sorted pos) where the keys would cost occupancy
#ifndef MF_MK_MAXR
#define MF_MK_MAXR 0  // largest R whose merged keys are stored (measured: the extra smem costs more occupancy than the saved load)
#endif
  static constexpr bool MK = R <= MF_MK_MAXR;
  // (u16 entries: 2*BS positions plus two pad entries per team lane, src_slot)
  static constexpr size_t sz_src = MK ? sizeof(U) * 2 * BS : sizeof(uint16_t) * (2 * BS + 2 * 32 * WP);
  static constexpr size_t sz_rab = sizeof(uint32_t) * BS;      // RA | RB << 16, transposed [t][lane]
  static constexpr int NWP = MF_ROWS_PAD ? NW + 1 : NW;  // row stride in words (rows[L][w] at L*NWP + w)
  static constexpr size_t sz_rows_bits = sizeof(uint32_t) * NWP * CH;
  static constexpr size_t sz_stage = sizeof(U) * (BS + BS / 32 + 1);
  // the rows area doubles as the output staging area after the walk
  // ... and as the key sort's scratch (runs, merged run) before the pair phase
  static constexpr size_t sz_scratch = sizeof(uint32_t) * 2 * WP * (32 * RS + RS);
  static constexpr size_t sz_rows0 = sz_rows_bits > sz_stage ? sz_rows_bits : sz_stage;
  static constexpr size_t sz_rows = (((KS && sz_scratch > sz_rows0) ? sz_scratch : sz_rows0) + 15) / 16 * 16;
  // A-side bits per word, only where two team lanes share a word (2R/WP < 32 positions per lane)
  static constexpr size_t sz_abits = 2 * R / WP == 32 ? 0 : sizeof(uint32_t) * NW;
  static constexpr size_t sz_warp = (sz_src + sz_rab + sz_rows + sz_abits + 15) / 16 * 16;  // per team
  static constexpr size_t smem = sz_sorted + W * sz_warp;
};

// Row L of the per-chunk live sets, word w.  Padded layout (MF_ROWS_PAD): rows[L][w] at
// L*NWP + w with an odd stride NWP, so the prefix pass (lane = word, loop over L: immediate
// offsets) and the walk (lane = L, data-dependent word) are both bank-spread.  Otherwise
// rows[L][w] at w*CH + (L ^ (w & (CH-1))).
template <int CH, int NWP>
__device__ __forceinline__ uint32_t row_addr(uint32_t L, uint32_t w) {
  if constexpr (MF_ROWS_PAD) return L * NWP + w;
  else return w * CH + (L ^ (w & (CH - 1)));
}

// A "team" of WP warps owns one block pair: it sorts the pair's B block together (WP warp
// sorts + a team merge level), runs the pair merge and the XOR prefix with 32*WP lanes,
// and its first warp walks the 32 chunks.  WP = 2 for the largest blocks halves the
// dependent merge chains that bound them at low occupancy.
#ifndef MF_MINB_R8
#define MF_MINB_R8 8  // resident CTAs the R = 8 kernel is compiled for (64-register cap with 4 teams per CTA)
#endif
#ifndef MF_MINB_R4
#define MF_MINB_R4 4  // (64 registers: k = 101 1.65 -> 1.45 ms)
#endif
#ifndef MF_MINB_R16
#define MF_MINB_R16 4  // 128 registers: 4 CTAs of 4 teams per SM (168 registers and 3 CTAs: k = 511 1.08 ms; 4: 1.04 ms)
#endif
#ifndef MF_MINB_R32
#define MF_MINB_R32 3  // 3 CTAs of 128 threads per SM is what shared memory allows: keep ptxas under 170 registers
                       // (unbounded it took 197 after a small change, 2 CTAs/SM, k = 1023 1.25 -> 1.42 ms)
#endif
#ifndef MF_MINB_R4_WIDE
#define MF_MINB_R4_WIDE 6  // R = 4, 64-bit keys (config 1): 6 CTAs of 4 teams per SM (80 registers); 4 CTAs (103
                           // registers): c1 0.0542 -> 0.0474 ms
#endif
template <int DT, int R> struct MediumMinBlocks {
  static constexpr bool wide = sizeof(typename Traits<DT>::U) == 8;
  static constexpr int value = R == 32 ? MF_MINB_R32 : R == 16 ? MF_MINB_R16 : R == 8 ? MF_MINB_R8
                               : R == 4 ? (wide ? MF_MINB_R4_WIDE : MF_MINB_R4) : 0;
};

// src[] holds one u16 entry per merged position q, in position order with two pad entries
// (one word) after each team lane's run of PL positions: the runs then start an odd number
// of words apart, so the merge's per-lane stores are conflict-free, and the walk's reads --
// every lane's cursor sits near the pair's median position -- fall on neighbouring words.
// (The earlier [q % PL][q / PL] layout put those reads on one bank: 13 wavefronts per load
// at k = 1023, 8.5 % of the kernel's shared-memory wavefronts.)
template <int PL, int TL>
__device__ __forceinline__ uint32_t src_slot(uint32_t q) {
  return q + 2 * (q >> __builtin_ctz(PL));
}

#ifndef MF_MERGE_NC32
#define MF_MERGE_NC32 1  // independent pair-merge chains per lane for R = 32 (measured: 2 is 7 % slower)
#endif
#ifndef MF_MERGE_NC8
#define MF_MERGE_NC8 1
#endif
template <int R> struct MergeChains { static constexpr int value = R == 32 ? MF_MERGE_NC32 : R == 8 ? MF_MERGE_NC8 : 1; };

template <int DT, int R, int W, int WP>
__global__ void __launch_bounds__(32 * W * WP, MediumMinBlocks<DT, R>::value) mf_medium_kernel(Geom g, uint64_t tiles_per_row, uint64_t total_tiles) {
  using C = MediumCfg<DT, R, W, WP>;
  using Tr = typename C::Tr;
  using U = typename C::U;
  using E = typename C::E;
  using TV = typename Tr::T;
  constexpr int NW = C::NW, PS = C::PS, SLOT = C::SLOT, RS = C::RS, CH = C::CH, SR = C::SR;
  constexpr int TL = 32 * WP;        // team lanes
  extern __shared__ __align__(16) unsigned char smem[];
  E* ring = reinterpret_cast<E*>(smem);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t team = warp / WP, sub = warp % WP, tl = sub * 32 + lane;
  const SyncTeam tbar{1 + team, (uint32_t)TL};
  auto team_sync = [&]() { if constexpr (WP > 1) tbar(); else __syncwarp(); };
  unsigned char* ws = smem + C::sz_sorted + team * C::sz_warp;
  uint16_t* src = reinterpret_cast<uint16_t*>(ws);
  uint32_t* rab = reinterpret_cast<uint32_t*>(ws + C::sz_src);
  uint32_t* rows = reinterpret_cast<uint32_t*>(ws + C::sz_src + C::sz_rab);
  uint32_t* abits = reinterpret_cast<uint32_t*>(ws + C::sz_src + C::sz_rab + C::sz_rows);
  U* ost = reinterpret_cast<U*>(rows);  // output staging reuses the rows area after the walk

  const uint32_t k = g.k, h = g.h;
  const uint32_t nq = 2 * k, nw = (nq + 31) / 32;
  // contiguous tile range of this CTA
  const uint64_t t_begin = total_tiles * blockIdx.x / gridDim.x;
  const uint64_t t_end = total_tiles * (blockIdx.x + 1) / gridDim.x;
  uint32_t base = 0;                 // physical slot of logical slot 0
  uint64_t prev_row = ~0ull, prev_tile = ~0ull;
  TV pre[RS];                        // this lane's part of the team's next block, loaded during phase 2
  bool have_pre = false;

  // sorted block into a ring slot; sorted position k holds a sentinel above every element,
  // so the pair merge needs no bounds checks
  auto sort_block = [&](E* sb, const TV (&raw)[RS]) {
    if constexpr (C::KS) {
      team_sort_keys<DT, RS, WP, PS, SR, CH>(sb, raw, k, sub, lane, tbar, rows, rab);
    } else {
      team_sort_raw<DT, RS, WP, C::BL>(sb, raw, k, sub, lane, tbar);
      if (sub == 0 && lane == 0) sb[pad<PS>(k)] = E::sentinel();
    }
  };

  // Pair merge of the key-sorted slots A, B (KS): team lane owns merged positions
  // [d, d + PL).  The cursors are shared-window byte addresses; elements carry ridx (the
  // transposed rab slot of their index, team_sort_keys), so the chunk is ridx % CH and the
  // rab entry 2*ridx + side.  Unless B holds a real all-ones key (its sentinel's bit 0),
  // plain key compares order the pair: A's sentinel then never ties with a live B element.
  // src[q] gets the byte offset of the key of merged position q.  Returns the A bits.
  auto merge_keys = [&](const auto* A, const auto* B, int d, uint32_t w0, uint32_t bo) -> uint32_t {
    constexpr int PL = 2 * R / WP;
    const uint32_t ringS = (uint32_t)__cvta_generic_to_shared(ring) + order_token();
    const uint32_t offA = (uint32_t)(reinterpret_cast<const unsigned char*>(A) - reinterpret_cast<const unsigned char*>(ring));
    const uint32_t offB = (uint32_t)(reinterpret_cast<const unsigned char*>(B) - reinterpret_cast<const unsigned char*>(ring));
    const int K = (int)k;
    const bool exact = (B[pad<PS>(K)].v & 1ull) != 0;
    uint16_t* rab16 = reinterpret_cast<uint16_t*>(rab);
    auto padk = [](uint32_t p) -> uint32_t { return p + (p >> PS); };  // slot of sorted position p
    auto run = [&](auto ex) -> uint32_t {
      constexpr bool EX = decltype(ex)::value;
      auto le = [&](uint2 a, uint2 b) -> bool {
        if constexpr (EX) {
          return (((uint64_t)a.y << 32) | (a.x & 0x80000000u)) <= (((uint64_t)b.y << 32) | (b.x & 0x80000000u));
        } else {
          return a.y <= b.y;
        }
      };
      auto at = [&](uint32_t off) -> uint2 {
        check_saddr(ringS + off, 8);
        uint2 v;
        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(ringS + off));
        return v;
      };
      // NC independent merge chains per lane (sub-ranges of PLC positions), interleaved
      // step by step: the dependent shared-load chain of each is NC times shorter
      constexpr int NC = MergeChains<R>::value, PLC = PL / NC;
      uint32_t lo[NC], hi[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const uint32_t dj = d + j * PLC;
        lo[j] = dj > (uint32_t)K ? dj - K : 0;
        hi[j] = dj < (uint32_t)K ? dj : K;
      }
      const int niter = 32 - __clz(K);          // >= ceil(log2(K + 1)) halvings
      for (int it = 0; it < niter; ++it) {
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const uint32_t dj = d + j * PLC;
          const bool act = lo[j] < hi[j];
          const uint32_t mid = (lo[j] + hi[j]) >> 1;
          const bool g = le(at(offA + 8 * padk(act ? mid : 0u)), at(offB + 8 * padk(act ? dj - 1 - mid : 0u)));
          lo[j] = act && g ? mid + 1 : lo[j];
          hi[j] = act && !g ? mid : hi[j];
        }
      }
      const uint32_t limA = offA + 8 * padk(K);
      const uint32_t sbase = (uint32_t)d + 2 * tl;  // src_slot(d): this lane's run of PL positions
      uint32_t relA[NC], relB[NC], bit[NC], am = 0;
      uint32_t ia[NC], ib[NC];                  // cursors (sorted positions) of the padded path
      uint2 ea[NC], eb[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const uint32_t dj = d + j * PLC;
        ia[j] = lo[j];
        ib[j] = dj - lo[j];
        if (dj >= nq) ia[j] = ib[j] = K;         // chains past the pair: both sides exhausted
        relA[j] = offA + 8 * padk(ia[j]);
        relB[j] = offB + 8 * padk(ib[j]);
        ea[j] = at(relA[j]);
        eb[j] = at(relB[j]);
        bit[j] = 1u << (bo + j * PLC);
      }
#pragma unroll 8
      for (int r = 0; r < PLC; ++r) {
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const uint32_t q = d + j * PLC + r;
          const bool takeA = le(ea[j], eb[j]);
          // past the pair both sides are the sentinel: ridx clamps to BS-1 >= k, whose rab
          // entry and row bits beyond 2k nobody reads -- no branch
          const uint32_t ri = min(takeA ? ea[j].x : eb[j].x, (uint32_t)C::BS - 1);
          MF_ASSERT(w0 < (uint32_t)C::NWP && src_slot<PL, 32 * WP>(q) < 2u * C::BS + 2u * TL);
          check_sptr(&rows[row_addr<CH, C::NWP>(ri & (CH - 1), w0)]);
          check_sptr(&rab16[2 * ri + 1]);
          atomicOr(&rows[row_addr<CH, C::NWP>(ri & (CH - 1), w0)], bit[j]);
          src[sbase + j * PLC + r] = (uint16_t)((takeA ? relA[j] : relB[j]) + 4);  // = src_slot(q)
          rab16[2 * ri + (takeA ? 0 : 1)] = (uint16_t)q;
          am |= takeA ? bit[j] : 0u;
          bit[j] <<= 1;
          uint2 nv;
          if constexpr (PS < 30) {  // padded slots: the next address from the advanced cursor
            ia[j] += takeA ? 1u : 0u;
            ib[j] += takeA ? 0u : 1u;
            // only A can pass its sentinel (ties go to A); B never passes it
            const uint32_t a = (takeA ? offA : offB) + 8 * padk(takeA ? min(ia[j], (uint32_t)K) : ib[j]);
            relA[j] = takeA ? a : relA[j];
            relB[j] = takeA ? relB[j] : a;
            nv = at(a);
          } else {
            relA[j] += takeA ? 8u : 0u;
            relB[j] += takeA ? 0u : 8u;
            nv = at(takeA ? min(relA[j], limA) : relB[j]);
          }
          ea[j] = takeA ? nv : ea[j];
          eb[j] = takeA ? eb[j] : nv;
        }
      }
      return am;
    };
    uint32_t am = exact ? run(std::true_type{}) : run(std::false_type{});
    if (d + PL > (int)nq) am &= d < (int)nq ? ((1u << (nq - d)) - 1u) << bo : 0u;
    return am;
  };

  // (row, tile-in-row) of the current tile, advanced incrementally (no 64-bit division per tile)
  uint64_t row = t_begin / tiles_per_row, tr = t_begin % tiles_per_row;
  for (uint64_t t = t_begin; t < t_end; ++t) {
    uint64_t nrow = row, ntr = tr + 1;
    if (ntr == tiles_per_row) { ntr = 0; ++nrow; }
    const uint64_t u0 = tr * W;
    const TV* __restrict__ x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
    TV* __restrict__ y = reinterpret_cast<TV*>(g.y) + row * g.ld_y;
    const bool carry = (row == prev_row && tr == prev_tile + 1);
    // ring arithmetic with one conditional subtract (base and logical are <= W)
    if (carry) { base += W; base -= base > (uint32_t)W ? W + 1 : 0; }
    auto slot = [&](uint32_t logical) {
      uint32_t b = base + logical;
      b -= b > (uint32_t)W ? W + 1 : 0;
      return ring + b * SLOT;
    };

    // ---------------- phase 1: team block sorts ----------------
    if (!carry && team == 0) {
      TV raw0[RS];
      team_load_block<TV, RS, WP>(raw0, x, g.n, k, u0, sub, lane);
      sort_block(slot(0), raw0);
    }
    if (!have_pre) team_load_block<TV, RS, WP>(pre, x, g.n, k, u0 + team + 1, sub, lane);
    sort_block(slot(team + 1), pre);
    __syncthreads();
    // prefetch this team's block of the next tile; it lands while phase 2 runs (large
    // blocks only: for small R the extra registers cost more occupancy than they hide)
    have_pre = R >= 16 && t + 1 < t_end;
    if (have_pre) {
      team_load_block<TV, RS, WP>(pre, reinterpret_cast<const TV*>(g.x) + nrow * g.ld_x, g.n, k,
                                  ntr * W + team + 1, sub, lane);
    }

    // ---------------- phase 2: per-pair postprocess ----------------
    const uint64_t u = u0 + team;
    if (u < g.units) {
      const uint64_t rem = g.keep - u * k;
      const uint32_t imax = rem < (uint64_t)k ? (uint32_t)rem : k;
      const E* A = slot(team);
      const E* B = slot(team + 1);

      constexpr int PL = 2 * R / WP;             // merged positions per team lane (divides 32)
      constexpr bool OWN = PL == 32;             // each lane owns one whole word of every row
      {
        uint4* r4 = reinterpret_cast<uint4*>(rows);
        for (uint32_t i = tl; i < (C::NWP * CH + 3) / 4; i += TL) r4[i] = make_uint4(0, 0, 0, 0);
        if constexpr (!OWN)
          for (uint32_t w = tl; w < NW; w += TL) abits[w] = 0;
      }
      team_sync();

      // merge path: team lane owns merged positions [tl*PL, tl*PL + PL), all inside word
      // w0 = d/32 of every row; branch-free steps
      const int d = tl * PL;
      const uint32_t w0 = (uint32_t)d >> 5, bo = (uint32_t)d & 31;
      uint32_t amask = 0;                        // A-side bits of this lane's positions (word w0)
      if constexpr (C::KS) {
        amask = merge_keys(A, B, d, w0, bo);
      } else {
        // merge path in the blocks' sort order, A before B on ties (E::merge_le); the
        // search and the steps use the same order, so the lanes' ranges tile [0, 2k).
        // Both blocks end in a sentinel at position k, so no step needs a bounds check.
        const int K = (int)k;
        int lo = d > K ? d - K : 0, hi = d < K ? d : K;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (E::merge_le(A[pad<PS>(mid)], B[pad<PS>(d - 1 - mid)])) lo = mid + 1; else hi = mid;
        }
        uint32_t ia = lo, ib = d - lo;
        if (d >= (int)nq) ia = ib = K;             // lanes past the pair: both sides exhausted
        E ea = A[pad<PS>(ia)], eb = B[pad<PS>(ib)];
        uint16_t* rab16 = reinterpret_cast<uint16_t*>(rab);
        constexpr int LSR = __builtin_ctz(SR);
#pragma unroll 8
        for (int r = 0; r < PL; ++r) {
          const uint32_t q = d + r;
          const bool takeA = E::merge_le(ea, eb);
          const E w = E::select(takeA, ea, eb);
          // past the pair (q >= 2k) both sides are the sentinel: its index clamps to slot
          // BS-1 >= k, whose rab entry and row bits beyond 2k nobody reads -- no branch
          const uint32_t idx = min(w.idx(), (uint32_t)C::BS - 1);
          const uint32_t c = idx >> LSR;         // owning team lane (chunk) of this element
          const uint32_t bit = 1u << (bo + r);
          atomicOr(&rows[row_addr<CH, C::NWP>(c, w0)], bit);
          if constexpr (C::MK) reinterpret_cast<U*>(src)[q] = w.key();
          else src[(uint32_t)d + 2 * tl + r] = (uint16_t)sel(takeA, ia, 0x8000u | ib);  // = src_slot(q)
          rab16[2 * ((idx & (SR - 1)) * CH + c) + (takeA ? 0 : 1)] = (uint16_t)q;
          amask |= takeA ? bit : 0u;
          ia += takeA;
          ib += !takeA;
          const E nv = (takeA ? A : B)[pad<PS>(min(sel(takeA, ia, ib), (uint32_t)K))];
          ea = E::select(takeA, nv, ea);
          eb = E::select(takeA, eb, nv);
        }
        if (d + PL > (int)nq) amask &= d < (int)nq ? ((1u << (nq - d)) - 1u) << bo : 0u;
      }
      if constexpr (!OWN)
        if (d < (int)nq) atomicOr(&abits[w0], amask);
      // XOR prefix over chunks: row_L = A_bits ^ (toggles of chunks < L).  A lane that owns
      // its word wrote every toggle of it itself, so it needs no barrier before its prefix.
      auto prefix = [&](uint32_t w, uint32_t acc) {
#pragma unroll 8
        for (uint32_t L = 0; L < (uint32_t)CH; ++L) {
          const uint32_t a = row_addr<CH, C::NWP>(L, w);
          const uint32_t dlt = rows[a];
          rows[a] = acc;
          acc ^= dlt;
        }
      };
      if constexpr (OWN) {
        if (w0 < nw) prefix(w0, amask);
      } else {
        team_sync();
        for (uint32_t w = tl; w < nw; w += TL) prefix(w, abits[w]);
      }
      team_sync();

      {
        const uint32_t ringK = (uint32_t)__cvta_generic_to_shared(ring);
        auto key_at = [&](uint32_t p) -> U {
          if constexpr (C::KS) {
            uint32_t v;
            MF_ASSERT(p < nq && src_slot<PL, TL>(p) < 2u * C::BS + 2u * TL);
            check_saddr(ringK + src[src_slot<PL, TL>(p)], 4);
            asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ringK + src[src_slot<PL, TL>(p)]));
            return (U)v;
          } else if constexpr (C::MK) {
            return reinterpret_cast<const U*>(src)[p];
          } else {
            const uint32_t s = src[src_slot<PL, TL>(p)];
            const E* blk = (s & 0x8000u) ? B : A;   // one load from the selected block
            return blk[pad<PS>(s & 0x7FFFu)].key();
          }
        };

        // walk: team lane L emits outputs [L*SR, L*SR + SR) of this unit
        const uint32_t i0 = tl * SR;
        U out[SR];
        if (i0 < imax) {
          // select the (h+1)-th live position of row_L, G independent words at a time
#ifndef MF_SEL_G_SMALL
#define MF_SEL_G_SMALL 1
#endif
#ifndef MF_SEL_G_LARGE
#define MF_SEL_G_LARGE 4
#endif
          constexpr int G = R >= 16 ? MF_SEL_G_LARGE : MF_SEL_G_SMALL;
          uint32_t cnt = 0, cw = 0, cb = 0;
          for (;; cw += G) {
            uint32_t wv[G], pc[G], sg = 0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
              wv[j] = rows[row_addr<CH, C::NWP>(tl, G > 1 ? min(cw + j, nw - 1) : cw)];
              pc[j] = (G == 1 || cw + j < nw) ? __popc(wv[j]) : 0u;
              sg += pc[j];
            }
            if (cnt + sg > h) {
#pragma unroll
              for (int j = 0; j < G - 1; ++j) {
                if (cnt + pc[0] > h) break;
                cnt += pc[0];
                ++cw;
                pc[0] = pc[j + 1];
                wv[0] = wv[j + 1];
              }
              cb = wv[0];
              break;
            }
            cnt += sg;
          }
          uint32_t p = cw * 32 + __fns(cb, 0, (int)(h - cnt) + 1);
          const uint32_t cw0 = cw;  // the written-through window is [cw0 - 1, cw0 + 1] (MF_WALK_WT = 2)
          (void)cw0;
          out[0] = key_at(p);
#pragma unroll
          for (int t = 1; t < SR; ++t) {
            if (i0 + t < imax) {
              const uint32_t ab = rab[(t - 1) * CH + tl];
              const uint32_t a = ab & 0xFFFF, b = ab >> 16;
              MF_ASSERT(a < nq && b < nq && tl < (uint32_t)CH);
              const uint32_t ba = 1u << (a & 31), bb = 1u << (b & 31);
              // Delete(A, i-1) and Undelete(B, i-1) on the cached cursor word; with MF_WALK_WT
              // also written through to the row (fire-and-forget atomics), else the row keeps its
              // chunk-start value and a word the cursor moves into is rebuilt from it and the
              // chunk's earlier steps (rare)
#if MF_WALK_WT == 1
              atomicAnd(&rows[row_addr<CH, C::NWP>(tl, a >> 5)], ~ba);
              atomicOr(&rows[row_addr<CH, C::NWP>(tl, b >> 5)], bb);
#elif MF_WALK_WT == 2
              if ((a >> 5) + 1 - cw0 <= 2u) atomicAnd(&rows[row_addr<CH, C::NWP>(tl, a >> 5)], ~ba);
              if ((b >> 5) + 1 - cw0 <= 2u) atomicOr(&rows[row_addr<CH, C::NWP>(tl, b >> 5)], bb);
#endif
              cb = sel((a >> 5) == cw, cb & ~ba, cb);
              cb = sel((b >> 5) == cw, cb | bb, cb);
              // the cursor moves up when the deletion is at or below it and the insertion above
              const bool up = a <= p && b > p;
              const bool down = a >= p && b < p;
              const uint32_t sh = p & 31;
              const uint32_t mu = cb & (0xFFFFFFFEu << sh);
              const uint32_t md = cb & ((1u << sh) - 1u);
              uint32_t m = sel(up, mu, md);
              if ((up || down) && m == 0) {  // the next live position is in another word (rare)
                const int dir = up ? 1 : -1;
                do {
                  cw += dir;
                  MF_ASSERT(cw < nw);
                  cb = rows[row_addr<CH, C::NWP>(tl, cw)];
#if MF_WALK_WT != 1
#pragma unroll 1
                  for (int tt = 1; tt <= (MF_WALK_WT == 2 && cw + 1 - cw0 <= 2u ? 0 : t); ++tt) {  // replay this chunk's steps so far on word cw
                    const uint32_t ab2 = rab[(tt - 1) * CH + tl];
                    const uint32_t a2 = ab2 & 0xFFFF, b2 = ab2 >> 16;
                    cb = sel((a2 >> 5) == cw, cb & ~(1u << (a2 & 31)), cb);
                    cb = sel((b2 >> 5) == cw, cb | (1u << (b2 & 31)), cb);
                  }
#endif
                  m = cb;
                } while (m == 0);
              }
              p = sel(up, cw * 32 + __ffs(m) - 1, sel(down, cw * 32 + 31 - __clz(m), p));
              out[t] = key_at(p);
            }
          }
        }
        team_sync();  // rows are dead: reuse them as the output staging area
        // a chunk's SR (<= 32, a power of two) outputs share one 32-group, so its padded
        // staging offset is one base plus the step
        const uint32_t ob = i0 + (i0 >> 5);
#pragma unroll
        for (int t = 0; t < SR; ++t)
          if (i0 + t < imax) {
            check_sptr(&ost[ob + t]);
            ost[ob + t] = out[t];
          }
        team_sync();
        TV* yo = y + u * k + tl;
        MF_ASSERT(u * k + imax <= g.keep);
        // team lane tl stores outputs tl + TL*j: fixed strides, so unrolled loads and stores
        // take immediate offsets
        const U* os = ost + tl + (tl >> 5);
#pragma unroll
        for (int j = 0; j < RS; ++j)
          if (tl + (uint32_t)(TL * j) < imax) yo[TL * j] = Tr::dec(os[(TL + WP) * j]);
      }
    }
    prev_row = row;
    prev_tile = tr;
    row = nrow;
    tr = ntr;
    __syncthreads();  // the ring slots are reused by the next tile
  }
}

}  // namespace mf
