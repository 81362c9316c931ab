// mf_medium.cuh -- fused median filter for medium windows (32 < k <= 32*R):
// one warp per block pair, both phases in one pass over HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155).
//   pad_to_blocks (filter.hpp:28-36)  -> virtual padding in the warp's loader
//   piecewise_sort (filter.hpp:41-54) -> warp block sort: every lane sorts R
//        (key, index) elements in registers (odd-even merge network), then five
//        warp-wide merge-path passes in shared memory produce the sorted block.
//   run_postprocess (filter.hpp:64-106) + Block (block.hpp:24-146) -> per pair:
//     (1) merge path over sorted A and sorted B (A wins ties: PAPER.md §6.3 "the
//         elements of A are considered to be smaller", filter.hpp:92-93) gives every
//         element its position in the pair's merged order, so Peek(A) vs Peek(B)
//         comparisons become position comparisons;
//     (2) the k steps of the pair are cut into 32 chunks of R steps, one per lane.
//         The state before any step is a pure function of (pi_A, pi_B, step)
//         (Eq. 4 / Lemma 1): the live set is {A: idx >= i} u
//         {B: idx < i}, and the median is its (h+1)-th smallest element.  Each
//         lane gets that live set as a 2k-bit row of the merged order (built for all
//         lanes at once by an XOR prefix over the per-chunk toggle sets), selects
//         its first median, then walks its R steps with Delete(A,i)/Undelete(B,i)
//         as bit clear/set and the median cursor moved by next/prev live bit --
//         the dancing-links list and the pair of cursors of Figure 7 folded into one
//         cursor over the merged order.
// Each block is read from HBM once per warp that needs it and every median is
// written once, coalesced.
#pragma once
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

template <int DT, int R, int W>
struct MediumCfg {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using E = Elem<U>;
  static constexpr int BS = 32 * R;        // block slot (>= k)
  static constexpr int NW = 2 * R;         // words per merged row (2k bits <= 64R)
  // per-CTA layout
  static constexpr size_t sz_sorted = sizeof(E) * BS * (W + 1);
  static constexpr size_t sz_mk = sizeof(U) * 2 * BS;         // merged keys
  static constexpr size_t sz_rab = sizeof(uint32_t) * BS;     // RA | RB << 16, transposed
  static constexpr size_t sz_rows = sizeof(uint32_t) * NW * 32;
  static constexpr size_t sz_abits = sizeof(uint32_t) * NW;
  static constexpr size_t sz_out = sizeof(U) * BS;
  static constexpr size_t sz_warp = sz_mk + sz_rab + sz_rows + sz_abits + sz_out;
  static constexpr size_t smem = sz_sorted + W * sz_warp;
};

// rows[L][w] lives at w*32 + (L ^ (w & 31)): the prefix pass (lane = word, loop
// over L) and the walk (lane = L, data-dependent word) are both bank-spread.
__device__ __forceinline__ uint32_t row_addr(uint32_t L, uint32_t w) { return w * 32 + (L ^ (w & 31)); }

template <int DT, int R, int W>
__global__ void __launch_bounds__(32 * W) mf_medium_kernel(Geom g) {
  using C = MediumCfg<DT, R, W>;
  using Tr = typename C::Tr;
  using U = typename C::U;
  using E = typename C::E;
  using TV = typename Tr::T;
  constexpr int BS = C::BS, NW = C::NW;
  extern __shared__ __align__(16) unsigned char smem[];
  E* sorted = reinterpret_cast<E*>(smem);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ws = smem + C::sz_sorted + warp * C::sz_warp;
  U* mk = reinterpret_cast<U*>(ws);
  uint32_t* rab = reinterpret_cast<uint32_t*>(ws + C::sz_mk);
  uint32_t* rows = reinterpret_cast<uint32_t*>(ws + C::sz_mk + C::sz_rab);
  uint32_t* abits = rows + NW * 32;
  U* ost = reinterpret_cast<U*>(ws + C::sz_mk + C::sz_rab + C::sz_rows + C::sz_abits);

  const uint32_t k = g.k, h = g.h;
  const uint64_t row = blockIdx.y;
  const uint64_t u0 = (uint64_t)blockIdx.x * W;
  const TV* __restrict__ x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  TV* __restrict__ y = reinterpret_cast<TV*>(g.y) + row * g.ld_y;

  // ---------------- phase 1: warp block sort ----------------
  auto sort_block = [&](uint32_t slot) {
    E* sb = sorted + slot * BS;
    const uint64_t blk = u0 + slot;
    E v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t e = lane + 32 * r;            // coalesced across the warp
      const uint64_t gp = blk * k + e;
      const U key = (e < k && gp < g.n) ? Tr::enc(x[gp]) : UMax<U>::v;
      v[r] = E::make(key, e);                      // padding: (UMAX, e) sorts last
    }
    sort_regs<R>(v);
#pragma unroll
    for (int r = 0; r < R; ++r) sb[lane * R + r] = v[r];
    __syncwarp();
#pragma unroll 1
    for (int run = R; run < BS; run *= 2) {
      const uint32_t gl = (2 * run) / R;           // lanes per merged run
      const uint32_t j = lane & (gl - 1);
      const E* X = sb + (lane / gl) * (2 * run);
      const E* Y = X + run;
      const int d = j * R;
      int lo = d > run ? d - run : 0, hi = d < run ? d : run;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (E::less(X[mid], Y[d - 1 - mid])) lo = mid + 1; else hi = mid;
      }
      int ia = lo, ib = d - lo;
      E xa = X[ia < run ? ia : run - 1], yb = Y[ib < run ? ib : run - 1];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool takeA = (ib >= run) || (ia < run && E::less(xa, yb));
        v[r] = takeA ? xa : yb;
        if (takeA) { ++ia; xa = X[ia < run ? ia : run - 1]; }
        else { ++ib; yb = Y[ib < run ? ib : run - 1]; }
      }
      __syncwarp();
      E* out = const_cast<E*>(X) + d;
#pragma unroll
      for (int r = 0; r < R; ++r) out[r] = v[r];
      __syncwarp();
    }
  };
  sort_block(warp + 1);
  if (warp == 0) sort_block(0);
  __syncthreads();

  // ---------------- phase 2: per-pair postprocess ----------------
  const uint64_t u = u0 + warp;
  if (u >= g.units) return;
  const uint64_t rem = g.keep - u * k;
  const uint32_t imax = rem < (uint64_t)k ? (uint32_t)rem : k;
  const E* A = sorted + warp * BS;
  const E* B = A + BS;
  const uint32_t nq = 2 * k;                 // merged positions
  const uint32_t nw = (nq + 31) / 32;

  for (uint32_t i = lane; i < NW * 32; i += 32) rows[i] = 0;
  for (uint32_t w = lane; w < NW; w += 32) abits[w] = 0;
  __syncwarp();

  // merge path: lane owns merged positions [lane*2R, lane*2R + 2R)
  {
    const int d = lane * 2 * R;
    if ((uint32_t)d < nq) {
      const int K = (int)k;
      int lo = d > K ? d - K : 0, hi = d < K ? d : K;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid].key() <= B[d - 1 - mid].key()) lo = mid + 1; else hi = mid;
      }
      int ia = lo, ib = d - lo;
#pragma unroll 4
      for (int r = 0; r < 2 * R; ++r) {
        const int q = d + r;
        if (q >= (int)nq) break;
        const bool takeA = (ib >= K) || (ia < K && A[ia].key() <= B[ib].key());
        const E e = takeA ? A[ia] : B[ib];
        const uint32_t idx = e.idx();
        mk[q] = e.key();
        const uint32_t c = idx / R;          // owning lane (chunk) of this element
        atomicOr(&rows[row_addr(c, q >> 5)], 1u << (q & 31));
        if (takeA) {
          atomicOr(&abits[q >> 5], 1u << (q & 31));
          reinterpret_cast<uint16_t*>(rab)[2 * ((idx % R) * 32 + c)] = (uint16_t)q;
          ++ia;
        } else {
          reinterpret_cast<uint16_t*>(rab)[2 * ((idx % R) * 32 + c) + 1] = (uint16_t)q;
          ++ib;
        }
      }
    }
  }
  __syncwarp();
  // XOR prefix over chunks: row_L = A_bits ^ (toggles of chunks < L)
  for (uint32_t w = lane; w < nw; w += 32) {
    uint32_t acc = abits[w];
#pragma unroll 8
    for (uint32_t L = 0; L < 32; ++L) {
      const uint32_t a = row_addr(L, w);
      const uint32_t dlt = rows[a];
      rows[a] = acc;
      acc ^= dlt;
    }
  }
  __syncwarp();

  // walk: lane L emits outputs [L*R, L*R + R) of this unit
  const uint32_t i0 = lane * R;
  if (i0 < imax) {
    // select the (h+1)-th live position of row_L
    uint32_t cnt = 0, p = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      const uint32_t word = rows[row_addr(lane, w)];
      const uint32_t pc = __popc(word);
      if (cnt + pc > h) { p = w * 32 + __fns(word, 0, (int)(h - cnt) + 1); break; }
      cnt += pc;
    }
    ost[i0] = mk[p];
#pragma unroll 4
    for (int t = 1; t < R; ++t) {
      const uint32_t i = i0 + t;
      if (i >= imax) break;
      const uint32_t ab = rab[(t - 1) * 32 + lane];
      const uint32_t a = ab & 0xFFFF, b = ab >> 16;
      const uint32_t wa = row_addr(lane, a >> 5), wb = row_addr(lane, b >> 5);
      rows[wa] &= ~(1u << (a & 31));
      rows[wb] |= 1u << (b & 31);
      int dir = 0;  // +1: next live above p, -1: previous live below p
      if (a == p) dir = b < p ? -1 : 1;
      else if (a < p && b > p) dir = 1;
      else if (a > p && b < p) dir = -1;
      if (dir > 0) {
        uint32_t w = (p + 1) >> 5;
        uint32_t word = (p + 1) & 31 ? rows[row_addr(lane, w)] & (0xFFFFFFFFu << ((p + 1) & 31))
                                     : rows[row_addr(lane, w)];
        while (word == 0) { ++w; word = rows[row_addr(lane, w)]; }
        p = w * 32 + __ffs(word) - 1;
      } else if (dir < 0) {
        uint32_t w = p >> 5;
        uint32_t word = rows[row_addr(lane, w)] & ((1u << (p & 31)) - 1u);
        while (word == 0) { --w; word = rows[row_addr(lane, w)]; }
        p = w * 32 + 31 - __clz(word);
      }
      ost[i] = mk[p];
    }
  }
  __syncwarp();
  // coalesced store of the unit's imax outputs
  TV* yo = y + u * k;
  for (uint32_t i = lane; i < imax; i += 32) yo[i] = Tr::dec(ost[i]);
}

}  // namespace mf
