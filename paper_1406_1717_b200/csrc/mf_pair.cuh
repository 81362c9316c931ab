// mf_pair.cuh -- fused pair phase of the large-k pipeline for 1023 < k <= 16383
// (config 4's range): one CTA per block pair keeps the pair's state in shared memory.
//
// Reference path replaced: run_postprocess (filter.hpp:64-106) with the Block dancing links
// (block.hpp:24-146).  The sorted blocks come from the pipeline's tile sort and merge passes
// (mf_large.cuh); ml_unit_merge + ml_walk write and re-read the merged keys, the origin table
// and the index -> position maps through HBM (about 4 GB per config-4 call).  Here they stay
// on chip:
//   org[q]   merged position q -> idx | isB << 15        (u16; k <= 16383 < 2^14)
//   rabA/B   index -> merged position                    (u16; 2k <= 32766)
//   isb/pre  side bitmap of the merged order and its word prefix counts: the sorted position
//            of the element at q is the number of same-side positions before q, so the
//            emitted key is read from the sorted block itself (L2-resident: this CTA merged
//            it moments before) -- no merged-key table
//   hist     live count of every 256-position superword at every chunk start
// Phases: (1) merge path of A and B in LQ-position tiles (merge_tile*, splits from
// ml_partition_units) filling org / rab / isb / hist; (2) prefix of the side bitmap and the
// per-chunk live counts; (3) PCH chunk walkers: select the (h+1)-th live position at the
// chunk's first step from the counts and on-demand live words, then walk it exactly like
// ml_walk (a 64-position window of the live set, Delete(A,i-1) / Undelete(B,i-1) per step,
// the cursor moving to the next or previous live position).
#pragma once
#include "mf_large.cuh"

namespace mf {

constexpr int PCH = 64;    // walk chunks per pair (two walking warps)
constexpr int PSW = 256;   // positions per superword (select granularity)
constexpr uint32_t kPairMaxK = 16383;

struct PairGeom {
  uint32_t NQP;   // merged positions rounded up to a superword
  uint32_t NS;    // superwords
  uint32_t CL;    // steps per chunk
  uint32_t off_org, off_rabA, off_rabB, off_isb, off_pre, off_hist, off_tile;
  uint32_t smem;  // bytes of dynamic shared memory
};

inline PairGeom pair_plan(uint32_t k, size_t tile_bytes) {
  PairGeom P{};
  const uint32_t nq = 2 * k;
  P.NQP = (nq + PSW - 1) / PSW * PSW;
  P.NS = P.NQP / PSW;
  P.CL = (k + PCH - 1) / PCH;
  auto al = [](uint32_t v) { return (v + 15) / 16 * 16; };
  uint32_t o = 0;
  P.off_org = o;  o = al(o + 2 * P.NQP);
  P.off_rabA = o; o = al(o + 2 * k);
  P.off_rabB = o; o = al(o + 2 * k);
  P.off_isb = o;  o = al(o + 4 * (P.NQP / 32));
  P.off_pre = o;  o = al(o + 4 * (P.NQP / 32));
  P.off_hist = o; o = al(o + 4 * 2 * P.NS * PCH);
  P.off_tile = o; o = al(o + (uint32_t)(tile_bytes > 2u * k ? tile_bytes : 2u * k));  // merge tile, then ps[k]
  P.smem = o;
  return P;
}

// live bits of merged positions [32w, 32w+32) before step i, from the u16 origin table:
// position q is live iff bit 15 of (org - i) is clear (the 16-bit form of live_word)
__device__ __forceinline__ uint32_t live_word16(const uint16_t* org, uint32_t w, uint32_t i, uint32_t nq) {
  const uint32_t* o32 = reinterpret_cast<const uint32_t*>(org) + w * 16;
  uint32_t dead = 0;
#pragma unroll
  for (int j = 15; j >= 0; --j) {
    const uint32_t v = o32[j];
    dead = (dead << 1) | ((((v >> 16) - i) >> 15) & 1u);
    dead = (dead << 1) | ((((v & 0xFFFFu) - i) >> 15) & 1u);
  }
  const uint32_t q0 = w * 32;
  const uint32_t valid = q0 + 32 <= nq ? 0xFFFFFFFFu : (q0 < nq ? (1u << (nq - q0)) - 1u : 0u);
  return ~dead & valid;
}

template <int DT>
__global__ void __launch_bounds__(LNT, 1) ml_pair(LargeGeom L, PairGeom P, const Elem<typename Traits<DT>::U>* S,
                                                   const uint2* splits) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using TV = typename Tr::T;
  using E = Elem<U>;
  constexpr bool SOA = kSoa<U, true>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* org = reinterpret_cast<uint16_t*>(smem_raw + P.off_org);
  uint16_t* rabA = reinterpret_cast<uint16_t*>(smem_raw + P.off_rabA);
  uint16_t* rabB = reinterpret_cast<uint16_t*>(smem_raw + P.off_rabB);
  uint32_t* isb = reinterpret_cast<uint32_t*>(smem_raw + P.off_isb);
  uint32_t* pre = reinterpret_cast<uint32_t*>(smem_raw + P.off_pre);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw + P.off_hist);  // [side][NS][PCH]
  unsigned char* tile = smem_raw + P.off_tile;
  const Geom& g = L.g;
  const uint64_t row = blockIdx.y, u = blockIdx.x;
  const uint32_t k = g.k, h = g.h, nq = 2 * k;
  const uint64_t ug = row * g.units + u;
  const E* A = S + (row * L.nb + u) * k;
  const E* B = A + k;
  const uint32_t NW = P.NQP / 32, NS = P.NS, CL = P.CL;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (uint32_t i = tid; i < NW; i += LNT) isb[i] = 0;
  for (uint32_t i = tid; i < 2 * NS * PCH; i += LNT) hist[i] = 0;
  __syncthreads();

  // ---- (1) merge path of the pair, LQ positions per round ----
  const int dd = (int)tid * LR2;
  for (uint32_t t = 0; t < L.tiles2; ++t) {
    const uint32_t d0 = t * LQ, d1 = min(d0 + LQ, nq);
    const uint2 sp = splits[ug * L.tiles2 + t];
    U vk[LR2];
    uint32_t vi[LR2];
    bool srcB[LR2];
    uint32_t nx;
    int cnt;
    if constexpr (SOA) {
      U* tk = reinterpret_cast<U*>(tile);
      uint32_t* ti = reinterpret_cast<uint32_t*>(tk + LQ + (LQ >> LPS) + 1);
      cnt = merge_tile_soa<true>(tk, ti, A, B, d0, d1, sp, vk, vi, srcB, nx);  // A first on key ties
    } else {
      auto before = [](const E& a, const E& c) { return a.key() <= c.key(); };
      E v[LR2];
      cnt = merge_tile(reinterpret_cast<E*>(tile), A, B, d0, d1, sp, before, v, srcB, nx);
#pragma unroll
      for (int r = 0; r < LR2; ++r) {
        vk[r] = v[r].key();
        vi[r] = v[r].idx();
      }
    }
    (void)vk;
    uint32_t bm = 0;
#pragma unroll
    for (int r = 0; r < LR2; ++r) {
      if (r < cnt) {
        const uint32_t q = d0 + dd + r, idx = vi[r];
        MF_ASSERT(q < nq && idx < k);
        org[q] = (uint16_t)(idx | (srcB[r] ? 0x8000u : 0u));
        (srcB[r] ? rabB : rabA)[idx] = (uint16_t)q;
        bm |= srcB[r] ? 1u << r : 0u;
        atomicAdd(&hist[((srcB[r] ? NS : 0u) + q / PSW) * PCH + idx / CL], 1u);
      }
    }
    if (cnt > 0) {
      const uint32_t q0 = d0 + dd;  // a multiple of LR2 = 16: one half of a bitmap word
      atomicOr(&isb[q0 >> 5], bm << (q0 & 31));
    }
    __syncthreads();  // the tile area is restaged by the next round
  }

  // ---- (2) side-bitmap prefix and live counts per (superword, chunk start) ----
  {
    // exclusive prefix of popc(isb[w]) over the NW words: per-thread runs, then a CTA scan
    const uint32_t per = (NW + LNT - 1) / LNT, w0 = tid * per, w1 = min(NW, w0 + per);
    uint32_t sum = 0;
    for (uint32_t w = w0; w < w1; ++w) sum += __popc(isb[w]);
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    uint32_t* wsum = reinterpret_cast<uint32_t*>(tile);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t base = inc - sum;
    for (uint32_t w = 0; w < warp; ++w) base += wsum[w];
    for (uint32_t w = w0; w < w1; ++w) {
      pre[w] = base;
      base += __popc(isb[w]);
    }
  }
  for (uint32_t s = warp; s < NS; s += LNT / 32) {
    // chunk c starts at step c*CL: live = A with chunk(idx) >= c plus B with chunk(idx) < c
    uint32_t* hA = hist + s * PCH;
    const uint32_t* hB = hist + (NS + s) * PCH;
    const uint32_t a0 = hA[lane], a1 = hA[32 + lane], b0 = hB[lane], b1 = hB[32 + lane];
    uint32_t sa0 = a0, sa1 = a1, sb0 = b0, sb1 = b1;  // inclusive scans over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x0 = __shfl_up_sync(0xFFFFFFFFu, sa0, o), x1 = __shfl_up_sync(0xFFFFFFFFu, sa1, o);
      const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, sb0, o), y1 = __shfl_up_sync(0xFFFFFFFFu, sb1, o);
      if (lane >= (uint32_t)o) { sa0 += x0; sa1 += x1; sb0 += y0; sb1 += y1; }
    }
    const uint32_t ta0 = __shfl_sync(0xFFFFFFFFu, sa0, 31), ta1 = __shfl_sync(0xFFFFFFFFu, sa1, 31);
    const uint32_t tb0 = __shfl_sync(0xFFFFFFFFu, sb0, 31);
    const uint32_t totA = ta0 + ta1;
    const uint32_t ea0 = sa0 - a0, ea1 = ta0 + sa1 - a1;  // exclusive prefixes of A
    const uint32_t eb0 = sb0 - b0, eb1 = tb0 + sb1 - b1;  // ... and of B
    __syncwarp();
    hA[lane] = (totA - ea0) + eb0;
    hA[32 + lane] = (totA - ea1) + eb1;
  }
  __syncthreads();

  // ---- (3) walk: chunk c = tid (< PCH) finds the median positions of steps [c*CL, c*CL + CL)
  // into ps[] (the tile area is free); (4) every thread then emits keys, coalesced, with all
  // key loads in flight (a load per step on the walk's chain would stall it on L2 latency)
  const uint64_t rem = g.keep - u * k;
  const uint32_t imax = rem < (uint64_t)k ? (uint32_t)rem : k;
  uint16_t* ps = reinterpret_cast<uint16_t*>(tile);
  auto word = [&](uint32_t w, uint32_t i) -> uint32_t { return w < NW ? live_word16(org, w, i, nq) : 0u; };
  const uint32_t i0 = tid * CL, i1 = min(imax, i0 + CL);
  if (tid < (uint32_t)PCH && i0 < i1) {
    // select the (h+1)-th live position before step i0
    uint32_t acc = 0, s = 0;
    for (; s < NS; ++s) {
      const uint32_t v = hist[s * PCH + tid];
      if (acc + v > h) break;
      acc += v;
    }
    MF_ASSERT(s < NS);
    uint32_t r = h - acc, cw = s * (PSW / 32), cb = 0;
    for (;; ++cw) {
      MF_ASSERT(cw < NW);
      cb = word(cw, i0);
      const uint32_t pc = __popc(cb);
      if (r < pc) break;
      r -= pc;
    }
    uint32_t p = cw * 32 + __fns(cb, 0, (int)r + 1);
    uint32_t cw0 = cw;
    uint64_t win = (uint64_t)cb | ((uint64_t)word(cw + 1, i0) << 32);
    ps[i0] = (uint16_t)p;
    for (uint32_t i = i0 + 1; i < i1; ++i) {
      const uint32_t a = rabA[i - 1], b = rabB[i - 1];  // Delete(A, i-1), Undelete(B, i-1)
      const uint32_t base = cw0 * 32;
      const uint32_t oa = a - base, ob = b - base, off = p - base;
      win &= ~(oa < 64 ? 1ull << oa : 0ull);
      win |= ob < 64 ? 1ull << ob : 0ull;
      const bool up = a <= p && b > p;
      const bool down = a >= p && b < p;
      uint64_t m = up ? (win & (0xFFFFFFFFFFFFFFFEull << off)) : (win & ((1ull << off) - 1ull));
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
      p = up ? cw0 * 32 + __ffsll((long long)m) - 1 : (down ? cw0 * 32 + 63 - __clzll((long long)m) : p);
      MF_ASSERT(p < nq);
      ps[i] = (uint16_t)p;
    }
  }
  __syncthreads();
  TV* y = reinterpret_cast<TV*>(g.y) + row * g.ld_y + u * k;
  for (uint32_t i = tid; i < imax; i += LNT) {
    const uint32_t p = ps[i], w = p >> 5, bits = isb[w];
    const uint32_t nB = pre[w] + __popc(bits & ((1u << (p & 31)) - 1u));
    const bool side = (bits >> (p & 31)) & 1u;
    const E* blk = side ? B : A;
    y[i] = Tr::dec(ldg_elem(blk + (side ? nB : p - nB)).key());
  }
}

}  // namespace mf
