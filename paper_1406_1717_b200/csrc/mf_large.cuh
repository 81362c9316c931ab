// mf_large.cuh -- median filter for large windows (k beyond the fused kernels'
// shared-memory budget, e.g. k = 10,001 and 100,001): multi-kernel pipeline with
// the per-pair state in L2/HBM.
//
// Reference path replaced: median_filter<T> (filter.hpp:149-155).
//   piecewise_sort (filter.hpp:41-54) -> segmented global merge sort: CTA tile sorts
//       (register network + CTA merge-path passes in smem), then log2(k/TS) global
//       merge-path passes; blocks are segments, (key, index) elements keep it stable.
//   run_postprocess (filter.hpp:64-106) -> per block pair (unit):
//     ml_unit_merge   merge path of sorted A and sorted B (A wins key ties,
//                     filter.hpp:92-93): merged keys, merged-position -> (block, index)
//                     and index -> merged position (Delete(A,i) / Undelete(B,i) targets);
//     ml_counts/ml_scan  live counts per 1024-position "superword" at every chunk start,
//                     the selection index for the chunk's first median;
//     ml_walk         one thread per chunk of CL steps.  The state before step i is the
//                     live set {A: idx >= i} u {B: idx < i} (Eq. 4 / Lemma 1,
//                     SURVEY.md §0.6); the thread keeps only the cursor p and the one
//                     32-position word of the live set around it, recomputing a word
//                     from the origin table when the cursor leaves it, so per-thread state
//                     is O(1) however large k is.
#pragma once
#include "mf_common.cuh"
#include "mf_sortnet.cuh"

namespace mf {

constexpr int LT = 256;          // threads per CTA
constexpr int LRT = 8;           // elements per thread
constexpr int LTS = LT * LRT;    // tile size (elements)

struct LargeGeom {
  Geom g;
  uint64_t nb;        // blocks per row (= units + 1)
  uint32_t tiles;     // tiles per block = ceil(k / LTS)
  uint32_t nq;        // merged positions per unit = 2k
  uint32_t nqp;       // padded stride (multiple of 32)
  uint32_t tiles2;    // tiles per unit merge = ceil(2k / LTS)
  uint32_t CL;        // steps per walk chunk
  uint32_t C;         // chunks per unit
  uint32_t NS;        // superwords (1024 positions) per unit
};

// CTA-wide merge passes over LTS elements in smem, runs from LRT up to LTS.
template <typename E>
__device__ __forceinline__ void cta_merge_passes(E* s, E (&v)[LRT]) {
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int run = LRT; run < LTS; run *= 2) {
    const int gl = (2 * run) / LRT;
    const int j = tid & (gl - 1);
    E* X = s + (tid / gl) * (2 * run);
    const E* Y = X + run;
    const int d = j * LRT;
    int lo = d > run ? d - run : 0, hi = d < run ? d : run;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (E::less(X[mid], Y[d - 1 - mid])) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d - lo;
    E xa = X[ia < run ? ia : run - 1], yb = Y[ib < run ? ib : run - 1];
#pragma unroll
    for (int r = 0; r < LRT; ++r) {
      const bool takeA = (ib >= run) || (ia < run && E::less(xa, yb));
      v[r] = takeA ? xa : yb;
      if (takeA) { ++ia; xa = X[ia < run ? ia : run - 1]; }
      else { ++ib; yb = Y[ib < run ? ib : run - 1]; }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < LRT; ++r) X[d + r] = v[r];
    __syncthreads();
  }
}

// ---- phase 1a: sort LTS-element tiles of every block ---------------------------------
template <int DT>
__global__ void __launch_bounds__(LT) ml_tile_sort(LargeGeom L, Elem<typename Traits<DT>::U>* out) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using E = Elem<U>;
  using TV = typename Tr::T;
  __shared__ E s[LTS];
  const Geom& g = L.g;
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.tiles;
  const uint32_t t = blockIdx.x % L.tiles;
  const TV* x = reinterpret_cast<const TV*>(g.x) + row * g.ld_x;
  const uint32_t k = g.k;
  E v[LRT];
#pragma unroll
  for (int r = 0; r < LRT; ++r) {
    const uint32_t e = t * LTS + threadIdx.x + LT * r;
    const uint64_t gp = b * k + e;
    const U key = (e < k && gp < g.n) ? Tr::enc(x[gp]) : UMax<U>::v;
    v[r] = E::make(key, e);
  }
  sort_regs<LRT>(v);
#pragma unroll
  for (int r = 0; r < LRT; ++r) s[threadIdx.x * LRT + r] = v[r];
  __syncthreads();
  cta_merge_passes<E>(s, v);
  const uint32_t len = min((uint32_t)LTS, k - t * LTS);
  E* o = out + (row * L.nb + b) * k + (uint64_t)t * LTS;
  for (uint32_t i = threadIdx.x; i < len; i += LT) o[i] = s[i];
}

// merge-path split of diagonal d over X[0,lx) and Y[0,ly) under `before(x, y)`
template <typename E, typename Before>
__device__ __forceinline__ uint32_t merge_split(const E* X, uint32_t lx, const E* Y, uint32_t ly,
                                                uint32_t d, Before before) {
  uint32_t lo = d > ly ? d - ly : 0, hi = d < lx ? d : lx;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (before(X[mid], Y[d - 1 - mid])) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- phase 1b: one global merge pass (runs of length `run` within every block) --------
template <int DT>
__global__ void __launch_bounds__(LT) ml_merge_pass(LargeGeom L, const Elem<typename Traits<DT>::U>* in,
                                                    Elem<typename Traits<DT>::U>* out, uint32_t run) {
  using U = typename Traits<DT>::U;
  using E = Elem<U>;
  __shared__ E sx[LTS];
  __shared__ uint32_t split[2];
  const uint64_t row = blockIdx.y;
  const uint64_t b = blockIdx.x / L.tiles;
  const uint32_t t = blockIdx.x % L.tiles;
  const uint32_t k = L.g.k;
  const uint64_t base = (row * L.nb + b) * k;
  const uint32_t p0 = t * LTS;
  const uint32_t x0 = p0 / (2 * run) * (2 * run);
  const uint32_t lx = min(run, k - x0);
  const uint32_t y0 = x0 + lx;
  const uint32_t ly = y0 < k ? min(run, k - y0) : 0;
  const E* X = in + base + x0;
  const E* Y = in + base + y0;
  const uint32_t d0 = p0 - x0;
  const uint32_t d1 = min(d0 + LTS, lx + ly);
  auto before = [](const E& a, const E& c) { return E::less(a, c); };
  if (threadIdx.x < 2) split[threadIdx.x] = merge_split(X, lx, Y, ly, threadIdx.x ? d1 : d0, before);
  __syncthreads();
  const uint32_t a0 = split[0], a1 = split[1];
  const uint32_t b0 = d0 - a0, b1 = d1 - a1;
  const uint32_t nx = a1 - a0, ny = b1 - b0;
  for (uint32_t i = threadIdx.x; i < nx + ny; i += LT) sx[i] = i < nx ? X[a0 + i] : Y[b0 + i - nx];
  __syncthreads();
  const E* SX = sx;
  const E* SY = sx + nx;
  const uint32_t dd = threadIdx.x * LRT;
  if (dd < nx + ny) {
    uint32_t ia = merge_split(SX, nx, SY, ny, dd, before), ib = dd - ia;
    E* o = out + base + x0 + d0 + dd;
    for (int r = 0; r < LRT && dd + r < nx + ny; ++r) {
      const bool takeA = (ib >= ny) || (ia < nx && E::less(SX[ia], SY[ib]));
      o[r] = takeA ? SX[ia++] : SY[ib++];
    }
  }
}

// ---- phase 2a: merge each pair (A = block u, B = block u+1) ---------------------------
template <int DT>
__global__ void __launch_bounds__(LT) ml_unit_merge(LargeGeom L, const Elem<typename Traits<DT>::U>* S,
                                                    typename Traits<DT>::U* mk, uint32_t* org, uint2* rab) {
  using U = typename Traits<DT>::U;
  using E = Elem<U>;
  __shared__ E sx[LTS];
  __shared__ uint32_t split[2];
  const uint64_t row = blockIdx.y;
  const uint64_t u = blockIdx.x / L.tiles2;
  const uint32_t t = blockIdx.x % L.tiles2;
  const uint32_t k = L.g.k;
  const E* A = S + (row * L.nb + u) * k;
  const E* B = A + k;
  const uint64_t ug = row * L.g.units + u;
  const uint32_t d0 = t * LTS, d1 = min(d0 + LTS, L.nq);
  auto before = [](const E& a, const E& c) { return a.key() <= c.key(); };  // A wins ties
  if (threadIdx.x < 2) split[threadIdx.x] = merge_split(A, k, B, k, threadIdx.x ? d1 : d0, before);
  __syncthreads();
  const uint32_t a0 = split[0], a1 = split[1];
  const uint32_t b0 = d0 - a0, b1 = d1 - a1;
  const uint32_t nx = a1 - a0, ny = b1 - b0;
  for (uint32_t i = threadIdx.x; i < nx + ny; i += LT) sx[i] = i < nx ? A[a0 + i] : B[b0 + i - nx];
  __syncthreads();
  const E* SX = sx;
  const E* SY = sx + nx;
  const uint32_t dd = threadIdx.x * LRT;
  if (dd < nx + ny) {
    uint32_t ia = merge_split(SX, nx, SY, ny, dd, before), ib = dd - ia;
    U* mko = mk + ug * L.nqp + d0 + dd;
    uint32_t* oo = org + ug * L.nqp + d0 + dd;
    uint2* ro = rab + ug * k;
    for (int r = 0; r < LRT && dd + r < nx + ny; ++r) {
      const uint32_t q = d0 + dd + r;
      const bool takeA = (ib >= ny) || (ia < nx && SX[ia].key() <= SY[ib].key());
      const E e = takeA ? SX[ia++] : SY[ib++];
      mko[r] = e.key();
      oo[r] = e.idx() | (takeA ? 0u : 0x80000000u);
      if (takeA) ro[e.idx()].x = q; else ro[e.idx()].y = q;
    }
  }
}

// ---- phase 2b: live counts per (chunk start, superword) ------------------------------
__global__ void __launch_bounds__(LT) ml_counts(LargeGeom L, const uint32_t* org, uint32_t* live) {
  extern __shared__ uint32_t hist[];  // hA[C], hB[C]
  const uint64_t ug = blockIdx.x / L.NS;
  const uint32_t S = blockIdx.x % L.NS;
  uint32_t* hA = hist;
  uint32_t* hB = hist + L.C;
  for (uint32_t c = threadIdx.x; c < 2 * L.C; c += LT) hist[c] = 0;
  __syncthreads();
  const uint32_t* og = org + ug * L.nqp;
  const uint32_t q1 = min((S + 1) * 1024u, L.nq);
  for (uint32_t q = S * 1024 + threadIdx.x; q < q1; q += LT) {
    const uint32_t v = og[q];
    const uint32_t c = (v & 0x7FFFFFFFu) / L.CL;
    atomicAdd((v >> 31) ? &hB[c] : &hA[c], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // hA -> suffix sums, hB -> exclusive prefix sums
    uint32_t acc = 0;
    for (int c = (int)L.C - 1; c >= 0; --c) { acc += hA[c]; hA[c] = acc; }
    acc = 0;
    for (uint32_t c = 0; c < L.C; ++c) { const uint32_t t = hB[c]; hB[c] = acc; acc += t; }
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < L.C; c += LT) live[(ug * L.C + c) * L.NS + S] = hA[c] + hB[c];
}

__global__ void ml_scan(LargeGeom L, uint32_t* live, uint64_t total) {
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= total) return;
  uint32_t* p = live + id * L.NS;
  uint32_t acc = 0;
  for (uint32_t S = 0; S < L.NS; ++S) { const uint32_t t = p[S]; p[S] = acc; acc += t; }
}

// live bits of merged positions [32w, 32w+32) just before step i (output i)
__device__ __forceinline__ uint32_t live_word(const uint32_t* og, uint32_t w, uint32_t i, uint32_t nq) {
  uint32_t bits = 0;
  const uint4* v4 = reinterpret_cast<const uint4*>(og + w * 32);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 v = __ldg(v4 + j);
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const uint32_t q = w * 32 + j * 4 + l;
      const uint32_t idx = vv[l] & 0x7FFFFFFFu;
      const bool isB = vv[l] >> 31;
      const bool lv = q < nq && (isB ? idx < i : idx >= i);
      bits |= (uint32_t)lv << (j * 4 + l);
    }
  }
  return bits;
}

// ---- phase 2c: chunked walk -----------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(LT) ml_walk(LargeGeom L, const typename Traits<DT>::U* mk, const uint32_t* org,
                                              const uint2* rab, const uint32_t* live, uint64_t total) {
  using Tr = Traits<DT>;
  using U = typename Tr::U;
  using TV = typename Tr::T;
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= total) return;
  const uint64_t ug = id / L.C;
  const uint32_t c = id % L.C;
  const Geom& g = L.g;
  const uint64_t row = ug / g.units, u = ug % g.units;
  const uint32_t k = g.k, h = g.h;
  const uint64_t rem = g.keep - u * k;
  const uint32_t imax = rem < (uint64_t)k ? (uint32_t)rem : k;
  const uint32_t i0 = c * L.CL;
  if (i0 >= imax) return;
  const uint32_t i1 = min(imax, i0 + L.CL);
  const uint32_t* og = org + ug * L.nqp;
  const U* mkg = mk + ug * L.nqp;
  const uint2* rb = rab + ug * k;
  const uint32_t* cum = live + (ug * L.C + c) * L.NS;
  TV* y = reinterpret_cast<TV*>(g.y) + row * g.ld_y + u * k;

  // select: superword with cum[S] <= h < cum[S+1], then words inside it
  uint32_t lo = 0, hi = L.NS - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(cum + mid) <= h) lo = mid; else hi = mid - 1;
  }
  uint32_t r = h - __ldg(cum + lo);
  uint32_t cw = lo * 32, cb = 0;
  for (;; ++cw) {
    cb = live_word(og, cw, i0, L.nq);
    const uint32_t pc = __popc(cb);
    if (r < pc) break;
    r -= pc;
  }
  uint32_t p = cw * 32 + __fns(cb, 0, (int)r + 1);
  y[i0] = Tr::dec(mkg[p]);
  for (uint32_t i = i0 + 1; i < i1; ++i) {
    const uint2 ab = __ldg(rb + i - 1);
    const uint32_t a = ab.x, b = ab.y;
    if ((a >> 5) == cw) cb &= ~(1u << (a & 31));
    if ((b >> 5) == cw) cb |= 1u << (b & 31);
    int dir = 0;
    if (a == p) dir = b < p ? -1 : 1;
    else if (a < p && b > p) dir = 1;
    else if (a > p && b < p) dir = -1;
    if (dir > 0) {
      const uint32_t sh = (p & 31) + 1;
      uint32_t m = sh < 32 ? cb & (0xFFFFFFFFu << sh) : 0;
      while (m == 0) { ++cw; cb = live_word(og, cw, i, L.nq); m = cb; }
      p = cw * 32 + __ffs(m) - 1;
    } else if (dir < 0) {
      uint32_t m = cb & ((1u << (p & 31)) - 1u);
      while (m == 0) { --cw; cb = live_word(og, cw, i, L.nq); m = cb; }
      p = cw * 32 + 31 - __clz(m);
    }
    y[i] = Tr::dec(mkg[p]);
  }
}

}  // namespace mf
