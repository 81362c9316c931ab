// mf_sortnet.cuh -- register sorting networks and the (key, index) element types.
//
// Phase 1 of the paper (piecewise sorting, filter.hpp:41-54) sorts (value, index)
// pairs so that equal values keep index order (stable).  On the GPU
// the pair is packed into one totally ordered element: for 32-bit keys a single
// u64 (key << 32 | index), for 64-bit keys a {key, index} pair compared
// lexicographically.  A total order makes any sorting network stable.
//
// The networks are Batcher odd-even merge sorts generated at compile time and
// pruned to K inputs (the pruned comparators only touch virtual +INF slots that
// never move in an all-ascending network), so a block of K elements sorts fully in
// registers with every index static.
#pragma once
#include <cstdint>
#include <utility>

#include "mf_common.cuh"

namespace mf {

struct NetList {
  int n;
  uint8_t a[1024];  // K <= 63: at most 543 comparators
  uint8_t b[1024];
};

constexpr NetList make_oem(int K) {
  NetList net{};
  net.n = 0;
  int N = 1;
  while (N < K) N <<= 1;
  for (int p = 1; p < N; p += p)
    for (int k = p; k > 0; k /= 2)
      for (int j = k % p; j + k < N; j += k + k)
        for (int i = 0; i < k && i < N - j - k; ++i)
          if ((i + j) / (p + p) == (i + j + k) / (p + p)) {
            const int lo = i + j, hi = i + j + k;
            if (hi < K) {
              net.a[net.n] = (uint8_t)lo;
              net.b[net.n] = (uint8_t)hi;
              ++net.n;
            }
          }
  return net;
}

template <int K> struct OEM { static constexpr NetList net = make_oem(K); };

// ---- element types --------------------------------------------------------------------
template <typename U> struct Elem;

// High word of a packed (key << 32 | index) element as a 32-bit register.  Written as a
// register-pair split because nvcc otherwise compares `(uint32_t)(v >> 32)` values as 64-bit
// numbers with a zero high word: an ISETP plus a useless ISETP.EX on (RZ, RZ) per exchange
// (378 of them in the k = 31 network).
__device__ __forceinline__ uint32_t hi32(uint64_t v) {
  uint32_t lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
  (void)lo;
  return hi;
}

template <> struct Elem<uint32_t> {
  static constexpr bool kFull = true;  // totally ordered by (key, index)
  uint64_t v;  // key << 32 | index
  __device__ __forceinline__ static Elem make(uint32_t key, uint32_t idx) {
    Elem e; e.v = ((uint64_t)key << 32) | idx; return e;
  }
  // greater than every real or padding element in the full order
  __device__ __forceinline__ static Elem sentinel() { Elem e; e.v = ~0ull; return e; }
  // merge order of two sorted blocks (A before B on ties): the sort order itself
  __device__ __forceinline__ static bool merge_le(const Elem& a, const Elem& b) { return a.v <= b.v; }
  __device__ __forceinline__ uint32_t key() const { return hi32(v); }
  __device__ __forceinline__ uint32_t idx() const { return (uint32_t)v; }
  __device__ __forceinline__ static bool less(const Elem& x, const Elem& y) { return x.v < y.v; }
  __device__ __forceinline__ static bool less_full(const Elem& x, const Elem& y) { return x.v < y.v; }
  __device__ __forceinline__ static void cswap(Elem& x, Elem& y) {
    const uint64_t lo = x.v < y.v ? x.v : y.v;
    const uint64_t hi = x.v < y.v ? y.v : x.v;
    x.v = lo; y.v = hi;
  }
  __device__ __forceinline__ static Elem select(bool c, const Elem& a, const Elem& b) {
    Elem e; e.v = sel(c, a.v, b.v); return e;
  }
};

template <> struct Elem<uint64_t> {
  static constexpr bool kFull = true;
  uint64_t k;
  uint32_t i;
  __device__ __forceinline__ static Elem make(uint64_t key, uint32_t idx) {
    Elem e; e.k = key; e.i = idx; return e;
  }
  __device__ __forceinline__ static Elem sentinel() { Elem e; e.k = ~0ull; e.i = ~0u; return e; }
  __device__ __forceinline__ static bool merge_le(const Elem& a, const Elem& b) { return !less(b, a); }
  __device__ __forceinline__ uint64_t key() const { return k; }
  __device__ __forceinline__ uint32_t idx() const { return i; }
  __device__ __forceinline__ static bool less(const Elem& x, const Elem& y) {
    return x.k < y.k || (x.k == y.k && x.i < y.i);
  }
  __device__ __forceinline__ static bool less_full(const Elem& x, const Elem& y) { return less(x, y); }
  __device__ __forceinline__ static void cswap(Elem& x, Elem& y) {
    const bool sw = less(y, x);
    const Elem t = x;
    x.k = sw ? y.k : x.k; x.i = sw ? y.i : x.i;
    y.k = sw ? t.k : y.k; y.i = sw ? t.i : y.i;
  }
  __device__ __forceinline__ static Elem select(bool c, const Elem& a, const Elem& b) {
    Elem e; e.k = sel(c, a.k, b.k); e.i = sel(c, a.i, b.i); return e;
  }
};

// Key-ordered elements: the same (key, index) payload, but comparisons look at the key
// only, so equal keys may end up in any order.  The filters need no more: the median of a
// window is a key (its bits are the sample's bits), and which of several equal samples is
// picked does not change it.  One compare instead of a 64-bit / two-part compare per
// exchange.  Decisions taken separately by two lanes about the same pair (bitonic
// cross-lane stages) use less_full, so both lanes agree on ties.  Phase-API sorts, whose
// permutation must match piecewise_sort (filter.hpp:41-54), keep Elem.
#ifndef MF_KE_PLAIN
#define MF_KE_PLAIN 1  // plain selects let ptxas schedule the network (measured: k = 31 small kernel 0.50 -> 0.46 ms)
#endif
struct KElem32 {
  static constexpr bool kFull = false;  // ordered by key only
  uint64_t v;  // key << 32 | index
  __device__ __forceinline__ static KElem32 make(uint32_t key, uint32_t idx) {
    KElem32 e; e.v = ((uint64_t)key << 32) | idx; return e;
  }
  __device__ __forceinline__ static KElem32 sentinel() { KElem32 e; e.v = ~0ull; return e; }
  // merge order of two key-sorted blocks: by key, A first on ties, except that the
  // sentinel (index bit 31) follows every real element of the same key
  __device__ __forceinline__ static bool merge_le(const KElem32& a, const KElem32& b) {
    return (a.v & 0xFFFFFFFF80000000ull) <= (b.v & 0xFFFFFFFF80000000ull);
  }
  __device__ __forceinline__ uint32_t key() const { return hi32(v); }
  __device__ __forceinline__ uint32_t idx() const { return (uint32_t)v; }
  __device__ __forceinline__ static bool less(const KElem32& x, const KElem32& y) { return x.key() < y.key(); }
  __device__ __forceinline__ static bool less_full(const KElem32& x, const KElem32& y) { return x.v < y.v; }
  __device__ __forceinline__ static void cswap(KElem32& x, KElem32& y) {
    const bool sw = y.key() < x.key();
    const uint64_t a = x.v, b = y.v;
#if MF_KE_PLAIN
    x.v = sw ? b : a;
    y.v = sw ? a : b;
#else
    x.v = sel(sw, b, a);
    y.v = sel(sw, a, b);
#endif
  }
  __device__ __forceinline__ static KElem32 select(bool c, const KElem32& a, const KElem32& b) {
    KElem32 e; e.v = sel(c, a.v, b.v); return e;
  }
};

struct KElem64 {
  static constexpr bool kFull = false;
  uint64_t k;
  uint32_t i;
  __device__ __forceinline__ static KElem64 make(uint64_t key, uint32_t idx) {
    KElem64 e; e.k = key; e.i = idx; return e;
  }
  __device__ __forceinline__ static KElem64 sentinel() { KElem64 e; e.k = ~0ull; e.i = ~0u; return e; }
  __device__ __forceinline__ static bool merge_le(const KElem64& a, const KElem64& b) {
    return a.k < b.k || (a.k == b.k && (a.i >> 31) <= (b.i >> 31));
  }
  __device__ __forceinline__ uint64_t key() const { return k; }
  __device__ __forceinline__ uint32_t idx() const { return i; }
  __device__ __forceinline__ static bool less(const KElem64& x, const KElem64& y) { return x.k < y.k; }
  __device__ __forceinline__ static bool less_full(const KElem64& x, const KElem64& y) {
    return x.k < y.k || (x.k == y.k && x.i < y.i);
  }
  __device__ __forceinline__ static void cswap(KElem64& x, KElem64& y) {
    const bool sw = y.k < x.k;
    const KElem64 t = x;
    x.k = sel(sw, y.k, x.k); x.i = sel(sw, y.i, x.i);
    y.k = sel(sw, t.k, y.k); y.i = sel(sw, t.i, y.i);
  }
  __device__ __forceinline__ static KElem64 select(bool c, const KElem64& a, const KElem64& b) {
    KElem64 e; e.k = sel(c, a.k, b.k); e.i = sel(c, a.i, b.i); return e;
  }
};

template <typename U> struct KeyOrd;
template <> struct KeyOrd<uint32_t> { using E = KElem32; };
template <> struct KeyOrd<uint64_t> { using E = KElem64; };

__device__ __forceinline__ KElem32 shfl_xor(const KElem32& e, int m) {
  KElem32 r; r.v = __shfl_xor_sync(0xFFFFFFFFu, e.v, m); return r;
}
__device__ __forceinline__ KElem64 shfl_xor(const KElem64& e, int m) {
  KElem64 r; r.k = __shfl_xor_sync(0xFFFFFFFFu, e.k, m); r.i = __shfl_xor_sync(0xFFFFFFFFu, e.i, m); return r;
}

__device__ __forceinline__ Elem<uint32_t> shfl_xor(const Elem<uint32_t>& e, int m) {
  Elem<uint32_t> r; r.v = __shfl_xor_sync(0xFFFFFFFFu, e.v, m); return r;
}
__device__ __forceinline__ Elem<uint64_t> shfl_xor(const Elem<uint64_t>& e, int m) {
  Elem<uint64_t> r; r.k = __shfl_xor_sync(0xFFFFFFFFu, e.k, m); r.i = __shfl_xor_sync(0xFFFFFFFFu, e.i, m); return r;
}

// read-only (non-coherent cache path) element loads
__device__ __forceinline__ Elem<uint32_t> ldg_elem(const Elem<uint32_t>* p) {
  Elem<uint32_t> r; r.v = __ldg(reinterpret_cast<const unsigned long long*>(&p->v)); return r;
}
__device__ __forceinline__ Elem<uint64_t> ldg_elem(const Elem<uint64_t>* p) {
  Elem<uint64_t> r;
  r.k = __ldg(reinterpret_cast<const unsigned long long*>(&p->k));
  r.i = __ldg(&p->i);
  return r;
}
__device__ __forceinline__ KElem32 ldg_elem(const KElem32* p) {
  KElem32 r; r.v = __ldg(reinterpret_cast<const unsigned long long*>(&p->v)); return r;
}
__device__ __forceinline__ KElem64 ldg_elem(const KElem64* p) {
  KElem64 r;
  r.k = __ldg(reinterpret_cast<const unsigned long long*>(&p->k));
  r.i = __ldg(&p->i);
  return r;
}

template <int K, int I> struct NetPair {
  static constexpr int a = OEM<K>::net.a[I], b = OEM<K>::net.b[I];
};
template <int K, typename E, int... I>
__device__ __forceinline__ void net_apply(E* v, std::integer_sequence<int, I...>) {
  (E::cswap(v[NetPair<K, I>::a], v[NetPair<K, I>::b]), ...);  // every index a constant
}

// Sort K register-resident elements (static indices only).
template <int K, typename E>
__device__ __forceinline__ void sort_regs(E (&v)[K]) {
  if constexpr (K > 1) net_apply<K>(v, std::make_integer_sequence<int, OEM<K>::net.n>{});
}

}  // namespace mf
