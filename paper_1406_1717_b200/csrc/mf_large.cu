// mf_large.cu -- workspace planning and launch sequence of the large-k pipeline,
// the phase-1 (piecewise_sort) entry, and the device input generators.
#include <algorithm>

#include "mf_launch.h"
#include "mf_large.cuh"
#include "mf_pair.cuh"

#ifndef MF_LARGE_KEYORD
#define MF_LARGE_KEYORD 1  // the filter's block sort compares keys only (the phase API never does)
#endif
#ifndef MF_PAIR
#define MF_PAIR 0  // 1: fused shared-memory pair phase (ml_pair, mf_pair.cuh) for 1023 < k <= 16383.
                   // Bit-exact (c4 golden, checked build) but slower: c4 11.59 ms against 8.32 ms for
                   // ml_unit_merge + ml_walk.  Its ~180 KB of pair state leaves one CTA (8 warps) per
                   // SM, so the phases (merge rounds with exposed staging latency, 64 walkers) run
                   // serialised at 7 % warps active (profiles/r02_pair_experiment.txt).
#endif
#ifndef MF_TILE_RADIX
#define MF_TILE_RADIX 0  // 1: LSD radix tile sort, 0: comparison network + merge levels
#endif

namespace mf {

namespace {

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <int DT>
LargeGeom plan(const Geom& g, uint64_t nb) {
  using U = typename Traits<DT>::U;
  LargeGeom L{};
  L.g = g;
  L.nb = nb;
  L.TS = TileSort<U>::TS;
  L.tiles = (g.k + L.TS - 1) / L.TS;
  L.mtiles = (g.k + LQ - 1) / LQ;
  L.nq = 2 * g.k;
  L.nqp = (uint32_t)align_up(L.nq, 32);
  L.tiles2 = (L.nq + LQ - 1) / LQ;
  // Chunk length: enough chunks per unit to fill the GPU, few enough that the
  // per-chunk selection table stays small (C * NS counters per unit).
  uint32_t cl = 64;
#ifndef MF_WALK_MAXC
#define MF_WALK_MAXC 128  // most chunks per unit before the chunk length doubles (256: c4 7.98 ms, 128: 7.73, 64: 7.72;
                          // c5 46.7 / 46.1 / 46.1 ms: each chunk pays a select of ~16 live words)
#endif
  while (cl < 1024 && (g.k + cl - 1) / cl > MF_WALK_MAXC) cl *= 2;
  while ((g.k + cl - 1) / cl > 4096) cl *= 2;  // bounds the per-CTA histogram (8C words)
  L.CL = cl;
  L.CLshift = 0;
  while ((1u << L.CLshift) < cl) ++L.CLshift;
  L.C = (g.k + cl - 1) / cl;
  L.NS = (L.nq + 1023) / 1024;
  return L;
}

// kernel attributes, per device (kernel_setup)
template <int DT>
cudaError_t configure(const LargeGeom& L) {
  using U = typename Traits<DT>::U;
  cudaError_t e;
  for (auto f : {ml_tile_sort<DT, true>, ml_tile_sort<DT, false>})
    if ((e = kernel_setup((const void*)f, TileSort<U>::smem, 0, nullptr)) != cudaSuccess) return e;
  if ((e = kernel_setup((const void*)ml_tile_radix<DT>, TileRadix<U>::smem, 0, nullptr)) != cudaSuccess) return e;
  if constexpr (sizeof(U) == 8)
    if ((e = kernel_setup((const void*)ml_tile_sort_soa<DT>, TileSoa::smem, 0, nullptr)) != cudaSuccess) return e;
  if ((e = kernel_setup((const void*)ml_merge_pass<DT, true>, merge_tile_bytes<U, kSoa<U, true>>(), 0, nullptr)) !=
      cudaSuccess)
    return e;
  if ((e = kernel_setup((const void*)ml_merge_pass<DT, false>, merge_tile_smem<U>(), 0, nullptr)) != cudaSuccess)
    return e;
  if ((e = kernel_setup((const void*)ml_walk<DT>, sizeof(U) * 32 * 9 * (LNT / 32), 0, nullptr)) != cudaSuccess)
    return e;
  const size_t um = merge_tile_bytes<U, kSoa<U, true>>() + sizeof(uint32_t) * 8 * L.C;
  return kernel_setup((const void*)ml_unit_merge<DT>, um, 0, nullptr);
}

template <int DT>
struct Layout {
  using U = typename Traits<DT>::U;
  using E = Elem<U>;
  size_t off_s0, off_s1, off_split, off_mk, off_org, off_rab, off_live, total;
  Layout(const LargeGeom& L, bool sort_only) {
    const uint64_t nel = (uint64_t)L.g.rows * L.nb * L.g.k;
    const uint64_t nu = (uint64_t)L.g.rows * L.g.units;
    size_t o = 0;
    off_s0 = o; o = align_up(o + sizeof(E) * nel, 256);
    off_s1 = o; o = align_up(o + sizeof(E) * nel, 256);
    const uint64_t ntiles = std::max<uint64_t>((uint64_t)L.g.rows * L.nb * L.mtiles,
                                               (uint64_t)L.g.rows * L.g.units * L.tiles2);
    off_split = o; o = align_up(o + sizeof(uint2) * ntiles, 256);
    off_mk = off_org = off_rab = off_live = o;
    if (!sort_only) {
      off_mk = o; o = align_up(o + sizeof(U) * nu * L.nqp, 256);
      off_org = o; o = align_up(o + sizeof(uint32_t) * nu * L.nqp, 256);
      off_rab = o; o = align_up(o + sizeof(uint2) * nu * L.C * L.CL, 256);
      off_live = o; o = align_up(o + sizeof(uint32_t) * nu * L.C * L.NS, 256);
    }
    total = o;
  }
};

// Segmented sort of every block into key order (KO) or (key, index) order; returns the
// buffer holding it.
template <int DT, bool KO>
cudaError_t sort_blocks(const LargeGeom& L, unsigned char* ws, const Layout<DT>& lay, cudaStream_t s,
                        uint64_t* launches, Elem<typename Traits<DT>::U>** result) {
  using U = typename Traits<DT>::U;
  using E = Elem<U>;
  cudaError_t e = configure<DT>(L);
  if (e != cudaSuccess) return e;
  E* bufs[2] = {reinterpret_cast<E*>(ws + lay.off_s0), reinterpret_cast<E*>(ws + lay.off_s1)};
  phase_mark(s, "large: tile sort");
#if MF_TILE_RADIX
  static_assert(TileRadix<U>::TS == TileSort<U>::TS, "tile size is shared with the merge passes");
  ml_tile_radix<DT><<<dim3((unsigned)(L.nb * L.tiles), L.g.rows), TileRadix<U>::NT, TileRadix<U>::smem, s>>>(
      L, bufs[0]);
#else
  if constexpr (MF_TS_SOA && KO && sizeof(U) == 8)
    ml_tile_sort_soa<DT><<<dim3((unsigned)(L.nb * L.tiles), L.g.rows), LNT, TileSoa::smem, s>>>(
        L, reinterpret_cast<Elem<uint64_t>*>(bufs[0]));
  else
    ml_tile_sort<DT, KO><<<dim3((unsigned)(L.nb * L.tiles), L.g.rows), LNT, TileSort<U>::smem, s>>>(L, bufs[0]);
#endif
  ++*launches;
  int cur = 0;
  uint2* splits = reinterpret_cast<uint2*>(ws + lay.off_split);
  const uint64_t ptiles = (uint64_t)L.g.rows * L.nb * L.mtiles;
  if ((uint64_t)L.TS < L.g.k) phase_mark(s, "large: merge passes");
  for (uint64_t run = L.TS; run < L.g.k; run *= 2) {
    ml_partition_pass<DT, KO><<<(unsigned)((ptiles + 127) / 128), 128, 0, s>>>(L, bufs[cur], splits, (uint32_t)run,
                                                                         ptiles);
    ml_merge_pass<DT, KO><<<dim3((unsigned)(L.nb * L.mtiles), L.g.rows), LNT, merge_tile_bytes<U, kSoa<U, KO>>(), s>>>(
        L, bufs[cur], bufs[cur ^ 1], (uint32_t)run, splits);
    *launches += 2;
    cur ^= 1;
  }
  *result = bufs[cur];
  return cudaGetLastError();
}

template <int DT>
cudaError_t run_large_dt(const Geom& g, void* wsv, size_t ws_bytes, cudaStream_t s, uint64_t* launches) {
  const LargeGeom L = plan<DT>(g, g.units + 1);
  const Layout<DT> lay(L, false);
  if (ws_bytes < lay.total) return cudaErrorMemoryAllocation;
  unsigned char* ws = static_cast<unsigned char*>(wsv);
  using U = typename Traits<DT>::U;
  Elem<U>* sorted = nullptr;
  cudaError_t e = sort_blocks<DT, MF_LARGE_KEYORD != 0>(L, ws, lay, s, launches, &sorted);
  if (e != cudaSuccess) return e;
  U* mk = reinterpret_cast<U*>(ws + lay.off_mk);
  uint32_t* org = reinterpret_cast<uint32_t*>(ws + lay.off_org);
  uint2* rab = reinterpret_cast<uint2*>(ws + lay.off_rab);
  uint32_t* live = reinterpret_cast<uint32_t*>(ws + lay.off_live);
  const uint64_t nu = (uint64_t)g.rows * g.units;
  const size_t um = merge_tile_bytes<U, kSoa<U, true>>() + sizeof(uint32_t) * 8 * L.C;
  uint2* splits = reinterpret_cast<uint2*>(ws + lay.off_split);
  const uint64_t utiles = (uint64_t)g.rows * g.units * L.tiles2;
  phase_mark(s, "large: pair merge");
  ml_partition_units<DT><<<(unsigned)((utiles + 127) / 128), 128, 0, s>>>(L, sorted, splits, utiles);
  if (MF_PAIR && g.k <= kPairMaxK) {
    const PairGeom P = pair_plan(g.k, merge_tile_bytes<U, kSoa<U, true>>());
    if (P.smem <= 227u * 1024u) {
      if ((e = kernel_setup((const void*)ml_pair<DT>, P.smem, 0, nullptr)) != cudaSuccess) return e;
      phase_mark(s, "large: fused pair merge + walk");
      ml_pair<DT><<<dim3((unsigned)g.units, g.rows), LNT, P.smem, s>>>(L, P, sorted, splits);
      *launches += 2;
      return cudaGetLastError();
    }
  }
  ml_unit_merge<DT><<<dim3((unsigned)(g.units * L.tiles2), g.rows), LNT, um, s>>>(L, sorted, mk, org, rab, live,
                                                                                  splits);
  *launches += 2;
  const uint64_t nchunks = nu * L.C;
  phase_mark(s, "large: walk");
  ml_walk<DT><<<(unsigned)((nchunks + LNT - 1) / LNT), LNT, sizeof(U) * 32 * 9 * (LNT / 32), s>>>(
      L, mk, org, rab, live, nchunks);
  ++*launches;
  return cudaGetLastError();
}

template <int DT>
__global__ void ml_extract_perm(LargeGeom L, const Elem<typename Traits<DT>::U>* S, uint32_t* perm, uint64_t total) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) perm[i] = S[i].idx();
}

template <int DT>
cudaError_t run_sort_dt(const Geom& g, uint64_t nb, void* wsv, uint32_t* perm, cudaStream_t s,
                        uint64_t* launches) {
  const LargeGeom L = plan<DT>(g, nb);
  const Layout<DT> lay(L, true);
  using U = typename Traits<DT>::U;
  Elem<U>* sorted = nullptr;
  cudaError_t e = sort_blocks<DT, false>(L, static_cast<unsigned char*>(wsv), lay, s, launches, &sorted);
  if (e != cudaSuccess) return e;
  const uint64_t total = (uint64_t)g.rows * nb * g.k;
  ml_extract_perm<DT><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(L, sorted, perm, total);
  ++*launches;
  return cudaGetLastError();
}

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  // value of the (i+1)-th next() of SplitMix64(seed) (generators.hpp:20-25)
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void gen_kernel(int kind, uint64_t seed, uint64_t mod, uint64_t offset, size_t n, void* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix_at(seed, offset + i);
    if (kind == 0) static_cast<float*>(out)[i] = (float)((double)(r >> 40) * 0x1.0p-24);
    else if (kind == 1) static_cast<double*>(out)[i] = (double)(r >> 11) * 0x1.0p-53;
    else static_cast<int32_t*>(out)[i] = (int32_t)(r % mod);
  }
}

}  // namespace

size_t large_workspace_bytes(int dt, const Geom& g) {
  switch (dt) {
    case DT_I32: return Layout<DT_I32>(plan<DT_I32>(g, g.units + 1), false).total;
    case DT_I64: return Layout<DT_I64>(plan<DT_I64>(g, g.units + 1), false).total;
    case DT_F32: return Layout<DT_F32>(plan<DT_F32>(g, g.units + 1), false).total;
    default: return Layout<DT_F64>(plan<DT_F64>(g, g.units + 1), false).total;
  }
}

cudaError_t run_large(int dt, const Geom& g, void* ws, size_t ws_bytes, cudaStream_t s, uint64_t* launches) {
  switch (dt) {
    case DT_I32: return run_large_dt<DT_I32>(g, ws, ws_bytes, s, launches);
    case DT_I64: return run_large_dt<DT_I64>(g, ws, ws_bytes, s, launches);
    case DT_F32: return run_large_dt<DT_F32>(g, ws, ws_bytes, s, launches);
    case DT_F64: return run_large_dt<DT_F64>(g, ws, ws_bytes, s, launches);
  }
  return cudaErrorInvalidValue;
}

size_t block_sort_workspace_bytes(int dt, const Geom& g, uint64_t nb) {
  switch (dt) {
    case DT_I32: return Layout<DT_I32>(plan<DT_I32>(g, nb), true).total;
    case DT_I64: return Layout<DT_I64>(plan<DT_I64>(g, nb), true).total;
    case DT_F32: return Layout<DT_F32>(plan<DT_F32>(g, nb), true).total;
    default: return Layout<DT_F64>(plan<DT_F64>(g, nb), true).total;
  }
}

cudaError_t run_block_sort(int dt, const Geom& g, uint64_t nb, void* ws, uint32_t* perm, cudaStream_t s,
                           uint64_t* launches) {
  switch (dt) {
    case DT_I32: return run_sort_dt<DT_I32>(g, nb, ws, perm, s, launches);
    case DT_I64: return run_sort_dt<DT_I64>(g, nb, ws, perm, s, launches);
    case DT_F32: return run_sort_dt<DT_F32>(g, nb, ws, perm, s, launches);
    case DT_F64: return run_sort_dt<DT_F64>(g, nb, ws, perm, s, launches);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_generate(int kind, uint64_t seed, uint64_t mod, uint64_t offset, size_t n, void* out,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 32);
  gen_kernel<<<blocks, 256, 0, s>>>(kind, seed, mod, offset, n, out);
  return cudaGetLastError();
}

}  // namespace mf
