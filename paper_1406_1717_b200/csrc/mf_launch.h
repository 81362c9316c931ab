// mf_launch.h -- host-side launchers shared by the translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "mf_common.cuh"

namespace mf {

// Per-(device, kernel) launch setup (mf_setup.cu): applies the dynamic-smem opt-in on the
// current device and returns its SM count and, for threads > 0, the resident CTAs per SM
// at (threads, smem).  Thread-safe; cached per device.
struct LaunchInfo {
  int sms;
  int resident;
};
cudaError_t kernel_setup(const void* func, size_t smem, int threads, LaunchInfo* out);

// Phase tracing (mf_setup.cu).  Launchers mark the start of each phase of a filter call
// (e.g. the large-k pipeline's tile sort, merge passes, pair merge and walk): an NVTX mark
// always (free without a tool attached), and -- while a context with MF_OPT_PROFILE runs a
// call on this thread -- a CUDA event on the launching stream, from which the C ABI
// reports per-phase device times (mf_context_last_phases).
struct PhaseTrace {
  static constexpr int kMax = 64;
  cudaEvent_t ev[kMax + 1] = {};
  const char* name[kMax] = {};
  int n = 0;          // phases marked by the last call
  bool open = false;  // a call is recording
};
void phase_begin(PhaseTrace* t);                 // this thread's calls record into t
void phase_mark(cudaStream_t s, const char* name);
void phase_end(cudaStream_t s);                  // closes the last phase, stops recording

// Largest k each fused class handles (per key width).
constexpr uint32_t kSmallMaxK = 31;        // 64-bit keys
#ifndef MF_SMALL_MAXK32
#define MF_SMALL_MAXK32 63
#endif
constexpr uint32_t kSmallMaxK32 = MF_SMALL_MAXK32;      // 32-bit keys (64-bit live masks past 31; the medium
                                           // kernel takes over at k = 65)
inline uint32_t small_max_k(int dt) { return (dt == DT_I32 || dt == DT_F32) ? kSmallMaxK32 : kSmallMaxK; }
constexpr uint32_t kMediumMaxK = 1023;
// Largest k of the large-k pipeline: it packs 2k merged positions (padded to a multiple of
// 32) into uint32 and a side flag into bit 31 of an in-block index.  The reference accepts
// k <= 2^32 - 2 (core.hpp:68-69); larger windows are rejected with MF_BAD_ARG.
constexpr uint64_t kLargeMaxK = (uint64_t(1) << 31) - 65;

// Fused small-k kernel (k odd, k <= small_max_k(dt)).
cudaError_t launch_small(int dt, const Geom& g, cudaStream_t s, uint64_t* launches);
// ... its 33 <= k <= 63 instantiations (32-bit keys; mf_small63.cu)
cudaError_t launch_small_k63(int dt, const Geom& g, cudaStream_t s);
// Fused medium-k kernel (k <= 1023).
cudaError_t launch_medium(int dt, const Geom& g, cudaStream_t s, uint64_t* launches);

// Large-k pipeline: workspace requirement and run.
size_t large_workspace_bytes(int dt, const Geom& g);
cudaError_t run_large(int dt, const Geom& g, void* ws, size_t ws_bytes, cudaStream_t s, uint64_t* launches);
// Phase-1 only (piecewise_sort): b*k permutation entries per row.
size_t block_sort_workspace_bytes(int dt, const Geom& g, uint64_t nb);
cudaError_t run_block_sort(int dt, const Geom& g, uint64_t nb, void* ws, uint32_t* perm, cudaStream_t s,
                           uint64_t* launches);

// Device generators.
cudaError_t launch_generate(int kind, uint64_t seed, uint64_t mod, uint64_t offset, size_t n, void* out,
                            cudaStream_t s);

}  // namespace mf
