/*
 * medfilt_gpu.h -- C ABI of the B200 median-filter library (libmedfilt_b200.so).
 *
 * The drop-in boundary for the reference's hot path
 *     template <std::signed_integral T>
 *     std::vector<T> medfilt::median_filter(std::span<const T> x, std::size_t k);
 *                                   (/root/reference/proj/include/medfilt/filter.hpp:149-155)
 * Plain pointers and sizes only; no exceptions and no C++/torch types cross it.
 * include/medfilt/gpu.hpp wraps it back into the reference's FilterFn<T> shape
 * (baselines.hpp:29-30) and rethrows the reference's exact error strings.
 *
 * Semantics (identical to the reference for every entry point):
 *   - y[i] = (h+1)-th smallest of x[i .. i+k-1], i in [0, n-k+1), k = 2h+1;
 *   - n < k gives an empty output, not an error (core.hpp:58-59, filter.hpp:69-79);
 *   - errors as core.hpp:62-76 (see mf_status and mf_error_message);
 *   - ties never change an output value (every median is an input element);
 *     float/double are ordered by IEEE totalOrder through the bit-key map of
 *     SURVEY.md §0.1 (an extension: the reference only takes signed integers).
 */
#ifndef MEDFILT_GPU_H
#define MEDFILT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MF_OK = 0,
  MF_EMPTY_INPUT = 1,     /* "input must not be empty"            core.hpp:63 */
  MF_K_ZERO = 2,          /* "window size must be positive"       core.hpp:64 */
  MF_K_EVEN = 3,          /* "even window size unsupported ..."   core.hpp:65-67 */
  MF_K_TOO_LARGE = 4,     /* "window size too large"              core.hpp:68-69 */
  MF_BAD_ARG = 5,         /* null pointer, short output buffer, bad dtype/stride */
  MF_CUDA_ERROR = 6,
  MF_OUT_OF_MEMORY = 7,
  MF_NO_DEVICE = 8
} mf_status;

typedef enum { MF_I32 = 0, MF_I64 = 1, MF_F32 = 2, MF_F64 = 3 } mf_dtype;

/* Kernel classes chosen by k: fused small (k <= 31; k <= 63 for 32-bit
 * keys; k = 3 is a direct selection kernel inside this class), fused medium (k <= 1023),
 * multi-kernel large. */
typedef enum { MF_CLASS_AUTO = -1, MF_CLASS_SMALL = 0, MF_CLASS_MEDIUM = 1, MF_CLASS_LARGE = 2 } mf_class;

typedef enum {
  MF_OPT_FORCE_CLASS = 0,     /* value: mf_class; a forced class must support k */
  MF_OPT_PIPELINE_CHUNK = 1,  /* value: largest host-pipeline chunk in samples (0 = default 2^22) */
  MF_OPT_PROFILE = 2          /* value 1: device entries record per-phase CUDA events (mf_context_last_phases) */
} mf_option;

typedef struct mf_context mf_context;

/* ---- status / arithmetic ---- */
const char* mf_status_string(mf_status s);
/* The reference's exception text for validation errors (core.hpp:63-69), else a description. */
const char* mf_error_message(mf_status s);
/* make_window_spec (core.hpp:62-76): h, b and output length; any out-pointer may be NULL. */
mf_status mf_window_spec(size_t n, size_t k, size_t* h, size_t* b, size_t* out_len);
/* Kernel class the library uses for (dtype, k). */
int mf_kernel_class(mf_dtype dtype, size_t k);

/* ---- context: device, stream and a grow-only device workspace (no per-call cudaMalloc) ---- */
mf_status mf_context_create(int device, mf_context** out);
/* Multi-device context over `ndev` CUDA devices (one sub-context each; a device may be
 * listed twice, e.g. for tests).  The host entries (mf_median_filter, mf_median_filter_rows)
 * shard their work across the devices, one host thread each: a single signal by contiguous
 * output ranges with a (k-1)-sample input halo, a batch by whole row groups (SURVEY.md
 * §8(e)); each device's D2H lands directly at its offset of the caller's output.  Outputs
 * are identical to a single-device call.  Device-pointer entries reject a multi-device
 * context only if the pointers are not device memory: with device pointers (on any one
 * "home" device), the device entries copy each shard peer to peer (peer access is enabled
 * here where the devices allow it: NVLink on a B200 box), filter it on its device and copy
 * its outputs back to the home buffer -- stream-ordered on the caller's stream. */
mf_status mf_context_create_multi(const int* devices, int ndev, mf_context** out);
/* Number of devices of ctx; writes up to `cap` device ids to `devices` (may be NULL). */
int mf_context_devices(const mf_context* ctx, int* devices, int cap);
void mf_context_destroy(mf_context* ctx);
mf_status mf_context_set_option(mf_context* ctx, mf_option opt, long value);
/* Number of kernels the last call on this context launched. */
uint64_t mf_context_last_launches(const mf_context* ctx);
/* Per-phase device times of the last device-entry call made with MF_OPT_PROFILE on: phase
 * names (static strings, e.g. "large: tile sort", "large: merge passes", "large: pair merge",
 * "large: walk") and milliseconds between consecutive phase marks; waits for the call to
 * finish.  Returns the number of phases (0 if none were recorded); fills at most `cap`.
 * Every call also emits NVTX ranges / marks (entries and phases) for nsys-style tools. */
int mf_context_last_phases(mf_context* ctx, const char** names, float* ms, int cap);

/* ---- host-buffer entry: the literal drop-in for median_filter<T> (filter.hpp:149-155).
 * x: n host samples; y: host buffer with capacity y_cap >= max(0, n-k+1); *y_len gets the
 * output length.  Synchronous: returns when y is filled. */
mf_status mf_median_filter(mf_context* ctx, mf_dtype dtype, const void* x, size_t n, size_t k,
                           void* y, size_t y_cap, size_t* y_len);

/* ---- device entry: d_x / d_y are device pointers on ctx's device; stream-ordered on
 * `stream` (a cudaStream_t; NULL = the default stream, as in the CUDA runtime); returns
 * after enqueueing.  The host entries use the context's own stream.  Calls on one context
 * may be issued on different streams: the context's large-k workspace is ordered across
 * them with an event, so such calls serialise on the device instead of sharing scratch.
 * k > 2^31 - 65 (large class) returns MF_BAD_ARG. */
mf_status mf_median_filter_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t n, size_t k,
                                  void* d_y, void* stream);

/* ---- batched rows: `rows` independent signals of n samples (row stride ld_x elements),
 * outputs n-k+1 per row (row stride ld_y elements).  Host and device flavours. */
mf_status mf_median_filter_rows(mf_context* ctx, mf_dtype dtype, const void* x, size_t rows, size_t n,
                                size_t ld_x, size_t k, void* y, size_t ld_y);
mf_status mf_median_filter_rows_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t rows,
                                       size_t n, size_t ld_x, size_t k, void* d_y, size_t ld_y,
                                       void* stream);

/* ---- phase API: piecewise_sort (filter.hpp:41-54) on the device.
 * d_perm gets b*k uint32 entries: d_perm[j*k + t] = index of the t-th smallest of block j
 * under the (value, index) order, the +INF padding of the last block sorting last. */
mf_status mf_block_sort_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t n, size_t k,
                               uint32_t* d_perm, void* stream);

/* ---- device-side input generators (SplitMix64, generators.hpp:16-29, jumped per index;
 * bit-identical to the sequential host stream; element j of the output is stream value
 * offset + j, so shards of one global signal are generated independently).  uniform_f32: (float)((next>>40)*2^-24);
 * uniform_f64: (next>>11)*2^-53; mod_i32: next % mod. ---- */
mf_status mf_generate_device(mf_context* ctx, int kind, uint64_t seed, uint64_t mod, uint64_t offset,
                             size_t n, void* d_out, void* stream);
enum { MF_GEN_UNIFORM_F32 = 0, MF_GEN_UNIFORM_F64 = 1, MF_GEN_MOD_I32 = 2 };
/* Host generator of the config-4 signal x_i = i/n + 0.01*sqrt(-2 ln(1-u1))*cos(2 pi u2)
 * (libm-dependent, so generated on the host; SURVEY.md §8(c) pitfall). */
void mf_generate_trend_f64_host(uint64_t seed, size_t n, double* out);

/* fold_checksum (io.hpp:17-28) on the host: FNV-1a over the 8 bytes of each value (32-bit
 * values sign-extended; float/double folded over their totalOrder keys).  Chainable:
 * start from MF_FOLD_INIT, and fold(a ++ b) = mf_fold_checksum(dt, b, nb, fold(a)). */
#define MF_FOLD_INIT 1469598103934665603ull
uint64_t mf_fold_checksum(mf_dtype dtype, const void* values, size_t n, uint64_t state);

#ifdef __cplusplus
}
#endif
#endif /* MEDFILT_GPU_H */
