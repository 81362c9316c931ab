// mf_capi.cu -- the extern "C" boundary (include/medfilt_gpu.h).
//
// Validation mirrors make_window_spec (core.hpp:62-76) check for check and in the
// same order; n < k returns an empty output (core.hpp:58-59).  There is no CPU
// fallback: every entry either runs the CUDA kernels or returns an error status.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/medfilt_gpu.h"
#include "mf_launch.h"

struct mf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  void* ws = nullptr;          // grow-only device workspace
  size_t ws_bytes = 0;
  void* io = nullptr;          // grow-only device buffers for the host entry points
  size_t io_bytes = 0;
  int force_class = MF_CLASS_AUTO;
  uint64_t launches = 0;
  std::mutex mu;
};

namespace {

size_t dtype_size(mf_dtype d) { return (d == MF_I64 || d == MF_F64) ? 8 : 4; }
bool dtype_ok(int d) { return d >= MF_I32 && d <= MF_F64; }

mf_status from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return MF_OK;
  if (e == cudaErrorMemoryAllocation) return MF_OUT_OF_MEMORY;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return MF_NO_DEVICE;
  return MF_CUDA_ERROR;
}

mf_status grow(void** p, size_t* cap, size_t need) {
  if (need <= *cap) return MF_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) { cudaGetLastError(); return from_cuda(e); }
  *cap = need;
  return MF_OK;
}

int class_for(mf_dtype, size_t k) {
  if (k <= mf::kSmallMaxK) return MF_CLASS_SMALL;
  if (k <= mf::kMediumMaxK) return MF_CLASS_MEDIUM;
  return MF_CLASS_LARGE;
}

// Core device path over `rows` independent signals; caller holds ctx->mu.
mf_status run_rows(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t rows, size_t n, size_t ld_x,
                   size_t k, void* d_y, size_t ld_y, cudaStream_t s) {
  size_t keep = 0;
  mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
  if (st != MF_OK) return st;
  if (!dtype_ok(dtype)) return MF_BAD_ARG;
  ctx->launches = 0;
  if (keep == 0 || rows == 0) return MF_OK;
  if (!d_x || !d_y || ld_x < n || ld_y < keep || rows > 65535) return MF_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  mf::Geom g{};
  g.x = d_x; g.y = d_y; g.n = n; g.ld_x = ld_x; g.ld_y = ld_y;
  g.k = (uint32_t)k; g.h = (uint32_t)((k - 1) / 2);
  g.keep = keep; g.units = (keep + k - 1) / k; g.rows = (uint32_t)rows;
  int cls = ctx->force_class == MF_CLASS_AUTO ? class_for(dtype, k) : ctx->force_class;
  if (cls == MF_CLASS_SMALL && k > mf::kSmallMaxK) return MF_BAD_ARG;
  if (cls == MF_CLASS_MEDIUM && k > mf::kMediumMaxK) return MF_BAD_ARG;
  cudaError_t e;
  if (cls == MF_CLASS_SMALL) {
    e = mf::launch_small(dtype, g, s, &ctx->launches);
  } else if (cls == MF_CLASS_MEDIUM) {
    e = mf::launch_medium(dtype, g, s, &ctx->launches);
  } else {
    const size_t need = mf::large_workspace_bytes(dtype, g);
    st = grow(&ctx->ws, &ctx->ws_bytes, need);
    if (st != MF_OK) return st;
    e = mf::run_large(dtype, g, ctx->ws, ctx->ws_bytes, s, &ctx->launches);
  }
  return from_cuda(e);
}

// Device entries follow the CUDA convention: NULL is the default stream.
cudaStream_t pick(mf_context*, void* stream) { return static_cast<cudaStream_t>(stream); }

}  // namespace

extern "C" {

const char* mf_status_string(mf_status s) {
  switch (s) {
    case MF_OK: return "MF_OK";
    case MF_EMPTY_INPUT: return "MF_EMPTY_INPUT";
    case MF_K_ZERO: return "MF_K_ZERO";
    case MF_K_EVEN: return "MF_K_EVEN";
    case MF_K_TOO_LARGE: return "MF_K_TOO_LARGE";
    case MF_BAD_ARG: return "MF_BAD_ARG";
    case MF_CUDA_ERROR: return "MF_CUDA_ERROR";
    case MF_OUT_OF_MEMORY: return "MF_OUT_OF_MEMORY";
    case MF_NO_DEVICE: return "MF_NO_DEVICE";
  }
  return "MF_UNKNOWN";
}

const char* mf_error_message(mf_status s) {
  switch (s) {  // the reference's std::invalid_argument texts, core.hpp:63-69
    case MF_EMPTY_INPUT: return "input must not be empty";
    case MF_K_ZERO: return "window size must be positive";
    case MF_K_EVEN: return "even window size unsupported (window must be k = 2h+1)";
    case MF_K_TOO_LARGE: return "window size too large";
    case MF_OK: return "ok";
    case MF_BAD_ARG: return "bad argument (null pointer, short output buffer, stride or dtype)";
    case MF_CUDA_ERROR: return "CUDA error";
    case MF_OUT_OF_MEMORY: return "out of device memory";
    case MF_NO_DEVICE: return "no CUDA device";
  }
  return "unknown status";
}

mf_status mf_window_spec(size_t n, size_t k, size_t* h, size_t* b, size_t* out_len) {
  if (n == 0) return MF_EMPTY_INPUT;                 // core.hpp:63
  if (k == 0) return MF_K_ZERO;                      // core.hpp:64
  if (k % 2 == 0) return MF_K_EVEN;                  // core.hpp:65-67
  if (k >= 0xFFFFFFFFull) return MF_K_TOO_LARGE;     // core.hpp:68-69
  if (h) *h = (k - 1) / 2;                           // core.hpp:73
  if (b) *b = (n + k - 1) / k;                       // core.hpp:74
  if (out_len) *out_len = n < k ? 0 : n - k + 1;     // core.hpp:58
  return MF_OK;
}

int mf_kernel_class(mf_dtype dtype, size_t k) { return class_for(dtype, k); }

mf_status mf_context_create(int device, mf_context** out) {
  if (!out) return MF_BAD_ARG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) { cudaGetLastError(); return MF_NO_DEVICE; }
  if (device < 0 || device >= count) return MF_BAD_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return MF_NO_DEVICE;
  mf_context* ctx = new mf_context();
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return MF_CUDA_ERROR;
  }
  *out = ctx;
  return MF_OK;
}

void mf_context_destroy(mf_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->io) cudaFree(ctx->io);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

mf_status mf_context_set_option(mf_context* ctx, mf_option opt, long value) {
  if (!ctx) return MF_BAD_ARG;
  if (opt == MF_OPT_FORCE_CLASS) {
    if (value < MF_CLASS_AUTO || value > MF_CLASS_LARGE) return MF_BAD_ARG;
    ctx->force_class = (int)value;
    return MF_OK;
  }
  return MF_BAD_ARG;
}

uint64_t mf_context_last_launches(const mf_context* ctx) { return ctx ? ctx->launches : 0; }

mf_status mf_median_filter_rows_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t rows,
                                       size_t n, size_t ld_x, size_t k, void* d_y, size_t ld_y,
                                       void* stream) {
  if (!ctx) return MF_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return run_rows(ctx, dtype, d_x, rows, n, ld_x, k, d_y, ld_y, pick(ctx, stream));
}

mf_status mf_median_filter_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t n, size_t k,
                                  void* d_y, void* stream) {
  size_t keep = 0;
  mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
  if (st != MF_OK) return st;
  return mf_median_filter_rows_device(ctx, dtype, d_x, 1, n, n, k, d_y, keep ? keep : 1, stream);
}

mf_status mf_median_filter_rows(mf_context* ctx, mf_dtype dtype, const void* x, size_t rows, size_t n,
                                size_t ld_x, size_t k, void* y, size_t ld_y) {
  if (!ctx) return MF_BAD_ARG;
  size_t keep = 0;
  mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
  if (st != MF_OK) return st;
  if (!dtype_ok(dtype)) return MF_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  ctx->launches = 0;
  if (keep == 0 || rows == 0) return MF_OK;
  if (!x || !y || ld_x < n || ld_y < keep) return MF_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  const size_t w = dtype_size(dtype);
  const size_t in_bytes = (rows * n * w + 255) / 256 * 256;
  const size_t out_bytes = rows * keep * w;
  st = grow(&ctx->io, &ctx->io_bytes, in_bytes + out_bytes);
  if (st != MF_OK) return st;
  char* d_x = static_cast<char*>(ctx->io);
  char* d_y = d_x + in_bytes;
  cudaStream_t s = ctx->stream;
  cudaError_t e = cudaMemcpy2DAsync(d_x, n * w, x, ld_x * w, n * w, rows, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return from_cuda(e);
  st = run_rows(ctx, dtype, d_x, rows, n, n, k, d_y, keep, s);
  if (st != MF_OK) return st;
  e = cudaMemcpy2DAsync(y, ld_y * w, d_y, keep * w, keep * w, rows, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return from_cuda(e);
  return from_cuda(cudaStreamSynchronize(s));
}

mf_status mf_median_filter(mf_context* ctx, mf_dtype dtype, const void* x, size_t n, size_t k, void* y,
                           size_t y_cap, size_t* y_len) {
  if (!ctx) return MF_BAD_ARG;
  size_t keep = 0;
  mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
  if (st != MF_OK) return st;
  if (y_len) *y_len = 0;
  if (keep > y_cap) return MF_BAD_ARG;
  st = mf_median_filter_rows(ctx, dtype, x, 1, n, n, k, y, keep ? keep : 1);
  if (st == MF_OK && y_len) *y_len = keep;
  return st;
}

mf_status mf_block_sort_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t n, size_t k,
                               uint32_t* d_perm, void* stream) {
  if (!ctx) return MF_BAD_ARG;
  size_t b = 0;
  mf_status st = mf_window_spec(n, k, nullptr, &b, nullptr);
  if (st != MF_OK) return st;
  if (!dtype_ok(dtype) || !d_x || !d_perm) return MF_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  ctx->launches = 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  mf::Geom g{};
  g.x = d_x; g.y = nullptr; g.n = n; g.ld_x = n; g.ld_y = 0;
  g.k = (uint32_t)k; g.h = (uint32_t)((k - 1) / 2);
  g.keep = n >= k ? n - k + 1 : 0; g.units = b; g.rows = 1;
  st = grow(&ctx->ws, &ctx->ws_bytes, mf::block_sort_workspace_bytes(dtype, g, b));
  if (st != MF_OK) return st;
  return from_cuda(mf::run_block_sort(dtype, g, b, ctx->ws, d_perm, pick(ctx, stream), &ctx->launches));
}

mf_status mf_generate_device(mf_context* ctx, int kind, uint64_t seed, uint64_t mod, uint64_t offset, size_t n,
                             void* d_out, void* stream) {
  if (!ctx || !d_out || kind < 0 || kind > 2 || (kind == 2 && mod == 0)) return MF_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  return from_cuda(mf::launch_generate(kind, seed, mod, offset, n, d_out, pick(ctx, stream)));
}

}  // extern "C"
