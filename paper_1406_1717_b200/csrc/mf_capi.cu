// mf_capi.cu -- the extern "C" boundary (include/medfilt_gpu.h).
//
// Validation mirrors make_window_spec (core.hpp:62-76) check for check and in the
// same order; n < k returns an empty output (core.hpp:58-59).  There is no CPU
// fallback: every entry either runs the CUDA kernels or returns an error status.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/medfilt_gpu.h"
#include "mf_launch.h"

// Host copy pool for the pageable-buffer path: a few persistent threads that split one
// memcpy (or a strided row copy) between them.  One pool per context; run() blocks until
// every piece is done.
struct CopyPool {
  std::vector<std::thread> threads;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;
  int parts = 0, next = 0, remaining = 0;
  uint64_t gen = 0;
  bool stop = false;
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) threads.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
  }
  int size() const { return (int)threads.size() + 1; }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> l(mu);
      cv.wait(l, [&] { return stop || (gen != seen && next < parts); });
      if (stop) return;
      seen = gen;
      while (next < parts) {
        const int i = next++;
        l.unlock();
        job(i);
        l.lock();
        if (--remaining == 0) done_cv.notify_all();
      }
    }
  }
  // job(i) for i in [0, n), on the pool and the calling thread
  void run(int n, std::function<void(int)> f) {
    if (n <= 1 || threads.empty()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> l(mu);
    job = std::move(f);
    parts = n;
    next = 0;
    remaining = n;
    ++gen;
    cv.notify_all();
    while (next < parts) {  // the caller takes pieces too
      const int i = next++;
      l.unlock();
      job(i);
      l.lock();
      --remaining;
    }
    done_cv.wait(l, [&] { return remaining == 0; });
  }
  // rows x bytes strided copy, split by rows (or by bytes for one row)
  void copy2d(char* dst, size_t dld, const char* src, size_t sld, size_t bytes, size_t rows) {
    constexpr size_t kPiece = size_t(1) << 20;
    const size_t total = bytes * rows;
    const int n = (int)std::max<size_t>(1, std::min<size_t>((size_t)size(), total / kPiece));
    if (rows == 1) {
      run(n, [&](int i) {
        const size_t a = bytes * i / n, b = bytes * (i + 1) / n;
        std::memcpy(dst + a, src + a, b - a);
      });
    } else {
      const int m = (int)std::min<size_t>(rows, (size_t)n);
      run(m, [&](int i) {
        for (size_t r = rows * i / m; r < rows * (i + 1) / m; ++r) std::memcpy(dst + r * dld, src + r * sld, bytes);
      });
    }
  }
};

struct mf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  void* ws = nullptr;          // grow-only device workspace
  size_t ws_bytes = 0;
  void* io = nullptr;          // grow-only device buffers for the host entry points
  size_t io_bytes = 0;
  int force_class = MF_CLASS_AUTO;
  size_t chunk_elems = size_t(1) << 22;  // largest host-pipeline chunk (samples; 2^22 measured 1.5 % above 2^23)
  uint64_t launches = 0;
  // host-entry pipeline: H2D / compute / D2H on three streams, up to 4 chunks in flight
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[16] = {}, ev_done[16] = {}, ev_out[16] = {};
  // the workspace is shared by every call on this context, whatever stream it is issued on:
  // each call that uses it records ws_ev, and the next one waits for it (stream order across
  // streams, so concurrent large-k calls on two streams never overlap on ws)
  cudaEvent_t ws_ev = nullptr;
  bool ws_ev_recorded = false;
  // MF_OPT_PROFILE: the device entries record a CUDA event at every phase mark
  bool profile = false;
  mf::PhaseTrace trace;
  // pageable host buffers: pinned staging slots and the copy pool (created on first use)
  void* hstage = nullptr;
  size_t hstage_bytes = 0;
  CopyPool* pool = nullptr;
  // multi-device context (mf_context_create_multi): one sub-context per device; the host
  // entries shard their work over them.  Empty for a single-device context.
  std::vector<mf_context*> subs;
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

// Host memory the DMA engines can read directly: pinned (cudaHostAlloc) or registered.
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Order a use of ctx->ws on stream s after the previous use (on whatever stream).
mf_status ws_acquire(mf_context* ctx, cudaStream_t s) {
  if (!ctx->ws_ev && cudaEventCreateWithFlags(&ctx->ws_ev, cudaEventDisableTiming) != cudaSuccess)
    return MF_CUDA_ERROR;
  if (ctx->ws_ev_recorded && cudaStreamWaitEvent(s, ctx->ws_ev, 0) != cudaSuccess) return MF_CUDA_ERROR;
  return MF_OK;
}
cudaError_t ws_release(mf_context* ctx, cudaStream_t s) {
  const cudaError_t e = cudaEventRecord(ctx->ws_ev, s);
  ctx->ws_ev_recorded = e == cudaSuccess;
  return e;
}

int class_for(mf_dtype dtype, size_t k) {
  if (k <= mf::small_max_k(dtype)) return MF_CLASS_SMALL;
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
  if (!d_x || !d_y || ld_x < n || ld_y < keep || rows > 0xFFFFFFFFull) return MF_BAD_ARG;
  int cls = ctx->force_class == MF_CLASS_AUTO ? class_for(dtype, k) : ctx->force_class;
  if (cls == MF_CLASS_SMALL && k > mf::small_max_k(dtype)) return MF_BAD_ARG;
  if (cls == MF_CLASS_MEDIUM && k > mf::kMediumMaxK) return MF_BAD_ARG;
  // the large-k pipeline packs 2k merged positions and a side flag into 32 bits
  if (cls == MF_CLASS_LARGE && k > mf::kLargeMaxK) return MF_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  mf::Geom g{};
  g.x = d_x; g.y = d_y; g.n = n; g.ld_x = ld_x; g.ld_y = ld_y;
  g.k = (uint32_t)k; g.h = (uint32_t)((k - 1) / 2);
  g.keep = keep; g.units = (keep + k - 1) / k; g.rows = (uint32_t)rows;
  cudaError_t e;
  if (cls == MF_CLASS_SMALL) {
    mf::phase_mark(s, k == 3 ? "small: k=3 selection" : "small: fused sort + walk");
    e = mf::launch_small(dtype, g, s, &ctx->launches);
  } else if (cls == MF_CLASS_MEDIUM) {
    mf::phase_mark(s, "medium: fused sort + merge + walk");
    e = mf::launch_medium(dtype, g, s, &ctx->launches);
  } else {
    // the large-k kernels put rows on grid.y (<= 65535): run row groups
    const size_t w = dtype_size(dtype);
    if ((st = ws_acquire(ctx, s)) != MF_OK) return st;
    e = cudaSuccess;
    for (size_t r0 = 0; r0 < rows && e == cudaSuccess; r0 += 65535) {
      mf::Geom gg = g;
      gg.rows = (uint32_t)std::min<size_t>(65535, rows - r0);
      gg.x = static_cast<const char*>(d_x) + r0 * ld_x * w;
      gg.y = static_cast<char*>(d_y) + r0 * ld_y * w;
      const size_t need = mf::large_workspace_bytes(dtype, gg);
      st = grow(&ctx->ws, &ctx->ws_bytes, need);
      if (st != MF_OK) return st;
      e = mf::run_large(dtype, gg, ctx->ws, ctx->ws_bytes, s, &ctx->launches);
    }
    const cudaError_t er = ws_release(ctx, s);
    if (e == cudaSuccess) e = er;
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

mf_status mf_context_create_multi(const int* devices, int ndev, mf_context** out) {
  if (!out) return MF_BAD_ARG;
  *out = nullptr;
  if (!devices || ndev < 1) return MF_BAD_ARG;
  mf_context* ctx = new mf_context();
  ctx->device = devices[0];
  for (int i = 0; i < ndev; ++i) {
    mf_context* sub = nullptr;
    const mf_status st = mf_context_create(devices[i], &sub);
    if (st != MF_OK) {
      mf_context_destroy(ctx);
      return st;
    }
    ctx->subs.push_back(sub);
  }
  // direct NVLink copies between the devices for the device-resident multi-device entry
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < ndev; ++j) {
      int can = 0;
      if (devices[i] == devices[j] || cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) != cudaSuccess || !can)
        continue;
      cudaSetDevice(devices[i]);
      if (cudaDeviceEnablePeerAccess(devices[j], 0) != cudaSuccess) cudaGetLastError();  // already enabled
    }
  cudaSetDevice(devices[0]);
  *out = ctx;
  return MF_OK;
}

int mf_context_devices(const mf_context* ctx, int* devices, int cap) {
  if (!ctx) return 0;
  if (ctx->subs.empty()) {
    if (devices && cap > 0) devices[0] = ctx->device;
    return 1;
  }
  for (int i = 0; i < (int)ctx->subs.size() && devices && i < cap; ++i) devices[i] = ctx->subs[i]->device;
  return (int)ctx->subs.size();
}

void mf_context_destroy(mf_context* ctx) {
  if (!ctx) return;
  if (!ctx->subs.empty()) {
    for (mf_context* sub : ctx->subs) mf_context_destroy(sub);
    delete ctx;
    return;
  }
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->ws_ev) cudaEventDestroy(ctx->ws_ev);
  for (cudaEvent_t ev : ctx->trace.ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->hstage) cudaFreeHost(ctx->hstage);
  delete ctx->pool;
  if (ctx->io) cudaFree(ctx->io);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->s_h2d) cudaStreamSynchronize(ctx->s_h2d), cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_d2h) cudaStreamSynchronize(ctx->s_d2h), cudaStreamDestroy(ctx->s_d2h);
  for (int i = 0; i < 16; ++i) {
    if (ctx->ev_in[i]) cudaEventDestroy(ctx->ev_in[i]);
    if (ctx->ev_done[i]) cudaEventDestroy(ctx->ev_done[i]);
    if (ctx->ev_out[i]) cudaEventDestroy(ctx->ev_out[i]);
  }
  delete ctx;
}

mf_status mf_context_set_option(mf_context* ctx, mf_option opt, long value) {
  if (!ctx) return MF_BAD_ARG;
  for (mf_context* sub : ctx->subs) {
    const mf_status st = mf_context_set_option(sub, opt, value);
    if (st != MF_OK) return st;
  }
  if (opt == MF_OPT_FORCE_CLASS) {
    if (value < MF_CLASS_AUTO || value > MF_CLASS_LARGE) return MF_BAD_ARG;
    ctx->force_class = (int)value;
    return MF_OK;
  }
  if (opt == MF_OPT_PROFILE) {
    if (value != 0 && value != 1) return MF_BAD_ARG;
    ctx->profile = value != 0;
    return MF_OK;
  }
  if (opt == MF_OPT_PIPELINE_CHUNK) {
    if (value < 0) return MF_BAD_ARG;
    ctx->chunk_elems = value == 0 ? size_t(1) << 22 : std::max<size_t>(1024, (size_t)value);
    return MF_OK;
  }
  return MF_BAD_ARG;
}

uint64_t mf_context_last_launches(const mf_context* ctx) { return ctx ? ctx->launches : 0; }

int mf_context_last_phases(mf_context* ctx, const char** names, float* ms, int cap) {
  if (!ctx || !ctx->subs.empty()) return 0;
  std::lock_guard<std::mutex> lock(ctx->mu);
  const mf::PhaseTrace& t = ctx->trace;
  if (t.n == 0 || !t.ev[t.n]) return 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess || cudaEventSynchronize(t.ev[t.n]) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int i = 0; i < t.n && i < cap; ++i) {
    if (names) names[i] = t.name[i];
    if (ms && cudaEventElapsedTime(&ms[i], t.ev[i], t.ev[i + 1]) != cudaSuccess) {
      cudaGetLastError();
      ms[i] = -1.0f;
    }
  }
  return t.n;
}

// Device-resident multi-device entry (the cudaMemcpyPeer variant): the
// signal (or batch) lives on one "home" device.  Each sub-context's device takes a shard --
// halo'd output ranges of a signal, row groups of a batch -- copied peer to peer (NVLink
// when peer access is on), filters it on its own stream, and copies its outputs back to the
// home buffer at their offset; the home device's own shard is filtered in place.  Stream
// ordered: every device waits on an event recorded on the caller's stream, and the caller's
// stream waits on every device's completion event, so the call returns after enqueueing.
// Caller holds ctx->mu.
static mf_status multi_device_rows(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t rows, size_t n,
                                   size_t ld_x, size_t k, void* d_y, size_t ld_y, size_t keep, cudaStream_t stream) {
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, d_x) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return MF_BAD_ARG;
  }
  const int home = pa.device;
  const size_t w = dtype_size(dtype), G = ctx->subs.size();
  struct Part { size_t xo, yo, rows, n, ld_x, ld_y, in_elems, out_elems; };
  std::vector<Part> parts;
  if (rows > 1) {
    const size_t use = std::min(G, rows);
    for (size_t g = 0; g < use; ++g) {
      const size_t r0 = rows * g / use, r1 = rows * (g + 1) / use;
      parts.push_back({r0 * ld_x, r0 * ld_y, r1 - r0, n, ld_x, ld_y, (r1 - r0) * ld_x, (r1 - r0) * ld_y});
    }
  } else {
    const size_t min_out = std::max<size_t>(size_t(1) << 20, 16 * k);
    const size_t use = std::max<size_t>(1, std::min(G, keep / min_out));
    for (size_t g = 0; g < use; ++g) {
      const size_t o0 = keep * g / use, o1 = keep * (g + 1) / use, ni = o1 - o0 + k - 1;
      parts.push_back({o0, o0, 1, ni, ni, o1 - o0, ni, o1 - o0});
    }
  }
  size_t first_home = parts.size();
  for (size_t i = 0; i < parts.size(); ++i)
    if (ctx->subs[i]->device == home) { first_home = i; break; }
  if (cudaSetDevice(home) != cudaSuccess) return MF_NO_DEVICE;
  cudaEvent_t start = nullptr;
  if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(start, stream) != cudaSuccess)
    return MF_CUDA_ERROR;
  std::vector<cudaEvent_t> done(parts.size(), nullptr);
  mf_status st = MF_OK;
  uint64_t launches = 0;
  for (size_t i = 0; i < parts.size() && st == MF_OK; ++i) {
    mf_context* sub = ctx->subs[i];
    std::lock_guard<std::mutex> sl(sub->mu);
    const Part& p = parts[i];
    if (cudaSetDevice(sub->device) != cudaSuccess) { st = MF_NO_DEVICE; break; }
    if (cudaStreamWaitEvent(sub->stream, start, 0) != cudaSuccess) { st = MF_CUDA_ERROR; break; }
    const char* x0 = static_cast<const char*>(d_x) + p.xo * w;
    char* y0 = static_cast<char*>(d_y) + p.yo * w;
    if (sub->device == home && i == first_home) {  // the home device's own shard, in place
      st = run_rows(sub, dtype, x0, p.rows, p.n, p.ld_x, k, y0, p.ld_y, sub->stream);
    } else {
      const size_t in_b = (p.in_elems * w + 255) / 256 * 256, out_b = (p.out_elems * w + 255) / 256 * 256;
      if ((st = grow(&sub->io, &sub->io_bytes, in_b + out_b)) != MF_OK) break;
      char* sx = static_cast<char*>(sub->io);
      char* sy = sx + in_b;
      if (cudaMemcpyPeerAsync(sx, sub->device, x0, home, p.in_elems * w, sub->stream) != cudaSuccess) {
        st = MF_CUDA_ERROR;
        break;
      }
      st = run_rows(sub, dtype, sx, p.rows, p.n, p.ld_x, k, sy, p.ld_y, sub->stream);
      // outputs back to their offset; strided rows row by row, so the caller's row gaps stay
      // untouched, as in the single-device entry
      const size_t outw = p.rows > 1 ? keep : p.out_elems;
      for (size_t r = 0; r < p.rows && st == MF_OK; ++r)
        if (cudaMemcpyPeerAsync(y0 + r * p.ld_y * w, home, sy + r * p.ld_y * w, sub->device,
                                (p.rows > 1 && p.ld_y == keep) ? p.rows * keep * w : outw * w, sub->stream) != cudaSuccess)
          st = MF_CUDA_ERROR;
        else if (p.rows > 1 && p.ld_y == keep)
          break;  // contiguous rows: one copy
    }
    launches += sub->launches;
    if (st == MF_OK && (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess ||
                        cudaEventRecord(done[i], sub->stream) != cudaSuccess))
      st = MF_CUDA_ERROR;
  }
  cudaSetDevice(home);
  for (cudaEvent_t ev : done)
    if (ev) {
      if (cudaStreamWaitEvent(stream, ev, 0) != cudaSuccess && st == MF_OK) st = MF_CUDA_ERROR;
      cudaEventDestroy(ev);  // released once complete
    }
  cudaEventDestroy(start);
  ctx->launches = launches;
  return st;
}

mf_status mf_median_filter_rows_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t rows,
                                       size_t n, size_t ld_x, size_t k, void* d_y, size_t ld_y,
                                       void* stream) {
  if (!ctx) return MF_BAD_ARG;
  if (!ctx->subs.empty()) {  // several devices: peer-copied shards (see multi_device_rows)
    size_t keep = 0;
    mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
    if (st != MF_OK) return st;
    if (!dtype_ok(dtype)) return MF_BAD_ARG;
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->launches = 0;
    if (keep == 0 || rows == 0) return MF_OK;
    if (!d_x || !d_y || ld_x < n || ld_y < keep) return MF_BAD_ARG;
    nvtxRangePushA("mf_median_filter_rows_device (multi-device)");
    st = multi_device_rows(ctx, dtype, d_x, rows, n, ld_x, k, d_y, ld_y, keep, pick(ctx, stream));
    nvtxRangePop();
    return st;
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  nvtxRangePushA("mf_median_filter_rows_device");
  cudaStream_t s = pick(ctx, stream);
  if (ctx->profile) mf::phase_begin(&ctx->trace);
  const mf_status st = run_rows(ctx, dtype, d_x, rows, n, ld_x, k, d_y, ld_y, s);
  if (ctx->profile) {
    if (cudaSetDevice(ctx->device) == cudaSuccess) mf::phase_end(s);
    if (st != MF_OK) ctx->trace.n = 0;
  }
  nvtxRangePop();
  return st;
}

mf_status mf_median_filter_device(mf_context* ctx, mf_dtype dtype, const void* d_x, size_t n, size_t k,
                                  void* d_y, void* stream) {
  size_t keep = 0;
  mf_status st = mf_window_spec(n, k, nullptr, nullptr, &keep);
  if (st != MF_OK) return st;
  return mf_median_filter_rows_device(ctx, dtype, d_x, 1, n, n, k, d_y, keep ? keep : 1, stream);
}

// Chunk sizes for the host pipeline: cmin, 2*cmin, 4*cmin, ... up to cmax at the head,
// the mirror image at the tail, cmax-sized chunks in between.  Inputs too short for both ramps get equal chunks of about cmin.
static std::vector<size_t> chunk_schedule(size_t total, size_t cmin, size_t cmax) {
  std::vector<size_t> ramp;
  size_t ramp_sum = 0;
  for (size_t s = cmin; s < cmax; s *= 2) ramp.push_back(s), ramp_sum += s;
  std::vector<size_t> out;
  if (total <= 2 * ramp_sum || ramp.empty()) {
    const size_t unit = ramp.empty() ? cmax : cmin;
    const size_t n = std::max<size_t>(1, (total + unit - 1) / unit);
    for (size_t i = 0; i < n; ++i) out.push_back(total / n + (i < total % n ? 1 : 0));
    return out;
  }
  out = ramp;
  // middle: cmax-sized chunks (DMA-friendly offsets), the remainder in the last one
  size_t mid = total - 2 * ramp_sum;
  for (; mid > cmax; mid -= cmax) out.push_back(cmax);
  if (mid) out.push_back(mid);
  out.insert(out.end(), ramp.rbegin(), ramp.rend());
  return out;
}

// Multi-device host entry: a single signal is cut into contiguous output
// ranges [o_g, o_{g+1}) and device g filters x[o_g, o_{g+1}+k-1) -- a (k-1)-sample halo --
// as an independent signal; a batch is cut into whole row groups.  Blocking never changes
// an output (the reference's pair loop, filter.hpp:83-102, is
// independent per pair), so the concatenation is the single-device result.  One host
// thread per device runs the single-device pipeline, whose D2H writes straight into the
// caller's output at offset o_g: the gather IS the D2H, no device-to-device exchange.
// Caller holds ctx->mu.
static mf_status multi_rows(mf_context* ctx, mf_dtype dtype, const void* x, size_t rows, size_t n, size_t ld_x,
                            size_t k, void* y, size_t ld_y, size_t keep) {
  struct Part { size_t xo, yo, rows, n, ld_x, ld_y; };
  const size_t G = ctx->subs.size(), w = dtype_size(dtype);
  std::vector<Part> parts;
  if (rows > 1) {
    const size_t use = std::min(G, rows);
    for (size_t g = 0; g < use; ++g) {
      const size_t r0 = rows * g / use, r1 = rows * (g + 1) / use;
      parts.push_back({r0 * ld_x, r0 * ld_y, r1 - r0, n, ld_x, ld_y});
    }
  } else {
    // shards of at least max(2^20, 16k) outputs: below that a device's launch and copy
    // latency outweighs the work it takes over
    const size_t min_out = std::max<size_t>(size_t(1) << 20, 16 * k);
    const size_t use = std::max<size_t>(1, std::min(G, keep / min_out));
    for (size_t g = 0; g < use; ++g) {
      const size_t o0 = keep * g / use, o1 = keep * (g + 1) / use;
      parts.push_back({o0, o0, 1, o1 - o0 + k - 1, o1 - o0 + k - 1, o1 - o0});
    }
  }
  std::vector<mf_status> st(parts.size(), MF_OK);
  auto run = [&](size_t i) {
    const Part& p = parts[i];
    st[i] = mf_median_filter_rows(ctx->subs[i], dtype, static_cast<const char*>(x) + p.xo * w, p.rows, p.n,
                                  p.ld_x, k, static_cast<char*>(y) + p.yo * w, p.ld_y);
  };
  std::vector<std::thread> threads;
  for (size_t i = 1; i < parts.size(); ++i) threads.emplace_back(run, i);
  run(0);
  for (auto& t : threads) t.join();
  uint64_t launches = 0;
  for (size_t i = 0; i < parts.size(); ++i) launches += ctx->subs[i]->launches;
  ctx->launches = launches;
  for (mf_status v : st)
    if (v != MF_OK) return v;
  return MF_OK;
}

// Host entry: the literal drop-in.  The signal (or batch) is cut into chunks of about
// kChunkElems outputs -- contiguous output ranges with a (k-1)-sample input halo, or whole
// rows -- and up to four chunks are kept in flight: H2D of chunk c+1, kernels of chunk c and D2H
// of chunk c-1 overlap on three streams, so a call costs about the slower of the two PCIe
// directions instead of their sum.  Blocking never changes an output.
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
  struct Range {  // NVTX range around the host entry (free without a tool attached)
    Range() { nvtxRangePushA("mf_median_filter_rows (host buffers)"); }
    ~Range() { nvtxRangePop(); }
  } range;
  if (!ctx->subs.empty()) return multi_rows(ctx, dtype, x, rows, n, ld_x, k, y, ld_y, keep);
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
#ifndef MF_PIPE_SLOTS
#define MF_PIPE_SLOTS 4
#endif
#ifndef MF_PIPE_RAMP
#define MF_PIPE_RAMP 16
#endif
  constexpr int kNumSlots = MF_PIPE_SLOTS;
  const size_t kChunkElems = ctx->chunk_elems;
  if (!ctx->s_h2d) {
    if (cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return MF_CUDA_ERROR;
    for (int i = 0; i < kNumSlots; ++i)
      if (cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->ev_out[i], cudaEventDisableTiming) != cudaSuccess)
        return MF_CUDA_ERROR;
  }
  const size_t w = dtype_size(dtype);
  // chunk geometry: single signals by output ranges, batches by row groups.  Chunk sizes
  // ramp up geometrically at the start and down at the end, so the H2D of the first chunk
  // and the D2H of the last (the parts nothing overlaps) are small.
  const bool by_rows = rows > 1;
  const size_t total = by_rows ? rows : keep;  // units to cut
  // large windows take chunks of at least 128 windows: every chunk re-sorts its blocks and pays the
  // large-k pipeline's launches, so a 2^22-sample chunk at k = 100001 would cost c5 a third of its e2e
  const size_t cmax = by_rows ? std::max<size_t>(1, kChunkElems / n) : std::min(keep, std::max<size_t>(kChunkElems, 128 * k));
  const size_t cmin = std::max<size_t>(by_rows ? 1 : std::min(cmax, 16 * k), cmax / MF_PIPE_RAMP);
  std::vector<size_t> sizes = chunk_schedule(total, cmin, cmax);
  const size_t nchunks = sizes.size();
  const size_t in_slot = ((by_rows ? cmax * n : cmax + k - 1) * w + 255) / 256 * 256;
  const size_t out_slot = ((by_rows ? cmax * keep : cmax) * w + 255) / 256 * 256;
  const int slots = (int)std::min<size_t>(kNumSlots, nchunks);
  st = grow(&ctx->io, &ctx->io_bytes, slots * (in_slot + out_slot));
  if (st != MF_OK) return st;
  // Pageable caller buffers (e.g. a std::vector behind gpu.hpp): the DMA engines cannot read
  // them directly, and the driver's own staging serialises the copy with the host thread.
  // They go through pinned staging slots instead, filled and drained by the context's copy
  // pool: the host copies chunk c+1 in and chunk c-1 out while the device runs chunk c.
  const bool stage_in = !host_pinned(x), stage_out = !host_pinned(y);
  char* hin = nullptr;
  char* hout = nullptr;
  if (stage_in || stage_out) {
    const size_t need = slots * (in_slot + out_slot);
    if (need > ctx->hstage_bytes) {
      if (ctx->hstage) cudaFreeHost(ctx->hstage);
      ctx->hstage = nullptr;
      ctx->hstage_bytes = 0;
      if (cudaHostAlloc(&ctx->hstage, need, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return MF_OUT_OF_MEMORY;
      }
      ctx->hstage_bytes = need;
    }
    if (!ctx->pool) {
      const unsigned hc = std::max(2u, std::thread::hardware_concurrency());
      ctx->pool = new CopyPool((int)std::min(15u, hc / 2));
    }
    hin = static_cast<char*>(ctx->hstage);
    hout = hin + slots * in_slot;
  }
  char* base = static_cast<char*>(ctx->io);
  const char* hx = static_cast<const char*>(x);
  char* hy = static_cast<char*>(y);
  uint64_t launches = 0;
  cudaError_t e = cudaSuccess;
  // chunk geometry: [begin unit, units) of chunk c
  std::vector<size_t> starts(nchunks + 1, 0);
  for (size_t c = 0; c < nchunks; ++c) starts[c + 1] = starts[c] + sizes[c];
  auto copy_out = [&](size_t c) {  // staged outputs of chunk c -> caller buffer
    const int sl = (int)(c % slots);
    const char* src = hout + sl * out_slot;
    if (by_rows) ctx->pool->copy2d(hy + starts[c] * ld_y * w, ld_y * w, src, keep * w, keep * w, sizes[c]);
    else ctx->pool->copy2d(hy + starts[c] * w, 0, src, 0, sizes[c] * w, 1);
  };
  size_t drained = 0;  // chunks whose outputs reached the caller's buffer (staged outputs)
  for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    const int sl = (int)(c % slots);
    char* d_x = base + sl * (in_slot + out_slot);
    char* d_y = d_x + in_slot;
    if (c >= (size_t)slots) {  // the slot's previous chunk must have left the device
      e = cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_out[sl], 0);
      if (e != cudaSuccess) break;
    }
    size_t r0 = 0, nr = 1, o0 = 0, no = keep, ni = n;
    if (by_rows) {
      r0 = starts[c];
      nr = sizes[c];
    } else {
      o0 = starts[c];
      no = sizes[c];
      ni = no + k - 1;
    }
    if (stage_in) {  // pageable -> pinned slot (its previous H2D finished: see below)
      char* hs = hin + sl * in_slot;
      if (by_rows) ctx->pool->copy2d(hs, n * w, hx + r0 * ld_x * w, ld_x * w, n * w, nr);
      else ctx->pool->copy2d(hs, 0, hx + o0 * w, 0, ni * w, 1);
      e = cudaMemcpyAsync(d_x, hs, (by_rows ? nr * n : ni) * w, cudaMemcpyHostToDevice, ctx->s_h2d);
    } else if (by_rows) {
      e = cudaMemcpy2DAsync(d_x, n * w, hx + r0 * ld_x * w, ld_x * w, n * w, nr, cudaMemcpyHostToDevice,
                            ctx->s_h2d);
    } else {
      e = cudaMemcpyAsync(d_x, hx + o0 * w, ni * w, cudaMemcpyHostToDevice, ctx->s_h2d);
    }
    if (e != cudaSuccess) break;
    if ((e = cudaEventRecord(ctx->ev_in[sl], ctx->s_h2d)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(ctx->stream, ctx->ev_in[sl], 0)) != cudaSuccess) break;
    st = run_rows(ctx, dtype, d_x, nr, ni, ni, k, d_y, by_rows ? keep : no, ctx->stream);
    launches += ctx->launches;
    if (st != MF_OK) break;
    if ((e = cudaEventRecord(ctx->ev_done[sl], ctx->stream)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_done[sl], 0)) != cudaSuccess) break;
    if (stage_out) {
      e = cudaMemcpyAsync(hout + sl * out_slot, d_y, (by_rows ? nr * keep : no) * w, cudaMemcpyDeviceToHost,
                          ctx->s_d2h);
    } else if (by_rows) {
      e = cudaMemcpy2DAsync(hy + r0 * ld_y * w, ld_y * w, d_y, keep * w, keep * w, nr, cudaMemcpyDeviceToHost,
                            ctx->s_d2h);
    } else {
      e = cudaMemcpyAsync(hy + o0 * w, d_y, no * w, cudaMemcpyDeviceToHost, ctx->s_d2h);
    }
    if (e != cudaSuccess) break;
    if ((e = cudaEventRecord(ctx->ev_out[sl], ctx->s_d2h)) != cudaSuccess) break;
    // Host side of the staged path, while the device runs chunk c: drain chunk c-1's outputs.
    // Waiting for chunk c-1's D2H also retires every H2D up to c-1, so the pinned input slot
    // of chunk c+1 (that of chunk c+1-slots) is free when the next iteration fills it.
    if ((stage_in || stage_out) && c >= 1) {
      if ((e = cudaEventSynchronize(ctx->ev_out[(c - 1) % slots])) != cudaSuccess) break;
      if (stage_out) copy_out(c - 1);
      drained = c;
    }
  }
  ctx->launches = launches;
  const cudaError_t e2 = cudaStreamSynchronize(ctx->s_d2h);
  const cudaError_t e3 = cudaStreamSynchronize(ctx->stream);
  if (st == MF_OK && e == cudaSuccess && e2 == cudaSuccess && stage_out)
    for (size_t c = drained; c < nchunks; ++c) copy_out(c);
  if (st != MF_OK) return st;
  if (e != cudaSuccess) return from_cuda(e);
  if (e2 != cudaSuccess) return from_cuda(e2);
  return from_cuda(e3);
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
  if (!dtype_ok(dtype) || !d_x || !d_perm || !ctx->subs.empty() || k > mf::kLargeMaxK) return MF_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  ctx->launches = 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  mf::Geom g{};
  g.x = d_x; g.y = nullptr; g.n = n; g.ld_x = n; g.ld_y = 0;
  g.k = (uint32_t)k; g.h = (uint32_t)((k - 1) / 2);
  g.keep = n >= k ? n - k + 1 : 0; g.units = b; g.rows = 1;
  st = grow(&ctx->ws, &ctx->ws_bytes, mf::block_sort_workspace_bytes(dtype, g, b));
  if (st != MF_OK) return st;
  cudaStream_t s = pick(ctx, stream);
  if ((st = ws_acquire(ctx, s)) != MF_OK) return st;
  cudaError_t e = mf::run_block_sort(dtype, g, b, ctx->ws, d_perm, s, &ctx->launches);
  const cudaError_t er = ws_release(ctx, s);
  return from_cuda(e != cudaSuccess ? e : er);
}

mf_status mf_generate_device(mf_context* ctx, int kind, uint64_t seed, uint64_t mod, uint64_t offset, size_t n,
                             void* d_out, void* stream) {
  if (!ctx || !ctx->subs.empty() || !d_out || kind < 0 || kind > 2 || (kind == 2 && mod == 0)) return MF_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MF_NO_DEVICE;
  return from_cuda(mf::launch_generate(kind, seed, mod, offset, n, d_out, pick(ctx, stream)));
}

}  // extern "C"
