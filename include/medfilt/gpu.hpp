// medfilt/gpu.hpp -- C++ drop-in over the C ABI (include/medfilt_gpu.h).
//
//   template <std::signed_integral T>
//   std::vector<T> medfilt::gpu::median_filter(std::span<const T> x, std::size_t k);
//
// has exactly the reference's FilterFn<T> shape (baselines.hpp:29-30), so it registers
// in the reference's dispatch tables (bench.hpp:51-59 lookup_filter, verify.hpp:60-70
// filter_table, medfilt_cli.cpp:45-50 run_algorithm) under the name "gpu".  Errors are
// rethrown as std::invalid_argument with the reference's texts (core.hpp:63-69); CUDA
// failures throw std::runtime_error.  Float/double overloads order by IEEE totalOrder.
#pragma once

#include <concepts>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../medfilt_gpu.h"

namespace medfilt::gpu {

namespace detail {

inline void check(mf_status st) {
  if (st == MF_OK) return;
  if (st == MF_EMPTY_INPUT || st == MF_K_ZERO || st == MF_K_EVEN || st == MF_K_TOO_LARGE)
    throw std::invalid_argument(mf_error_message(st));
  throw std::runtime_error(std::string(mf_status_string(st)) + ": " + mf_error_message(st));
}

// Devices the calling thread's context spans: set_devices(), else the environment
// variable MEDFILT_GPU_DEVICES ("0,1,2,3" or "all"), else device 0.
inline std::vector<int> env_devices() {
  std::vector<int> d;
  const char* e = std::getenv("MEDFILT_GPU_DEVICES");
  if (!e || !*e) return {0};
  if (std::string(e) == "all") {
    mf_context* probe = nullptr;
    for (int i = 0; mf_context_create(i, &probe) == MF_OK; ++i) {
      mf_context_destroy(probe);
      d.push_back(i);
    }
    return d.empty() ? std::vector<int>{0} : d;
  }
  for (const char* p = e; *p;) {
    char* end = nullptr;
    const long v = std::strtol(p, &end, 10);
    if (end == p) break;
    d.push_back((int)v);
    p = *end == ',' ? end + 1 : end;
  }
  return d.empty() ? std::vector<int>{0} : d;
}

// One context per host thread (contexts are not shared across threads).
struct Holder {
  mf_context* ctx = nullptr;
  std::vector<int> devices = env_devices();
  ~Holder() { mf_context_destroy(ctx); }
};
inline Holder& holder() {
  thread_local Holder h;
  return h;
}

inline mf_context* context() {
  Holder& h = holder();
  if (!h.ctx) {
    if (h.devices.size() == 1) check(mf_context_create(h.devices[0], &h.ctx));
    else check(mf_context_create_multi(h.devices.data(), (int)h.devices.size(), &h.ctx));
  }
  return h.ctx;
}

template <typename T> constexpr mf_dtype dtype_of();
template <> constexpr mf_dtype dtype_of<std::int32_t>() { return MF_I32; }
template <> constexpr mf_dtype dtype_of<std::int64_t>() { return MF_I64; }
template <> constexpr mf_dtype dtype_of<float>() { return MF_F32; }
template <> constexpr mf_dtype dtype_of<double>() { return MF_F64; }

template <typename T>
std::vector<T> run(std::span<const T> x, std::size_t k) {
  std::size_t keep = 0;
  check(mf_window_spec(x.size(), k, nullptr, nullptr, &keep));  // core.hpp:62-76
  std::vector<T> y(keep);
  if (keep == 0) return y;                                        // n < k: empty
  std::size_t len = 0;
  check(mf_median_filter(context(), dtype_of<T>(), x.data(), x.size(), k, y.data(), y.size(), &len));
  y.resize(len);
  return y;
}

}  // namespace detail

/// Devices the calling thread's median_filter calls use (SURVEY.md §8(b) "Multi-GPU entry:
/// a device list").  With more than one device every call shards its signal (contiguous
/// output ranges with a (k-1)-sample halo) or its rows across them; outputs are unchanged.
inline void set_devices(std::vector<int> devices) {
  if (devices.empty()) throw std::invalid_argument("device list must not be empty");
  detail::Holder& h = detail::holder();
  mf_context_destroy(h.ctx);
  h.ctx = nullptr;
  h.devices = std::move(devices);
}

/// median_filter<T> (filter.hpp:149-155) on the B200.
template <std::signed_integral T>
  requires(sizeof(T) == 4 || sizeof(T) == 8)
std::vector<T> median_filter(std::span<const T> x, std::size_t k) {
  using W = std::conditional_t<sizeof(T) == 4, std::int32_t, std::int64_t>;
  if constexpr (std::same_as<T, W>) {
    return detail::run<T>(x, k);
  } else {  // e.g. long vs long long of the same width
    auto y = detail::run<W>(std::span<const W>(reinterpret_cast<const W*>(x.data()), x.size()), k);
    return std::vector<T>(y.begin(), y.end());
  }
}

/// Float/double extension (the reference takes signed integers only).
inline std::vector<float> median_filter(std::span<const float> x, std::size_t k) {
  return detail::run<float>(x, k);
}
inline std::vector<double> median_filter(std::span<const double> x, std::size_t k) {
  return detail::run<double>(x, k);
}

/// sort_via_median_filter (filter.hpp:177-205) with the filter on the GPU: each block of
/// h+1 samples is surrounded by h copies of the type's minimum and h of its maximum, one
/// median filter with k = 2h+1 runs over the whole gadget, and each block's sorted image
/// is read out of the output.
template <std::signed_integral T>
std::vector<std::vector<T>> sort_via_median_filter(std::span<const std::vector<T>> blocks, std::size_t h) {
  for (const auto& block : blocks)
    if (block.size() != h + 1) throw std::invalid_argument("each block must hold h+1 samples");
  if (blocks.empty()) return {};
  const std::size_t k = 2 * h + 1, unit = 3 * h + 1;
  std::vector<T> gadget;
  gadget.reserve(blocks.size() * unit);
  for (const auto& block : blocks) {
    gadget.insert(gadget.end(), h, std::numeric_limits<T>::min());
    gadget.insert(gadget.end(), block.begin(), block.end());
    gadget.insert(gadget.end(), h, std::numeric_limits<T>::max());
  }
  const std::vector<T> med = median_filter<T>(std::span<const T>(gadget), k);
  std::vector<std::vector<T>> sorted(blocks.size());
  for (std::size_t j = 0; j < blocks.size(); ++j)
    sorted[j].assign(med.begin() + j * unit, med.begin() + j * unit + h + 1);
  return sorted;
}

}  // namespace medfilt::gpu
